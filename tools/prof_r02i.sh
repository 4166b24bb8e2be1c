# gn_partial_kernel<16> at B = 512 with source-level counters
set -x
python tools/sweep_hp.py 512 1 0 > gpurun_out/plain_gn.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gn_partial" -s 2 -c 1 -o gpurun_out/r02_gn_src python tools/sweep_hp.py 512 1 0 > gpurun_out/ncu_gn.log 2>&1
ls -la gpurun_out/r02_gn_src*
