# Config-4 kernels at B = 512 (tools/sweep_hp.py: the first march is 512 instances)
set -x
python tools/sweep_hp.py 512 1 0 > gpurun_out/plain_sweep.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hyperpair_engine|gn_partial|positions_clusters_mma" -s 3 -c 3 -o gpurun_out/r02_c4k python tools/sweep_hp.py 512 1 0 > gpurun_out/ncu_c4k.log 2>&1
ls -la gpurun_out/r02_c4k*
