# hyperpair_engine_kernel at B = 512 (config 4): launch list and one full capture
set -x
python tools/sweep_hp.py 512 1 0 > gpurun_out/plain_hp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hyperpair_engine" -s 2 -c 1 -o gpurun_out/r02_hp_engine512 python tools/sweep_hp.py 512 1 0 > gpurun_out/ncu_hp.log 2>&1
ls -la gpurun_out/r02_hp_engine512*
