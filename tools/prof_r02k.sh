# persistent FOM kernel (config 1) under ncu: one full capture of the whole-trajectory launch
set -x
python tools/fom_time_probe.py > gpurun_out/plain_fom.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fom_persistent -s 1 -c 1 -o gpurun_out/r02_fom_persistent python tools/fom_time_probe.py > gpurun_out/ncu_fom.log 2>&1
ls -la gpurun_out/r02_fom_persistent*
