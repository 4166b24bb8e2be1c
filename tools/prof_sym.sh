python bench.py --workload config2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:allpairs_sym -s 3 -c 1 -o gpurun_out/r02_sym python bench.py --workload config2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sym.log 2>&1
