# round-2 evidence: hyperpair (current code) full capture, the config-5
# all-pairs launch's DRAM traffic, and the default bench's launch list
set -x
python tools/bench_ptrom.py --inst 512 --steps 1 --batch 512 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hyperpair -s 30 -c 1 -o gpurun_out/r02_hyperpair_cur python tools/bench_ptrom.py --inst 512 --steps 1 --batch 512 > gpurun_out/ncu_c4.log 2>&1
python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:allpairs_f64 -c 1 --csv --log-file gpurun_out/r02_allpairs_c5_metrics.csv python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_default.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out | tail -8
