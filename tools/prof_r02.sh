set -x
python tools/prof_live.py config4 512 2 > gpurun_out/live_c4.txt 2>&1
python tools/prof_live.py config3 > gpurun_out/live_c3.txt 2>&1
python tools/prof_live.py config1 > gpurun_out/live_c1.txt 2>&1
python tools/bench_ptrom.py --inst 512 --steps 1 --batch 512 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hyperpair -s 1 -c 1 -o gpurun_out/r02_hyperpair python tools/bench_ptrom.py --inst 512 --steps 1 --batch 512 > gpurun_out/ncu_c4.log 2>&1
python tools/bench_tree.py 1048576 1 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"bh_eval|morton_subtree|morton_levels|morton_large" -s 4 -c 4 -o gpurun_out/r02_tree python tools/bench_tree.py 1048576 1 > gpurun_out/ncu_c3.log 2>&1
ls -la gpurun_out/
