set -x
python tools/bench_ptrom.py --inst 512 --steps 1 --batch 512 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hyperpair|positions_clusters_mma|gn_partial" -s 30 -c 3 -o gpurun_out/r02_c4 python tools/bench_ptrom.py --inst 512 --steps 1 --batch 512 > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out
