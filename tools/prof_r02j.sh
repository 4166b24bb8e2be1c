# new batch-engine test + the transposed cluster-position kernel under ncu (B = 512)
set -x

python tools/sweep_hp.py 512 1 0 > gpurun_out/plain_pos.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"positions_clusters_mma" -s 2 -c 1 -o gpurun_out/r02_pos2 python tools/sweep_hp.py 512 1 0 > gpurun_out/ncu_pos.log 2>&1
ls -la gpurun_out/r02_pos2*
