# Round-2 (session 2) captures: the engine hyperpair kernel (config 4) and the
# BH far field with source-level counters (config 3). Each ncu pass only
# after its plain command exited 0.
set -x
timeout 900 python -m pytest tests/test_rom_gpu.py -m gpu -x -q -k "variants or batch_affine or ptrom_simulate_parity" > gpurun_out/t_hpvar.log 2>&1
python tools/bench_ptrom.py --inst 512 --steps 1 --batch 512 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hyperpair_engine -s 1 -c 1 -o gpurun_out/r02_hp_engine python tools/bench_ptrom.py --inst 512 --steps 1 --batch 512 > gpurun_out/ncu_c4.log 2>&1
python tools/bench_tree.py 1048576 1 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"bh_eval" -s 1 -c 1 -o gpurun_out/r02_bh_src python tools/bench_tree.py 1048576 1 > gpurun_out/ncu_c3.log 2>&1
ls -la gpurun_out/
