for s in 2048 1024 512 256 128; do
  echo "seq_max=$s"; PTROM_TREE_SEQ_MAX=$s python tools/bench_tree.py 1048576 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(d[k],4) if isinstance(d[k],float) else d[k] for k in ('total_ms','build_ms','eval_ms','resolved_targets','interactions')})"
done
PTROM_TREE_SEQ_MAX=256 python -m pytest tests/test_tree_gpu.py -x -q -m gpu 2>&1 | tail -2
