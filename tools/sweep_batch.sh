# config-4 PTROM march over the instance batch size (instances marched together per launch)
for b in 256 512 1024 2048; do
  echo "batch=$b"
  python tools/bench_ptrom.py --inst 4096 --steps 5 --batch $b 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['instance_steps_per_s'], d['seconds'])"
done
