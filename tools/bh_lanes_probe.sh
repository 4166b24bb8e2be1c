# far-field time against the targets per warp (PTROM_BH_LANES): how the warp-union walk grows
# with the slot window (32 slots touch ~3.1 leaves, 16 ~2.0, 8 ~1.5 at config 3)
for l in 32 24 16 12 8; do
  echo "lanes=$l"
  PTROM_BH_LANES=$l python tools/bench_tree.py 1048576 5 2>/dev/null | python -c "
import json,sys
t=sys.stdin.read()
i=t.find('{'); d=json.loads(t[i:]) if i>=0 else None
print(json.dumps(d)[:400] if d else t[-300:])"
done
