"""Per-rank compute of the target-sharded config-2 evaluation on one GPU:
times ptrom_dev_pairwise_velocity_f64 for rows [0, N/G) against all N
sources (what each of G ranks runs after the position all-gather), G = 1..8.
Reports the compute-only strong-scaling efficiency T1 / (G · T_G); the NCCL
all-gather (2 x 8N/G bytes per rank per step) is not included."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import device as dev  # noqa: E402
from paper_2103_01983_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = workloads.config2(n=n) if n == 65536 else workloads.config5(n=n)
x = torch.tensor(w.x0, device="cuda")
g = torch.tensor(w.gamma, device="cuda")
ctx = pt.default_context(0)
res = {}
for G in (1, 2, 4, 8):
    m = n // G
    out = torch.empty(2 * m, dtype=torch.float64, device="cuda")
    for _ in range(3):
        dev.pairwise_velocity(x, g, w.delta, 0, None, 0, m, out, ctx=ctx)
    torch.cuda.synchronize()
    reps = max(3, min(50, int(2e11 / (m * n))))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        dev.pairwise_velocity(x, g, w.delta, 0, None, 0, m, out, ctx=ctx)
    b.record()
    torch.cuda.synchronize()
    res[G] = a.elapsed_time(b) / reps
for G, ms in res.items():
    print(json.dumps({"n": n, "G": G, "targets_per_rank": n // G, "ms": ms,
                      "compute_efficiency": res[1] / (G * ms)}))
