"""Sweeps the velocity-kernel shape table (csrc/allpairs.cu PTROM_VEL_VARIANTS)
at config 2 (N = 65,536, fp64) and prints ms / TFLOP/s per variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import device as dev  # noqa: E402
from paper_2103_01983_b200 import workloads  # noqa: E402

n_var = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
w = workloads.config2(n=n)
x = torch.tensor(w.x0, device="cuda")
g = torch.tensor(w.gamma, device="cuda")
ref = None
res = []
for v in range(n_var):
    os.environ["PTROM_ALLPAIRS_VARIANT"] = str(v)
    ctx = pt.Context(0)
    out = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        dev.pairwise_velocity(x, g, w.delta, out=out, ctx=ctx)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    reps = 10
    for _ in range(reps):
        dev.pairwise_velocity(x, g, w.delta, out=out, ctx=ctx)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    if ref is None:
        ref = out.clone()
    err = float((out - ref).norm() / ref.norm())
    tf = 12 * n * (n - 1) / (ms * 1e-3) / 1e12
    res.append({"variant": v, "ms": ms, "tflops": tf, "rel_vs_v0": err})
    print(json.dumps(res[-1]), flush=True)
    ctx.close()
