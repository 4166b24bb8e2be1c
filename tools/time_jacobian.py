"""Device time of one full-set self-block Jacobian evaluation (config 2 and
config 5 inputs): unordered pairs (default) and one-sided
(PTROM_ALLPAIRS_SYM=0 in the environment).

    python tools/time_jacobian.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import device as dev, workloads  # noqa: E402

out = {"sym": os.environ.get("PTROM_ALLPAIRS_SYM", "1") != "0"}
for name, w, reps in (("config2", workloads.config2(), 20), ("config5", workloads.config5(), 1)):
    n = w.n
    x = torch.tensor(w.x0, device="cuda")
    g = torch.tensor(w.gamma, device="cuda")
    ctx = pt.default_context()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    dev.inexact_kernel_jacobian(x, g, w.delta, ctx=ctx)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        dev.inexact_kernel_jacobian(x, g, w.delta, ctx=ctx)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    out[name] = {"ms": ms, "pairs_per_s": n * (n - 1) / (ms * 1e-3),
                 "tflops_21_per_pair": 21 * n * (n - 1) / (ms * 1e-3) / 1e12}
print(json.dumps(out))
