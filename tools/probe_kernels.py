"""Throughput of the all-pairs variants at config 2 (N = 65,536): fp64
velocity, fp64 Jacobian (Newton blocks), fp32 velocity, hamiltonian."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import device as dev  # noqa: E402
from paper_2103_01983_b200 import workloads  # noqa: E402

w = workloads.config2()
n = w.n
x = torch.tensor(w.x0, device="cuda")
g = torch.tensor(w.gamma, device="cuda")
x32, g32 = x.float(), g.float()
ctx = pt.default_context(0)
inv = torch.empty((n, 4), dtype=torch.float64, device="cuda")
out = torch.empty(2 * n, dtype=torch.float64, device="cuda")
out32 = torch.empty(2 * n, dtype=torch.float32, device="cuda")
cases = {
    "vel_f64": (lambda: dev.pairwise_velocity(x, g, w.delta, 0, None, 0, n, out, ctx=ctx), 12),
    "jac_f64_newton_blocks": (lambda: dev.newton_blocks(x, g, w.delta, 0, 1e-3, 0, n, inv, ctx=ctx), 21),
    "vel_f32": (lambda: dev.pairwise_velocity(x32, g32, w.delta, 0, None, 0, n, out32, ctx=ctx), 12),
    "hamiltonian_f64": (lambda: dev.hamiltonian(x, g, ctx=ctx), None),
}
for name, (fn, flops) in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    pairs = n * (n - 1) if name != "hamiltonian_f64" else n * (n - 1) // 2
    d = {"kernel": name, "ms": ms, "pairs_per_s": pairs / (ms * 1e-3)}
    if flops:
        d["tflops"] = flops * pairs / (ms * 1e-3) / 1e12
    print(json.dumps(d))
