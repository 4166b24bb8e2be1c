"""Small driver for ncu captures of the all-pairs kernels (config 2, fp64 by
default): a few evaluations through the device C ABI."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2103_01983_b200 import device as dev  # noqa: E402
from paper_2103_01983_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", choices=["vel64", "vel32", "jac64"], default="vel64")
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
w = workloads.config2(n=a.n)
dt = torch.float32 if a.mode == "vel32" else torch.float64
x = torch.tensor(w.x0, device="cuda", dtype=dt)
g = torch.tensor(w.gamma, device="cuda", dtype=dt)
for _ in range(a.reps):
    if a.mode == "jac64":
        dev.inexact_kernel_jacobian(x, g, w.delta)
    else:
        dev.pairwise_velocity(x, g, w.delta)
dev.synchronize()
print("ok", a.mode)
