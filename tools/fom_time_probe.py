"""Wall time of the config-1 trajectory through the host entry point
(ptrom_fom_simulate_f64) and the device entry point (ptrom_dev_fom_simulate_f64)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import device as dev  # noqa: E402
from paper_2103_01983_b200 import workloads  # noqa: E402

w = workloads.config1()
sysm = pt.ParticleSystem(w.gamma, w.delta)
grid = pt.TimeGrid(w.dt, w.n_steps)
for _ in range(3):
    pt.fom_simulate(w.x0, sysm, grid)
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    run = pt.fom_simulate(w.x0, sysm, grid)
    ts.append(time.perf_counter() - t0)
print(f"host API: median {np.median(ts)*1e3:.2f} ms, min {min(ts)*1e3:.2f} ms, updates {int(np.sum(run.iterations))}")
x0 = torch.tensor(w.x0, device="cuda")
g = torch.tensor(w.gamma, device="cuda")
snaps = torch.empty(w.n_steps, 2 * w.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    dev.fom_simulate(x0, g, w.delta, w.dt, w.n_steps, snapshots=snaps)
ts = []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = dev.fom_simulate(x0, g, w.delta, w.dt, w.n_steps, snapshots=snaps)
    ts.append(time.perf_counter() - t0)
print(f"device API: median {np.median(ts)*1e3:.2f} ms, min {min(ts)*1e3:.2f} ms, evals {r[4]} + {r[5]}")
