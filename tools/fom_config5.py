"""Config 5 on one GPU, end to end: the 20-step implicit-trapezoidal FOM
(config-1 integrator, dt = 1e-3) at N = 4,194,304 through the reference-facing
fom_simulate (host state in, snapshots out). Reports the wall time, the Newton
updates per step and the pair rate over the whole trajectory.

    python tools/fom_config5.py [n] [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = workloads.config5(n=n)
sysm = pt.ParticleSystem(w.gamma, w.delta)
pt.reset_kernel_eval_count()
t0 = time.perf_counter()
run = pt.fom_simulate(w.x0, sysm, pt.TimeGrid(1e-3, steps))
wall = time.perf_counter() - t0
pairs = pt.kernel_eval_count()
snap = run.snapshots
out = {"workload": w.name, "n": n, "steps": steps, "wall_s": wall, "newton_updates": run.iterations,
       "converged": run.converged, "velocity_pairs": pairs, "velocity_evaluations": pairs / (n * (n - 1)),
       "pairs_per_s_incl_jacobians_and_io": pairs / wall, "finite": bool(np.isfinite(snap).all()),
       "max_displacement": float(np.abs(snap[:, -1] - w.x0).max())}
print(json.dumps(out))
