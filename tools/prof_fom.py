"""Live per-kernel device times of the config-1 FOM trajectory (CUPTI via
torch.profiler, no replay): python tools/prof_fom.py"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import workloads  # noqa: E402

w = workloads.config1()
sysm = pt.ParticleSystem(w.gamma, w.delta)
pt.fom_simulate(w.x0, sysm, pt.TimeGrid(w.dt, 5))
t0 = time.perf_counter()
run = pt.fom_simulate(w.x0, sysm, pt.TimeGrid(w.dt, w.n_steps))
t = time.perf_counter() - t0
it = int(np.sum(run.iterations))
print(f"config1 FOM: {t * 1e3:.2f} ms for {w.n_steps} steps, {it} Newton updates")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    pt.fom_simulate(w.x0, sysm, pt.TimeGrid(w.dt, w.n_steps))
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    k = e.name.replace("(anonymous namespace)::", "").split("(")[0][:90]
    agg[k][0] += 1
    agg[k][1] += e.device_time_total
tot = sum(v[1] for v in agg.values())
print(f"kernel time {tot / 1e3:.2f} ms")
for k, (c, tt) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{tt / 1e3:9.3f} ms {c:6d} {tt / max(c, 1):8.1f} us  {k}")
