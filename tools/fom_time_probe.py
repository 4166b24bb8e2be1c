import time, numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2103_01983_b200 as pt
from paper_2103_01983_b200 import workloads
w = workloads.config1()
sysm = pt.ParticleSystem(w.gamma, w.delta)
pt.fom_simulate(w.x0, sysm, pt.TimeGrid(w.dt, 5))
t0 = time.perf_counter()
run = pt.fom_simulate(w.x0, sysm, pt.TimeGrid(w.dt, w.n_steps))
t = time.perf_counter() - t0
it = int(np.sum(run.iterations))
print(f"config1 FOM: {t*1e3:.1f} ms for {w.n_steps} steps, {it} Newton updates, {t*1e6/(it+w.n_steps):.1f} us per velocity eval")
