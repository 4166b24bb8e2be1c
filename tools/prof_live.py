"""Live per-kernel device times (CUPTI through torch.profiler, no replay,
warm caches) for one workload step:

    python tools/prof_live.py config4 [batch] [steps]
    python tools/prof_live.py config3
"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import workloads  # noqa: E402


def table(prof, title):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        k = e.name.replace("(anonymous namespace)::", "").split("(")[0][:80]
        agg[k][0] += 1
        agg[k][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    tot = sum(v[1] for v in agg.values())
    print(f"== {title}: {tot / 1e3:.2f} ms kernel time")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        print(f"{t / 1e3:10.3f} ms {c:6d}  {t / max(c, 1):9.1f} us/launch  {k}")


what = sys.argv[1]
# PTROM_TUNING="key=value,...": ptrom_set_tuning on the default context (A/B of engine variants)
for kv in filter(None, os.environ.get("PTROM_TUNING", "").split(",")):
    k_, v_ = kv.split("=")
    pt.default_context().set_tuning(k_, int(v_))
if what == "config4":
    from paper_2103_01983_b200 import rom
    from paper_2103_01983_b200.tree import ClusterCriterion
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    w = workloads.config4(n_inst=B)
    ids = rom.greedy_sample(w.phi_r, w.n_samples)
    A = rom.build_gnat_operator(w.phi_r, ids)
    g1 = w.gamma_a + w.gamma_b
    basis = rom.PODBasis(w.phi, w.sv, w.x0)
    op = rom.GnatOperator(basis, ids, A)
    sur = rom.SurrogateSourceBasis.cluster_pod(basis, g1, ids, ClusterCriterion.neighbor(1.0), 1)
    cfg = rom.RomConfig(1e-300, 5, 1.0)
    sys_ = pt.ParticleSystem(g1, w.delta)
    rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, w.mu[:B], sys_, pt.TimeGrid(w.dt, 1), cfg, batch=B)
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, w.mu[:B], sys_, pt.TimeGrid(w.dt, steps), cfg,
                                 batch=B)
        torch.cuda.synchronize()
    print(f"wall {time.perf_counter() - t0:.3f} s for {B} x {steps} instance-steps")
    table(prof, f"config4 B={B} steps={steps}")
    t0 = time.perf_counter()
    rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, w.mu[:B], sys_, pt.TimeGrid(w.dt, steps), cfg,
                             batch=B)
    print(f"wall (no profiler) {time.perf_counter() - t0:.3f} s")
    # single-instance drop-in (exact reassign per query)
    t0 = time.perf_counter()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        rom.ptrom_simulate(basis, op, sur, pt.ParticleSystem(w.gamma_a + 1.3 * w.gamma_b, w.delta),
                           pt.TimeGrid(w.dt, 2), cfg)
        torch.cuda.synchronize()
    print(f"single instance, 2 steps: wall {time.perf_counter() - t0:.3f} s")
    table(prof, "ptrom_simulate single instance")
elif what == "config1":
    w = workloads.config1()
    sysm = pt.ParticleSystem(w.gamma, w.delta)
    pt.fom_simulate(w.x0, sysm, pt.TimeGrid(w.dt, 3))
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pt.fom_simulate(w.x0, sysm, pt.TimeGrid(w.dt, w.n_steps))
        torch.cuda.synchronize()
    table(prof, "config1 FOM 100 steps")
elif what == "config3":
    import ctypes
    w = workloads.config3()
    ctx = pt.default_context()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    x = torch.tensor(w.x0, device="cuda")
    g = torch.tensor(w.gamma, device="cuda")
    f = torch.empty(2 * w.n, dtype=torch.float64, device="cuda")
    cnt = ctypes.c_uint64()
    step = lambda: ctx.check(ctx.lib.ptrom_dev_barnes_hut_velocity_f64(ctx.handle, w.n, x.data_ptr(), g.data_ptr(),
                                                                       w.delta, 0, 0, 0.5, 32, None, f.data_ptr(),
                                                                       ctypes.byref(cnt)))
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            step()
        torch.cuda.synchronize()
    table(prof, "config3 x5")
