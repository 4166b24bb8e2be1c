"""Config 4 kernel variants (ptrom_set_tuning "hyperpair_variant", or the key given as the 4th argument):
per variant, one batched march of B instances x S steps; prints the average
hyperpair launch (library CUDA events around the launch), the march time and
whether x̂ is bit-identical to variant 1 (the generic kernel).

    python tools/sweep_hp.py [B] [steps] [variants, comma-separated] [tuning key]
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import rom, workloads  # noqa: E402
from paper_2103_01983_b200.tree import ClusterCriterion  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
variants = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "1,0,2,3,4").split(",")]
key = sys.argv[4] if len(sys.argv) > 4 else "hyperpair_variant"  # or gn_variant
w = workloads.config4(n_inst=B)
ctx = pt.default_context()
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ids = rom.greedy_sample(w.phi_r, w.n_samples)
A = rom.build_gnat_operator(w.phi_r, ids)
g1 = w.gamma_a + w.gamma_b
basis = rom.PODBasis(w.phi, w.sv, w.x0)
op = rom.GnatOperator(basis, ids, A)
sur = rom.SurrogateSourceBasis.cluster_pod(basis, g1, ids, ClusterCriterion.neighbor(1.0), 1)
cfg = rom.RomConfig(1e-300, 5, 1.0)
sys_ = pt.ParticleSystem(g1, w.delta)
lib = ctx.lib
ref = None
for v in variants:
    ctx.set_tuning(key, v)
    rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, w.mu[:B], sys_, pt.TimeGrid(w.dt, 1), cfg, batch=B)
    torch.cuda.synchronize()
    lib.ptrom_profile_begin(ctx.handle)
    t0 = time.perf_counter()
    tr = rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, w.mu[:B], sys_, pt.TimeGrid(w.dt, steps), cfg,
                                  batch=B)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms, nl = ctypes.c_double(), ctypes.c_int64()
    ctx.check(lib.ptrom_profile_end(ctx.handle, ctypes.byref(ms), ctypes.byref(nl)))
    xh = np.asarray(tr.x_hat)
    if ref is None:
        ref = xh
    same = bool(np.array_equal(xh, ref))
    print(json.dumps({"variant": v, "hp_avg_ms": ms.value / max(1, nl.value), "launches": nl.value,
                      "march_s": wall, "inst_steps_per_s": B * steps / wall, "bitwise_vs_first": same,
                      "max_rel_vs_first": float(np.max(np.abs(xh - ref)) / max(1e-300, np.max(np.abs(ref))))}),
          flush=True)
