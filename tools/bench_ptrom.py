"""Config 4 (BASELINE.json configs[3]) on one B200: offline tables built on
the device by the product, then the batched PTROM online march over n_inst
μ instances. Reports instance-steps/s (T = reassign + march, offline build
excluded, as BASELINE.md §2)."""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2103_01983_b200 as pt  # noqa: E402
from paper_2103_01983_b200 import rom, workloads  # noqa: E402
from paper_2103_01983_b200.tree import ClusterCriterion  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--inst", type=int, default=4096)
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()

t0 = time.perf_counter()
w = workloads.config4(n=a.n, n_inst=a.inst, n_steps=a.steps)
t_gen = time.perf_counter() - t0
ctx = pt.default_context()
t0 = time.perf_counter()
ids = rom.greedy_sample(w.phi_r, w.n_samples)
t_greedy = time.perf_counter() - t0
t0 = time.perf_counter()
A = rom.build_gnat_operator(w.phi_r, ids)
t_op = time.perf_counter() - t0
g1 = w.gamma_a + w.gamma_b
basis = rom.PODBasis(w.phi, w.sv, w.x0)
op = rom.GnatOperator(basis, ids, A)
t0 = time.perf_counter()
sur = rom.SurrogateSourceBasis.cluster_pod(basis, g1, ids, ClusterCriterion.neighbor(1.0), 1)
t_sur = time.perf_counter() - t0
L = sur.export_lists()
cfg = rom.RomConfig(1e-300, 5, 1.0)
grid = pt.TimeGrid(w.dt, a.steps)
sys_ = pt.ParticleSystem(g1, w.delta)
# warm-up on a small batch
rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, w.mu[:min(8, a.inst)], sys_, pt.TimeGrid(w.dt, 1), cfg,
                         batch=a.batch)
lib = ctx.lib
if a.profile:
    lib.ptrom_profile_begin(ctx.handle)
pt.reset_kernel_eval_count()
t0 = time.perf_counter()
tr = rom.ptrom_simulate_batch(basis, op, sur, w.gamma_a, w.gamma_b, w.mu, sys_, grid, cfg, batch=a.batch)
T = time.perf_counter() - t0
pairs = pt.kernel_eval_count()
hp_ms = None
if a.profile:
    ms, nl = ctypes.c_double(), ctypes.c_int64()
    ctx.check(lib.ptrom_profile_end(ctx.handle, ctypes.byref(ms), ctypes.byref(nl)))
    hp_ms = (ms.value, nl.value)
nt = len(ids)
evals = a.inst * (1 + a.steps * 6)
out = {
    "workload": w.name, "n": a.n, "n_inst": a.inst, "steps": a.steps, "batch": a.batch, "n_samples": nt,
    "n_clusters": sur.n_clusters, "n_direct": sur.n_direct,
    "interactions_per_target": (len(L["cl_list"]) + len(L["d_list"])) / nt,
    "seconds": T, "instance_steps_per_s": a.inst * a.steps / T,
    "hyperpair_interactions": pairs, "interactions_per_s": pairs / T,
    "ac_gflop": a.inst * a.steps * 5 * 2 * 32 * 16 * 2 * nt / 1e9,
    "offline_s": {"generate_inputs_host": t_gen, "greedy_sample": t_greedy, "gnat_operator": t_op,
                  "cluster_pod": t_sur},
    "hyperpair_kernel_ms": hp_ms, "finite": bool(np.all(np.isfinite(tr.x_hat))),
    "iterations_per_step": float(np.mean(tr.iterations)),
}
print(json.dumps(out), flush=True)
