import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2103_01983_b200 as pt
from paper_2103_01983_b200 import rom, workloads
from paper_2103_01983_b200.tree import ClusterCriterion
from oracle import pyoracle
# bit-exactness at scale with big clusters (N = 200k; neighbor clusters reach > 4096 members)
w = workloads.config4(n=200000, n_inst=2)
ids = rom.greedy_sample(w.phi_r, w.n_samples)
g1 = w.gamma_a + w.gamma_b
basis = rom.PODBasis(w.phi, w.sv, w.x0)
sur = rom.SurrogateSourceBasis.cluster_pod(basis, g1, ids, ClusterCriterion.neighbor(1.0), 1)
L = sur.export_lists()
sizes = np.diff(L["mem_off"])
print("clusters", len(sizes), "max members", sizes.max(), "> 4096:", (sizes > 4096).sum())
osur = pyoracle.Surrogate(w.phi, w.sv, w.x0, g1, ids, 1, 1.0, 1)
g = w.gamma_a + 1.37 * w.gamma_b
osur.reassign(g)
torch.cuda.synchronize()
t0 = time.perf_counter()
sur.reassign_cluster_circulation(g, basis)
torch.cuda.synchronize()
print("device reassign %.2f ms" % ((time.perf_counter() - t0) * 1e3))
e = sur.export()
for k in ("phi_tilde", "x0_tilde", "gamma_tilde"):
    assert np.array_equal(e[k], getattr(osur, k)), k
print("bitwise equal to the oracle")
# full config4 size timing
w = workloads.config4(n_inst=2)
ids = rom.greedy_sample(w.phi_r, w.n_samples)
g1 = w.gamma_a + w.gamma_b
basis = rom.PODBasis(w.phi, w.sv, w.x0)
sur = rom.SurrogateSourceBasis.cluster_pod(basis, g1, ids, ClusterCriterion.neighbor(1.0), 1)
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sur.reassign_cluster_circulation(w.gamma_a + (1.1 + r) * w.gamma_b, basis)
    torch.cuda.synchronize()
    print("config4 reassign %.2f ms" % ((time.perf_counter() - t0) * 1e3))
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sur.reassign_cluster_circulation(w.gamma_a + 1.7 * w.gamma_b, basis)
    torch.cuda.synchronize()
for e in prof.key_averages():
    if e.device_type.name == "CUDA":
        print(f"{e.key[:60]:60s} {e.count:4d} {e.device_time_total/1e3:9.3f} ms")
