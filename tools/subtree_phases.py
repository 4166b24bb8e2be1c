"""Phase breakdown of morton_subtree_kernel (PTROM_SUBTREE_PROFILE clocks):
builds the config-3 tree once with the per-subtree clock64 dump enabled and
prints, per phase, the summed and the per-subtree mean cycles.

    python tools/subtree_phases.py [n]
"""
import os
import sys
import tempfile

path = os.path.join(tempfile.gettempdir(), "ptrom_subtree_prof.csv")
os.environ["PTROM_SUBTREE_PROFILE"] = path
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2103_01983_b200 import workloads  # noqa: E402
from paper_2103_01983_b200.tree import QuadTree  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
w = workloads.config3(n=n)
for _ in range(2):
    QuadTree(w.x0[:n], w.x0[n:], w.gamma, 32)
p = np.loadtxt(path, delimiter=",", dtype=np.int64)
ph = np.diff(p[:, :8], axis=1)
names = ["members", "topology", "records", "id sort", "partitions", "chains", "abs sums"]
m = p[:, 8]
print(f"subtrees {len(p)}, members min/median/max {m.min()}/{int(np.median(m))}/{m.max()}, "
      f"nodes median {int(np.median(p[:, 9] // 100))}, levels median {int(np.median(p[:, 9] % 100))}")
tot = ph.sum()
for i, nm in enumerate(names):
    print(f"{nm:11s} {ph[:, i].sum() / tot * 100:5.1f}%  mean {ph[:, i].mean():9.0f} cyc  max {ph[:, i].max():9d}")
big = m > 1024
print(f"subtrees > 1024 members: {big.sum()}, their share of cycles {ph[big].sum() / tot * 100:.1f}%")
print(f"mean cycles per subtree {ph.sum(1).mean():.0f}, max {ph.sum(1).max()}")
