"""Dump config 4's surrogate lists (cluster / near-field CSR) and target ids for
offline analysis of list overlap between spatially adjacent targets."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench_extra import _config4_setup  # noqa: E402

pt, rom, w, ctx, ids, A, basis, op, sur, off = _config4_setup(None)
L = sur.export_lists()
np.savez_compressed(sys.argv[1], cl_off=L["cl_off"], cl_list=L["cl_list"].astype(np.int32), d_off=L["d_off"],
                    d_list=L["d_list"].astype(np.int32), targets=np.asarray(ids), x0=w.x0)
print("saved", {k: v.shape for k, v in L.items()})
