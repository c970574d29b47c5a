"""One preconditioner application at config 3 with dense groups, for a per-kernel launch list
(dev tool):  ncu --metrics gpu__time_duration.sum --csv ... python tools/prof_groups.py [keep]"""
import sys
from pathlib import Path

import numpy as np
from scipy.sparse import linalg as spla

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402
from paper_2303_01760_b200.solver import _DeviceLU  # noqa: E402

keep = int(sys.argv[1]) if len(sys.argv) > 1 else 50
ns = nodesets.hybrid_hole_2d(500, seed=2)
ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings(), factorize=True)
host_lu = spla.splu(ops.poisson_matrix.tocsc())
lu = _DeviceLU(host_lu, keep_levels=keep)
t = L.torch()
b = L.to_device(np.random.default_rng(0).normal(size=lu.n))
x = L.empty(lu.n, t.float64)
for _ in range(3):
    lu.solve(b, x)
t.cuda.synchronize()
print("done", lu.group_rows, lu.sL.n_phases)
