"""A/B of the U-solve tile inverses (hn_sptrsv_super_inv with / without tinv) on config 3 (dev tool)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402
from paper_2303_01760_b200.solver import _DeviceLU  # noqa: E402


def main():
    t = L.torch()
    ns = nodesets.hybrid_hole_2d(500, seed=2)
    _DeviceLU.TILE_INVERSE = True  # the schedules compute their tile inverses at setup
    _DeviceLU.TILE_INVERSE_L = True
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings())
    lu = ops._d_lu
    b = L.to_device(np.random.default_rng(0).normal(size=lu.n))
    x = L.empty(lu.n, t.float64)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    res = {}
    for rep in range(3):
        for on in ("none", "L", "U", "LU"):
            _DeviceLU.TILE_INVERSE_L = on in ("L", "LU")
            _DeviceLU.TILE_INVERSE = on in ("U", "LU")
            for _ in range(3):
                lu.solve(b, x)
            ts = []
            for _ in range(15):
                e0.record()
                lu.solve(b, x)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            res.setdefault(on, []).append(float(np.median(ts)))
            if rep == 0:
                res[("x", on)] = x.cpu().numpy().copy()
    for on in ("none", "L", "U", "LU"):
        print(f"tile inverse {on}: L+U solve median ms per rep {['%.3f' % v for v in res[on]]}", flush=True)
    a = res[("x", "none")]
    for on in ("L", "U", "LU"):
        print(on, "max rel diff vs substitution", float(np.abs(res[("x", on)] - a).max() / np.abs(a).max()))
    _DeviceLU.TILE_INVERSE = False
    _DeviceLU.TILE_INVERSE_L = False


if __name__ == "__main__":
    main()
