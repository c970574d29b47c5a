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
    _DeviceLU.TILE_INVERSE = True  # the U schedule computes its tile inverses at setup
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings())
    lu = ops._d_lu
    b = L.to_device(np.random.default_rng(0).normal(size=lu.n))
    x = L.empty(lu.n, t.float64)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    res = {}
    for rep in range(3):
        for on in (False, True):
            _DeviceLU.TILE_INVERSE = on
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
    for on in (False, True):
        print(f"tile inverse {on}: L+U solve median ms per rep {['%.3f' % v for v in res[on]]}", flush=True)
    a, c = res[("x", False)], res[("x", True)]
    print("max rel diff", float(np.abs(a - c).max() / np.abs(a).max()))
    _DeviceLU.TILE_INVERSE = False


if __name__ == "__main__":
    main()
