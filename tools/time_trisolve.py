"""Time the L and U supernodal solves and one full preconditioner application on config 3
(dev tool; CUDA events, median of 20)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402


def timeit(fn, reps=20):
    t = L.torch()
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    t = L.torch()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    ns = nodesets.hybrid_hole_2d(M, seed=2)
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings())
    lu = ops._d_lu
    b = L.to_device(np.random.default_rng(0).normal(size=lu.n))
    x = L.empty(lu.n, t.float64)
    s = L.stream_handle()
    tl = timeit(lambda: lu._tri(lu.sL, lu.L, None, b, lu.z, s))
    tu = timeit(lambda: lu._tri(lu.sU, lu.U, lu.diag, b, lu.w, s))
    tp = timeit(lambda: lu.solve(b, x))
    print(f"L {tl:.3f} ms  U {tu:.3f} ms  precond {tp:.3f} ms  (L+U nnz {lu.L.nnz + lu.U.nnz})", flush=True)


if __name__ == "__main__":
    main()
