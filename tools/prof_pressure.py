"""Time the pieces of one pressure solve on config 3 (dev tool)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402


def levels(csr, lower=True):
    """Dependency depth of a triangular CSR (host, for diagnostics)."""
    n = csr.shape[0]
    lev = np.zeros(n, dtype=np.int64)
    ip, ix = csr.indptr, csr.indices
    rng = range(n) if lower else range(n - 1, -1, -1)
    for i in rng:
        c = ix[ip[i]:ip[i + 1]]
        if len(c):
            lev[i] = lev[c].max() + 1
    return lev


def main():
    t = L.torch()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    ns = nodesets.hybrid_hole_2d(M, seed=2)
    t0 = time.perf_counter()
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings())
    print(f"N={len(ns)} build_operators {time.perf_counter() - t0:.1f}s", flush=True)
    lu = ops._d_lu
    print(f"L nnz {lu.L.nnz:,} U nnz {lu.U.nnz:,} A nnz {ops._d_poisson.nnz:,}", flush=True)
    n1 = lu.n
    b = L.to_device(np.random.default_rng(0).normal(size=n1))
    x = L.empty(n1, t.float64)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)

    def timeit(fn, reps=3):
        fn()
        t.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0.record()
            fn()
            e1.record()
            t.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts)

    s = L.stream_handle()
    print("A matvec ms", timeit(lambda: ops._d_poisson.matvec(b, x)), flush=True)
    print("L solve ms", timeit(lambda: L.call("hn_sptrsv", 1, L.ptr(lu.L.rowptr), L.ptr(lu.L.cols),
                                              L.ptr(lu.L.vals), None, L.ptr(b), L.ptr(x), n1, L.ptr(lu.ticket), s)),
          flush=True)
    print("U solve ms", timeit(lambda: L.call("hn_sptrsv", 0, L.ptr(lu.U.rowptr), L.ptr(lu.U.cols),
                                              L.ptr(lu.U.vals), L.ptr(lu.diag), L.ptr(b), L.ptr(x), n1,
                                              L.ptr(lu.ticket), s)), flush=True)
    print("precond ms", timeit(lambda: lu.solve(b, x)), flush=True)
    # correctness of the device LU solve vs SuperLU
    got = x.cpu().numpy()
    want = ops.poisson_precond @ b.cpu().numpy()
    print("precond rel err", np.abs(got - want).max() / np.abs(want).max(), flush=True)
    Lh = lu.L
    import scipy.sparse as sp
    Lc = sp.csr_matrix((Lh.vals.cpu().numpy(), Lh.cols.cpu().numpy(), Lh.rowptr.cpu().numpy()), shape=(n1, n1))
    Uc = sp.csr_matrix((lu.U.vals.cpu().numpy(), lu.U.cols.cpu().numpy(), lu.U.rowptr.cpu().numpy()), shape=(n1, n1))
    t0 = time.perf_counter()
    lv = levels(Lc)
    lu_ = levels(Uc, lower=False)
    print(f"L depth {lv.max()} U depth {lu_.max()} (host level sweep {time.perf_counter() - t0:.1f}s)", flush=True)
    rowlen = np.diff(Lc.indptr)
    print("L row nnz mean", rowlen.mean(), "max", rowlen.max(), flush=True)


if __name__ == "__main__":
    main()
