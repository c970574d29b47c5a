"""Sweep the scheduled triangular-solve parameters on config 3's SuperLU factors (dev tool)."""
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp
from scipy.sparse import linalg as spla

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402
from paper_2303_01760_b200.operators import DeviceCSR  # noqa: E402
from paper_2303_01760_b200.solver import plan_triangular_tasks  # noqa: E402


def main():
    t = L.torch()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    ns = nodesets.hybrid_hole_2d(M, seed=2)
    ops = hn.build_operators(ns, {"wall:x-"}, hn.PoissonSolveSettings())
    lu = spla.splu(ops.poisson_matrix.tocsc())
    Lm = sp.tril(sp.csr_matrix(lu.L), k=-1, format="csr")
    Um = sp.csr_matrix(lu.U)
    diag = Um.diagonal()
    Us = sp.triu(Um, k=1, format="csr")
    n = Lm.shape[0]
    for name, m in (("L", Lm), ("U", Us)):
        rl = np.diff(m.indptr)
        p = plan_triangular_tasks(m, name == "L", 256)
        lev = p["levels"]
        per_level_nnz = np.bincount(lev, weights=rl)
        per_level_rows = np.bincount(lev)
        print(f"{name}: nnz {m.nnz:,} depth {p['depth']} rows/level mean {per_level_rows.mean():.1f} "
              f"max row {rl.max()} ; nnz/level p50 {np.median(per_level_nnz):.0f} p99 {np.percentile(per_level_nnz, 99):.0f}"
              f" max {per_level_nnz.max():.0f}; rows>1024: {(rl > 1024).sum()}", flush=True)
    dL, dU = DeviceCSR(Lm), DeviceCSR(Us)
    dd = L.to_device(diag)
    b = L.to_device(np.random.default_rng(0).normal(size=n))
    x = L.empty(n, t.float64)
    ticket = L.zeros(1, t.int64)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    for chunk in (64, 256):
        plans = {nm: plan_triangular_tasks(m, nm == "L", chunk) for nm, m in (("L", Lm), ("U", Us))}
        dev = {}
        for nm, pl in plans.items():
            dev[nm] = dict(row=L.to_device(pl["row"]), beg=L.to_device(pl["beg"]), len=L.to_device(pl["len"]),
                           part=L.to_device(pl["part"]), np=L.to_device(pl["np"]),
                           partial=L.empty(max(pl["npartial"], 1), t.float64), nt=pl["ntasks"], npart=pl["npartial"])
        for wps in (4, 8, 16, 32, 64):
            res = []
            for nm, m, dg in (("L", dL, None), ("U", dU, dd)):
                d = dev[nm]

                def run():
                    L.call("hn_sptrsv_tasks", 0 if dg is None else 1, L.ptr(d["row"]), L.ptr(d["beg"]), L.ptr(d["len"]),
                           L.ptr(d["part"]), L.ptr(d["np"]), d["nt"], L.ptr(m.cols), L.ptr(m.vals), L.ptr(dg), L.ptr(b),
                           L.ptr(x), n, L.ptr(d["partial"]), d["npart"], L.ptr(ticket), wps, L.stream_handle())
                run()
                t.cuda.synchronize()
                e0.record()
                run()
                e1.record()
                t.cuda.synchronize()
                res.append(e0.elapsed_time(e1))
            print(f"chunk {chunk:5d} warps/SM {wps:3d}: L {res[0]:8.2f} ms  U {res[1]:8.2f} ms", flush=True)
    # reference: host SuperLU solve time
    t0 = time.perf_counter()
    lu.solve(np.random.default_rng(1).normal(size=n))
    print(f"host SuperLU solve {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
