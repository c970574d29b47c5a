"""A/B the RBF weight kernels (static order vs searching) on configs 1 and 4 (dev tool).

For each variant: cold-L2 kernel time, LAPACK-count TFLOP/s, row-normwise max difference
against the searching kernel (variant 100) and against numpy dgesv on a sample, and the
number of stencils bit-identical to the searching kernel (= flagged and re-solved by it).
  python tools/ab_rbf.py [2d|3d|all] [variants, e.g. 100,0,101]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01760_b200 import _lib as L  # noqa: E402
from paper_2303_01760_b200 import nodesets  # noqa: E402
from paper_2303_01760_b200._device import device_nodes  # noqa: E402
from oracle import hn_oracle as O  # noqa: E402  (checker only)

FLOPS = {(2, 12): 5613, (3, 20): 24625, (3, 30): 54500}


def run(ns, d, n, rows, variants, fine=False):
    t = L.torch()
    dn = device_nodes(ns)
    st = dn.knn(n, rows=L.to_device(rows.astype(np.int32)), **({"fine": True} if fine else {}))
    K = len(rows)
    nops = d + 1
    kinds = L.host_ints([0] + [1] * d)
    axes = L.host_ints([0] + list(range(d)))
    nrm = L.host_dbls([0] * (3 * nops))
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    flush = L.empty(64 * 2 ** 20, t.float64)
    st_h = st.cpu().numpy().astype(np.int64)
    samp = np.random.default_rng(0).choice(K, size=min(K, 4000), replace=False)
    ops = [("lap",)] + [("d", a) for a in range(d)]
    wref = O.rbf_solve(ns.positions, st_h[samp], ops)  # (k, n, ops) stencil order
    base = None
    for v in variants:
        L.lib().hn_weights_rbf_set_variant(v)
        oi = L.empty((n, K), t.int32)
        ow = L.empty((nops, n, K), t.float64)
        info = L.zeros(K, t.int32)
        times = []
        for rep in range(7):
            flush.fill_(rep)
            e0.record()
            L.call("hn_weights_rbf", L.ptr(dn.pos), d, L.ptr(st), K, n, nops, kinds, axes, nrm, None, None,
                   L.ptr(oi), L.ptr(ow), L.ptr(info), L.stream_handle())
            e1.record()
            t.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        w = ow.cpu().numpy()
        idx = oi.cpu().numpy()
        ms = float(np.median(times[1:]))
        # numpy reference in table order: sort each stencil's weights by node id
        order = np.argsort(st_h[samp], axis=1, kind="stable")
        want = np.take_along_axis(wref, order[:, :, None], 1)  # (k, n, ops)
        got = np.transpose(w[:, :, samp], (2, 1, 0))
        ok_idx = np.array_equal(idx[:, samp].T, np.take_along_axis(st_h[samp], order, 1))
        e_np = (np.abs(got - want).max(axis=1) / np.abs(want).max(axis=1)).max()
        line = (f"  variant {v:3d}: {ms * 1e3:8.1f} us  {K * FLOPS[(d, n)] / ms / 1e9:6.2f} TFLOP/s  "
                f"vs dgesv {e_np:.1e} idx_ok {ok_idx} singular {int((info != 0).sum().item())}")
        if base is None:
            base = w
        else:
            diff = np.abs(w - base).max(axis=1) / np.abs(base).max(axis=1)
            same = int(np.sum(np.all(w == base, axis=(0, 1))))
            line += f"  vs v{variants[0]} {diff.max():.1e}  identical rows {same}"
        print(line, flush=True)
    L.lib().hn_weights_rbf_set_variant(0)


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    variants = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [100, 0, 101]
    if which in ("2d", "all"):
        ns = nodesets.jittered_box(315, seed=1)
        rows = np.nonzero(ns.kind != 2)[0]
        print(f"config 1: K = {len(rows)} (2D n=12)", flush=True)
        run(ns, 2, 12, rows, variants)
    if which in ("3d", "all"):
        ns = nodesets.hybrid_sphere_3d(94, seed=4, refine=2.8)
        rows = np.nonzero(ns.kind == 1)[0]
        for n in (20, 30):
            print(f"config 4 scattered rows: K = {len(rows)} (3D n={n})", flush=True)
            run(ns, 3, n, rows, variants, fine=True)


if __name__ == "__main__":
    main()
