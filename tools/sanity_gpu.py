"""Early GPU sanity run: drive libhn.so directly on small synthetic inputs and compare
with numpy/scipy.  Development tool (not part of the product path)."""

import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp
from scipy.spatial import cKDTree

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01760_b200 import _lib as L  # noqa: E402


def pad_pos(p):
    d = p.shape[1]
    s = 2 if d == 2 else 4
    out = np.zeros((len(p), s))
    out[:, :d] = p
    return out


def knn_ref(p, q_idx, n):
    tree = cKDTree(p)
    k = min(len(p), n + 8)
    while True:
        d, idx = tree.query(p[q_idx], k=k)
        if k == len(p) or np.all(d[:, -1] > d[:, n - 1] * (1 + 1e-12)):
            break
        k = min(len(p), 2 * k)
    order = np.lexsort((idx, d), axis=1)
    return np.take_along_axis(idx, order, axis=1)[:, :n]


def main():
    t = L.torch()
    lib = L.lib()
    print("hn_version", lib.hn_version())
    # fp64 peak probe
    out = L.zeros(1, t.float64)
    blocks, iters = 148 * 8, 4096
    L.call("hn_bench_dfma", L.ptr(out), blocks, iters, L.stream_handle())
    t.cuda.synchronize()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    e0.record()
    L.call("hn_bench_dfma", L.ptr(out), blocks, iters, L.stream_handle())
    e1.record()
    t.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    flops = blocks * 256 * iters * 16 * 2
    print(f"DFMA probe: {flops / ms / 1e9:.1f} TFLOP/s ({ms:.3f} ms)")

    rng = np.random.default_rng(0)
    M = 315
    h = 1.0 / M
    ij = np.array([(i, j) for i in range(1, M) for j in range(1, M)], float)
    pts = ij * h + rng.uniform(-0.35 * h, 0.35 * h, ij.shape)
    n = len(pts)
    d = 2
    dp = L.to_device(pad_pos(pts))
    lo = pts.min(axis=0)
    hi = pts.max(axis=0)
    cell = h
    dims = [int(np.floor((hi[a] - lo[a]) / cell)) + 1 for a in range(d)]
    ncells = int(np.prod(dims))
    cs = L.empty(ncells + 1, t.int32)
    ci = L.empty(n, t.int32)
    cp = L.empty((n, 2), t.float64)
    sc = L.empty(ncells, t.int32)
    spc = L.empty(n, t.int32)
    L.call("hn_celllist_build", L.ptr(dp), n, d, L.host_dbls(lo), cell, L.host_ints(dims), L.ptr(cs), L.ptr(ci),
           L.ptr(cp), L.ptr(sc), L.ptr(spc), L.stream_handle())
    nst = 12
    oi = L.empty((n, nst), t.int32)
    od = L.empty((n, nst), t.float64)
    t.cuda.synchronize()
    t0 = time.perf_counter()
    L.call("hn_knn", L.ptr(dp), d, L.host_dbls(lo), cell, L.host_ints(dims), L.ptr(cs), L.ptr(ci), L.ptr(cp),
           None, None, n, nst, None, L.ptr(oi), L.ptr(od), L.stream_handle())
    t.cuda.synchronize()
    print(f"knn {n} queries: {1e3 * (time.perf_counter() - t0):.2f} ms (incl. launch)")
    got = oi.cpu().numpy()
    ref = knn_ref(pts, np.arange(n), nst)
    print("knn bit-exact:", np.array_equal(got, ref), "mismatch rows:", int(np.sum(np.any(got != ref, axis=1))))

    # RBF weights for Lap, dx, dy
    kinds = [0, 1, 1]
    axes = [0, 0, 1]
    K = n
    widx = L.empty((nst, K), t.int32)
    ww = L.empty((3, nst, K), t.float64)
    info = L.empty(K, t.int32)
    st = t.from_numpy(ref.astype(np.int32)).cuda()
    L.call("hn_weights_rbf", L.ptr(dp), d, L.ptr(st), K, nst, 3, L.host_ints(kinds), L.host_ints(axes), None,
           None, None, L.ptr(widx), L.ptr(ww), L.ptr(info), L.stream_handle())
    t.cuda.synchronize()
    for rep in range(3):
        e0.record()
        L.call("hn_weights_rbf", L.ptr(dp), d, L.ptr(st), K, nst, 3, L.host_ints(kinds), L.host_ints(axes), None,
               None, None, L.ptr(widx), L.ptr(ww), L.ptr(info), L.stream_handle())
        e1.record()
        t.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"rbf weights {K}: {ms:.3f} ms -> {K * 5613 / ms / 1e9:.2f} TFLOP/s (LAPACK-count)")
    print("info nonzero:", int((info != 0).sum()))
    # numpy reference for a subset
    sub = rng.choice(K, 500, replace=False)
    P = pts[ref[sub]]
    rel = P - P[:, :1]
    scale = np.max(np.linalg.norm(rel, axis=-1), axis=1)
    loc = rel / scale[:, None, None]
    diff = loc[:, :, None, :] - loc[:, None, :, :]
    A = np.sqrt((diff ** 2).sum(-1)) ** 3
    ex = [(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)]
    Pm = np.stack([loc[..., 0] ** a * loc[..., 1] ** b for a, b in ex], -1)
    S = np.zeros((len(sub), 18, 18))
    S[:, :12, :12] = A
    S[:, :12, 12:] = Pm
    S[:, 12:, :12] = Pm.transpose(0, 2, 1)
    r = np.linalg.norm(loc, axis=-1)
    R = np.zeros((len(sub), 18, 3))
    R[:, :12, 0] = 9 * r
    R[:, :12, 1] = -3 * r * loc[..., 0]
    R[:, :12, 2] = -3 * r * loc[..., 1]
    R[:, 12 + 3, 0] = 2
    R[:, 12 + 5, 0] = 2
    R[:, 12 + 1, 1] = 1
    R[:, 12 + 2, 2] = 1
    sol = np.linalg.solve(S, R)[:, :12]
    sol[:, :, 0] /= scale[:, None] ** 2
    sol[:, :, 1:] /= scale[:, None, None]
    order = np.argsort(ref[sub], axis=1)
    wref = np.take_along_axis(sol, order[:, :, None], axis=1)
    gi = widx.cpu().numpy().T[sub]
    gw = ww.cpu().numpy().transpose(2, 1, 0)[sub]
    print("rbf idx sorted equal:", np.array_equal(gi, np.sort(ref[sub], axis=1)))
    err = np.abs(gw - wref).max(axis=1) / np.abs(wref).max(axis=1)
    print("rbf weights max rel (row-normwise) err:", err.max())

    # apply bit-exact vs scipy CSR
    f = np.sin(3 * pts[:, 0]) * np.cos(2 * pts[:, 1])
    df = L.to_device(f)
    outp = L.empty((3, n), t.float64)
    rows = t.arange(n, dtype=t.int32, device="cuda")
    L.call("hn_apply_ell", 1, L.host_i64([K]), L.host_ints([nst]), L.host_ptrs([rows]), L.host_ptrs([widx]),
           L.host_ptrs([ww]), 3, L.host_ints([0, 1, 2]), L.ptr(df), L.ptr(outp), n, L.stream_handle())
    t.cuda.synchronize()
    I = widx.cpu().numpy().T
    W = ww.cpu().numpy().transpose(0, 2, 1)
    ok = True
    for o in range(3):
        csr = sp.csr_matrix((W[o].ravel(), I.ravel(), np.arange(0, n * nst + 1, nst)), shape=(n, n))
        ok &= np.array_equal(csr @ f, outp[o].cpu().numpy())
    print("apply bit-exact vs scipy csr:", ok)
    for rep in range(3):
        e0.record()
        L.call("hn_apply_ell", 1, L.host_i64([K]), L.host_ints([nst]), L.host_ptrs([rows]), L.host_ptrs([widx]),
               L.host_ptrs([ww]), 3, L.host_ints([0, 1, 2]), L.ptr(df), L.ptr(outp), n, L.stream_handle())
        e1.record()
        t.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        byt = 28 * n * nst + 8 * n + 24 * n
        print(f"apply 3 ops: {ms * 1e3:.1f} us -> {byt / ms / 1e6:.0f} GB/s (warm L2)")

    # MON 2D lattice stencil check
    hh = 0.1
    lat = np.array([[i * hh, j * hh] for i in range(5) for j in range(5)])
    dl = L.to_device(pad_pos(lat))
    stm = t.tensor([[12, 7, 11, 13, 17]], dtype=t.int32, device="cuda")
    mi = L.empty((5, 1), t.int32)
    mw = L.empty((3, 5, 1), t.float64)
    minfo = L.empty(1, t.int32)
    L.call("hn_weights_mon", L.ptr(dl), 2, L.ptr(stm), 1, 3, L.host_ints(kinds), L.host_ints(axes), None,
           L.ptr(mi), L.ptr(mw), L.ptr(minfo), L.stream_handle())
    t.cuda.synchronize()
    print("MON idx", mi.cpu().numpy().ravel(), "lap", mw[0].cpu().numpy().ravel(), "dx", mw[1].cpu().numpy().ravel())


if __name__ == "__main__":
    main()
