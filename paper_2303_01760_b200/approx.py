"""Stencils and differentiation weights on the GPU (drop-in for hybridnodes.approx).

Same names, signatures, return types and errors as pkg/src/hybridnodes/approx.py; the
arithmetic runs in libhn.so:

  classify_methods / select_method  -> hn_classify (+ hn_knn probes without a lattice)
  _mon_stencils / find_stencil      -> hn_mon_stencils / hn_knn  (bit-exact indices)
  _batched_mon_weights              -> hn_weights_mon   (thread per stencil)
  _batched_rbf_weights              -> hn_weights_rbf   (warp-cooperative Gauss-Jordan)
  compute_weights                   -> all of the above, results kept in HBM as ELL bins

`tree` arguments (scipy cKDTree in the reference) are accepted and ignored: the device
cell list replaces them.  Condition numbers (with_kappa / WeightRow.kappa) -- the reference's
numpy SVD diagnostic (approx.py:100-105, 229-233, 285-289) -- run on the GPU
(hn_condition_numbers) for the stencil sizes the library has kernels for, else on the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._device import Bin, DeviceTable, bins_args, device_nodes
from .errors import SingularSystemError
from .nodegen import KIND_BOUNDARY, KIND_REGULAR, LATTICE_NONE

MON_SIZE = {2: 5, 3: 7}
RBF_SIZE = {2: 12, 3: 30}  # read at call time, like the reference (approx.py:25, 388, 420)
POLY_COUNT = {2: 6, 3: 10}

METHOD_MON = 0
METHOD_RBFFD = 1
METHOD_NONE = -1


@dataclass(frozen=True)
class Laplacian:
    order: int = 2


@dataclass(frozen=True)
class Partial:
    axis: int
    order: int = 1


@dataclass(frozen=True)
class NormalDerivative:
    normal: tuple
    order: int = 1


@dataclass(frozen=True)
class StencilSpec:
    center: int
    neighbors: np.ndarray
    method: str


@dataclass
class WeightRow:
    neighbors: np.ndarray
    weights: dict
    kappa: float


# ---------------------------------------------------------------- operator codes
def _op_code(op, dim: int):
    """(kind, axis, normal) for HN_OP_*; accepts this package's or the reference's op classes."""
    name = type(op).__name__
    if name == "Laplacian":
        return 0, 0, (0.0,) * dim
    if name == "Partial":
        return 1, int(op.axis), (0.0,) * dim
    if name == "NormalDerivative":
        nrm = tuple(float(v) for v in op.normal)
        if len(nrm) != dim:
            raise ValueError("normal has the wrong dimension")
        return 2, 0, nrm
    raise TypeError(f"unknown operator kind {op!r}")


def _op_args(ops, dim):
    codes = [_op_code(op, dim) for op in ops]
    return (L.host_ints([c[0] for c in codes]), L.host_ints([c[1] for c in codes]),
            L.host_dbls([v for c in codes for v in c[2]]))


def _op_order(op) -> int:
    return int(getattr(op, "order", 2 if type(op).__name__ == "Laplacian" else 1))


# ---------------------------------------------------------------- diagnostics (host)
def condition_number(matrix: np.ndarray) -> float:
    """Spectral condition number sigma_max / sigma_min (+inf when singular)."""
    s = np.linalg.svd(np.asarray(matrix, dtype=float), compute_uv=False)
    if s[-1] == 0.0:
        return float("inf")
    return float(s[0] / s[-1])


def _exps(dim):
    out = [(0,) * dim]
    for a in range(dim):
        e = [0] * dim
        e[a] = 1
        out.append(tuple(e))
    for a in range(dim):
        for b in range(a, dim):
            e = [0] * dim
            e[a] += 1
            e[b] += 1
            out.append(tuple(e))
    return out


def _local(positions, stencils):
    pts = positions[stencils]
    rel = pts - pts[:, :1, :]
    scale = np.max(np.linalg.norm(rel, axis=-1), axis=1)
    return rel / scale[:, None, None]


def _kappa_host(positions: np.ndarray, stencils: np.ndarray, mon: bool) -> np.ndarray:
    """kappa of the local systems (approx.py:229-233, 285-289); host SVD diagnostic."""
    loc = _local(positions, stencils)
    k, n, dim = loc.shape
    if mon:
        m = np.empty((k, n, n))
        m[:, 0, :] = 1.0
        for a in range(dim):
            m[:, 1 + a, :] = loc[:, :, a]
            m[:, 1 + dim + a, :] = loc[:, :, a] ** 2
    else:
        ex = _exps(dim)
        q = len(ex)
        m = np.zeros((k, n + q, n + q))
        diff = loc[:, :, None, :] - loc[:, None, :, :]
        m[:, :n, :n] = np.sqrt(np.sum(diff * diff, axis=-1)) ** 3
        p = np.ones((k, n, q))
        for j, e in enumerate(ex):
            for a in range(dim):
                if e[a]:
                    p[:, :, j] *= loc[:, :, a] ** e[a]
        m[:, :n, n:] = p
        m[:, n:, :n] = np.transpose(p, (0, 2, 1))
    s = np.linalg.svd(m, compute_uv=False)
    with np.errstate(divide="ignore"):
        return np.where(s[:, -1] > 0, s[:, 0] / s[:, -1], np.inf)


_KAPPA_SIZES = {(2, 5, True), (3, 7, True), (2, 12, False), (3, 20, False), (3, 30, False)}


def _kappa_bin(dn, d_idx, rs: int, cs: int, d_centers, K: int, n: int, mon: bool):
    """kappa of K device stencils (hn_condition_numbers) -> device fp64 (K,)."""
    t = L.torch()
    out = L.empty(max(K, 1), t.float64)
    if K:
        L.call("hn_condition_numbers", L.ptr(dn.pos), dn.stride, dn.dim, L.ptr(d_idx), rs, cs, L.ptr(d_centers), K, n,
               1 if mon else 0, L.ptr(out), L.stream_handle())
    return out[:K]


def _kappa(nodeset_or_positions, stencils: np.ndarray, mon: bool) -> np.ndarray:
    """kappa of host stencils (K, n), centre first: GPU for the library's sizes, else host SVD."""
    positions = np.asarray(getattr(nodeset_or_positions, "positions", nodeset_or_positions), float)
    stencils = np.atleast_2d(np.asarray(stencils, dtype=np.int64))
    k, n = stencils.shape
    if (positions.shape[1], n, bool(mon)) not in _KAPPA_SIZES:
        return _kappa_host(positions, stencils, mon)
    from ._device import DeviceNodes
    dn = device_nodes(nodeset_or_positions) if hasattr(nodeset_or_positions, "positions") else None
    if dn is None:
        dn = _PosOnly(positions)
    st = L.to_device(np.ascontiguousarray(stencils, dtype=np.int32))
    return _kappa_bin(dn, st, n, 1, None, k, n, mon).cpu().numpy()


class _PosOnly:
    """Device copy of bare coordinates for hn_condition_numbers (per-stencil API calls)."""

    def __init__(self, positions: np.ndarray):
        self.dim = positions.shape[1]
        self.stride = self.dim
        self.pos = L.to_device(np.ascontiguousarray(positions, dtype=np.float64))


# ---------------------------------------------------------------- device solves
def _solve_bin(dn, stencils_dev, d_rows, ops, mon: bool, row_normals=None):
    """Weights for a batch of stencils straight into an ELL bin (ascending node order).
    Returns (Bin, info); info[k] != 0 marks a singular stencil (checked by _check_info)."""
    t = L.torch()
    K, n = int(stencils_dev.shape[0]), int(stencils_dev.shape[1])
    nops = len(ops)
    d_idx = L.empty((n, max(K, 1)), t.int32)
    d_w = L.empty((nops, n, max(K, 1)), t.float64)
    info = L.zeros(max(K, 1), t.int32)
    if K:
        kinds, axes, normals = _op_args(ops, dn.dim)
        if mon:
            if n != 2 * dn.dim + 1:
                raise SingularSystemError(f"singular MON system: stencil size {n} != {2 * dn.dim + 1}")
            L.call("hn_weights_mon", L.ptr(dn.pos), dn.dim, L.ptr(stencils_dev), K, nops, kinds, axes, normals,
                   L.ptr(d_idx), L.ptr(d_w), L.ptr(info), L.stream_handle())
        else:
            ws = None
            if L.lib().hn_weights_rbf_is_tuned(dn.dim, n, nops) != 0:
                ws = L.empty(int(L.lib().hn_weights_rbf_workspace(dn.dim, n, nops, K)), t.float64)
            rn = L.to_device(np.ascontiguousarray(row_normals, dtype=float)) if row_normals is not None else None
            L.call("hn_weights_rbf", L.ptr(dn.pos), dn.dim, L.ptr(stencils_dev), K, n, nops, kinds, axes, normals,
                   L.ptr(rn), L.ptr(ws), L.ptr(d_idx), L.ptr(d_w), L.ptr(info), L.stream_handle())
    b = Bin(None, n, d_idx[:, :K] if K else d_idx[:, :0], d_w[:, :, :K] if K else d_w[:, :, :0], d_rows=d_rows, K=K)
    b.mon = mon
    return b, info[:K]


def _check_info(pairs):
    """One device reduction + one read-back for every bin's singular flags (approx.py:223-226, 278-281)."""
    pairs = [(b, i) for b, i in pairs if b.K]
    if not pairs:
        return
    t = L.torch()
    flags = t.stack([t.count_nonzero(i) for _, i in pairs]).cpu().numpy()
    for (b, info), bad in zip(pairs, flags):
        if bad:
            first = int(t.nonzero(info)[0].item())
            kind = "MON" if b.mon else "RBF-FD saddle"
            raise SingularSystemError(f"singular {kind} system: Singular matrix ({int(bad)} stencil(s), first at "
                                      f"node {int(b.d_rows[first].item())})")


def _solve_points(points: np.ndarray, ops, mon: bool, row_normals=None):
    """Weights of one or more stencils given directly as point arrays (K, n, d)."""
    pts = np.asarray(points, dtype=float)
    k, n, dim = pts.shape

    class _Tmp:
        pass

    tmp = _Tmp()
    tmp.positions = pts.reshape(k * n, dim)
    tmp.kind = np.ones(k * n, dtype=np.int8)
    dn = device_nodes_uncached(tmp)
    st = L.to_device(np.arange(k * n, dtype=np.int32).reshape(k, n))
    b, info = _solve_bin(dn, st, L.to_device(np.arange(k, dtype=np.int32)), ops, mon, row_normals)
    _check_info([(b, info)])
    idx = b.d_idx.cpu().numpy().T.reshape(k, n)          # local ids, ascending = stencil order ids
    w = b.d_w.cpu().numpy().transpose(0, 2, 1)           # (nops, K, n) ascending local id
    return idx, w


def device_nodes_uncached(obj):
    from ._device import DeviceNodes
    return DeviceNodes(obj)


# ---------------------------------------------------------------- public API
def select_method(index: int, nodeset, tree=None) -> str:
    """MON for regular nodes whose 2d axis neighbours all exist; else RBF-FD (approx.py:114-130)."""
    if nodeset.kind[index] != KIND_REGULAR:
        return "rbffd"
    dim = nodeset.dim
    lat, lidx = getattr(nodeset, "lattice", None), getattr(nodeset, "lattice_idx", None)
    if lat is not None and lidx is not None and lidx[index][0] != LATTICE_NONE:
        m = int(device_nodes(nodeset).classify()[index].item())
        return "mon" if m == METHOD_MON else "rbffd"
    h = nodeset.spacing[index]
    pos = nodeset.positions[index]
    probes = np.concatenate([pos + h * np.eye(dim), pos - h * np.eye(dim)])
    _, dist = device_nodes(nodeset).knn(1, points=probes, with_dist=True)
    return "mon" if bool(np.all(dist.cpu().numpy()[:, 0] < 1e-9 * h)) else "rbffd"


def find_stencil(center: int, nodeset, n: int, tree=None) -> StencilSpec:
    """The n nearest nodes (centre included) by (distance, index) (approx.py:149-155)."""
    total = len(nodeset)
    if n > total:
        raise ValueError(f"stencil size {n} exceeds node count {total}")
    idx = device_nodes(nodeset).knn(n, rows=np.array([center], dtype=np.int32)).cpu().numpy()[0].astype(np.int64)
    method = "mon" if n == MON_SIZE[nodeset.dim] and nodeset.kind[center] == KIND_REGULAR else "rbffd"
    return StencilSpec(center, idx, method)


def _single(stencil, positions, op, mon: bool) -> WeightRow:
    nb = np.asarray(stencil.neighbors, dtype=np.int64)
    pts = np.asarray(positions, float)[nb][None]
    kappa = float(_kappa(np.asarray(positions, float), nb[None], mon)[0])
    if not np.isfinite(kappa):
        kind = "MON" if mon else "RBF-FD"
        raise SingularSystemError(f"singular {kind} system (duplicate nodes?)", kappa)
    _, w = _solve_points(pts, [op], mon)  # local ids 0..n-1 are the stencil order
    order = np.argsort(nb)
    return WeightRow(nb[order], {op: w[0, 0][order]}, kappa)


def mon_weights(stencil: StencilSpec, positions: np.ndarray, op) -> WeightRow:
    """Monomial collocation weights for one stencil and one operator (approx.py:293-299)."""
    return _single(stencil, positions, op, True)


def rbf_fd_weights(stencil: StencilSpec, positions: np.ndarray, op) -> WeightRow:
    """PHS + monomial RBF-FD weights for one stencil and one operator (approx.py:302-308)."""
    return _single(stencil, positions, op, False)


class WeightTable:
    """Per-node stencil indices and weights (approx.py:311-329), resident in HBM.

    The host arrays (indices (N, n_max) -1 padded, sizes, weights {op: (N, n_max)},
    method, kappa) are materialised from the device bins on first access; assigning a
    field detaches the table from its device copy so edits are honoured downstream.
    """

    def __init__(self, indices=None, sizes=None, weights=None, method=None, kappa=None, _device=None):
        self._dev = _device
        self._indices, self._sizes, self._weights = indices, sizes, weights
        self._method = method
        self.kappa = kappa

    def _materialize(self):
        if self._indices is None and self._dev is not None:
            self._indices, self._sizes, self._weights = self._dev.host_arrays()

    def _detach(self):
        self._materialize()
        _ = self.method
        self._dev = None

    @property
    def indices(self):
        self._materialize()
        return self._indices

    @indices.setter
    def indices(self, v):
        self._detach()
        self._indices = v

    @property
    def sizes(self):
        if self._sizes is None and self._dev is not None:
            self._sizes = self._dev.sizes()
        return self._sizes

    @sizes.setter
    def sizes(self, v):
        self._detach()
        self._sizes = v

    @property
    def weights(self):
        self._materialize()
        return self._weights

    @weights.setter
    def weights(self, v):
        self._detach()
        self._weights = v

    @property
    def method(self):
        if self._method is None and self._dev is not None:
            self._method = self._dev.method
        return self._method

    @method.setter
    def method(self, v):
        self._method = v

    @property
    def ops(self):
        return self._dev.ops if self._dev is not None else list(self._weights.keys())

    def device_table(self, dim: int) -> DeviceTable:
        """The HBM bins (rebuilt from the host arrays if the table was edited)."""
        if self._dev is None:
            self._dev = DeviceTable.from_host(np.asarray(self._indices), np.asarray(self._sizes),
                                              self._weights, list(self._weights.keys()), dim)
            self._dev.method = self._method
        return self._dev

    def row(self, i: int) -> WeightRow:
        m = self.sizes[i]
        w = {op: tab[i, :m].copy() for op, tab in self.weights.items()}
        return WeightRow(self.indices[i, :m].copy(), w,
                         float(self.kappa[i]) if self.kappa is not None else float("nan"))


def classify_methods(nodeset, tree=None) -> np.ndarray:
    """METHOD_MON / METHOD_RBFFD per interior node, METHOD_NONE on boundary (approx.py:332-357)."""
    dn = device_nodes(nodeset)
    lat, lidx = getattr(nodeset, "lattice", None), getattr(nodeset, "lattice_idx", None)
    method = dn.classify().cpu().numpy().astype(np.int8)
    if lat is None or lidx is None:
        # no lattice map: probe +-h e_a with a 1-NN query (approx.py:124-130)
        regular = np.nonzero(np.asarray(nodeset.kind) == KIND_REGULAR)[0]
        if len(regular):
            dim = nodeset.dim
            h = np.asarray(nodeset.spacing)[regular]
            pos = np.asarray(nodeset.positions)[regular]
            eye = np.concatenate([np.eye(dim), -np.eye(dim)])
            probes = (pos[:, None, :] + h[:, None, None] * eye[None]).reshape(-1, dim)
            _, dist = dn.knn(1, points=probes, with_dist=True)
            ok = np.all(dist.cpu().numpy()[:, 0].reshape(len(regular), 2 * dim) < 1e-9 * h[:, None], axis=1)
            method[regular[ok]] = METHOD_MON
    return method


def _interior_device_table(nodeset, ops, n_rbf: int | None = None, host_copy: bool = False) -> DeviceTable:
    """classify -> device partition [MON | RBF | NONE] -> stencils -> solves, all in HBM;
    one 12-byte read-back (the class sizes) and one deferred singular check."""
    dim = nodeset.dim
    n = len(nodeset)
    n_rbf = RBF_SIZE[dim] if n_rbf is None else n_rbf
    dn = device_nodes(nodeset)
    t = L.torch()
    has_lattice = getattr(nodeset, "lattice", None) is not None and getattr(nodeset, "lattice_idx", None) is not None
    if has_lattice or not np.any(np.asarray(nodeset.kind) == KIND_REGULAR):
        method_d = dn.classify()
    else:  # probe path without a lattice map (approx.py:352-356)
        method_d = L.to_device(classify_methods(nodeset))
    rows_d = L.empty(max(n, 1), t.int32)
    counts_d = L.empty(3, t.int32)
    scratch = L.empty(3 * (n // 256 + 1) + 1, t.int32)
    L.call("hn_partition_methods", L.ptr(method_d), n, L.ptr(rows_d), L.ptr(counts_d), L.ptr(scratch),
           L.stream_handle())
    kind = np.asarray(nodeset.kind)
    if not np.any(kind == KIND_REGULAR):
        # no regular node: every interior node is RBF-FD (approx.py:346-350), so the class
        # sizes are known here and the device partition runs without a read-back
        k_rbf = int(np.count_nonzero(kind != KIND_BOUNDARY))
        k_mon, k_none = 0, n - k_rbf
    else:
        k_mon, k_rbf, k_none = (int(v) for v in counts_d.cpu().numpy())
    bins, pending = [], []
    if k_mon:
        d_rows = rows_d[:k_mon]
        st = dn.mon_stencils(d_rows) if has_lattice else dn.knn(MON_SIZE[dim], rows=d_rows)
        pending.append(_solve_bin(dn, st, d_rows, ops, True))
    if k_rbf:
        if n_rbf > n:
            raise ValueError(f"stencil size {n_rbf} exceeds node count {n}")
        d_rows = rows_d[k_mon:k_mon + k_rbf]
        pending.append(_solve_bin(dn, dn.knn(n_rbf, rows=d_rows, fine=True), d_rows, ops, False))
    bins = [b for b, _ in pending]
    if k_none:
        d_rows = rows_d[k_mon + k_rbf:n]
        bins.append(Bin(None, 0, L.empty((0, k_none), t.int32), L.empty((len(ops), 0, k_none), t.float64),
                        d_rows=d_rows, K=k_none))
    dev = DeviceTable(n, dim, list(ops), bins, n_rbf, method_d[:n])
    if host_copy:
        dev.start_host_copy()  # the result D2H completes under the flag read below
    _check_info(pending)
    return dev


_COPY_STREAMS: dict = {}


def _copy_stream():
    t = L.torch()
    dev = t.cuda.current_device()
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = t.cuda.Stream()
    return _COPY_STREAMS[dev]


NATIVE_CHUNKS = 8  # RBF chunks of the native pipeline's overlapped copy-back


def _native_ok(nodeset, ops, n_rbf: int | None = None) -> bool:
    """hn_weights_pipeline covers the lattice / no-regular-node cases with a tuned RBF size."""
    dim = nodeset.dim
    n_rbf = RBF_SIZE[dim] if n_rbf is None else n_rbf
    has_lattice = getattr(nodeset, "lattice", None) is not None and getattr(nodeset, "lattice_idx", None) is not None
    return (has_lattice or not np.any(np.asarray(nodeset.kind) == KIND_REGULAR)) and len(nodeset) >= n_rbf and \
        L.lib().hn_weights_rbf_is_tuned(dim, n_rbf, len(list(ops))) == 0


def _interior_native(nodeset, ops, n_rbf: int | None = None, host_copy: bool = True) -> DeviceTable:
    """The public orchestration as one native call (hn_weights_pipeline): classify ->
    partition -> MON stencils + solves -> kNN + RBF-FD solves, plus (host_copy) the padded
    WeightTable layout and its overlapped copy into pinned host memory.  host_copy=False
    keeps the ELL bins in HBM (operator assembly)."""
    dim = nodeset.dim
    n = len(nodeset)
    n_rbf = RBF_SIZE[dim] if n_rbf is None else n_rbf
    nops = len(ops)
    dn = device_nodes(nodeset)
    t = L.torch()
    g = dn.grid(dn.fine_cell) if dn.fine_cell is not None else dn.grid(dn.cell, exact=True)
    kind = np.asarray(nodeset.kind)
    # no regular node: the RBF rows are the non-boundary nodes, ascending -- only their count
    # and the chunk cut ids are needed, from the (few) boundary ids
    bnd = np.flatnonzero(kind == KIND_BOUNDARY) if not np.any(kind == KIND_REGULAR) else None
    k_rbf_host = n - len(bnd) if bnd is not None else -1
    has_lat = dn.lattice_grid is not None
    nmon = 2 * dim + 1
    cap_mon = n if k_rbf_host < 0 else 1  # no regular node -> no MON rows
    cap_rbf = n
    # three device pools + two pinned pools (allocation count is this call's host cost)
    i32_sizes = [max(n, 1), 3, 3 * (n // 256 + 1) + 1, nmon * cap_mon, nmon * cap_mon, cap_mon,
                 n_rbf * cap_rbf, n_rbf * cap_rbf, cap_rbf, 4]
    pool_i = L.empty(sum(i32_sizes), t.int32)
    rows, counts, scratch, mon_st, mon_idx, mon_info, rbf_st, rbf_idx, rbf_info, summary = \
        t.split(pool_i, i32_sizes)
    tab = nops * max(n, 1) * n_rbf if host_copy else 0
    pool_f = L.empty(nops * nmon * cap_mon + nops * n_rbf * cap_rbf + tab, t.float64)
    mon_w, rbf_w, d_w = t.split(pool_f, [nops * nmon * cap_mon, nops * n_rbf * cap_rbf, tab])
    method = L.empty(max(n, 1), t.int8)
    h_small = t.empty(16 + max(n, 1), dtype=t.int8, pin_memory=True)  # 4 int32 summary + method
    h_sum, h_m = h_small[:16].view(t.int32), h_small[16:]
    d_idx = d_sizes = h_idx = h_sizes = h_w = None
    if host_copy:
        pool_l = L.empty(max(n, 1) * (n_rbf + 1), t.int64)
        d_idx, d_sizes = pool_l[: max(n, 1) * n_rbf], pool_l[max(n, 1) * n_rbf:]
        h_l = t.empty(max(n, 1) * (n_rbf + 1), dtype=t.int64, pin_memory=True)
        h_w = t.empty((nops, max(n, 1), n_rbf), dtype=t.float64, pin_memory=True)
        h_idx, h_sizes = h_l[: max(n, 1) * n_rbf].view(max(n, 1), n_rbf), h_l[max(n, 1) * n_rbf:]
    kinds, axes, normals = _op_args(ops, dim)
    cnt = (L.C.c_int64 * 3)()
    # node-ordered RBF chunks: each chunk's table slice is copied back while the next computes
    chunks = NATIVE_CHUNKS if (k_rbf_host != 0 and host_copy) else 1
    cut = None
    if bnd is not None and chunks > 1 and k_rbf_host > 0:
        kb = (k_rbf_host * np.arange(1, chunks)) // chunks
        # id of the kb-th non-boundary node = kb + #{boundary ids b_j with b_j - j <= kb}
        cut = L.host_i64(kb + np.searchsorted(bnd - np.arange(len(bnd)), kb, side="right"))
    L.call("hn_weights_pipeline", L.ptr(dn.pos), dim, n, L.ptr(dn.kind), L.ptr(dn.lattice_idx if has_lat else None),
           L.ptr(dn.lattice_grid if has_lat else None), L.host_ints(dn.grid_dims if has_lat else [1, 1, 1]),
           L.host_dbls(dn.lo), g.cell, L.host_ints(g.dims), L.ptr(g.start), L.ptr(g.items), L.ptr(g.pos),
           L.ptr(dn.spacing), nops, kinds, axes, normals, n_rbf, 0, k_rbf_host, L.ptr(method), L.ptr(rows),
           L.ptr(counts), L.ptr(scratch), L.ptr(mon_st), L.ptr(mon_idx), L.ptr(mon_w), L.ptr(mon_info),
           L.ptr(rbf_st), L.ptr(rbf_idx), L.ptr(rbf_w), L.ptr(rbf_info), L.ptr(d_idx), L.ptr(d_sizes), L.ptr(d_w),
           L.ptr(h_idx), L.ptr(h_sizes), L.ptr(h_w), L.ptr(h_m), cnt, L.ptr(summary), L.ptr(h_sum),
           chunks, cut, L.stream_handle())
    k_mon, k_rbf, k_none = int(cnt[0]), int(cnt[1]), int(cnt[2])
    chunks = max(1, min(chunks, k_rbf, 64)) if k_rbf else 1
    kb = [(k_rbf * c) // chunks for c in range(chunks + 1)]
    if host_copy:
        L.TRAFFIC["d2h"] += h_idx.nbytes + h_sizes.nbytes + h_w.nbytes + n + 16
    bins = []
    if k_mon:
        b = Bin(None, nmon, mon_idx[: nmon * k_mon].view(nmon, k_mon),
                mon_w[: nops * nmon * k_mon].view(nops, nmon, k_mon), d_rows=rows[:k_mon], K=k_mon)
        b.mon = True
        bins.append(b)
    for c in range(chunks if k_rbf else 0):  # one ELL bin per chunk (DeviceTable.compact merges them)
        k0, kc = kb[c], kb[c + 1] - kb[c]
        if not kc:
            continue
        b = Bin(None, n_rbf, rbf_idx[n_rbf * k0: n_rbf * (k0 + kc)].view(n_rbf, kc),
                rbf_w[nops * n_rbf * k0: nops * n_rbf * (k0 + kc)].view(nops, n_rbf, kc),
                d_rows=rows[k_mon + k0:k_mon + k0 + kc], K=kc)
        b.mon = False
        bins.append(b)
    if k_none:
        bins.append(Bin(None, 0, L.empty((0, k_none), t.int32), L.empty((nops, 0, k_none), t.float64),
                        d_rows=rows[k_mon + k_rbf:n], K=k_none))
    dev = DeviceTable(n, dim, list(ops), bins, n_rbf, method[:n])
    if host_copy:
        dev._pending = (h_idx, h_sizes, h_w, h_m, (d_idx, d_sizes, d_w.view(nops, max(n, 1), n_rbf)))
    t.cuda.current_stream().synchronize()  # the one synchronisation (flags + table copies)
    hs = h_sum.numpy()
    for cnt_, first, kind_, off in ((hs[0], hs[1], "MON", 0), (hs[2], hs[3], "RBF-FD saddle", k_mon)):
        if cnt_:
            node = int(rows[off + int(first)].item())
            raise SingularSystemError(f"singular {kind_} system: Singular matrix ({int(cnt_)} stencil(s), first at "
                                      f"node {node})")
    return dev


class WeightsPipeline:
    """The public orchestration (hn_weights_pipeline, as compute_weights calls it) for a fixed
    node set with the class sizes frozen from one eager pass: no read-back, no host copy, the
    bins stay in HBM -- so one step is host-sync-free and can be replayed as a CUDA graph
    (bench.py's device-resident `value`).  `check()` verifies the frozen sizes and the
    singular flags after replays."""

    def __init__(self, nodeset, ops, rbf_n: int | None = None):
        from ._device import DeviceNodes
        t = L.torch()
        self.ops = list(ops)
        self.dim = dim = nodeset.dim
        self.n = n = len(nodeset)
        self.n_rbf = RBF_SIZE[dim] if rbf_n is None else rbf_n
        if not _native_ok(nodeset, self.ops, self.n_rbf):
            raise NotImplementedError("WeightsPipeline needs the native orchestration (lattice map or no regular "
                                      "node, tuned RBF size)")
        self.dn = dn = DeviceNodes(nodeset)
        self.method = L.empty(max(n, 1), t.int8)
        self.rows = L.empty(max(n, 1), t.int32)
        self.counts = L.empty(3, t.int32)
        self.part_scratch = L.empty(3 * (n // 256 + 1) + 1, t.int32)
        self.gq = dn.grid(dn.fine_cell) if dn.fine_cell is not None else dn.grid(dn.cell, exact=True)
        s = L.stream_handle()  # eager classification: the frozen class sizes
        L.call("hn_classify", L.ptr(dn.kind), L.ptr(dn.lattice_idx), L.ptr(dn.lattice_grid),
               L.host_ints(dn.grid_dims if dn.lattice_grid is not None else [1, 1, 1]), n, dim, L.ptr(self.method),
               s)
        L.call("hn_partition_methods", L.ptr(self.method), n, L.ptr(self.rows), L.ptr(self.counts),
               L.ptr(self.part_scratch), s)
        self.k_mon, self.k_rbf, self.k_none = (int(v) for v in self.counts.cpu().numpy())
        if self.k_rbf and self.n_rbf > n:
            raise ValueError(f"stencil size {self.n_rbf} exceeds node count {n}")
        nops = len(self.ops)
        km, kr = max(self.k_mon, 1), max(self.k_rbf, 1)
        nmon = 2 * dim + 1
        self.mon_st = L.empty((km, nmon), t.int32)
        self.rbf_st = L.empty((kr, self.n_rbf), t.int32)
        self.mon_idx, self.mon_w = L.empty((nmon, km), t.int32), L.empty((nops, nmon, km), t.float64)
        self.rbf_idx, self.rbf_w = L.empty((self.n_rbf, kr), t.int32), L.empty((nops, self.n_rbf, kr), t.float64)
        self.mon_info, self.rbf_info = L.zeros(km, t.int32), L.zeros(kr, t.int32)
        self._args = _op_args(self.ops, dim)
        self._cnt = (L.C.c_int64 * 3)()
        self.graph = None

    def run(self):
        """The whole step, launched on the current stream, no host synchronisation."""
        dn, g = self.dn, self.gq
        dn.build_grid(g)  # the cell list the RBF-FD queries search (K1)
        has_lat = dn.lattice_grid is not None
        kinds, axes, normals = self._args
        L.call("hn_weights_pipeline", L.ptr(dn.pos), self.dim, self.n, L.ptr(dn.kind),
               L.ptr(dn.lattice_idx if has_lat else None), L.ptr(dn.lattice_grid if has_lat else None),
               L.host_ints(dn.grid_dims if has_lat else [1, 1, 1]), L.host_dbls(dn.lo), g.cell, L.host_ints(g.dims),
               L.ptr(g.start), L.ptr(g.items), L.ptr(g.pos), L.ptr(dn.spacing), len(self.ops), kinds, axes, normals,
               self.n_rbf, self.k_mon, self.k_rbf, L.ptr(self.method), L.ptr(self.rows), L.ptr(self.counts),
               L.ptr(self.part_scratch), L.ptr(self.mon_st), L.ptr(self.mon_idx), L.ptr(self.mon_w),
               L.ptr(self.mon_info), L.ptr(self.rbf_st), L.ptr(self.rbf_idx), L.ptr(self.rbf_w),
               L.ptr(self.rbf_info), None, None, None, None, None, None, None, self._cnt, None, None,
               1, None, L.stream_handle())

    def capture(self):
        t = L.torch()
        self.run()  # warm every code path on the capture stream's device
        t.cuda.synchronize()
        self.graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self.graph):
            self.run()
        return self

    def replay(self):
        self.graph.replay()

    def check(self):
        """Frozen sizes still hold and no stencil was singular (one read-back)."""
        t = L.torch()
        flags = t.stack([self.counts.to(t.int64)[0], self.counts.to(t.int64)[1],
                         t.count_nonzero(self.mon_info[: self.k_mon]), t.count_nonzero(self.rbf_info[: self.k_rbf])])
        k_mon, k_rbf, bad_mon, bad_rbf = (int(v) for v in flags.cpu().numpy())
        if (k_mon, k_rbf) != (self.k_mon, self.k_rbf):
            raise RuntimeError("node classification changed under a frozen WeightsPipeline")
        if bad_mon or bad_rbf:
            raise SingularSystemError(f"singular systems: {bad_mon} MON, {bad_rbf} RBF-FD")

    def table(self) -> DeviceTable:
        t = L.torch()
        bins = []
        nmon = 2 * self.dim + 1
        if self.k_mon:
            bins.append(Bin(None, nmon, self.mon_idx[:, : self.k_mon], self.mon_w[:, :, : self.k_mon],
                            d_rows=self.rows[: self.k_mon], K=self.k_mon))
        if self.k_rbf:
            bins.append(Bin(None, self.n_rbf, self.rbf_idx[:, : self.k_rbf], self.rbf_w[:, :, : self.k_rbf],
                            d_rows=self.rows[self.k_mon: self.k_mon + self.k_rbf], K=self.k_rbf))
        if self.k_none:
            bins.append(Bin(None, 0, L.empty((0, self.k_none), t.int32), L.empty((len(self.ops), 0, self.k_none),
                                                                                  t.float64),
                            d_rows=self.rows[self.k_mon + self.k_rbf: self.n], K=self.k_none))
        return DeviceTable(self.n, self.dim, self.ops, bins, self.n_rbf, self.method[: self.n])


def compute_weights(nodeset, ops, with_kappa: bool = False, tree=None, rbf_n: int | None = None) -> WeightTable:
    """Stencils and weights for every interior node, batched per method (approx.py:379-413).

    `rbf_n` (extension) overrides RBF_SIZE[d] for this call, as the reference allows by
    rebinding its module constant.  The host arrays are copied back under the
    call's one synchronisation; operator assembly (solver.build_operators) uses
    _compute_weights(host_copy=False) and keeps the table in HBM."""
    return _compute_weights(nodeset, ops, with_kappa, rbf_n, host_copy=True)



def _compute_weights(nodeset, ops, with_kappa: bool = False, rbf_n: int | None = None,
                     host_copy: bool = False) -> WeightTable:
    ops = list(ops)
    for op in ops:
        _op_code(op, nodeset.dim)
    if _native_ok(nodeset, ops, rbf_n):  # the native orchestration (lattice or no regular node, tuned size)
        dev = _interior_native(nodeset, ops, rbf_n, host_copy=host_copy)
    else:  # the same library calls driven stage by stage (host-probed classes, untuned sizes)
        dev = _interior_device_table(nodeset, ops, rbf_n, host_copy=host_copy)
    table = WeightTable(_device=dev)
    if with_kappa:
        kappa = np.full(len(nodeset), np.nan)
        dn = device_nodes(nodeset)
        for b in dev.bins:
            if b.width == 0 or b.K == 0:
                continue
            mon = b.width == MON_SIZE[nodeset.dim] and bool(np.all(dev.method[b.rows_host] == METHOD_MON))
            if (nodeset.dim, b.width, mon) in _KAPPA_SIZES:  # on the device, straight from the ELL bin
                kappa[b.rows_host] = _kappa_bin(dn, b.d_idx, 1, b.K, b.d_rows, b.K, b.width, mon).cpu().numpy()
            else:
                idx = table.indices[b.rows_host, : b.width]
                kappa[b.rows_host] = _kappa_host(np.asarray(nodeset.positions, float),
                                                 _stencil_order(b.rows_host, idx), mon)
        table.kappa = kappa
    return table


def _stencil_order(rows, idx_sorted):
    """Centre first (kappa is invariant to the order of the other nodes)."""
    out = np.empty_like(idx_sorted)
    for r, (row, ids) in enumerate(zip(rows, idx_sorted)):
        out[r] = np.concatenate([[row], ids[ids != row]])
    return out


def _boundary_stencils(nodeset, rows: np.ndarray, exclude: np.ndarray | None):
    """[self] + nearest allowed nodes (exclude given) or plain kNN (approx.py:416-434).

    Returns (device stencils, tie_rows): tie_rows are the requested rows whose
    (size-1)-th and size-th allowed candidates tie exactly in distance -- where the
    reference keeps cKDTree's traversal choice instead of the (distance, index) rule
    (SURVEY §8(a) A5)."""
    t = L.torch()
    dim = nodeset.dim
    size = RBF_SIZE[dim]
    dn = device_nodes(nodeset)
    d_rows = L.to_device(rows.astype(np.int32))
    if exclude is None:
        if size > len(nodeset):
            raise ValueError(f"stencil size {size} exceeds node count {len(nodeset)}")
        return dn.knn(size, rows=d_rows), np.empty(0, dtype=np.int64)
    exclude = np.asarray(exclude, dtype=bool)
    if not np.all(exclude[rows]):
        raise ValueError("exclude mask must cover the requested rows")
    allowed = int((~exclude).sum())
    k = min(allowed, size - 1)
    kq = min(allowed, k + 1)
    idx, dist = dn.knn(kq, rows=d_rows, exclude=exclude.astype(np.uint8), with_dist=True)
    tie_rows = np.empty(0, dtype=np.int64)
    if kq > k and len(rows):
        dd = dist.cpu().numpy()
        tie_rows = rows[dd[:, k - 1] == dd[:, k]]
    st = t.cat([d_rows.view(-1, 1), idx[:, :k]], dim=1).contiguous()
    return st, tie_rows


def _boundary_table(nodeset, rows, exclude, ops, normals: bool, override=None) -> tuple[DeviceTable, np.ndarray]:
    rows = np.asarray(rows, dtype=np.int64)
    n = len(nodeset)
    dim = nodeset.dim
    dn = device_nodes(nodeset)
    bins = []
    ties = np.empty(0, dtype=np.int64)
    size = RBF_SIZE[dim]
    if len(rows):
        order = np.argsort(rows, kind="stable")
        rows_sorted = rows[order]
        st, ties = _boundary_stencils(nodeset, rows_sorted, exclude)
        size = int(st.shape[1])
        if override is not None:
            # explicit stencils for chosen rows (e.g. the reference's cKDTree choice on the
            # exact-tie rows of SURVEY §8(a) A5), given as (rows, (k, size) stencils)
            o_rows, o_st = np.asarray(override[0], dtype=np.int64), np.asarray(override[1])
            pos = np.searchsorted(rows_sorted, o_rows)
            if len(o_rows) and (np.any(pos >= len(rows_sorted)) or np.any(rows_sorted[pos] != o_rows)):
                raise ValueError("override rows must be among the requested rows")
            if len(o_rows):
                st[L.to_device(pos.astype(np.int64))] = L.to_device(o_st.astype(np.int32))
        rn = np.asarray(nodeset.normals, float)[rows_sorted] if normals else None
        b, info = _solve_bin(dn, st, L.to_device(rows_sorted.astype(np.int32)), ops, False, row_normals=rn)
        b._rows_host = rows_sorted
        _check_info([(b, info)])
        bins.append(b)
    rest = np.setdiff1d(np.arange(n), rows)
    if len(rest):
        t = L.torch()
        bins.append(Bin(rest, 0, L.empty((0, len(rest)), t.int32), L.empty((len(ops), 0, len(rest)), t.float64)))
    method = np.full(n, METHOD_NONE, dtype=np.int8)
    method[rows] = METHOD_RBFFD
    return DeviceTable(n, dim, list(ops), bins, size, method), ties


def normal_derivative_table(nodeset, rows: np.ndarray, tree=None, exclude: np.ndarray | None = None) -> WeightTable:
    """One-sided RBF-FD normal-derivative rows at boundary nodes (approx.py:437-465)."""
    dim = nodeset.dim
    dev, ties = _boundary_table(nodeset, rows, exclude, [NormalDerivative((0.0,) * dim)], True)
    dev.ops = ["normal"]
    t = WeightTable(method=dev.method, _device=dev)
    t.tie_rows = ties
    return t


def boundary_partial_table(nodeset, rows: np.ndarray, tree=None, exclude: np.ndarray | None = None,
                           stencil_override=None) -> WeightTable:
    """One-sided RBF-FD first-derivative rows at boundary nodes, all axes (approx.py:468-491).

    `stencil_override=(rows, stencils)` (extension) fixes the stencils of chosen rows;
    `table.tie_rows` lists rows whose (d, idx) choice may differ from cKDTree's."""
    ops = [Partial(a) for a in range(nodeset.dim)]
    dev, ties = _boundary_table(nodeset, rows, exclude, ops, False, stencil_override)
    t = WeightTable(method=dev.method, _device=dev)
    t.tie_rows = ties
    return t
