"""Device-resident forms of the hot-path data (HBM layout).

* DeviceNodes  -- padded AoS positions (stride 2 in 2D, 4 in 3D), kind, lattice map and
                  the uniform cell list; one per NodeSet, cached.
* Bin          -- one ELL slab of rows sharing a stencil width: rows[K], idx[W][K],
                  w[op][W][K] (column-major so a warp of rows reads each column coalesced).
* DeviceTable  -- the bins of one weight table (MON / RBF / boundary), with the host
                  WeightTable arrays produced on demand.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _lib as L

INT32_MIN = np.iinfo(np.int32).min
ELL_WIDTHS = (0, 5, 7, 12, 20, 30)


def _pos_stride(dim: int) -> int:
    return 2 if dim == 2 else 4


def pad_positions(positions: np.ndarray) -> np.ndarray:
    n, d = positions.shape
    out = np.zeros((n, _pos_stride(d)))
    out[:, :d] = positions
    return out


class DeviceNodes:
    """Device copy of a node set plus its cell list (replaces cKDTree, approx.py:386)."""

    def __init__(self, nodeset):
        t = L.torch()
        pos = np.asarray(nodeset.positions, dtype=float)
        self.n, self.dim = pos.shape
        if self.dim not in (2, 3):
            raise ValueError("node sets must be 2D or 3D")
        self.stride = _pos_stride(self.dim)
        # raw host arrays go up as they are (pinned DMA); padding, dtype narrowing and the
        # bounding box / mean scattered spacing are computed on the device, with one small
        # read-back -- the host-side numpy passes cost ~25 ms at N = 1e6
        kind_h = np.asarray(nodeset.kind, dtype=np.int8)
        spacing = getattr(nodeset, "spacing", None)
        up = [pos, kind_h] + ([np.asarray(spacing, dtype=float)] if spacing is not None else [])
        got = L.to_device_many(up)  # one pinned staging buffer, one DMA
        raw, self.kind = got[0], got[1]
        self.spacing = got[2] if spacing is not None else None  # per-node spacing: kNN first radius
        if self.stride == self.dim:
            self.pos = raw
        else:
            self.pos = L.zeros((self.n, self.stride), t.float64)
            self.pos[:, : self.dim] = raw
        self.lattice_grid = self.lattice_idx = None
        self.grid_dims = None
        lat = getattr(nodeset, "lattice", None)
        lidx = getattr(nodeset, "lattice_idx", None)
        if lat is not None and lidx is not None:
            grid = np.asarray(lat.grid)
            self.grid_dims = list(grid.shape)
            g_d, li = L.to_device_many([grid, np.asarray(lidx)])
            self.lattice_grid = g_d.to(t.int32)
            if li.dtype == t.int64:
                li = t.where(li == np.iinfo(np.int64).min, INT32_MIN, li)
            self.lattice_idx = li.to(t.int32).contiguous()
        if self.n:
            # bounding box + mean scattered spacing in one kernel pass, one small read-back
            st_d = L.empty(2 * self.dim + 2, t.float64)
            scratch = L.empty(8, t.int64)
            L.call("hn_node_stats", L.ptr(raw), self.n, self.dim, L.ptr(self.kind), L.ptr(self.spacing),
                   L.ptr(st_d), L.ptr(scratch), L.stream_handle())
            st = st_d.cpu().numpy()
            lo, hi = st[: self.dim], st[self.dim: 2 * self.dim]
            mean_h = st[2 * self.dim] / st[2 * self.dim + 1] if self.spacing is not None and st[-1] > 0 else None
        else:
            lo, hi, mean_h = np.zeros(self.dim), np.ones(self.dim), None
        # uniform cell list: ~1 node per cell in 2D, ~2 in 3D
        self.lo, self.hi = lo.astype(float), hi.astype(float)
        ext = np.maximum(hi - lo, 1e-300)
        vol = float(np.prod(ext))
        cell = (vol / max(self.n, 1)) ** (1.0 / self.dim) * (1.0 if self.dim == 2 else 1.25)
        if not np.isfinite(cell) or cell <= 0:
            cell = float(np.max(ext)) or 1.0
        self._grids = {}
        g = self.grid(cell, exact=True)
        self.cell, self.dims = g.cell, g.dims
        self.cell_start, self.cell_items, self.cell_pos = g.start, g.items, g.pos
        # graded sets: queries on the finest nodes get a grid sized to their own spacing
        self.fine_cell = None
        if mean_h is not None:
            fine = float(mean_h) * (1.0 if self.dim == 2 else 1.25)
            if fine < 0.7 * self.cell:
                self.fine_cell = fine

    class _Grid:
        pass

    def grid(self, cell: float, exact: bool = False):
        """Uniform cell list with (about) the requested cell size; built once, cached."""
        t = L.torch()
        ext = np.maximum(self.hi - self.lo, 1e-300)
        dims = [int(np.floor(ext[a] / cell)) + 1 for a in range(self.dim)]
        while int(np.prod(dims)) > 8 * max(self.n, 1) + 64:
            cell *= 1.25
            dims = [int(np.floor(ext[a] / cell)) + 1 for a in range(self.dim)]
        key = round(float(cell), 15)
        if key in self._grids:
            return self._grids[key]
        g = DeviceNodes._Grid()
        g.cell, g.dims = float(cell), dims
        ncells = int(np.prod(dims))
        g.start = L.empty(ncells + 1, t.int32)
        g.items = L.empty(max(self.n, 1), t.int32)
        g.pos = L.empty((max(self.n, 1), self.stride), t.float64)
        g.scratch = L.empty(ncells, t.int32)
        g.scratch2 = L.empty(max(self.n, 1), t.int32)
        self.build_grid(g)
        self._grids[key] = g
        return g

    def build_grid(self, g):
        """(Re)build a cell list from the resident positions (K1)."""
        L.call("hn_celllist_build", L.ptr(self.pos), self.n, self.dim, L.host_dbls(self.lo), g.cell,
               L.host_ints(g.dims), L.ptr(g.start), L.ptr(g.items), L.ptr(g.pos), L.ptr(g.scratch),
               L.ptr(g.scratch2), L.stream_handle())

    def knn(self, n: int, rows=None, points: np.ndarray | None = None, exclude=None, with_dist: bool = False,
            fine: bool = False):
        """n nearest nodes by (fl-distance, index) for node ids `rows` or query `points`.
        fine=True: the queries sit on the finest (scattered) nodes -> use their grid.
        Any grid gives the same (exact) answer; the choice only changes the work."""
        t = L.torch()
        g = self.grid(self.fine_cell) if (fine and self.fine_cell is not None) else self.grid(self.cell, exact=True)
        qpos = None
        if points is not None:
            pts = np.atleast_2d(np.asarray(points, float))
            nq = len(pts)
            qpos = L.to_device(pad_positions(pts))
            q = None
        elif rows is None:
            nq = self.n
            q = None
        else:
            q = rows if hasattr(rows, "data_ptr") else L.to_device(np.asarray(rows, dtype=np.int32))
            nq = int(q.numel())
        out = L.empty((max(nq, 1), n), t.int32)
        dist = L.empty((max(nq, 1), n), t.float64) if with_dist else None
        ex = None
        if exclude is not None:
            ex = exclude if hasattr(exclude, "data_ptr") else L.to_device(np.asarray(exclude, dtype=np.uint8))
        if nq and qpos is None and self.spacing is not None:
            L.call("hn_knn_spacing", L.ptr(self.pos), self.dim, L.host_dbls(self.lo), g.cell, L.host_ints(g.dims),
                   L.ptr(g.start), L.ptr(g.items), L.ptr(g.pos), L.ptr(q), None,
                   nq, n, L.ptr(ex), L.ptr(self.spacing), L.ptr(out), L.ptr(dist), L.stream_handle())
        elif nq:
            L.call("hn_knn", L.ptr(self.pos), self.dim, L.host_dbls(self.lo), g.cell, L.host_ints(g.dims),
                   L.ptr(g.start), L.ptr(g.items), L.ptr(g.pos), L.ptr(q), L.ptr(qpos),
                   nq, n, L.ptr(ex), L.ptr(out), L.ptr(dist), L.stream_handle())
        out = out[:nq]
        return (out, dist[:nq]) if with_dist else out

    def classify(self):
        t = L.torch()
        method = L.empty(max(self.n, 1), t.int8)
        has_lat = self.lattice_grid is not None
        L.call("hn_classify", L.ptr(self.kind), L.ptr(self.lattice_idx if has_lat else None),
               L.ptr(self.lattice_grid if has_lat else None),
               L.host_ints(self.grid_dims if has_lat else [1, 1, 1]), self.n, self.dim, L.ptr(method),
               L.stream_handle())
        return method[: self.n]

    def mon_stencils(self, rows):
        t = L.torch()
        k = int(rows.numel())
        out = L.empty((max(k, 1), 2 * self.dim + 1), t.int32)
        if k:
            L.call("hn_mon_stencils", L.ptr(rows), k, L.ptr(self.pos), L.ptr(self.lattice_idx),
                   L.ptr(self.lattice_grid), L.host_ints(self.grid_dims), self.dim, L.ptr(out), L.stream_handle())
        return out[:k]


_NODE_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _node_key(nodeset):
    """Identity of everything DeviceNodes snapshots (positions, kind, spacing, lattice map)
    plus a strided fingerprint of the positions, so replaced arrays and most in-place edits
    rebuild the device copy.  Node sets are treated as immutable inputs, as the reference's
    per-call cKDTree implies; edit a copy (or a new NodeSet) to be sure."""
    pos = nodeset.positions
    lat = getattr(nodeset, "lattice", None)
    arrays = (pos, getattr(nodeset, "kind", None), getattr(nodeset, "spacing", None),
              getattr(nodeset, "lattice_idx", None), getattr(lat, "grid", None))
    flat = np.asarray(pos).reshape(-1)
    step = max(1, flat.size // 4096)
    return (tuple(id(a) for a in arrays), tuple(getattr(a, "shape", None) for a in arrays),
            flat[::step].tobytes())


def device_nodes(nodeset) -> DeviceNodes:
    """Cached DeviceNodes for a node set (rebuilt when _node_key changes)."""
    key = _node_key(nodeset)
    try:
        ent = _NODE_CACHE.get(nodeset)
    except TypeError:
        ent = None
    if ent is not None and ent[0] == key:
        return ent[2]
    dn = DeviceNodes(nodeset)
    try:
        _NODE_CACHE[nodeset] = (key, None, dn)
    except TypeError:
        pass
    return dn


class Bin:
    """ELL slab: K rows of stencil width W and n_ops weight planes (device)."""

    def __init__(self, rows_host, width: int, d_idx, d_w, d_rows=None, K: int | None = None):
        self._rows_host = None if rows_host is None else np.asarray(rows_host, dtype=np.int64)
        self.K = int(K) if K is not None else len(self._rows_host)
        self.width = int(width)
        self.d_rows = d_rows if d_rows is not None else L.to_device(self._rows_host.astype(np.int32))
        self.d_idx = d_idx  # (W, K) int32
        self.d_w = d_w      # (nops, W, K) fp64

    @property
    def rows_host(self) -> np.ndarray:
        """Node ids of the bin's rows (copied from HBM on first use)."""
        if self._rows_host is None:
            self._rows_host = self.d_rows[: self.K].cpu().numpy().astype(np.int64)
        return self._rows_host


def bins_args(bins):
    """ctypes argument block (nbins, K[], W[], rows*[], idx*[], w*[]) for the ELL kernels."""
    live = [b for b in bins if b.K > 0]
    return (len(live), L.host_i64([b.K for b in live]), L.host_ints([b.width for b in live]),
            L.host_ptrs([b.d_rows for b in live]), L.host_ptrs([b.d_idx for b in live]),
            L.host_ptrs([b.d_w for b in live]), live)


class DeviceTable:
    """All bins of one weight table (rows of every node appear in exactly one bin)."""

    def __init__(self, n: int, dim: int, ops: list, bins: list, n_max: int, method=None):
        self.n, self.dim, self.ops, self.bins, self.n_max = n, dim, list(ops), bins, n_max
        self._method = method  # host array, or a device tensor copied on first use

    @property
    def method(self):
        if self._method is not None and hasattr(self._method, "is_cuda"):
            self._method = self._method.cpu().numpy().astype(np.int8)
        return self._method

    @method.setter
    def method(self, v):
        self._method = v

    @property
    def ell_ok(self) -> bool:
        if len([b for b in self.bins if b.K]) > 4:
            self.compact()
        return all(b.width in ELL_WIDTHS for b in self.bins) and len([b for b in self.bins if b.K]) <= 4

    def compact(self):
        """Merge bins of equal width (e.g. the row chunks of compute_weights' overlapped
        copy-back) into one ELL slab each: rows, idx and weights concatenated along K."""
        t = L.torch()
        by_w = {}
        for b in self.bins:
            by_w.setdefault(b.width, []).append(b)
        merged = []
        for w, group in by_w.items():
            group = [b for b in group if b.K] or group[:1]
            if len(group) == 1:
                merged.append(group[0])
                continue
            K = sum(b.K for b in group)
            rows = t.cat([b.d_rows[: b.K] for b in group])
            idx = t.cat([b.d_idx[:, : b.K] for b in group], dim=1).contiguous()
            wts = t.cat([b.d_w[:, :, : b.K] for b in group], dim=2).contiguous()
            nb = Bin(None, w, idx, wts, d_rows=rows, K=K)
            nb.mon = getattr(group[0], "mon", False)
            merged.append(nb)
        self.bins = merged

    def sizes(self) -> np.ndarray:
        s = np.zeros(self.n, dtype=np.int64)
        for b in self.bins:
            s[b.rows_host] = b.width
        return s

    def start_host_copy(self):
        """Enqueue the WeightTable layout (hn_ell_to_table) and its D2H into pinned memory on
        the current stream, without waiting: compute_weights issues this before its one
        synchronising read (the singular flags), so the copy rides on that sync."""
        if getattr(self, "_pending", None) is not None or getattr(self, "_pinned", None) is not None:
            return
        t = L.torch()
        n, m, nops = self.n, self.n_max, len(self.ops)
        d_idx = L.empty((max(n, 1), m), t.int64)
        d_sizes = L.zeros(max(n, 1), t.int64)
        d_w = L.empty((nops, max(n, 1), m), t.float64)
        nb, K, W, R, I, Wt, live = bins_args(self.bins)
        if nb:
            L.call("hn_ell_to_table", nb, K, W, R, I, Wt, nops, m, n, L.ptr(d_idx), L.ptr(d_sizes), L.ptr(d_w),
                   L.stream_handle())
        h_idx = t.empty(d_idx.shape, dtype=t.int64, pin_memory=True)
        h_sizes = t.empty(d_sizes.shape, dtype=t.int64, pin_memory=True)
        h_w = t.empty(d_w.shape, dtype=t.float64, pin_memory=True)
        h_idx.copy_(d_idx, non_blocking=True)
        h_sizes.copy_(d_sizes, non_blocking=True)
        h_w.copy_(d_w, non_blocking=True)
        h_m = None
        if self._method is not None and hasattr(self._method, "is_cuda"):
            h_m = t.empty(self._method.shape, dtype=self._method.dtype, pin_memory=True)
            h_m.copy_(self._method, non_blocking=True)
        L.TRAFFIC["d2h"] += h_idx.nbytes + h_sizes.nbytes + h_w.nbytes + (h_m.nbytes if h_m is not None else 0)
        self._pending = (h_idx, h_sizes, h_w, h_m, (d_idx, d_sizes, d_w))

    def host_arrays(self):
        """(indices (N, n_max) int64 -1 padded, sizes, {op: (N, n_max)}) -- the WeightTable
        layout, produced on the device (hn_ell_to_table) and copied once into pinned memory."""
        t = L.torch()
        self.start_host_copy()
        if self._pending is not None:
            t.cuda.current_stream().synchronize()
            h_idx, h_sizes, h_w, h_m, _ = self._pending
            self._pending = None
            self._pinned = (h_idx, h_sizes, h_w)  # numpy views below keep these alive via this table
            if h_m is not None:
                self._method = h_m.numpy().astype(np.int8)
        h_idx, h_sizes, h_w = self._pinned
        n = self.n
        w_np = h_w.numpy()
        weights = {op: w_np[j, :n] for j, op in enumerate(self.ops)}
        return h_idx.numpy()[:n], h_sizes.numpy()[:n], weights

    @staticmethod
    def from_host(indices: np.ndarray, sizes: np.ndarray, weights: dict, ops: list, dim: int) -> "DeviceTable":
        """Bins from WeightTable arrays (rows grouped by stencil size)."""
        t = L.torch()
        n, n_max = indices.shape
        bins = []
        for w in np.unique(sizes):
            rows = np.nonzero(sizes == w)[0]
            w = int(w)
            if w == 0:
                bins.append(Bin(rows, 0, L.empty((0, len(rows)), t.int32), L.empty((len(ops), 0, len(rows)), t.float64)))
                continue
            idx = np.ascontiguousarray(indices[rows, :w].T.astype(np.int32))
            wt = np.stack([np.ascontiguousarray(weights[op][rows, :w].T) for op in ops])
            bins.append(Bin(rows, w, L.to_device(idx), L.to_device(wt)))
        return DeviceTable(n, dim, ops, bins, n_max)
