"""Global sparse operators applied on the GPU (drop-in for hybridnodes.operators).

Reference: pkg/src/hybridnodes/operators.py.  `SparseOperator.matrix` stays a scipy CSR
(callers and tests read it), but `apply` never touches it: operators assembled from a
weight table run the binned ELL kernel (hn_apply_ell) on the table's HBM bins, any other
matrix runs the sequential CSR kernel (hn_csr_matvec).  Both reproduce scipy's
csr_matvec bit for bit.  Inputs may be numpy arrays (copied in and out) or
CUDA tensors (results stay on the device).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy import sparse

from . import _lib as L
from ._device import bins_args


@dataclass
class FieldState:
    """Velocity, pressure and temperature over all nodes (operators.py:14-31)."""

    velocity: np.ndarray
    pressure: np.ndarray
    temperature: np.ndarray

    @staticmethod
    def zeros(n: int, dim: int) -> "FieldState":
        return FieldState(np.zeros((n, dim)), np.zeros(n), np.zeros(n))

    def copy(self) -> "FieldState":
        return FieldState(self.velocity.copy(), self.pressure.copy(), self.temperature.copy())

    def finite(self) -> bool:
        return bool(np.all(np.isfinite(self.velocity)) and np.all(np.isfinite(self.pressure))
                    and np.all(np.isfinite(self.temperature)))


def _is_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


class DeviceCSR:
    """A scipy CSR matrix mirrored in HBM (int64 row pointers, int32 columns)."""

    def __init__(self, m):
        m = sparse.csr_matrix(m)
        self.shape = m.shape
        self.nnz = m.nnz
        self.rowptr = L.to_device(np.asarray(m.indptr, dtype=np.int64))
        self.cols = L.to_device(np.asarray(m.indices, dtype=np.int32))
        self.vals = L.to_device(np.asarray(m.data, dtype=np.float64))

    def matvec(self, x, y):
        L.call("hn_csr_matvec", L.ptr(self.rowptr), L.ptr(self.cols), L.ptr(self.vals), L.ptr(x), self.shape[0],
               L.ptr(y), L.stream_handle())
        return y

    def residual(self, x, b, y):
        L.call("hn_csr_residual", L.ptr(self.rowptr), L.ptr(self.cols), L.ptr(self.vals), L.ptr(x), L.ptr(b),
               self.shape[0], L.ptr(y), L.stream_handle())
        return y


class SparseOperator:
    """Row-compressed operator; row i holds node i's stencil weights (operators.py:34-58)."""

    def __init__(self, matrix, kind, row_sizes: np.ndarray, _table=None, _plane: int | None = None):
        self._matrix = matrix
        self.kind = kind
        self.row_sizes = row_sizes
        self._table = _table      # DeviceTable (ELL bins) when assembled from weights
        self._plane = _plane
        self._csr = None

    @property
    def matrix(self):
        if self._matrix is None:
            self._matrix = _table_csr(self._table, self._plane)
        return self._matrix

    @matrix.setter
    def matrix(self, m):
        self._matrix = m
        self._table = None
        self._csr = None

    @property
    def shape(self):
        if self._matrix is None and self._table is not None:
            return (self._table.n, self._table.n)
        return self.matrix.shape

    def _apply_device(self, f, out):
        if self._table is not None and self._table.ell_ok:
            nb, K, W, R, I, Wt, _ = bins_args(self._table.bins)
            L.call("hn_apply_ell", nb, K, W, R, I, Wt, 1, L.host_ints([self._plane]), L.ptr(f), L.ptr(out),
                   out.numel(), L.stream_handle())
        else:
            if self._csr is None:
                self._csr = DeviceCSR(self.matrix)
            self._csr.matvec(f, out)
        return out

    def apply(self, field):
        n_cols = self.shape[1]
        if field.shape[0] != n_cols:
            raise ValueError(f"field length {field.shape[0]} != N {n_cols}")
        t = L.torch()
        if _is_cuda(field):
            f = field.to(t.float64).contiguous()
            out = L.empty(self.shape[0], t.float64)
            return self._apply_device(f, out)
        f = L.to_device(np.asarray(field, dtype=np.float64))
        out = L.empty(self.shape[0], t.float64)
        return self._apply_device(f, out).cpu().numpy()

    def row(self, i: int):
        m = self.matrix
        sl = slice(m.indptr[i], m.indptr[i + 1])
        return m.indices[sl], m.data[sl]


def _table_csr(table, plane: int):
    """scipy CSR of one weight plane of a DeviceTable (host materialisation for the API)."""
    indices, sizes, weights = table.host_arrays()
    op = table.ops[plane]
    n = table.n
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(sizes, out=indptr[1:])
    cols = np.arange(indices.shape[1])[None, :] < sizes[:, None]
    return sparse.csr_matrix((weights[op][cols], indices[cols], indptr), shape=(n, n))


def assemble(nodeset, table, kind) -> SparseOperator:
    """One operator kind from a weight table, row order = node order (operators.py:61-77)."""
    ops = table.ops
    if kind not in ops:
        raise KeyError(f"weight table has no operator {kind!r}")
    sizes = np.asarray(table.sizes)
    missing = np.nonzero(np.asarray(nodeset.interior_mask) & (sizes == 0))[0]
    if len(missing):
        raise ValueError(f"missing weight row for interior node {int(missing[0])}")
    dev = table.device_table(nodeset.dim)
    return SparseOperator(None, kind, sizes.copy(), _table=dev, _plane=list(dev.ops).index(kind))


def apply(op: SparseOperator, field):
    """out_i = sum_j w_ij field_j (operators.py:80-82)."""
    return op.apply(field)


def divergence(partials, velocity):
    """Sum of axis-derivative applications over velocity components (operators.py:85-90).

    Accumulated on the device in the reference order ((D0 v0 + D1 v1) + D2 v2)."""
    t = L.torch()
    on_dev = _is_cuda(velocity)
    v = velocity.to(t.float64) if on_dev else L.to_device(np.asarray(velocity, dtype=np.float64))
    n = v.shape[0]
    out = partials[0].apply(v[:, 0].contiguous())
    for a in range(1, len(partials)):
        term = partials[a].apply(v[:, a].contiguous())
        L.call("hn_bicg_update", 1, L.ptr(out), L.ptr(term), None, 1.0, 0.0, n, L.stream_handle())
    return out if on_dev else out.cpu().numpy()
