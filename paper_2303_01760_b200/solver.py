"""Explicit-Euler natural-convection solver with Chorin projection, GPU-resident.

Drop-in for pkg/src/hybridnodes/solver.py: same dataclasses, OperatorSet attributes,
step functions and `run`.  Per step, everything runs in libhn.so on HBM-resident state:

  momentum_predict + apply_velocity_bc  -> hn_momentum            (K7)
  divergence / dt -> Poisson rhs        -> hn_div_rhs             (K8)
  pressure_solve (bicgstab + LU precond) -> hn_csr_residual/matvec, hn_sptrsv x2, hn_permute,
                                           hn_reduce, hn_bicg_update   (K9, scipy's algebra)
  velocity_correct + temperature_step   -> hn_correct_temperature (K10)
  apply_temperature_bc                  -> hn_temperature_bc      (K11)
  finite probe / Nusselt / divergence   -> flags + hn_reduce      (K12)

Setup (`build_operators`) computes every weight table on the GPU; the one-time algebra
that builds the bordered Poisson matrix and its complete LU factorisation stays on the
host with scipy/SuperLU, exactly as the reference does (solver.py:168-213) -- it is not
part of the per-step hot path.  The factors are then moved to HBM and
applied by sync-free triangular solves.
"""

from __future__ import annotations

import ctypes as C
import time
import weakref
from dataclasses import dataclass, field

import numpy as np
from scipy import sparse
from scipy.sparse import linalg as spla

from . import _lib as L
from ._device import bins_args
from .approx import (Laplacian, Partial, _compute_weights, boundary_partial_table, compute_weights,
                     normal_derivative_table)
from .errors import PoissonConvergenceError, SolverDivergenceError
from .nodegen import ROLE_DIRICHLET, ROLE_NEUMANN
from .operators import DeviceCSR, FieldState, SparseOperator, assemble

INT32_MAX = np.iinfo(np.int32).max


@dataclass
class PhysicsParams:
    Ra: float
    Pr: float
    g: np.ndarray = None
    t_ref: float = 0.0
    dissipation: float = 0.0

    def __post_init__(self):
        if self.Ra <= 0 or self.Pr <= 0:
            raise ValueError("Ra and Pr must be positive")
        if self.g is not None:
            self.g = np.asarray(self.g, dtype=float)
            if abs(np.linalg.norm(self.g) - 1.0) > 1e-12:
                raise ValueError("gravity direction must be a unit vector")

    def gravity(self, dim: int) -> np.ndarray:
        if self.g is not None:
            return self.g
        g = np.zeros(dim)
        g[-1] = -1.0
        return g


@dataclass
class TimeControls:
    dt: float
    t_end: float
    steady_tol: float = 1e-6
    nu_window: int = 40
    nu_stride: int = 20

    @staticmethod
    def from_spacing(h_min: float, t_end: float, Ra: float | None = None, **kwargs) -> "TimeControls":
        """dt = min(0.1 h_min^2 / 2, 40/Ra) (solver.py:60-73)."""
        dt = 0.1 * h_min ** 2 / 2.0
        if Ra is not None:
            dt = min(dt, 40.0 / Ra)
        return TimeControls(dt=dt, t_end=t_end, **kwargs)


@dataclass
class PoissonSolveSettings:
    tol: float = 1e-8
    maxiter: int = 2000
    gauge: int | None = None
    stabilization: float = 0.1

    def __post_init__(self):
        if not 0 < self.tol < 1:
            raise ValueError("relative tolerance must lie in (0, 1)")
        if not 0 <= self.stabilization <= 1:
            raise ValueError("stabilization must lie in [0, 1]")


_MAX_PAIRS = 512  # kSnMaxPairs (csrc/pressure.cu): (row, 256-entry chunk) pairs per task


def _split_by_chunks(outside: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    """Refine helper row ranges so no task has more than _MAX_PAIRS (row, chunk) pairs."""
    chunks = np.maximum(1, -(-outside // 256))
    out = [int(bounds[0])]
    for a, b in zip(bounds[:-1], bounds[1:]):
        a, b = int(a), int(b)
        while chunks[a:b].sum() > _MAX_PAIRS:
            if b - a == 1:
                raise ValueError("a factor row has more than 131,072 off-block entries")
            m = a + int(np.searchsorted(np.cumsum(chunks[a:b]), _MAX_PAIRS, side="right"))
            m = min(max(m, a + 1), b - 1)
            out.append(m)
            a = m
        out.append(b)
    return np.asarray(out)


def plan_supernodal_blocks(m: sparse.csr_matrix, lower: bool, cap: int = 256, helper_nnz: int = 4096,
                           batch: int = 8, batch_row_nnz: int = 32, rect: bool = True,
                           extra_outside: np.ndarray | None = None) -> dict:
    """Host planning of hn_sptrsv_super: dense-triangle row blocks in dependency-level order.
    Consecutive small blocks (w <= 32, every row's outside part <= batch_row_nnz) of one
    level are grouped `batch` to a task (kind 3, one warp each); heavy blocks get helper
    tasks (kind 1) for their outside sums.  rect: a block task whose rows all couple densely
    to the adjacent predecessor block (the pieces of one supernode cut at `cap`) takes those
    columns off its off-block sums and applies them itself from packed rectangle panels, tile
    by tile as the predecessor solves them (t_rw = the rectangle's width).  extra_outside: per
    row, off-block entries the device rows carry beyond `m` -- counted into the outside sums'
    work, not into the structure."""
    n = m.shape[0]
    rowptr = np.ascontiguousarray(m.indptr, dtype=np.int64)
    cols = np.ascontiguousarray(m.indices, dtype=np.int32)
    r0 = np.zeros(max(n, 1), dtype=np.int32)
    w = np.zeros(max(n, 1), dtype=np.int32)
    vp = L._vp
    nb = int(L.lib().hn_host_supernodes(rowptr.ctypes.data_as(vp), cols.ctypes.data_as(vp), n, 1 if lower else 0,
                                        cap, r0.ctypes.data_as(vp), w.ctypes.data_as(vp)))
    r0, w = r0[:nb].copy(), w[:nb].copy()
    lev = np.zeros(nb, dtype=np.int32)
    L.call("hn_host_block_levels", rowptr.ctypes.data_as(vp), cols.ctypes.data_as(vp), n, 1 if lower else 0, nb,
           r0.ctypes.data_as(vp), w.ctypes.data_as(vp), lev.ctypes.data_as(vp))
    order = np.lexsort((r0, lev))
    r0, w, lev = r0[order], w[order], lev[order]
    # heavy blocks: their outside sums go to helper tasks (kind 1) that run on other SMs,
    # the block itself (kind 2) only solves the dense triangle
    rowlen = np.diff(rowptr)
    owner_r0 = np.repeat(r0, w)
    owner_w = np.repeat(w, w)
    rows = np.concatenate([np.arange(a, a + b) for a, b in zip(r0, w)]) if nb else np.empty(0, np.int64)
    rr = rows - owner_r0
    inside = rr if lower else owner_w - 1 - rr
    outside = rowlen[rows] - inside
    starts = np.concatenate([[0], np.cumsum(w)[:-1]]) if nb else np.empty(0, np.int64)
    extra = np.asarray(extra_outside, dtype=outside.dtype)[rows] if extra_outside is not None and nb else 0
    block_maxout = np.maximum.reduceat(outside + extra, starts) if nb else np.empty(0)
    small = (w <= 32) & (block_maxout <= batch_row_nnz) if batch else np.zeros(nb, bool)
    rect_w = np.zeros(nb, dtype=np.int64)
    if rect and nb:
        by_r0 = {int(a): k for k, a in enumerate(r0)}
        by_end = {int(a) + int(b): k for k, (a, b) in enumerate(zip(r0, w))}
        for k in np.nonzero(~small)[0]:
            pk = by_end.get(int(r0[k])) if lower else by_r0.get(int(r0[k]) + int(w[k]))
            if pk is None:
                continue
            pw = int(w[pk])
            sl = slice(starts[k], starts[k] + w[k])
            rk, ins, outk = rows[sl], inside[sl], outside[sl]
            if (outk < pw).any():
                continue
            if lower:
                e_first, e_last, c_first = rowptr[rk + 1] - ins - pw, rowptr[rk + 1] - ins - 1, int(r0[pk])
            else:
                e_first, e_last, c_first = rowptr[rk] + ins, rowptr[rk] + ins + pw - 1, int(r0[k] + w[k])
            if (cols[e_first] == c_first).all() and (cols[e_last] == c_first + pw - 1).all():
                rect_w[k] = pw
                outside[sl] -= pw
    outside = outside + extra
    block_out = np.add.reduceat(outside, starts) if nb else np.empty(0)
    kinds, tr0, tw, trb, trc, trw = [], [], [], [], [], []
    members = []  # (r0, w) of batched small blocks, appended after the task list (kind 3)
    heavy = set(np.nonzero((block_out > helper_nnz) & (w > 1))[0].tolist())
    pending = []  # consecutive small blocks of one level -> one warp each

    def flush():
        if len(pending) == 1:
            k = pending[0]
            kinds.append(0); tr0.append(r0[k]); tw.append(w[k]); trb.append(0); trc.append(w[k]); trw.append(0)
        elif pending:
            kinds.append(3); tr0.append(0); tw.append(0); trb.append(len(members)); trc.append(len(pending))
            trw.append(0)
            members.extend((int(r0[k]), int(w[k])) for k in pending)
        pending.clear()

    for k in range(nb):
        if small[k] and k not in heavy:
            if pending and (lev[pending[0]] != lev[k] or len(pending) == batch):
                flush()
            pending.append(k)
            continue
        flush()
        if k in heavy:
            o = outside[starts[k]: starts[k] + w[k]]
            cut = np.searchsorted(np.cumsum(o), np.arange(1, int(np.ceil(o.sum() / helper_nnz))) * helper_nnz)
            bounds = np.unique(np.concatenate([[0], cut, [w[k]]]))
            bounds = _split_by_chunks(o, bounds)
            for a, b in zip(bounds[:-1], bounds[1:]):
                kinds.append(1); tr0.append(r0[k]); tw.append(w[k]); trb.append(a); trc.append(b - a)
                trw.append(rect_w[k])
            kinds.append(2); tr0.append(r0[k]); tw.append(w[k]); trb.append(0); trc.append(w[k]); trw.append(rect_w[k])
        else:
            o = outside[starts[k]: starts[k] + w[k]]
            if np.maximum(1, -(-o // 256)).sum() > _MAX_PAIRS:
                raise ValueError("a one-row block has more than 131,072 off-block entries")
            kinds.append(0); tr0.append(r0[k]); tw.append(w[k]); trb.append(0); trc.append(w[k]); trw.append(rect_w[k])
    flush()
    ntasks = len(kinds)
    for idx, (a, b) in enumerate(members):  # member entries: the kernel never tickets past ntasks
        kinds.append(4); tr0.append(a); tw.append(b); trb.append(0); trc.append(b); trw.append(0)
    trb = [v + ntasks if kd == 3 else v for kd, v in zip(kinds, trb)]
    as32 = lambda v: np.asarray(v, dtype=np.int32)  # noqa: E731
    return {"nblk": nb, "r0": r0, "w": w, "levels": lev, "depth": int(lev.max()) + 1 if nb else 0,
            "ntasks": ntasks, "kind": as32(kinds), "t_r0": as32(tr0), "t_w": as32(tw), "t_rb": as32(trb),
            "t_rc": as32(trc), "t_rw": as32(trw), "heavy": len(heavy), "batched": len(members),
            "rects": int((rect_w > 0).sum())}


def dense_group_runs(m: sparse.csr_matrix, lower_plan: dict, keep_levels: int, upper: sparse.csr_matrix | None = None,
                     max_bytes: float = 3e9):
    """Row runs at the top of the elimination tree: the rows of L's blocks at level >=
    keep_levels (everything above them is then `keep_levels` cheap levels deep), closed under
    both solves' dependencies (no other row of L reads a chosen row; a chosen row of U reads
    only chosen rows), as maximal contiguous ranges.  keep_levels rises until the runs' inverse
    triangles fit max_bytes.  Returns (starts, ends) or None."""
    n = m.shape[0]
    r0, w, lev = lower_plan["r0"], lower_plan["w"], lower_plan["levels"]
    depth = int(lower_plan["depth"])
    rows_l = np.repeat(np.arange(n), np.diff(m.indptr))
    rows_u = np.repeat(np.arange(n), np.diff(upper.indptr)) if upper is not None else None
    keep = int(keep_levels)
    while keep < depth:
        sel = lev >= keep
        chosen = np.zeros(n, dtype=bool)
        chosen[np.concatenate([np.arange(a, a + b) for a, b in zip(r0[sel], w[sel])])] = True
        for _ in range(64):  # closure (a fixed point in one or two rounds: the set is the tree's top)
            before = int(chosen.sum())
            chosen[rows_l[chosen[m.indices]]] = True            # a row of L reading a chosen column
            if upper is not None:
                chosen[upper.indices[chosen[rows_u]]] = True    # a column a chosen row of U reads
            if int(chosen.sum()) == before:
                break
        idx = np.nonzero(chosen)[0]
        if len(idx) == 0:
            return None
        brk = np.nonzero(np.diff(idx) > 1)[0]
        starts = np.concatenate([[idx[0]], idx[brk + 1]]).astype(np.int64)
        ends = np.concatenate([idx[brk] + 1, [idx[-1] + 1]]).astype(np.int64)
        if 4.0 * float(((ends - starts).astype(np.float64) ** 2).sum()) <= max_bytes and len(idx) <= n // 2:
            return starts, ends
        keep += max(1, (depth - keep) // 4)
    return None


def group_arrays(m: sparse.csr_matrix, g: dict, lower: bool) -> dict:
    """Host arrays of the dense groups (pure numpy): the coupling CSR over the chosen rows in
    (phase, row) order -- a row's entries outside its run are a prefix (L: columns < a) or a
    suffix (U: columns >= b) of its sorted CSR row -- and, per row, where its slice of the
    run's row-packed inverse triangle starts (g_off), how long it is (g_cnt) and which y entry
    its first column multiplies (g_ystart)."""
    rows, starts, ends, run_of = g["rows"], g["starts"], g["ends"], g["run_of"]
    n = m.shape[0]
    a_of, b_of = starts[run_of[rows]], ends[run_of[rows]]
    indptr = np.asarray(m.indptr, dtype=np.int64)
    cnt_out = np.zeros(len(rows), dtype=np.int64)
    e0 = np.zeros(len(rows), dtype=np.int64)
    for q, r in enumerate(rows):  # searchsorted in each chosen row (26 K rows at config 3)
        c = m.indices[indptr[r]: indptr[r + 1]]
        if lower:
            k = int(np.searchsorted(c, a_of[q], side="left"))
            cnt_out[q], e0[q] = k, indptr[r]
        else:
            k = int(np.searchsorted(c, b_of[q], side="left"))
            cnt_out[q], e0[q] = len(c) - k, indptr[r] + k
    cpl_ptr = np.concatenate([[0], np.cumsum(cnt_out)]).astype(np.int64)
    take = np.repeat(e0 - cpl_ptr[:-1], cnt_out) + np.arange(cpl_ptr[-1], dtype=np.int64)
    widths = (ends - starts)[g["order"]]
    tri = widths * (widths + 1) // 2
    run_off = np.zeros(len(starts), dtype=np.int64)
    run_off[g["order"]] = np.concatenate([[0], np.cumsum(tri)[:-1]])
    i = rows - a_of  # row inside its run
    wv = b_of - a_of
    if lower:
        g_off = run_off[run_of[rows]] + i * (i + 1) // 2
        g_cnt, g_ystart = i + 1, a_of
    else:
        g_off = run_off[run_of[rows]] + i * wv - i * (i - 1) // 2
        g_cnt, g_ystart = wv - i, rows
    return {"cpl_ptr": cpl_ptr, "cpl_cols": np.ascontiguousarray(m.indices[take], dtype=np.int32),
            "cpl_vals": np.ascontiguousarray(m.data[take], dtype=np.float64), "run_off": run_off,
            "inv_entries": int(tri.sum()), "g_off": g_off.astype(np.int64), "g_cnt": g_cnt.astype(np.int32),
            "g_ystart": g_ystart.astype(np.int32)}


def group_task_matrix(m: sparse.csr_matrix, chosen: np.ndarray) -> sparse.csr_matrix:
    """The task kernel's matrix once the groups took their rows: the chosen rows are empty
    (trivial tasks x = b / 1; for U the groups put their solution into b first, so the trivial
    task reproduces it).  The other rows of U keep their group columns: x of the groups is
    final before the tasks run.  (Moving those columns into a streaming product ahead of the
    tasks -- 23 M entries, 87 us -- was built and measured: the task kernel did not get
    shorter, U 0.837 -> 0.866 ms; dropped.)"""
    n = m.shape[0]
    ent_row = np.repeat(np.arange(n), np.diff(m.indptr))
    ent = ~chosen[ent_row]
    indptr = np.concatenate([[0], np.cumsum(np.bincount(ent_row[ent], minlength=n))]).astype(np.int64)
    return sparse.csr_matrix((m.data[ent], m.indices[ent], indptr), shape=m.shape)


def plan_groups(m: sparse.csr_matrix, groups, lower: bool, max_phases: int = 16):
    """Phases of the runs for one factor: a run's phase = 1 + the highest phase among the runs
    it reads (L: earlier rows, U: later rows); rows ordered by (phase, row)."""
    starts, ends = (np.asarray(v, dtype=np.int64) for v in groups)
    n, nr = m.shape[0], len(starts)
    if nr == 0:
        return None
    run_of = np.full(n, -1, dtype=np.int64)
    chosen = np.zeros(n, dtype=bool)
    for k, (a, b) in enumerate(zip(starts, ends)):
        run_of[a:b] = k
        chosen[a:b] = True
    phase = np.zeros(nr, dtype=np.int64)
    for k in (range(nr) if lower else range(nr - 1, -1, -1)):
        a, b = starts[k], ends[k]
        cols = m.indices[m.indptr[a]: m.indptr[b]]
        out = cols[cols < a] if lower else cols[cols >= b]
        deps = np.unique(run_of[out])
        deps = deps[deps >= 0]
        if len(deps):
            phase[k] = phase[deps].max() + 1
    if int(phase.max()) + 1 > max_phases:
        return None
    order = np.lexsort((starts, phase))
    rows = np.concatenate([np.arange(starts[k], ends[k]) for k in order])
    counts = np.bincount(phase, weights=(ends - starts).astype(float), minlength=int(phase.max()) + 1)
    return {"starts": starts, "ends": ends, "order": order, "phase": phase, "rows": rows, "chosen": chosen,
            "run_of": run_of, "phase_ptr": np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)}


class _SuperSchedule:
    """Device task list of one supernodal triangular solve: the planned tasks plus the packed
    dense triangles of the block tasks (hn_host_pack_panels), and optionally the dense groups:
    row runs at the top of the elimination tree that leave the task list and are solved
    through the explicit inverses of their triangles (csrc/pressure.cu, 'dense groups')."""

    MAX_PHASES = 16

    def __init__(self, m: sparse.csr_matrix, lower: bool, diag: np.ndarray | None = None, inverse: int = 0,
                 groups=None, **plan_kw):
        n = m.shape[0]
        self.n, self.lower = n, bool(lower)
        self.groups = None
        g = self._plan_groups(m, groups) if groups is not None else None
        dg = np.ascontiguousarray(diag if diag is not None else np.ones(1), dtype=np.float64)
        if g is not None:
            # the task kernel's matrix: the chosen rows are empty (trivial tasks x = b / 1; for U
            # the groups put their solution into b first, so the trivial task reproduces it)
            lead = group_task_matrix(m, g["chosen"])
            if diag is not None:
                dg = dg.copy()
                dg[g["chosen"]] = 1.0
        else:
            lead = m
        lead.sort_indices()
        plan = plan_supernodal_blocks(lead, lower, **plan_kw)
        self.csr = DeviceCSR(lead)
        self.inverse = int(inverse)  # 0 substitution, 1 diagonal-tile inverses, 2 whole-block inverses
        self.nblk, self.depth, self.ntasks = plan["nblk"], plan["depth"], plan["ntasks"]
        kind, r0, w, rw = plan["kind"], plan["t_r0"], plan["t_w"], plan["t_rw"]
        vp = L._vp
        rowptr = np.ascontiguousarray(lead.indptr, dtype=np.int64)
        cols = np.ascontiguousarray(lead.indices, dtype=np.int32)
        vals = np.ascontiguousarray(lead.data, dtype=np.float64)
        off = np.empty(len(kind), dtype=np.int64)
        args = (rowptr.ctypes.data_as(vp), cols.ctypes.data_as(vp), vals.ctypes.data_as(vp), dg.ctypes.data_as(vp),
                1 if lower else 0, int(inverse), self.ntasks, kind.ctypes.data_as(vp), r0.ctypes.data_as(vp),
                w.ctypes.data_as(vp), rw.ctypes.data_as(vp), off.ctypes.data_as(vp))
        total = int(L.lib().hn_host_pack_panels(*args, None))
        packed = np.empty(max(total, 2), dtype=np.float64)
        if int(L.lib().hn_host_pack_panels(*args, packed.ctypes.data_as(vp))) != total:
            raise RuntimeError("hn_host_pack_panels: a planned block's in-block triangle is not dense")
        off[self.ntasks:] = -1
        self.kind, self.r0, self.w = L.to_device(kind), L.to_device(r0), L.to_device(w)
        self.rb, self.rc = L.to_device(plan["t_rb"]), L.to_device(plan["t_rc"])
        self.off, self.packed = L.to_device(off), L.to_device(packed)
        self.rw = L.to_device(rw)
        self.rects = plan["rects"]
        self.packed_bytes = 8 * total
        self.nnz = int(lead.nnz)
        self.d_diag = L.to_device(dg) if diag is not None else None
        self.inv_entries = 0
        self.n_phases, self.group_rows = 0, 0
        phase_ptr = (C.c_int64 * 17)()
        gp = [None] * 9
        if g is not None:
            gp = self._upload_groups(m, g, diag) + [L.empty(n, L.torch().float64)]  # + the y scratch
            for k, v in enumerate(g["phase_ptr"]):
                phase_ptr[k] = int(v)
        self._plan = L.TriPlan(
            1 if lower else 0, self.inverse, self.ntasks, self.kind.data_ptr(), self.r0.data_ptr(),
            self.w.data_ptr(), self.rb.data_ptr(), self.rc.data_ptr(), self.off.data_ptr(), self.rw.data_ptr(),
            self.csr.rowptr.data_ptr(), self.csr.cols.data_ptr(), self.csr.vals.data_ptr(),
            self.d_diag.data_ptr() if self.d_diag is not None else None, self.packed.data_ptr(),
            self.n_phases, phase_ptr, *[t.data_ptr() if t is not None else None for t in gp])
        self._group_tensors = gp

    # ---- dense groups ----
    def _plan_groups(self, m, groups):
        return plan_groups(m, groups, self.lower, self.MAX_PHASES)

    def _upload_groups(self, m, g, diag):
        """Coupling CSR (the chosen rows' entries outside their run), the runs' inverse
        triangles (row-packed; one dense triangular solve per run on the device, setup only) and
        the per-row descriptors."""
        t = L.torch()
        lower = self.lower
        arr = group_arrays(m, g, lower)
        starts, ends = g["starts"], g["ends"]
        inv = L.empty(int(arr["inv_entries"]), t.float64)
        for k in g["order"]:
            a, b = int(starts[k]), int(ends[k])
            wk = b - a
            blk = np.asarray(m[a:b, a:b].todense(), dtype=np.float64)
            blk[np.diag_indices(wk)] = 1.0 if lower else np.asarray(diag, dtype=np.float64)[a:b]
            d_blk = L.to_device(blk)
            x = t.linalg.solve_triangular(d_blk, t.eye(wk, dtype=t.float64, device=d_blk.device), upper=not lower)
            mask = t.ones((wk, wk), dtype=t.bool, device=d_blk.device)
            mask = t.tril(mask) if lower else t.triu(mask)
            o = int(arr["run_off"][k])
            inv[o: o + wk * (wk + 1) // 2].copy_(x[mask])
            del d_blk, x, mask
        self.n_phases = len(g["phase_ptr"]) - 1
        self.group_rows = len(g["rows"])
        self.nnz += int(arr["cpl_ptr"][-1])
        self.inv_entries = int(arr["inv_entries"])
        self.groups = g
        return [L.to_device(g["rows"].astype(np.int32)), L.to_device(arr["cpl_ptr"]), L.to_device(arr["cpl_cols"]),
                L.to_device(arr["cpl_vals"]), L.to_device(arr["g_off"]), L.to_device(arr["g_cnt"]),
                L.to_device(arr["g_ystart"]), inv]

    def plan_struct(self):
        return self._plan


class _DeviceLU:
    """SuperLU factors Pr A Pc = L U in HBM: strict-lower L, strict-upper U + diag, perms,
    and the supernodal task lists of both solves."""

    CTAS_PER_SM = 2
    # diagonal 32-row tiles of the packed triangles applied as precomputed inverses (x = T^-1 y,
    # no substitution chain) for the L / U solve.  Config 3 (tools/ab_inverse.py): L 1.10 ->
    # 0.91 ms, U 1.27 -> 1.06 ms; the solve moves from 1.2e-11 to 1.1e-10 of SuperLU's (max
    # norm, random rhs) and the fields after 50 full steps by <= 1.1e-12 (relative).
    # (2 = whole-block inverses -- the packed panels hold the inverse of a block's entire dense
    # triangle, x = B^-1 y panel by panel with no tile-to-tile chain -- measured slower: L 0.726
    # -> 0.777 ms with a 4096-row dense tail, 5e-10 from SuperLU: a block's x is then published only
    # at its end, while the tile scheme feeds the next piece of a supernode tile by tile.)
    TILE_INVERSE_L = 1
    TILE_INVERSE_U = 1
    # dense groups: the rows of L's block levels >= KEEP_LEVELS (the top of the elimination tree:
    # separators, nearly dense supernodes that can only be solved one 256-wide piece after the
    # other) leave the task chain and are solved through explicit inverses, phase by phase
    # (csrc/pressure.cu).  Config 3 at 50: 12.4 K rows in 8 runs, 4 phases, L's 96 and U's 77 block
    # levels -> 50 and 44.  Measured L + U (tools/time_trisolve.py): none 1.913 ms, keep 60 1.509, 50
    # 1.469, 40 1.536, 30 1.573 (more rows = more inverse bytes and phases).  0 = off.
    KEEP_LEVELS = 50
    # max-norm relative distance to SuperLU's solve on a random rhs (tests): U is ill-conditioned
    # (block kappa up to 7e7), two exact substitution orders differ by ~6e-11; the diagonal-tile
    # inverses move it to ~1.1e-10 (fields: <= 1.1e-12 after 50 steps, see above)
    PARITY_TOL = {False: 1e-10, True: 1e-9}

    def __init__(self, lu, inverse: int | None = None, keep_levels: int | None = None, **plan_kw):
        Lm = sparse.csr_matrix(lu.L)
        Um = sparse.csr_matrix(lu.U)
        self.n = Lm.shape[0]
        Ls = sparse.tril(Lm, k=-1, format="csr")
        Us = sparse.triu(Um, k=1, format="csr")
        Ls.sort_indices()
        Us.sort_indices()
        udiag = np.asarray(Um.diagonal(), dtype=np.float64)
        keep = self.KEEP_LEVELS if keep_levels is None else int(keep_levels)
        groups = None
        if keep > 0:
            full = plan_supernodal_blocks(Ls, True, **plan_kw)
            if full["depth"] > keep + 4:
                groups = dense_group_runs(Ls, full, keep, upper=Us)
        self.sL = _SuperSchedule(Ls, lower=True, inverse=self.TILE_INVERSE_L if inverse is None else inverse,
                                 groups=groups, **plan_kw)
        self.sU = _SuperSchedule(Us, lower=False, diag=udiag, inverse=self.TILE_INVERSE_U if inverse is None else inverse,
                                 groups=groups, **plan_kw)
        self.group_rows = self.sL.group_rows
        self.L, self.U = self.sL.csr, self.sU.csr  # the rows the task kernels read
        self.diag = self.sU.d_diag
        self.perm_r = L.to_device(np.asarray(lu.perm_r, dtype=np.int32))
        self.perm_c = L.to_device(np.asarray(lu.perm_c, dtype=np.int32))
        t = L.torch()
        self.y = L.empty(self.n, t.float64)
        self.z = L.empty(self.n, t.float64)
        self.w = L.empty(self.n, t.float64)
        self.ticket = L.zeros(1, t.int64)
        self.ysum = L.empty(self.n, t.float64)
        self.nnz = int(Ls.nnz + Us.nnz + self.n)  # the factors as SuperLU holds them
        # bytes one application reads: 12 B per sparse entry the kernels touch (task rows and the
        # groups' coupling) + 8 B per entry of the groups' inverse triangles + the U diagonal
        self.solve_bytes = 12 * (self.sL.nnz + self.sU.nnz) + 8 * (self.sL.inv_entries + self.sU.inv_entries) \
            + 8 * self.n
        self.parity_tol = self.PARITY_TOL[bool(self.sL.inverse or self.sU.inverse or self.group_rows)]

    def plans(self):
        """(L, U) as hn_tri_plan structs for hn_pressure_setup (the arrays stay owned here)."""
        return self.sL.plan_struct(), self.sU.plan_struct()

    def solve(self, b, x):
        """x = Pc U^-1 L^-1 Pr b (scipy SuperLU.solve semantics)."""
        s = L.stream_handle()
        L.call("hn_permute", 0, L.ptr(self.perm_r), L.ptr(b), self.n, L.ptr(self.y), s)
        self._tri(self.sL, self.L, None, self.y, self.z, s)
        self._tri(self.sU, self.U, self.diag, self.z, self.w, s)
        L.call("hn_permute", 1, L.ptr(self.perm_c), L.ptr(self.w), self.n, L.ptr(x), s)
        return x

    def _tri(self, sch, m, diag, b, x, s):
        """One triangular solve (m and diag are the schedule's own arrays; kept in the signature
        for the dev tools).  The upper solve with dense groups overwrites the groups' entries of
        b with their solution (solve() passes its own scratch)."""
        L.call("hn_sptrsv_plan", C.byref(sch.plan_struct()), L.ptr(b), L.ptr(x), L.ptr(self.ysum), self.n,
               L.ptr(self.ticket), self.CTAS_PER_SM, s)


def _free_pressure(handle: int):
    try:
        L.lib().hn_pressure_free(handle)
    except Exception:  # interpreter shutdown
        pass


class _NativePressure:
    """The device-driven BiCGStab of the bordered Poisson system (hn_pressure_setup /
    hn_pressure_solve, csrc/bicgstab.cu): scipy's algorithm with every scalar on the device,
    the loop a CUDA-graph WHILE node; no host round trip per solve."""

    def __init__(self, A: "DeviceCSR", lu: _DeviceLU):
        pl, pu = lu.plans()
        h = C.c_int64(0)
        L.call("hn_pressure_setup", lu.n, L.ptr(A.rowptr), L.ptr(A.cols), L.ptr(A.vals), C.byref(pl), C.byref(pu),
               L.ptr(lu.perm_r), L.ptr(lu.perm_c), lu.CTAS_PER_SM, C.byref(h))
        self.handle = h.value
        self._keep = (A, lu)
        self._finalizer = weakref.finalize(self, _free_pressure, self.handle)

    def solve(self, b, x0, x, rtol: float, maxiter: int, status):
        """Enqueue one solve on the current stream: x0 None = zero start, x0 is x = warm start
        from x; status (device int32[2]) <- [scipy info, passes]."""
        L.call("hn_pressure_solve", self.handle, L.ptr(b), L.ptr(x0), L.ptr(x), float(rtol), int(maxiter),
               L.ptr(status), L.stream_handle())


class OperatorSet:
    """Assembled operators, boundary index sets and factorised helpers (solver.py:96-125),
    with their HBM mirrors."""

    def __init__(self, nodeset, lap, partials, gauge: int, poisson_matrix, poisson_precond, neumann_rows,
                 neumann_lu, nu_rows, cold_idx, nu_scale, lu=None, neumann_diag=None):
        self.nodeset = nodeset
        self.lap = lap
        self.partials = partials
        self.gauge = gauge
        self.poisson_matrix = poisson_matrix
        self.poisson_precond = poisson_precond
        self.neumann_lu = neumann_lu
        self.cold_idx = cold_idx
        self.nu_scale = nu_scale
        self._poisson_lambda = 0.0
        self.interior_idx = np.nonzero(nodeset.interior_mask)[0]
        self.boundary_idx = np.nonzero(nodeset.boundary_mask)[0]
        self.dirichlet_idx = np.nonzero(nodeset.role == ROLE_DIRICHLET)[0]
        self.neumann_idx = np.nonzero(nodeset.role == ROLE_NEUMANN)[0]
        self._w_neumann = neumann_rows
        self._nu_rows = nu_rows
        t = L.torch()
        n = len(nodeset)
        self.n = n
        # ---- HBM mirrors ----
        self._table = lap._table
        ops = list(self._table.ops)
        self._lap_plane = ops.index(lap.kind)
        self._d_planes = [ops.index(p.kind) for p in partials]
        self._d_poisson = DeviceCSR(poisson_matrix) if poisson_matrix is not None else None
        self._d_lu = _DeviceLU(lu) if lu is not None else None
        self._d_press = _NativePressure(self._d_poisson, self._d_lu) if self._d_lu is not None else None
        self._d_pstatus = L.zeros(2, t.int32)
        self._d_dir_idx = L.to_device(self.dirichlet_idx.astype(np.int32))
        self.dirichlet_values = nodeset.bc_value[self.dirichlet_idx]
        self._d_neu = None
        if neumann_rows is not None:
            self._d_neu = DeviceCSR(neumann_rows)
            self._d_neu_idx = L.to_device(self.neumann_idx.astype(np.int32))
            self._d_neu_diag = L.to_device(np.asarray(neumann_diag, dtype=np.float64))
            mask = np.zeros(n, dtype=np.uint8)
            mask[self.neumann_idx] = 1
            self._d_is_neu = L.to_device(mask)
        self._d_nu = DeviceCSR(nu_rows) if nu_rows is not None else None
        self._d_interior = L.to_device(self.interior_idx.astype(np.int32))
        self._red = L.empty(512, t.float64)
        self._scalar = L.empty(8, t.float64)

    @property
    def dim(self) -> int:
        return self.nodeset.dim

    @property
    def dirichlet_values(self):
        return self._dirichlet_values

    @dirichlet_values.setter
    def dirichlet_values(self, v):
        self._dirichlet_values = np.asarray(v, dtype=float)
        self._d_dir_val = L.to_device(self._dirichlet_values.astype(np.float64))

    # ---- device helpers ----
    def _bins(self):
        return bins_args(self._table.bins)

    def reduce(self, op: int, a, b=None, idx=None, n=None) -> float:
        n = int(a.numel()) if n is None and idx is None else (int(idx.numel()) if idx is not None else n)
        L.call("hn_reduce", op, L.ptr(a), L.ptr(b), L.ptr(idx), n, L.ptr(self._red), L.ptr(self._scalar),
               L.stream_handle())
        return float(self._scalar[0].item())


def _table_to_csr(table, key, n: int) -> sparse.csr_matrix:
    cols = np.arange(table.indices.shape[1])[None, :] < table.sizes[:, None]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(table.sizes, out=indptr[1:])
    return sparse.csr_matrix((table.weights[key][cols], table.indices[cols], indptr), shape=(n, n))


def build_operators(nodeset, cold_origins: set, settings: PoissonSolveSettings,
                    timings: dict | None = None, boundary_override=None, interior_rbf_n: int | None = None,
                    factorize: bool = True) -> OperatorSet:
    """Weights on the GPU, one-time host assembly + SuperLU, factors to HBM (solver.py:133-232).

    Extensions: `boundary_override=(rows, stencils)` pins chosen boundary-gradient
    stencils (SURVEY §8(a) A5 tie rows); `interior_rbf_n` sets the interior RBF-FD stencil
    size while the boundary tables keep RBF_SIZE (config 4: n = 20 inside, 30 at walls, H9);
    `factorize=False` skips the bordered Poisson matrix and its LU (explicit kernels only,
    e.g. config 4 at N = 1e6 where the reference's SuperLU treatment is infeasible, H8)."""
    timings = timings if timings is not None else {}
    dim = nodeset.dim
    n = len(nodeset)
    ops_wanted = [Laplacian()] + [Partial(a) for a in range(dim)]
    boundary_idx = np.nonzero(nodeset.boundary_mask)[0]
    neumann_idx = np.nonzero(nodeset.role == ROLE_NEUMANN)[0]
    cold_idx = np.array([i for i in boundary_idx if nodeset.origin[i] in cold_origins], dtype=np.int64)

    t0 = time.perf_counter()
    table = _compute_weights(nodeset, ops_wanted, rbf_n=interior_rbf_n)
    boundary_grad = boundary_partial_table(nodeset, boundary_idx, exclude=nodeset.boundary_mask,
                                           stencil_override=boundary_override)
    nu_table = normal_derivative_table(nodeset, cold_idx) if len(cold_idx) else None
    L.torch().cuda.synchronize()
    timings["weights"] = time.perf_counter() - t0

    t0 = time.perf_counter()
    lap = assemble(nodeset, table, Laplacian())
    partials = [assemble(nodeset, table, Partial(a)) for a in range(dim)]
    grad_rows = [_table_to_csr(boundary_grad, Partial(a), n) for a in range(dim)]
    normals_safe = np.where(np.isfinite(nodeset.normals), nodeset.normals, 0.0)
    normal_matrix = sum(sparse.diags(normals_safe[:, a]) @ grad_rows[a] for a in range(dim)).tocsr()

    interior = nodeset.interior_mask
    if settings.gauge is None:
        centroid = nodeset.positions[interior].mean(axis=0)
        cand = np.nonzero(interior)[0]
        gauge = int(cand[np.argmin(np.linalg.norm(nodeset.positions[cand] - centroid, axis=1))])
    else:
        gauge = int(settings.gauge)
    poisson = precond = lu = None
    if factorize:
        grad_full = [p.matrix + g for p, g in zip(partials, grad_rows)]
        div_grad = sum(p.matrix @ g for p, g in zip(partials, grad_full))
        beta = settings.stabilization
        blended = (1.0 - beta) * div_grad + beta * lap.matrix
        core = (sparse.diags(interior.astype(float)) @ blended
                + sparse.diags(nodeset.boundary_mask.astype(float)) @ normal_matrix).tocsr()
        core.eliminate_zeros()
        core = core.tocoo()
        n_int = int(interior.sum())
        rows = np.concatenate([core.row, np.nonzero(interior)[0], [n]])
        cols = np.concatenate([core.col, np.full(n_int, n), [gauge]])
        data = np.concatenate([core.data, np.ones(n_int), [1.0]])
        poisson = sparse.csr_matrix((data, (rows, cols)), shape=(n + 1, n + 1))
        lu = spla.splu(poisson.tocsc())
        precond = spla.LinearOperator(poisson.shape, lu.solve)

    neumann_rows = neumann_lu = neumann_diag = None
    if len(neumann_idx):
        neumann_rows = normal_matrix[neumann_idx]
        block = neumann_rows[:, neumann_idx].tocsr()
        off = block - sparse.diags(block.diagonal())
        off.eliminate_zeros()
        if off.nnz:
            raise NotImplementedError("Neumann reconstruction block is not diagonal; the GPU path solves it "
                                      "as an elementwise division (boundary stencils must exclude each other)")
        neumann_diag = block.diagonal()
        neumann_lu = spla.splu(block.tocsc())
    nu_rows = _table_to_csr(nu_table, "normal", n)[cold_idx] if nu_table is not None else None

    dirichlet_idx = np.nonzero(nodeset.role == ROLE_DIRICHLET)[0]
    values = nodeset.bc_value[dirichlet_idx]
    t_span = (values.max() - values.min()) if len(values) else 1.0
    nu_scale = float(np.max(nodeset.positions.max(axis=0) - nodeset.positions.min(axis=0)))
    nu_scale /= t_span if t_span > 0 else 1.0
    opset = OperatorSet(nodeset, lap, partials, gauge, poisson, precond, neumann_rows, neumann_lu, nu_rows,
                        cold_idx, nu_scale, lu=lu, neumann_diag=neumann_diag)
    opset.boundary_tie_rows = getattr(boundary_grad, "tie_rows", np.empty(0, dtype=np.int64))
    L.torch().cuda.synchronize()
    timings["solver_setup"] = time.perf_counter() - t0
    return opset


# ============================================================ device step pieces
def _lap2_dev(ops: OperatorSet, f, out):
    """out = lap(lap(f)) with the inner result's boundary rows at 0 (solver.py:245-247): two
    bit-exact ELL applies; boundary rows have empty stencils, so they already give 0."""
    t = L.torch()
    tmp = L.empty(ops.n, t.float64)
    nb, K, W, R, I, Wt, _ = ops._bins()
    sel = L.host_ints([ops._lap_plane])
    L.call("hn_apply_ell", nb, K, W, R, I, Wt, 1, sel, L.ptr(f), L.ptr(tmp), ops.n, L.stream_handle())
    L.call("hn_apply_ell", nb, K, W, R, I, Wt, 1, sel, L.ptr(tmp), L.ptr(out), ops.n, L.stream_handle())
    return out


def _hyper_coef(ops: OperatorSet, coeff: float):
    """-coeff * spacing**3, evaluated by numpy exactly as the reference does (cached in HBM)."""
    cache = ops.__dict__.setdefault("_hyper_cache", {})
    if coeff not in cache:
        cache[coeff] = L.to_device(-coeff * np.asarray(ops.nodeset.spacing, dtype=float) ** 3)
    return cache[coeff]


def _momentum_dev(ops: OperatorSet, params: PhysicsParams, dt: float, v_soa, T, out, zero_boundary: bool):
    dim = ops.dim
    g = params.gravity(dim)
    buoy = [params.Ra * params.Pr * g[c] for c in range(dim)]  # ((Ra*Pr)*g_c), solver.py:270
    hc = l2 = None
    if params.dissipation:  # hyper-dissipation (solver.py:235-247, 271-272)
        t = L.torch()
        hc = _hyper_coef(ops, float(params.dissipation))
        l2 = L.empty((dim, ops.n), t.float64)
        for c in range(dim):
            _lap2_dev(ops, v_soa[c], l2[c])
    nb, K, W, R, I, Wt, _ = ops._bins()
    L.call("hn_momentum", nb, K, W, R, I, Wt, ops._lap_plane, L.host_ints(ops._d_planes), dim, L.ptr(v_soa),
           L.ptr(T), ops.n, float(dt), float(params.Pr), float(params.t_ref), L.host_dbls(buoy),
           1 if zero_boundary else 0, L.ptr(hc), L.ptr(l2), L.ptr(out), L.stream_handle())
    return out


def _div_rhs_dev(ops: OperatorSet, vstar_soa, dt: float, rhs):
    nb, K, W, R, I, Wt, _ = ops._bins()
    L.call("hn_div_rhs", nb, K, W, R, I, Wt, L.host_ints(ops._d_planes), ops.dim, L.ptr(vstar_soa), ops.n,
           float(dt), L.ptr(rhs), L.stream_handle())
    return rhs


def _correct_temp_dev(ops: OperatorSet, vstar_soa, p, T, dt: float, vout, Tout, flags, dissipation: float = 0.0):
    hc = l2 = None
    if dissipation:  # hyper-dissipation of T with the corrected velocity's speed (solver.py:355-356)
        t = L.torch()
        hc = _hyper_coef(ops, float(dissipation))
        l2 = _lap2_dev(ops, T, L.empty(ops.n, t.float64))
    nb, K, W, R, I, Wt, _ = ops._bins()
    L.call("hn_correct_temperature", nb, K, W, R, I, Wt, ops._lap_plane, L.host_ints(ops._d_planes), ops.dim,
           L.ptr(vstar_soa), L.ptr(p), L.ptr(T), ops.n, float(dt), L.ptr(vout), L.ptr(Tout), L.ptr(flags),
           L.ptr(hc), L.ptr(l2), L.stream_handle())


def _temperature_bc_dev(ops: OperatorSet, T, flags=None, latch=None, pstatus=None):
    """K11 in one launch; with `latch` (and int32[3] flags) the end-of-step latch rides along."""
    nd = len(ops.dirichlet_idx)
    neu = ops._d_neu
    L.call("hn_temperature_bc", L.ptr(ops._d_dir_idx), L.ptr(ops._d_dir_val), nd,
           L.ptr(neu.rowptr if neu else None), L.ptr(neu.cols if neu else None), L.ptr(neu.vals if neu else None),
           L.ptr(ops._d_neu_idx if neu else None), L.ptr(ops._d_neu_diag if neu else None),
           L.ptr(ops._d_is_neu if neu else None), len(ops.neumann_idx) if neu else 0, L.ptr(T), L.ptr(flags),
           L.ptr(latch), L.ptr(pstatus), L.stream_handle())
    return T


class _GMRES:
    """Retry solver after a BiCGStab failure, standing in for scipy's lgmres (reference
    solver.py:306-312): restarted GMRES(m) with the same LU preconditioner (right
    preconditioning, modified Gram-Schmidt) and the same stopping rule
    ||b - A x|| <= rtol ||b||, on device vectors with libhn reductions and updates.  It only
    runs when BiCGStab reports a failure, so its host-side Hessenberg algebra is off the
    per-step path."""

    RESTART = 30

    def __init__(self, ops: OperatorSet):
        self.ops = ops
        self.n1 = ops.n + 1
        t = L.torch()
        m = self.RESTART
        self.V = L.empty((m + 1, self.n1), t.float64)
        self.Z = L.empty((m, self.n1), t.float64)
        self.w = L.empty(self.n1, t.float64)

    def _dot(self, a, b):
        return self.ops.reduce(0, a, b, n=self.n1)

    def _axpy(self, y, x, alpha):
        L.call("hn_bicg_update", 1, L.ptr(y), L.ptr(x), None, float(alpha), 0.0, self.n1, L.stream_handle())

    def solve(self, b, x0, rtol: float, maxiter: int):
        ops, m = self.ops, self.RESTART
        bnrm = float(np.sqrt(self._dot(b, b)))
        if not np.isfinite(bnrm):
            return x0, -1
        atol = float(rtol) * bnrm
        x = x0.clone() if x0 is not None else L.zeros(self.n1, L.torch().float64)
        if bnrm == 0:
            return x.zero_(), 0
        V, Z, w = self.V, self.Z, self.w
        for _ in range(max(1, maxiter)):
            ops._d_poisson.residual(x, b, w)
            beta = float(np.sqrt(self._dot(w, w)))
            if beta <= atol:
                return x, 0
            V[0].zero_()
            self._axpy(V[0], w, 1.0 / beta)
            H = np.zeros((m + 1, m))
            cs, sn = np.zeros(m), np.zeros(m)
            g = np.zeros(m + 1)
            g[0] = beta
            k = 0
            for j in range(m):
                ops._d_lu.solve(V[j], Z[j])
                ops._d_poisson.matvec(Z[j], w)
                for i in range(j + 1):
                    H[i, j] = self._dot(w, V[i])
                    self._axpy(w, V[i], -H[i, j])
                H[j + 1, j] = float(np.sqrt(self._dot(w, w)))
                if H[j + 1, j] > 0:
                    V[j + 1].zero_()
                    self._axpy(V[j + 1], w, 1.0 / H[j + 1, j])
                for i in range(j):  # apply the previous Givens rotations to column j
                    a, c = H[i, j], H[i + 1, j]
                    H[i, j], H[i + 1, j] = cs[i] * a + sn[i] * c, -sn[i] * a + cs[i] * c
                r = np.hypot(H[j, j], H[j + 1, j])
                cs[j], sn[j] = (H[j, j] / r, H[j + 1, j] / r) if r > 0 else (1.0, 0.0)
                H[j, j], H[j + 1, j] = r, 0.0
                g[j + 1] = -sn[j] * g[j]
                g[j] = cs[j] * g[j]
                k = j + 1
                if abs(g[j + 1]) <= atol or H[j + 1, j] == 0 and r == 0:
                    break
            y = np.linalg.lstsq(np.triu(H[:k, :k]), g[:k], rcond=None)[0]
            for i in range(k):
                self._axpy(x, Z[i], y[i])
        ops._d_poisson.residual(x, b, w)
        return x, (0 if float(np.sqrt(self._dot(w, w))) <= atol else maxiter)


def _pressure_dev(ops: OperatorSet, rhs, x0, settings: PoissonSolveSettings, x, status=None):
    """One checked pressure solve into x (device, n+1): the native BiCGStab, the status read
    back, and on failure the reference's retry (lgmres there, the GMRES stand-in here) from the
    same x0 before PoissonConvergenceError (solver.py:304-313).  x0 must not alias x."""
    if ops._d_press is None:
        raise RuntimeError("operators were built with factorize=False: no pressure solve available")
    status = ops._d_pstatus if status is None else status
    ops._d_press.solve(rhs, x0, x, settings.tol, settings.maxiter, status)
    info = int(status[0].item())
    if info != 0:
        retry = getattr(ops, "_gmres", None) or _GMRES(ops)
        ops._gmres = retry
        xr, info = retry.solve(rhs, x0, settings.tol, settings.maxiter)
        if info != 0:
            tt = L.torch()
            res_vec = L.empty(ops.n + 1, tt.float64)
            ops._d_poisson.residual(xr, rhs, res_vec)
            res = np.sqrt(ops.reduce(0, res_vec, res_vec)) / max(np.sqrt(ops.reduce(0, rhs, rhs)), 1e-300)
            raise PoissonConvergenceError(f"pressure Poisson solve did not converge (info={info})",
                                          residual=float(res))
        x.copy_(xr)
    return x


# ============================================================ public step functions (host arrays)
def _soa(v: np.ndarray):
    return L.to_device(np.ascontiguousarray(np.asarray(v, dtype=np.float64).T))


def momentum_predict(state: FieldState, ops: OperatorSet, params: PhysicsParams, dt: float) -> np.ndarray:
    """Intermediate velocity v* without the pressure gradient (solver.py:250-274)."""
    t = L.torch()
    v = _soa(state.velocity)
    T = L.to_device(np.asarray(state.temperature, dtype=np.float64))
    out = L.empty((ops.dim, ops.n), t.float64)
    _momentum_dev(ops, params, dt, v, T, out, zero_boundary=False)
    return out.cpu().numpy().T.copy()


def apply_velocity_bc(v: np.ndarray, ops: OperatorSet) -> np.ndarray:
    """No-slip on every boundary node (in place, solver.py:277-280)."""
    v[ops.boundary_idx] = 0.0
    return v


def pressure_solve(vstar: np.ndarray, ops: OperatorSet, settings: PoissonSolveSettings, dt: float,
                   x0: np.ndarray | None = None, wall_gradient: np.ndarray | None = None) -> np.ndarray:
    """Solve the bordered Poisson system for p (solver.py:283-314) on the GPU."""
    t = L.torch()
    n = ops.n
    rhs = L.empty(n + 1, t.float64)
    _div_rhs_dev(ops, _soa(vstar), dt, rhs)
    if wall_gradient is not None:
        bidx = L.to_device(ops.boundary_idx.astype(np.int64))
        rhs.index_copy_(0, bidx, L.to_device(np.broadcast_to(np.asarray(wall_gradient, float),
                                                             ops.boundary_idx.shape).copy()))
    x0d = None
    if x0 is not None:  # the reference appends the last lambda to an n-vector (solver.py:302-303)
        x0 = np.asarray(x0, dtype=np.float64)
        x0d = L.to_device(np.concatenate([x0, [ops._poisson_lambda]]) if len(x0) == n else x0)
    x = _pressure_dev(ops, rhs, x0d, settings, L.empty(n + 1, t.float64))
    p = x.cpu().numpy()
    ops._poisson_lambda = float(p[n])
    return p[:n].copy()


def velocity_correct(vstar: np.ndarray, p: np.ndarray, ops: OperatorSet, dt: float) -> np.ndarray:
    """v = v* - dt grad p inside, no-slip on boundaries (solver.py:317-331)."""
    t = L.torch()
    vout = L.empty((ops.dim, ops.n), t.float64)
    Tout = L.empty(ops.n, t.float64)
    flags = L.to_device(np.array([0, INT32_MAX], dtype=np.int32))
    zeros = L.zeros(ops.n, t.float64)
    _correct_temp_dev(ops, _soa(vstar), L.to_device(np.asarray(p, dtype=np.float64)), zeros, dt, vout, Tout, flags)
    return vout.cpu().numpy().T.copy()


def apply_temperature_bc(t_field: np.ndarray, ops: OperatorSet) -> np.ndarray:
    """Dirichlet values reset; insulated nodes solved from their Neumann rows (solver.py:334-342)."""
    T = L.to_device(np.asarray(t_field, dtype=np.float64))
    _temperature_bc_dev(ops, T)
    t_field[:] = T.cpu().numpy()
    return t_field


def temperature_step(state: FieldState, ops: OperatorSet, dt: float, dissipation: float = 0.0) -> np.ndarray:
    """T += dt * (-v . grad T + lap T) inside; boundary values re-imposed (solver.py:345-358)."""
    t = L.torch()
    v = _soa(state.velocity)
    T = L.to_device(np.asarray(state.temperature, dtype=np.float64))
    vout = L.empty((ops.dim, ops.n), t.float64)
    Tout = L.empty(ops.n, t.float64)
    flags = L.to_device(np.array([0, INT32_MAX], dtype=np.int32))
    zeros = L.zeros(ops.n, t.float64)
    # with p = 0 the fused kernel's corrected velocity is v itself (v - dt*0 = v)
    _correct_temp_dev(ops, v, zeros, T, dt, vout, Tout, flags, dissipation)
    _temperature_bc_dev(ops, Tout)
    return Tout.cpu().numpy()


def nusselt_average(state: FieldState, ops: OperatorSet) -> float:
    """Mean of L/(T_H - T_C) |dT/dn| over the cold-boundary nodes (solver.py:361-365)."""
    if ops._d_nu is None:
        return float("nan")
    T = L.to_device(np.asarray(state.temperature, dtype=np.float64))
    return _nusselt_dev(ops, T)


def _nusselt_dev(ops: OperatorSet, T) -> float:
    t = L.torch()
    m = ops._d_nu.shape[0]
    g = L.empty(m, t.float64)
    ops._d_nu.matvec(T, g)
    return float(ops.nu_scale * (ops.reduce(2, g, n=m) / m))


def interior_divergence(v: np.ndarray, ops: OperatorSet) -> float:
    t = L.torch()
    return _interior_divergence_dev(ops, _soa(v))


def _interior_divergence_dev(ops: OperatorSet, v_soa) -> float:
    t = L.torch()
    rhs = L.empty(ops.n + 1, t.float64)
    _div_rhs_dev(ops, v_soa, 1.0, rhs)  # div / 1.0 is exact
    return ops.reduce(1, rhs, idx=ops._d_interior)


# ============================================================ device-resident stepping
def _pinned_view(t, a: np.ndarray):
    """A torch view of a host array for an async DMA: the array itself when it lives in pinned
    memory, else a pinned staging copy (torch's caching host allocator)."""
    src = t.from_numpy(a)
    if src.is_pinned():
        return src
    stage = t.empty(src.shape, dtype=src.dtype, pin_memory=True)
    stage.copy_(src)
    return stage


class DeviceStepper:
    """One explicit step = K7 -> K8 -> K9 -> K10 -> K11 on HBM-resident state (replicates the
    loop body of run(), solver.py:439-452).

    After the first (eager) step every step is ONE CUDA-graph replay on the stepper's own
    stream: momentum, divergence, the device-driven BiCGStab (a WHILE node, warm-started from
    the previous [p, lambda] as the reference's x0), correction + temperature, boundary
    conditions and the end-of-step latch -- no host synchronisation.  The latch records the
    first non-finite step and the first step whose BiCGStab failed; `check_finite` (called
    every nu_stride steps by run()) reads it.  A BiCGStab failure rolls the fields back to the
    last check and replays the steps one by one with the reference's failure handling (the
    lgmres stand-in, then PoissonConvergenceError at that step)."""

    def __init__(self, ops: OperatorSet, params: PhysicsParams, settings: PoissonSolveSettings, dt: float,
                 state: FieldState, graphs: bool = True):
        t = L.torch()
        self.ops, self.params, self.settings, self.dt = ops, params, settings, float(dt)
        n, d = ops.n, ops.dim
        self.v = _soa(state.velocity)
        self.T = L.to_device(np.asarray(state.temperature, dtype=np.float64))
        # x = [p, lambda]: the pressure is a view of the Krylov solution (warm start of the next step)
        self.x = L.to_device(np.concatenate([np.asarray(state.pressure, dtype=np.float64),
                                             [getattr(ops, "_poisson_lambda", 0.0)]]))
        self.p = self.x[:n]
        self.x0 = L.empty(n + 1, t.float64)
        self.vstar = L.empty((d, n), t.float64)
        self.v_next = L.empty((d, n), t.float64)
        self.T_next = L.empty(n, t.float64)
        self.rhs = L.empty(n + 1, t.float64)
        self.status = L.zeros(2, t.int32)
        self.flags = L.to_device(np.array([0, INT32_MAX, 0], dtype=np.int32))  # [bad, node, blocks done]
        # [steps done, first non-finite step (0: none), its lowest non-finite T node, first step
        # whose BiCGStab failed (0: none), its info] (hn_step_latch)
        self.latch = L.to_device(np.array([0, 0, INT32_MAX, 0, 0], dtype=np.int32))
        self.have_p = False
        self.steps = 0
        self.graphs_enabled = bool(graphs) and ops._d_press is not None
        self.stream = t.cuda.Stream()
        self._graphs = {}
        self._bufs = (self.v, self.v_next, self.T, self.T_next)
        self._snapshot()

    # ---- one step, enqueued on the current stream ----
    def _explicit_front(self):
        ops = self.ops
        _momentum_dev(ops, self.params, self.dt, self.v, self.T, self.vstar, zero_boundary=True)
        _div_rhs_dev(ops, self.vstar, self.dt, self.rhs)

    def _explicit_back(self, pstatus):
        ops = self.ops
        _correct_temp_dev(ops, self.vstar, self.p, self.T, self.dt, self.v_next, self.T_next, self.flags,
                          self.params.dissipation)
        _temperature_bc_dev(ops, self.T_next, self.flags, self.latch, pstatus)  # + end-of-step latch

    def _body(self):
        """Unchecked step (graph body): warm-started device solve, status -> latch."""
        self._explicit_front()
        self.ops._d_press.solve(self.rhs, self.x if self.have_p else None, self.x, self.settings.tol,
                                self.settings.maxiter, self.status)
        self._explicit_back(self.status)

    def _checked_step(self):
        """Eager step with the status read back and the reference's failure handling."""
        self._explicit_front()
        x0 = None
        if self.have_p:
            self.x0.copy_(self.x)
            x0 = self.x0
        _pressure_dev(self.ops, self.rhs, x0, self.settings, self.x, self.status)
        self._explicit_back(None)

    def _swap(self):
        self.v, self.v_next = self.v_next, self.v
        self.T, self.T_next = self.T_next, self.T
        self.steps += 1

    def step(self):
        t = L.torch()
        self.stream.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(self.stream):
            if not self.graphs_enabled:
                if self.ops._d_press is None:
                    raise RuntimeError("operators were built with factorize=False: no pressure solve available")
                self._checked_step()
            elif not self.have_p:
                self._body()  # first step: zero start, no warm-start pointer in the graph
            else:
                key = self.v.data_ptr()
                g = self._graphs.get(key)
                if g is None:
                    g = t.cuda.CUDAGraph()
                    with t.cuda.graph(g, stream=self.stream, capture_error_mode="relaxed"):
                        self._body()
                    self._graphs[key] = g
                g.replay()
        t.cuda.current_stream().wait_stream(self.stream)
        self.have_p = True
        self._swap()

    def explicit_step(self):
        """The explicit part of a step only (K7, K8, K10, K11) with the pressure held at its
        current value -- for measuring the HBM-bound kernels in isolation (bench).  Replayed
        as a CUDA graph like the full step, so host launch latency does not enter."""
        t = L.torch()
        self.stream.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(self.stream):
            key = ("explicit", self.v.data_ptr())
            g = self._graphs.get(key)
            if g is None:
                self._explicit_front()  # eager once (lazy caches, e.g. hyper-dissipation)
                self._explicit_back(None)
                g = t.cuda.CUDAGraph()
                with t.cuda.graph(g, stream=self.stream, capture_error_mode="relaxed"):
                    self._explicit_front()
                    self._explicit_back(None)
                self._graphs[key] = g
            g.replay()
        t.cuda.current_stream().wait_stream(self.stream)
        self.v, self.v_next = self.v_next, self.v
        self.T, self.T_next = self.T_next, self.T

    # ---- checks, rollback ----
    def _snapshot(self):
        self._snap = (self.v.clone(), self.T.clone(), self.x.clone(), self.latch.clone(), self.steps, self.have_p)

    def _restore(self):
        v, T, x, latch, steps, have_p = self._snap
        self.v.copy_(v)
        self.T.copy_(T)
        self.x.copy_(x)
        self.latch.copy_(latch)
        self.steps, self.have_p = steps, have_p

    def check_finite(self, step: int | None = None):
        """Read the device latch (one 20-byte copy).  A BiCGStab failure (before any non-finite
        step) rolls back to the last check and replays with the reference's handling: the
        lgmres stand-in, else PoissonConvergenceError at that step (solver.py:304-313).  Then
        SolverDivergenceError for the first step whose fields went non-finite, with the
        reference's step number (counted from this stepper's first step) and node (the lowest
        non-finite temperature index, -1 if only the velocity was), solver.py:448-452."""
        f = self.latch.cpu().numpy()
        if f[3] and (f[1] == 0 or f[3] <= f[1]):
            target = self.steps
            self._restore()
            t = L.torch()
            with t.cuda.stream(self.stream):
                while self.steps < target:
                    self._checked_step()
                    self.have_p = True
                    self._swap()
            t.cuda.current_stream().wait_stream(self.stream)
            f = self.latch.cpu().numpy()
        if f[1]:
            bad = int(f[1])
            node = int(f[2]) if f[2] != INT32_MAX else -1
            raise SolverDivergenceError(f"non-finite field at step {bad}", step=bad, node=node)
        self._snapshot()

    def state(self) -> FieldState:
        """The fields on the host: one device pass puts [v (n x d) | p, lambda | T] into one
        contiguous buffer, one DMA into pinned memory (torch's caching host allocator), one
        synchronisation; the returned arrays are views of that pinned block, so a later
        load_state() of them is a direct DMA again."""
        t = L.torch()
        n, d = self.ops.n, self.ops.dim
        dev = L.empty(n * d + (n + 1) + n, t.float64)
        dev[: n * d].view(n, d).copy_(self.v.t())
        dev[n * d: n * d + n + 1].copy_(self.x)
        dev[n * d + n + 1:].copy_(self.T)
        host = t.empty(dev.shape, dtype=t.float64, pin_memory=True)
        host.copy_(dev, non_blocking=True)
        t.cuda.current_stream().synchronize()
        L.TRAFFIC["d2h"] += host.nbytes
        h = host.numpy()
        self.ops._poisson_lambda = float(h[n * d + n])
        return FieldState(h[: n * d].reshape(n, d), h[n * d: n * d + n], h[n * d + n + 1:])

    def load_state(self, state: FieldState):
        """Replace the device fields with a host state (the pressure also warm-starts the next
        solve, as p_prev does in the reference loop).  Pinned host arrays (e.g. from state())
        go by direct DMA; others through a pinned staging block."""
        t = L.torch()
        n, d = self.ops.n, self.ops.dim
        for dst, src, shape in ((self.T, state.temperature, (n,)), (self.p, state.pressure, (n,))):
            a = np.ascontiguousarray(np.asarray(src, dtype=np.float64).reshape(shape))
            dst.copy_(_pinned_view(t, a), non_blocking=True)
        v = np.ascontiguousarray(np.asarray(state.velocity, dtype=np.float64).reshape(n, d))
        tmp = L.empty((n, d), t.float64)
        tmp.copy_(_pinned_view(t, v), non_blocking=True)
        self.v.copy_(tmp.t())
        self.x[self.ops.n] = float(getattr(self.ops, "_poisson_lambda", 0.0))
        L.TRAFFIC["h2d"] += self.v.nbytes + self.T.nbytes + self.p.nbytes
        self.have_p = True
        self._snapshot()
        t.cuda.current_stream().synchronize()  # the caller may reuse its host arrays at once

    def nusselt(self) -> float:
        return _nusselt_dev(self.ops, self.T) if self.ops._d_nu is not None else float("nan")

    def divergence(self, which: str = "v") -> float:
        return _interior_divergence_dev(self.ops, self.vstar if which == "vstar" else self.v)


@dataclass
class RunResult:
    case: str
    discretization: str
    final_nu: float
    nu_steps: np.ndarray
    nu_times: np.ndarray
    nu_values: np.ndarray
    counts: tuple
    n_total: int
    timings: dict
    dt: float
    steps: int
    t_final: float
    status: str = "ok"
    diagnostics: dict = field(default_factory=dict)
    state: FieldState | None = None
    nodeset: object = None


def run(config, spec=None, nodeset=None) -> RunResult:
    """Build operators and integrate the case to t_end (solver.py:395-490), GPU-resident.

    `config` needs the CaseConfig fields run() reads (Ra, Pr, t_cold, t_hot, t_init, t_end,
    poisson_tol, poisson_maxiter, steady_tol, nu_window, nu_stride, case, discretization)
    and a `cold_origins(spec)` method or attribute.  Without a `nodeset` the case's node set
    is generated on the device (generate.hybrid_discretize, reference nodegen.py:436-518)."""
    timings: dict = {}
    t0 = time.perf_counter()
    if spec is None and callable(getattr(config, "cold_origins", None)):
        # the reference always builds the domain first (solver.py:412-415): its
        # CaseConfig.cold_origins(spec) reads spec.obstacles, even with a precomputed node set
        from .config import build_domain
        spec = build_domain(config)
    if nodeset is None:
        from .generate import hybrid_discretize
        nodeset = hybrid_discretize(config, spec)
    timings["nodegen"] = time.perf_counter() - t0
    settings = PoissonSolveSettings(tol=config.poisson_tol, maxiter=config.poisson_maxiter)
    cold = config.cold_origins(spec) if callable(getattr(config, "cold_origins", None)) else set(config.cold_origins)
    ops = build_operators(nodeset, cold, settings, timings=timings)
    params = PhysicsParams(config.Ra, config.Pr, t_ref=0.5 * (config.t_cold + config.t_hot))
    controls = TimeControls.from_spacing(float(np.min(nodeset.spacing)), config.t_end, Ra=config.Ra,
                                         steady_tol=config.steady_tol, nu_window=config.nu_window,
                                         nu_stride=config.nu_stride)
    n = len(nodeset)
    state = FieldState.zeros(n, nodeset.dim)
    state.temperature[:] = config.t_init
    apply_temperature_bc(state.temperature, ops)
    dt = controls.dt
    n_steps = max(1, int(np.ceil(controls.t_end / dt - 1e-12)))
    monitor_stride = max(1, controls.nu_stride)
    stepper = DeviceStepper(ops, params, settings, dt, state)
    nu_steps, nu_times, nu_values, div_samples = [], [], [], []
    t0 = time.perf_counter()
    step = 0
    for step in range(1, n_steps + 1):
        stepper.step()
        if step % monitor_stride == 0 or step == n_steps:
            stepper.check_finite(step)
            nu_steps.append(step)
            nu_times.append(step * dt)
            nu_values.append(stepper.nusselt())
            if len(div_samples) < 64 or step == n_steps:
                div_samples.append((step, stepper.divergence("vstar"), stepper.divergence("v")))
            w = controls.nu_window
            if controls.steady_tol > 0 and len(nu_values) >= 2 * w:
                m1 = float(np.mean(nu_values[-w:]))
                m0 = float(np.mean(nu_values[-2 * w:-w]))
                span = (nu_times[-1] - nu_times[-w - 1]) or 1.0
                if abs(m1 - m0) / (max(abs(m1), 1e-12) * span) < controls.steady_tol:
                    break
    stepper.check_finite(step)
    L.torch().cuda.synchronize()
    timings["stepping"] = time.perf_counter() - t0
    timings["total"] = sum(timings.values())
    final = stepper.state()
    nr, ns_, nb = nodeset.counts
    return RunResult(case=getattr(config, "case", "custom"), discretization=getattr(config, "discretization", ""),
                     final_nu=nu_values[-1] if nu_values else float("nan"), nu_steps=np.asarray(nu_steps),
                     nu_times=np.asarray(nu_times), nu_values=np.asarray(nu_values), counts=(nr, ns_, nb),
                     n_total=n, timings=timings, dt=dt, steps=step, t_final=step * dt,
                     diagnostics={"divergence_samples": div_samples,
                                  "temperature_range": (float(final.temperature.min()),
                                                        float(final.temperature.max()))},
                     state=final, nodeset=nodeset)


def write_outputs(result: RunResult, out_dir) -> None:
    """The run artifacts the reference's bench layer writes (pkg/src/hybridnodes/bench.py:28-44),
    same files and columns: nu_series.csv (step, t, Nu), timings.csv (phase, seconds, sorted)
    and, with a final state, fields_<t>.csv (coordinates, velocity, p, T, h; t with '.' -> 'p')."""
    import csv
    from pathlib import Path

    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)

    def dump(name, header, rows):
        with open(out / name, "w", newline="") as fh:
            wr = csv.writer(fh)
            wr.writerow(header)
            wr.writerows(rows)

    dump("nu_series.csv", ["step", "t", "Nu"], zip(result.nu_steps, result.nu_times, result.nu_values))
    dump("timings.csv", ["phase", "seconds"], sorted(result.timings.items()))
    if result.state is None or result.nodeset is None:
        return
    ns, st = result.nodeset, result.state
    dim = ns.positions.shape[1]
    header = [*"xyz"[:dim], *"uvw"[:dim], "p", "T", "h"]
    table = np.column_stack([ns.positions, st.velocity, st.pressure, st.temperature, ns.spacing])
    dump("fields_%s.csv" % ("%g" % result.t_final).replace(".", "p"), header, table)
