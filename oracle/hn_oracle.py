"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference hot path (arXiv 2303.01760, package
`hybridnodes`, /root/reference/pkg/src/hybridnodes).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline leg (`--impl reference` / `cpu_baseline`) may import it, and
only as the checker / the timed CPU reference -- never as the product path.

The reference is pure Python; its arithmetic lives in third-party numerics that are not
vendored under /root/reference (pyproject pins only lower bounds):
    numpy 2.3.5 (np.linalg.solve -> OpenBLAS 0.3.30 LAPACK dgesv), scipy 1.18.1
    (cKDTree, CSR csr_matvec, SuperLU splu, bicgstab).
The oracle calls the same numerics in the same order, so on the same host it reproduces
the reference bit for bit; pinning: tests/test_oracle_golden.py checks it against golden
vectors produced by running the reference itself (oracle/make_golden.py ->
tests/golden/*.npz).

Operators are given as tuples: ("lap",), ("d", axis), ("n", normal-tuple).
"""

from __future__ import annotations

import math

import numpy as np
from scipy import sparse
from scipy.sparse import linalg as spla
from scipy.spatial import cKDTree

KIND_REGULAR, KIND_SCATTERED, KIND_BOUNDARY = 0, 1, 2
ROLE_DIRICHLET, ROLE_NEUMANN = 1, 2
NONE_KEY = np.iinfo(np.int64).min
MON_N = {2: 5, 3: 7}
RBF_N = {2: 12, 3: 30}


def op_tuple(op):
    """Map this package's / the reference's operator objects to oracle tuples."""
    if isinstance(op, tuple):
        return op
    name = type(op).__name__
    if name == "Laplacian":
        return ("lap",)
    if name == "Partial":
        return ("d", int(op.axis))
    if name == "NormalDerivative":
        return ("n", tuple(float(v) for v in op.normal))
    if op == "normal":
        return ("nrow",)
    raise TypeError(op)


def op_order(op) -> int:
    return 2 if op[0] == "lap" else 1


# ------------------------------------------------------------------ stencils
def knn_by_key(positions, queries, n):
    """n nearest by (fl-distance, index): cKDTree query widened past cutoff ties, then
    lexsort -- reference approx.py:133-146."""
    total = len(positions)
    if n > total:
        raise ValueError(f"stencil size {n} exceeds node count {total}")
    tree = cKDTree(positions)
    k = min(total, n + 8)
    while True:
        d, idx = tree.query(queries, k=k)
        d = np.atleast_2d(d)
        idx = np.atleast_2d(idx)
        if k == total or np.all(d[:, -1] > d[:, n - 1] * (1 + 1e-12)):
            break
        k = min(total, 2 * k)
    order = np.lexsort((idx, d), axis=1)
    return np.take_along_axis(idx, order, axis=1)[:, :n]


def _axis_offsets(dim):
    eye = np.eye(dim, dtype=np.int64)
    return np.concatenate([eye, -eye])


def classify(ns):
    """-1 boundary / 0 MON / 1 RBF-FD -- reference approx.py:332-357."""
    n = len(ns.positions)
    dim = ns.positions.shape[1]
    kind = np.asarray(ns.kind)
    out = np.where(kind != KIND_BOUNDARY, 1, -1).astype(np.int8)
    reg = np.nonzero(kind == KIND_REGULAR)[0]
    if not len(reg):
        return out
    if ns.lattice is not None and ns.lattice_idx is not None:
        keys = np.asarray(ns.lattice_idx)[reg]
        on = keys[:, 0] != NONE_KEY
        good = np.ones(int(on.sum()), dtype=bool)
        grid = np.asarray(ns.lattice.grid)
        for off in _axis_offsets(dim):
            kk = keys[on] + off
            good &= grid[tuple(kk[:, a] for a in range(dim))] >= 0
        out[reg[on][good]] = 0
        return out
    tree = cKDTree(ns.positions)
    for i in reg:
        h = ns.spacing[i]
        probes = np.concatenate([ns.positions[i] + h * np.eye(dim), ns.positions[i] - h * np.eye(dim)])
        dd, _ = tree.query(probes, k=1)
        if np.all(dd < 1e-9 * h):
            out[i] = 0
    return out


def mon_stencils(ns, rows):
    """[row] + lattice axis neighbours by (norm, index) -- reference approx.py:360-376."""
    dim = ns.positions.shape[1]
    if ns.lattice is None or ns.lattice_idx is None:
        return knn_by_key(ns.positions, ns.positions[rows], MON_N[dim])
    keys = np.asarray(ns.lattice_idx)[rows]
    grid = np.asarray(ns.lattice.grid)
    nb = np.stack([grid[tuple((keys + off)[:, a] for a in range(dim))] for off in _axis_offsets(dim)], axis=1)
    dist = np.linalg.norm(ns.positions[nb] - ns.positions[rows][:, None, :], axis=-1)
    srt = np.lexsort((nb, dist), axis=1)
    return np.concatenate([rows[:, None], np.take_along_axis(nb, srt, axis=1)], axis=1)


def boundary_stencils(ns, rows, exclude, size):
    """[self] + (size-1) nearest allowed (no widening) -- reference approx.py:416-431."""
    if exclude is None:
        return knn_by_key(ns.positions, ns.positions[rows], size)
    exclude = np.asarray(exclude, dtype=bool)
    allowed = np.nonzero(~exclude)[0]
    k = min(len(allowed), size - 1)
    d, idx = cKDTree(ns.positions[allowed]).query(ns.positions[rows], k=k)
    d, idx = np.atleast_2d(d), np.atleast_2d(idx)
    srt = np.lexsort((allowed[idx], d), axis=1)
    return np.concatenate([rows[:, None], allowed[np.take_along_axis(idx, srt, axis=1)]], axis=1)


# ------------------------------------------------------------------ local systems
def _local(positions, stencils):
    p = positions[stencils]
    rel = p - p[:, 0, :][:, None, :]
    scale = np.max(np.linalg.norm(rel, axis=-1), axis=1)
    return rel / scale[:, None, None], scale


def _exponents(dim):
    ex = [(0,) * dim]
    for deg in (1, 2):
        for combo in _combos(dim, deg):
            e = [0] * dim
            for a in combo:
                e[a] += 1
            ex.append(tuple(e))
    return ex


def _combos(dim, deg):
    if deg == 1:
        return [(a,) for a in range(dim)]
    return [(a, b) for a in range(dim) for b in range(a, dim)]


def mon_solve(positions, stencils, ops):
    """(K, n, n_ops) MON weights in stencil order -- reference approx.py:212-234."""
    loc, scale = _local(positions, stencils)
    k, n, dim = loc.shape
    M = np.empty((k, n, n))
    M[:, 0, :] = 1.0
    for a in range(dim):
        M[:, 1 + a, :] = loc[:, :, a]
        M[:, 1 + dim + a, :] = loc[:, :, a] ** 2
    rhs = np.zeros((n, len(ops)))
    for j, op in enumerate(ops):
        if op[0] == "lap":
            rhs[1 + dim:, j] = 2.0
        elif op[0] == "d":
            rhs[1 + op[1], j] = 1.0
        else:
            rhs[1:1 + dim, j] = np.asarray(op[1], dtype=float)
    w = np.linalg.solve(M, rhs)
    for j, op in enumerate(ops):
        w[:, :, j] /= scale[:, None] ** op_order(op)
    return w


def rbf_solve(positions, stencils, ops, normals=None):
    """(K, n, n_ops) PHS r^3 + degree-2 RBF-FD weights -- reference approx.py:237-290."""
    loc, scale = _local(positions, stencils)
    k, n, dim = loc.shape
    ex = _exponents(dim)
    q = len(ex)
    S = np.zeros((k, n + q, n + q))
    dif = loc[:, :, None, :] - loc[:, None, :, :]
    S[:, :n, :n] = np.sqrt(np.sum(dif * dif, axis=-1)) ** 3
    P = np.ones((k, n, q))
    for j, e in enumerate(ex):
        for a in range(dim):
            if e[a]:
                P[:, :, j] *= loc[:, :, a] ** e[a]
    S[:, :n, n:] = P
    S[:, n:, :n] = np.transpose(P, (0, 2, 1))
    r = np.linalg.norm(loc, axis=-1)
    if normals is not None:
        R = np.zeros((k, n + q, 1))
        R[:, :n, 0] = -3.0 * r * np.einsum("knd,kd->kn", loc, normals)
        for j, e in enumerate(ex):
            if sum(e) == 1:
                R[:, n + j, 0] = normals[:, e.index(1)]
        orders = [1]
    else:
        R = np.zeros((k, n + q, len(ops)))
        for j, op in enumerate(ops):
            if op[0] == "lap":
                R[:, :n, j] = 3.0 * (dim + 1) * r
            elif op[0] == "d":
                R[:, :n, j] = -3.0 * r * loc[:, :, op[1]]
            else:
                R[:, :n, j] = -3.0 * r * (loc @ np.asarray(op[1], dtype=float))
            for m, e in enumerate(ex):
                if op[0] == "lap":
                    R[:, n + m, j] = sum(2.0 for a in range(dim) if e[a] == 2 and sum(e) == 2)
                elif sum(e) == 1:
                    ax = e.index(1)
                    R[:, n + m, j] = (1.0 if ax == op[1] else 0.0) if op[0] == "d" else op[1][ax]
        orders = [op_order(op) for op in ops]
    sol = np.linalg.solve(S, R)
    w = sol[:, :n, :]
    for j, o in enumerate(orders):
        w[:, :, j] /= scale[:, None] ** o
    return w


# ------------------------------------------------------------------ tables
def _store(table, rows, stencils, w, keys):
    order = np.argsort(stencils, axis=1)
    table["indices"][rows, : stencils.shape[1]] = np.take_along_axis(stencils, order, axis=1)
    for j, key in enumerate(keys):
        table["weights"][key][rows, : stencils.shape[1]] = np.take_along_axis(w[:, :, j], order, axis=1)
    table["sizes"][rows] = stencils.shape[1]


def _empty_table(n, width, keys):
    return {"indices": np.full((n, width), -1, dtype=np.int64), "sizes": np.zeros(n, dtype=np.int64),
            "weights": {k: np.zeros((n, width)) for k in keys}, "method": np.full(n, -1, dtype=np.int8)}


def compute_weights(ns, ops, rbf_n=None, chunk=4096):
    """Interior stencils + weights -- reference approx.py:379-413."""
    keys = list(ops)
    ops = [op_tuple(o) for o in keys]
    dim = ns.positions.shape[1]
    n = len(ns.positions)
    rbf_n = RBF_N[dim] if rbf_n is None else rbf_n
    method = classify(ns)
    table = _empty_table(n, rbf_n, keys)  # n_max = RBF_SIZE[dim] at call time (approx.py:388)
    table["method"] = method
    for meth, solver in ((0, mon_solve), (1, rbf_solve)):
        rows = np.nonzero(method == meth)[0]
        if not len(rows):
            continue
        st = mon_stencils(ns, rows) if meth == 0 else knn_by_key(ns.positions, ns.positions[rows], rbf_n)
        table.setdefault("stencils", {})[meth] = (rows, st)
        for lo in range(0, len(rows), chunk):
            sl = slice(lo, lo + chunk)
            _store(table, rows[sl], st[sl], solver(ns.positions, st[sl], ops), keys)
    return table


def boundary_table(ns, rows, exclude, ops=None, normals=False, size=None, chunk=4096):
    """boundary_partial_table / normal_derivative_table -- reference approx.py:437-491."""
    rows = np.asarray(rows, dtype=np.int64)
    dim = ns.positions.shape[1]
    size = RBF_N[dim] if size is None else size
    keys = ["normal"] if normals else [("d", a) for a in range(dim)]
    st = boundary_stencils(ns, rows, exclude, size)
    table = _empty_table(len(ns.positions), st.shape[1], keys)
    table["stencils"] = st
    for lo in range(0, len(rows), chunk):
        sl = slice(lo, lo + chunk)
        if normals:
            w = rbf_solve(ns.positions, st[sl], None, normals=np.asarray(ns.normals)[rows[sl]])
        else:
            w = rbf_solve(ns.positions, st[sl], keys)
        _store(table, rows[sl], st[sl], w, keys)
        table["method"][rows[sl]] = 1
    return table


def csr(table, key, n):
    """CSR of one weight plane -- reference operators.py:61-77 / solver.py:127-130."""
    cols = np.arange(table["indices"].shape[1])[None, :] < table["sizes"][:, None]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(table["sizes"], out=indptr[1:])
    return sparse.csr_matrix((table["weights"][key][cols], table["indices"][cols], indptr), shape=(n, n))


def apply(matrix, field):
    """scipy csr_matvec -- reference operators.py:51-54."""
    return matrix @ field


def apply_sequential(matrix, field):
    """Plain-loop restatement of csr_matvec: acc = 0; acc += w*f in stored order."""
    out = np.zeros(matrix.shape[0])
    ip, ix, dv = matrix.indptr, matrix.indices, matrix.data
    for i in range(matrix.shape[0]):
        acc = 0.0
        for k in range(ip[i], ip[i + 1]):
            acc += dv[k] * field[ix[k]]
        out[i] = acc
    return out


# ------------------------------------------------------------------ solver
class Operators:
    """Everything solver.build_operators produces (reference solver.py:133-232)."""


def build_operators(ns, cold_origins, beta=0.1, gauge=None, rbf_n=None, table=None):
    dim = ns.positions.shape[1]
    n = len(ns.positions)
    o = Operators()
    o.n, o.dim = n, dim
    keys = [("lap",)] + [("d", a) for a in range(dim)]
    bidx = np.nonzero(np.asarray(ns.kind) == KIND_BOUNDARY)[0]
    bmask = np.asarray(ns.kind) == KIND_BOUNDARY
    interior = ~bmask
    o.table = table if table is not None else compute_weights(ns, keys, rbf_n=rbf_n)
    o.bgrad = boundary_table(ns, bidx, bmask)
    cold = np.array([i for i in bidx if ns.origin[i] in cold_origins], dtype=np.int64)
    o.nu_table = boundary_table(ns, cold, None, normals=True) if len(cold) else None
    o.lap = csr(o.table, ("lap",), n)
    o.d = [csr(o.table, ("d", a), n) for a in range(dim)]
    grows = [csr(o.bgrad, ("d", a), n) for a in range(dim)]
    nsafe = np.where(np.isfinite(ns.normals), ns.normals, 0.0)
    normal = sum(sparse.diags(nsafe[:, a]) @ grows[a] for a in range(dim)).tocsr()
    if gauge is None:
        cen = ns.positions[interior].mean(axis=0)
        cand = np.nonzero(interior)[0]
        gauge = int(cand[np.argmin(np.linalg.norm(ns.positions[cand] - cen, axis=1))])
    o.gauge = gauge
    full = [p + g for p, g in zip(o.d, grows)]
    div_grad = sum(p @ g for p, g in zip(o.d, full))
    blended = (1.0 - beta) * div_grad + beta * o.lap
    core = (sparse.diags(interior.astype(float)) @ blended + sparse.diags(bmask.astype(float)) @ normal).tocsr()
    core.eliminate_zeros()
    core = core.tocoo()
    ni = int(interior.sum())
    o.poisson = sparse.csr_matrix(
        (np.concatenate([core.data, np.ones(ni), [1.0]]),
         (np.concatenate([core.row, np.nonzero(interior)[0], [n]]), np.concatenate([core.col, np.full(ni, n), [gauge]]))),
        shape=(n + 1, n + 1))
    o.lu = spla.splu(o.poisson.tocsc())
    o.precond = spla.LinearOperator(o.poisson.shape, o.lu.solve)
    o.boundary_idx = bidx
    o.interior_idx = np.nonzero(interior)[0]
    o.dirichlet_idx = np.nonzero(np.asarray(ns.role) == ROLE_DIRICHLET)[0]
    o.dirichlet_values = np.asarray(ns.bc_value)[o.dirichlet_idx]
    o.neumann_idx = np.nonzero(np.asarray(ns.role) == ROLE_NEUMANN)[0]
    o.w_neu = o.neu_lu = None
    if len(o.neumann_idx):
        o.w_neu = normal[o.neumann_idx]
        o.neu_lu = spla.splu(o.w_neu[:, o.neumann_idx].tocsc())
    o.nu_rows = csr(o.nu_table, "normal", n)[cold] if o.nu_table is not None else None
    vals = o.dirichlet_values
    span = (vals.max() - vals.min()) if len(vals) else 1.0
    o.nu_scale = float(np.max(ns.positions.max(axis=0) - ns.positions.min(axis=0))) / (span if span > 0 else 1.0)
    o.lam = 0.0
    o.spacing = np.asarray(ns.spacing, dtype=float)
    return o


def hyper_dissipation(o, field, speed, coeff):
    """-coeff * h^3 |v| lap(lap(field)), inner boundary rows zeroed -- reference solver.py:235-247."""
    inner = o.lap @ field
    inner[o.boundary_idx] = 0.0
    return -coeff * o.spacing ** 3 * speed * (o.lap @ inner)


def momentum(o, v, T, Ra, Pr, t_ref, dt, g=None, dissipation=0.0):
    """v* (no BC) -- reference solver.py:250-274."""
    dim = o.dim
    if g is None:
        g = np.zeros(dim)
        g[-1] = -1.0
    tdelta = T - t_ref
    out = np.empty_like(v)
    speed = np.linalg.norm(v, axis=1)
    grads = [[o.d[a] @ v[:, c] for a in range(dim)] for c in range(dim)]
    for c in range(dim):
        adv = v[:, 0] * grads[c][0]
        for a in range(1, dim):
            adv += v[:, a] * grads[c][a]
        rhs = -adv + Pr * (o.lap @ v[:, c]) - Ra * Pr * g[c] * tdelta
        if dissipation:
            rhs += hyper_dissipation(o, v[:, c], speed, dissipation)
        out[:, c] = v[:, c] + dt * rhs
    return out


def pressure(o, vstar, dt, x0=None, tol=1e-8, maxiter=2000):
    """Bordered Poisson via bicgstab + complete-LU preconditioner -- reference solver.py:283-314."""
    n = o.n
    rhs = np.empty(n + 1)
    div = o.d[0] @ vstar[:, 0]
    for a in range(1, o.dim):
        div += o.d[a] @ vstar[:, a]
    rhs[:n] = div / dt
    rhs[o.boundary_idx] = 0.0
    rhs[n] = 0.0
    if x0 is not None and len(x0) == n:
        x0 = np.concatenate([x0, [o.lam]])
    p, info = spla.bicgstab(o.poisson, rhs, x0=x0, M=o.precond, rtol=tol, atol=0.0, maxiter=maxiter)
    if info != 0:
        raise RuntimeError(f"oracle bicgstab info={info}")
    o.lam = float(p[n])
    return p[:n]


def correct(o, vstar, p, dt):
    """reference solver.py:317-331."""
    v = vstar.copy()
    for a in range(o.dim):
        v[:, a] -= dt * (o.d[a] @ p)
    v[o.boundary_idx] = 0.0
    return v


def temperature_bc(o, T):
    """reference solver.py:334-342 (in place)."""
    T[o.dirichlet_idx] = o.dirichlet_values
    if o.neu_lu is not None:
        t0 = T.copy()
        t0[o.neumann_idx] = 0.0
        T[o.neumann_idx] = o.neu_lu.solve(-(o.w_neu @ t0))
    return T


def temperature(o, v, T, dt, dissipation=0.0):
    """reference solver.py:345-358."""
    conv = v[:, 0] * (o.d[0] @ T)
    for a in range(1, o.dim):
        conv += v[:, a] * (o.d[a] @ T)
    rhs = -conv + (o.lap @ T)
    if dissipation:
        rhs += hyper_dissipation(o, T, np.linalg.norm(v, axis=1), dissipation)
    out = T + dt * rhs
    return temperature_bc(o, out)


def nusselt(o, T):
    """reference solver.py:361-365."""
    if o.nu_rows is None:
        return float("nan")
    return float(o.nu_scale * np.mean(np.abs(o.nu_rows @ T)))


def step(o, state, Ra, Pr, t_ref, dt, p_prev=None, tol=1e-8, dissipation=0.0):
    """One run() loop body -- reference solver.py:439-452."""
    v, T = state
    vstar = momentum(o, v, T, Ra, Pr, t_ref, dt, dissipation=dissipation)
    vstar[o.boundary_idx] = 0.0
    p = pressure(o, vstar, dt, x0=p_prev, tol=tol)
    v_new = correct(o, vstar, p, dt)
    T_new = temperature(o, v_new, T, dt, dissipation=dissipation)
    probe = float(np.sum(T_new)) + float(np.sum(v_new))
    if not math.isfinite(probe):
        raise FloatingPointError("non-finite field")
    return (v_new, T_new), p


def dt_rule(h_min, Ra):
    """reference solver.py:60-73."""
    return min(0.1 * h_min ** 2 / 2.0, 40.0 / Ra)
