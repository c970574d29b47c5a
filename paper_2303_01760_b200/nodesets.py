"""Seeded synthetic node sets for the five BASELINE configurations.

The reference's own generators (advancing-front fill, SDF geometry; reference
nodegen.py:182-518, geometry.py) are outside the hot path.  These
builder-defined generators follow SURVEY Appendix B and produce NodeSets with every
field the hot path reads (kind, role, bc_value, normals, origin tags and the lattice
index map), in the reference's node order: regular, scattered, boundary.

Boundary conditions everywhere follow the reference's dvd policy (config.py:112-124):
the x = lo wall is Dirichlet t_cold (tag ``wall:x-``), x = hi is Dirichlet t_hot,
every other wall and every obstacle is insulated (Neumann).  Corners/edges belong to
the x walls first, then the lowest-axis wall (reference geometry.py:384-450).

  config0  regular_box(199)              N = 40,000   (the reference's dvd pure-regular set)
  config1  jittered_box(315, seed)       N = 99,856   (100,000 is not a square lattice + ring)
  config2  hybrid_hole_2d(500, seed)     N ~ 247,600  (~23 % scattered, band around the hole)
  config3  = config2 node set, time stepping
  config4  hybrid_sphere_3d(M, seed)     N ~ 1e6      (scattered band refined 2x toward the sphere)
"""

from __future__ import annotations

import numpy as np

from .nodegen import (KIND_BOUNDARY, KIND_REGULAR, KIND_SCATTERED, LATTICE_NONE, ROLE_DIRICHLET,
                      ROLE_INTERIOR, ROLE_NEUMANN, LatticeInfo, NodeSet)

T_COLD, T_HOT = -0.5, 0.5


def _box_walls(M: int, dim: int):
    """Lattice-aligned box wall nodes at spacing 1/M: (keys, normals, origins)."""
    keys, normals, origins = [], [], []
    if dim == 2:
        for xi, tag, nx in ((0, "x-", -1.0), (M, "x+", 1.0)):
            for yj in (0, M):
                keys.append((xi, yj)); normals.append((nx, 0.0)); origins.append(f"wall:{tag}")
        inner = np.arange(1, M)
        for axis, side in ((0, 0), (0, 1), (1, 0), (1, 1)):
            val = 0 if side == 0 else M
            sgn = -1.0 if side == 0 else 1.0
            tag = f"wall:{'xy'[axis]}{'-' if side == 0 else '+'}"
            for t in inner:
                k = [0, 0]
                k[axis] = val
                k[1 - axis] = int(t)
                nrm = [0.0, 0.0]
                nrm[axis] = sgn
                keys.append(tuple(k)); normals.append(tuple(nrm)); origins.append(tag)
        return np.array(keys, np.int64), np.array(normals), origins
    # 3D: corners (x walls), edges (lowest non-edge axis), face interiors
    for xi, tag, nx in ((0, "x-", -1.0), (M, "x+", 1.0)):
        for yj in (0, M):
            for zk in (0, M):
                keys.append((xi, yj, zk)); normals.append((nx, 0.0, 0.0)); origins.append(f"wall:{tag}")
    inner = np.arange(1, M)
    for axis in range(3):
        u, v = [a for a in range(3) if a != axis]
        for uv in (0, M):
            for vv in (0, M):
                sgn = -1.0 if uv == 0 else 1.0
                nrm = [0.0, 0.0, 0.0]
                nrm[u] = sgn
                tag = f"wall:{'xyz'[u]}{'-' if sgn < 0 else '+'}"
                for t in inner:
                    k = [0, 0, 0]
                    k[axis] = int(t); k[u] = uv; k[v] = vv
                    keys.append(tuple(k)); normals.append(tuple(nrm)); origins.append(tag)
    face_keys = []
    for axis in range(3):
        u, v = [a for a in range(3) if a != axis]
        for side in (0, 1):
            val = 0 if side == 0 else M
            uu, vv = np.meshgrid(inner, inner, indexing="ij")
            k = np.zeros((uu.size, 3), np.int64)
            k[:, axis] = val
            k[:, u] = uu.ravel()
            k[:, v] = vv.ravel()
            nrm = np.zeros((uu.size, 3))
            nrm[:, axis] = -1.0 if side == 0 else 1.0
            face_keys.append((k, nrm, [f"wall:{'xyz'[axis]}{'-' if side == 0 else '+'}"] * uu.size))
    keys = np.concatenate([np.array(keys, np.int64)] + [f[0] for f in face_keys])
    normals = np.concatenate([np.array(normals)] + [f[1] for f in face_keys])
    origins = origins + sum((f[2] for f in face_keys), [])
    return keys, normals, origins


def _wall_bc(origins):
    role = np.array([ROLE_DIRICHLET if o in ("wall:x-", "wall:x+") else ROLE_NEUMANN for o in origins], np.int8)
    val = np.array([T_COLD if o == "wall:x-" else (T_HOT if o == "wall:x+" else 0.0) for o in origins])
    return role, val


def _assemble(dim, M, reg_keys, scat_pos, scat_h, wall_keys, wall_normals, wall_origins,
              extra_pos=None, extra_normals=None, extra_origins=None, extra_h=None) -> NodeSet:
    h = 1.0 / M
    step = np.full(dim, h)
    reg_pos = reg_keys * h
    wall_pos = wall_keys * h
    n_r, n_s = len(reg_pos), len(scat_pos)
    bpos = [wall_pos]
    bnorm = [wall_normals]
    borig = list(wall_origins)
    bh = [np.full(len(wall_pos), h)]
    if extra_pos is not None and len(extra_pos):
        bpos.append(extra_pos); bnorm.append(extra_normals); borig += list(extra_origins); bh.append(extra_h)
    bpos = np.concatenate(bpos)
    n_b = len(bpos)
    positions = np.concatenate([reg_pos, scat_pos.reshape(-1, dim), bpos])
    spacing = np.concatenate([np.full(n_r, h), scat_h, np.concatenate(bh)])
    kind = np.concatenate([np.full(n_r, KIND_REGULAR), np.full(n_s, KIND_SCATTERED),
                           np.full(n_b, KIND_BOUNDARY)]).astype(np.int8)
    wrole, wval = _wall_bc(wall_origins)
    n_extra = n_b - len(wall_pos)
    role = np.concatenate([np.full(n_r + n_s, ROLE_INTERIOR), wrole, np.full(n_extra, ROLE_NEUMANN)]).astype(np.int8)
    bc_value = np.concatenate([np.full(n_r + n_s, np.nan), wval, np.zeros(n_extra)])
    normals = np.concatenate([np.full((n_r + n_s, dim), np.nan), np.concatenate(bnorm)])
    origin = [""] * (n_r + n_s) + borig
    lattice = LatticeInfo(np.zeros(dim), step, tuple([M] * dim))
    lattice_idx = np.full((len(positions), dim), LATTICE_NONE, dtype=np.int64)
    if n_r:
        lattice_idx[:n_r] = reg_keys
        lattice.grid[tuple(reg_keys[:, a] for a in range(dim))] = np.arange(n_r)
    # wall nodes sit on lattice lines and join the index map (reference nodegen.py:505-516)
    wid = n_r + n_s + np.arange(len(wall_pos))
    free = lattice.grid[tuple(wall_keys[:, a] for a in range(dim))] < 0
    lattice.grid[tuple(wall_keys[free][:, a] for a in range(dim))] = wid[free]
    lattice_idx[wid[free]] = wall_keys[free]
    return NodeSet(positions, spacing, kind, role, bc_value, normals, origin, lattice, lattice_idx)


def _interior_keys(M: int, dim: int) -> np.ndarray:
    r = np.arange(1, M)
    grids = np.meshgrid(*([r] * dim), indexing="ij")
    return np.stack([g.ravel() for g in grids], axis=-1).astype(np.int64)


def regular_box(M: int = 199, dim: int = 2) -> NodeSet:
    """Pure lattice box with (M+1)^d nodes: config 0 is regular_box(199) (N = 40,000, h = 1/199)."""
    wk, wn, wo = _box_walls(M, dim)
    return _assemble(dim, M, _interior_keys(M, dim), np.empty((0, dim)), np.empty(0), wk, wn, wo)


def jittered_box(M: int = 315, seed: int = 1, jitter: float = 0.35, dim: int = 2) -> NodeSet:
    """Config 1: interior lattice nodes jittered by U(+-jitter*h)^d, all scattered; wall ring at h."""
    rng = np.random.default_rng(seed)
    h = 1.0 / M
    keys = _interior_keys(M, dim)
    pos = keys * h + rng.uniform(-jitter * h, jitter * h, keys.shape)
    wk, wn, wo = _box_walls(M, dim)
    ns = _assemble(dim, M, np.empty((0, dim), np.int64), pos, np.full(len(pos), h), wk, wn, wo)
    return ns


def _separation_thin(pts, rad, rng):
    """Random-priority maximal independent set of the conflict graph |p_i - p_j| <
    max(rad_i, rad_j) (Luby rounds, vectorised): every kept pair is >= its radius apart and
    every dropped candidate has a kept neighbour inside its radius (Poisson-disk quality)."""
    from scipy.spatial import cKDTree
    n = len(pts)
    if n == 0:
        return np.zeros(0, bool)
    pairs = cKDTree(pts).query_pairs(float(rad.max()), output_type="ndarray")
    if len(pairs):
        d = np.linalg.norm(pts[pairs[:, 0]] - pts[pairs[:, 1]], axis=1)
        pairs = pairs[d < np.maximum(rad[pairs[:, 0]], rad[pairs[:, 1]])]
    a = np.concatenate([pairs[:, 0], pairs[:, 1]]) if len(pairs) else np.zeros(0, np.int64)
    b = np.concatenate([pairs[:, 1], pairs[:, 0]]) if len(pairs) else np.zeros(0, np.int64)
    prio = rng.permutation(n)
    state = np.zeros(n, np.int8)  # 0 open, 1 kept, -1 dropped
    while (state == 0).any():
        live = (state[a] == 0) & (state[b] == 0)
        aa, bb = a[live], b[live]
        top = np.full(n, -1, dtype=prio.dtype)
        np.maximum.at(top, aa, prio[bb])
        win = (state == 0) & (prio > top)
        state[win] = 1
        state[bb[win[aa]]] = -1
    return state == 1


def _graded_band(rng, M, dim, center, radius, band, refine, jitter, regular_keys_mask_fn, separation=0.7):
    """Jittered fine lattice (spacing h/refine) inside the band around a round obstacle,
    thinned to a target spacing growing linearly from h/refine at the surface to h at the
    band edge; candidates too close to the surface or to a kept regular node are dropped.
    Thinning keeps every pair >= separation * target apart (_separation_thin): random
    Bernoulli thinning leaves near-coincident pairs whose RBF-FD Laplacian rows carry
    growing modes under the explicit step (config 3 diverged at step 35 on that set)."""
    h = 1.0 / M
    hf = h / refine
    Mf = int(np.floor(1.0 / hf))
    lo = np.floor((np.asarray(center) - radius - band) / hf).astype(int) - 1
    hi = np.ceil((np.asarray(center) + radius + band) / hf).astype(int) + 1
    axes = [np.arange(max(1, lo[a]), min(Mf, hi[a])) for a in range(dim)]
    g = np.meshgrid(*axes, indexing="ij")
    fk = np.stack([x.ravel() for x in g], axis=-1)
    pts = fk * hf + rng.uniform(-jitter * hf, jitter * hf, fk.shape)
    dist = np.linalg.norm(pts - np.asarray(center), axis=1) - radius
    target = hf + (h - hf) * np.clip(dist / band, 0.0, 1.0)
    keep = (dist > 0.5 * hf) & (dist < band)
    pts, target = pts[keep], target[keep]
    # stay >= 0.5*target away from the nearest lattice node if that node is regular
    near = np.rint(pts / h).astype(np.int64)
    dnear = np.linalg.norm(pts - near * h, axis=1)
    is_reg = regular_keys_mask_fn(near)
    ok = ~(is_reg & (dnear < 0.5 * target))
    pts, target = pts[ok], target[ok]
    sel = _separation_thin(pts, separation * target, rng)
    return pts[sel], target[sel]


def hybrid_hole_2d(M: int = 500, seed: int = 2, radius: float = 0.2, band: float = 0.08,
                   refine: int = 2, jitter: float = 0.35, center=(0.5, 0.5)) -> NodeSet:
    """Configs 2/3: unit square minus a hole; regular 5-point lattice away from the hole,
    scattered graded band of width `band` around it (hole-only band, H10)."""
    rng = np.random.default_rng(seed)
    h = 1.0 / M
    c = np.asarray(center, float)
    keys = _interior_keys(M, 2)
    d_lat = np.linalg.norm(keys * h - c, axis=1) - radius
    reg_keys = keys[d_lat >= band]

    def is_regular(k):
        inside = np.all((k >= 1) & (k <= M - 1), axis=1)
        d = np.linalg.norm(k * h - c, axis=1) - radius
        return inside & (d >= band)

    spts, sh = _graded_band(rng, M, 2, c, radius, band, refine, jitter, is_regular)
    hf = h / refine
    nb = int(round(2 * np.pi * radius / hf))
    th = 2 * np.pi * np.arange(nb) / nb
    nrm = np.stack([np.cos(th), np.sin(th)], axis=1)
    hole = c + radius * nrm
    wk, wn, wo = _box_walls(M, 2)
    return _assemble(2, M, reg_keys, spts, sh, wk, wn, wo, hole, nrm, ["obstacle:0"] * nb, np.full(nb, hf))


def _fibonacci_sphere(center, radius, n):
    i = np.arange(n) + 0.5
    phi = np.arccos(1 - 2 * i / n)
    theta = np.pi * (1 + 5 ** 0.5) * i
    u = np.stack([np.cos(theta) * np.sin(phi), np.sin(theta) * np.sin(phi), np.cos(phi)], axis=1)
    return np.asarray(center) + radius * u, u


def hybrid_sphere_3d(M: int = 92, seed: int = 4, radius: float = 0.2, band: float = 0.08,
                     refine: int = 2, jitter: float = 0.35, center=(0.5, 0.5, 0.5)) -> NodeSet:
    """Config 4: unit cube minus a sphere; regular 7-point lattice away from the sphere,
    graded scattered band around it (2x refined toward the surface, H10)."""
    rng = np.random.default_rng(seed)
    h = 1.0 / M
    c = np.asarray(center, float)
    keys = _interior_keys(M, 3)
    d_lat = np.linalg.norm(keys * h - c, axis=1) - radius
    reg_keys = keys[d_lat >= band]

    def is_regular(k):
        inside = np.all((k >= 1) & (k <= M - 1), axis=1)
        d = np.linalg.norm(k * h - c, axis=1) - radius
        return inside & (d >= band)

    spts, sh = _graded_band(rng, M, 3, c, radius, band, refine, jitter, is_regular)
    hf = h / refine
    nsph = max(8, int(round(8 * np.pi * radius ** 2 / (np.sqrt(3.0) * hf * hf))))
    sph, nrm = _fibonacci_sphere(c, radius, nsph)
    wk, wn, wo = _box_walls(M, 3)
    return _assemble(3, M, reg_keys, spts, sh, wk, wn, wo, sph, nrm, ["obstacle:0"] * nsph, np.full(nsph, hf))


def sinusoid_field(positions: np.ndarray, seed: int = 7, terms: int = 16) -> np.ndarray:
    """BASELINE test field u = sum_k a_k prod_a sin(k_a pi x_a), (k) ~ U{1..8}^d, a ~ N(0,1)."""
    rng = np.random.default_rng(seed)
    dim = positions.shape[1]
    ks = rng.integers(1, 9, size=(terms, dim))
    amp = rng.normal(size=terms)
    out = np.zeros(len(positions))
    for k, a in zip(ks, amp):
        term = np.full(len(positions), a)
        for ax in range(dim):
            term = term * np.sin(k[ax] * np.pi * positions[:, ax])
        out += term
    return out


CONFIGS = {
    0: dict(name="config0: 2D regular 200x200 (N=40,000), MON 5-point", build=lambda: regular_box(199)),
    1: dict(name="config1: 2D scattered jittered M=315 (N=99,856), RBF-FD n=12 (18x18)",
            build=lambda: jittered_box(315, seed=1)),
    2: dict(name="config2: 2D hybrid hole M=500 (N~247.6K), MON 5 + RBF-FD 12",
            build=lambda: hybrid_hole_2d(500, seed=2)),
    4: dict(name="config4: 3D hybrid sphere (N~1e6), MON 7 + RBF-FD n=20 (30x30)",
            build=lambda: hybrid_sphere_3d(92, seed=4)),
}
