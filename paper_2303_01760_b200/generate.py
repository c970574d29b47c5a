"""Node-set generation on the device: lattice fill, region cut,
advancing-front scattered fill and the lattice index map, as K12 kernels (csrc/nodegen.cu).

Reference: pkg/src/hybridnodes/nodegen.py -- SpacingFunction :33-60, RegularFill /
regular_fill :182-216, carve_transition :219-227, _wave_candidates :270-294,
scattered_fill :297-381, _scattered_region :384-433, hybrid_discretize :436-518.

Same names, arguments, results and errors as the reference.  The random draws of every
front wave come from the reference's own numpy Generator calls (standard_normal, then
random, per wave), so a wave's candidate directions are the reference's; the candidates,
the in-domain / region tests, the first-fit acceptance (csrc/nodegen.cu: pre-test + in-order
sync-free resolution, the sequential loop's exact accept set) and the append all run on the
device, one host read of the new-node count per wave.  Box / circle / sphere domains give
the reference's node sets bit for bit; star / ellipse obstacles agree to rounding (device
sin/cos).  Boundary sampling is O(surface) set-up (geometry.discretize_boundary).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigurationError
from .geometry import (REGION_ALL, REGION_LAYER, REGION_NONE, REGION_QUARTERS, REGION_SPLIT, BoundarySet,
                       DeviceGeometry, DomainSpec, discretize_boundary)
from .nodegen import (KIND_BOUNDARY, KIND_REGULAR, KIND_SCATTERED, LATTICE_NONE, ROLE_DIRICHLET, ROLE_INTERIOR,
                      ROLE_NEUMANN, LatticeInfo, NodeSet)

ACCEPT = 0.995  # nodegen.py:31


@dataclass
class SpacingFunction:
    """Target spacing: h_s on the obstacles, growing linearly to h_r at delta_h*h_r, h_r beyond
    (reference nodegen.py:33-60).  boundary_distance: a DomainSpec's obstacle_distance (or None)."""

    h_r: float
    h_s: float
    delta_h: float
    boundary_distance: object = None

    def __post_init__(self):
        if self.h_s > self.h_r:
            raise ConfigurationError("h_s must not exceed h_r")

    @property
    def transition_width(self) -> float:
        return self.delta_h * self.h_r

    def __call__(self, pts) -> np.ndarray:
        pts = np.atleast_2d(np.asarray(pts, dtype=float))
        if self.boundary_distance is None or self.h_s == self.h_r or self.delta_h == 0:
            return np.full(len(pts), self.h_r)
        return _device_geometry(_spec_of(self), self).eval(pts, 2)


def _spec_of(spacing):
    """The domain whose obstacle_distance grades `spacing` (bound method of a DomainSpec)."""
    bd = getattr(spacing, "boundary_distance", None)
    spec = getattr(bd, "__self__", None)
    if spec is None or not hasattr(spec, "obstacles"):
        raise TypeError("spacing.boundary_distance must be a DomainSpec's obstacle_distance "
                        "(the device evaluates the domain's own geometry)")
    return spec


_GEOM_CACHE: dict = {}


def _device_geometry(spec, spacing=None, region=None) -> DeviceGeometry:
    """DeviceGeometry per (domain, spacing, region) -- one upload of the obstacle tables."""
    key = (id(spec), None if spacing is None else (spacing.h_r, spacing.h_s, spacing.delta_h,
                                                   spacing.boundary_distance is not None),
           None if region is None else (region.code, region.axis, region.rc, region.rt))
    hit = _GEOM_CACHE.get(key)
    if hit is not None and hit.spec is spec:
        return hit
    if len(_GEOM_CACHE) > 64:
        _GEOM_CACHE.clear()
    g = DeviceGeometry(spec, spacing, region)
    _GEOM_CACHE[key] = g
    return g


@dataclass(frozen=True)
class Region:
    """A scattered-region predicate the device evaluates (reference nodegen.py:384-433):
    code REGION_*, split axis, quarters centre rc, thresholds rt = (region, near-region)."""

    spec: object
    code: int
    axis: int = 0
    rc: tuple = (0.0, 0.0)
    rt: tuple = (0.0, 0.0)
    near: bool = False

    def __call__(self, pts) -> np.ndarray:
        pts = np.atleast_2d(np.asarray(pts, dtype=float))
        return _device_geometry(self.spec, None, self).eval(pts, 5 if self.near else 4) != 0.0

    def dilated(self) -> "Region":
        return Region(self.spec, self.code, self.axis, self.rc, self.rt, True)


def _scattered_region(config, spec, step_max: float):
    """(region, near_region) of the case (reference nodegen.py:384-433); (None, None) = no
    scattered zone."""
    mode = config.discretization
    reach = 2.0 * step_max
    if mode == "pure-regular":
        return None, None
    if mode == "pure-scattered":
        r = Region(spec, REGION_ALL)
        return r, r.dilated()
    if config.case == "dvd":
        c = (spec.lo + spec.hi) / 2.0
        r = Region(spec, REGION_QUARTERS, rc=(float(c[0]), float(c[1])), rt=(0.0, reach))
        return r, r.dilated()
    if config.case == "dvd-split":
        axis = 1 if config.split_orientation == "horizontal" else 0
        cut = spec.lo[axis] + config.delta_h * step_max
        r = Region(spec, REGION_SPLIT, axis=axis, rt=(float(cut), float(cut + reach)))
        return r, r.dilated()
    if not spec.obstacles:
        return None, None
    width = config.delta_h * step_max
    r = Region(spec, REGION_LAYER, rt=(float(width), float(width + reach)))
    return r, r.dilated()


@dataclass
class RegularFill:
    """Interior lattice nodes (reference nodegen.py:182-193)."""

    positions: np.ndarray
    indices: np.ndarray
    origin: np.ndarray
    step: np.ndarray
    cells: tuple

    def __len__(self) -> int:
        return len(self.positions)


def _lattice_frame(spec, h_r: float):
    if h_r <= 0:
        raise ConfigurationError("h_r must be positive")
    extent = spec.hi - spec.lo
    if np.any(h_r > extent):
        raise ConfigurationError(f"h_r={h_r} exceeds the domain extent {extent}")
    cells = tuple(max(1, round(float(e) / h_r)) for e in extent)
    step = extent / np.asarray(cells)
    return cells, step


def _lattice_device(spec, cells, step, region=None, carve: float = 0.0):
    """Kept lattice nodes on the device: (positions (K, d), keys (K, d) int64)."""
    d = len(spec.lo)
    total = int(np.prod([c - 1 for c in cells]))
    thr = -0.5 * float(np.max(step)) * (1 - 1e-12)
    pos = _lib.empty((max(total, 1), d), _lib.torch().float64)
    key = _lib.empty((max(total, 1), d), _lib.torch().int64)
    cnt = C.c_int64(0)
    g = _device_geometry(spec, None, region)
    _lib.call("hn_lattice_fill", g.ref(), _lib.host_i64(cells), _lib.host_dbls(step), thr,
              int(region is not None), float(carve), _lib.ptr(pos), _lib.ptr(key), C.byref(cnt), _lib.stream_handle())
    k = int(cnt.value)
    return pos[:k], key[:k]


def regular_fill(spec, h_r: float) -> RegularFill:
    """Axis-aligned interior lattice, nodes within h_r/2 of the boundary excluded; the spacing
    snaps to extent/round(extent/h_r) (reference nodegen.py:196-216)."""
    cells, step = _lattice_frame(spec, h_r)
    pos, key = _lattice_device(spec, cells, step)
    return RegularFill(pos.cpu().numpy(), key.cpu().numpy(), np.asarray(spec.lo, float).copy(), step, cells)


def carve_transition(fill: RegularFill, spec, delta_h: float, h_r: float) -> RegularFill:
    """Drop lattice nodes within delta_h*h_r of an obstacle surface (reference nodegen.py:219-227)."""
    if delta_h == 0 or not spec.obstacles:
        return fill
    keep = _device_geometry(spec).eval(fill.positions, 1) >= delta_h * h_r
    return RegularFill(fill.positions[keep], fill.indices[keep], fill.origin, fill.step, fill.cells)


class _Front:
    """Device state of one advancing-front fill: node positions / spacings with room to grow."""

    def __init__(self, seeds_dev, h_dev):
        t = _lib.torch()
        self.d = seeds_dev.shape[1]
        self.count = seeds_dev.shape[0]
        self.pts = t.empty((max(2 * self.count, 1024), self.d), dtype=t.float64, device=seeds_dev.device)
        self.hs = t.empty((self.pts.shape[0],), dtype=t.float64, device=seeds_dev.device)
        self.pts[: self.count] = seeds_dev
        self.hs[: self.count] = h_dev

    def reserve(self, extra: int):
        need = self.count + extra
        if need <= self.pts.shape[0]:
            return
        t = _lib.torch()
        cap = max(need, 2 * self.pts.shape[0])
        pts = t.empty((cap, self.d), dtype=t.float64, device=self.pts.device)
        hs = t.empty((cap,), dtype=t.float64, device=self.pts.device)
        pts[: self.count] = self.pts[: self.count]
        hs[: self.count] = self.hs[: self.count]
        self.pts, self.hs = pts, hs


def _fill_device(spec, seeds_dev, spacing, rng_seed: int, region=None, seed_regular=None, h_regular=None,
                 queue_filter=None) -> "_Front":
    """scattered_fill on device-resident seeds; returns the _Front (seeds first, then the
    accepted nodes in acceptance order)."""
    t = _lib.torch()
    d = seeds_dev.shape[1]
    n_seeds = seeds_dev.shape[0]
    _spacing_ok = spacing.boundary_distance is None or spacing.h_s == spacing.h_r or spacing.delta_h == 0
    spec_g = spec if _spacing_ok else _spec_of(spacing)
    dev_region = region if isinstance(region, Region) else None
    g = _device_geometry(spec_g if spec_g is not None else spec, spacing, dev_region)
    h_seed = g.eval_device(seeds_dev, 2)
    front = _Front(seeds_dev, h_seed)
    rng = np.random.default_rng(rng_seed)
    seam = 0.9 * h_regular if h_regular is not None else 0.0
    cell = max(float(spacing.h_r), seam) * (1 + 1e-12)
    lo, hi = _lib.host_dbls(spec.lo), _lib.host_dbls(spec.hi)
    sreg = None
    if seed_regular is not None and h_regular is not None:
        sreg = _lib.to_device(np.asarray(seed_regular, dtype=np.uint8))
    if queue_filter is None:
        front_ids, k, front_lo = None, n_seeds, 0
    else:
        ids = np.nonzero(np.asarray(queue_filter))[0].astype(np.int64)
        front_ids, k, front_lo = (_lib.to_device(ids) if len(ids) else None), len(ids), 0
    n_dir = 3 * d + 1
    while k > 0:
        rnd = rng.standard_normal((k, d + 1, d))
        u = rng.random((k, n_dir))
        drnd, du = _lib.to_device_many([rnd, u])
        m = k * n_dir
        cand = t.empty((m, d), dtype=t.float64, device=seeds_dev.device)
        hcand = t.empty((m,), dtype=t.float64, device=seeds_dev.device)
        ok = t.empty((m,), dtype=t.uint8, device=seeds_dev.device)
        _lib.call("hn_front_candidates", g.ref(), _lib.ptr(front.pts), _lib.ptr(front.hs), _lib.ptr(front_ids),
                  front_lo, k, _lib.ptr(drnd), _lib.ptr(du), int(dev_region is not None), _lib.ptr(cand),
                  _lib.ptr(hcand), _lib.ptr(ok), _lib.stream_handle())
        if region is not None and dev_region is None:
            # a caller-supplied Python predicate (e.g. a lambda) runs where it lives
            mask = np.asarray(region(cand.cpu().numpy()), dtype=bool)
            ok &= _lib.to_device(mask.astype(np.uint8))
        front.reserve(m)
        new = C.c_int64(0)
        _lib.call("hn_front_accept", d, _lib.ptr(front.pts), _lib.ptr(front.hs), front.count, front.pts.shape[0],
                  _lib.ptr(sreg), n_seeds if sreg is not None else 0, _lib.ptr(cand), _lib.ptr(hcand),
                  _lib.ptr(ok), m, seam, lo, hi, cell, C.byref(new), _lib.stream_handle())
        front_ids, front_lo, k = None, front.count, int(new.value) - front.count
        front.count = int(new.value)
    return front


def scattered_fill(spec, seed_positions, spacing, rng_seed: int, region=None, seed_regular_mask=None,
                   h_regular: float | None = None, queue_filter=None) -> np.ndarray:
    """Advancing-front fill of the scattered region (reference nodegen.py:297-381): FIFO waves,
    candidates on spheres of the local target spacing around the popped nodes, accepted when
    inside the domain (and region) and no closer than 0.995 of their own spacing to any
    node (0.9*h_regular to regular seeds).  Deterministic for a fixed rng_seed."""
    seeds = np.atleast_2d(np.asarray(seed_positions, dtype=float))
    if len(seeds) == 0 or seeds.size == 0:
        return np.empty((0, spec.dim if hasattr(spec, "dim") else len(spec.lo)))
    front = _fill_device(spec, _lib.to_device(seeds), spacing, rng_seed, region, seed_regular_mask, h_regular,
                         queue_filter)
    return front.pts[len(seeds): front.count].cpu().numpy()


def _bc_policy(config, spec):
    if callable(getattr(config, "bc_policy", None)):
        return config.bc_policy(spec)
    from .config import bc_policy
    return bc_policy(config, spec)


def hybrid_discretize(config, spec=None) -> NodeSet:
    """The case's node set: lattice, region cut, boundary, scattered fill, lattice map
    (reference nodegen.py:436-518); every per-node step on the device."""
    if spec is None:
        from .config import build_domain
        spec = build_domain(config)
    t = _lib.torch()
    d = len(spec.lo)
    cells, step = _lattice_frame(spec, config.h_r)
    step_max = float(np.max(step))
    h_s = config.h_s if config.h_s < config.h_r else step_max
    spacing = SpacingFunction(step_max, h_s, config.delta_h, spec.obstacle_distance if spec.obstacles else None)
    region, near = _scattered_region(config, spec, step_max)
    if config.discretization == "pure-scattered":
        kept_pos = t.empty((0, d), dtype=t.float64, device=_lib.device())
        kept_key = t.empty((0, d), dtype=t.int64, device=_lib.device())
    else:
        kept_pos, kept_key = _lattice_device(spec, cells, step, region)
    boundary = discretize_boundary(spec, spacing, _bc_policy(config, spec))
    bpos = _lib.to_device(boundary.positions)
    n_r, n_b = kept_pos.shape[0], len(boundary)
    if config.discretization == "pure-regular" or region is None:
        scat = t.empty((0, d), dtype=t.float64, device=_lib.device())
        scat_h = t.empty((0,), dtype=t.float64, device=_lib.device())
    else:
        seeds = t.cat([bpos, kept_pos]) if n_r else bpos
        seed_reg = np.concatenate([np.zeros(n_b, bool), np.ones(n_r, bool)])
        queue = _device_geometry(spec, None, near).eval_device(seeds, 5).cpu().numpy() != 0.0
        front = _fill_device(spec, seeds, spacing, config.rng_seed, region, seed_reg, step_max, queue)
        scat, scat_h = front.pts[n_b + n_r: front.count], front.hs[n_b + n_r: front.count]
    n_s = scat.shape[0]
    if n_r + n_s == 0:
        raise ConfigurationError("discretization produced zero interior nodes")
    g = _device_geometry(spec, spacing)
    h = t.cat([t.full((n_r,), step_max, dtype=t.float64, device=_lib.device()), g.eval_device(scat, 2),
               g.eval_device(bpos, 2)])
    positions = t.cat([kept_pos, scat, bpos]).cpu().numpy()
    kind = np.concatenate([np.full(n_r, KIND_REGULAR), np.full(n_s, KIND_SCATTERED),
                           np.full(n_b, KIND_BOUNDARY)]).astype(np.int8)
    role = np.concatenate([np.full(n_r + n_s, ROLE_INTERIOR),
                           [ROLE_DIRICHLET if k == "dirichlet" else ROLE_NEUMANN for k in boundary.bc_kind]])
    bc_value = np.concatenate([np.full(n_r + n_s, np.nan), boundary.bc_value])
    normals = np.concatenate([np.full((n_r + n_s, d), np.nan), boundary.normals])
    origin = [""] * (n_r + n_s) + list(boundary.origin)
    lattice = LatticeInfo(np.asarray(spec.lo, float).copy(), step, cells,
                          grid=np.empty(tuple(c + 1 for c in cells), dtype=np.int64))
    grid = t.empty(int(np.prod([c + 1 for c in cells])), dtype=t.int64, device=_lib.device())
    bkey = t.empty((max(n_b, 1), d), dtype=t.int64, device=_lib.device())
    _lib.call("hn_lattice_map", d, _lib.host_i64(cells), _lib.host_dbls(spec.lo), _lib.host_dbls(step),
              1e-9 * step_max, _lib.ptr(kept_key), n_r, _lib.ptr(bpos), n_b, n_r + n_s, _lib.ptr(grid),
              _lib.ptr(bkey), _lib.stream_handle())
    lattice.grid = grid.cpu().numpy().reshape(tuple(c + 1 for c in cells))
    lattice_idx = np.full((len(positions), d), LATTICE_NONE, dtype=np.int64)
    lattice_idx[:n_r] = kept_key.cpu().numpy()
    lattice_idx[n_r + n_s:] = bkey[:n_b].cpu().numpy()
    return NodeSet(positions, h.cpu().numpy(), kind, role, bc_value, normals, origin, lattice, lattice_idx)


__all__ = ["SpacingFunction", "RegularFill", "Region", "regular_fill", "carve_transition", "scattered_fill",
           "hybrid_discretize", "BoundarySet", "DomainSpec"]
