"""Domains for node generation: box minus obstacles, evaluated by the K12 device kernels.

Reference: pkg/src/hybridnodes/geometry.py (shapes :37-199, DomainSpec :253-312,
boundary sampling :362-518).  Shapes and the domain are plain parameter records here;
every signed-distance / spacing / region query over many points goes to `hn_geom_eval`
(csrc/nodegen.cu) -- box, circle and sphere in the reference's exact operation order
(bit-identical), star and ellipse by the same table + Newton scheme with the device's
sin/cos (equal to rounding).  Boundary sampling is O(surface) host set-up built from the
same numpy calls as the reference, with its spacing evaluated on the device.  A reference
`hybridnodes.geometry.DomainSpec` (or any object with lo / hi / obstacles whose shapes carry
the reference's fields) is accepted wherever a DomainSpec is.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib
from .errors import ConfigurationError

CURVE_TABLE = 1024  # geometry.py:21
DENSE_ARC = 4096    # geometry.py:22

BCPolicy = Callable[[str, np.ndarray], tuple]


def _points(x, dim: int):
    pts = np.asarray(x, dtype=float)
    single = pts.ndim == 1
    pts = np.atleast_2d(pts)
    if pts.shape[1] != dim:
        raise ValueError(f"expected points of dimension {dim}, got shape {pts.shape}")
    return pts, single


# ------------------------------------------------------------------ shapes
@dataclass(frozen=True)
class Circle:
    """Circle (2D) / sphere (3D) (reference geometry.py:37-54)."""

    center: tuple
    radius: float

    def __post_init__(self):
        if self.radius <= 0:
            raise ConfigurationError(f"degenerate obstacle: radius {self.radius} <= 0")
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))

    @property
    def dim(self) -> int:
        return len(self.center)

    def signed_distance(self, pts) -> np.ndarray:
        return _shape_eval(self, pts)


class _Curve:
    """Closed 2D curve parametrised by angle (reference geometry.py:57-101)."""

    @property
    def dim(self) -> int:
        return 2

    def signed_distance(self, pts) -> np.ndarray:
        return _shape_eval(self, pts)

    def boundary_points(self, spacing):
        """Samples at the local target spacing by arc-length inversion; (points, outward normals)."""
        t = np.linspace(0.0, 2 * np.pi, DENSE_ARC + 1)
        pts = _curve_point(self, t)
        speed = np.linalg.norm(_curve_velocity(self, t), axis=-1)
        dens = speed / spacing(pts)
        tau = np.concatenate([[0.0], np.cumsum((dens[1:] + dens[:-1]) / 2 * np.diff(t))])
        n = max(3, round(tau[-1]))
        ts = np.interp(np.arange(n) * tau[-1] / n, tau, t)
        p = _curve_point(self, ts)
        v = _curve_velocity(self, ts)
        nrm = np.stack([v[:, 1], -v[:, 0]], axis=-1)
        nrm /= np.linalg.norm(nrm, axis=-1, keepdims=True)
        return p, nrm


@dataclass(frozen=True)
class Ellipse(_Curve):
    """Rotated ellipse (reference geometry.py:104-145)."""

    center: tuple
    semi_axes: tuple
    angle: float = 0.0

    def __post_init__(self):
        if min(self.semi_axes) <= 0:
            raise ConfigurationError(f"degenerate obstacle: semi-axes {self.semi_axes}")
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))
        object.__setattr__(self, "semi_axes", tuple(float(a) for a in self.semi_axes))


@dataclass(frozen=True)
class Star(_Curve):
    """r(t) = mean + amplitude cos(lobes t + phase) (reference geometry.py:148-197)."""

    center: tuple
    mean_radius: float
    amplitude: float
    lobes: int
    phase: float = 0.0

    def __post_init__(self):
        if self.mean_radius <= 0:
            raise ConfigurationError(f"degenerate obstacle: radius {self.mean_radius} <= 0")
        if not 0 <= self.amplitude < self.mean_radius:
            raise ConfigurationError("star amplitude must satisfy 0 <= amplitude < mean radius")
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))


def _kind(shape) -> int:
    """0 circle/sphere, 1 star, 2 ellipse -- by the fields, so reference shapes drop in."""
    if hasattr(shape, "lobes"):
        return 1
    if hasattr(shape, "semi_axes"):
        return 2
    if hasattr(shape, "radius"):
        return 0
    raise TypeError(f"unsupported obstacle shape {type(shape).__name__}")


def _rot(shape):
    c, s = math.cos(shape.angle), math.sin(shape.angle)
    return np.array([[c, -s], [s, c]])


def _curve_point(shape, t):
    c = np.asarray(shape.center)
    if _kind(shape) == 1:
        r = shape.mean_radius + shape.amplitude * np.cos(shape.lobes * t + shape.phase)
        return c + r[..., None] * np.stack([np.cos(t), np.sin(t)], axis=-1)
    a, b = shape.semi_axes
    return c + np.stack([a * np.cos(t), b * np.sin(t)], axis=-1) @ _rot(shape).T


def _curve_velocity(shape, t):
    if _kind(shape) == 1:
        u = np.stack([np.cos(t), np.sin(t)], axis=-1)
        du = np.stack([-np.sin(t), np.cos(t)], axis=-1)
        arg = shape.lobes * t + shape.phase
        rp = -shape.amplitude * shape.lobes * np.sin(arg)
        r = shape.mean_radius + shape.amplitude * np.cos(arg)
        return rp[..., None] * u + r[..., None] * du
    a, b = shape.semi_axes
    return np.stack([-a * np.sin(t), b * np.cos(t)], axis=-1) @ _rot(shape).T


@dataclass(frozen=True)
class Obstacle:
    """Solid obstacle: Dirichlet wall temperature, or insulated if None (geometry.py:202-210)."""

    shape: object
    temperature: float | None = None

    def signed_distance(self, pts) -> np.ndarray:
        return self.shape.signed_distance(pts)


class BoundarySet:
    """Array-of-fields boundary samples (reference geometry.py:221-250)."""

    def __init__(self, positions, normals, bc_kind, bc_value, origin):
        self.positions = np.asarray(positions, dtype=float)
        self.normals = np.asarray(normals, dtype=float)
        self.bc_kind = list(bc_kind)
        self.bc_value = np.asarray(bc_value, dtype=float)
        self.origin = list(origin)

    def __len__(self) -> int:
        return len(self.positions)

    @staticmethod
    def concatenate(parts):
        parts = [p for p in parts if len(p)]
        if not parts:
            raise ValueError("no boundary samples")
        return BoundarySet(np.concatenate([p.positions for p in parts]),
                           np.concatenate([p.normals for p in parts]),
                           [k for p in parts for k in p.bc_kind], np.concatenate([p.bc_value for p in parts]),
                           [o for p in parts for o in p.origin])


# ------------------------------------------------------------------ domain
class DomainSpec:
    """Axis-aligned box minus non-overlapping obstacles (reference geometry.py:253-312)."""

    def __init__(self, lo, hi, obstacles=()):
        self.lo = np.asarray(lo, dtype=float)
        self.hi = np.asarray(hi, dtype=float)
        if self.lo.shape != self.hi.shape or self.lo.ndim != 1:
            raise ConfigurationError("box corners must be points of equal dimension")
        if not np.all(self.hi > self.lo):
            raise ConfigurationError("box upper corner must exceed lower corner")
        self.obstacles = tuple(obstacles)
        if self.dim not in (2, 3):
            raise ConfigurationError(f"only 2D and 3D domains supported, got d={self.dim}")
        for obs in self.obstacles:
            if obs.shape.dim != self.dim:
                raise ConfigurationError("obstacle dimension does not match the box")
            if self.dim == 3 and _kind(obs.shape) != 0:
                raise ConfigurationError("3D domains support spherical obstacles only")

    @property
    def dim(self) -> int:
        return len(self.lo)

    @property
    def extent(self) -> np.ndarray:
        return self.hi - self.lo

    def _eval(self, x, mode):
        pts, single = _points(x, self.dim)
        out = DeviceGeometry(self).eval(pts, mode)
        return out[0] if single else out

    def box_signed_distance(self, x):
        return self._eval(x, 3)

    def obstacle_distance(self, x):
        """Signed distance to the nearest obstacle surface (+inf with no obstacles)."""
        return self._eval(x, 1)

    def signed_distance(self, x):
        return self._eval(x, 0)

    def contains(self, x, margin: float = 0.0):
        return self.signed_distance(x) <= -margin

    def validate_clearances(self, min_gap: float) -> None:
        """Obstacles strictly inside the box with min_gap between surfaces (geometry.py:308-319)."""
        validate_clearances(self, min_gap)


def signed_distance(spec, x):
    """Signed distance to the fluid region: negative inside, zero on the boundary."""
    pts, single = _points(x, len(spec.lo))
    out = DeviceGeometry(spec).eval(pts, 0)
    return out[0] if single else out


def _probe_surface(shape, n: int = 512) -> np.ndarray:
    if _kind(shape) == 0 and shape.dim == 3:
        return fibonacci_sphere(np.asarray(shape.center), shape.radius, n)
    t = np.linspace(0, 2 * np.pi, n, endpoint=False)
    if _kind(shape) == 0:
        return np.asarray(shape.center) + shape.radius * np.stack([np.cos(t), np.sin(t)], axis=-1)
    return _curve_point(shape, t)


def validate_clearances(spec, min_gap: float) -> None:
    for i, obs in enumerate(spec.obstacles):
        pts = _probe_surface(obs.shape)
        if np.any(DeviceGeometry(spec).eval(pts, 3) > -min_gap):
            raise ConfigurationError(f"obstacle {i} too close to the box walls")
        for j, other in enumerate(spec.obstacles):
            if j != i and np.any(_shape_eval(other.shape, pts) < min_gap):
                raise ConfigurationError(f"obstacles {i} and {j} closer than {min_gap}")


def fibonacci_sphere(center, radius: float, n: int) -> np.ndarray:
    """Fibonacci lattice on a sphere (reference geometry.py:334-341)."""
    i = np.arange(n)
    z = 1.0 - 2.0 * (i + 0.5) / n
    phi = i * np.pi * (3.0 - np.sqrt(5.0))
    rho = np.sqrt(1.0 - z * z)
    return np.asarray(center) + radius * np.stack([rho * np.cos(phi), rho * np.sin(phi), z], axis=-1)


def default_bc_policy(spec) -> BCPolicy:
    """Insulated walls; obstacles Dirichlet at their temperature, else insulated."""

    def policy(origin, position):
        if origin.startswith("obstacle:"):
            t = spec.obstacles[int(origin.split(":")[1])].temperature
            return ("neumann", 0.0) if t is None else ("dirichlet", float(t))
        return ("neumann", 0.0)

    return policy


# ------------------------------------------------------------------ device geometry
class _Geom(C.Structure):
    """hn_geom (include/hn.h)."""
    _fields_ = [("dim", C.c_int), ("n_obs", C.c_int), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("graded", C.c_int), ("h_r", C.c_double), ("h_s", C.c_double), ("width", C.c_double),
                ("obs_kind", C.c_void_p), ("obs_par", C.c_void_p), ("curve_t", C.c_void_p),
                ("curve_tab", C.c_void_p), ("region", C.c_int), ("axis", C.c_int), ("rc", C.c_double * 2),
                ("rt", C.c_double * 2)]


REGION_NONE, REGION_ALL, REGION_QUARTERS, REGION_SPLIT, REGION_LAYER = range(5)


class DeviceGeometry:
    """The hn_geom record of a domain (+ spacing function + scattered region), with the
    obstacle parameters and curve tables resident on the device."""

    def __init__(self, spec, spacing=None, region=None):
        self.spec = spec
        d = len(spec.lo)
        g = _Geom()
        g.dim = d
        g.n_obs = len(spec.obstacles)
        for a in range(d):
            g.lo[a], g.hi[a] = float(spec.lo[a]), float(spec.hi[a])
        self._keep = []
        if spec.obstacles:
            kinds, par, tabs = [], np.zeros((len(spec.obstacles), 8)), np.zeros((len(spec.obstacles), CURVE_TABLE, 2))
            t_tab = np.linspace(0.0, 2 * np.pi, CURVE_TABLE, endpoint=False)
            for j, obs in enumerate(spec.obstacles):
                sh = obs.shape
                k = _kind(sh)
                kinds.append(k)
                if k == 0:
                    par[j, :d] = sh.center
                    par[j, d] = sh.radius
                elif k == 1:
                    par[j, :6] = (*sh.center, sh.mean_radius, sh.amplitude, float(sh.lobes), sh.phase)
                else:
                    c, s = _rot(sh)[0, 0], _rot(sh)[1, 0]
                    par[j, :6] = (*sh.center, *sh.semi_axes, c, s)
                if k:
                    tabs[j] = _curve_point(sh, t_tab)
            dk, dp, dt, dtab = _lib.to_device_many([np.asarray(kinds, np.int32), par, t_tab, tabs])
            self._keep += [dk, dp, dt, dtab]
            g.obs_kind, g.obs_par, g.curve_t, g.curve_tab = (x.data_ptr() for x in (dk, dp, dt, dtab))
        g.graded = 0
        g.h_r = g.h_s = 1.0
        if spacing is not None:
            g.h_r, g.h_s = float(spacing.h_r), float(spacing.h_s)
            g.width = float(spacing.delta_h * spacing.h_r)
            g.graded = int(spacing.boundary_distance is not None and spacing.h_s != spacing.h_r
                           and spacing.delta_h != 0)
        g.region = REGION_NONE
        if region is not None:
            g.region = region.code
            g.axis = region.axis
            g.rc[0], g.rc[1] = region.rc
            g.rt[0], g.rt[1] = region.rt
        self.g = g

    def ref(self) -> int:
        return C.addressof(self.g)

    def eval(self, pts, mode: int) -> np.ndarray:
        """mode 0 sd, 1 obstacle distance, 2 spacing, 3 box sd, 4 region, 5 near-region."""
        pts = np.ascontiguousarray(pts, dtype=float)
        if len(pts) == 0:
            return np.empty(0)
        dp = _lib.to_device(pts)
        out = _lib.empty((len(pts),), _lib.torch().float64)
        _lib.call("hn_geom_eval", self.ref(), _lib.ptr(dp), len(pts), mode, _lib.ptr(out), _lib.stream_handle())
        return out.cpu().numpy()

    def eval_device(self, dpts, mode: int):
        out = _lib.empty((dpts.shape[0],), _lib.torch().float64)
        if dpts.shape[0]:
            _lib.call("hn_geom_eval", self.ref(), _lib.ptr(dpts), dpts.shape[0], mode, _lib.ptr(out),
                      _lib.stream_handle())
        return out


def _shape_eval(shape, pts) -> np.ndarray:
    """One shape's signed distance (negative inside the solid) on the device."""
    pts, single = _points(pts, shape.dim)
    d = len(shape.center)
    box = DomainSpec(np.full(d, -1e300), np.full(d, 1e300), (Obstacle(shape),))
    out = DeviceGeometry(box).eval(pts, 1)
    return out[0] if single else out


# ------------------------------------------------------------------ boundary sampling
def _sample_segment(a, b, spacing, include_ends: bool = False) -> np.ndarray:
    """Points along a -> b at the local target spacing (geometry.py:362-377)."""
    a, b = np.asarray(a, float), np.asarray(b, float)
    length = float(np.linalg.norm(b - a))
    s = np.linspace(0.0, 1.0, DENSE_ARC + 1)
    dens = length / spacing(a + s[:, None] * (b - a))
    tau = np.concatenate([[0.0], np.cumsum((dens[1:] + dens[:-1]) / 2 * np.diff(s))])
    n = max(1, round(tau[-1]))
    targets = np.arange(n + 1) * tau[-1] / n if include_ends else np.arange(1, n) * tau[-1] / n
    return a + np.interp(targets, tau, s)[:, None] * (b - a)


def _box_walls_2d(spec, spacing) -> BoundarySet:
    """Corners (owned by the x walls), then the x-, x+, y-, y+ wall interiors (geometry.py:380-405)."""
    lo, hi = spec.lo, spec.hi
    pos = [np.array([lo[0], lo[1]]), np.array([lo[0], hi[1]]), np.array([hi[0], lo[1]]), np.array([hi[0], hi[1]])]
    nrm = [np.array([-1.0, 0.0])] * 2 + [np.array([1.0, 0.0])] * 2
    tags = ["wall:x-"] * 2 + ["wall:x+"] * 2
    walls = (("wall:x-", (lo[0], lo[1]), (lo[0], hi[1]), (-1.0, 0.0)),
             ("wall:x+", (hi[0], lo[1]), (hi[0], hi[1]), (1.0, 0.0)),
             ("wall:y-", (lo[0], lo[1]), (hi[0], lo[1]), (0.0, -1.0)),
             ("wall:y+", (lo[0], hi[1]), (hi[0], hi[1]), (0.0, 1.0)))
    for tag, a, b, n in walls:
        seg = _sample_segment(np.array(a), np.array(b), spacing)
        pos += list(seg)
        nrm += [np.array(n)] * len(seg)
        tags += [tag] * len(seg)
    return BoundarySet(np.array(pos), np.array(nrm), ["neumann"] * len(pos), np.zeros(len(pos)), tags)


def _box_walls_3d(spec, spacing) -> BoundarySet:
    """Corners (x walls), edges (lowest non-edge axis), face interiors (geometry.py:408-458)."""
    lo, hi = spec.lo, spec.hi
    pos, nrm, tags = [], [], []
    for xi, xv in enumerate((lo[0], hi[0])):
        for yv in (lo[1], hi[1]):
            for zv in (lo[2], hi[2]):
                pos.append(np.array([xv, yv, zv], float))
                nrm.append(np.array([-1.0 if xi == 0 else 1.0, 0.0, 0.0]))
                tags.append(f"wall:x{'-+'[xi]}")
    for axis in range(3):
        u, v = [a for a in range(3) if a != axis]
        for uv in (lo[u], hi[u]):
            for vv in (lo[v], hi[v]):
                a, b = np.zeros(3), np.zeros(3)
                a[axis], b[axis] = lo[axis], hi[axis]
                a[u] = b[u] = uv
                a[v] = b[v] = vv
                sgn = -1.0 if uv == lo[u] else 1.0
                n_vec = np.zeros(3)
                n_vec[u] = sgn
                h_edge = float(np.min(spacing(a + np.linspace(0, 1, 33)[:, None] * (b - a))))
                n = max(1, round(float(np.linalg.norm(b - a)) / h_edge))
                for s in np.arange(1, n) / n:
                    pos.append(a + s * (b - a))
                    nrm.append(n_vec)
                    tags.append(f"wall:{'xyz'[u]}{'-' if sgn < 0 else '+'}")
    for axis in range(3):
        u, v = [a for a in range(3) if a != axis]
        for side, val in ((0, lo[axis]), (1, hi[axis])):
            n_vec = np.zeros(3)
            n_vec[axis] = -1.0 if side == 0 else 1.0
            probe = np.zeros((17 * 17, 3))
            probe[:, axis] = val
            probe[:, u] = np.repeat(np.linspace(lo[u], hi[u], 17), 17)
            probe[:, v] = np.tile(np.linspace(lo[v], hi[v], 17), 17)
            h_face = float(np.min(spacing(probe)))
            nu = max(1, round((hi[u] - lo[u]) / h_face))
            nv = max(1, round((hi[v] - lo[v]) / h_face))
            su = lo[u] + np.arange(1, nu) * (hi[u] - lo[u]) / nu
            sv = lo[v] + np.arange(1, nv) * (hi[v] - lo[v]) / nv
            face = np.zeros((len(su) * len(sv), 3))
            face[:, axis] = val
            face[:, u] = np.repeat(su, len(sv))
            face[:, v] = np.tile(sv, len(su))
            pos += list(face)
            nrm += [n_vec] * len(face)
            tags += [f"wall:{'xyz'[axis]}{'-' if side == 0 else '+'}"] * len(face)
    return BoundarySet(np.array(pos), np.array(nrm), ["neumann"] * len(pos), np.zeros(len(pos)), tags)


def _obstacle_samples(spec, idx: int, spacing) -> BoundarySet:
    """Fibonacci sphere at hexagonal-packing density (3D) or arc-length samples (2D)
    (geometry.py:461-477)."""
    shape = spec.obstacles[idx].shape
    k = _kind(shape)
    if k == 0 and shape.dim == 3:
        c = np.asarray(shape.center)
        h = float(np.min(spacing(c[None, :] + np.array([[shape.radius, 0.0, 0.0]]))))
        n = max(8, round(8 * np.pi * shape.radius**2 / (np.sqrt(3.0) * h * h)))
        pts = fibonacci_sphere(c, shape.radius, n)
        nrm = (pts - c) / shape.radius
    elif k == 0:
        pts, nrm = Star(shape.center, shape.radius, 0.0, 1).boundary_points(spacing)
    else:
        pts, nrm = _Curve.boundary_points(shape, spacing)
    return BoundarySet(pts, nrm, ["neumann"] * len(pts), np.zeros(len(pts)), [f"obstacle:{idx}"] * len(pts))


def discretize_boundary(spec, spacing, bc_policy: BCPolicy | None = None) -> BoundarySet:
    """Whole domain boundary at the local target spacing, with BCs from the policy
    (reference geometry.py:498-518)."""
    for obs in spec.obstacles:
        radius = getattr(obs.shape, "radius", None) or getattr(obs.shape, "mean_radius", 1.0)
        if radius <= 0:
            raise ConfigurationError("degenerate obstacle: radius <= 0")
    policy = bc_policy if bc_policy is not None else default_bc_policy(spec)
    parts = [_box_walls_2d(spec, spacing) if len(spec.lo) == 2 else _box_walls_3d(spec, spacing)]
    parts += [_obstacle_samples(spec, i, spacing) for i in range(len(spec.obstacles))]
    out = BoundarySet.concatenate(parts)
    for i in range(len(out)):
        kind, value = policy(out.origin[i], out.positions[i])
        if kind not in ("dirichlet", "neumann"):
            raise ConfigurationError(f"unknown boundary condition kind {kind!r}")
        out.bc_kind[i] = kind
        out.bc_value[i] = value
    return out
