"""Node-set container consumed by the hot path (mirror of the reference container).

Reference: pkg/src/hybridnodes/nodegen.py:22-23 (KIND_*/ROLE_*), :73-87 (LatticeInfo),
:90-179 (NodeSet).  Every API here accepts any object with the NodeSet attributes, so a
`hybridnodes.nodegen.NodeSet` built by the reference drops in unchanged.  The node
generators (regular fill, advancing front, hybrid_discretize) run on the
device: `generate.py`.  Seeded Appendix-B generators for the benchmark configs live in
`nodesets.py`.
"""

from __future__ import annotations

import csv
import ctypes as C
from dataclasses import dataclass

import numpy as np

KIND_REGULAR, KIND_SCATTERED, KIND_BOUNDARY = 0, 1, 2
ROLE_INTERIOR, ROLE_DIRICHLET, ROLE_NEUMANN = 0, 1, 2

_KIND_NAMES = {KIND_REGULAR: "regular", KIND_SCATTERED: "scattered", KIND_BOUNDARY: "boundary"}
_ROLE_NAMES = {ROLE_INTERIOR: "interior", ROLE_DIRICHLET: "dirichlet", ROLE_NEUMANN: "neumann"}

LATTICE_NONE = np.iinfo(np.int64).min


@dataclass
class LatticeInfo:
    """Regular-lattice index map (reference nodegen.py:73-87): grid[key] = node id or -1."""

    origin: np.ndarray
    step: np.ndarray
    cells: tuple
    grid: np.ndarray = None

    def __post_init__(self):
        if self.grid is None:
            self.grid = np.full(tuple(c + 1 for c in self.cells), -1, dtype=np.int64)

    def occupied(self, keys: np.ndarray) -> np.ndarray:
        keys = np.atleast_2d(keys)
        return self.grid[tuple(keys[:, a] for a in range(keys.shape[1]))]


class NodeSet:
    """Array-of-fields node container (reference nodegen.py:90-179)."""

    LATTICE_NONE = LATTICE_NONE

    def __init__(self, positions, spacing, kind, role, bc_value, normals, origin=None,
                 lattice: LatticeInfo | None = None, lattice_idx: np.ndarray | None = None):
        self.positions = np.asarray(positions, dtype=float)
        self.spacing = np.asarray(spacing, dtype=float)
        self.kind = np.asarray(kind, dtype=np.int8)
        self.role = np.asarray(role, dtype=np.int8)
        self.bc_value = np.asarray(bc_value, dtype=float)
        self.normals = np.asarray(normals, dtype=float)
        self.origin = list(origin) if origin is not None else [""] * len(self.positions)
        self.lattice = lattice
        self.lattice_idx = lattice_idx
        n = len(self.positions)
        if not (len(self.spacing) == len(self.kind) == len(self.role) == n):
            raise ValueError("field lengths disagree")
        if np.any(self.spacing <= 0):
            raise ValueError("node spacing must be positive")

    def __len__(self) -> int:
        return len(self.positions)

    @property
    def dim(self) -> int:
        return self.positions.shape[1]

    @property
    def counts(self) -> tuple[int, int, int]:
        return (int(np.sum(self.kind == KIND_REGULAR)), int(np.sum(self.kind == KIND_SCATTERED)),
                int(np.sum(self.kind == KIND_BOUNDARY)))

    @property
    def interior_mask(self) -> np.ndarray:
        return self.kind != KIND_BOUNDARY

    @property
    def boundary_mask(self) -> np.ndarray:
        return self.kind == KIND_BOUNDARY

    def to_csv(self, path) -> None:
        axes = "xyz"[: self.dim]
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(list(axes) + ["h", "kind", "role", "bc_value"] + [f"n{a}" for a in axes])
            for i in range(len(self)):
                w.writerow([repr(float(v)) for v in self.positions[i]]
                           + [repr(float(self.spacing[i])), _KIND_NAMES[int(self.kind[i])],
                              _ROLE_NAMES[int(self.role[i])], repr(float(self.bc_value[i]))]
                           + [repr(float(v)) for v in self.normals[i]])

    @staticmethod
    def from_csv(path) -> "NodeSet":
        kinds = {v: k for k, v in _KIND_NAMES.items()}
        roles = {v: k for k, v in _ROLE_NAMES.items()}
        with open(path, newline="") as f:
            rows = list(csv.reader(f))
        header, rows = rows[0], rows[1:]
        d = sum(1 for c in header if c in ("x", "y", "z"))
        num = np.array([[float(r[a]) for a in range(d + 1)] for r in rows])
        return NodeSet(num[:, :d], num[:, d], [kinds[r[d + 1]] for r in rows], [roles[r[d + 2]] for r in rows],
                       [float(r[d + 3]) for r in rows], [[float(r[d + 4 + a]) for a in range(d)] for r in rows])

    # ---- compact array form (fixtures, process boundaries) ----
    def to_arrays(self) -> dict:
        out = dict(positions=self.positions, spacing=self.spacing, kind=self.kind, role=self.role,
                   bc_value=self.bc_value, normals=self.normals,
                   origin=np.array(self.origin, dtype="U16"))
        if self.lattice is not None and self.lattice_idx is not None:
            out.update(lattice_origin=np.asarray(self.lattice.origin, float),
                       lattice_step=np.asarray(self.lattice.step, float),
                       lattice_cells=np.asarray(self.lattice.cells, np.int64),
                       lattice_grid=self.lattice.grid, lattice_idx=self.lattice_idx)
        return out

    @staticmethod
    def from_arrays(a) -> "NodeSet":
        lattice = lattice_idx = None
        if "lattice_grid" in a:
            lattice = LatticeInfo(np.asarray(a["lattice_origin"]), np.asarray(a["lattice_step"]),
                                  tuple(int(c) for c in a["lattice_cells"]), np.asarray(a["lattice_grid"]))
            lattice_idx = np.asarray(a["lattice_idx"])
        return NodeSet(a["positions"], a["spacing"], a["kind"], a["role"], a["bc_value"], a["normals"],
                       [str(s) for s in a["origin"]], lattice, lattice_idx)

    # ---- reference NodeSet helpers (nodegen.py:135-148) ----
    def node(self, i: int) -> "Node":
        normal = self.normals[i] if self.kind[i] == KIND_BOUNDARY else None
        return Node(self.positions[i], float(self.spacing[i]), int(self.kind[i]), int(self.role[i]),
                    float(self.bc_value[i]), normal)

    def min_distance_violations(self) -> int:
        """Pairs closer than 0.5*min(h_i, h_j) - 1e-12, counted on the device (hn_close_pairs)."""
        from . import _lib
        if len(self) < 2:
            return 0
        pos = np.ascontiguousarray(self.positions)
        lo, hi = pos.min(axis=0), pos.max(axis=0)
        dp, dh = _lib.to_device_many([pos, np.ascontiguousarray(self.spacing)])
        out = C.c_int64(0)
        _lib.call("hn_close_pairs", self.dim, _lib.ptr(dp), _lib.ptr(dh), len(self), _lib.host_dbls(lo),
                  _lib.host_dbls(hi), 0.5 * float(np.max(self.spacing)) * (1 + 1e-9), C.byref(out),
                  _lib.stream_handle())
        return int(out.value)


@dataclass(frozen=True)
class Node:
    """Single-node view into a NodeSet (reference nodegen.py:63-70)."""

    position: np.ndarray
    h: float
    kind: int
    role: int
    bc_value: float
    normal: np.ndarray | None
