"""Row-sharded explicit step over several GPUs.

The reference loop body (solver.py:439-452) is single-process; this is its one-process-per-GPU
form.  Nodes are cut into spatial slabs (`partition_nodes`); a rank keeps its owned rows first
and then the halo nodes its stencils reach, so the step kernels of csrc/step.cu run unchanged
on the rank's local numbering.  Per step:

    K7 momentum (owned rows)            -> halo exchange of v*          (d planes)
    K8 divergence / right-hand side     -> all-gather of the owned rows (N fp64 in total)
    K9 pressure: replicated (the reference's sparse direct LU does not shard: replicas only)
    K10 correction + temperature        -> halo exchange of (v, T)      (d + 1 planes)
    K11 temperature boundary conditions -> halo exchange of T           (1 plane)

Every exchange is pack (hn_halo_gather) -> NCCL send/recv on the same stream -> unpack
(hn_halo_scatter); nothing synchronises with the host.  Rows are computed by the same kernels
in the same per-row order as on one GPU, and the replicated pressure solve sees the same
right-hand side on every rank, so the sharded fields are bitwise equal to DeviceStepper's.

`HaloPlan`, `partition_nodes` and `build_halo_plan` are pure host logic (numpy) and are tested
with world_size-2 gloo processes on CPU; `ShardedStepper` needs a GPU per rank.  `LocalTransport`
runs R virtual ranks in ONE process in lockstep (each phase for every rank, then the copies
between their buffers): it is how the single-GPU test checks the sharded step against
DeviceStepper without ranks that wait on one another."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .errors import PoissonConvergenceError, SolverDivergenceError
from .operators import FieldState

INT32_MAX = np.iinfo(np.int32).max


# ============================================================ host logic (no GPU)
def partition_nodes(positions: np.ndarray, world: int, axis: int | None = None) -> np.ndarray:
    """Owner rank per node: equal-count slabs along `axis` (default: the longest extent), ties
    by node id.  Slabs keep the halo a thin strip, as §8(e)'s 'node range (spatially sorted)'."""
    pos = np.asarray(positions, dtype=float)
    n = len(pos)
    if world < 1:
        raise ValueError("world must be >= 1")
    if axis is None:
        axis = int(np.argmax(pos.max(axis=0) - pos.min(axis=0))) if n else 0
    order = np.argsort(pos[:, axis], kind="stable")
    owner = np.empty(n, dtype=np.int32)
    cuts = (np.arange(world + 1, dtype=np.int64) * n) // world
    for r in range(world):
        owner[order[cuts[r]: cuts[r + 1]]] = r
    return owner


@dataclass
class HaloPlan:
    """One rank's local numbering and exchange lists.

    Local ids: [0, n_own) = own_glob (ascending node id), then the halo grouped by owner rank
    (ascending), ascending node id inside a group -- the order the owner packs them in."""
    rank: int
    world: int
    n_global: int
    own_glob: np.ndarray           # (n_own,) int64
    halo_glob: np.ndarray          # (n_halo,) int64
    recv_counts: np.ndarray        # (world,) halo nodes owned by each peer
    send_counts: np.ndarray        # (world,) owned nodes each peer needs
    send_loc: np.ndarray           # (sum send_counts,) local ids, grouped by peer
    own_counts: np.ndarray         # (world,) owned rows of every rank
    gather_pos: np.ndarray         # (n_global,) position of node g in the padded all-gather buffer
    glob2loc: np.ndarray = field(repr=False, default=None)  # (n_global,) int32, -1 = not local

    @property
    def n_own(self) -> int:
        return len(self.own_glob)

    @property
    def n_halo(self) -> int:
        return len(self.halo_glob)

    @property
    def n_loc(self) -> int:
        return self.n_own + self.n_halo

    @property
    def max_own(self) -> int:
        return int(self.own_counts.max()) if len(self.own_counts) else 0

    @property
    def loc2glob(self) -> np.ndarray:
        return np.concatenate([self.own_glob, self.halo_glob])

    def pack_map(self, ncomp: int, stride: int) -> np.ndarray:
        """Source offsets of the send buffer [peer][component][node] in an SoA block whose
        planes are `stride` apart."""
        out, o = np.empty(len(self.send_loc) * ncomp, dtype=np.int64), 0
        s = 0
        for p in range(self.world):
            c = int(self.send_counts[p])
            seg = self.send_loc[s: s + c]
            for k in range(ncomp):
                out[o: o + c] = k * stride + seg
                o += c
            s += c
        return out

    def unpack_map(self, ncomp: int, stride: int) -> np.ndarray:
        """Destination offsets of the receive buffer [peer][component][node] (the halo tail)."""
        out, o = np.empty(self.n_halo * ncomp, dtype=np.int64), 0
        h = self.n_own
        for p in range(self.world):
            c = int(self.recv_counts[p])
            for k in range(ncomp):
                out[o: o + c] = k * stride + h + np.arange(c, dtype=np.int64)
                o += c
            h += c
        return out


def halo_requests(owner: np.ndarray, ref_rows: np.ndarray, ref_cols: np.ndarray) -> list:
    """For every rank q: the nodes its owned rows read but do not own, ordered by (owner, id)."""
    owner = np.asarray(owner)
    n = len(owner)
    world = int(owner.max()) + 1 if n else 1
    ro, co = owner[ref_rows].astype(np.int64), owner[ref_cols]
    cross = ro != co
    key = np.unique(ro[cross] * n + np.asarray(ref_cols, dtype=np.int64)[cross])
    req, node = key // n, key % n
    out = []
    for q in range(world):
        mine = node[req == q]
        out.append(mine[np.lexsort((mine, owner[mine]))])
    return out


def build_halo_plan(owner: np.ndarray, ref_rows: np.ndarray, ref_cols: np.ndarray, rank: int,
                    world: int | None = None) -> HaloPlan:
    """The plan of `rank`, derived from the replicated stencil references: every rank computes
    the same request lists, so send and receive lists agree without a handshake."""
    owner = np.asarray(owner, dtype=np.int32)
    n = len(owner)
    world = int(world if world is not None else owner.max() + 1)
    requests = halo_requests(owner, ref_rows, ref_cols)
    requests += [np.empty(0, dtype=np.int64)] * (world - len(requests))
    own = np.nonzero(owner == rank)[0].astype(np.int64)
    halo = requests[rank].astype(np.int64)
    g2l = np.full(n, -1, dtype=np.int32)
    g2l[own] = np.arange(len(own), dtype=np.int32)
    g2l[halo] = len(own) + np.arange(len(halo), dtype=np.int32)
    recv_counts = np.bincount(owner[halo], minlength=world).astype(np.int64)
    send, send_counts = [], np.zeros(world, dtype=np.int64)
    for p in range(world):
        if p == rank:
            continue
        need = requests[p]
        need = need[owner[need] == rank]  # ascending id: the order p lays its halo group out in
        send.append(g2l[need].astype(np.int64))
        send_counts[p] = len(need)
    own_counts = np.bincount(owner, minlength=world).astype(np.int64)
    max_own = int(own_counts.max()) if n else 0
    gather_pos = np.empty(n, dtype=np.int64)
    for q in range(world):
        ids = np.nonzero(owner == q)[0]
        gather_pos[ids] = q * max_own + np.arange(len(ids), dtype=np.int64)
    return HaloPlan(rank, world, n, own, halo, recv_counts, send_counts,
                    np.concatenate(send) if send else np.empty(0, dtype=np.int64), own_counts, gather_pos, g2l)


# ============================================================ transports
class TorchDistTransport:
    """torch.distributed (NCCL on GPUs, gloo in the CPU tests): grouped send/recv for the halo,
    all_gather_into_tensor for the owned rows.  Works on whatever device the buffers live on."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def halo(self, parts):
        (plan, send, recv, ncomp), = parts
        dist, ops = self.dist, []
        so = ro = 0
        for p in range(self.world):
            ns, nr = int(plan.send_counts[p]) * ncomp, int(plan.recv_counts[p]) * ncomp
            peer = dist.get_global_rank(self.group, p) if self.group is not None else p
            if ns:
                ops.append(dist.P2POp(dist.isend, send[so: so + ns], peer, self.group))
            if nr:
                ops.append(dist.P2POp(dist.irecv, recv[ro: ro + nr], peer, self.group))
            so, ro = so + ns, ro + nr
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def gather(self, parts):
        (mine, out), = parts
        self.dist.all_gather_into_tensor(out, mine, group=self.group)


class LocalTransport:
    """R virtual ranks stepped in lockstep inside one process: the exchange is plain copies
    between their buffers (test and single-GPU verification; no rank waits on another)."""

    def __init__(self, world: int):
        self.world = world

    def halo(self, parts):
        assert len(parts) == self.world
        send_off = [np.concatenate([[0], np.cumsum(pl.send_counts * nc)]) for pl, _, _, nc in parts]
        for p, (plan, _, recv, nc) in enumerate(parts):
            ro = 0
            for q in range(self.world):
                nr = int(plan.recv_counts[q]) * nc
                if nr:
                    a = int(send_off[q][p])
                    recv[ro: ro + nr].copy_(parts[q][1][a: a + nr])
                ro += nr

    def gather(self, parts):
        assert len(parts) == self.world
        m = parts[0][0].numel()
        for _, out in parts:
            for q, (mine, _) in enumerate(parts):
                out[q * m: (q + 1) * m].copy_(mine)


# ============================================================ the rank's slice of the operators
def stencil_references(ops) -> tuple[np.ndarray, np.ndarray]:
    """(row, column) node ids of everything a step reads across rows: the interior operator
    table and the Neumann reconstruction rows (K11)."""
    rows, cols = [], []
    for b in ops._table.bins:
        if b.K == 0 or b.width == 0:
            continue
        idx = b.d_idx[:, : b.K].cpu().numpy().astype(np.int64)
        rows.append(np.broadcast_to(b.rows_host[None, :], idx.shape).ravel())
        cols.append(idx.ravel())
    if ops._w_neumann is not None:
        m = ops._w_neumann.tocoo()
        rows.append(np.asarray(ops.neumann_idx, dtype=np.int64)[m.row])
        cols.append(m.col.astype(np.int64))
    if not rows:
        return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64)
    return np.concatenate(rows), np.concatenate(cols)


class _LocalBin:
    def __init__(self, K, width, d_rows, d_idx, d_w):
        self.K, self.width, self.d_rows, self.d_idx, self.d_w = int(K), int(width), d_rows, d_idx, d_w


class _LocalCSR:
    def __init__(self, rowptr, cols, vals, shape):
        self.rowptr, self.cols, self.vals, self.shape = rowptr, cols, vals, shape


class LocalOperators:
    """What the step kernels need from an OperatorSet, cut to one rank's owned rows and
    renumbered to its local ids (duck-types solver.OperatorSet for the _*_dev helpers)."""

    def __init__(self, ops, plan: HaloPlan):
        from ._device import bins_args
        t = L.torch()
        self._bins_args = bins_args
        self.plan, self.dim, self.n = plan, ops.dim, plan.n_loc
        self.nodeset = None
        self._lap_plane, self._d_planes = ops._lap_plane, list(ops._d_planes)
        g2l = L.to_device(plan.glob2loc.astype(np.int32))
        owner_mask = np.zeros(plan.n_global, dtype=bool)
        owner_mask[plan.own_glob] = True
        bad = L.zeros(1, t.int32)
        self.bins = []
        for b in ops._table.bins:
            if b.K == 0:
                continue
            sel_h = np.nonzero(owner_mask[b.rows_host])[0]
            if len(sel_h) == 0:
                continue
            sel = L.to_device(sel_h.astype(np.int64))
            rows = L.to_device(plan.glob2loc[b.rows_host[sel_h]].astype(np.int32))
            if b.width == 0:
                self.bins.append(_LocalBin(len(sel_h), 0, rows, L.empty((0, len(sel_h)), t.int32),
                                           L.empty((len(ops._table.ops), 0, len(sel_h)), t.float64)))
                continue
            idx_g = b.d_idx[:, : b.K].index_select(1, sel).contiguous()
            idx = t.empty_like(idx_g)
            L.call("hn_remap_indices", L.ptr(idx_g), L.ptr(g2l), idx_g.numel(), L.ptr(idx), L.ptr(bad),
                   L.stream_handle())
            w = b.d_w[:, :, : b.K].index_select(2, sel).contiguous()
            self.bins.append(_LocalBin(len(sel_h), b.width, rows, idx, w))
        # K11: owned Dirichlet nodes, owned Neumann rows (columns renumbered)
        own_dir = owner_mask[ops.dirichlet_idx]
        self.dirichlet_idx = plan.glob2loc[ops.dirichlet_idx[own_dir]]
        self._d_dir_idx = L.to_device(self.dirichlet_idx.astype(np.int32))
        self._d_dir_val = L.to_device(np.asarray(ops.dirichlet_values, dtype=np.float64)[own_dir])
        self._d_neu = None
        self.neumann_idx = np.empty(0, dtype=np.int64)
        if ops._w_neumann is not None:
            own_neu = np.nonzero(owner_mask[ops.neumann_idx])[0]
            m = ops._w_neumann.tocsr()[own_neu]
            cols = plan.glob2loc[m.indices]
            if len(cols) and cols.min() < 0:
                raise RuntimeError("halo plan misses a Neumann-row column")
            self.neumann_idx = plan.glob2loc[ops.neumann_idx[own_neu]].astype(np.int64)
            self._d_neu = _LocalCSR(L.to_device(m.indptr.astype(np.int64)), L.to_device(cols.astype(np.int32)),
                                    L.to_device(m.data.astype(np.float64)), (len(own_neu), plan.n_loc))
            self._d_neu_idx = L.to_device(self.neumann_idx.astype(np.int32))
            self._d_neu_diag = L.to_device(ops._d_neu_diag.cpu().numpy()[own_neu])
            mask = np.zeros(plan.n_loc, dtype=np.uint8)  # halo Neumann nodes too: t0 zeroes them as columns
            is_neu_glob = np.zeros(plan.n_global, dtype=bool)
            is_neu_glob[ops.neumann_idx] = True
            mask[is_neu_glob[plan.loc2glob]] = 1
            self._d_is_neu = L.to_device(mask)
        if int(bad.item()):
            raise RuntimeError("halo plan misses a stencil column")

    def _bins(self):
        return self._bins_args(self.bins)


# ============================================================ the stepper
class ShardedStepper:
    """One rank of the row-sharded step.  `ops` is the replicated OperatorSet (every rank builds
    or loads the same one: the pressure factor is replicated anyway); `state` the global initial
    FieldState.  step() enqueues the whole step on the current stream."""

    def __init__(self, ops, params, settings, dt: float, state: FieldState, rank: int, world: int,
                 transport=None, owner: np.ndarray | None = None):
        t = L.torch()
        if getattr(params, "dissipation", 0.0):
            raise NotImplementedError("hyper-dissipation reads lap(lap(f)): a 2-hop halo, not built")
        if ops._d_press is None:
            raise RuntimeError("operators were built with factorize=False: no pressure solve available")
        self.ops, self.params, self.settings, self.dt = ops, params, settings, float(dt)
        self.rank, self.world = int(rank), int(world)
        self.transport = transport
        owner = partition_nodes(ops.nodeset.positions, world) if owner is None else np.asarray(owner, np.int32)
        self.owner = owner
        rr, cc = stencil_references(ops)
        self.plan = plan = build_halo_plan(owner, rr, cc, rank, world)
        self.local = LocalOperators(ops, plan)
        n, d, nl = ops.n, ops.dim, plan.n_loc
        self.n_global, self.dim = n, d
        l2g = plan.loc2glob
        # (v | T) share one SoA block per buffer so the post-K10 exchange is one message
        self._blk = [L.empty((d + 1, nl), t.float64), L.empty((d + 1, nl), t.float64)]
        self._blk[0][:d].copy_(L.to_device(np.ascontiguousarray(np.asarray(state.velocity, float)[l2g].T)))
        self._blk[0][d].copy_(L.to_device(np.asarray(state.temperature, float)[l2g]))
        self._blk[1].zero_()
        self.cur = 0
        self.vstar = L.zeros((d, nl), t.float64)
        self.rhs_loc = L.zeros(nl + 1, t.float64)
        self.p_loc = L.zeros(nl, t.float64)
        self.x = L.to_device(np.concatenate([np.asarray(state.pressure, float),
                                             [getattr(ops, "_poisson_lambda", 0.0)]]))
        self.rhs = L.zeros(n + 1, t.float64)
        self.status = L.zeros(2, t.int32)
        self.flags = L.to_device(np.array([0, INT32_MAX, 0], dtype=np.int32))
        self.latch = L.to_device(np.array([0, 0, INT32_MAX, 0, 0], dtype=np.int32))
        self.have_p = False
        self.steps = 0
        self._d_loc2glob = L.to_device(l2g.astype(np.int64))
        self._d_gather_pos = L.to_device(plan.gather_pos)
        self._own_pad = L.zeros(max(plan.max_own, 1), t.float64)
        self._gathered = L.zeros(max(plan.max_own, 1) * world, t.float64)
        self._maps = {}
        self._send = L.empty(max(len(plan.send_loc), 1) * (d + 1), t.float64)
        self._recv = L.empty(max(plan.n_halo, 1) * (d + 1), t.float64)

    # ---- views of the current / next buffers ----
    @property
    def v(self):
        return self._blk[self.cur][: self.dim]

    @property
    def T(self):
        return self._blk[self.cur][self.dim]

    @property
    def _next(self):
        return self._blk[1 - self.cur]

    # ---- exchange pieces (pack / transfer / unpack are separate so virtual ranks can run in lockstep) ----
    def _map(self, ncomp):
        m = self._maps.get(ncomp)
        if m is None:
            nl = self.plan.n_loc
            m = (L.to_device(self.plan.pack_map(ncomp, nl)), L.to_device(self.plan.unpack_map(ncomp, nl)))
            self._maps[ncomp] = m
        return m

    def _pack(self, block, ncomp):
        """block: contiguous (>= ncomp, n_loc) view whose first ncomp planes are exchanged."""
        pm, _ = self._map(ncomp)
        n = pm.numel()
        L.call("hn_halo_gather", L.ptr(block), L.ptr(pm), n, L.ptr(self._send), L.stream_handle())
        return (self.plan, self._send[:n], self._recv[: self.plan.n_halo * ncomp], ncomp)

    def _unpack(self, block, ncomp):
        _, um = self._map(ncomp)
        L.call("hn_halo_scatter", L.ptr(self._recv), L.ptr(um), um.numel(), L.ptr(block), L.stream_handle())

    # ---- phases ----
    def _phase_momentum(self):
        from .solver import _momentum_dev
        _momentum_dev(self.local, self.params, self.dt, self.v, self.T, self.vstar, zero_boundary=True)
        return self._pack(self.vstar, self.dim)

    def _phase_rhs(self):
        from .solver import _div_rhs_dev
        self._unpack(self.vstar, self.dim)
        _div_rhs_dev(self.local, self.vstar, self.dt, self.rhs_loc)
        self._own_pad[: self.plan.n_own].copy_(self.rhs_loc[: self.plan.n_own])
        return (self._own_pad, self._gathered)

    def _phase_pressure_correct(self):
        from .solver import _correct_temp_dev
        n = self.n_global
        L.call("hn_halo_gather", L.ptr(self._gathered), L.ptr(self._d_gather_pos), n, L.ptr(self.rhs),
               L.stream_handle())
        self.ops._d_press.solve(self.rhs, self.x if self.have_p else None, self.x, self.settings.tol,
                                self.settings.maxiter, self.status)
        L.call("hn_halo_gather", L.ptr(self.x), L.ptr(self._d_loc2glob), self.plan.n_loc, L.ptr(self.p_loc),
               L.stream_handle())
        nxt = self._next
        _correct_temp_dev(self.local, self.vstar, self.p_loc, self.T, self.dt, nxt[: self.dim], nxt[self.dim],
                          self.flags, 0.0)
        return self._pack(nxt, self.dim + 1)

    def _phase_bc(self):
        from .solver import _temperature_bc_dev
        nxt = self._next
        self._unpack(nxt, self.dim + 1)
        _temperature_bc_dev(self.local, nxt[self.dim], self.flags, self.latch, self.status)
        return self._pack(nxt[self.dim:], 1)

    def _phase_finish(self):
        self._unpack(self._next[self.dim:], 1)
        self.cur = 1 - self.cur
        self.have_p = True
        self.steps += 1

    def step(self):
        step_lockstep([self], self.transport)

    # ---- results ----
    def state(self) -> FieldState:
        """The global fields on the host (owned rows of every rank all-gathered; the pressure is
        replicated).  Collective: every rank calls it."""
        return gather_states([self], self.transport)[0]

    def latch_host(self) -> np.ndarray:
        """[steps, first non-finite step, its lowest non-finite T node (GLOBAL id), first failed
        pressure step, its info] of this rank's rows."""
        f = self.latch.cpu().numpy().astype(np.int64)
        if f[2] != INT32_MAX:
            f[2] = int(self.plan.loc2glob[f[2]])
        return f

    def check_finite(self, peers_latches=None):
        """Raise as DeviceStepper.check_finite does, over all ranks' latches (pass the list of
        every rank's latch_host(); one rank alone checks its own rows)."""
        rows = np.asarray(peers_latches if peers_latches is not None else [self.latch_host()])
        pfail = rows[:, 3][rows[:, 3] > 0]
        bad = rows[:, 1][rows[:, 1] > 0]
        first_bad = int(bad.min()) if len(bad) else 0
        if len(pfail) and (first_bad == 0 or int(pfail.min()) <= first_bad):
            raise PoissonConvergenceError(f"pressure Poisson solve did not converge at step {int(pfail.min())}",
                                          residual=float("nan"))
        if first_bad:
            nodes = rows[rows[:, 1] == first_bad, 2]
            nodes = nodes[nodes != INT32_MAX]
            raise SolverDivergenceError(f"non-finite field at step {first_bad}", step=first_bad,
                                        node=int(nodes.min()) if len(nodes) else -1)


def step_lockstep(steppers, transport):
    """One step of every stepper in the list: one rank with its TorchDistTransport, or all R
    virtual ranks of a LocalTransport."""
    transport.halo([s._phase_momentum() for s in steppers])
    transport.gather([s._phase_rhs() for s in steppers])
    transport.halo([s._phase_pressure_correct() for s in steppers])
    transport.halo([s._phase_bc() for s in steppers])
    for s in steppers:
        s._phase_finish()


def gather_states(steppers, transport):
    """Global FieldState per stepper (all-gather of the owned rows, plane by plane)."""
    t = L.torch()
    d, n = steppers[0].dim, steppers[0].n_global
    outs = [L.empty((d + 1, n), t.float64) for _ in steppers]
    for k in range(d + 1):
        parts = []
        for s in steppers:
            s._own_pad[: s.plan.n_own].copy_(s._blk[s.cur][k, : s.plan.n_own])
            parts.append((s._own_pad, s._gathered))
        transport.gather(parts)
        for s, o in zip(steppers, outs):
            L.call("hn_halo_gather", L.ptr(s._gathered), L.ptr(s._d_gather_pos), n, L.ptr(o[k]), L.stream_handle())
    res = []
    for s, o in zip(steppers, outs):
        h = o.cpu().numpy()
        x = s.x.cpu().numpy()
        res.append(FieldState(np.ascontiguousarray(h[:d].T), x[:n].copy(), h[d].copy()))
    return res


# ============================================================ row-sharded weight computation
def row_cuts(k: int, world: int) -> np.ndarray:
    """Equal-count cuts of a class's node-ordered row list ('shard interior rows
    by node range ... concatenate outputs')."""
    return (np.arange(world + 1, dtype=np.int64) * int(k)) // world


class WeightShard:
    """One rank's slice of the interior weight table: the MON and RBF-FD rows it computed
    (ELL slabs over its node range) plus the replicated classification."""

    def __init__(self, nodeset, ops, rank: int, world: int, rbf_n: int | None = None):
        from . import approx as A
        from ._device import device_nodes
        t = L.torch()
        dim, n = nodeset.dim, len(nodeset)
        self.ops, self.dim, self.n, self.rank, self.world = list(ops), dim, n, rank, world
        for op in self.ops:
            A._op_code(op, dim)
        self.n_rbf = A.RBF_SIZE[dim] if rbf_n is None else int(rbf_n)
        dn = device_nodes(nodeset)
        has_lattice = getattr(nodeset, "lattice", None) is not None and getattr(nodeset, "lattice_idx", None) is not None
        if not (has_lattice or not np.any(np.asarray(nodeset.kind) == A.KIND_REGULAR)):
            raise NotImplementedError("sharded weights need the lattice map (or no regular node)")
        self.method_d = dn.classify()
        rows_d = L.empty(max(n, 1), t.int32)
        counts_d = L.empty(3, t.int32)
        scratch = L.empty(3 * (n // 256 + 1) + 1, t.int32)
        L.call("hn_partition_methods", L.ptr(self.method_d), n, L.ptr(rows_d), L.ptr(counts_d), L.ptr(scratch),
               L.stream_handle())
        self.k_mon, self.k_rbf, self.k_none = (int(v) for v in counts_d.cpu().numpy())
        self.rows_d = rows_d
        self.local, self.pending = {}, []
        for name, k, off, mon in (("mon", self.k_mon, 0, True), ("rbf", self.k_rbf, self.k_mon, False)):
            if k == 0:
                continue
            cuts = row_cuts(k, world)
            mine = rows_d[off + int(cuts[rank]): off + int(cuts[rank + 1])]
            if mon:
                st = dn.mon_stencils(mine) if has_lattice else dn.knn(A.MON_SIZE[dim], rows=mine)
            else:
                if self.n_rbf > n:
                    raise ValueError(f"stencil size {self.n_rbf} exceeds node count {n}")
                st = dn.knn(self.n_rbf, rows=mine, fine=True)
            b, info = A._solve_bin(dn, st, mine, self.ops, mon)
            self.local[name] = b
            self.pending.append((b, info))

    def check(self):
        from . import approx as A
        A._check_info(self.pending)


def _gather_cols(per_rank, counts, transport):
    """per_rank[i]: (R_, K_q) tensor of virtual rank i (one entry for a real rank); returns the
    (R_, sum K) concatenation along the last axis in rank order, one per entry."""
    t = L.torch()
    kmax, world = int(max(counts)), len(counts)
    rows = per_rank[0].shape[0]
    parts = []
    for x in per_rank:
        mine = t.zeros((rows, kmax), dtype=x.dtype, device=x.device)
        mine[:, : x.shape[1]].copy_(x)
        parts.append((mine.reshape(-1), t.empty(world * rows * kmax, dtype=x.dtype, device=x.device)))
    transport.gather(parts)
    return [t.cat([out.view(world, rows, kmax)[q, :, : int(counts[q])] for q in range(world)], dim=1).contiguous()
            for _, out in parts]


def merge_weight_shards(shards, transport):
    """All-gather the shards' slabs into the full interior table on every rank (bitwise the
    single-GPU table: each stencil's arithmetic does not depend on its batch).  `shards`: the one
    WeightShard of this rank (TorchDistTransport) or every virtual rank's (LocalTransport)."""
    from ._device import Bin, DeviceTable
    from .approx import WeightTable
    t = L.torch()
    s0 = shards[0]
    world, nops = s0.world, len(s0.ops)
    tables = [[] for _ in shards]
    for name, k, off in (("mon", s0.k_mon, 0), ("rbf", s0.k_rbf, s0.k_mon)):
        if k == 0:
            continue
        counts = np.diff(row_cuts(k, world))
        width = s0.local[name].width
        idx = _gather_cols([s.local[name].d_idx[:, : s.local[name].K] for s in shards], counts, transport)
        wts = _gather_cols([s.local[name].d_w[:, :, : s.local[name].K].reshape(nops * width, -1) for s in shards],
                           counts, transport)
        for i, s in enumerate(shards):
            b = Bin(None, width, idx[i], wts[i].view(nops, width, k), d_rows=s.rows_d[off: off + k], K=k)
            b.mon = name == "mon"
            tables[i].append(b)
    out = []
    for i, s in enumerate(shards):
        if s.k_none:
            tables[i].append(Bin(None, 0, L.empty((0, s.k_none), t.int32), L.empty((nops, 0, s.k_none), t.float64),
                                 d_rows=s.rows_d[s.k_mon + s.k_rbf: s.n], K=s.k_none))
        s.check()
        out.append(WeightTable(_device=DeviceTable(s.n, s.dim, s.ops, tables[i], s.n_rbf, s.method_d[: s.n])))
    return out


def compute_weights_sharded(nodeset, ops, rank: int, world: int, transport, rbf_n: int | None = None):
    """compute_weights (approx.py:379-413) with the interior rows sharded over `world` ranks:
    positions replicated, each rank solves its node range, one all-gather per slab."""
    return merge_weight_shards([WeightShard(nodeset, ops, rank, world, rbf_n)], transport)[0]


__all__ = ["HaloPlan", "partition_nodes", "halo_requests", "build_halo_plan", "stencil_references",
           "TorchDistTransport", "LocalTransport", "LocalOperators", "ShardedStepper", "step_lockstep",
           "gather_states", "row_cuts", "WeightShard", "merge_weight_shards", "compute_weights_sharded"]
