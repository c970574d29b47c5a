"""Benchmark for the hybrid RBF-FD hot path on B200 (contract: see DESIGN.md §6).

Default workload: config 4, the largest single-GPU configuration of BASELINE.json (3D
hybrid sphere set, N = 1,054,026, 22 % scattered) -- one step = cell list + classify + MON
7-point stencils and solves + kNN n = 20 + RBF-FD PHS r^3 + degree-2 30x30 fp64 solves
(Laplacian, d/dx, d/dy, d/dz) for every interior row, written into HBM ELL slabs.  `value`
= stencil weights/s over the whole job; `e2e` = the same through the public API
compute_weights() with host NodeSet in and host WeightTable out; `roofline` = the dominant
kernel (the RBF-FD solve) vs the live DFMA peak; `cpu_baseline` = the reference's algorithm
(oracle port, 1 thread, the reference's protocol) on the same host.  The metric's second
half rides on the same line as `time_steps`: config 3 (the 2D hybrid set at full N = 243,955,
explicit Boussinesq steps with the reference's LU-preconditioned BiCGStab pressure) in
node-updates/s, its full-step and explicit-part HBM fractions, e2e with host fields in and
out every step, and the oracle step on the same host (1 thread).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 0|1|2|3|4]
                  [--no-steps] [--no-cpu-baseline]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FLOPS_PER_STENCIL = {("rbf", 2, 12): 5613, ("rbf", 3, 20): 24625, ("rbf", 3, 30): 54500, ("mon", 2, 5): 205,
                     ("mon", 3, 7): 567}
L2_FLUSH_BYTES = 256 << 20


class L2Flush:
    """Flush L2 between timed launches: write a 256 MiB buffer (> the 126 MB L2), then read a
    second one, so the next launch starts with L2 full of *clean* lines -- a write-only flush
    leaves ~100 MB of dirty lines whose write-back would land inside the timed kernel."""

    def __init__(self, L):
        t = L.torch()
        self.a = L.empty(L2_FLUSH_BYTES // 8, t.float64)
        self.b = L.zeros(L2_FLUSH_BYTES // 8, t.float64)
        self.s = L.empty((), t.float64)
        self.t = t

    def __call__(self, v=1.0):
        self.a.fill_(v)
        self.t.sum(self.b, dim=0, out=self.s)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 200 for weight configs, 50 for config 3)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-steps", action="store_true", help="weights line without the config-3 steps object")
    ap.add_argument("--sharded", action="store_true",
                    help="--phase steps with --gpus N > 1: ONE node set row-sharded over the ranks (halo "
                         "exchange per gather pass, replicated pressure; strong scaling) instead of replicas")
    ap.add_argument("--phase", default=None, choices=["weights", "steps"],
                    help="config 4 has both: weight computation (default) or the Boussinesq steps")
    return ap.parse_args()


# ----------------------------------------------------------------------------- distributed plumbing
def dist_init(n):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend)
    return rank, world


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_seed(base: int, rank: int) -> int:
    """Weak scaling: every rank owns an independent node set of the config's size."""
    return base + 1000 * rank


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def _lines(self):
        self.file.flush()
        return len([ln for ln in Path(self.file.name).read_text().splitlines() if ln[:1].isdigit()])

    def _wait_for(self, count, timeout):
        t0 = time.perf_counter()
        while self._lines() < count and time.perf_counter() - t0 < timeout:
            time.sleep(0.002)

    def __enter__(self):
        try:
            idx = os.environ.get("LOCAL_RANK", "0")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", idx, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "10"],
                                         stdout=self.file, stderr=subprocess.DEVNULL)
            # nvidia-smi needs ~0.1-0.5 s before its first sample: wait for it, so even a short
            # timed region is bracketed by samples
            self._wait_for(1, 5.0)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self._wait_for(self._lines() + 1, 0.5)  # one sample at/after the end of the region
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.file.flush()
        rows = []
        for line in Path(self.file.name).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6 and parts[0].isdigit():
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [int(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------- workloads
def build_nodeset(cfg: int, seed_off: int = 0):
    from paper_2303_01760_b200 import nodesets
    if cfg == 0:
        return nodesets.regular_box(199)
    if cfg == 1:
        return nodesets.jittered_box(315, seed=1 + seed_off)
    if cfg in (2, 3):
        return nodesets.hybrid_hole_2d(500, seed=2 + seed_off)
    return nodesets.hybrid_sphere_3d(94, seed=4 + seed_off, refine=2.8)


def measure_dfma_peak(L):
    t = L.torch()
    out = L.zeros(1, t.float64)
    blocks, iters = 148 * 8, 8192
    for _ in range(2):
        L.call("hn_bench_dfma", L.ptr(out), blocks, iters, L.stream_handle())
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(3):
        e0.record()
        L.call("hn_bench_dfma", L.ptr(out), blocks, iters, L.stream_handle())
        e1.record()
        t.cuda.synchronize()
        best = max(best, blocks * 256 * iters * 16 * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


class LaunchCounter:
    """Kernels each libhn entry point launches (fixed per call; see csrc/*.cu)."""
    # hn_pressure_solve: 6 set-up kernels + one WHILE-body pass + 1 finish kernel.  The
    # complete-LU preconditioner converges at its first half-step check, so a pass is its
    # first half (7 Krylov kernels + 1 preconditioner application), the IF-condition kernel and
    # the end-of-pass kernel; the second half sits in an IF node that is not entered.  One
    # application = 2 permutes + per factor (reset + task kernel + 2 kernels per dense-group
    # phase); steps_measure sets the entry from the factors' phase counts.
    KERNELS = {"hn_celllist_build": 5, "hn_partition_methods": 6, "hn_sptrsv_super": 2,
               "hn_knn": 1, "hn_knn_spacing": 1, "hn_classify": 1, "hn_mon_stencils": 1, "hn_weights_mon": 2,
               "hn_weights_rbf": 1, "hn_apply_ell": 1, "hn_momentum": 1, "hn_div_rhs": 1,
               "hn_correct_temperature": 1, "hn_temperature_bc": 1, "hn_csr_matvec": 1, "hn_csr_residual": 1,
               "hn_pressure_solve": 22, "hn_permute": 1, "hn_reduce": 2, "hn_bicg_update": 1, "hn_bench_dfma": 1}

    def __init__(self, L):
        self.L = L
        self.count = 0
        self.enabled = False
        self._orig = L.call

        def counted(name, *args):
            if self.enabled:
                self.count += self.KERNELS.get(name, 1)
            return self._orig(name, *args)

        L.call = counted


def run_weights_bench(args, rank, world):
    import paper_2303_01760_b200 as hn
    from paper_2303_01760_b200 import _device, _lib as L, approx
    t = L.torch()
    counter = LaunchCounter(L)
    cfg = args.config
    ns = build_nodeset(cfg, shard_seed(0, rank) if world > 1 else 0)
    dim = ns.dim
    ops = [hn.Laplacian()] + [hn.Partial(a) for a in range(dim)]
    rbf_n = 20 if dim == 3 else None
    n_int = int(ns.interior_mask.sum())
    flush = L2Flush(L)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)

    # ---- device-resident step: positions in HBM; the whole pipeline (cell list ->
    # classify -> partition -> stencils -> solves) replayed as one CUDA graph ----
    pipe = approx.WeightsPipeline(ns, ops, rbf_n)
    # hn_weights_pipeline's kernels (no table, no summary): classify 1, partition 6, MON
    # stencils 1 + solve 2, kNN (3D: warp kernel + box fallback), RBF-FD (3D: null-space +
    # searching fallback; 2D: one launch, in-kernel fallback)
    counter.KERNELS["hn_weights_pipeline"] = 14 if dim == 3 else 12
    counter.enabled = True
    pipe.run()
    launches = counter.count  # kernels per step (counted from one eager pass)
    counter.enabled = False
    pipe.capture()
    for _ in range(args.warmup):
        pipe.replay()
    t.cuda.synchronize()
    pipe.check()
    barrier(world)
    times = []
    with ClockSampler() as clocks:
        for _ in range(args.steps):
            flush(1.0)
            e0.record()
            pipe.replay()
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    t.cuda.synchronize()
    pipe.check()
    barrier(world)
    ms = max_over_ranks(float(np.mean(times)), world)
    value = world * n_int / (ms * 1e-3)

    # ---- dominant kernel: the RBF (or MON for config 0) weight solve, timed alone ----
    dev = approx._interior_device_table(ns, ops, rbf_n)
    method = dev.method
    big = "rbf" if (method == 1).sum() >= (method == 0).sum() * (0.05 if dim == 2 else 0.2) or cfg == 1 else "mon"
    rows = np.nonzero(method == (1 if big == "rbf" else 0))[0]
    dn = _device.device_nodes(ns)
    if big == "rbf":
        st = dn.knn(rbf_n or 12, rows=L.to_device(rows.astype(np.int32)))
        nst = rbf_n or 12
    else:
        st = dn.mon_stencils(L.to_device(rows.astype(np.int32)))
        nst = 2 * dim + 1
    K = len(rows)
    kinds, axes, normals = approx._op_args(ops, dim)
    oi = L.empty((nst, K), t.int32)
    ow = L.empty((len(ops), nst, K), t.float64)
    info = L.zeros(K, t.int32)

    def solve():
        if big == "rbf":
            counter._orig("hn_weights_rbf", L.ptr(dn.pos), dim, L.ptr(st), K, nst, len(ops), kinds, axes, normals,
                          None, None, L.ptr(oi), L.ptr(ow), L.ptr(info), L.stream_handle())
        else:
            counter._orig("hn_weights_mon", L.ptr(dn.pos), dim, L.ptr(st), K, len(ops), kinds, axes, normals,
                          L.ptr(oi), L.ptr(ow), L.ptr(info), L.stream_handle())

    for _ in range(3):
        solve()
    kt = []
    for _ in range(min(max(5, args.steps), 30)):
        flush(2.0)
        e0.record()
        solve()
        e1.record()
        e1.synchronize()
        kt.append(e0.elapsed_time(e1))
    k_ms = float(np.median(kt))
    fps = FLOPS_PER_STENCIL[(big, dim, nst)]
    mon_bytes = nst * 4 + 8 * dim + nst * 4 + len(ops) * nst * 8  # ids in, own position, idx + weights out
    achieved = K * fps / (k_ms * 1e-3) / 1e12
    peak = measure_dfma_peak(L)
    traffic = None
    tj = ROOT / "profiles" / "traffic.json"
    if tj.exists():
        traffic = json.loads(tj.read_text()).get(f"weights_config{cfg}")

    # ---- secondary: fused 3/4-op apply over the same table (HBM roofline) ----
    f = L.to_device(build_field(ns))
    out = L.empty((len(ops), len(ns)), t.float64)
    nb, bK, bW, bR, bI, bWt, live = _device.bins_args(dev.bins)
    op_sel = L.host_ints(list(range(len(ops))))

    def app():
        counter._orig("hn_apply_ell", nb, bK, bW, bR, bI, bWt, len(ops), op_sel, L.ptr(f), L.ptr(out), len(ns),
                      L.stream_handle())

    for _ in range(3):
        app()
    at = []
    for _ in range(min(max(10, args.steps), 30)):
        flush(3.0)
        e0.record()
        app()
        e1.record()
        e1.synchronize()
        at.append(e0.elapsed_time(e1))
    a_ms = float(np.median(at))
    wt = []  # warm: 20 launches back to back, table and field L2-resident (labelled as such)
    for _ in range(5):
        e0.record()
        for _ in range(20):
            app()
        e1.record()
        e1.synchronize()
        wt.append(e0.elapsed_time(e1) / 20)
    a_warm_ms = float(np.median(wt))
    S = int(sum(b.K * b.width for b in live))
    a_bytes = (4 + 8 * len(ops)) * S + 8 * len(ns) + 8 * len(ops) * len(ns) + 4 * len(ns)
    peaks = load_peaks()

    # ---- end to end through the public API: host NodeSet in, host WeightTable out ----
    from paper_2303_01760_b200.nodegen import NodeSet
    e2e_t = []
    h2d = d2h = 0
    e2e_steps = min(args.steps, 10)
    e2e_warm = max(args.warmup, 5)  # untimed: allocator pools and pinned pages reach steady state
    for k in range(e2e_warm + e2e_steps):
        fresh = NodeSet(ns.positions, ns.spacing, ns.kind, ns.role, ns.bc_value, ns.normals, ns.origin, ns.lattice,
                        ns.lattice_idx)
        flush(4.0)
        t.cuda.synchronize()
        b0 = dict(L.TRAFFIC)
        t0 = time.perf_counter()
        table = hn.compute_weights(fresh, ops, rbf_n=rbf_n) if rbf_n else hn.compute_weights(fresh, ops)
        idx = table.indices
        w = table.weights
        t.cuda.synchronize()
        if k >= e2e_warm:
            e2e_t.append(time.perf_counter() - t0)
        # bytes the call moved (package counters: every H2D upload and the result D2H)
        h2d, d2h = L.TRAFFIC["h2d"] - b0["h2d"], L.TRAFFIC["d2h"] - b0["d2h"]
        del table, idx, w  # the caller is done with this table: its pinned pages go back to the cache
    e2e_s = max_over_ranks(float(np.mean(e2e_t)), world)

    line = {
        "metric": "stencil weights/sec", "value": value, "unit": "stencils/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded node sets, SURVEY Appendix B)",
        "config": weights_config(cfg, ns, world, pipe.k_mon, pipe.k_rbf, len(ops)),
        "e2e": {"value": world * n_int / e2e_s, "unit": "stencils/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "api": "paper_2303_01760_b200.compute_weights(NodeSet, ops)",
                "samples_ms": [round(1e3 * x, 3) for x in e2e_t]},
        "roofline": ({"bound": "fp64", "kernel": (f"rbf_ns_kernel<{dim},{nst}>" if dim == 3 else f"rbf_static_kernel<{dim},{nst}>"), "achieved": achieved,
                      "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                      "algorithmic": f"{fps} flop/stencil (LAPACK getrf+getrs count, SURVEY §8(d)) x {K} stencils",
                      "kernel_ms": k_ms,
                      "peak_source": "live DFMA probe (hn_bench_dfma); MEASURED_PEAKS.json has no fp64 entry"}
                     if big == "rbf" else
                     # the MON solve is ~205 flop per 176 B: bound by memory, not the FP64 pipe
                     {"bound": "hbm", "kernel": f"mon_weights_kernel<{dim}>",
                      "achieved": K * mon_bytes / (k_ms * 1e-3) / 1e9, "peak": load_peaks().get("hbm_gbs", 6526.8),
                      "unit": "GB/s", "frac": K * mon_bytes / (k_ms * 1e-3) / 1e9 / load_peaks().get("hbm_gbs", 6526.8),
                      "traffic": traffic,
                      "algorithmic": f"{mon_bytes} B/stencil (stencil ids in, own position, idx + weights out) x {K}",
                      "kernel_ms": k_ms, "fp64_tflops": achieved, "fp64_frac": achieved / peak,
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy test)"}),
        "apply": {"metric": "fused multi-op application", "kernel": "apply_ell_kernel", "ms": a_ms,
                  "bytes": a_bytes, "achieved_gbs": a_bytes / (a_ms * 1e-3) / 1e9, "peak_gbs": peaks.get("hbm_gbs"),
                  "frac": a_bytes / (a_ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6526.8),
                  "frac_of_8tbs_nominal": a_bytes / (a_ms * 1e-3) / 8e12,
                  "warm_l2_ms": a_warm_ms, "warm_l2_gbs": a_bytes / (a_warm_ms * 1e-3) / 1e9,
                  "node_updates_per_s": len(ns) / (a_ms * 1e-3),
                  "bytes_formula": "(4 + 8*ops)*S + 8N (field) + 8*ops*N (out) + 4N (row ids)"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_weights(ns, ops, rbf_n)
    return line


def build_field(ns):
    from paper_2303_01760_b200 import nodesets
    return nodesets.sinusoid_field(ns.positions)


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def config_name(cfg, ns):
    c = ns.counts
    return {0: f"config0: 2D regular 200x200, N={len(ns)}, MON 5-point, Lap/dx/dy weights",
            1: f"config1: 2D scattered jittered M=315, N={len(ns)}, kNN n=12 + RBF-FD 18x18, Lap/dx/dy weights",
            2: f"config2: 2D hybrid hole M=500, N={len(ns)} ({c[1] / len(ns):.1%} scattered), kNN + MON/RBF weights",
            3: f"config3: config-2 set, explicit Boussinesq steps Ra=1e6 Pr=0.71 with reference pressure",
            4: f"config4: 3D hybrid sphere, N={len(ns)} ({c[1] / len(ns):.1%} scattered), MON 7 + RBF-FD n=20 (30x30)",
            }[cfg]


def stencil_mix(dev):
    return {f"w{b.width}": int(b.K) for b in dev.bins if b.width}


def weights_config(cfg, ns, world, k_mon, k_rbf, ops):
    """The `config` object of a weights line -- identical for both arms (same_config)."""
    dim = ns.dim
    mix = {}
    if k_mon:
        mix[f"w{2 * dim + 1}"] = int(k_mon)
    if k_rbf:
        mix[f"w{20 if dim == 3 else 12}"] = int(k_rbf)
    return {"workload": config_name(cfg, ns), "N": len(ns), "interior_rows": int(k_mon + k_rbf), "stencils": mix,
            "ops": int(ops), "l2": "flushed between steps (256 MiB write + 256 MiB read: L2 left clean)",
            "parallelism": f"weak x{world} (independent node set per rank)"}


def cpu_baseline_weights(ns, ops, rbf_n):
    """The reference algorithm (oracle port: cKDTree + LAPACK dgesv, 1 thread) on the same
    host, bounded sample = the whole config once or more (about 3-15 s)."""
    from oracle import hn_oracle as O
    from threadpoolctl import threadpool_limits
    keys = [O.op_tuple(o) for o in ops]
    n_int = int(ns.interior_mask.sum())
    reps, t_total = 0, 0.0
    # one BLAS thread for the oracle only (the reference's protocol); a process-wide
    # OMP_NUM_THREADS=1 would also serialise torch's host copies on the GPU arm's e2e path
    with threadpool_limits(1):
        while t_total < 3.0 and reps < 5:
            t0 = time.perf_counter()
            O.compute_weights(ns, keys, rbf_n=rbf_n)
            t_total += time.perf_counter() - t0
            reps += 1
    return {"value": reps * n_int / t_total, "unit": "stencils/s", "cores": 1, "kind": "port",
            "sample": f"oracle compute_weights on the full workload x{reps} ({t_total:.1f} s), "
                      f"OPENBLAS_NUM_THREADS=1 (reference protocol, cli.py:7-10)",
            "host_cpu": cpu_model()}


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- config 3: time steps
def _stepper(hn, ns, factorize, Ra, seed=3, rbf_n=None):
    dim = ns.dim
    settings = hn.PoissonSolveSettings()
    if rbf_n is None:
        rbf_n = 20 if dim == 3 else None
    ops = hn.build_operators(ns, {"wall:x-"}, settings, interior_rbf_n=rbf_n, factorize=factorize)
    dt = hn.TimeControls.from_spacing(float(np.min(ns.spacing)), 1.0, Ra=Ra).dt
    T0 = (ns.positions[:, 0] - 0.5) + 1e-3 * np.random.default_rng(seed).normal(size=len(ns))
    st = hn.FieldState(np.zeros((len(ns), dim)), np.zeros(len(ns)), T0)
    hn.apply_temperature_bc(st.temperature, ops)
    return hn.DeviceStepper(ops, hn.PhysicsParams(Ra, 0.71), settings, dt, st), ops, dt


def _explicit_roofline(L, stepper, ns, steps, flush):
    """The HBM-bound explicit part (K7 + K8 + K10 + K11) timed alone, L2 flushed per step."""
    t = L.torch()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    for _ in range(3):
        stepper.explicit_step()
    ts = []
    for _ in range(max(10, min(steps, 50))):
        flush(5.0)
        e0.record()
        stepper.explicit_step()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    d, n = ns.dim, len(ns)
    S = int(sum(b.K * b.width for b in stepper.ops._table.bins))
    nbytes = S * (28 + 24 * d) + 40 * n * (d + 1)
    peak = load_peaks().get("hbm_gbs", 6526.8)
    return {"kernels": "momentum_kernel + div_rhs_kernel + correct_temp_kernel + temperature BC", "ms": ms,
            "node_updates_per_s": n / (ms * 1e-3), "bytes": nbytes,
            "bytes_formula": "S(28+24d) + 40N(d+1) (SURVEY §8(d))", "achieved_gbs": nbytes / (ms * 1e-3) / 1e9,
            "peak_gbs": peak, "frac": nbytes / (ms * 1e-3) / 1e9 / peak,
            "frac_of_8tbs_nominal": nbytes / (ms * 1e-3) / 8e12}


def pressure_bytes(ops) -> int:
    """Algorithmic HBM bytes of one warm pressure solve (one BiCGStab half-step, SURVEY §8(a)
    A17): 2 A-matvecs (12 B/nnz + int64 row pointer + x gather/y write), one preconditioner
    application (L and U: 12 B per sparse entry the task kernels and the dense groups' coupling read,
    8 B per entry of the groups' inverse triangles, the U diagonal, the two permutations in and out) and the
    BiCGStab vector algebra (~12 vector passes of 8 B/element)."""
    n1 = ops.n + 1
    a_nnz = int(ops._d_poisson.nnz)
    lu = ops._d_lu
    return 2 * (12 * a_nnz + 24 * n1) + int(lu.solve_bytes) + 4 * 12 * n1 + 12 * 8 * n1


def steps_measure(args, rank, world, cfg=3, flush=None, with_cpu=True):
    """Config 3 (2D, full N, reference pressure treatment) -> node-updates/s of full steps.
    Config 4 (3D): full steps (with the reference's SuperLU pressure) at a reduced-N twin of
    the same generator -- SuperLU at N = 1e6 is infeasible -- plus the explicit
    part at the full N = 1.05e6."""
    import paper_2303_01760_b200 as hn
    from paper_2303_01760_b200 import _lib as L, nodesets
    t = L.torch()
    counter = LaunchCounter(L)
    flush = flush or L2Flush(L)
    off = shard_seed(0, rank) if world > 1 else 0
    if cfg == 3:
        ns, Ra = build_nodeset(3, off), 1e6
    else:
        ns, Ra = nodesets.hybrid_sphere_3d(24, seed=4 + off, refine=2.8), 1e5
    # 3D full steps: interior n = 30 (the reference's RBF_SIZE[3]).  With BASELINE's n = 20 the
    # explicit scheme is unstable on this set -- |v| grows x1.2 per step and the run blows up
    # at step 42, in the CPU oracle of the reference algorithm exactly as on the GPU
    # (DESIGN.md §5); the explicit part at the full N below keeps n = 20.
    t_setup = time.perf_counter()
    stepper, ops, dt = _stepper(hn, ns, True, Ra, rbf_n=30 if cfg == 4 else None)
    t_setup = time.perf_counter() - t_setup
    lu_dev = ops._d_lu
    counter.KERNELS = dict(counter.KERNELS, hn_pressure_solve=16 + (6 + 2 * (lu_dev.sL.n_phases + lu_dev.sU.n_phases)),
                           hn_sptrsv_plan=2 + 2 * max(lu_dev.sL.n_phases, lu_dev.sU.n_phases))
    steps = args.steps_steps
    # a step is one CUDA-graph replay (no libhn call from the host), so the kernels of a step
    # are counted where they are enqueued: the warm-up steps (eager first step, then the
    # capture of the two ping-pong graphs) each enqueue exactly one step's kernels
    counter.enabled = True
    for _ in range(args.warmup):
        stepper.step()
    counter.enabled = False
    launches_per_step = counter.count // max(1, args.warmup)
    t.cuda.synchronize()
    barrier(world)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    with ClockSampler() as clocks:
        e0.record(stepper.stream)
        for _ in range(steps):
            stepper.step()
        e1.record(stepper.stream)
        t.cuda.synchronize()
    stepper.check_finite()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, world)
    explicit = _explicit_roofline(L, stepper, ns, steps, flush)
    d, n = ns.dim, len(ns)
    peak = load_peaks().get("hbm_gbs", 6526.8)
    pb = pressure_bytes(ops)
    full_bytes = explicit["bytes"] + pb

    # ---- e2e: host fields in (pinned staging), one step, host fields out, every step ----
    from paper_2303_01760_b200.operators import FieldState
    host = stepper.state()
    e2e_t = []
    b0 = dict(L.TRAFFIC)
    for k in range(3 + min(steps, 10)):
        t.cuda.synchronize()
        t0 = time.perf_counter()
        stepper.load_state(host)
        stepper.step()
        host = stepper.state()
        if k >= 3:
            e2e_t.append(time.perf_counter() - t0)
    stepper.check_finite()
    e2e_ms = max_over_ranks(1e3 * float(np.mean(e2e_t)), world)
    h2d = (L.TRAFFIC["h2d"] - b0["h2d"]) // (3 + min(steps, 10))
    d2h = (d + 2) * 8 * n
    out = {"metric": "node-updates/sec per step", "value": world * n / (ms * 1e-3), "unit": "node-updates/s",
           "ms_per_step": ms, "steps": steps, "warmup": args.warmup,
           "config": {"workload": config_name(cfg, ns), "N": n, "dt": dt, "Ra": Ra,
                      "pressure": "LU-preconditioned BiCGStab (SuperLU factors in HBM, supernodal sync-free "
                                  "trisolves), device-driven (graph WHILE node), one graph replay per step",
                      "setup_s": round(t_setup, 2),
                      "l2": "not flushed between full steps (each step moves > 1 GB); explicit part: flushed"},
           "hbm_full_step": {"bytes": full_bytes, "explicit_bytes": explicit["bytes"], "pressure_bytes": pb,
                             "bytes_formula": "explicit S(28+24d)+40N(d+1) + pressure (bench.pressure_bytes)",
                             "achieved_gbs": full_bytes / (ms * 1e-3) / 1e9, "peak_gbs": peak,
                             "frac": full_bytes / (ms * 1e-3) / 1e9 / peak},
           "explicit": explicit,
           "e2e": {"value": world * n / (e2e_ms * 1e-3), "unit": "node-updates/s", "ms_per_step": e2e_ms,
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                   "api": "DeviceStepper.load_state(host FieldState) + step() + state() -> host, every step"},
           "gpu_launches": launches_per_step, "clocks": clocks.summary()}
    if cfg == 4:
        out["config"]["workload"] = out["config"]["workload"].replace("n=20 (30x30)", "n=30 (40x40)")
        big = build_nodeset(4, off)
        st_big, _, _ = _stepper(hn, big, False, Ra)
        out["explicit_full_N"] = dict(_explicit_roofline(L, st_big, big, steps, flush), N=len(big))
        out["config"]["note"] = ("full steps at a reduced-N twin (hybrid_sphere_3d(24)) with interior n=30 "
                                 "(n=20 diverges at step 42 in the reference algorithm too); the explicit part "
                                 "at the full N=%d with n=20" % len(big))
    if with_cpu and rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_steps(ns, Ra, rbf_n=30 if cfg == 4 else None)
    return out


def cpu_baseline_steps(ns, Ra, rbf_n=None, budget_s=8.0):
    """The reference's run-loop body (oracle port of solver.py:439-452: scipy csr_matvec +
    bicgstab with the SuperLU preconditioner) on the same host, 1 thread; build_operators
    (splu) is setup, reported separately.  Bounded sample: as many steps as fit in ~8 s."""
    from oracle import hn_oracle as O
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        t0 = time.perf_counter()
        o = O.build_operators(ns, {"wall:x-"}, rbf_n=rbf_n)
        setup = time.perf_counter() - t0
        dt = O.dt_rule(float(np.min(ns.spacing)), Ra)
        T = O.temperature_bc(o, (ns.positions[:, 0] - 0.5) + 1e-3 * np.random.default_rng(3).normal(size=len(ns)))
        state, p = (np.zeros((len(ns), ns.dim)), T), None
        state, p = O.step(o, state, Ra, 0.71, 0.0, dt, p_prev=p)  # cold first step: not timed
        k, t_steps = 0, 0.0
        while t_steps < budget_s and k < 200:
            t0 = time.perf_counter()
            state, p = O.step(o, state, Ra, 0.71, 0.0, dt, p_prev=p)
            t_steps += time.perf_counter() - t0
            k += 1
    return {"value": len(ns) * k / t_steps, "unit": "node-updates/s", "cores": 1, "kind": "port",
            "ms_per_step": 1e3 * t_steps / k,
            "sample": f"oracle run-loop body x{k} warm steps ({t_steps:.1f} s) on the same node set, after "
                      f"build_operators (setup {setup:.1f} s, not timed), OPENBLAS_NUM_THREADS=1 (cli.py:7-10)",
            "setup_s": round(setup, 2), "host_cpu": cpu_model()}


def sharded_steps_measure(args, rank, world, cfg=3):
    """Strong scaling of the config-3 step: one node set, rows sharded over the ranks
    (paper_2303_01760_b200.sharded: halo exchange of v*, (v, T) and T per step over NCCL, the
    right-hand side all-gathered, the pressure solve replicated).  Time = max over ranks."""
    import paper_2303_01760_b200 as hn
    from paper_2303_01760_b200 import _lib as L, nodesets, sharded as S
    t = L.torch()
    if cfg == 3:
        ns, Ra, rbf_n = build_nodeset(3, 0), 1e6, None
    else:
        ns, Ra, rbf_n = nodesets.hybrid_sphere_3d(24, seed=4, refine=2.8), 1e5, 30
    single, ops, dt = _stepper(hn, ns, True, Ra, rbf_n=rbf_n)
    st0 = single.state()
    tr = S.TorchDistTransport() if world > 1 else S.LocalTransport(1)
    stepper = S.ShardedStepper(ops, single.params, single.settings, dt, st0, rank, world, transport=tr)
    for _ in range(args.warmup):
        stepper.step()
    t.cuda.synchronize()
    barrier(world)
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    steps = args.steps_steps
    with ClockSampler() as clocks:
        e0.record()
        for _ in range(steps):
            stepper.step()
        e1.record()
        t.cuda.synchronize()
    stepper.check_finite()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, world)
    n, d, pl = len(ns), ns.dim, stepper.plan
    return {"metric": "node-updates/sec per step", "value": n / (ms * 1e-3), "unit": "node-updates/s",
            "ms_per_step": ms, "steps": steps, "warmup": args.warmup, "scaling": "strong",
            "config": {"workload": config_name(cfg, ns), "N": n, "dt": dt, "Ra": Ra,
                       "parallelism": f"rows sharded x{world} (slabs), replicated pressure solve",
                       "rows_this_rank": pl.n_own, "halo_this_rank": pl.n_halo,
                       "exchange_bytes_per_step": int(8 * (2 * d + 2) * (pl.n_halo + len(pl.send_loc)) + 8 * n)},
            "clocks": clocks.summary()}


def run_steps_bench(args, rank, world):
    m = (sharded_steps_measure if getattr(args, "sharded", False) else steps_measure)(args, rank, world,
                                                                                     cfg=args.config)
    line = {"metric": m["metric"], "value": m["value"], "unit": m["unit"], "n_gpus": world,
            "steps": m["steps"], "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic"}
    line.update({k: v for k, v in m.items() if k not in line and k != "metric"})
    line["scaling"] = m.get("scaling", "weak")
    return line


# ----------------------------------------------------------------------------- reference arm
_REF = {}  # workload shared with forked reference workers (copy-on-write, no pickling)


def _ref_worker_init():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)  # one BLAS thread per worker process: P processes = P cores
    except ImportError:
        pass


def _ref_chunk(job):
    """One worker's share of the reference algorithm (oracle port of approx.py:379-413):
    kNN by (fl-distance, index) through cKDTree + LAPACK dgesv per 4096-stencil batch."""
    from oracle import hn_oracle as O
    meth, lo, hi = job
    ns, ops, rbf_n, rows_by = _REF["ns"], _REF["ops"], _REF["rbf_n"], _REF["rows"]
    rows = rows_by[meth][lo:hi]
    if meth == 0:
        st = O.mon_stencils(ns, rows)
        solver = O.mon_solve
    else:
        st = O.knn_by_key(ns.positions, ns.positions[rows], rbf_n)
        solver = O.rbf_solve
    for k in range(0, len(rows), 4096):
        w = solver(ns.positions, st[k:k + 4096], ops)
        O._store(_REF["table"], rows[k:k + 4096], st[k:k + 4096], w, _REF["keys"])  # shared-memory table
    return hi - lo


def run_reference(args, rank, world):
    """The reference's CPU implementation of the path (oracle port; the Python reference
    cannot travel to the GPU box) on this host with every core: the interior rows are split
    over P forked worker processes (one BLAS thread each) and the WeightTable is assembled
    in the parent -- the per-row work is independent."""
    if world > 1 and rank != 0:
        return None
    import multiprocessing as mp
    from oracle import hn_oracle as O
    cfg = args.config
    ns = build_nodeset(cfg)
    dim = ns.dim
    keys = [("lap",)] + [("d", a) for a in range(dim)]
    ops = [O.op_tuple(k) for k in keys]
    n_int = int(ns.interior_mask.sum())
    rbf_n = 20 if dim == 3 else 12
    P = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    method = O.classify(ns)

    def shared(shape, dtype, fill):
        n = int(np.prod(shape))
        buf = mp.RawArray("b", max(1, n * np.dtype(dtype).itemsize))
        a = np.frombuffer(buf, dtype=dtype, count=n).reshape(shape)
        a[...] = fill
        return a
    # the WeightTable lives in shared memory: workers fill their rows in place (no pickling)
    table = {"indices": shared((len(ns), rbf_n), np.int64, -1), "sizes": shared((len(ns),), np.int64, 0),
             "weights": {k: shared((len(ns), rbf_n), np.float64, 0.0) for k in keys}, "method": method}
    _REF.update(ns=ns, ops=ops, keys=keys, rbf_n=rbf_n, table=table,
                rows={m: np.nonzero(method == m)[0] for m in (0, 1)})
    jobs = []
    for m in (0, 1):
        rows = _REF["rows"][m]
        per = max(1, -(-len(rows) // P))
        jobs += [(m, lo, min(lo + per, len(rows))) for lo in range(0, len(rows), per)]

    def one_step(pool):
        return sum(pool.imap_unordered(_ref_chunk, jobs))

    ctx = mp.get_context("fork")
    with ctx.Pool(P, initializer=_ref_worker_init) as pool:
        for _ in range(min(args.warmup, 1)):
            one_step(pool)
        ts = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            one_step(pool)
            ts.append(time.perf_counter() - t0)
    s = float(np.mean(ts))
    v = n_int / s
    return {"impl": "reference", "metric": "stencil weights/sec", "value": v, "unit": "stencils/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": weights_config(cfg, ns, world, int((method == 0).sum()), int((method == 1).sum()), len(keys)),
            "cpu_baseline": {"value": v, "unit": "stencils/s", "cores": P, "kind": "port",
                             "sample": f"full workload per step, {args.steps} steps: numpy/scipy oracle port of the "
                                       f"reference (cKDTree + batched LAPACK dgesv) over {P} worker processes, "
                                       "1 BLAS thread each, writing one shared-memory WeightTable",
                             "host_cpu": cpu_model()},
            "e2e": {"value": v, "unit": "stencils/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if args.steps is None:
        args.steps = 50 if args.config == 3 else (3 if args.impl == "reference" else 20)
    if args.phase is None:
        args.phase = "steps" if args.config == 3 else "weights"
    args.steps_steps = args.steps if args.phase == "steps" else 50  # steps timed for the `steps` object
    rank, world = dist_init(args.gpus)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    elif args.phase == "steps" and args.config in (3, 4):
        line = run_steps_bench(args, rank, world)
    else:
        line = run_weights_bench(args, rank, world)
        if args.config == 4 and not args.no_steps:
            # the metric's second half (node-updates/s per step, % HBM) on BASELINE config 3
            line["time_steps"] = steps_measure(args, rank, world, cfg=3)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
