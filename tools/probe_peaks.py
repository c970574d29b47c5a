"""Measure fp64 DFMA and DMMA (tensor) throughput on this GPU (dev tool)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01760_b200 import _lib as L  # noqa: E402


def run(name, flops_per_launch, blocks, iters):
    t = L.torch()
    out = L.zeros(1, t.float64)
    for _ in range(2):
        L.call(name, L.ptr(out), blocks, iters, L.stream_handle())
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    best = 0
    for _ in range(3):
        e0.record(); L.call(name, L.ptr(out), blocks, iters, L.stream_handle()); e1.record(); t.cuda.synchronize()
        best = max(best, flops_per_launch / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


for blocks in (148 * 4, 148 * 8):
    print(f"DFMA blocks={blocks}: {run('hn_bench_dfma', blocks * 256 * 8192 * 16 * 2, blocks, 8192):.1f} TFLOP/s")
    print(f"DMMA blocks={blocks}: {run('hn_bench_dmma', blocks * 8 * 4096 * 4 * 512, blocks, 4096):.1f} TFLOP/s")
