"""Timeline of one public-API compute_weights call on config 1: host spans vs device
kernels/copies (torch.profiler), to see where the e2e milliseconds go (dev tool)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, nodesets  # noqa: E402
from paper_2303_01760_b200.nodegen import NodeSet  # noqa: E402


def call(ns, ops):
    fresh = NodeSet(ns.positions, ns.spacing, ns.kind, ns.role, ns.bc_value, ns.normals, ns.origin, ns.lattice,
                    ns.lattice_idx)
    table = hn.compute_weights(fresh, ops)
    return table.indices, table.weights, table.method


def main():
    t = L.torch()
    from torch.profiler import profile, ProfilerActivity
    ns = nodesets.jittered_box(315, seed=1)
    ops = [hn.Laplacian(), hn.Partial(0), hn.Partial(1)]
    for _ in range(5):
        call(ns, ops)
    t.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        call(ns, ops)
    print(f"e2e call {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms", flush=True)
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            call(ns, ops)
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    tot = {}
    for e in ev:
        tot[e.name] = tot.get(e.name, 0.0) + e.device_time / 3
    print("device time per call (us):")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
        print(f"  {v:9.1f}  {k[:100]}")
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=30))
    prof.export_chrome_trace("gpurun_out/e2e_trace.json")


if __name__ == "__main__":
    main()
