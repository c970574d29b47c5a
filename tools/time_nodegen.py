"""Time the device hybrid_discretize on reference cases (dev tool)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2303_01760_b200 as hn

cases = [dict(case="dvd", h_r=0.01), dict(case="spheres3d", h_r=0.05), dict(case="obstacles2d", h_r=0.02),
         dict(case="spheres3d", h_r=0.02), dict(case="spheres3d", h_r=0.01), dict(case="dvd", h_r=0.002)]
for kw in cases[: int(sys.argv[1]) if len(sys.argv) > 1 else None]:
    cfg = hn.CaseConfig(**kw)
    spec = hn.build_domain(cfg)
    hn.hybrid_discretize(cfg, spec) if kw["h_r"] >= 0.02 else None
    t = time.perf_counter()
    ns = hn.hybrid_discretize(cfg, spec)
    dt = time.perf_counter() - t
    print(kw, "N", len(ns), "counts", ns.counts, f"{dt * 1e3:.1f} ms", f"{len(ns) / dt:.3e} nodes/s", flush=True)
