"""Host-side profile of one config-1 weights step (dev tool)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2303_01760_b200 as hn  # noqa: E402
from paper_2303_01760_b200 import _lib as L, approx, nodesets  # noqa: E402
from paper_2303_01760_b200 import _device  # noqa: E402


def main():
    t = L.torch()
    ns = nodesets.jittered_box(315, seed=1)
    ops = [hn.Laplacian(), hn.Partial(0), hn.Partial(1)]
    _device.device_nodes(ns)
    for _ in range(5):
        approx._interior_device_table(ns, ops)
    t.cuda.synchronize()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        approx._interior_device_table(ns, ops)
    t.cuda.synchronize()
    print(f"steady step (no cell list rebuild): {(time.perf_counter() - t0) / n * 1e3:.3f} ms", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(n):
        approx._interior_device_table(ns, ops)
    t.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
