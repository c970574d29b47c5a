"""PCIe copy bandwidth probe: pinned H2D / D2H of the config-1 table sizes (dev tool)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_01760_b200 import _lib as L  # noqa: E402


def main():
    t = L.torch()
    for mb in (4.9, 39.2, 200.0):
        n = int(mb * 1e6 / 8)
        d = t.empty(n, dtype=t.float64, device="cuda")
        h = t.empty(n, dtype=t.float64, pin_memory=True)
        for direction in ("d2h", "h2d"):
            for _ in range(3):
                (h.copy_(d, non_blocking=True) if direction == "d2h" else d.copy_(h, non_blocking=True))
            t.cuda.synchronize()
            ts = []
            for _ in range(10):
                t0 = time.perf_counter()
                (h.copy_(d, non_blocking=True) if direction == "d2h" else d.copy_(h, non_blocking=True))
                t.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            ts.sort()
            print(f"{direction} {mb:6.1f} MB: {ts[len(ts) // 2] * 1e3:.3f} ms = {mb / 1e3 / ts[len(ts) // 2]:.1f} GB/s",
                  flush=True)


if __name__ == "__main__":
    main()
