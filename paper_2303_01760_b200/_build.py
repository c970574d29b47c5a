"""Build libhn.so (all CUDA kernels + the C ABI) in-tree for sm_100a.

Plain nvcc, one object per .cu file, linked into paper_2303_01760_b200/libhn.so so the
built library travels with the repo snapshot to the GPU box.  Objects are rebuilt when
their source or any header is newer.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG.parent / "build" / "hn"
LIB = PKG / "libhn.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "--expt-relaxed-constexpr", "-I", str(CSRC), "-I", str(INCLUDE)]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def build(verbose: bool = False, ptxas_info: bool = False, force: bool = False, trace: bool = False) -> Path:
    """trace=True: a dev build (libhn_trace.so, -DHN_TRACE) with the trisolve task timeline
    hook hn_debug_sptrsv_trace (tools/trace_sptrsv.py); the product library never has it."""
    build_dir = BUILD.parent / "hn_trace" if trace else BUILD
    lib_path = PKG / "libhn_trace.so" if trace else LIB
    build_dir.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    newest_header = max((h.stat().st_mtime for h in headers), default=0.0)
    objs = []
    nvcc = _nvcc()
    procs = []
    for src in sources():
        obj = build_dir / (src.stem + ".o")
        objs.append(obj)
        stale = force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, newest_header)
        if not stale:
            continue
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *(["-DHN_TRACE"] if trace else []), "-c", str(src), "-o", str(obj)]
        if ptxas_info:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose or ptxas_info:
            sys.stdout.write(out)
        if p.returncode != 0:
            failed.append(src.name)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    lib_stale = force or not lib_path.exists() or any(o.stat().st_mtime > lib_path.stat().st_mtime for o in objs)
    if lib_stale:
        cmd = [nvcc, *ARCH, "-shared", "-o", str(lib_path), *map(str, objs), "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return lib_path


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, ptxas_info="--ptxas" in sys.argv, force="-f" in sys.argv,
                trace="--trace" in sys.argv))
