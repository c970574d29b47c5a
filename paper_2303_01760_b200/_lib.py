"""ctypes binding of libhn.so (include/hn.h) plus the device-memory plumbing.

torch provides device memory and the current CUDA stream only; every computation on
the hot path is a libhn.so kernel.  There is no CPU fallback: if the library or a GPU
is missing, `lib()` raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("HN_LIB_PATH", _PKG / "libhn.so"))  # env override: A/B builds (dev)

_c_int_p = C.POINTER(C.c_int)
_c_i64_p = C.POINTER(C.c_int64)
_c_dbl_p = C.POINTER(C.c_double)
_vp = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_d = C.c_double

class TriPlan(C.Structure):
    """hn_tri_plan (include/hn.h): one triangular factor's supernodal task list."""
    _fields_ = [("lower", _i), ("inv", _i), ("ntasks", _i64), ("kind", _vp), ("r0", _vp), ("w", _vp), ("rb", _vp),
                ("rc", _vp), ("off", _vp), ("rw", _vp), ("rowptr", _vp), ("cols", _vp), ("vals", _vp), ("diag", _vp),
                ("packed", _vp), ("n_phases", _i), ("phase_ptr", _i64 * 17), ("g_row", _vp), ("g_cpl_rowptr", _vp),
                ("g_cpl_cols", _vp), ("g_cpl_vals", _vp), ("g_inv_off", _vp), ("g_cnt", _vp), ("g_ystart", _vp),
                ("g_inv", _vp), ("g_y", _vp)]


# name -> (restype, argtypes); mirrors include/hn.h exactly (tests check the export list)
SIGNATURES: dict[str, tuple] = {
    "hn_version": (_i, []),
    "hn_bench_dfma": (_i, [_vp, _i, _i, _vp]),
    "hn_bench_dmma": (_i, [_vp, _i, _i, _vp]),
    "hn_node_stats": (_i, [_vp, _i64, _i, _vp, _vp, _vp, _vp, _vp]),
    "hn_celllist_build": (_i, [_vp, _i64, _i, _c_dbl_p, _d, _c_int_p, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hn_knn": (_i, [_vp, _i, _c_dbl_p, _d, _c_int_p, _vp, _vp, _vp, _vp, _vp, _i64, _i, _vp, _vp, _vp, _vp]),
    "hn_knn_spacing": (_i, [_vp, _i, _c_dbl_p, _d, _c_int_p, _vp, _vp, _vp, _vp, _vp, _i64, _i, _vp, _vp, _vp, _vp,
                            _vp]),
    "hn_weights_pipeline": (_i, [_vp, _i, _i64, _vp, _vp, _vp, _c_int_p, _c_dbl_p, _d, _c_int_p, _vp, _vp, _vp,
                                 _vp, _i, _c_int_p, _c_int_p, _c_dbl_p, _i, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64_p, _vp,
                                 _vp, _i, _c_i64_p, _vp]),
    "hn_classify": (_i, [_vp, _vp, _vp, _c_int_p, _i64, _i, _vp, _vp]),
    "hn_mon_stencils": (_i, [_vp, _i64, _vp, _vp, _vp, _c_int_p, _i, _vp, _vp]),
    "hn_weights_mon": (_i, [_vp, _i, _vp, _i64, _i, _c_int_p, _c_int_p, _c_dbl_p, _vp, _vp, _vp, _vp]),
    "hn_weights_rbf": (_i, [_vp, _i, _vp, _i64, _i, _i, _c_int_p, _c_int_p, _c_dbl_p, _vp, _vp, _vp, _vp,
                            _vp, _vp]),
    "hn_weights_rbf_is_tuned": (_i, [_i, _i, _i]),
    "hn_weights_rbf_workspace": (_i64, [_i, _i, _i, _i64]),
    "hn_weights_rbf_set_variant": (None, [_i]),
    "hn_knn_set_variant": (None, [_i]),
    "hn_apply_set_threads": (None, [_i]),
    "hn_apply_ell": (_i, [_i, _c_i64_p, _c_int_p, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), _i,
                          _c_int_p, _vp, _vp, _i64, _vp]),
    "hn_ell_to_table": (_i, [_i, _c_i64_p, _c_int_p, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), _i, _i, _i64,
                             _vp, _vp, _vp, _vp]),
    "hn_momentum": (_i, [_i, _c_i64_p, _c_int_p, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), _i, _c_int_p,
                         _i, _vp, _vp, _i64, _d, _d, _d, _c_dbl_p, _i, _vp, _vp, _vp, _vp]),
    "hn_div_rhs": (_i, [_i, _c_i64_p, _c_int_p, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), _c_int_p, _i,
                        _vp, _i64, _d, _vp, _vp]),
    "hn_correct_temperature": (_i, [_i, _c_i64_p, _c_int_p, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), _i,
                                    _c_int_p, _i, _vp, _vp, _vp, _i64, _d, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hn_temperature_bc": (_i, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "hn_csr_matvec": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "hn_csr_residual": (_i, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "hn_sptrsv_super": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i, _vp,
                             _vp, _vp, _i64, _vp, _i, _vp]),
    "hn_host_pack_panels": (_i64, [_vp, _vp, _vp, _vp, _i, _i, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hn_host_supernodes": (_i64, [_vp, _vp, _i64, _i, _i, _vp, _vp]),
    "hn_host_block_levels": (_i, [_vp, _vp, _i64, _i, _i64, _vp, _vp, _vp]),
    "hn_partition_methods": (_i, [_vp, _i64, _vp, _vp, _vp, _vp]),
    "hn_permute": (_i, [_i, _vp, _vp, _i64, _vp, _vp]),
    "hn_sptrsv_plan": (_i, [C.POINTER(TriPlan), _vp, _vp, _vp, _i64, _vp, _i, _vp]),
    "hn_halo_gather": (_i, [_vp, _vp, _i64, _vp, _vp]),
    "hn_halo_scatter": (_i, [_vp, _vp, _i64, _vp, _vp]),
    "hn_remap_indices": (_i, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "hn_condition_numbers": (_i, [_vp, _i, _i, _vp, _i64, _i64, _vp, _i64, _i, _i, _vp, _vp]),
    "hn_pressure_setup": (_i, [_i64, _vp, _vp, _vp, C.POINTER(TriPlan), C.POINTER(TriPlan), _vp, _vp, _i, _c_i64_p]),
    "hn_pressure_solve": (_i, [_i64, _vp, _vp, _vp, _d, _i, _vp, _vp]),
    "hn_pressure_free": (_i, [_i64]),
    "hn_reduce": (_i, [_i, _vp, _vp, _vp, _i64, _vp, _vp, _vp]),
    "hn_bicg_update": (_i, [_i, _vp, _vp, _vp, _d, _d, _i64, _vp]),
    "hn_geom_eval": (_i, [_vp, _vp, _i64, _i, _vp, _vp]),
    "hn_lattice_fill": (_i, [_vp, _c_i64_p, _c_dbl_p, _d, _i, _d, _vp, _vp, _c_i64_p, _vp]),
    "hn_front_candidates": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _i, _vp, _vp, _vp, _vp]),
    "hn_front_accept": (_i, [_i, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _d, _c_dbl_p, _c_dbl_p,
                             _d, _c_i64_p, _vp]),
    "hn_lattice_map": (_i, [_i, _c_i64_p, _c_dbl_p, _c_dbl_p, _d, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp]),
    "hn_close_pairs": (_i, [_i, _vp, _vp, _i64, _c_dbl_p, _c_dbl_p, _d, _c_i64_p, _vp]),
}

_LIB = None


class NativeError(RuntimeError):
    """A libhn.so call failed (CUDA error or bad argument)."""


def lib():
    """Load libhn.so once; raises if it is missing (no CPU fallback exists)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python -m paper_2303_01760_b200._build)")
        handle = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
        ab_build = "HN_LIB_PATH" in os.environ  # dev A/B against an older build: tolerate new symbols
        for name, (res, args) in SIGNATURES.items():
            if ab_build and not hasattr(handle, name):
                continue
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
        if os.environ.get("HN_RBF_VARIANT"):  # dev A/B of the weight kernels (tools/ab_rbf.py)
            handle.hn_weights_rbf_set_variant(int(os.environ["HN_RBF_VARIANT"]))
    return _LIB


def call(name: str, *args) -> int:
    rc = getattr(lib(), name)(*args)
    if rc < 0:
        raise NativeError(f"{name}: CUDA error {-rc}")
    if rc > 0:
        raise NativeError(f"{name}: invalid argument (code {rc})")
    return rc


# ---------------------------------------------------------------- torch plumbing
_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        if not t.cuda.is_available():
            raise NativeError("no CUDA device: the hybridnodes-b200 hot path runs on the GPU only")
        _torch = t
    return _torch


def device():
    return torch().device("cuda", torch().cuda.current_device())


def stream_handle():
    return _vp(torch().cuda.current_stream().cuda_stream)


def ptr(t) -> _vp:
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return _vp(0)
    return _vp(t.data_ptr())


def host_ints(vals) -> C.Array:
    arr = (C.c_int * max(1, len(vals)))(*[int(v) for v in vals])
    return arr


def host_i64(vals) -> C.Array:
    return (C.c_int64 * max(1, len(vals)))(*[int(v) for v in vals])


def host_dbls(vals) -> C.Array:
    vals = list(vals)
    return (C.c_double * max(1, len(vals)))(*[float(v) for v in vals])


def host_ptrs(tensors) -> C.Array:
    return (_vp * max(1, len(tensors)))(*[t.data_ptr() if t is not None else 0 for t in tensors])


# host<->device bytes moved by this package (bench.py reports the per-call deltas as e2e traffic)
TRAFFIC = {"h2d": 0, "d2h": 0}


def to_device(a: np.ndarray, dtype=None):
    """Copy a host array to the current device (pinned staging for large arrays)."""
    t = torch()
    arr = np.ascontiguousarray(a if dtype is None else a.astype(dtype, copy=False))
    TRAFFIC["h2d"] += arr.nbytes
    src = t.from_numpy(arr)
    if arr.nbytes < (64 << 10):
        return src.to(device(), non_blocking=False)
    # pinned staging (torch's caching host allocator keeps the block until the copy's
    # event completes), then an async DMA: no pageable bounce through the driver
    stage = t.empty(src.shape, dtype=src.dtype, pin_memory=True)
    stage.copy_(src)
    return stage.to(device(), non_blocking=True)


def to_device_many(arrays):
    """Upload several host arrays with one pinned staging buffer and one DMA; returns device
    tensors (8-byte aligned segments of one allocation)."""
    t = torch()
    arrs = [np.ascontiguousarray(a) for a in arrays]
    offs, total = [], 0
    for a in arrs:
        offs.append(total)
        total += (a.nbytes + 7) // 8 * 8
    stage = t.empty(max(total, 8), dtype=t.uint8, pin_memory=True)
    for a, o in zip(arrs, offs):  # torch's CPU copy is multi-threaded (numpy's is not)
        stage[o:o + a.nbytes].copy_(t.from_numpy(a.reshape(-1).view(np.uint8)))
    dev = stage.to(device(), non_blocking=True)
    TRAFFIC["h2d"] += total
    out = []
    for a, o in zip(arrs, offs):
        tt = _np_to_torch_dtype(a.dtype)
        seg = dev[o:o + (a.nbytes + 7) // 8 * 8].view(tt)
        out.append(seg[: a.size].view(a.shape))
    return out


def _np_to_torch_dtype(dt):
    t = torch()
    return {np.dtype(np.float64): t.float64, np.dtype(np.int64): t.int64, np.dtype(np.int32): t.int32,
            np.dtype(np.int8): t.int8, np.dtype(np.uint8): t.uint8}[np.dtype(dt)]


def empty(shape, dtype):
    return torch().empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype):
    return torch().zeros(shape, dtype=dtype, device=device())


def loaded_library_path() -> str:
    return os.fspath(LIB_PATH)
