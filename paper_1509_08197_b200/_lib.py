"""ctypes binding of the C ABI in include/hdp_stereo.h (libhdpstereo.so).

The product path has no CPU fallback: if the in-tree CUDA library is missing
or no CUDA device is visible, every device entry point raises.  Status codes
map one-to-one onto the reference's error classes (treestereo/errors.py).
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, DataError, InternalError

_HERE = os.path.dirname(os.path.abspath(__file__))
# HDP_LIB: load another build of the library (A/B comparisons of build variants)
LIB_PATH = os.environ.get("HDP_LIB") or os.path.join(_HERE, "libhdpstereo.so")
ABI_VERSION = 1

_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_F = C.c_float
_D = C.c_double

# name -> (restype, argtypes); mirrors include/hdp_stereo.h
SIGNATURES = {
    "hdp_abi_version": (_I, []),
    "hdp_last_error": (C.c_char_p, []),
    "hdp_launch_count": (_I64, []),
    "hdp_u8_to_f64": (_I, [_P, _P, _I64, _P]),
    "hdp_block_mean": (_I, [_P, _P, _I, _I, _I, _I, _I, _P]),
    "hdp_prepare": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "hdp_argsort_u64": (_I, [_P, _I64, _P, _P]),
    "hdp_cost_volume": (_I, [_P, _P, _I, _I, _I, _I, _P, _I, _F, _F, _F, _P, _P]),
    "hdp_grid_edges": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "hdp_grid_edge_weights64": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "hdp_median3x3": (_I, [_P, _P, _I, _I, _I, _I, _P]),
    "hdp_mst": (_I, [_I64, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "hdp_prepare_u8": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "hdp_grid_edges_u8": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P]),
    "hdp_predict_masks": (_I, [_P, _I64, _I, _D, _P, _I, _P]),
    "hdp_priors_from_counts": (_I, [_P, _P, _I, _I, _P, _P]),
    "hdp_bayes": (_I, [_P, _P, _I, _I, _I, _P, _P, _P]),
    "hdp_mst_grid": (_I, [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "hdp_prior_counts": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _D, _D, _D,
                              _P, _P, _I, _P]),
    "hdp_check_exact_division": (_I, [_I64, C.c_uint64, _P, _P]),
    "hdp_assign_rows": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P]),
    "hdp_hdpf": (_I, [_I, _I64, _I64, _P, _P, _P, _P, _P, _I, _I, _D, _P, _D, _P, _P, _P, _P, _P]),
    "hdp_segment_tree": (_I, [_I, _I, _I, _P, _P, _P, _P, _D, _P, _P, _P, _P]),
    "hdp_forest_create": (_I, [_I64, _I64, _P, _P, _P, _P, _P, _F, C.POINTER(_P), _P]),
    "hdp_forest_stats": (_I, [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64),
                              C.POINTER(_I64)]),
    "hdp_forest_export": (_I, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "hdp_forest_set_lanes": (_I, [_P, _P, _I, _P]),
    "hdp_forest_set_lanes_range": (_I, [_P, _I, _I, _P]),
    "hdp_forest_set_lanes_nodes": (_I, [_P, _P, _I, _P]),
    "hdp_forest_entries": (_I, [_P, C.POINTER(_I64), _P, _P]),
    "hdp_aggregate_wta": (_I, [_P, _P, _P, _I, _I, _I, _F, _F, _F, _P, _P, _P, _P, _P, _P]),
    "hdp_forest_pair_stats": (_I, [_P, _I, _I64, _P, _P, _P]),
    "hdp_forest_pair_stats_device": (_I, [_P, _I, _I64, _P, _P]),
    "hdp_forest_set_timing": (_I, [_P, _I]),
    "hdp_forest_stage_ms": (_I, [_P, _P, _P]),
    "hdp_forest_destroy": (None, [_P]),
    "hdp_keys_unpack": (_I, [_P, _I64, _I, _P, _P, _P]),
    "hdp_keys_pack": (_I, [_P, _P, _I64, _I, _P, _P]),
    "hdp_error_counts": (_I, [_P, _P, _P, _P, _P, _I, _I64, _P, _I, _P, _P]),
    "hdp_occlusion_from_gt": (_I, [_P, _P, _P, _P, _I, _I, _I, _P, _P]),
    "hdp_rows_first_argmin": (_I, [_P, _I64, _I, _P, _P, _P]),
    "hdp_gather_ragged": (_I, [_P, _I, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "hdp_set_early_cost": (_I, [_I]),
    "hdp_pool_reserve": (_I, [_I64, _P]),
    "hdp_dense_pipeline": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _F, _F, _F, _F, _I, _P, _P, _P, _P, _P, _P]),
}

_lib = None


def load():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"CUDA extension missing: {LIB_PATH} (build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'`); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.hdp_abi_version() != ABI_VERSION:
        raise RuntimeError("libhdpstereo.so ABI version mismatch; rebuild")
    _lib = lib
    return lib


_ERRORS = {2: ConfigError, 3: DataError, 4: InternalError, 5: InternalError}


def check(status: int) -> None:
    if status == 0:
        return
    msg = load().hdp_last_error().decode(errors="replace")
    raise _ERRORS.get(status, InternalError)(msg or f"hdp status {status}")


# diagnostics: HDP_DIAG_SLOWCALL=<ms> reports every library call whose host time exceeds it
_SLOW_MS = float(os.environ.get("HDP_DIAG_SLOWCALL", "0") or 0)


def call(name: str, *args) -> None:
    if _SLOW_MS > 0:
        import sys
        import time

        t = time.perf_counter()
        status = getattr(load(), name)(*args)
        dt = 1e3 * (time.perf_counter() - t)
        if dt > _SLOW_MS:
            print(f"[hdp slow call] {name}: {dt:.0f} ms", file=sys.stderr, flush=True)
        check(status)
        return
    check(getattr(load(), name)(*args))


def torch_mod():
    import torch

    return torch


def device():
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required (the B200 path has no CPU fallback)")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch_mod().cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
