"""ctypes binding of libgenoiht_cuda.so (include/genoiht_cuda.h).

The library is the product's only compute path.  It is built in-tree by
``__graft_entry__.build()`` (``make -C paper_1608_01398_b200/csrc``); there is
no CPU fallback: if the shared object or a CUDA device is missing, every entry
point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GI_LIB_PATH") or os.path.join(_HERE, "libgenoiht_cuda.so")

_lib = None
_lock = threading.Lock()

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_u64 = ctypes.c_uint64


class NativeError(RuntimeError):
    """A CUDA-side failure reported through gi_last_error()."""


class FitConfig(ctypes.Structure):
    """gi_fit_config (IhtConfig, iht.py:120-140)."""

    _fields_ = [("k", c_i64), ("max_iter", c_i64), ("tol", c_dbl), ("c_omega", c_dbl),
                ("max_backtracks", c_i64), ("flags", c_i64)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(c_int, c_vp, ctypes.POINTER(c_dbl), c_i64, c_int)
ALLGATHER_FN = ctypes.CFUNCTYPE(c_int, c_vp, ctypes.POINTER(c_dbl), c_i64, ctypes.POINTER(c_dbl))


class FitOut(ctypes.Structure):
    """gi_fit_result (FitResult, iht.py:172-180)."""

    _fields_ = [("support", c_vp), ("weights", c_vp), ("support_cap", c_i64), ("nnz", c_i64),
                ("covar", c_vp), ("loss_trace", c_vp), ("trace_cap", c_i64),
                ("trace_len", c_i64), ("iterations", c_i64), ("backtracks", c_i64),
                ("kernel_launches", c_i64), ("aty_ms_total", c_dbl), ("aty_launches", c_i64),
                ("reason", c_int), ("heldout_sse", c_dbl), ("heldout_n", c_i64),
                ("xtr_kernel", c_int)]


class FitJob(ctypes.Structure):
    """gi_fit_job: one fit of gi_fit_many."""

    _fields_ = [("h", c_vp), ("y", c_vp), ("C", c_vp), ("c", c_i64), ("keep", c_vp),
                ("u", c_vp), ("v", c_vp), ("cfg", ctypes.POINTER(FitConfig)),
                ("warm_idx", c_vp), ("warm_w", c_vp), ("warm_k", c_i64), ("bcov0", c_vp),
                ("res", ctypes.POINTER(FitOut)), ("warm_from", c_i64), ("status", c_int),
                ("error", ctypes.c_char * 256)]


def _declare(lib):
    P = c_vp
    sig = {
        "gi_version": ([], c_int),
        "gi_last_error": ([], ctypes.c_char_p),
        "gi_device_count": ([P], c_int),
        "gi_device_info": ([c_int, P, P, P], c_int),
        "gi_device_sync": ([c_int], c_int),
        "gi_matrix_from_bed": ([P, c_i64, c_i64, c_int, P], c_int),
        "gi_matrix_create": ([c_i64, c_i64, c_int, P], c_int),
        "gi_matrix_upload_bed": ([P, c_i64, c_i64, P], c_int),
        "gi_matrix_finalize": ([P], c_int),
        "gi_matrix_synth": ([c_u64, c_i64, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_int, P], c_int),
        "gi_matrix_with_stats": ([P, P, P, P], c_int),
        "gi_matrix_subset_rows": ([P, P, c_i64, P], c_int),
        "gi_matrix_free": ([P], c_int),
        "gi_matrix_shape": ([P, P, P, P], c_int),
        "gi_matrix_xtr_format": ([P, c_int, P], c_int),
        "gi_matrix_stats": ([P, P, P], c_int),
        "gi_matrix_read_bed": ([P, c_i64, c_i64, P], c_int),
        "gi_matrix_missing_counts": ([P, P], c_int),
        "gi_matrix_device_stats": ([P, P, P], c_int),
        "gi_matrix_masked_stats": ([P, P, P, P], c_int),
        "gi_aty": ([P, P, c_dbl, P, c_int], c_int),
        "gi_aty_batched": ([P, P, P, P, P, c_i64, P, c_int], c_int),
        "gi_ax_cols": ([P, P, P, c_i64, P], c_int),
        "gi_decompress": ([P, P, c_i64, P], c_int),
        "gi_dev_ax": ([P, P, P, P, P, c_i64, P, c_int, P], c_int),
        "gi_dev_aty_fast": ([P, P, P, P, P, P, c_dbl, P, P], c_int),
        "gi_dev_aty_exact": ([P, P, P, P, P, c_dbl, P, P], c_int),
        "gi_padded_samples": ([P], c_i64),
        "gi_dev_stats": ([P, P, P, P, P, P], c_int),
        "gi_red_partials": ([], c_i64),
        "gi_dev_residual": ([c_i64, P, P, P, c_i64, P, P, c_dbl, P, P, P, P, P], c_int),
        "gi_dev_center": ([c_i64, c_i64, P, P, P, P, P, P, P], c_int),
        "gi_dev_covgrad": ([c_i64, P, c_i64, P, P, P, P, P], c_int),
        "gi_dev_maxabs": ([c_i64, P, P, c_int, P, P, P], c_int),
        "gi_dev_sumsq": ([c_i64, P, P, c_int, P, P, P], c_int),
        "gi_dev_add_cov": ([c_i64, P, c_i64, P, P, P], c_int),
        "gi_topk_slots": ([c_i64, c_i64], c_i64),
        "gi_dev_topk": ([c_i64, c_i64, c_int, P, P, c_dbl, c_i64, P, P, P, P, P, P, P, P], c_int),
        "gi_dev_scatter": ([c_i64, P, P, P, P], c_int),
        "gi_dev_gather": ([c_i64, P, P, P, P], c_int),
        "gi_fit": ([P, P, P, c_i64, P, P, P, ctypes.POINTER(FitConfig), P, P, c_i64, P,
                    ctypes.POINTER(FitOut)], c_int),
        "gi_fit_sharded": ([P, P, c_i64, P, P, c_i64, P, P, P, ctypes.POINTER(FitConfig), P, P,
                            c_i64, P, ctypes.POINTER(FitOut)], c_int),
        "gi_comm_nccl_available": ([], c_int),
        "gi_comm_nccl_unique_id": ([P], c_int),
        "gi_comm_create_nccl": ([P, c_int, c_int, c_int, P], c_int),
        "gi_comm_create_callbacks": ([c_int, c_int, P, P, P, P], c_int),
        "gi_comm_free": ([P], c_int),
        "gi_matrix_with_masked_stats": ([P, P, P], c_int),
        "gi_fit_many": ([P, P, c_i64, c_int], c_int),
        "gi_cv": ([P, P, P, c_i64, P, c_int, P, c_i64, ctypes.POINTER(FitConfig), c_int, c_int,
                   c_int, P],
                  c_int),
        "gi_batch_create": ([P, c_int, P], c_int),
        "gi_batch_stats": ([P, P, P], c_int),
        "gi_batch_free": ([P], c_int),
        "gi_fit_batched": ([P, P, P, P, c_i64, P, P, P, ctypes.POINTER(FitConfig), P, P, c_i64, P,
                            ctypes.POINTER(FitOut)], c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def lib():
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeError(
                        f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                        "(there is no CPU fallback)")
                h = ctypes.CDLL(LIB_PATH)
                _declare(h)
                _lib = h
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().gi_last_error()
        raise NativeError(msg.decode() if msg else "unknown CUDA failure")


def device_count() -> int:
    out = c_int(0)
    check(lib().gi_device_count(ctypes.byref(out)))
    return int(out.value)


def require_device(device: int = 0) -> None:
    count = device_count()
    if count == 0:
        raise NativeError("no CUDA device is visible; the genoiht B200 path has no CPU fallback")
    if not 0 <= device < count:
        raise NativeError(f"CUDA device {device} out of range (0..{count - 1})")


def device_info(device: int = 0):
    sms = c_int(0)
    mem = c_i64(0)
    l2 = c_i64(0)
    check(lib().gi_device_info(device, ctypes.byref(sms), ctypes.byref(mem), ctypes.byref(l2)))
    return int(sms.value), int(mem.value), int(l2.value)


def ptr(array) -> int:
    """Address of a numpy array, torch tensor or None."""
    if array is None:
        return None
    if hasattr(array, "data_ptr"):
        return array.data_ptr()
    return array.ctypes.data
