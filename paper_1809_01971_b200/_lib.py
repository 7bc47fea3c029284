"""ctypes binding of libfraclap_b200.so (the C ABI in include/fraclap_b200.h).

The library is the product path: there is no CPU fallback.  Loading fails
loudly when the shared object is missing or when no CUDA device is present
at call time.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FL_LIB_OVERRIDE: A/B timing of kernel variants (dev tools only)
LIB_PATH = os.environ.get("FL_LIB_OVERRIDE") or os.path.join(_HERE, "libfraclap_b200.so")

FL_OK, FL_EINVAL, FL_ECUDA, FL_ENOMEM = 0, 1, 2, 3
TAGS = ("g1", "g2", "g3", "g4")

_lock = threading.Lock()
_lib = None

c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_int = ctypes.c_int
P = ctypes.POINTER

# name -> (restype, argtypes); must mirror include/fraclap_b200.h
SIGNATURES = {
    "fl_version": (c_int, []),
    "fl_last_error": (ctypes.c_char_p, []),
    "fl_sm_count": (c_int, []),
    "fl_prepare": (c_int, [c_i64]),
    "fl_dst1": (c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, c_dbl, c_vp]),
    "fl_dst1_core": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_dbl, c_vp]),
    "fl_basis_apply": (c_int, [c_vp, c_int, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp]),
    "fl_core_eval": (c_int, [c_vp, c_int, P(c_i64), P(c_vp), c_int, c_dbl, c_dbl, c_dbl, c_int, c_vp]),
    "fl_cp_to_dense": (c_int, [c_vp, c_int, P(c_i64), c_i64, c_vp, P(c_vp), c_vp]),
    "fl_sinc_factor": (c_int, [c_vp, c_vp, c_i64, c_vp, c_i64, c_dbl, c_vp]),
    "fl_apply_full": (c_int, [c_vp, c_vp, c_vp, c_int, P(c_i64), c_dbl, c_vp]),
    "fl_apply_full_padded": (c_int, [c_vp, c_vp, c_vp, c_vp, c_int, P(c_i64), c_i64, c_dbl, c_vp]),
    "fl_apply_full_lanes": (c_int, [c_vp, c_vp, c_vp, c_vp, c_int, P(c_i64), c_dbl, c_vp]),
    "fl_dst1_core_lanes": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_dbl, c_vp]),
    "fl_dst1_core_lanes_mode0": (c_int, [c_vp, c_vp, c_vp, c_i64, c_dbl, c_vp]),
    "fl_dst1_pass": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_i64, c_i64, c_i64, P(c_i64), P(c_i64), c_dbl, c_vp]),
    "fl_transform_full": (c_int, [c_vp, c_vp, c_int, P(c_i64), c_dbl, c_vp]),
    "fl_cp_apply_mode": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_dbl, c_vp]),
    "fl_cp_gram": (c_int, [c_int, P(c_i64), P(c_vp), c_i64, P(c_vp), c_i64, c_vp, c_vp]),
    "fl_svd_batched": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp]),
    "fl_svd_left_pivoted": (c_int, [c_vp, c_int, c_int, c_vp, c_vp, c_vp]),
    "fl_kr_contract": (c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "fl_qr_r": (c_int, [c_int, P(c_vp), P(c_int), P(c_i64), P(c_i64), P(c_i64), P(c_vp), c_vp]),
    "fl_left_sv_wide": (c_int, [c_int, P(c_vp), P(c_int), P(c_i64), P(c_i64), P(c_i64), P(c_vp), P(c_vp), c_vp]),
    "fl_col_norms": (c_int, [c_vp, c_i64, c_i64, c_vp, c_vp]),
    "fl_col_scale": (c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "fl_pcg_spectral": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl, c_int, c_vp, c_vp, c_vp]),
    "fl_pcg_phase": (c_int, [c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp]),
}
FL_PCG_WORK = 8192


class FraclapError(RuntimeError):
    """A CUDA-side failure inside libfraclap_b200."""


def load():
    """Load (once) and return the shared library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                "libfraclap_b200.so not built (%s); run `python -m paper_1809_01971_b200.build`"
                % LIB_PATH)
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols():
    return sorted(SIGNATURES)


def check(rc):
    if rc == FL_OK:
        return
    msg = load().fl_last_error().decode(errors="replace")
    if rc == FL_EINVAL:
        raise ValueError(msg)
    raise FraclapError("fraclap_b200 error %d: %s" % (rc, msg))


def require_cuda(t=None):
    if not torch.cuda.is_available():
        raise RuntimeError("fraclap_b200 needs a CUDA device (no CPU fallback)")
    if t is not None and not t.is_cuda:
        raise ValueError("expected a CUDA tensor")


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dims_arr(dims):
    return (c_i64 * len(dims))(*[int(n) for n in dims])


def ptr_arr(tensors):
    return (c_vp * len(tensors))(*[t.data_ptr() for t in tensors])


def call(name, *args):
    fn = getattr(load(), name)
    rc = fn(*args)
    if rc == FL_ENOMEM:
        # the library's stream-ordered scratch and torch's caching allocator
        # share the device: hand torch's cached blocks back and retry once
        torch.cuda.empty_cache()
        rc = fn(*args)
    check(rc)
