"""ctypes binding of libsbt200.so (the C ABI declared in include/sbt200.h).

The library is the ONLY compute path: there is no CPU fallback.  Loading fails
loudly when the shared object is missing or lacks a declared symbol.
"""
from __future__ import annotations

import ctypes
import threading
from ctypes import c_double, c_float, c_int, c_int64, c_void_p
from pathlib import Path

import os

# SBT_LIB: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = Path(os.environ.get("SBT_LIB") or
                Path(__file__).resolve().parent / "lib" / "libsbt200.so")

SBT_OK = 0
SBT_EINVAL = -1
SBT_EUNSUPPORTED = -2
SBT_ECUDA = -3

_I = c_int64
_P = c_void_p


def _core_sig(real):
    # m, n, k, alpha, a, oa, ars, acs, b, ob, brs, bcs, beta, c, oc, crs, ccs, stream
    return [_I, _I, _I, real, _P, _I, _I, _I, _P, _I, _I, _I, real, _P, _I, _I, _I, _P]


def _batched_sig(real, stream=True):
    sig = [_I, _I, _I, real, _P, _I, _I, _I, _I, _P, _I, _I, _I, _I, real, _P, _I, _I, _I, _I, _I]
    return sig + [_P] if stream else sig


def _batched2_sig(real):
    return [_I, _I, _I, real, _P, _I, _I, _I, _I, _I, _P, _I, _I, _I, _I, _I, real, _P, _I, _I,
            _I, _I, _I, _I, _I, _P]


class GemmDesc(ctypes.Structure):
    """sbt_gemm_desc (include/sbt200.h): one problem of a grouped call."""
    _fields_ = [("m", c_int64), ("n", c_int64), ("k", c_int64),
                ("alpha", c_double), ("beta", c_double),
                ("a", c_void_p), ("oa", c_int64), ("ars", c_int64), ("acs", c_int64),
                ("apt", c_int64), ("apt2", c_int64),
                ("b", c_void_p), ("ob", c_int64), ("brs", c_int64), ("bcs", c_int64),
                ("bpt", c_int64), ("bpt2", c_int64),
                ("c", c_void_p), ("oc", c_int64), ("crs", c_int64), ("ccs", c_int64),
                ("cpt", c_int64), ("cpt2", c_int64),
                ("batch", c_int64), ("batch2", c_int64)]


# every symbol include/sbt200.h declares, with its ctypes signature
SIGNATURES = {
    "sbt_version": ([], c_int),
    "sbt_last_error": ([], ctypes.c_char_p),
    "sbt_launch_count": ([], c_int64),
    "sbt_last_kernel": ([], ctypes.c_char_p),
    "sbt_set_kernel_override": ([c_int], c_int),
    "sbt_set_accumulation": ([c_int], c_int),
    "sbt_probe_fp64_peak": ([c_int, ctypes.POINTER(c_double)], c_int),
    "sbt_probe_tf32_peak": ([ctypes.POINTER(c_double)], c_int),
    "sbt_probe_tf32_sustained": ([c_double, ctypes.POINTER(c_double)], c_int),
    "sbt_permute_f64": ([c_int, ctypes.POINTER(c_int64), _P, ctypes.POINTER(c_int64), _P, _P],
                        c_int),
    "sbt_permute_f32": ([c_int, ctypes.POINTER(c_int64), _P, ctypes.POINTER(c_int64), _P, _P],
                        c_int),
    "sbt_ritz_f64": ([_P, _P, c_int64, c_int, c_int, c_double, _P, _P, _P, _P, _P, _P, _P],
                     c_int),
    "sbt_hooi_factor_ws_bytes": ([c_int, ctypes.POINTER(c_int64), c_int, c_int], ctypes.c_size_t),
    "sbt_hooi_factor_f32": ([_P, c_int, ctypes.POINTER(c_int64), c_int, _P, c_int64, c_int, c_int,
                             c_double, _P, ctypes.c_size_t, _P, _P, _P, _P, _P, _P, _P], c_int),
    "sbt_hooi_factor_f64": ([_P, c_int, ctypes.POINTER(c_int64), c_int, _P, c_int64, c_int, c_int,
                             c_double, _P, ctypes.c_size_t, _P, _P, _P, _P, _P, _P, _P], c_int),
    "sbt_mode_product_acc64_f32": ([_P, c_int, ctypes.POINTER(c_int64), c_int, _P, c_int64, c_int,
                                    _P, _P], c_int),
    "sbt_mode_product_acc64_f64": ([_P, c_int, ctypes.POINTER(c_int64), c_int, _P, c_int64, c_int,
                                    _P, _P], c_int),
    "sbt_hooi_status_f32": ([_P, c_int64, _P, c_int, _P, _P], c_int),
    "sbt_hooi_status_f64": ([_P, c_int64, _P, c_int, _P, _P], c_int),
    "sbt_batched_core_group_f32": ([c_int, ctypes.POINTER(GemmDesc), _P], c_int),
    "sbt_batched_core_group_f64": ([c_int, ctypes.POINTER(GemmDesc), _P], c_int),
    "sbt_gemm_core_f64": (_core_sig(c_double), c_int),
    "sbt_gemm_core_f32": (_core_sig(c_float), c_int),
    "sbt_batched_core_f64": (_batched_sig(c_double), c_int),
    "sbt_batched_core_f32": (_batched_sig(c_float), c_int),
    "sbt_ext_batched_core_f64": (_batched_sig(c_double), c_int),
    "sbt_ext_batched_core_f32": (_batched_sig(c_float), c_int),
    "sbt_batched2_core_f64": (_batched2_sig(c_double), c_int),
    "sbt_batched2_core_f32": (_batched2_sig(c_float), c_int),
    "sbt_batched_core_host_f64": (_batched_sig(c_double, stream=False), c_int),
    "sbt_batched_core_host_f32": (_batched_sig(c_float, stream=False), c_int),
}

_lock = threading.Lock()
_lib = None


class LibraryError(RuntimeError):
    pass


def load():
    """Load (once) and return the CDLL with argtypes set."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise LibraryError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1606_05696_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (args, res) in SIGNATURES.items():
            if os.environ.get("SBT_LIB") and not hasattr(lib, name):
                continue  # A/B experiments with an older build: tolerate new symbols
            fn = getattr(lib, name)  # AttributeError = missing export -> loud failure
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc == SBT_OK:
        return
    msg = load().sbt_last_error().decode(errors="replace")
    if rc == SBT_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({rc}): {msg}")


def launch_count() -> int:
    return int(load().sbt_launch_count())


def last_kernel() -> str:
    return load().sbt_last_kernel().decode()


def set_kernel_override(which) -> None:
    """0/'auto', 1/'generic', 2/'tensor', 3/'small'."""
    names = {"auto": 0, "generic": 1, "tensor": 2, "small": 3}
    which = names.get(which, which)
    check(load().sbt_set_kernel_override(int(which)), "sbt_set_kernel_override")


class fast_accumulation:
    """Context manager: narrow fp32 tensor-core tiles launched by this thread
    inside the block use the fast (truncating) accumulator instead of the
    unbiased default (``sbt_set_accumulation``)."""

    def __enter__(self):
        self.prev = load().sbt_set_accumulation(0)
        return self

    def __exit__(self, *exc):
        load().sbt_set_accumulation(self.prev)
        return False


def probe_fp64_peak(kind: str = "dmma") -> float:
    """Measured fp64 TFLOP/s of the DMMA tensor pipe ("dmma") or DFMA ("dfma")."""
    out = c_double(0.0)
    check(load().sbt_probe_fp64_peak(0 if kind == "dmma" else 1, ctypes.byref(out)),
          "sbt_probe_fp64_peak")
    return out.value


def probe_tf32_peak() -> float:
    """Measured dense TF32 TFLOP/s of the tcgen05 tensor pipe (3xTF32 peak = / 3)."""
    out = c_double(0.0)
    check(load().sbt_probe_tf32_peak(ctypes.byref(out)), "sbt_probe_tf32_peak")
    return out.value


def probe_tf32_sustained(seconds: float = 3.0) -> float:
    """Dense TF32 TFLOP/s of the tcgen05 pipe under sustained load (power cap)."""
    out = c_double(0.0)
    check(load().sbt_probe_tf32_sustained(float(seconds), ctypes.byref(out)),
          "sbt_probe_tf32_sustained")
    return out.value
