"""Loader for the sm_100a shared library (the C ABI in include/epsgraph_b200.h).

The library is built in-tree (``python -c "import __graft_entry__ as g;
g.build()"`` or :func:`build`) and loaded with ctypes; ctypes releases the
GIL for the duration of every call.  There is no fallback: if the library is
missing or no CUDA device is visible, compute entry points raise.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.environ.get("EG_LIB_PATH") or os.path.join(_HERE, "_native", "libepsgraph_b200.so")
_SRC_DIR = os.path.join(_HERE, "csrc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]

EG_OK, EG_ERR_ARG, EG_ERR_CUDA, EG_ERR_CAPACITY, EG_ERR_WORKSPACE, EG_ERR_UNSUPPORTED = range(6)
METRIC_COSINE, METRIC_EUCLIDEAN = 0, 1
MAX_LENGTH, MAX_BLOCKS = 256, 64

_lock = threading.Lock()
_lib = None


def sources():
    return sorted(os.path.join(_SRC_DIR, f) for f in os.listdir(_SRC_DIR)
                  if f.endswith((".cu", ".cuh")))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/capi.cu (which includes the other sources) for sm_100a."""
    srcs = sources() + [os.path.join(_ROOT, "include", "epsgraph_b200.h")]
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(s) for s in srcs)):
        return LIB_PATH
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    tmp = LIB_PATH + ".tmp"
    cmd = ["nvcc", *NVCC_FLAGS, "-o", tmp, os.path.join(_SRC_DIR, "capi.cu")]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def _declare(lib):
    P, i32, i64, sz, dbl = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t,
                            ctypes.c_double)
    I = ctypes.c_int
    sig = {
        "eg_last_error": ([], ctypes.c_char_p),
        "eg_set_option": ([ctypes.c_char_p, ctypes.c_longlong], I),
        "eg_reset_options": ([], None),
        "eg_version": ([], I),
        "eg_device_sm_count": ([], I),
        "eg_launch_count": ([], ctypes.c_longlong),
        "eg_profile_enable": ([I], None),
        "eg_profile_class_name": ([I], ctypes.c_char_p),
        "eg_profile_read": ([P, P, I], I),
        "eg_row_stats": ([P, I, i64, i32, P, P, P], I),
        "eg_debug_set_tc_dump": ([P], None),
        "eg_debug_msm_stats": ([P, I], I),
        "eg_project_workspace": ([i64, i32, i32, i32], sz),
        "eg_project": ([P, I, i64, i32, P, P, P, i32, i32, P, P, sz, P, P], I),
        "eg_project_rows": ([P, I, i64, i32, P, P, P, P, i32, i32, P, P, sz, P, P], I),
        "eg_msm_workspace": ([i64, i32, i32], sz),
        "eg_msm_plan_workspace": ([i32, i32, i32], sz),
        "eg_msm_plan": ([P, i64, i32, i32, i32, dbl, P, P, P, sz, P], I),
        "eg_msm_estimate_pairs": ([P, i64, i32, i32, i32, P, P, sz, P], I),
        "eg_msm_pairs": ([P, i64, i32, i32, P, i32, i32, P, P, i64, P, P, i64, P, P, sz, P], I),
        "eg_msm_pairs_design": ([P, i64, i32, i32, P, i32, i32, P, P, i64, P, i32, P, P, i64, P, P,
                                 sz, P], I),
        "eg_msm_design": ([i32, i32, i32, P, i32], I),
        "eg_xrep_filter": ([P, P, i64, P, i64, i32, i32, i32, P, P, P], I),
        "eg_xrep_filter_async": ([P, P, i64, P, i64, i32, i32, i32, P, P, P], I),
        "eg_hamming_filter_async": ([P, P, i64, P, i64, i32, i32, i32, P, P, P], I),
        "eg_grouped_sort_workspace": ([i64, i32], sz),
        "eg_grouped_sort": ([P, i64, i32, P, i32, ctypes.c_uint64, i32, P, P, P, P, sz, P], I),
        "eg_first_witness": ([P, i64, P, i32, i32, i32, P, P], I),
        "eg_sort_workspace": ([i64, I], sz),
        "eg_sort_keys": ([P, P, i64, i32, P, sz, P], I),
        "eg_sort_pair_keys": ([P, i64, i64, P, sz, P], I),
        "eg_merge_runs_workspace": ([i64, I], sz),
        "eg_merge_runs": ([P, P, P, i32, P, sz, P], I),
        "eg_compact_workspace": ([i64], sz),
        "eg_compact_keys": ([P, P, i64, P, P, P, sz, P], I),
        "eg_verify_workspace": ([i64], sz),
        "eg_verify": ([P, I, i64, i32, P, P, i64, i32, dbl, P, P, P, P, sz, P], I),
        "eg_bf_cosine_workspace": ([i64, i32], sz),
        "eg_bf_cosine_candidates": ([P, I, i64, i32, P, dbl, P, i64, P, P, sz, P], I),
        "eg_bf_hamming_workspace": ([], sz),
        "eg_bf_hamming": ([P, i64, i32, i32, P, i64, P, P, sz, P], I),
        "eg_format_edges_workspace": ([i64], sz),
        "eg_format_edges": ([P, P, i64, P, i64, P, P, sz, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def lib():
    """The loaded library; raises if it is missing (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"CUDA extension not built: {LIB_PATH} is missing "
                    "(run __graft_entry__.build()); there is no CPU fallback")
            _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


class NativeError(RuntimeError):
    pass


def check(rc: int, what: str):
    """Map a C-ABI status to the reference's exception types."""
    if rc == EG_OK:
        return
    msg = lib().eg_last_error().decode(errors="replace")
    if rc == EG_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    if rc == EG_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")


class Profile:
    """Per-kernel-class CUDA-event timing collected inside the library."""

    def __init__(self):
        self.lib = lib()

    def start(self):
        self.lib.eg_profile_read(None, None, 0)   # drop stale records
        self.lib.eg_profile_enable(1)

    def stop(self) -> dict:
        self.lib.eg_profile_enable(0)
        nc = 32
        ms = (ctypes.c_double * nc)()
        cnt = (ctypes.c_longlong * nc)()
        k = self.lib.eg_profile_read(ctypes.addressof(ms), ctypes.addressof(cnt), nc)
        out = {}
        for c in range(k):
            if cnt[c]:
                out[self.lib.eg_profile_class_name(c).decode()] = {"ms": ms[c], "count": int(cnt[c])}
        return out


class options:
    """Context manager for the library's path overrides (eg_set_option):
    ``with options(project_path=1): ...`` -- tests use it to reach the
    alternative kernels; the defaults are restored on exit."""

    def __init__(self, **kw):
        self.kw = kw

    def __enter__(self):
        for k, v in self.kw.items():
            check(lib().eg_set_option(k.encode(), int(v)), f"option {k}")
        return self

    def __exit__(self, *exc):
        lib().eg_reset_options()
        return False


def launch_count() -> int:
    return int(lib().eg_launch_count())
