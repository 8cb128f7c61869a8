"""ctypes binding of libgespmm.so (the C ABI declared in include/gespmm/gespmm.h).

There is no CPU fallback: if the library is missing and cannot be built, or
no CUDA device is present when a compute entry point is called, the call
raises.  The host-only helpers (generators, checksum, reduce/variant lookup)
work without a GPU, which is what the CPU test suite exercises.
"""
from __future__ import annotations

import ctypes as C
import os
import shutil
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# GESPMM_LIB: an alternative build of the same library (A/B kernel experiments,
# tools/variant_build.py); the default is the in-tree build.
# GESPMM_EXPERIMENTAL=1 selects the build with the measured-slower options
# (libgespmm_exp.so, _build.build(experimental=True)).
LIB_PATH = os.environ.get("GESPMM_LIB") or os.path.join(
    _HERE, "libgespmm_exp.so" if os.environ.get("GESPMM_EXPERIMENTAL") == "1" else "libgespmm.so")

# gespmm_status_t
OK, EINVAL, EDIM, ENONCANON, ECUDA, ENOMEM, EUNSUPPORTED = range(7)
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "EDIM", 3: "ENONCANON", 4: "ECUDA", 5: "ENOMEM",
                6: "EUNSUPPORTED"}
# gespmm_reduce_t
SUM, MEAN, MAX, MIN = range(4)
REDUCE = {"sum": SUM, "mean": MEAN, "max": MAX, "min": MIN}
# gespmm_variant_t
VARIANT_TUNED, VARIANT_NAIVE, VARIANT_CRC, VARIANT_CRC_CWM = range(4)
ARG_EDGE, ARG_COLUMN = 0, 1

# Every symbol include/gespmm/gespmm.h declares (checked by the CPU tests).
EXPORTS = [
    "gespmm_options_default", "gespmm_last_error", "gespmm_spmm_device", "gespmm_spmm_host",
    "gespmm_plan_create", "gespmm_plan_execute", "gespmm_plan_describe", "gespmm_plan_launches",
    "gespmm_plan_destroy", "gespmm_validate_device", "gespmm_select_variant",
    "gespmm_reduce_by_name", "gespmm_checksum", "gespmm_make_random_dense",
    "gespmm_randomize_values", "gespmm_gen_uniform", "gespmm_gen_powerlaw", "gespmm_abi_version",
    "gespmm_device_info", "gespmm_launch_count", "gespmm_diag_gather",
    "gespmm_csr_transpose_device", "gespmm_validate_device_as", "gespmm_csr1_write",
    "gespmm_csr1_header", "gespmm_csr1_read_host", "gespmm_csr1_load_device",
    "gespmm_diag_gather_hub", "gespmm_diag_gather_mode", "gespmm_plan_execute_gather",
    "gespmm_peer_barrier", "gespmm_peer_alloc", "gespmm_peer_free", "gespmm_ipc_get_handle",
    "gespmm_ipc_open_handle", "gespmm_ipc_close", "gespmm_multicast_alloc",
    "gespmm_multicast_free", "gespmm_build_flags", "gespmm_from_coo", "gespmm_validate_host",
    "gespmm_mtx_parse", "gespmm_from_coo_device", "gespmm_to_coo_device",
    "gespmm_release_workspace",
]
BUILD_EXPERIMENTAL = 1
MAX_GATHER_DSTS = 8


class Csr(C.Structure):
    _fields_ = [("n_rows", C.c_uint32), ("n_cols", C.c_uint32), ("nnz", C.c_uint64),
                ("row_ptr", C.c_void_p), ("col_ind", C.c_void_p), ("vals", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("variant", C.c_int32), ("cf", C.c_uint32), ("exact", C.c_int32),
                ("arg_kind", C.c_int32), ("validate", C.c_int32),
                ("fault_skip_tail", C.c_int32), ("l2_hints", C.c_int32),
                ("hub_threshold", C.c_int32), ("l2_persist", C.c_int32),
                ("l2_hot_mb", C.c_int32), ("tuned_cf", C.c_int32),
                ("col_slices", C.c_int32), ("rows_per_warp", C.c_int32),
                ("cluster_hot", C.c_int32), ("h2d_pack", C.c_int32),
                ("hot_rows_mb", C.c_int32), ("overlap_prev", C.c_int32)]


_lock = threading.Lock()
_lib = None


class LibraryMissing(RuntimeError):
    """libgespmm.so is absent and could not be built (no silent fallback)."""


def _ensure_built():
    if os.path.exists(LIB_PATH):
        return
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not (os.path.exists(nvcc) or shutil.which("nvcc")):
        raise LibraryMissing(f"{LIB_PATH} is missing and nvcc is unavailable to build it")
    from . import _build
    _build.build()
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(f"build did not produce {LIB_PATH}")


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        _ensure_built()
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32
        L.gespmm_options_default.argtypes = [C.POINTER(Options)]
        L.gespmm_options_default.restype = None
        L.gespmm_last_error.restype = C.c_char_p
        L.gespmm_last_error.argtypes = []
        L.gespmm_spmm_device.argtypes = [C.POINTER(Csr), vp, u32, C.c_int, vp, vp,
                                         C.POINTER(Options), vp]
        L.gespmm_spmm_device.restype = C.c_int
        L.gespmm_spmm_host.argtypes = [C.POINTER(Csr), vp, u32, u32, C.c_int, vp, vp,
                                       C.POINTER(Options)]
        L.gespmm_spmm_host.restype = C.c_int
        L.gespmm_plan_create.argtypes = [C.POINTER(Csr), u32, C.c_int, C.POINTER(Options), vp,
                                         C.POINTER(vp)]
        L.gespmm_plan_create.restype = C.c_int
        L.gespmm_plan_execute.argtypes = [vp, vp, vp, vp, vp]
        L.gespmm_plan_execute.restype = C.c_int
        L.gespmm_plan_describe.argtypes = [vp]
        L.gespmm_plan_describe.restype = C.c_char_p
        L.gespmm_plan_launches.argtypes = [vp]
        L.gespmm_plan_launches.restype = i32
        L.gespmm_plan_destroy.argtypes = [vp]
        L.gespmm_plan_destroy.restype = None
        L.gespmm_validate_device.argtypes = [C.POINTER(Csr), vp]
        L.gespmm_validate_device.restype = C.c_int
        L.gespmm_validate_device_as.argtypes = [C.POINTER(Csr), vp, C.c_char_p]
        L.gespmm_validate_device_as.restype = C.c_int
        L.gespmm_select_variant.argtypes = [u32, C.POINTER(i32), C.POINTER(u32)]
        L.gespmm_select_variant.restype = None
        L.gespmm_reduce_by_name.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.gespmm_reduce_by_name.restype = C.c_int
        L.gespmm_checksum.argtypes = [vp, u32, u32]
        L.gespmm_checksum.restype = u64
        L.gespmm_make_random_dense.argtypes = [u32, u32, u64, vp]
        L.gespmm_make_random_dense.restype = None
        L.gespmm_randomize_values.argtypes = [vp, u64, u64]
        L.gespmm_randomize_values.restype = None
        L.gespmm_gen_uniform.argtypes = [u32, u64, u64, i32, vp, vp, vp]
        L.gespmm_gen_uniform.restype = C.c_int
        L.gespmm_gen_powerlaw.argtypes = [u32, u64, u32, C.c_double, u64, i32, vp, vp, vp]
        L.gespmm_gen_powerlaw.restype = C.c_int
        L.gespmm_abi_version.argtypes = []
        L.gespmm_abi_version.restype = i32
        L.gespmm_from_coo.argtypes = [u32, u32, u64, vp, vp, vp, i32, vp, vp, vp,
                                      C.POINTER(u64)]
        L.gespmm_from_coo.restype = C.c_int
        L.gespmm_validate_host.argtypes = [C.POINTER(Csr), u64, u64, u64, C.c_char_p, u64,
                                           C.POINTER(u64)]
        L.gespmm_validate_host.restype = u64
        L.gespmm_mtx_parse.argtypes = [C.c_char_p, u64, C.POINTER(u32), C.POINTER(u32),
                                       C.POINTER(u64), vp, vp, vp]
        L.gespmm_mtx_parse.restype = C.c_int
        L.gespmm_build_flags.argtypes = []
        L.gespmm_build_flags.restype = i32
        L.gespmm_device_info.argtypes = [C.POINTER(i32), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int64), C.POINTER(i32), C.POINTER(i32)]
        L.gespmm_device_info.restype = C.c_int
        L.gespmm_diag_gather.argtypes = [vp, u64, vp, u32, vp, i32, i32, vp]
        L.gespmm_diag_gather.restype = C.c_int
        L.gespmm_diag_gather_hub.argtypes = [vp, u64, vp, u32, vp, i32, vp]
        L.gespmm_diag_gather_hub.restype = C.c_int
        L.gespmm_diag_gather_mode.argtypes = [vp, u64, vp, vp, i32, i32, vp]
        L.gespmm_diag_gather_mode.restype = C.c_int
        L.gespmm_csr_transpose_device.argtypes = [C.POINTER(Csr), vp, vp, vp, vp]
        L.gespmm_csr_transpose_device.restype = C.c_int
        L.gespmm_from_coo_device.argtypes = [u32, u32, u64, vp, vp, vp, i32, vp, vp, vp,
                                             C.POINTER(u64), vp]
        L.gespmm_from_coo_device.restype = C.c_int
        L.gespmm_to_coo_device.argtypes = [C.POINTER(Csr), vp, vp, vp, vp]
        L.gespmm_to_coo_device.restype = C.c_int
        L.gespmm_release_workspace.argtypes = []
        L.gespmm_release_workspace.restype = None
        L.gespmm_csr1_write.argtypes = [C.c_char_p, C.POINTER(Csr)]
        L.gespmm_csr1_write.restype = C.c_int
        L.gespmm_csr1_header.argtypes = [C.c_char_p, C.POINTER(u32), C.POINTER(u32),
                                         C.POINTER(u64)]
        L.gespmm_csr1_header.restype = C.c_int
        L.gespmm_csr1_read_host.argtypes = [C.c_char_p, vp, vp, vp]
        L.gespmm_csr1_read_host.restype = C.c_int
        L.gespmm_csr1_load_device.argtypes = [C.c_char_p, vp, vp, vp, i32, vp]
        L.gespmm_csr1_load_device.restype = C.c_int
        L.gespmm_plan_execute_gather.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp]
        L.gespmm_plan_execute_gather.restype = C.c_int
        L.gespmm_peer_barrier.argtypes = [vp, i32, i32, u32, u32, vp, vp]
        L.gespmm_peer_barrier.restype = C.c_int
        L.gespmm_peer_alloc.argtypes = [u64, C.POINTER(vp)]
        L.gespmm_peer_alloc.restype = C.c_int
        L.gespmm_peer_free.argtypes = [vp]
        L.gespmm_peer_free.restype = C.c_int
        L.gespmm_ipc_get_handle.argtypes = [vp, C.c_char_p]
        L.gespmm_ipc_get_handle.restype = C.c_int
        L.gespmm_ipc_open_handle.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.gespmm_ipc_open_handle.restype = C.c_int
        L.gespmm_ipc_close.argtypes = [vp]
        L.gespmm_ipc_close.restype = C.c_int
        L.gespmm_multicast_alloc.argtypes = [u64, C.POINTER(vp), C.POINTER(vp)]
        L.gespmm_multicast_alloc.restype = C.c_int
        L.gespmm_multicast_free.argtypes = [vp]
        L.gespmm_multicast_free.restype = C.c_int
        L.gespmm_launch_count.argtypes = []
        L.gespmm_launch_count.restype = u64
        _lib = L
    return _lib


def last_error() -> str:
    return lib().gespmm_last_error().decode(errors="replace")


def default_options(**kw) -> Options:
    o = Options()
    lib().gespmm_options_default(C.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, int(v))
    return o


def experimental_built() -> bool:
    """True when the loaded library carries the experimental (measured-slower)
    options: GESPMM_EXPERIMENTAL=1 build, or GESPMM_LIB pointing at one."""
    return bool(lib().gespmm_build_flags() & BUILD_EXPERIMENTAL)


def launch_count() -> int:
    return int(lib().gespmm_launch_count())
