"""ctypes binding of the C ABI in include/absp.h (libabsp.so, built in-tree).

The product path has no fallback: if the library is missing or fails to load,
importing the runtime raises. Status codes map onto Python exceptions that
mirror the reference's C++ exception classes:

    ABSP_EINVAL    -> InvalidArgument (ValueError)      std::invalid_argument
    ABSP_ERANGE    -> OutOfRange (IndexError)           std::out_of_range
    ABSP_ECAPACITY -> CapacityError (RuntimeError)      std::runtime_error
    ABSP_ESTATE    -> LogicError (RuntimeError)         std::logic_error
    ABSP_ECUDA     -> CudaError (RuntimeError)
    ABSP_ENOMEM    -> MemoryError
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libabsp.so"
# ABSP_LIB=<file name in lib/> loads another build of the same ABI (A/B measurements)
if os.environ.get("ABSP_LIB"):
    LIB_PATH = LIB_PATH.with_name(os.path.basename(os.environ["ABSP_LIB"]))

ABSP_MAX_CANDIDATES = 16

EXPORTED = [
    "absp_abi_version", "absp_last_error", "absp_config_validate", "absp_ctx_create",
    "absp_ctx_destroy", "absp_set_assignment", "absp_kv_bind", "absp_build_store", "absp_append", "absp_select",
    "absp_attend", "absp_attend_selected", "absp_decode_step", "absp_decode_step_host", "absp_last_selection",
    "absp_get_layer_info", "absp_download_store", "absp_download_scores", "absp_download_selection", "absp_download_filter_scores",
    "absp_fill_synthetic_bf16", "absp_launch_count", "absp_attend_validate", "absp_layout_version", "absp_set_filter_diagnostics",
    "absp_engine_create", "absp_engine_destroy", "absp_engine_prefill", "absp_engine_step", "absp_engine_info",
    "absp_full_attention", "absp_attention_recall", "absp_profile_sample", "absp_select_step",
]


class AbspError(Exception):
    status = -1


class InvalidArgument(AbspError, ValueError):
    status = 1


class OutOfRange(AbspError, IndexError):
    status = 2


class CapacityError(AbspError, RuntimeError):
    status = 3


class LogicError(AbspError, RuntimeError):
    status = 4


class CudaError(AbspError, RuntimeError):
    status = 5


class DeviceMemoryError(AbspError, MemoryError):
    status = 6


_ERRORS = {c.status: c for c in (InvalidArgument, OutOfRange, CapacityError, LogicError, CudaError,
                                 DeviceMemoryError)}


class Config(C.Structure):
    _fields_ = [
        ("num_kv_heads", C.c_uint32),
        ("num_q_heads", C.c_uint32),
        ("head_dim", C.c_uint32),
        ("page_size", C.c_uint32),
        ("num_candidates", C.c_uint32),
        ("candidate_block_sizes", C.c_uint32 * ABSP_MAX_CANDIDATES),
        ("token_budget", C.c_uint32),
        ("centroid_method", C.c_uint32),
        ("quant_bits", C.c_uint32),
        ("quant_mode", C.c_uint32),
        ("max_batch", C.c_uint32),
        ("max_seq_len", C.c_uint32),
        ("num_layers", C.c_uint32),
    ]


class LayerInfo(C.Structure):
    _fields_ = [
        ("batch", C.c_uint32),
        ("max_select", C.c_uint32),
        ("total_centroids", C.c_uint64),
        ("store_bytes", C.c_uint64),
        ("kv_bytes_selected", C.c_uint64),
        ("code_bytes", C.c_uint64),
    ]


_lib = None


def load(path: Path | str | None = None) -> C.CDLL:
    """Load libabsp.so; raises if it is absent (no silent fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise FileNotFoundError(f"{p} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
    L = C.CDLL(str(p))
    vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
    u32p = C.POINTER(u32)
    L.absp_abi_version.restype = C.c_int
    L.absp_last_error.restype = C.c_char_p
    L.absp_config_validate.argtypes = [C.POINTER(Config)]
    L.absp_ctx_create.argtypes = [C.c_int, C.POINTER(Config), C.POINTER(vp)]
    L.absp_ctx_destroy.argtypes = [vp]
    L.absp_set_assignment.argtypes = [vp, u32, u32p]
    L.absp_kv_bind.argtypes = [vp, u32, vp, vp, u64, vp, u32, u32p, u32]
    L.absp_build_store.argtypes = [vp, u32, vp]
    L.absp_append.argtypes = [vp, u32, vp, vp, vp]
    L.absp_select.argtypes = [vp, u32, vp, vp, u32, vp, vp]
    L.absp_attend.argtypes = [vp, u32, vp, vp, u32, vp, vp, vp]
    L.absp_attend_selected.argtypes = [vp, u32, vp, vp, vp]
    L.absp_decode_step.argtypes = [vp, u32, vp, vp, vp]
    L.absp_select_step.argtypes = [vp, u32, vp, vp]
    L.absp_decode_step_host.argtypes = [vp, u32, vp, vp, vp]
    L.absp_last_selection.argtypes = [vp, u32, C.POINTER(vp), u32p, C.POINTER(vp)]
    L.absp_get_layer_info.argtypes = [vp, u32, C.POINTER(LayerInfo)]
    L.absp_download_store.argtypes = [vp, u32, u32] + [vp] * 9
    L.absp_download_scores.argtypes = [vp, u32, u32, vp]
    L.absp_download_selection.argtypes = [vp, u32, vp, vp]
    L.absp_download_filter_scores.argtypes = [vp, u32, u32, vp, vp]
    L.absp_fill_synthetic_bf16.argtypes = [vp, u64, u64, u64, vp]
    L.absp_attend_validate.argtypes = [vp, u32, vp]
    L.absp_set_filter_diagnostics.argtypes = [vp, u32, C.c_int]
    L.absp_layout_version.argtypes = [vp, u32]
    L.absp_layout_version.restype = u64
    L.absp_engine_create.argtypes = [C.c_int, C.POINTER(Config), u32p, u64, C.POINTER(vp)]
    L.absp_engine_destroy.argtypes = [vp]
    L.absp_engine_prefill.argtypes = [vp, vp, u64, vp, u64, u64]
    L.absp_engine_step.argtypes = [vp, vp, u64, vp, u64, vp, u64, vp, vp, u32, vp, C.POINTER(C.c_int)]
    L.absp_engine_info.argtypes = [vp, C.POINTER(u64), C.POINTER(u32), C.POINTER(vp)]
    L.absp_full_attention.argtypes = [vp, u32, vp, vp, vp, u64, vp]
    L.absp_attention_recall.argtypes = [vp, u32, vp, u64, vp, u32, vp, vp, vp]
    L.absp_profile_sample.argtypes = [C.c_int, C.POINTER(Config), vp, vp, vp, u64, u32p, vp, vp]
    L.absp_launch_count.argtypes = [vp]
    L.absp_launch_count.restype = u64
    for name in EXPORTED:
        if name not in ("absp_abi_version", "absp_last_error", "absp_launch_count"):
            getattr(L, name).restype = C.c_int
    if path is None:
        _lib = L
    return L


def check(status: int) -> None:
    if status != 0:
        msg = load().absp_last_error().decode(errors="replace")
        raise _ERRORS.get(status, AbspError)(msg)
