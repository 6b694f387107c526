"""ctypes binding of the C ABI in include/elattn_gpu.h.

The shared library is built in-tree (``paper_2105_04779_b200/libelattn_gpu.so``)
by ``__graft_entry__.build()``.  There is no fallback: if the library is
missing or fails to load, every call raises :class:`ElattnUnavailable`.
"""
from __future__ import annotations

import ctypes
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().with_name("libelattn_gpu.so")

# Status codes (include/elattn_gpu.h) -> reference exception types (errors.hpp:8-36).
OK, ERR_SHAPE, ERR_PARAM, ERR_STATE, ERR_NUMERIC, ERR_CUDA, ERR_OOM, ERR_UNSUPPORTED = range(8)
DTYPE_F32, DTYPE_BF16 = 0, 1

# Every symbol declared in include/elattn_gpu.h (checked by tests/test_capi_load.py).
EXPORTED_SYMBOLS = (
    "elattn_gpu_version",
    "elattn_gpu_last_error_message",
    "elattn_gpu_params_create",
    "elattn_gpu_params_destroy",
    "elattn_gpu_params_info",
    "elattn_gpu_build_el_query",
    "elattn_gpu_el_attention_folded",
    "elattn_gpu_el_attention_step",
    "elattn_gpu_el_attention_step_indexed",
    "elattn_gpu_el_attention_decode",
    "elattn_gpu_workspace_size",
    "elattn_gpu_decode_kernel_kind",
    "elattn_gpu_launch_count",
    "elattn_gpu_decoder_create",
    "elattn_gpu_decoder_run",
    "elattn_gpu_decoder_destroy",
    "elattn_gpu_decoder_kernels_per_run",
    "elattn_gpu_cache_append",
    "elattn_gpu_cache_gather",
    "elattn_gpu_cache_append_indexed",
    "elattn_gpu_cache_fork_workspace",
    "elattn_gpu_cache_fork",
    "elattn_gpu_kv_append",
    "elattn_gpu_mixed_self_attention",
    "elattn_gpu_mixed_workspace_size",
    "elattn_gpu_beam_candidates",
    "elattn_gpu_lane_gather",
    "elattn_gpu_reset_launch_count",
    "elattn_gpu_mha_kv_build",
    "elattn_gpu_mha_workspace_size",
    "elattn_gpu_mha_attention",
)


class ElattnError(RuntimeError):
    """Base of the library's errors (mirrors std::exception in the reference)."""

    status = -1


class ShapeError(ElattnError, ValueError):
    status = ERR_SHAPE


class ParamError(ElattnError, ValueError):
    status = ERR_PARAM


class StateError(ElattnError):
    status = ERR_STATE


class NumericError(ElattnError):
    status = ERR_NUMERIC


class CudaError(ElattnError):
    status = ERR_CUDA


class OutOfMemoryError(ElattnError):
    status = ERR_OOM


class UnsupportedError(ElattnError):
    status = ERR_UNSUPPORTED


class ElattnUnavailable(ElattnError):
    """The CUDA library is not built / not loadable: no silent fallback exists."""


_ERRORS = {c.status: c for c in (ShapeError, ParamError, StateError, NumericError, CudaError,
                                 OutOfMemoryError, UnsupportedError)}

_lock = threading.Lock()
_lib = None

vp, sz, i32, i64, dp = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)


def _declare(lib: ctypes.CDLL) -> None:
    lib.elattn_gpu_version.restype = ctypes.c_char_p
    lib.elattn_gpu_last_error_message.restype = ctypes.c_char_p
    lib.elattn_gpu_params_create.argtypes = [i32, i32, i32, i32, i32, i32] + [vp] * 8 + [ctypes.POINTER(vp)]
    lib.elattn_gpu_params_destroy.argtypes = [vp]
    lib.elattn_gpu_params_info.argtypes = [vp] + [ctypes.POINTER(i32)] * 4
    lib.elattn_gpu_build_el_query.argtypes = [vp, vp, i32, vp, vp, vp, sz, vp]
    lib.elattn_gpu_el_attention_folded.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, vp, vp, sz, vp]
    lib.elattn_gpu_el_attention_step.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp, vp, sz, vp]
    lib.elattn_gpu_el_attention_step_indexed.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, vp, vp, sz, vp]
    lib.elattn_gpu_el_attention_decode.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp, vp]
    lib.elattn_gpu_workspace_size.argtypes = [vp, i32, i32, i32]
    lib.elattn_gpu_workspace_size.restype = sz
    lib.elattn_gpu_decode_kernel_kind.argtypes = [vp, i32]
    lib.elattn_gpu_launch_count.restype = i64
    lib.elattn_gpu_decoder_create.argtypes = [ctypes.POINTER(vp), i32, vp, vp, i32, i32, i32, vp, vp,
                                              ctypes.POINTER(vp)]
    lib.elattn_gpu_decoder_run.argtypes = [vp, vp]
    lib.elattn_gpu_decoder_destroy.argtypes = [vp]
    lib.elattn_gpu_decoder_kernels_per_run.argtypes = [vp]
    lib.elattn_gpu_decoder_kernels_per_run.restype = i64
    lib.elattn_gpu_cache_append.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp]
    lib.elattn_gpu_cache_gather.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp]
    lib.elattn_gpu_cache_append_indexed.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, vp]
    lib.elattn_gpu_cache_fork_workspace.argtypes = [i32, i32, i32]
    lib.elattn_gpu_cache_fork_workspace.restype = sz
    lib.elattn_gpu_cache_fork.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, i32, i32, i32, vp, sz, vp]
    lib.elattn_gpu_kv_append.argtypes = [vp, vp, i32, vp, vp, i32, i32, vp]
    lib.elattn_gpu_mixed_self_attention.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp, vp, i32, i32, vp, vp, sz, vp]
    lib.elattn_gpu_mixed_workspace_size.argtypes = [vp, i32, i32]
    lib.elattn_gpu_mixed_workspace_size.restype = sz
    lib.elattn_gpu_beam_candidates.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp, vp, vp, vp]
    lib.elattn_gpu_lane_gather.argtypes = [vp, vp, vp, i32, i32, ctypes.c_int64, vp]
    lib.elattn_gpu_mha_kv_build.argtypes = [vp, vp, i32, i32, vp, vp, vp]
    lib.elattn_gpu_mha_workspace_size.argtypes = [vp, i32, i32]
    lib.elattn_gpu_mha_workspace_size.restype = sz
    lib.elattn_gpu_mha_attention.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, vp, vp, sz, vp]
    for name in EXPORTED_SYMBOLS:
        fn = getattr(lib, name)
        if fn.restype is ctypes.c_int and name not in ("elattn_gpu_decode_kernel_kind",
                                                       "elattn_gpu_cache_fork_workspace"):
            fn.restype = i32


def lib() -> ctypes.CDLL:
    """Load libelattn_gpu.so once (raises ElattnUnavailable if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ElattnUnavailable(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            try:
                handle = ctypes.CDLL(str(LIB_PATH))
            except OSError as exc:  # pragma: no cover - loader failure is environment specific
                raise ElattnUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
            _declare(handle)
            _lib = handle
    return _lib


def check(rc: int) -> None:
    """Raise the reference-typed exception for a non-zero status."""
    if rc == OK:
        return
    msg = lib().elattn_gpu_last_error_message().decode(errors="replace")
    raise _ERRORS.get(rc, ElattnError)(msg or f"elattn status {rc}")


def version() -> str:
    return lib().elattn_gpu_version().decode()
