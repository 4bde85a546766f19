"""ctypes binding of the C ABI in include/obtree_b200.h.

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a)
into ``paper_2211_00391_b200/_lib/libobtree_b200.so``.  There is no fallback:
if the library is missing or no CUDA device is visible, every GPU entry point
raises ``NativeUnavailable`` naming the cause.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "libobtree_b200.so"
LIB_PATH = Path(__file__).resolve().parent / "_lib" / LIB_NAME

OBT_OK = 0
OBT_E_INVALID = -1
OBT_E_CUDA = -2
OBT_E_UNSUPPORTED = -3
OBT_E_NOMEM = -4

LAYOUT_OBJECT_MAJOR = 0
LAYOUT_FEATURE_MAJOR = 1
SHARD_OBJECTS = 0
SHARD_TREES = 1
PRECISION_BINARY64 = 0
PRECISION_BINARY16 = 1

LEAF_STORAGE_NAMES = {0: "fp64", 1: "fp32", 2: "fp16"}

# Every symbol include/obtree_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED_SYMBOLS = (
    "obt_model_create",
    "obt_model_destroy",
    "obt_model_info",
    "obt_model_quantize_kernel",
    "obt_model_multi_kernel",
    "obt_workspace_size",
    "obt_predict_dev",
    "obt_predict_host",
    "obt_predict_sharded",
    "obt_quantize_dev",
    "obt_leaf_indices_dev",
    "obt_predict_dev_marked",
    "obt_event_create",
    "obt_event_record",
    "obt_event_elapsed_ms",
    "obt_event_destroy",
    "obt_last_launch_count",
    "obt_last_error",
    "obt_abi_version",
    "obt_set_path_option",
    "obt_get_path_option",
)

# Planner choices a caller may force (obt_set_path_option; -1 = automatic).
PATH_OPTIONS = ("desc_source", "tpw", "wide", "fan", "pdl", "tail_split", "quant_lut", "lut_cells",
                "leaf_storage", "multi_staged", "leaf_select")


class NativeUnavailable(RuntimeError):
    """The CUDA library cannot be used (not built, or no GPU)."""


class NativeError(RuntimeError):
    """A C ABI call returned an error code."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class ModelDesc(ctypes.Structure):
    _fields_ = [
        ("n_features", ctypes.c_int32),
        ("n_trees", ctypes.c_int32),
        ("max_depth", ctypes.c_int32),
        ("n_outputs", ctypes.c_int32),
        ("border_counts", ctypes.c_void_p),
        ("borders", ctypes.c_void_p),
        ("border_stride", ctypes.c_int32),
        ("split_feature", ctypes.c_void_p),
        ("split_ordinal", ctypes.c_void_p),
        ("leaves", ctypes.c_void_p),
        ("leaves_f16", ctypes.c_void_p),
        ("scale", ctypes.c_double),
        ("bias", ctypes.c_double),
        ("precision", ctypes.c_int32),
    ]


_lib = None


def library_path() -> Path:
    override = os.environ.get("OBTREE_B200_LIB")
    return Path(override) if override else LIB_PATH


def load_library() -> ctypes.CDLL:
    """Load the shared library and declare signatures (no GPU needed to load)."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(str(path))
    i32, i64, vp, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    p_i32 = ctypes.POINTER(ctypes.c_int32)
    sig = {
        "obt_model_create": (ctypes.c_int, [ctypes.POINTER(ModelDesc), ctypes.c_int, ctypes.POINTER(vp)]),
        "obt_model_destroy": (ctypes.c_int, [vp]),
        "obt_model_info": (ctypes.c_int, [vp, p_i32, p_i32, p_i32, p_i32, p_i32, p_i32, p_i32]),
        "obt_model_quantize_kernel": (ctypes.c_int, [vp, p_i32, p_i32]),
        "obt_model_multi_kernel": (ctypes.c_int, [vp, p_i32]),
        "obt_workspace_size": (ctypes.c_int, [vp, i64, ctypes.POINTER(sz)]),
        "obt_predict_dev": (ctypes.c_int, [vp, vp, i64, i32, vp, vp, sz, vp]),
        "obt_predict_host": (ctypes.c_int, [vp, vp, i64, i32, vp, vp]),
        "obt_predict_sharded": (ctypes.c_int, [ctypes.POINTER(vp), i32, i32, vp, i64, i32, ctypes.c_double,
                                               ctypes.c_double, vp]),
        "obt_quantize_dev": (ctypes.c_int, [vp, vp, i64, i32, vp, vp]),
        "obt_leaf_indices_dev": (ctypes.c_int, [vp, vp, i64, i32, i32, i32, vp, vp]),
        "obt_predict_dev_marked": (ctypes.c_int, [vp, vp, i64, i32, vp, vp, sz, vp, vp, vp, vp]),
        "obt_event_create": (ctypes.c_int, [ctypes.POINTER(vp)]),
        "obt_event_record": (ctypes.c_int, [vp, vp]),
        "obt_event_elapsed_ms": (ctypes.c_int, [vp, vp, ctypes.POINTER(ctypes.c_float)]),
        "obt_event_destroy": (ctypes.c_int, [vp]),
        "obt_last_launch_count": (ctypes.c_int, []),
        "obt_last_error": (ctypes.c_char_p, []),
        "obt_abi_version": (ctypes.c_int, []),
        "obt_set_path_option": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int]),
        "obt_get_path_option": (ctypes.c_int, [ctypes.c_char_p, p_i32]),
    }
    for name, (restype, argtypes) in sig.items():
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


def check(code: int) -> None:
    if code != OBT_OK:
        lib = load_library()
        msg = lib.obt_last_error().decode("utf-8", "replace")
        raise NativeError(code, msg)


def require_gpu() -> ctypes.CDLL:
    """The library, after confirming a CUDA device exists (fails loudly otherwise)."""
    lib = load_library()
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device is visible; the B200 kernels have no CPU fallback")
    return lib


def set_path_option(name: str, value: int) -> None:
    """Force one planner choice process-wide (see include/obtree_b200.h); -1 = automatic."""
    check(load_library().obt_set_path_option(name.encode(), int(value)))


def get_path_option(name: str) -> int:
    v = ctypes.c_int32()
    check(load_library().obt_get_path_option(name.encode(), ctypes.byref(v)))
    return int(v.value)


class path_options:
    """Context manager forcing planner choices for the duration of a block, then
    restoring the previous values: ``with path_options(wide=1, fan=0): ...``."""

    def __init__(self, **opts):
        self.opts = opts
        self.saved = {}

    def __enter__(self):
        for k, v in self.opts.items():
            self.saved[k] = get_path_option(k)
            set_path_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            set_path_option(k, v)
        return False


class Event:
    """A timing CUDA event owned by the library's runtime (works on torch streams)."""

    def __init__(self):
        self._lib = load_library()
        self.handle = ctypes.c_void_p()
        check(self._lib.obt_event_create(ctypes.byref(self.handle)))

    def record(self, stream: int) -> None:
        check(self._lib.obt_event_record(self.handle, stream))

    def elapsed_ms(self, end: "Event") -> float:
        ms = ctypes.c_float()
        check(self._lib.obt_event_elapsed_ms(self.handle, end.handle, ctypes.byref(ms)))
        return float(ms.value)

    def __del__(self):
        try:
            if self.handle.value:
                self._lib.obt_event_destroy(self.handle)
        except Exception:
            pass


def current_stream_handle(device=None) -> int:
    import torch

    return int(torch.cuda.current_stream(device).cuda_stream)
