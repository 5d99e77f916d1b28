"""ctypes binding of libpreft.so (the C ABI declared in include/preft.h).

The library is built in-tree by `_build.build_library()` (or
`__graft_entry__.build()`).  There is no CPU fallback anywhere in this
package: every compute entry point goes through this binding and raises if
the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import DeviceError, status_to_error

LIB_PATH = Path(__file__).resolve().parent / "libpreft.so"

DTYPE_F32 = 0
DTYPE_BF16 = 1
DTYPE_F64 = 2

ENTRY_DECODE = 1
ENTRY_ALL_POSITIONS = 2

META_ERR_E_RANGE = 1
META_ERR_T_RANGE = 2
META_ERR_QSL = 4
META_ERR_TILES = 8
META_ERR_UNITS = 16

CTR_SEL_TOKENS = 0
CTR_SEGMENTS = 1
CTR_TILES = 2
CTR_ERR = 3
CTR_SEL_ENTRIES = 4
CTR_T = 5
CTR_E = 6
CTR_SPLIT = 7
CTR_CHUNKS = 8
CTR_UNITS = 9
CTR_LORA_UNITS = 10
CTR_LORA_CHUNKS = 11
NUM_COUNTERS = 12
CHUNK_ROWS = 16
UNIT_CHUNKS = 4
META_UNIT_ORDER = 1
SLOT_SPLIT_ALL_LORA = 2**31 - 1  # every slot is a LoRA-class slot
MAX_ENTRIES = 4096

ABI_VERSION = 2


class PreftMeta(ctypes.Structure):
    _fields_ = [
        ("entries", ctypes.c_void_p),
        ("mask", ctypes.c_void_p),
        ("tokens", ctypes.c_void_p),
        ("segments", ctypes.c_void_p),
        ("tiles", ctypes.c_void_p),
        ("entry_offset", ctypes.c_void_p),
        ("counters", ctypes.c_void_p),
        ("E_cap", ctypes.c_int32),
        ("T_cap", ctypes.c_int32),
        ("tile_cap", ctypes.c_int32),
        ("tile_tokens", ctypes.c_int32),
        ("slot_split", ctypes.c_int32),
        ("rows_hint", ctypes.c_int32),
        ("chunks", ctypes.c_void_p),
        ("units", ctypes.c_void_p),
        ("chunk_cap", ctypes.c_int32),
        ("meta_flags", ctypes.c_int32),
        ("lora_part", ctypes.c_void_p),
        ("lora_part_floats", ctypes.c_int64),
    ]


XCHG_MAX_TP = 8


class PreftXchg(ctypes.Structure):
    """preft_xchg_t: one rank's view of the fused kernel's exchange regions."""

    _fields_ = [
        ("tp_size", ctypes.c_int32),
        ("tp_rank", ctypes.c_int32),
        ("planes", ctypes.c_int32),
        ("T_cap", ctypes.c_int32),
        ("U_cap", ctypes.c_int32),
        ("peer_sys", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("part", ctypes.c_void_p * XCHG_MAX_TP),
        ("flag", ctypes.c_void_p * XCHG_MAX_TP),
        ("state", ctypes.c_void_p),
        ("spin_ns", ctypes.c_int64),
    ]


class PreftLoraSite(ctypes.Structure):
    _fields_ = [
        ("A", ctypes.c_void_p),
        ("Bt", ctypes.c_void_p),
        ("scale", ctypes.c_void_p),
        ("bias", ctypes.c_void_p),
        ("y", ctypes.c_void_p),
        ("ldy", ctypes.c_int64),
        ("n", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("Bt_tc", ctypes.c_void_p),
    ]


# name -> (restype, argtypes); the exported surface of include/preft.h
SIGNATURES = {
    "preft_meta_entries_words": (ctypes.c_size_t, [ctypes.c_int32]),
    "preft_meta_build": (ctypes.c_int, [ctypes.POINTER(PreftMeta), ctypes.c_void_p]),
    "preft_lora_apply": (
        ctypes.c_int,
        [
            ctypes.POINTER(PreftMeta),
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_int32,
            ctypes.POINTER(PreftLoraSite),
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_void_p,
        ],
    ),
    "preft_reft_apply": (
        ctypes.c_int,
        [
            ctypes.POINTER(PreftMeta),
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.c_int32,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_void_p,
        ],
    ),
    "preft_set_reft_variant": (ctypes.c_int, [ctypes.c_int32]),
    "preft_set_reft_tc_flags": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32]),
    "preft_lora_shrink": (
        ctypes.c_int,
        [
            ctypes.POINTER(PreftMeta),
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.c_int32,
            ctypes.POINTER(PreftLoraSite),
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_void_p,
        ],
    ),
    "preft_lora_expand": (
        ctypes.c_int,
        [
            ctypes.POINTER(PreftMeta),
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.POINTER(PreftLoraSite),
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_void_p,
        ],
    ),
    "preft_xchg_region_bytes": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "preft_xchg_init": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_int32, ctypes.c_int32, ctypes.c_int32],
    ),
    "preft_lora_fused": (
        ctypes.c_int,
        [
            ctypes.POINTER(PreftMeta),
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.c_int32,
            ctypes.POINTER(PreftLoraSite),
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_void_p,
            ctypes.c_void_p,
        ],
    ),
    "preft_xchg_errors": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32)]),
    "preft_dev_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "preft_dev_free": (ctypes.c_int, [ctypes.c_void_p]),
    "preft_ipc_handle": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "preft_ipc_open": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "preft_ipc_close": (ctypes.c_int, [ctypes.c_void_p]),
    "preft_set_split_variant": (ctypes.c_int, [ctypes.c_int32]),
    "preft_diag_split": (ctypes.c_int, [ctypes.c_void_p]),
    "preft_lora_part_floats": (ctypes.c_int64, [ctypes.POINTER(PreftMeta)]),
    "preft_diag_reft_tc": (ctypes.c_int, [ctypes.c_void_p]),
    "preft_convert_2d": (
        ctypes.c_int,
        [
            ctypes.c_void_p,
            ctypes.c_int32,
            ctypes.c_int64,
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.c_void_p,
        ],
    ),
    "preft_plan_create": (ctypes.c_void_p, [ctypes.POINTER(PreftMeta)]),
    "preft_plan_destroy": (None, [ctypes.c_void_p]),
    "preft_plan_set_slot_split": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "preft_plan_set_rows_hint": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "preft_plan_refresh_meta": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PreftMeta)]),
    "preft_plan_add_lora": (
        ctypes.c_int,
        [
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_int32,
            ctypes.POINTER(PreftLoraSite),
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_int32,
        ],
    ),
    "preft_plan_add_reft": (
        ctypes.c_int,
        [
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_int64,
            ctypes.c_int32,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_int32,
            ctypes.c_int32,
            ctypes.c_int32,
        ],
    ),
    "preft_plan_num_ops": (ctypes.c_int, [ctypes.c_void_p]),
    "preft_plan_set_timing": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]),
    "preft_plan_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "preft_plan_collect_timing": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)],
    ),
    "preft_set_lora_variant": (ctypes.c_int, [ctypes.c_int32]),
    "preft_tc_selftest": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_void_p],
    ),
    "preft_abi_version": (ctypes.c_int, []),
    "preft_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "preft_last_cuda_error": (ctypes.c_char_p, []),
    "preft_num_sms": (ctypes.c_int, []),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load libpreft.so once (raises if it was never built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise DeviceError(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.preft_abi_version() != ABI_VERSION:
            raise DeviceError("libpreft ABI version mismatch; rebuild the library")
        _lib = lib
        return lib


def check(status: int, what: str) -> None:
    if status == 0:
        return
    err = status_to_error(status, what)
    if status == 16:
        detail = load().preft_last_cuda_error()
        err = type(err)(f"{err} ({detail.decode() if detail else 'no detail'})")
    raise err


def require_cuda(device=None):
    """Return a torch.device for the CUDA extension or raise (no CPU fallback)."""
    import torch

    load()
    if not torch.cuda.is_available():
        raise DeviceError("libpreft needs a CUDA device (sm_100a); no CPU fallback exists")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise DeviceError(f"libpreft runs on CUDA devices only, got {dev}")
    return dev
