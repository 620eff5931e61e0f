"""ctypes binding of libpearl_b200.so (declared in include/pearl_b200.h).

There is no fallback: if the shared library is missing, or no CUDA device is
present, every product entry point raises.  (The CPU oracle under oracle/ is
test infrastructure and is never imported from here.)
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import AllZeroResidual, DeviceError, InvalidDistribution, ZeroDraftProb

PEARL_OK = 0
PEARL_ERR_INVALID_DISTRIBUTION = 1
PEARL_ERR_ALL_ZERO_RESIDUAL = 2
PEARL_ERR_ZERO_DRAFT_PROB = 3
PEARL_ERR_VALUE = 4
PEARL_ERR_TIMEOUT = 5

ROWS_PROBS64 = 0
ROWS_LOGITS32 = 1

F_GREEDY = 1
F_BONUS = 2
F_ADVANCE = 4
F_PROBE = 8

# PEARL_LIB_PATH: a diagnostic build of the same library (e.g. -DPEARL_TRACE_PICK)
LIB_PATH = os.environ.get("PEARL_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                            "libpearl_b200.so")

_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_f32 = ctypes.c_float
_sz = ctypes.c_size_t


class VerifyResultC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("status", "accepted", "correction", "examined", "draws_used", "bonus", "fallback",
                 "reserved")]


# (name, restype, argtypes) for every symbol include/pearl_b200.h declares.
SIGNATURES = {
    "pearl_version": (_i32, []),
    "pearl_last_error": (ctypes.c_char_p, []),
    "pearl_launch_count": (ctypes.c_ulonglong, []),
    "pearl_verify_work_bytes": (_sz, [_i32]),
    "pearl_prepare_vocab": (_i32, [_i32]),
    "pearl_spec_verify": (_i32, [_i32, _vp, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _f32, _i32, _vp, _vp,
                                 _vp, _vp]),
    "pearl_sample_rows": (_i32, [_i32, _vp, _i32, _i32, _vp, _i32, _vp, _f32, _i32, _vp, _vp, _vp, _vp,
                                 _vp]),
    "pearl_spec_verify_multi": (_i32, [_i32, _vp, _i32, _i32, _i32, _i32, _f32, _i32, _vp]),
    "pearl_sample_rows_multi": (_i32, [_i32, _vp, _i32, _i32, _vp, _i32, _vp, _f32, _i32, _vp, _vp, _vp]),
    "pearl_logits_to_probs": (_i32, [_vp, _i32, _i32, _f32, _vp, _vp, _vp]),
    "pearl_residual": (_i32, [_vp, _vp, _i32, _vp, _vp, _vp]),
    # model runtime (csrc/llama.cu)
    "pearl_llama_create": (_i32, [_vp, _vp, _i32, _vp]),
    "pearl_llama_destroy": (_i32, [_vp]),
    "pearl_llama_forward": (_i32, [_vp, _vp, _i32, _vp, _i32, _vp, _vp]),
    "pearl_llama_workspace_bytes": (_sz, [_vp, _i32]),
    "pearl_llama_forward_slots": (_i32, [_vp, _vp, _i32, _vp, _vp, _vp, _vp]),
    "pearl_llama_profile": (_i32, [_vp, _vp, _i32, _vp, _vp, _vp, _vp]),
    "pearl_llama_set_l2_window": (_i32, [_vp, _vp, ctypes.c_size_t, _vp]),
    "pearl_green_streams": (_i32, [_i32, _vp, _vp, _vp, _vp]),
    "pearl_llama_debug_buffer": (_i32, [_vp, _i32, _vp, ctypes.c_size_t, _vp]),
    "pearl_gemm": (_i32, [_i32, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "pearl_gemm_splits": (_i32, [_i32, _i32]),
    "pearl_kv_rollback": (_i32, [_vp, _vp, _i32, _vp]),
    "pearl_pearl_commit": (_i32, [_vp, _vp]),
    "pearl_step_assemble": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    # K6 split-pair exchange (csrc/exchange.cu)
    "pearl_mailbox_bytes": (_sz, [_i32, _i32]),
    "pearl_mailbox_alloc": (_i32, [_sz, _vp]),
    "pearl_mailbox_free": (_i32, [_vp]),
    "pearl_ipc_export": (_i32, [_vp, _vp]),
    "pearl_ipc_import": (_i32, [_vp, _vp]),
    "pearl_ipc_close": (_i32, [_vp]),
    "pearl_xfer_send": (_i32, [_vp, _vp]),
    "pearl_xfer_send_copy": (_i32, [_vp, _vp, _vp]),
    "pearl_peer_storable": (_i32, [ctypes.c_char_p]),
    "pearl_pci_bus_id": (_i32, [ctypes.c_char_p, _i32]),
    "pearl_xfer_wait": (_i32, [_vp, _vp, _vp, _i32, _vp, ctypes.c_longlong, _vp]),
}

MAILBOX_IDS_OFFSET = 256
MAILBOX_MAX_IDS = 1024
MAILBOX_ROWS_OFFSET = 256 + 4 * 1024
IPC_HANDLE_BYTES = 64

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load the extension (once).  Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2408_11850_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(code: int, what: str = "") -> None:
    """Map a C-ABI status code onto the reference's exception classes."""
    if code == PEARL_OK:
        return
    if code == PEARL_ERR_INVALID_DISTRIBUTION:
        raise InvalidDistribution(f"{what}: invalid distribution")
    if code == PEARL_ERR_ALL_ZERO_RESIDUAL:
        raise AllZeroResidual("target and draft distributions are identical")
    if code == PEARL_ERR_ZERO_DRAFT_PROB:
        raise ZeroDraftProb(f"{what}: drafted token has zero draft probability")
    if code == PEARL_ERR_VALUE:
        raise ValueError(f"{what}: invalid value")
    if code == PEARL_ERR_TIMEOUT:
        raise DeviceError(f"{what}: split-pair peer did not deliver before the exchange timeout")
    msg = load().pearl_last_error()
    raise DeviceError(f"{what}: libpearl_b200 error {code}: {msg.decode() if msg else ''}")


_prepared = set()


def prepare_vocab(V: int) -> None:
    if V in _prepared:
        return
    check(load().pearl_prepare_vocab(int(V)), "pearl_prepare_vocab")
    _prepared.add(V)
