"""ctypes binding of ``libspmoe.so`` (the C ABI in ``include/spmoe.h``).

The product path has no CPU fallback: if the library is missing or fails to
load, every compute entry point raises :class:`NativeUnavailable`.  The
library is built in-tree by :mod:`paper_2510_10302_b200.build`.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libspmoe.so"


class NativeUnavailable(RuntimeError):
    """The sm_100a library could not be loaded (no fallback exists)."""


class SpmoeError(RuntimeError):
    """A C-ABI entry point returned a non-zero status."""

    def __init__(self, fn: str, status: int, text: str):
        super().__init__(f"{fn} failed with status {status}: {text}")
        self.status = status


_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_f = C.c_float
_sz = C.c_size_t

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "spmoe_abi_version": (_i, []),
    "spmoe_status_string": (C.c_char_p, [_i]),
    "spmoe_router_topk": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p]),
    "spmoe_moe_permute": (_i, [_p, _i, _i, _i, _p, _p, _p, _p]),
    "spmoe_expert_ffn": (_i, [_p, _i64, _p, _u64, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _i, _p]),
    "spmoe_expert_ffn_up": (_i, [_p, _i64, _p, _u64, _p, _i, _i, _i, _i, _i, _p, _p, _p, _i, _p]),
    "spmoe_expert_ffn_down": (_i, [_p, _i64, _p, _u64, _i, _i, _i, _i, _i, _p, _p, _p, _i, _p]),
    "spmoe_expert_ffn_tc": (_i, [_p, _i64, _p, _u64, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _i, _i, _p]),
    "spmoe_expert_ffn_tc_fused": (_i, [_p, _i64, _p, _u64, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _i, _p, _p]),
    "spmoe_expert_ffn_tc_units": (_i, [_p, _i64, _p, _u64, _p, _i, _i, _i, _i, _i, _p, _p, _i, _p, _p, _p, _p, _p]),
    "spmoe_expert_ffn_tc_units_workspace_floats": (_i64, [_i, _i, _i]),
    "spmoe_k3_timing": (_i, [_p, _p]),
    "spmoe_moe_combine": (_i, [_p, _p, _p, _i, _i, _i, _p, _p, _p, _p, _p]),
    "spmoe_gather_rows": (_i, [_p, _p, _i, _i, _i64, _p, _p]),
    "spmoe_greedy_accept": (_i, [_p, _i64, _p, _i, _i, _i, _p, _p, _p]),
    "spmoe_argmax_rows": (_i, [_p, _i64, _i, _i, _p, _p]),
    "spmoe_h2d_batch": (_i, [_p, _p, _p, _i, _p]),
    "spmoe_rms_norm": (_i, [_p, _p, _i, _i, _f, _p, _p]),
    "spmoe_rope_kv": (_i, [_p, _p, _p, _p, _i, _i, _i, _i, _i, _i, _i, _p, _p, _p, _p]),
    "spmoe_linear": (_i, [_p, _p, _i64, _i, _i, _i, _p, _f, _p, _i64, _p, _p, _p]),
    "spmoe_attention": (_i, [_p, _p, _p, _p, _i, _i, _i, _i, _i, _i, _f, _p, _p]),
    "spmoe_fill_normal_bf16": (_i, [_p, _i64, _u64, _u64, _f, _p]),
    "spmoe_rt_create": (_p, [_i, _i, _i, _p, _p, _p, _sz, _p, _i]),
    "spmoe_rt_destroy": (None, [_p]),
    "spmoe_rt_lookup": (_i, [_p, _i, _i, _i]),
    "spmoe_rt_slot_of": (_i, [_p, _i, _i]),
    "spmoe_rt_insert_batch": (_i, [_p, _p, _p, _i, _i, _p]),
    "spmoe_rt_pin": (_i, [_p, _p, _p, _i]),
    "spmoe_rt_unpin": (None, [_p, _p, _p, _i]),
    "spmoe_rt_lru_order": (_i, [_p, _p, _p, _i]),
    "spmoe_rt_counters": (None, [_p, _p]),
    "spmoe_rt_reset_stats": (None, [_p]),
    "spmoe_rt_demand_load": (_i, [_p, _p, _p, _i, _p]),
    "spmoe_rt_wait_slot": (_i, [_p, _i, _p]),
    "spmoe_rt_mark_read": (_i, [_p, _i, _p]),
    "spmoe_rt_slot_ready": (_i, [_p, _i]),
    "spmoe_rt_worker_start": (_i, [_p]),
    "spmoe_rt_push_task": (_i, [_p, _i, _p, _i, _p, _i]),
    "spmoe_rt_push_task_flag": (_i, [_p, _i, _p, _i, _p, _i, _i]),
    "spmoe_signal_bump": (_i, [_p, _p]),
    "spmoe_rt_drain": (_i, [_p]),
    "spmoe_k3_devtiming": (_i, [_p]),
    "spmoe_xc_decode_segments_timed": (_i, [_p, _p, _i, _i, _p, _p, _p]),
    "spmoe_rt_debug_fail_copies": (_i, [_p, _i]),
    "spmoe_rt_abort_pending": (_i, [_p]),
    "spmoe_rt_worker_stop": (_i, [_p]),
    "spmoe_rt_transfer_log": (_i, [_p, _p, _p, _i]),
    "spmoe_rt_transfer_experts": (_i, [_p, _i, _p, _i]),
    "spmoe_rt_clear_log": (None, [_p]),
    "spmoe_rt_transfer_wire_bytes": (_i64, [_p, _i]),
    "spmoe_rt_transfer_copy_end_ms": (C.c_double, [_p, _i]),
    "spmoe_rt_set_codec": (_i, [_p, _sz, _p, _sz, _i, _p]),
    "spmoe_rt_wire_bytes": (None, [_p, _p]),
    "spmoe_rt_decode_timing": (_i, [_p, _i]),
    "spmoe_rt_decode_stats": (_i, [_p, _p, _p, _p]),
    "spmoe_xc_work_bytes": (_sz, [_i, _p]),
    "spmoe_xc_plan": (_i, [_p, _i, _p, _p, _p, _p]),
    "spmoe_xc_encode": (_i, [_p, _p, _p, _p, _p]),
    "spmoe_xc_decode": (_i, [_p, _p, _p, _p]),
    "spmoe_xc_decode_segments": (_i, [_p, _p, _i, _i, _p, _p]),
    "spmoe_rt_since_epoch_ms": (C.c_double, [_p, _p]),
    "spmoe_host_alloc_mapped": (_i, [_sz, _p, _p]),
    "spmoe_host_free": (_i, [_p]),
    "spmoe_host_register": (_i, [_p, _sz]),
    "spmoe_host_unregister": (_i, [_p]),
    "spmoe_event_create": (_i, [_p]),
    "spmoe_event_destroy": (_i, [_p]),
    "spmoe_event_record_external": (_i, [_p, _p]),
    "spmoe_event_synchronize": (_i, [_p]),
}

_lib = None
_lock = threading.Lock()


def load(build_if_missing: bool = False) -> C.CDLL:
    """Load (once) and return the library with all signatures bound."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            if build_if_missing:
                from .build import build

                build()
            else:
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing; run `python -m paper_2510_10302_b200.build` "
                    "(there is no CPU fallback)"
                )
        try:
            lib = C.CDLL(str(LIB_PATH))
        except OSError as exc:  # pragma: no cover - depends on the box
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(fn: str, status: int) -> None:
    if status != 0:
        lib = load()
        raise SpmoeError(fn, status, lib.spmoe_status_string(status).decode())


def call(fn: str, *args) -> int:
    """Call a status-returning entry point and raise on failure."""
    lib = load()
    st = getattr(lib, fn)(*args)
    check(fn, st)
    return st
