"""ctypes declarations for librx.so (include/rx.h).  Argument marshalling only.

Loading fails loudly (ImportError) if the in-tree library is missing: there is
no fallback path of any kind.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librx.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python paper_2312_07104_b200/build.py` "
                      "(or __graft_entry__.build()); there is no CPU fallback")

# RX_LIB_OVERRIDE: load a sanitizer build of the HOST half instead (scripts/asan_host.sh);
# device entry points are then absent and only the tree/router tests may run.
_override = os.environ.get("RX_LIB_OVERRIDE")
lib = C.CDLL(_override if _override else LIB_PATH)

i32, i64, f32, vp, sz = C.c_int32, C.c_int64, C.c_float, C.c_void_p, C.c_size_t
P32 = C.POINTER(C.c_int32)
P64 = C.POINTER(C.c_int64)


class AttnCfg(C.Structure):
    _fields_ = [("h_q", i32), ("h_kv", i32), ("head_dim", i32), ("sm_scale", f32)]


class TpOut(C.Structure):
    _fields_ = [("d_o", vp * 8), ("world", i32), ("h_q_total", i32), ("head_offset", i32)]


EVICT_CB = C.CFUNCTYPE(None, vp, P32, i64)
EVICT_PATH_CB = C.CFUNCTYPE(None, vp, P32, i64, i64, P32, i64)
STEP_EVENT_CB = C.CFUNCTYPE(None, vp, i32, P64, P32, i64)

# symbol -> (restype, argtypes); the set of names is exactly include/rx.h's declarations
SIGNATURES = {
    "rx_status_str": (C.c_char_p, [C.c_int]),
    "rx_version": (C.c_char_p, []),
    "rx_cache_create": (C.c_int, [i64, C.POINTER(vp)]),
    "rx_cache_destroy": (None, [vp]),
    "rx_match_prefix": (C.c_int, [vp, P32, i64, P64, P64, P32]),
    "rx_insert": (C.c_int, [vp, P32, P32, i64, P64, P64]),
    "rx_inc_ref": (C.c_int, [vp, i64, P64]),
    "rx_dec_ref": (C.c_int, [vp, i64, P64]),
    "rx_evict": (C.c_int, [vp, i64, P64, EVICT_CB, vp]),
    "rx_alloc": (C.c_int, [vp, i64, P32]),
    "rx_free": (C.c_int, [vp, P32, i64]),
    "rx_alloc_evict": (C.c_int, [vp, i64, P32, P64, EVICT_CB, vp]),
    "rx_evict_paths": (C.c_int, [vp, i64, P64, EVICT_PATH_CB, vp]),
    "rx_router_create": (C.c_int, [i32, C.POINTER(vp)]),
    "rx_router_destroy": (None, [vp]),
    "rx_router_affinity": (C.c_int, [vp, P32, i64, P64]),
    "rx_router_dispatch": (C.c_int, [vp, i32, P32, P64, P64, C.c_double, P32, P64]),
    "rx_router_insert": (C.c_int, [vp, i32, P32, i64]),
    "rx_router_queue_evict": (C.c_int, [vp, i32, P32, i64, i64]),
    "rx_router_sync": (i64, [vp]),
    "rx_router_queue_len": (i64, [vp]),
    "rx_router_dump_json": (i64, [vp, C.c_char_p, i64]),
    "rx_match_prefix_batch": (C.c_int, [vp, i32, P32, P64, P64, P64, P32]),
    "rx_inc_ref_batch": (C.c_int, [vp, i32, P64, P64]),
    "rx_finish_batch": (C.c_int, [vp, i32, P64, P32, P64, P32, P64, P64, P64]),
    "rx_schedule": (C.c_int, [vp, i32, P32, P64, P64, i32, C.POINTER(C.c_uint64), P64, P64, P32, P32,
                              C.POINTER(i32), P64]),
    "rx_decode_steps": (C.c_int, [vp, i32, P32, i64, P32, P32, P32, P64, P32, P64, P32, C.POINTER(i32), i32,
                                  P32, i64, P64, C.POINTER(i32), STEP_EVENT_CB, vp]),
    "rx_fsm_create": (C.c_int, [C.c_char_p, i64, C.POINTER(vp)]),
    "rx_fsm_destroy": (None, [vp]),
    "rx_fsm_num_states": (i32, [vp]),
    "rx_fsm_step": (i32, [vp, i32, i32]),
    "rx_fsm_is_accepting": (i32, [vp, i32]),
    "rx_fsm_allowed": (i32, [vp, i32, C.POINTER(C.c_uint8)]),
    "rx_fsm_jump": (i32, [vp, i32, C.POINTER(C.c_uint8), i32, C.POINTER(i32)]),
    "rx_evictable_size": (i64, [vp]),
    "rx_total_cached": (i64, [vp]),
    "rx_available": (i64, [vp]),
    "rx_num_slots": (i64, [vp]),
    "rx_clock": (i64, [vp]),
    "rx_dump_json": (i64, [vp, C.c_char_p, i64]),
    "rx_store_kv": (C.c_int, [C.POINTER(AttnCfg), i64, vp, vp, vp, vp, vp, i64, vp, vp, vp]),
    "rx_extend": (C.c_int, [C.POINTER(AttnCfg), i32, vp, i64, vp, vp, vp, vp, i64, i32, i32,
                            vp, vp, vp, vp, vp, i64, vp, vp, sz, vp]),
    "rx_extend_workspace_bytes": (sz, [C.POINTER(AttnCfg), i32, i32]),
    "rx_extend_cascade": (C.c_int, [C.POINTER(AttnCfg), i32, vp, i64, vp, vp, vp, vp, i64, i32, i32, i32,
                                    vp, vp, vp, vp, vp, i64, vp, vp, sz, vp]),
    "rx_extend_cascade_workspace_bytes": (sz, [C.POINTER(AttnCfg), i64, i32]),
    "rx_decode": (C.c_int, [C.POINTER(AttnCfg), i32, vp, i64, vp, vp, i32, vp, vp, vp, i64, vp, vp, sz, vp]),
    "rx_decode_append": (C.c_int, [C.POINTER(AttnCfg), i32, vp, i64, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, i64,
                                   vp, vp, sz, vp]),
    "rx_decode_workspace_bytes": (sz, [C.POINTER(AttnCfg), i32, i32]),
    "rx_decode_cascade_append": (C.c_int, [C.POINTER(AttnCfg), i32, vp, i64, vp, vp, vp, i32, i32, vp, vp, vp, vp,
                                           vp, vp, i64, vp, vp, sz, vp]),
    "rx_decode_cascade_workspace_bytes": (sz, [C.POINTER(AttnCfg), i32, i32, i32]),
    "rx_decode_run": (C.c_int, [C.POINTER(AttnCfg), i32, P32, P32, i32, vp, i64, vp, P64, i32, C.POINTER(vp),
                                C.POINTER(vp), C.POINTER(vp), vp, vp, i64, C.POINTER(vp), i32, i32, i32, vp, sz, vp]),
    "rx_decode_append_tp": (C.c_int, [C.POINTER(AttnCfg), i32, vp, i64, vp, vp, vp, i32, i32, vp, vp, vp, vp,
                                      vp, vp, i64, C.POINTER(TpOut), vp, sz, vp]),
    "rx_last_launch_count": (i32, []),
    "rx_copy_h2d": (C.c_int, [vp, vp, i64, vp]),
    "rx_tp_buffer_bytes": (sz, [i32, i64]),
    "rx_tp_ipc_handle": (C.c_int, [vp, vp]),
    "rx_tp_ipc_offset": (i64, [vp]),
    "rx_tp_ipc_open": (C.c_int, [vp, C.POINTER(vp)]),
    "rx_tp_ipc_close": (C.c_int, [vp]),
    "rx_tp_allgather": (C.c_int, [vp, i64, C.POINTER(vp), i32, i32, i64, i64, vp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    if _override and not hasattr(lib, _name):
        continue
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

STATUS = {0: "RX_OK", -1: "RX_E_INVALID", -2: "RX_E_NOMEM", -3: "RX_E_UNDERFLOW", -4: "RX_E_STALE",
          -5: "RX_E_UNSUPPORTED", -6: "RX_E_CUDA", -7: "RX_E_WORKSPACE", -8: "RX_E_CAPACITY"}


class RxError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {STATUS.get(status, status)}")
        self.status = status
