"""B200-native RadixAttention hot path (arXiv 2312.07104).

librx.so (C ABI, include/rx.h): host radix tree over a token-slot KV pool +
sm_100a kernels for KV store, extend (tcgen05/TMEM) and decode (split-KV,
GQA-grouped).  This package is the thin Python binding plus the request-flow
harness that drives it.  It never imports ``oracle/``.
"""
from .api import (RadixCache, Fsm, attn_cfg, rx_store_kv, rx_extend, rx_decode, rx_decode_append, rx_decode_cascade_append,
                  rx_decode_cascade_workspace_bytes, rx_extend_workspace_bytes, rx_extend_cascade,
                  rx_extend_cascade_workspace_bytes,
                  rx_decode_workspace_bytes, rx_last_launch_count, rx_copy_h2d, rx_decode_run,
                  rx_decode_append_tp, tp_out)
from ._lib import RxError, LIB_PATH

__all__ = ["RadixCache", "Fsm", "attn_cfg", "rx_store_kv", "rx_extend", "rx_decode", "rx_decode_append", "rx_decode_cascade_append",
           "rx_decode_cascade_workspace_bytes", "rx_extend_workspace_bytes", "rx_extend_cascade",
           "rx_extend_cascade_workspace_bytes",
           "rx_decode_workspace_bytes", "rx_last_launch_count", "rx_copy_h2d", "rx_decode_run",
           "rx_decode_append_tp", "tp_out", "RxError", "LIB_PATH"]
