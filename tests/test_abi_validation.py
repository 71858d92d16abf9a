"""Argument validation of the device entry points (include/rx.h), on the CPU: every call below
fails its host-side checks before any CUDA call, so no GPU is needed.  Status codes as the header
documents them."""
import ctypes as C

from paper_2312_07104_b200._lib import lib, AttnCfg

INVALID, UNSUPPORTED, WORKSPACE = -1, -5, -7


def cfg(h_q=32, h_kv=8, hd=128):
    return AttnCfg(h_q, h_kv, hd, 0.088)


def test_unsupported_shapes():
    for c in (cfg(hd=96), cfg(h_q=30, h_kv=8), cfg(h_q=48, h_kv=3)):
        assert lib.rx_extend(C.byref(c), 1, None, 8, None, None, None, None, 1, 1, 0, None, None, None, None, None,
                             16, None, None, 0, None) == UNSUPPORTED
        assert lib.rx_decode(C.byref(c), 1, None, 8, None, None, 1, None, None, None, 16, None, None, 0,
                             None) == UNSUPPORTED
    assert lib.rx_extend(None, 1, None, 8, None, None, None, None, 1, 1, 0, None, None, None, None, None, 16, None,
                         None, 0, None) == INVALID


def test_empty_calls_are_ok_and_null_buffers_invalid():
    c = cfg()
    # empty batch / no new rows: nothing to do
    assert lib.rx_extend(C.byref(c), 0, None, 8, None, None, None, None, 0, 0, 0, None, None, None, None, None, 16,
                         None, None, 0, None) == 0
    assert lib.rx_decode(C.byref(c), 0, None, 8, None, None, 0, None, None, None, 16, None, None, 0, None) == 0
    # work requested but null device buffers
    assert lib.rx_extend(C.byref(c), 2, None, 8, None, None, None, None, 5, 3, 2, None, None, None, None, None, 16,
                         None, None, 0, None) == INVALID
    assert lib.rx_decode(C.byref(c), 2, None, 8, None, None, 4, None, None, None, 16, None, None, 0, None) == INVALID
    assert lib.rx_decode_append(C.byref(c), 2, None, 8, None, None, None, 4, None, None, None, None, None, None, 16,
                                None, None, 0, None) == INVALID
    assert lib.rx_extend_cascade(C.byref(c), 2, None, 8, None, None, None, None, 5, 3, 2, -1, None, None, None, None,
                                 None, 16, None, None, 0, None) == INVALID


def test_workspace_queries():
    c = cfg()
    assert lib.rx_extend_workspace_bytes(C.byref(c), 4, 100) == 256      # the work-counter header (rx.h)
    assert lib.rx_extend_workspace_bytes(C.byref(c), 0, 100) == 0
    small = lib.rx_decode_workspace_bytes(C.byref(c), 256, 512)
    big = lib.rx_decode_workspace_bytes(C.byref(c), 4, 65536)
    assert small == 0 and big > 0                       # one split needs no workspace; splits do
    assert lib.rx_decode_cascade_workspace_bytes(C.byref(c), 128, 8320, 8192) > 0
    assert lib.rx_extend_cascade_workspace_bytes(C.byref(c), 4096, 1024) > 0
    assert lib.rx_extend_cascade_workspace_bytes(C.byref(c), 4096, 0) == 0
    assert lib.rx_decode_workspace_bytes(C.byref(cfg(hd=96)), 4, 100) == 0
