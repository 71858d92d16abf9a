"""Counter-based bf16 value generator for q / k / v.

value(h, head, kind, d):
    base = splitmix64(h XOR splitmix64(4*head + kind + 1))
    r    = splitmix64(base + d * GOLDEN)                 (wrapping)
    S    = sum of the four 16-bit fields of r            (integer in [0, 262140])
    x    = float32(S - 131070) * float32(sqrt(3) / 65536) * scale
    out  = bf16(x)  (round to nearest even)

S is an Irwin-Hall(4) draw on a 2^-16 grid: mean 0, variance 1 after scaling,
bell-shaped, |x| <= 3.46.  Every step is integer arithmetic except one fp32
multiply of two exactly representable numbers (correctly rounded under IEEE
754 on any device) and the RNE cast, so CPU and GPU produce identical bits.
(SURVEY.md §8(c) suggested Box-Muller; DESIGN.md "Readings" records why this
generator replaces it: transcendental functions are not bit-reproducible
across devices.)  ``scale`` must be a power of two so the scaling is exact.

kind: 0 = K, 1 = V, 2 = Q.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from .hashing import GOLDEN, _s64, splitmix64_np, splitmix64_t, splitmix64_int, MASK64

KIND_K, KIND_V, KIND_Q = 0, 1, 2
_C = np.float32(math.sqrt(3.0) / 65536.0)


def _head_salt(head: int, kind: int) -> int:
    return splitmix64_int(4 * head + kind + 1)


def gen_values(hashes, heads, kind: int, hd: int, scale: float = 1.0,
               device=None, chunk: int = 8192) -> torch.Tensor:
    """hashes: uint64 numpy array or int64 torch tensor [N]; returns bf16 [N, len(heads), hd]."""
    assert scale > 0 and math.log2(scale) == int(math.log2(scale)), "scale must be a power of 2"
    if isinstance(hashes, np.ndarray):
        hashes = torch.from_numpy(hashes.astype(np.uint64).view(np.int64))
    if device is not None:
        hashes = hashes.to(device)
    dev = hashes.device
    n = hashes.shape[0]
    heads = list(heads)
    out = torch.empty((n, len(heads), hd), dtype=torch.bfloat16, device=dev)
    salts = torch.tensor([_s64(_head_salt(h, kind)) for h in heads], dtype=torch.int64, device=dev)
    dstep = torch.arange(hd, dtype=torch.int64, device=dev) * _s64(GOLDEN)
    c = torch.tensor(float(_C), dtype=torch.float32, device=dev)
    sc = torch.tensor(scale, dtype=torch.float32, device=dev)
    for s in range(0, n, chunk):
        h = hashes[s:s + chunk]
        base = splitmix64_t(h[:, None] ^ salts[None, :])                 # [n, H]
        r = splitmix64_t(base[:, :, None] + dstep[None, None, :])       # [n, H, hd]
        tot = (r & 0xFFFF) + ((r >> 16) & 0xFFFF) + ((r >> 32) & 0xFFFF) + ((r >> 48) & 0xFFFF)
        x = (tot - 131070).to(torch.float32) * c
        if scale != 1.0:
            x = x * sc
        out[s:s + chunk] = x.to(torch.bfloat16)
    return out


def _bf16_rne_np(x: np.ndarray) -> np.ndarray:
    """float32 -> float32 holding the bf16 round-to-nearest-even value (finite inputs)."""
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = (u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32)


def gen_values_np(hashes: np.ndarray, heads, kind: int, hd: int, scale: float = 1.0) -> np.ndarray:
    """Independent numpy form of gen_values (float32 holding bf16 values)."""
    hashes = np.asarray(hashes, dtype=np.uint64)
    heads = list(heads)
    salts = np.array([_head_salt(h, kind) for h in heads], dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = splitmix64_np(hashes[:, None] ^ salts[None, :])
        r = splitmix64_np(base[:, :, None] + np.arange(hd, dtype=np.uint64)[None, None, :] * np.uint64(GOLDEN))
    m = np.uint64(0xFFFF)
    tot = (r & m) + ((r >> np.uint64(16)) & m) + ((r >> np.uint64(32)) & m) + ((r >> np.uint64(48)) & m)
    x = (tot.astype(np.int64) - 131070).astype(np.float32) * _C
    x = (x * np.float32(scale)).astype(np.float32)
    return _bf16_rne_np(x)
