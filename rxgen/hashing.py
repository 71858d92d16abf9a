"""splitmix64 in three interchangeable forms (python int, numpy uint64, torch int64).

splitmix64(x) = mix(x + 0x9E3779B97F4A7C15) with the standard Stafford-13
finaliser; splitmix64(0) == 0xE220A8397B1DCDAF (the published first output of
the splitmix64 stream seeded with 0; pinned in tests/test_rxgen.py).

The torch form runs on CPU or CUDA with wrapping int64 arithmetic; logical
right shifts are emulated with a mask.  All three forms must agree bit for bit
(tests/test_rxgen.py).
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
# salt for the mock model's "next token" draw
NEXT_SALT = 0x6A09E667F3BCC909


def _s64(u: int) -> int:
    """uint64 -> the int64 with the same bits."""
    u &= MASK64
    return u - (1 << 64) if u >= (1 << 63) else u


def splitmix64_int(x: int) -> int:
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * _M1) & MASK64
    z = ((z ^ (z >> 27)) * _M2) & MASK64
    return z ^ (z >> 31)


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        return z ^ (z >> np.uint64(31))


def _srl(t, s: int):
    """Logical right shift of an int64 tensor."""
    return (t >> s) & ((1 << (64 - s)) - 1)


def splitmix64_t(x):
    """torch int64 tensor -> torch int64 tensor (same bits as the uint64 form)."""
    z = x + _s64(GOLDEN)
    z = (z ^ _srl(z, 30)) * _s64(_M1)
    z = (z ^ _srl(z, 27)) * _s64(_M2)
    return z ^ _srl(z, 31)


def prefix_hashes(tokens, seed: int) -> np.ndarray:
    """h_p = splitmix64(h_{p-1} XOR tok_p), h_{-1} = seed; returns uint64[n]."""
    toks = np.asarray(tokens, dtype=np.uint64)
    out = np.empty(len(toks), dtype=np.uint64)
    h = seed & MASK64
    for i, t in enumerate(toks.tolist()):
        h = splitmix64_int(h ^ t)
        out[i] = h
    return out


def extend_hashes(h_prev: int, tokens) -> np.ndarray:
    """Continue a prefix-hash chain from h_prev over more tokens."""
    return prefix_hashes(tokens, h_prev)


def next_token(h: int, vocab: int) -> int:
    """Mock model: the token generated after a prefix whose hash is h."""
    return 1 + splitmix64_int((h ^ NEXT_SALT) & MASK64) % (vocab - 1)


def sched_keys(seed: int, wave: int, n: int) -> np.ndarray:
    """Random-schedule priority keys (the P:432 "Random Schedule" ablation): key i of a wave is
    splitmix64(seed ^ (wave << 32) ^ i).  An input, drawn identically for the oracle and the library."""
    x = np.arange(n, dtype=np.uint64) ^ np.uint64((int(seed) ^ (int(wave) << 32)) & MASK64)
    return splitmix64_np(x)


FSM_SALT = 0xBB67AE8584CAA73B


def fsm_choice(h: int, n: int) -> int:
    """Mock model under a regex constraint (reading R28): after a prefix with hash h, pick option
    splitmix64(h ^ FSM_SALT) mod n of the n allowed options (allowed bytes ascending, then STOP if
    the state is accepting)."""
    return splitmix64_int((int(h) ^ FSM_SALT) & MASK64) % n
