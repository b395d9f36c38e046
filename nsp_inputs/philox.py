"""Counter-based Philox4x32-10 generator + Box-Muller, vectorised in numpy.

Seeded-input generator shared by the oracle and the CUDA path's harness (the
only code both sides may use; it holds none of the method's arithmetic).
Reading SURVEY.md §8(c) C7: key = seed, counter = (element index lo, element
index hi, stream id, 0); two 53-bit uniforms in (0,1) from the 4x32-bit output,
then the Box-Muller cosine branch.  The paper only says "the same seed"
(§5) and "entries from the standard normal distribution"
(PAPER.md:1172-1173); the generator itself is this build's documented choice.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint32(0x9E3779B9)
_W1 = np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)

# stream ids (SURVEY.md §8(d) "Seeds": Omega 0, x*/b 1, field 2, RGG points 3, RGG weights 4)
STREAM_OMEGA = 0
STREAM_XSTAR = 1
STREAM_FIELD = 2
STREAM_POINTS = 3
STREAM_WEIGHTS = 4


def philox4x32_10(ctr: np.ndarray, key: tuple[int, int]) -> np.ndarray:
    """ctr: (..., 4) uint32 counters; key: (k0, k1). Returns (..., 4) uint32."""
    c = [ctr[..., i].astype(np.uint64) for i in range(4)]
    k0 = np.uint32(key[0] & 0xFFFFFFFF)
    k1 = np.uint32(key[1] & 0xFFFFFFFF)
    for _ in range(10):
        p0 = _M0 * c[0]
        p1 = _M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
        k0 = np.uint32((int(k0) + int(_W0)) & 0xFFFFFFFF)
        k1 = np.uint32((int(k1) + int(_W1)) & 0xFFFFFFFF)
    return np.stack([x.astype(np.uint32) for x in c], axis=-1)


def _raw(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    idx = np.arange(start, start + count, dtype=np.uint64)
    ctr = np.empty((count, 4), dtype=np.uint32)
    ctr[:, 0] = (idx & _MASK32).astype(np.uint32)
    ctr[:, 1] = (idx >> np.uint64(32)).astype(np.uint32)
    ctr[:, 2] = np.uint32(stream)
    ctr[:, 3] = 0
    return philox4x32_10(ctr, (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))


def _uniform_pair(r: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Two doubles in the open interval (0,1) from 4x u32 (53 bits each)."""
    a = r[:, 0].astype(np.uint64) >> np.uint64(5)   # 27 bits
    b = r[:, 1].astype(np.uint64) >> np.uint64(6)   # 26 bits
    c = r[:, 2].astype(np.uint64) >> np.uint64(5)
    d = r[:, 3].astype(np.uint64) >> np.uint64(6)
    scale = 1.0 / 9007199254740992.0               # 2^-53
    u1 = ((a * np.uint64(67108864) + b).astype(np.float64) + 0.5) * scale
    u2 = ((c * np.uint64(67108864) + d).astype(np.float64) + 0.5) * scale
    return u1, u2


def _chunks(count: int, chunk: int = 1 << 22):
    for s in range(0, count, chunk):
        yield s, min(count, s + chunk)


def uniform(seed: int, stream: int, count: int) -> np.ndarray:
    """count doubles in (0,1): element e uses counter e (first uniform of the pair)."""
    out = np.empty(count, dtype=np.float64)
    for s, e in _chunks(count):
        u1, _ = _uniform_pair(_raw(seed, stream, s, e - s))
        out[s:e] = u1
    return out


def gaussian(seed: int, stream: int, count: int) -> np.ndarray:
    """count i.i.d. N(0,1) doubles: element e = sqrt(-2 ln u1) cos(2 pi u2) from counter e."""
    out = np.empty(count, dtype=np.float64)
    for s, e in _chunks(count):
        u1, u2 = _uniform_pair(_raw(seed, stream, s, e - s))
        out[s:e] = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return out


def gaussian_block(seed: int, stream: int, rows: int, cols: int) -> np.ndarray:
    """Row-major rows x cols N(0,1) block; element (i, j) uses counter i*cols + j."""
    return gaussian(seed, stream, rows * cols).reshape(rows, cols)
