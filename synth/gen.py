"""Counter-based generator: splitmix64 -> uniforms -> Box-Muller normals -> bf16 (RNE).

Recipe (SURVEY.md §8(d) "Synthetic inputs"):
  * every tensor has its own stream id; element i of a stream is
    ``mix64(seed * 0x100000001B3 + stream * 0xD1B54A32D192ED03 + (i+1) * GOLDEN)``,
    i.e. a pure function of (seed, stream, i) — order independent, vectorised;
  * uniforms use the top 53 bits: u = (x >> 11 + 0.5) * 2^-53, never 0 or 1;
  * normals: Box-Muller on consecutive uniform pairs, fp64;
  * bf16: fp64 -> fp32 (numpy RNE) -> bf16 (RNE on the bit pattern).
Returned bf16 tensors are ``numpy.uint16`` bit patterns.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_SEED_MUL = np.uint64(0x100000001B3)
_STREAM_MUL = np.uint64(0xD1B54A32D192ED03)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


def splitmix64(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    """n raw 64-bit outputs of stream ``stream`` starting at element ``offset``."""
    with np.errstate(over="ignore"):
        base = (np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * _SEED_MUL
                + np.uint64(stream & 0xFFFFFFFFFFFFFFFF) * _STREAM_MUL)
        idx = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        return _mix64(base + idx * GOLDEN)


def uniform01(seed: int, stream: int, n: int) -> np.ndarray:
    x = splitmix64(seed, stream, n)
    return ((x >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def normal(seed: int, stream: int, n: int) -> np.ndarray:
    m = (n + 1) // 2
    u = uniform01(seed, stream, 2 * m)
    u1, u2 = u[0::2], u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * m, dtype=np.float64)
    z[0::2] = r * np.cos(2.0 * np.pi * u2)
    z[1::2] = r * np.sin(2.0 * np.pi * u2)
    return z[:n]


def bf16_bits_from_f64(x: np.ndarray) -> np.ndarray:
    """fp64 -> fp32 (RNE) -> bf16 bits (RNE). NaN stays NaN (quiet)."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    b = f.view(np.uint32)
    lsb = (b >> np.uint32(16)) & np.uint32(1)
    with np.errstate(over="ignore"):
        r = ((b + np.uint32(0x7FFF) + lsb) >> np.uint32(16)).astype(np.uint16)
    nan = np.isnan(f)
    if nan.any():
        r[nan] = np.uint16(0x7FC0)
    return r


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def normal_bf16(seed: int, stream: int, shape, std: float = 1.0) -> np.ndarray:
    n = int(np.prod(shape)) if len(shape) else 1
    return bf16_bits_from_f64(normal(seed, stream, n) * std).reshape(shape)


def int_bf16(seed: int, stream: int, shape, lo: int, hi: int) -> np.ndarray:
    """Integers uniform in [lo, hi] as bf16 bits (exact for |v| <= 256)."""
    n = int(np.prod(shape))
    x = splitmix64(seed, stream, n)
    v = lo + (x % np.uint64(hi - lo + 1)).astype(np.int64)
    return bf16_bits_from_f64(v.astype(np.float64)).reshape(shape)


def sparse_int_bf16(seed: int, stream: int, shape, nnz_per_line: int, axis: int,
                    lo: int, hi: int) -> np.ndarray:
    """Integer matrix with at most ``nnz_per_line`` nonzeros along each line of
    ``axis`` (axis=1: per row; axis=0: per column), values in [lo, hi]."""
    rows, cols = shape
    lines, length = (rows, cols) if axis == 1 else (cols, rows)
    x = splitmix64(seed, stream, lines * nnz_per_line * 2).reshape(lines, nnz_per_line, 2)
    pos = (x[..., 0] % np.uint64(length)).astype(np.int64)
    val = lo + (x[..., 1] % np.uint64(hi - lo + 1)).astype(np.int64)
    m = np.zeros((lines, length), dtype=np.float64)
    for ln in range(lines):          # later duplicates overwrite: still <= nnz per line
        m[ln, pos[ln]] = val[ln]
    if axis == 0:
        m = m.T
    return bf16_bits_from_f64(m)


def seq_lengths(seed: int, stream: int, n: int, lo: int, hi: int) -> np.ndarray:
    """len = lo + (u64 % (hi - lo + 1))."""
    x = splitmix64(seed, stream, n)
    return (lo + (x % np.uint64(hi - lo + 1)).astype(np.int64)).astype(np.int32)


class Stream:
    """Hands out consecutive stream ids for one seed, so every tensor of a
    workload gets its own stream in a fixed order."""

    def __init__(self, seed: int, first: int = 1):
        self.seed = seed
        self.next_id = first

    def take(self) -> int:
        s = self.next_id
        self.next_id += 1
        return s
