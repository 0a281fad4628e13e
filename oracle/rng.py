"""Oracle (TEST INFRASTRUCTURE ONLY): counter-based generator, numpy side.

Bit-for-bit restatement of ``paper_2501_10375_b200/csrc/rng.cuh``.  The
reference has no weights (pkg/README.md:16-18); this generator is builder
defined so that 90 GB of Mixtral-shaped random-init weights never has to be
stored: any element is a pure function of (seed, tag, index).

    mix64(z)     = splitmix64 finaliser
    key(seed,tag)= mix64(seed * G ^ mix64(tag + G))
    bits(key,i)  = mix64(key + (i + 1) * G)
    u(key,i)     = float32(bits >> 40) * 2^-23 - 1        in [-1, 1), exact
    value        = bf16_rne(float32(u * scale))            (weights)
                 = float32(u * scale)                      (fp32 tensors)
"""

from __future__ import annotations

import numpy as np

G = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

# tag kinds (top byte of the 64-bit tag)
KIND_EXPERT = 1   # matrix 0 = W1 (ffn,d), 1 = W3 (ffn,d), 2 = W2 (d,ffn)
KIND_GATE = 2     # (E, d) router rows of one layer
KIND_NORM = 3     # (d,) RMSNorm weight of one layer
KIND_INPUT = 4    # activations: layer field = stream id, expert field = step


def make_tag(kind: int, layer: int = 0, expert: int = 0, matrix: int = 0) -> int:
    return (kind << 56) | (layer << 32) | (expert << 16) | matrix


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * M1
    z = z ^ (z >> np.uint64(27))
    z = z * M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, tag: int) -> np.uint64:
    with np.errstate(over="ignore"):
        t = _mix64(np.array([np.uint64(tag) + G], dtype=np.uint64))
        s = np.array([np.uint64(seed) * G], dtype=np.uint64)
        return _mix64(s ^ t)[0]


def uniform_pm1(seed: int, tag: int, index: np.ndarray) -> np.ndarray:
    """float32 values in [-1, 1) for the given flat indices."""
    key = stream_key(seed, tag)
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        b = _mix64(key + (idx + np.uint64(1)) * G)
    u = (b >> np.uint64(40)).astype(np.float32)
    return u * np.float32(2.0 ** -23) - np.float32(1.0)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 bit pattern (uint16)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (b >> np.uint32(16)) & np.uint32(1)
    return ((b + np.uint32(0x7FFF) + r) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 value, returned as float32."""
    return bf16_bits_to_f32(f32_to_bf16_bits(x))


def tensor_f32(seed: int, tag: int, shape, scale: float, offset: int = 0) -> np.ndarray:
    n = int(np.prod(shape))
    u = uniform_pm1(seed, tag, np.arange(offset, offset + n, dtype=np.uint64))
    return (u * np.float32(scale)).reshape(shape)


def tensor_bf16(seed: int, tag: int, shape, scale: float, offset: int = 0) -> np.ndarray:
    """bf16-valued tensor returned as float32 (exact)."""
    return round_bf16(tensor_f32(seed, tag, shape, scale, offset))


def norm_weight(seed: int, layer: int, d: int) -> np.ndarray:
    """RMSNorm weight: bf16(1 + 0.25 * u)."""
    u = uniform_pm1(seed, make_tag(KIND_NORM, layer), np.arange(d, dtype=np.uint64))
    return round_bf16(np.float32(1.0) + np.float32(0.25) * u)
