"""numpy restatement of the reference's LIN1 forward path (test oracle only).

Every function cites the reference line it restates (paths relative to
/root/reference/pkg/src/ensemblegate/).
"""

from __future__ import annotations

import json

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64(seed: int, n: int) -> list[int]:
    """fixtures.py:22-30 -- plain-integer SplitMix64 (n outputs)."""
    out = []
    state = seed & MASK64
    for _ in range(n):
        state = (state + 0x9E3779B97F4A7C15) & MASK64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        out.append(z ^ (z >> 31))
    return out


def symmetric_floats(seed: int, n: int) -> np.ndarray:
    """fixtures.py:39-42 -- (z >> 40) / 2^23 - 1, exact in fp32."""
    z = np.asarray(splitmix64(seed, n), dtype=np.uint64)
    return ((z >> np.uint64(40)).astype(np.float64) / float(1 << 23) - 1.0)


def gen_model_arrays(seed: int, k: int, d: int) -> tuple[np.ndarray, np.ndarray]:
    """fixtures.py:45-74 -- the weights (K, D) then bias (K) of gen_model, same stream order."""
    v = symmetric_floats(seed, k * d + k)
    return v[: k * d].reshape(k, d).astype(np.float32), v[k * d:].astype(np.float32)


def preprocess(x: np.ndarray, channels: int, mean, std) -> np.ndarray:
    """models.py:254-259 -- ((x.reshape(B, C, HW) - mean_f32) / std_f32), fp32."""
    mean = np.asarray(mean, dtype=np.float32).reshape(-1, 1)
    std = np.asarray(std, dtype=np.float32).reshape(-1, 1)
    b, d = x.shape
    return ((x.reshape(b, channels, d // channels) - mean) / std).reshape(b, d)


def u8_to_f32(pixels: np.ndarray, pixel_scale: float) -> np.ndarray:
    """wire.py:71 -- pixels.astype(f32) / f32(pixel_scale)."""
    return pixels.astype(np.float32) / np.float32(pixel_scale)


def linear_scores(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """models.py:275-278 -- fp64 einsum, bias added after the sum."""
    s = np.einsum("bd,kd->bk", x.astype(np.float64), w.astype(np.float64))
    s += b.astype(np.float64)
    return s


def argmax_lowest(scores: np.ndarray) -> np.ndarray:
    """models.py:279 -- np.argmax (first maximum = lowest index on ties)."""
    return np.argmax(scores, axis=1)


def forward(members, x_raw: np.ndarray, channels: int, mean, std) -> list[list[int]]:
    """ensemble.py:248-250 -- preprocess once, then every member in manifest order.

    members: list of (weights (K, D) f32, bias (K,) f32).
    """
    xp = preprocess(np.asarray(x_raw, dtype=np.float32), channels, mean, std)
    return [argmax_lowest(linear_scores(xp, w, b)).tolist() for w, b in members]


def apply_policy(kind: str, k, votes) -> list[int]:
    """policy.py:66-76 -- any = max, all = min, at_least = colsum >= k."""
    arr = np.asarray(votes, dtype=np.int64)
    if kind == "any":
        return arr.max(axis=0).tolist()
    if kind == "all":
        return arr.min(axis=0).tolist()
    return (arr.sum(axis=0) >= k).astype(np.int64).tolist()


def canonical(obj) -> bytes:
    """jsonio.py:28-36 -- sorted keys, compact separators."""
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), allow_nan=False,
                      ensure_ascii=True).encode("utf-8")


def unit_floats(seed: int, n: int) -> np.ndarray:
    """fixtures.py:33-36 -- (z >> 40) / 2^24 in [0, 1), exact in fp32."""
    z = np.asarray(splitmix64(seed, n), dtype=np.uint64)
    return ((z >> np.uint64(40)).astype(np.float64) / float(1 << 24)).astype(np.float32)
