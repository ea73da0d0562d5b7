"""Deterministic synthetic inputs (no datasets are available offline).

SplitMix64 is the reference's cross-language generator (eg/fixtures.py:22-30);
here it is vectorised with numpy uint64 wrap-around arithmetic.  Images are u8
HWC.  ``kind="noise"`` is the survey's plain recipe (byte = z >> 56, seed =
1234 + image index); ``kind="structured"`` mixes that noise with a per-image
colour gradient so that random-init classifiers do not collapse every image onto
one class.
"""

from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Outputs start .. start + n - 1 of the SplitMix64 stream for ``seed`` (uint64)."""
    with np.errstate(over="ignore"):
        state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + _GAMMA * np.arange(
            start + 1, start + n + 1, dtype=np.uint64)
        z = state
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def noise_image(seed: int, h: int, w: int, c: int = 3) -> np.ndarray:
    return (splitmix64(seed, h * w * c) >> np.uint64(56)).astype(np.uint8).reshape(h, w, c)


def structured_image(seed: int, h: int, w: int, c: int = 3) -> np.ndarray:
    noise = noise_image(seed, h, w, c).astype(np.float32)
    p = (splitmix64(seed ^ 0x5EED, 8) >> np.uint64(40)).astype(np.float64) / float(1 << 24)
    yy, xx = np.meshgrid(np.linspace(-1, 1, h), np.linspace(-1, 1, w), indexing="ij")
    ang = 2 * np.pi * p[0]
    freq = 1.0 + 6.0 * p[1]
    wave = np.sin(freq * (np.cos(ang) * xx + np.sin(ang) * yy) * np.pi + 2 * np.pi * p[2])
    base = np.stack([p[3 + (i % 3)] for i in range(c)]) * 255.0
    img = base[None, None, :] * (0.5 + 0.5 * wave[..., None]) * (0.4 + 1.2 * p[6])
    img = 0.7 * img + 0.3 * noise
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def images(n: int, h: int, w: int, c: int = 3, seed0: int = 1234, kind: str = "structured") -> np.ndarray:
    fn = structured_image if kind == "structured" else noise_image
    return np.stack([fn(seed0 + i, h, w, c) for i in range(n)])


def images_fast(n: int, h: int, w: int, c: int = 3, seed0: int = 1234, first_row: int = 0) -> np.ndarray:
    """Large batches for benchmarking: one SplitMix64 stream, byte = z >> 56.  Rows
    first_row .. first_row + n - 1 of that stream's images (a rank's shard of a global
    batch is the same bytes as the global batch's rows)."""
    px = h * w * c
    return (splitmix64(seed0, n * px, first_row * px) >> np.uint64(56)).astype(np.uint8).reshape(n, h, w, c)
