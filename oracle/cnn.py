"""CPU fp32 oracle for CNN members (test infrastructure only).

Algorithm: torchvision 0.26.0+cu128 / torch 2.11.0+cu128 eager fp32 on the CPU
(third-party; the reference has no CNN code).  Model construction
is the member format's own definition (paper_2003_01538_b200.zoo.build_torch_model:
seeded init + seeded BN statistics); the oracle's job is the arithmetic.

Input semantics follow the reference exactly up to the model input: u8 pixels
/ pixel_scale in fp32 (eg/wire.py:71), then (x - mean) / std in fp32
(eg/models.py:254-259), laid out NCHW.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import lin1


def preprocess_u8(pixels_hwc: np.ndarray, mean, std, pixel_scale: float = 255.0) -> torch.Tensor:
    """(B, H, W, C) u8 -> normalised fp32 NCHW, the reference's fp32 op order."""
    b, h, w, c = pixels_hwc.shape
    x = lin1.u8_to_f32(np.ascontiguousarray(pixels_hwc.transpose(0, 3, 1, 2)), pixel_scale)
    x = lin1.preprocess(x.reshape(b, -1), c, mean, std)
    return torch.from_numpy(x.reshape(b, c, h, w))


def resize(x_nchw: torch.Tensor, size: int) -> torch.Tensor:
    """Bilinear, align_corners=False, no antialias (torch.nn.functional.interpolate)."""
    return torch.nn.functional.interpolate(x_nchw, size=(size, size), mode="bilinear",
                                           align_corners=False)


def set_threads() -> int:
    n = len(os.sched_getaffinity(0))
    torch.set_num_threads(n)
    return n


@torch.no_grad()
def logits(model: torch.nn.Module, x_nchw: torch.Tensor) -> np.ndarray:
    """fp32 eager forward on the CPU."""
    return model.float().eval()(x_nchw.float()).numpy()


def topk_order(scores: np.ndarray, k: int) -> np.ndarray:
    """Indices by (score desc, index asc) -- the combine kernel's documented order."""
    return np.argsort(-scores, axis=-1, kind="stable")[..., :k]


def softmax(scores: np.ndarray) -> np.ndarray:
    z = scores - scores.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def decisive(scores: np.ndarray, k: int, tol: float) -> np.ndarray:
    """Samples whose first k+1 ranked scores are separated by more than 2*tol.

    For those, any implementation within the logit tolerance must reproduce the
    oracle's top-k order exactly (SURVEY.md §7.3 protocol (ii)).
    """
    s = -np.sort(-scores, axis=-1)[..., : k + 1]
    gaps = s[..., :-1] - s[..., 1:]
    return (gaps > 2 * tol).all(axis=-1)
