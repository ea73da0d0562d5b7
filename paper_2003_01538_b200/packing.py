"""Host-side weight packing for the sm_100a conv/GEMM kernel (K2/K3).

The kernel reads weights as a dense, K-major bf16 matrix W[N = Cout, K] through a
2-D TMA map with 128-byte swizzle, 64 K-elements per block.  The K ordering has to
match the order in which the A operand (activations) is gathered:

* ``im2col`` (any kh x kw, stride, padding): K = (tap, channel) with the channel
  axis padded to a multiple of 64 per tap -- one TMA im2col load per (tap,
  64-channel chunk);
* ``tiled`` (1x1, stride 1): K = channel padded to 64;
* ``c8`` (the stem, Cin <= 8): K = (filter row, 8 pixel slots, 8 channels) --
  one 64-wide K block per filter row, slots >= kw and channels >= Cin are zero;
* ``flatten`` (FC on an H x W x C feature map): K = NHWC order of the feature
  map (torchvision flattens NCHW, so the columns are permuted here), padded to 64.

Padding is zero, so padded K positions contribute exactly 0.
"""

from __future__ import annotations

import numpy as np
import torch


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def conv_mode(kh: int, kw: int, sh: int, sw: int, ph: int, pw: int, cin: int, stem: bool) -> str:
    if stem:
        # stride-2 stems read even/odd column planes: their K groups list even taps first
        return "c8s2" if sw == 2 else "c8"
    if kh == kw == 1 and sh == sw == 1 and ph == pw == 0:
        return "tiled"
    return "im2col"


def pack_conv_weight(w: torch.Tensor, mode: str, hw: tuple[int, int] | None = None) -> torch.Tensor:
    """fp32 [Cout, Cin, kh, kw] (or [Cout, C*H*W] for flatten) -> bf16 [Cout, Kpad]."""
    w = w.detach().to(torch.float32).cpu()
    if mode == "flatten":
        cout, feat = w.shape
        h, wd = hw
        c = feat // (h * wd)
        w = w.reshape(cout, c, h, wd).permute(0, 2, 3, 1).reshape(cout, feat)
        out = torch.zeros(cout, _round_up(feat, 64), dtype=torch.float32)
        out[:, :feat] = w
        return out.to(torch.bfloat16).contiguous()
    cout, cin, kh, kw = w.shape
    taps = kh * kw
    wt = w.permute(0, 2, 3, 1).reshape(cout, taps, cin)  # (Cout, tap, Cin)
    if mode in ("c8", "c8s2"):
        # one 64-wide K block per filter row: 8 K groups (taps) x 8 channels; "c8s2" orders
        # the groups as taps 0, 2, 4, 6, 1, 3, 5, 7 (csrc/conv_umma.cu, stem planes mode)
        if cin > 8 or kw > 8:
            raise ValueError("c8 packing needs Cin <= 8 and kw <= 8")
        out = torch.zeros(cout, kh, 8, 8, dtype=torch.float32)
        wr = wt.reshape(cout, kh, kw, cin)
        for g in range(8):
            tap = (2 * g if g < 4 else 2 * (g - 4) + 1) if mode == "c8s2" else g
            if tap < kw:
                out[:, :, g, :cin] = wr[:, :, tap, :]
    else:
        cpad = _round_up(cin, 64)
        out = torch.zeros(cout, taps, cpad, dtype=torch.float32)
        out[:, :, :cin] = wt
    return out.reshape(cout, -1).to(torch.bfloat16).contiguous()


def fold_bn(weight: torch.Tensor, bias: torch.Tensor | None, bn) -> tuple[torch.Tensor, torch.Tensor]:
    """Fold an eval-mode BatchNorm that follows a conv into the conv's weight/bias."""
    scale = bn.weight.detach().double() / torch.sqrt(bn.running_var.detach().double() + bn.eps)
    shift = bn.bias.detach().double() - bn.running_mean.detach().double() * scale
    w = weight.detach().double() * scale.reshape(-1, *([1] * (weight.dim() - 1)))
    b = shift if bias is None else bias.detach().double() * scale + shift
    return w.float(), b.float()


def bn_affine(bn) -> tuple[torch.Tensor, torch.Tensor]:
    """Per-channel (scale, shift) of an eval-mode BatchNorm: y = x * scale + shift."""
    scale = bn.weight.detach().double() / torch.sqrt(bn.running_var.detach().double() + bn.eps)
    shift = bn.bias.detach().double() - bn.running_mean.detach().double() * scale
    return scale.float(), shift.float()


def u8_lut(mean, std, pixel_scale: float, channels: int) -> np.ndarray:
    """The reference's fp32 preprocess of every byte value, per channel.

    ((np.float32(v) / np.float32(pixel_scale)) - mean_c) / std_c with numpy's
    fp32 ops, i.e. exactly eg/wire.py:71 followed by eg/models.py:254-259.
    """
    mean = np.asarray(mean, dtype=np.float32).reshape(-1)
    std = np.asarray(std, dtype=np.float32).reshape(-1)
    v = np.arange(256, dtype=np.float32) / np.float32(pixel_scale)
    lut = np.empty((channels, 256), dtype=np.float32)
    for c in range(channels):
        m = mean[0] if mean.size == 1 else mean[c]
        s = std[0] if std.size == 1 else std[c]
        lut[c] = (v - m) / s
    return lut


def pick_block_n(cout: int, groups: int = 1) -> int:
    """The N-tile width the native planner uses (runtime.cu pick_block_n)."""
    bn = 32 if cout <= 32 else 64 if cout <= 64 else 128 if cout <= 128 else (256 if cout % 256 == 0 else 128)
    if groups > 1:  # (runtime.cu plan_conv: 64-wide block-diagonal tiles when a group fits)
        return min(bn, 64) if cout // groups <= 64 else min(bn, 128)
    return bn


def pack_grouped_conv_weight(w: torch.Tensor, groups: int, block_n: int) -> torch.Tensor:
    """Grouped conv (Cin == Cout) as block-diagonal N tiles.

    fp32 [Cout, Cout/groups, kh, kw] -> bf16 [Cout, taps * ceil(BN/64)*64]: output row o
    (tile t = o // BN) holds its group's weights at input positions relative to the
    tile's channel window [t*BN, t*BN + BN); everything else is zero.
    """
    w = w.detach().to(torch.float32).cpu()
    cout, cpg, kh, kw = w.shape
    if block_n % cpg != 0:
        raise ValueError("a group must not straddle N tiles")
    taps = kh * kw
    bpad = _round_up(block_n, 64)
    out = torch.zeros(cout, taps, bpad, dtype=torch.float32)
    wt = w.permute(0, 2, 3, 1).reshape(cout, taps, cpg)
    for o in range(cout):
        g = o // cpg
        rel = g * cpg - (o // block_n) * block_n
        out[o, :, rel:rel + cpg] = wt[o]
    return out.reshape(cout, -1).to(torch.bfloat16).contiguous()


def pack_conv_weight_f32(w: torch.Tensor, cin_pad: int | None = None,
                         hw: tuple[int, int] | None = None) -> torch.Tensor:
    """fp32-faithful mode (csrc/ref32.cu): fp32 [Cout, Cin/groups, kh, kw] ->
    [Cout, kh, kw, Cin'] (channels zero-padded to ``cin_pad``: a stem reads the 8-channel
    K1 image); an FC after an H x W map (``hw``) -> [Cout, H*W*C] in NHWC order."""
    w = w.detach().to(torch.float32).cpu()
    if hw is not None:
        cout, feat = w.shape
        h, wd = hw
        c = feat // (h * wd)
        return w.reshape(cout, c, h, wd).permute(0, 2, 3, 1).reshape(cout, feat).contiguous()
    if w.dim() == 2:
        w = w.reshape(w.shape[0], -1, 1, 1)
    out = w.permute(0, 2, 3, 1)
    if cin_pad is not None and cin_pad > out.shape[3]:
        pad = torch.zeros(*out.shape[:3], cin_pad - out.shape[3])
        out = torch.cat([out, pad], dim=3)
    return out.reshape(out.shape[0], -1).contiguous()
