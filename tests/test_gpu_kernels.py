"""Kernel-level parity on the B200: every conv class the model families use,
against a plain fp32 PyTorch CPU convolution of the same bf16-rounded operands."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2003_01538_b200 import _lib
from paper_2003_01538_b200.packing import (conv_mode, pack_conv_weight, pack_grouped_conv_weight,
                                          pick_block_n, u8_lut)

pytestmark = pytest.mark.gpu

DEV = "cuda"


def _p(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def run_conv(x_nhwc, ldx, cin, w, bias, res, relu, kh, kw, sh, sw, ph, pw, *, y_ld=None,
             y_off=0, out_f32=False, stem=False, split_k=0, block_n=0, pre=None, groups=1):
    lib = _lib.load()
    B, H, W, _ = x_nhwc.shape
    cout = w.shape[0]
    Ho = (H + 2 * ph - kh) // sh + 1
    Wo = (W + 2 * pw - kw) // sw + 1
    if groups > 1:
        wp = pack_grouped_conv_weight(w, groups, block_n or pick_block_n(cout, groups)).to(DEV)
    else:
        wp = pack_conv_weight(w, conv_mode(kh, kw, sh, sw, ph, pw, cin, stem)).to(DEV)
    ld = y_ld or cout
    y = torch.zeros(B, Ho, Wo, ld, device=DEV, dtype=torch.float32 if out_f32 else torch.bfloat16)
    ws = torch.empty(2 * 148 * 128 * 256, device=DEV, dtype=torch.float32)
    b = bias.to(DEV) if bias is not None else None
    pre_s = pre_t = None
    if pre is not None:
        kpad = (cin + 63) // 64 * 64
        pre_s = torch.zeros(kpad, device=DEV)
        pre_t = torch.zeros(kpad, device=DEV)
        pre_s[:cin] = pre[0].to(DEV)
        pre_t[:cin] = pre[1].to(DEV)
    _lib.check(lib.eb_k_conv(
        _p(x_nhwc), B, H, W, ldx, cin, _p(wp), _p(b), _p(res), res.shape[-1] if res is not None else 0,
        _p(y), ld, y_off, cout, kh, kw, sh, sw, ph, pw, int(relu), int(out_f32), int(stem),
        split_k, block_n, groups, _p(ws), _p(pre_s), _p(pre_t), None))
    torch.cuda.synchronize()
    return y


def ref_conv(x_nhwc, cin, w, bias, res, relu, kh, kw, sh, sw, ph, pw, groups=1):
    x = x_nhwc[..., :cin].float().cpu().permute(0, 3, 1, 2)
    wr = w.to(torch.bfloat16).float()
    y = F.conv2d(x, wr, None if bias is None else bias.float(), stride=(sh, sw), padding=(ph, pw),
                 groups=groups)
    y = y.permute(0, 2, 3, 1)
    if res is not None:
        y = y + res.float().cpu()
    if relu:
        y = torch.relu(y)
    return y


CASES = [
    # name, B, H, W, cin, cout, kh, kw, sh, sw, ph, pw
    ("1x1", 2, 14, 14, 256, 128, 1, 1, 1, 1, 0, 0),
    ("3x3", 2, 14, 14, 64, 64, 3, 3, 1, 1, 1, 1),
    ("3x3s2", 3, 28, 28, 128, 256, 3, 3, 2, 2, 1, 1),
    ("1x1s2", 2, 28, 28, 256, 512, 1, 1, 2, 2, 0, 0),
    ("7x7tail", 5, 7, 7, 512, 512, 3, 3, 1, 1, 1, 1),
    ("1x7", 2, 17, 17, 128, 192, 1, 7, 1, 1, 0, 3),
    ("7x1", 2, 17, 17, 128, 192, 7, 1, 1, 1, 3, 0),
    ("5x5", 2, 35, 35, 48, 64, 5, 5, 1, 1, 2, 2),
    ("3x3s2valid", 2, 35, 35, 96, 96, 3, 3, 2, 2, 0, 0),
    ("growth32", 2, 56, 56, 128, 32, 3, 3, 1, 1, 1, 1),
    # taps-in-N mode edges: partial N tiles, ragged Cin, odd image sizes, 1x3 filters
    ("3x3c48", 3, 15, 13, 64, 48, 3, 3, 1, 1, 1, 1),
    ("3x3c24ragged", 2, 9, 11, 40, 24, 3, 3, 1, 1, 1, 1),
    ("1x3c64", 2, 8, 8, 96, 64, 1, 3, 1, 1, 0, 1),
    ("3x3c64big", 4, 30, 30, 64, 64, 3, 3, 1, 1, 1, 1),
    # tall taps-in-N (Cout 32, Cin > 64, one load per channel chunk): 7x7 tail images,
    # a ragged second chunk, 4 chunks, and the widest grid one 256-row box covers (Wp = 64)
    ("tall7", 5, 7, 7, 256, 32, 3, 3, 1, 1, 1, 1),
    ("tall14c96", 3, 14, 14, 96, 32, 3, 3, 1, 1, 1, 1),
    ("tall28c256", 2, 28, 28, 256, 32, 3, 3, 1, 1, 1, 1),
    ("tallWp64", 2, 10, 62, 128, 32, 3, 3, 1, 1, 1, 1),
    ("tallWp66", 2, 6, 64, 128, 32, 3, 3, 1, 1, 1, 1),
    ("tallc512", 2, 14, 14, 512, 32, 3, 3, 1, 1, 1, 1),  # weights too large: regular taps-in-N
    # unpadded 3x3 stride-1 (Inception-v3 Conv2d_2a / 4a): padded-grid modes with Wp = W
    ("valid3x3c32", 2, 37, 37, 32, 32, 3, 3, 1, 1, 0, 0),
    ("valid3x3c192", 2, 19, 19, 80, 192, 3, 3, 1, 1, 0, 0),
    ("valid3x3c64", 3, 21, 17, 64, 64, 3, 3, 1, 1, 0, 0),
    ("valid3x3tall", 2, 16, 16, 128, 32, 3, 3, 1, 1, 0, 0),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_conv_matches_fp32(case):
    _, B, H, W, cin, cout, kh, kw, sh, sw, ph, pw = case
    g = torch.Generator().manual_seed(hash(case[0]) & 0xFFFF)
    x = torch.randn(B, H, W, cin, generator=g).to(torch.bfloat16).to(DEV)
    w = torch.randn(cout, cin, kh, kw, generator=g) / np.sqrt(cin * kh * kw)
    bias = torch.randn(cout, generator=g) * 0.1
    y = run_conv(x, cin, cin, w, bias, None, True, kh, kw, sh, sw, ph, pw)
    r = ref_conv(x, cin, w, bias, None, True, kh, kw, sh, sw, ph, pw)
    err = (y.float().cpu() - r).abs().max().item()
    assert err <= 0.02 * r.abs().max().item() + 1e-2, err


def test_conv_stem_c8():
    g = torch.Generator().manual_seed(7)
    B, H, W = 2, 56, 56
    x3 = torch.randn(B, H, W, 3, generator=g)
    x = torch.zeros(B, H, W, 8)
    x[..., :3] = x3
    x = x.to(torch.bfloat16).to(DEV)
    w = torch.randn(64, 3, 7, 7, generator=g) / np.sqrt(147)
    bias = torch.randn(64, generator=g) * 0.1
    y = run_conv(x, 8, 8, w, bias, None, True, 7, 7, 2, 2, 3, 3, stem=True)
    r = ref_conv(x, 3, w, bias, None, True, 7, 7, 2, 2, 3, 3)
    err = (y.float().cpu() - r).abs().max().item()
    assert err <= 0.02 * r.abs().max().item() + 1e-2, err


STEM_CASES = [
    # name, B, H, W, cout, kh, kw, s, p  (the image has 3 real channels, padded to 8)
    ("vgg_rows", 2, 30, 26, 64, 3, 3, 1, 1),
    ("resnet_planes", 3, 57, 61, 64, 7, 7, 2, 3),
    ("grouped_planes", 2, 40, 44, 128, 7, 7, 2, 3),
    ("inception_planes", 2, 37, 41, 32, 3, 3, 2, 0),
    ("wide_planes", 1, 20, 300, 64, 7, 7, 2, 3),   # Wo > 128: two tiles per output row
]


@pytest.mark.parametrize("case", STEM_CASES, ids=[c[0] for c in STEM_CASES])
@pytest.mark.parametrize("layout", [1, 2], ids=["gather", "relayout"])
def test_stem_layouts(case, layout):
    """Stems through the cp.async gather (c8_stem = 1) and through the padded rows /
    even-odd planes layouts (c8_stem = 2 after eb_k_stem_relayout)."""
    lib = _lib.load()
    _, B, H, W, cout, kh, kw, st, pd = case
    g = torch.Generator().manual_seed(H * W + cout)
    x = torch.zeros(B, H, W, 8)
    x[..., :3] = torch.randn(B, H, W, 3, generator=g)
    x = x.to(torch.bfloat16).to(DEV)
    w = torch.randn(cout, 3, kh, kw, generator=g) / np.sqrt(3 * kh * kw)
    bias = torch.randn(cout, generator=g) * 0.1
    Ho, Wo = (H + 2 * pd - kh) // st + 1, (W + 2 * pd - kw) // st + 1
    wp = pack_conv_weight(w, conv_mode(kh, kw, st, st, pd, pd, 3, True)).to(DEV)
    src = x
    if layout == 2:
        nbytes = ctypes.c_uint64(0)
        _lib.check(lib.eb_k_stem_layout(B, H, W, kh, kw, st, st, pd, pd, ctypes.byref(nbytes)))
        src = torch.full((nbytes.value // 2,), float("nan"), device=DEV).to(torch.bfloat16)
        _lib.check(lib.eb_k_stem_relayout(_p(x), B, H, W, kh, kw, st, st, pd, pd, _p(src), None))
    y = torch.full((B, Ho, Wo, cout), float("nan"), device=DEV).to(torch.bfloat16)
    _lib.check(lib.eb_k_conv(
        _p(src), B, H, W, 8, 8, _p(wp), _p(bias.to(DEV)), None, 0, _p(y), cout, 0, cout, kh, kw,
        st, st, pd, pd, 1, 0, layout, 0, 0, 1, None, None, None, None))
    torch.cuda.synchronize()
    r = ref_conv(x, 3, w, bias, None, True, kh, kw, st, st, pd, pd)
    yy = y.float().cpu()
    assert torch.isfinite(yy).all()
    err = (yy - r).abs().max().item()
    assert err <= 0.02 * r.abs().max().item() + 1e-2, err


def test_conv_slices_residual():
    # DenseNet-style: read a channel prefix of a wider buffer, write into a slice.
    g = torch.Generator().manual_seed(3)
    B, H, W, ld, cin, cout = 3, 14, 14, 192, 96, 32
    x = torch.randn(B, H, W, ld, generator=g).to(torch.bfloat16).to(DEV)
    w = torch.randn(cout, cin, 3, 3, generator=g) / np.sqrt(cin * 9)
    res = torch.randn(B, H, W, cout, generator=g).to(torch.bfloat16).to(DEV)
    y = run_conv(x, ld, cin, w, None, res, True, 3, 3, 1, 1, 1, 1, y_ld=128, y_off=64)
    r = ref_conv(x, cin, w, None, res, True, 3, 3, 1, 1, 1, 1)
    yy = y.float().cpu()
    assert (yy[..., :64] == 0).all() and (yy[..., 96:] == 0).all()
    err = (yy[..., 64:96] - r).abs().max().item()
    assert err <= 0.02 * r.abs().max().item() + 1e-2, err


@pytest.mark.parametrize("split", [1, 0, 4])
def test_fc_f32_splitk(split):
    g = torch.Generator().manual_seed(11)
    B, cin, cout = 5, 2048, 1000
    x = torch.randn(B, 1, 1, cin, generator=g).to(torch.bfloat16).to(DEV)
    w = torch.randn(cout, cin, 1, 1, generator=g) / np.sqrt(cin)
    bias = torch.randn(cout, generator=g)
    y = run_conv(x, cin, cin, w, bias, None, False, 1, 1, 1, 1, 0, 0, out_f32=True, split_k=split)
    r = ref_conv(x, cin, w, bias, None, False, 1, 1, 1, 1, 0, 0)
    err = (y.cpu() - r).abs().max().item()
    assert err <= 2e-3 * r.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("bn", [32, 64, 128, 256])
def test_block_n_variants(bn):
    g = torch.Generator().manual_seed(bn)
    x = torch.randn(2, 14, 14, 128, generator=g).to(torch.bfloat16).to(DEV)
    w = torch.randn(256, 128, 3, 3, generator=g) / np.sqrt(128 * 9)
    y = run_conv(x, 128, 128, w, None, None, False, 3, 3, 1, 1, 1, 1, block_n=bn)
    r = ref_conv(x, 128, w, None, None, False, 3, 3, 1, 1, 1, 1)
    err = (y.float().cpu() - r).abs().max().item()
    assert err <= 0.02 * r.abs().max().item() + 1e-2, err


def test_preprocess_u8_lut_exact():
    lib = _lib.load()
    rng = np.random.default_rng(0)
    B, H, W, C = 3, 17, 9, 3
    px = rng.integers(0, 256, size=(B, H, W, C), dtype=np.uint8)
    mean, std = (0.485, 0.456, 0.406), (0.229, 0.224, 0.225)
    lut = u8_lut(mean, std, 255.0, C)
    d_x = torch.from_numpy(px).to(DEV)
    d_lut = torch.from_numpy(lut).to(DEV)
    d_y = torch.empty(B, H, W, 8, dtype=torch.bfloat16, device=DEV)
    _lib.check(lib.eb_k_preprocess_u8_nhwc8(_p(d_x), _p(d_y), B, C, H * W, _p(d_lut), None))
    torch.cuda.synchronize()
    # reference semantics: wire.py:71 then models.py:254-259, fp32, then bf16
    x = px.astype(np.float32) / np.float32(255.0)
    ref = (x - np.asarray(mean, np.float32)) / np.asarray(std, np.float32)
    ref_bf16 = torch.from_numpy(ref).to(torch.bfloat16)
    got = d_y.cpu()
    assert torch.equal(got[..., :C], ref_bf16)
    assert (got[..., C:].float() == 0).all()


@pytest.mark.parametrize("geom", [(2, 224, 224, 3, 3, 1, 1), (2, 224, 224, 7, 7, 2, 3),
                                  (3, 19, 23, 3, 3, 1, 1), (2, 21, 25, 7, 7, 2, 3),
                                  (1, 20, 300, 7, 7, 2, 3)],
                         ids=["vgg_rows", "grouped_planes", "rows_ragged", "planes_ragged", "wide"])
def test_preprocess_u8_layout_equals_relayout(geom):
    """K1 straight into a stem layout == K1 to NHWC8 then eb_k_stem_relayout, byte for byte
    (the engine's u8 path uses the former)."""
    lib = _lib.load()
    B, H, W, kh, kw, st, pd = geom
    rng = np.random.default_rng(H * W + kh)
    px = torch.from_numpy(rng.integers(0, 256, size=(B, H, W, 3), dtype=np.uint8)).to(DEV)
    lut = torch.from_numpy(u8_lut((0.485, 0.456, 0.406), (0.229, 0.224, 0.225), 255.0, 3)).to(DEV)
    img8 = torch.empty(B, H, W, 8, dtype=torch.bfloat16, device=DEV)
    _lib.check(lib.eb_k_preprocess_u8_nhwc8(_p(px), _p(img8), B, 3, H * W, _p(lut), None))
    nbytes = ctypes.c_uint64(0)
    _lib.check(lib.eb_k_stem_layout(B, H, W, kh, kw, st, st, pd, pd, ctypes.byref(nbytes)))
    a = torch.full((nbytes.value // 2,), 7.0, device=DEV).to(torch.bfloat16)
    b = torch.full((nbytes.value // 2,), -7.0, device=DEV).to(torch.bfloat16)
    _lib.check(lib.eb_k_stem_relayout(_p(img8), B, H, W, kh, kw, st, st, pd, pd, _p(a), None))
    _lib.check(lib.eb_k_preprocess_u8_layout(_p(px), B, 3, H, W, _p(lut), kh, kw, st, st, pd, pd,
                                             _p(b), None))
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int16).cpu(), b.view(torch.int16).cpu())


def test_preprocess_f32_bit_exact():
    lib = _lib.load()
    rng = np.random.default_rng(1)
    B, C, H, W = 4, 3, 13, 11
    x = rng.random((B, C * H * W), dtype=np.float32)
    mean = np.asarray([0.485, 0.456, 0.406], np.float32)
    std = np.asarray([0.229, 0.224, 0.225], np.float32)
    ref = ((x.reshape(B, C, H * W) - mean.reshape(-1, 1)) / std.reshape(-1, 1)).reshape(B, -1)
    d_x = torch.from_numpy(x).to(DEV)
    d_y = torch.empty_like(d_x)
    d_mean, d_std = torch.from_numpy(mean).to(DEV), torch.from_numpy(std).to(DEV)
    _lib.check(lib.eb_k_preprocess_f32(_p(d_x), _p(d_y), B, C, H * W, _p(d_mean), _p(d_std), 3, None))
    torch.cuda.synchronize()
    assert np.array_equal(d_y.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_pool_and_gap():
    lib = _lib.load()
    g = torch.Generator().manual_seed(5)
    B, H, W, C = 2, 14, 14, 64
    x = torch.randn(B, H, W, C, generator=g).to(torch.bfloat16).to(DEV)
    for mode, k, s, p in [(0, 3, 2, 1), (0, 2, 2, 0), (1, 2, 2, 0), (1, 3, 1, 1)]:
        Ho = (H + 2 * p - k) // s + 1
        y = torch.zeros(B, Ho, Ho, C, dtype=torch.bfloat16, device=DEV)
        _lib.check(lib.eb_k_pool(_p(x), C, _p(y), C, 0, B, H, W, C, k, s, p, mode, None, None, None))
        torch.cuda.synchronize()
        xc = x.float().cpu().permute(0, 3, 1, 2)
        if mode == 0:
            r = F.max_pool2d(xc, k, s, p)
        else:
            r = F.avg_pool2d(xc, k, s, p, count_include_pad=True)
        r = r.permute(0, 2, 3, 1)
        assert (y.float().cpu() - r).abs().max().item() < 0.02
    y = torch.zeros(B, C, dtype=torch.bfloat16, device=DEV)
    _lib.check(lib.eb_k_gap(_p(x), C, _p(y), B, H * W, C, None, None, None))
    torch.cuda.synchronize()
    r = x.float().cpu().mean(dim=(1, 2))
    assert (y.float().cpu() - r).abs().max().item() < 0.01


@pytest.mark.parametrize("C,ldx,k,s,p,mode", [
    (288, 320, 2, 2, 0, 1),    # DenseNet transition: 36 channel groups, strided source
    (40, 40, 3, 2, 1, 0),      # 5 groups (CTA of 255 threads)
    (512, 512, 2, 2, 0, 0),    # VGG: 64 groups
    (24, 48, 3, 1, 1, 2),      # exclude-pad average
])
def test_pool_geometries_bnrelu(C, ldx, k, s, p, mode):
    lib = _lib.load()
    g = torch.Generator().manual_seed(C + k)
    B, H, W = 3, 15, 13
    x = torch.randn(B, H, W, ldx, generator=g).to(torch.bfloat16).to(DEV)
    scale = (torch.rand(C, generator=g) + 0.5).to(DEV)
    shift = (torch.randn(C, generator=g) * 0.1).to(DEV)
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    ldy, y_off = C + 16, 8
    y = torch.zeros(B, Ho, Wo, ldy, dtype=torch.bfloat16, device=DEV)
    _lib.check(lib.eb_k_pool(_p(x), ldx, _p(y), ldy, y_off, B, H, W, C, k, s, p, mode,
                             _p(scale), _p(shift), None))
    torch.cuda.synchronize()
    xa = torch.relu(x[..., :C].float().cpu() * scale.cpu() + shift.cpu()).permute(0, 3, 1, 2)
    if mode == 0:
        r = F.max_pool2d(xa, k, s, p)
    else:
        r = F.avg_pool2d(xa, k, s, p, count_include_pad=(mode == 1))
    r = r.permute(0, 2, 3, 1)
    yy = y.float().cpu()
    assert (yy[..., :y_off] == 0).all() and (yy[..., y_off + C:] == 0).all()
    assert (yy[..., y_off:y_off + C] - r).abs().max().item() < 0.03


def test_combine_argmax_topk_policy():
    lib = _lib.load()
    B, K = 6, 10
    l32 = torch.zeros(B, 2 * K)
    l32[:, :K] = torch.arange(K).float()  # member 0: argmax K-1
    l32[:, K:] = 1.0                      # member 1: all tied -> index 0
    l32[0, K + 3] = 2.0
    l64 = torch.tensor([[0.25, 0.5], [0.5, 0.5], [0.7, 0.1], [0.1, 0.2], [0.3, 0.3], [1.0, 0.0]],
                       dtype=torch.float64)
    kind = torch.tensor([0, 0, 1], dtype=torch.int32)
    koff = torch.tensor([0, K, 0], dtype=torch.int32)
    kcnt = torch.tensor([K, K, 2], dtype=torch.int32)
    d = {n: t.to(DEV) for n, t in dict(l32=l32, l64=l64, kind=kind, koff=koff, kcnt=kcnt).items()}
    labels = torch.zeros(3, B, dtype=torch.int32, device=DEV)
    tk = torch.zeros(3, B, 3, dtype=torch.int32, device=DEV)
    tp = torch.zeros(3, B, 3, dtype=torch.float32, device=DEV)
    comb = torch.zeros(B, dtype=torch.int32, device=DEV)
    _lib.check(lib.eb_k_combine(_p(d["l32"]), 2 * K, _p(d["l64"]), 2, _p(d["kind"]), _p(d["koff"]),
                                _p(d["kcnt"]), 3, B, _p(labels), 3, _p(tk), _p(tp), 0, 0, _p(comb),
                                None))
    torch.cuda.synchronize()
    lab = labels.cpu().numpy()
    assert (lab[0] == K - 1).all()
    assert lab[1, 0] == 3 and (lab[1, 1:] == 0).all()
    assert lab[2].tolist() == [1, 0, 0, 1, 0, 0]
    assert tk.cpu()[0, 0].tolist() == [K - 1, K - 2, K - 3]
    assert tk.cpu()[1, 1].tolist() == [0, 1, 2]
    p = torch.softmax(l32[0, :K], 0)
    assert torch.allclose(tp.cpu()[0, 0], p.flip(0)[:3], atol=1e-5)


@pytest.mark.parametrize("B,K", [(7, 5), (70, 16), (9, 40), (70, 130)])
def test_lin1_f64_scores(B, K):
    """K6 (both the small-K warp kernel and the 64 x 64 tiled one) against the fp64 einsum
    of eg/models.py:275-278; each sample's scores are bitwise the same alone."""
    lib = _lib.load()
    rng = np.random.default_rng(2)
    D, ns = 3000, 3
    x = rng.standard_normal((B, D)).astype(np.float32)
    w = rng.standard_normal((K, D)).astype(np.float32)
    b = rng.standard_normal(K).astype(np.float32)
    ref = np.einsum("bd,kd->bk", x.astype(np.float64), w.astype(np.float64)) + b.astype(np.float64)
    dx, dw, db = (torch.from_numpy(a).to(DEV) for a in (x, w, b))
    part = torch.empty(ns * B * K, dtype=torch.float64, device=DEV)
    out = torch.empty(B, K, dtype=torch.float64, device=DEV)
    _lib.check(lib.eb_k_lin1(_p(dx), _p(dw), _p(db), _p(part), _p(out), B, K, D, ns, None))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-9)
    assert (got.argmax(1) == ref.argmax(1)).all()
    one = torch.empty(1, K, dtype=torch.float64, device=DEV)
    _lib.check(lib.eb_k_lin1(_p(dx[B - 1:]), _p(dw), _p(db), _p(part), _p(one), 1, K, D, ns, None))
    torch.cuda.synchronize()
    assert np.array_equal(one.cpu().numpy()[0], got[B - 1])


def test_conv_pre_activation_bnrelu():
    """DenseNet: relu(x * s + t) on the (sliced) input, fused into the A path."""
    g = torch.Generator().manual_seed(13)
    B, H, W, ld, cin, cout = 3, 28, 28, 256, 160, 128
    x = torch.randn(B, H, W, ld, generator=g).to(torch.bfloat16).to(DEV)
    w = torch.randn(cout, cin, 1, 1, generator=g) / np.sqrt(cin)
    bias = torch.randn(cout, generator=g) * 0.1
    s = torch.rand(cin, generator=g) + 0.5
    t = torch.randn(cin, generator=g) * 0.3
    y = run_conv(x, ld, cin, w, bias, None, True, 1, 1, 1, 1, 0, 0, pre=(s, t))
    xa = torch.relu(x[..., :cin].float().cpu() * s + t).to(torch.bfloat16)
    r = ref_conv(xa, cin, w, bias, None, True, 1, 1, 1, 1, 0, 0)
    err = (y.float().cpu() - r).abs().max().item()
    assert err <= 0.02 * r.abs().max().item() + 1e-2, err


@pytest.mark.parametrize("width,stride", [(128, 1), (256, 2), (512, 1), (1024, 1)])
def test_grouped_conv_resnext(width, stride):
    """ResNeXt 3x3 grouped conv (32 groups) as block-diagonal N tiles."""
    g = torch.Generator().manual_seed(width + stride)
    B, H = 2, 14
    x = torch.randn(B, H, H, width, generator=g).to(torch.bfloat16).to(DEV)
    w = torch.randn(width, width // 32, 3, 3, generator=g) / np.sqrt(9 * width // 32)
    bias = torch.randn(width, generator=g) * 0.1
    y = run_conv(x, width, width, w, bias, None, True, 3, 3, stride, stride, 1, 1, groups=32)
    r = ref_conv(x, width, w, bias, None, True, 3, 3, stride, stride, 1, 1, groups=32)
    err = (y.float().cpu() - r).abs().max().item()
    assert err <= 0.02 * r.abs().max().item() + 1e-2, err


@pytest.mark.parametrize("hw,out", [((299, 299), (224, 224)), ((224, 224), (299, 299)), ((17, 9), (8, 12))])
def test_resize_bilinear_matches_interpolate(hw, out):
    lib = _lib.load()
    g = torch.Generator().manual_seed(17)
    B, C = 3, 8
    x = torch.randn(B, hw[0], hw[1], C, generator=g).to(torch.bfloat16).to(DEV)
    y = torch.zeros(B, out[0], out[1], C, dtype=torch.bfloat16, device=DEV)
    _lib.check(lib.eb_k_resize(_p(x), C, _p(y), C, B, hw[0], hw[1], C, out[0], out[1], None))
    torch.cuda.synchronize()
    r = F.interpolate(x.float().cpu().permute(0, 3, 1, 2), size=out, mode="bilinear",
                      align_corners=False).permute(0, 2, 3, 1)
    assert (y.float().cpu() - r).abs().max().item() < 0.03


GUARD_CASES = [
    # name, B, H, W, cin, cout, kh, kw, s, p, stem   (exercise every store path at odd sizes)
    ("tapn32", 3, 13, 11, 128, 32, 3, 3, 1, 1, False),
    ("tapn64", 2, 17, 9, 64, 64, 3, 3, 1, 1, False),
    ("tapshift96", 2, 15, 13, 64, 96, 3, 3, 1, 1, False),
    ("pair256", 2, 14, 14, 512, 256, 3, 3, 1, 1, False),
    ("im2col_s2", 3, 15, 15, 64, 128, 3, 3, 2, 1, False),
    ("tiled", 3, 9, 7, 192, 64, 1, 1, 1, 0, False),
    ("stem_rows", 2, 19, 23, 8, 64, 3, 3, 1, 1, True),
    ("stem_planes", 2, 21, 25, 8, 128, 7, 7, 2, 3, True),
]


@pytest.mark.parametrize("case", GUARD_CASES, ids=[c[0] for c in GUARD_CASES])
def test_conv_writes_stay_inside_output(case):
    """Bounds check without a sanitizer: the output lives inside a larger buffer filled with
    a sentinel; after the conv every element outside the [B, Ho, Wo, cout] slice (guard
    rows before/after, and the channels past cout in a wider row) must be untouched, and
    the slice must match the fp32 reference."""
    lib = _lib.load()
    _, B, H, W, cin, cout, kh, kw, st, pd, stem = case
    g = torch.Generator().manual_seed(sum(map(ord, case[0])))
    if stem:
        x = torch.zeros(B, H, W, 8)
        x[..., :3] = torch.randn(B, H, W, 3, generator=g)
        cin_real = 3
    else:
        x = torch.randn(B, H, W, cin, generator=g)
        cin_real = cin
    x = x.to(torch.bfloat16).to(DEV)
    w = torch.randn(cout, cin_real, kh, kw, generator=g) / np.sqrt(cin_real * kh * kw)
    bias = torch.randn(cout, generator=g) * 0.1
    Ho, Wo = (H + 2 * pd - kh) // st + 1, (W + 2 * pd - kw) // st + 1
    wp = pack_conv_weight(w, conv_mode(kh, kw, st, st, pd, pd, cin_real, stem)).to(DEV)
    ld = cout + 24                       # wider rows: channels [cout, ld) must stay untouched
    guard = 4096                         # elements before and after the tensor
    n = B * Ho * Wo * ld
    SENT = -12352.0  # exactly representable in bf16
    buf = torch.full((guard + n + guard,), SENT, device=DEV).to(torch.bfloat16)
    y = buf[guard:guard + n].view(B, Ho, Wo, ld)
    src = x
    layout = 1 if stem else 0
    if stem:
        nbytes = ctypes.c_uint64(0)
        _lib.check(lib.eb_k_stem_layout(B, H, W, kh, kw, st, st, pd, pd, ctypes.byref(nbytes)))
        src = torch.zeros(nbytes.value // 2, device=DEV, dtype=torch.bfloat16)
        _lib.check(lib.eb_k_stem_relayout(_p(x), B, H, W, kh, kw, st, st, pd, pd, _p(src), None))
        layout = 2
    ws = torch.zeros(4 << 20, device=DEV)
    _lib.check(lib.eb_k_conv(
        _p(src), B, H, W, x.shape[-1], x.shape[-1] if stem else cin, _p(wp), _p(bias.to(DEV)), None, 0,
        _p(y), ld, 0, cout, kh, kw, st, st, pd, pd, 1, 0, layout, 0, 0, 1, _p(ws), None, None, None))
    torch.cuda.synchronize()
    b = buf.float().cpu()
    assert (b[:guard] == SENT).all() and (b[guard + n:] == SENT).all(), "write before/after the tensor"
    yy = y.float().cpu()
    assert (yy[..., cout:] == SENT).all(), "write past cout in a row"
    r = ref_conv(x, cin_real, w, bias, None, True, kh, kw, st, st, pd, pd)
    err = (yy[..., :cout] - r).abs().max().item()
    assert err <= 0.02 * r.abs().max().item() + 1e-2, err


POOL2_CASES = [  # B, H, W, Cin, Cout
    (2, 224, 224, 64, 64),   # VGG16 conv1_2 + pool1 geometry
    (3, 20, 26, 64, 32),     # one segment, ragged (26 < 60)
    (2, 14, 122, 48, 64),    # 3 segments, the last partial; Cin < 64
    (2, 12, 16, 128, 32),    # 2 K blocks per filter row (3-plane epilogue)
    (1, 2, 2, 64, 64),       # a single pooled pixel
]


@pytest.mark.parametrize("case", POOL2_CASES, ids=[f"{c[1]}x{c[2]}c{c[3]}-{c[4]}" for c in POOL2_CASES])
def test_conv_maxpool2_fused_bit_exact(case):
    """eb_k_conv_maxpool2 == eb_k_conv then eb_k_pool(2, 2, max), bit for bit, and no write
    outside the pooled slice (guard sentinel, wider rows)."""
    lib = _lib.load()
    B, H, W, cin, cout = case
    g = torch.Generator().manual_seed(B * 1000 + H * 7 + cin)
    x = torch.randn(B, H, W, cin, generator=g).to(torch.bfloat16).to(DEV)
    w = torch.randn(cout, cin, 3, 3, generator=g) / np.sqrt(cin * 9)
    bias = (torch.randn(cout, generator=g) * 0.1).to(DEV)
    # the reference conv in the fused kernel's arithmetic: classic three-plane taps-in-N
    # (a standalone conv of this class may fold tap 2 or run tall, summing in another order)
    import os
    saved = {k: os.environ.get(k) for k in ("EB_TAPN2", "EB_TAPN_TALL")}
    os.environ["EB_TAPN2"], os.environ["EB_TAPN_TALL"] = "0", "0"
    try:
        y_full = run_conv(x, cin, cin, w, bias.cpu(), None, True, 3, 3, 1, 1, 1, 1)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    Ho2, Wo2 = H // 2, W // 2
    ref = torch.zeros(B, Ho2, Wo2, cout, device=DEV, dtype=torch.bfloat16)
    _lib.check(lib.eb_k_pool(_p(y_full), cout, _p(ref), cout, 0, B, H, W, cout, 2, 2, 0, 0,
                             None, None, None))
    wp = pack_conv_weight(w, conv_mode(3, 3, 1, 1, 1, 1, cin, False)).to(DEV)
    ld, off, guard = cout + 16, 8, 2048
    SENT = -12352.0
    n = B * Ho2 * Wo2 * ld
    buf = torch.full((guard + n + guard,), SENT, device=DEV).to(torch.bfloat16)
    y = buf[guard:guard + n].view(B, Ho2, Wo2, ld)
    _lib.check(lib.eb_k_conv_maxpool2(_p(x), B, H, W, cin, cin, _p(wp), _p(bias), _p(y), ld, off,
                                      cout, 3, 3, 1, 1, 1, None))
    torch.cuda.synchronize()
    b = buf.float().cpu()
    assert (b[:guard] == SENT).all() and (b[guard + n:] == SENT).all(), "write outside the tensor"
    yy = y.cpu()
    assert (yy[..., :off].float() == SENT).all() and (yy[..., off + cout:].float() == SENT).all()
    got = yy[..., off:off + cout]
    assert torch.equal(got, ref.cpu()), "fused pool differs from conv + pool"
    r = F.max_pool2d(ref_conv(x, cin, w, bias.cpu(), None, True, 3, 3, 1, 1, 1, 1).permute(0, 3, 1, 2), 2)
    err = (got.float() - r.permute(0, 2, 3, 1)).abs().max().item()
    assert err <= 0.02 * r.abs().max().item() + 1e-2, err


def test_conv_maxpool2_rejects_unsupported():
    lib = _lib.load()
    x = torch.zeros(1, 8, 8, 64, device=DEV, dtype=torch.bfloat16)
    wp = torch.zeros(1 << 16, device=DEV, dtype=torch.bfloat16)
    y = torch.zeros(1, 4, 4, 256, device=DEV, dtype=torch.bfloat16)
    # Cout 256 (not taps-in-N) and an odd output size are refused, not mis-computed
    assert lib.eb_k_conv_maxpool2(_p(x), 1, 8, 8, 64, 64, _p(wp), None, _p(y), 256, 0, 256, 3, 3, 1, 1,
                                  1, None) != 0
    assert lib.eb_k_conv_maxpool2(_p(x), 1, 7, 7, 64, 64, _p(wp), None, _p(y), 64, 0, 64, 3, 3, 1, 1,
                                  1, None) != 0


def test_gap_with_bnrelu_prologue():
    """Global average pool with the fused BN-ReLU prologue (DenseNet norm5 + relu + pool),
    against fp32 torch on the same bf16 input."""
    lib = _lib.load()
    g = torch.Generator().manual_seed(77)
    B, H, W, C = 3, 7, 7, 1024
    x = torch.randn(B, H, W, C, generator=g).to(torch.bfloat16).to(DEV)
    scale = (torch.rand(C, generator=g) + 0.5).to(DEV)
    shift = (torch.randn(C, generator=g) * 0.2).to(DEV)
    y = torch.empty(B, C, device=DEV, dtype=torch.bfloat16)
    _lib.check(lib.eb_k_gap(_p(x), C, _p(y), B, H * W, C, _p(scale), _p(shift), None))
    torch.cuda.synchronize()
    ref = torch.relu(x.float() * scale + shift).mean(dim=(1, 2))
    assert torch.allclose(y.float(), ref, atol=1e-2, rtol=1e-2)
