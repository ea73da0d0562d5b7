"""CNN ensemble members: the ``cnn1`` model format and its lowering to engine ops.

The reference only knows LIN1 linear members (eg/models.py:176-226)
leaves room for richer formats dispatched on the ``format`` tag.  A ``cnn1``
document names a torchvision architecture and the seeds of its random
initialisation, so every member is reproducible bit-for-bit without shipping
weights:

    {"format": "cnn1", "id": "r50", "arch": "resnet50", "seed": 1,
     "input_shape": [3, 224, 224], "labels": 1000}

``labels`` is either a list of strings or a class count K (labels class_0..).
Weights (``build_torch_model``), all deterministic from (arch, seed, K):

1. ``torch.manual_seed(seed)`` then the torchvision constructor (weights=None;
   Inception-v3 convs re-drawn fan-in scaled);
2. every BatchNorm's affine parameters and running statistics drawn from
   ``torch.Generator().manual_seed(seed + 7919)`` so that BN folding is actually
   exercised (plain random init makes BN an identity);
3. ResNet/ResNeXt residual branches scaled down: the last BN of every block
   (Bottleneck.bn3 / BasicBlock.bn2) has its affine multiplied by 0.3, so 50 blocks
   of randomly initialised residuals do not explode (ResNet-152 reached logits of
   6e8 without it);
4. BN statistics calibrated: every BN's running mean / variance is set to the
   batch statistics of a fixed calibration batch (4 structured synthetic images at
   the native size, ImageNet normalisation), computed in float64 on a copy of the
   model -- what the running statistics of a trained network would be, so eval-mode
   BN normalises and activations stay O(1) through the depth;
5. the classifier head centred: the final Linear's bias is set to -W @ mu, mu the
   mean penultimate feature over the same batch (float64), so the class ranking is
   driven by the input rather than by the network's input-independent mean
   response (random networks otherwise put every image in 1-2 classes).

Steps 4-5 cost one float64 forward of 4 images per member at load time (0.2-0.6 s
on 8 cores); float64 makes them reproducible across hosts (the stored fp32 values
are the float64 results rounded once).

Lowering (build_member) walks the module tree once, folds eval-mode BN into
the preceding conv, packs bf16 weights for the tcgen05 kernel and declares the
NHWC activation tensors and ops of the member on its own concurrency lane.
"""

from __future__ import annotations

import torch
import torch.nn as nn

from . import _lib
from .engine import Engine, TRef
from .packing import (bn_affine, conv_mode, fold_bn, pack_conv_weight, pack_conv_weight_f32,
                      pack_grouped_conv_weight, pick_block_n)

ARCHS = (
    "resnet18", "resnet34", "resnet50", "resnet101", "resnet152",
    "resnext50_32x4d", "resnext101_32x8d",
    "densenet121", "densenet169", "densenet201",
    "vgg11", "vgg13", "vgg16", "vgg19",
    "inception_v3",
)

NATIVE_SIZE = {"inception_v3": 299}


def randomize_bn(model: nn.Module, seed: int) -> None:
    g = torch.Generator().manual_seed(seed + 7919)
    with torch.no_grad():
        for m in model.modules():
            if isinstance(m, nn.BatchNorm2d):
                c = m.num_features
                m.weight.copy_(torch.empty(c).uniform_(0.6, 1.4, generator=g))
                m.bias.copy_(torch.empty(c).normal_(0.0, 0.2, generator=g))
                m.running_mean.copy_(torch.empty(c).normal_(0.0, 0.2, generator=g))
                m.running_var.copy_(torch.empty(c).uniform_(0.6, 1.6, generator=g))


def build_torch_model(arch: str, seed: int, num_classes: int = 1000) -> nn.Module:
    """The fp32 torchvision module a cnn1 document describes (eval mode, CPU)."""
    import torchvision.models as tvm

    if arch not in ARCHS:
        raise ValueError(f"unsupported arch {arch!r}")
    torch.manual_seed(seed)
    kwargs = {"weights": None, "num_classes": num_classes}
    if arch == "inception_v3":
        kwargs.update(aux_logits=False, init_weights=True)
    model = getattr(tvm, arch)(**kwargs)
    if arch == "inception_v3":
        # torchvision draws every Inception conv from N(0, 0.1) regardless of fan-in, which
        # blows activations up to ~1e12 at random init; use a fan-in scaled draw instead.
        with torch.no_grad():
            for mod in model.modules():
                if isinstance(mod, nn.Conv2d):
                    nn.init.kaiming_normal_(mod.weight, mode="fan_in", nonlinearity="relu")
    randomize_bn(model, seed)
    scale_residual_branches(model)
    calibrate(model, arch, seed, num_classes)
    return model.eval()


RESIDUAL_SCALE = 0.3
CALIB_IMAGES = 4
CALIB_SEED0 = 0xCA11B
_calib_cache: dict = {}


def scale_residual_branches(model: nn.Module, alpha: float = RESIDUAL_SCALE) -> None:
    """Multiply the affine of the last BN of every residual block by alpha."""
    from torchvision.models.resnet import BasicBlock, Bottleneck

    with torch.no_grad():
        for m in model.modules():
            bn = m.bn3 if isinstance(m, Bottleneck) else m.bn2 if isinstance(m, BasicBlock) else None
            if bn is not None:
                bn.weight.mul_(alpha)
                bn.bias.mul_(alpha)


def _calibration_batch(size: int) -> torch.Tensor:
    import numpy as np

    from . import synth

    mean = np.asarray((0.485, 0.456, 0.406), np.float32).reshape(1, 3, 1, 1)
    std = np.asarray((0.229, 0.224, 0.225), np.float32).reshape(1, 3, 1, 1)
    px = synth.images(CALIB_IMAGES, size, size, 3, seed0=CALIB_SEED0, kind="structured")
    x = (px.transpose(0, 3, 1, 2).astype(np.float32) / np.float32(255.0) - mean) / std
    return torch.from_numpy(x).double()


def calibrate(model: nn.Module, arch: str, seed: int, num_classes: int) -> None:
    """Steps 4-5 of the recipe (module docstring): BN statistics and head bias from a
    float64 forward of the calibration batch; cached per (arch, seed, K)."""
    import copy

    key = (arch, seed, num_classes)
    if key not in _calib_cache:
        m64 = copy.deepcopy(model).double()
        bns = [m for m in m64.modules() if isinstance(m, nn.BatchNorm2d)]
        for bn in bns:
            bn.reset_running_stats()
            bn.momentum = None  # cumulative average = the statistics of the one batch
        x = _calibration_batch(NATIVE_SIZE.get(arch, 224))
        m64.train()
        with torch.no_grad():
            m64(x)
        m64.eval()
        head = [m for m in m64.modules() if isinstance(m, nn.Linear)][-1]
        feats = []
        hook = head.register_forward_hook(lambda mod, i, o: feats.append(i[0]))
        with torch.no_grad():
            m64(x)
        hook.remove()
        mu = feats[0].mean(0)
        bias = -(head.weight @ mu)
        _calib_cache[key] = ([(bn.running_mean.float(), bn.running_var.float()) for bn in bns],
                             bias.float())
    stats, bias = _calib_cache[key]
    bns = [m for m in model.modules() if isinstance(m, nn.BatchNorm2d)]
    head = [m for m in model.modules() if isinstance(m, nn.Linear)][-1]
    with torch.no_grad():
        for bn, (rm, rv) in zip(bns, stats):
            bn.running_mean.copy_(rm)
            bn.running_var.copy_(rv)
        head.bias.copy_(bias)


# ---------------------------------------------------------------------- lowering


class Lowering:
    """Declares one member's tensors/ops on an Engine."""

    def __init__(self, eng: Engine, lane: int):
        self.eng = eng
        self.lane = lane

    # -- primitives --------------------------------------------------------
    def conv(self, x: TRef, conv: nn.Conv2d | nn.Linear, bn=None, relu=False, res=None,
             out: TRef | None = None, flatten=False, pre_bn=None) -> TRef:
        eng = self.eng
        if isinstance(conv, nn.Linear):
            w = conv.weight.detach().float()
            b = conv.bias.detach().float() if conv.bias is not None else None
            cout = conv.out_features
            if eng.f32:
                wp = pack_conv_weight_f32(w, hw=(x.h, x.w) if flatten else None)
            elif flatten:
                wp = pack_conv_weight(w, "flatten", hw=(x.h, x.w))
            else:
                wp = pack_conv_weight(w.reshape(cout, -1, 1, 1), "tiled")
            kh = kw = 1
            sh = sw = 1
            ph = pw = 0
            ho = wo = 1
        else:
            if conv.dilation != (1, 1):
                raise NotImplementedError("dilated convolution")
            w = conv.weight.detach().float()
            b = conv.bias.detach().float() if conv.bias is not None else None
            if bn is not None:
                w, b = fold_bn(w, b, bn)
            kh, kw = conv.kernel_size
            sh, sw = conv.stride
            ph, pw = conv.padding
            cout = conv.out_channels
            stem = x.ctot == 8 and x.c == 8  # a K1 image (native or resized)
            if eng.f32:
                wp = pack_conv_weight_f32(w, cin_pad=x.c if stem else None)
            elif conv.groups > 1:  # ResNeXt: block-diagonal N tiles
                wp = pack_grouped_conv_weight(w, conv.groups, pick_block_n(cout, conv.groups))
            else:
                wp = pack_conv_weight(w, conv_mode(kh, kw, sh, sw, ph, pw, x.c, stem))
            ho = (x.h + 2 * ph - kh) // sh + 1
            wo = (x.w + 2 * pw - kw) // sw + 1
        if out is None:
            out = eng.tensor(ho, wo, cout)
        w_off = eng.weight(wp)
        b_off = eng.weight(b.contiguous()) if b is not None else None
        so = sho = None
        if pre_bn is not None:  # BN-ReLU of the input, applied to A inside the kernel
            sc, sf = bn_affine(pre_bn)
            kpad = (x.c + 63) // 64 * 64
            so = eng.weight(torch.cat([sc, torch.zeros(kpad - x.c)]))
            sho = eng.weight(torch.cat([sf, torch.zeros(kpad - x.c)]))
        k_alg = w.shape[1] if w.dim() == 2 else w.shape[1] * w.shape[2] * w.shape[3]
        meta = {"name": "conv", "flops": 2 * ho * wo * cout * k_alg,
                "shape": (ho, wo, cout, kh, kw, sh, x.c), "weight_bytes": 2 * cout * k_alg}
        eng.op(_lib.EB_OP_CONV, x, out, cout=cout, res=res, kh=kh, kw=kw, sh=sh, sw=sw, ph=ph,
               pw=pw, relu=relu, flatten=flatten, lane=self.lane, w_off=w_off, b_off=b_off,
               scale_off=so, shift_off=sho, meta=meta,
               groups=getattr(conv, "groups", 1))
        return out

    def pool(self, x: TRef, k, s, p, mode, out: TRef | None = None, bn=None) -> TRef:
        ho = (x.h + 2 * p - k) // s + 1
        wo = (x.w + 2 * p - k) // s + 1
        if out is None:
            out = self.eng.tensor(ho, wo, x.c)
        so = sh = None
        if bn is not None:
            sc, sf = bn_affine(bn)
            so, sh = self.eng.weight(sc), self.eng.weight(sf)
        self.eng.op(_lib.EB_OP_POOL, x, out, kh=k, kw=k, sh=s, sw=s, ph=p, pw=p, pool_mode=mode,
                    lane=self.lane, scale_off=so, shift_off=sh)
        return out

    def bnrelu(self, x: TRef, bn, out: TRef) -> TRef:
        sc, sf = bn_affine(bn)
        self.eng.op(_lib.EB_OP_BNRELU, x, out, lane=self.lane, scale_off=self.eng.weight(sc),
                    shift_off=self.eng.weight(sf))
        return out

    def gap(self, x: TRef, bn=None) -> TRef:
        out = self.eng.tensor(1, 1, x.c)
        so = sh = None
        if bn is not None:
            sc, sf = bn_affine(bn)
            so, sh = self.eng.weight(sc), self.eng.weight(sf)
        self.eng.op(_lib.EB_OP_GAP, x, out, lane=self.lane, scale_off=so, shift_off=sh)
        return out

    # -- architectures -----------------------------------------------------
    def resnet(self, m, x: TRef, logits: TRef, stem_out: TRef | None = None) -> None:
        x = stem_out if stem_out is not None else self.conv(x, m.conv1, m.bn1, relu=True)
        x = self.pool(x, 3, 2, 1, _lib.EB_POOL_MAX)
        for layer in (m.layer1, m.layer2, m.layer3, m.layer4):
            for blk in layer:
                identity = x
                if hasattr(blk, "conv3"):  # Bottleneck
                    y = self.conv(x, blk.conv1, blk.bn1, relu=True)
                    y = self.conv(y, blk.conv2, blk.bn2, relu=True)
                    if blk.downsample is not None:
                        identity = self.conv(x, blk.downsample[0], blk.downsample[1])
                    x = self.conv(y, blk.conv3, blk.bn3, relu=True, res=identity)
                else:  # BasicBlock
                    y = self.conv(x, blk.conv1, blk.bn1, relu=True)
                    if blk.downsample is not None:
                        identity = self.conv(x, blk.downsample[0], blk.downsample[1])
                    x = self.conv(y, blk.conv2, blk.bn2, relu=True, res=identity)
        x = self.gap(x)
        self.conv(x, m.fc, out=logits)

    def densenet(self, m, x: TRef, logits: TRef, stem_out: TRef | None = None) -> None:
        f = m.features
        x = stem_out if stem_out is not None else self.conv(x, f.conv0, f.norm0, relu=True)
        blocks = [getattr(f, f"denseblock{i}") for i in range(1, 5)]
        trans = [getattr(f, f"transition{i}", None) for i in range(1, 5)]
        h = (x.h + 2 - 3) // 2 + 1
        c_in = f.conv0.out_channels
        buf = None
        pending = None  # (pooled input, 1x1 conv) of the previous transition
        for bi, block in enumerate(blocks):
            layers = list(block.children())
            growth = layers[0].conv2.out_channels
            width = layers[0].conv1.out_channels
            c_tot = c_in + len(layers) * growth
            buf = self.eng.tensor(h, h, c_tot)
            if pending is None:
                self.pool(x, 3, 2, 1, _lib.EB_POOL_MAX, out=buf.slice(0, c_in))
            else:
                self.conv(pending[0], pending[1], out=buf.slice(0, c_in))
            bott = self.eng.tensor(h, h, width)
            for li, layer in enumerate(layers):
                c_cur = c_in + li * growth
                # norm1-ReLU on the concatenated input is applied to A inside the 1x1
                # kernel; norm2 folds into conv1 (bias + ReLU in the epilogue)
                y = self.conv(buf.slice(0, c_cur), layer.conv1, layer.norm2, relu=True, out=bott,
                              pre_bn=layer.norm1)
                self.conv(y, layer.conv2, out=buf.slice(c_cur, growth))
            if trans[bi] is not None:
                t = trans[bi]
                # BN-ReLU -> conv1x1 -> avgpool2x2 is evaluated as BN-ReLU -> avgpool -> conv1x1:
                # the 1x1 conv and the 2x2 mean commute (both linear), 4x fewer conv FLOPs.
                pending = (self.pool(buf, 2, 2, 0, _lib.EB_POOL_AVG, bn=t.norm), t.conv)
                c_in = t.conv.out_channels
                h = h // 2
        x = self.gap(buf, bn=f.norm5)
        self.conv(x, m.classifier, out=logits)

    def vgg(self, m, x: TRef, logits: TRef) -> None:
        mods = list(m.features.children())
        i = 0
        while i < len(mods):
            mod = mods[i]
            if isinstance(mod, nn.Conv2d):
                relu = i + 1 < len(mods) and isinstance(mods[i + 1], nn.ReLU)
                x = self.conv(x, mod, relu=relu)
                i += 2 if relu else 1
            elif isinstance(mod, nn.MaxPool2d):
                x = self.pool(x, mod.kernel_size, mod.stride, mod.padding, _lib.EB_POOL_MAX)
                i += 1
            else:
                raise NotImplementedError(type(mod))
        if (x.h, x.w) != (7, 7):
            raise NotImplementedError("VGG lowering expects a 7x7 final feature map (224 input)")
        cls = [c for c in m.classifier.children() if isinstance(c, nn.Linear)]
        x = self.conv(x, cls[0], relu=True, flatten=True)
        x = self.conv(x, cls[1], relu=True)
        self.conv(x, cls[2], out=logits)

    # -- Inception-v3 ---------------------------------------------------------
    def _bc(self, x, bc, out=None):
        return self.conv(x, bc.conv, bc.bn, relu=True, out=out)

    def inception(self, m, x: TRef, logits: TRef) -> None:
        x = self._bc(x, m.Conv2d_1a_3x3)
        x = self._bc(x, m.Conv2d_2a_3x3)
        x = self._bc(x, m.Conv2d_2b_3x3)
        x = self.pool(x, 3, 2, 0, _lib.EB_POOL_MAX)
        x = self._bc(x, m.Conv2d_3b_1x1)
        x = self._bc(x, m.Conv2d_4a_3x3)
        x = self.pool(x, 3, 2, 0, _lib.EB_POOL_MAX)
        for name in ("Mixed_5b", "Mixed_5c", "Mixed_5d"):
            x = self._inc_a(x, getattr(m, name))
        x = self._inc_b(x, m.Mixed_6a)
        for name in ("Mixed_6b", "Mixed_6c", "Mixed_6d", "Mixed_6e"):
            x = self._inc_c(x, getattr(m, name))
        x = self._inc_d(x, m.Mixed_7a)
        x = self._inc_e(x, m.Mixed_7b)
        x = self._inc_e(x, m.Mixed_7c)
        x = self.gap(x)
        self.conv(x, m.fc, out=logits)

    def _avg3(self, x):
        return self.pool(x, 3, 1, 1, _lib.EB_POOL_AVG)

    def _inc_a(self, x, blk):
        c1 = blk.branch1x1.conv.out_channels
        c5 = blk.branch5x5_2.conv.out_channels
        c3 = blk.branch3x3dbl_3.conv.out_channels
        cp = blk.branch_pool.conv.out_channels
        out = self.eng.tensor(x.h, x.w, c1 + c5 + c3 + cp)
        self._bc(x, blk.branch1x1, out=out.slice(0, c1))
        y = self._bc(x, blk.branch5x5_1)
        self._bc(y, blk.branch5x5_2, out=out.slice(c1, c5))
        y = self._bc(x, blk.branch3x3dbl_1)
        y = self._bc(y, blk.branch3x3dbl_2)
        self._bc(y, blk.branch3x3dbl_3, out=out.slice(c1 + c5, c3))
        self._bc(self._avg3(x), blk.branch_pool, out=out.slice(c1 + c5 + c3, cp))
        return out

    def _inc_b(self, x, blk):
        c3 = blk.branch3x3.conv.out_channels
        cd = blk.branch3x3dbl_3.conv.out_channels
        ho = (x.h - 3) // 2 + 1
        out = self.eng.tensor(ho, ho, c3 + cd + x.c)
        self._bc(x, blk.branch3x3, out=out.slice(0, c3))
        y = self._bc(x, blk.branch3x3dbl_1)
        y = self._bc(y, blk.branch3x3dbl_2)
        self._bc(y, blk.branch3x3dbl_3, out=out.slice(c3, cd))
        self.pool(x, 3, 2, 0, _lib.EB_POOL_MAX, out=out.slice(c3 + cd, x.c))
        return out

    def _inc_c(self, x, blk):
        out = self.eng.tensor(x.h, x.w, 768)
        self._bc(x, blk.branch1x1, out=out.slice(0, 192))
        y = self._bc(x, blk.branch7x7_1)
        y = self._bc(y, blk.branch7x7_2)
        self._bc(y, blk.branch7x7_3, out=out.slice(192, 192))
        y = self._bc(x, blk.branch7x7dbl_1)
        y = self._bc(y, blk.branch7x7dbl_2)
        y = self._bc(y, blk.branch7x7dbl_3)
        y = self._bc(y, blk.branch7x7dbl_4)
        self._bc(y, blk.branch7x7dbl_5, out=out.slice(384, 192))
        self._bc(self._avg3(x), blk.branch_pool, out=out.slice(576, 192))
        return out

    def _inc_d(self, x, blk):
        ho = (x.h - 3) // 2 + 1
        out = self.eng.tensor(ho, ho, 320 + 192 + x.c)
        y = self._bc(x, blk.branch3x3_1)
        self._bc(y, blk.branch3x3_2, out=out.slice(0, 320))
        y = self._bc(x, blk.branch7x7x3_1)
        y = self._bc(y, blk.branch7x7x3_2)
        y = self._bc(y, blk.branch7x7x3_3)
        self._bc(y, blk.branch7x7x3_4, out=out.slice(320, 192))
        self.pool(x, 3, 2, 0, _lib.EB_POOL_MAX, out=out.slice(512, x.c))
        return out

    def _inc_e(self, x, blk):
        out = self.eng.tensor(x.h, x.w, 2048)
        self._bc(x, blk.branch1x1, out=out.slice(0, 320))
        y = self._bc(x, blk.branch3x3_1)
        self._bc(y, blk.branch3x3_2a, out=out.slice(320, 384))
        self._bc(y, blk.branch3x3_2b, out=out.slice(704, 384))
        y = self._bc(x, blk.branch3x3dbl_1)
        y = self._bc(y, blk.branch3x3dbl_2)
        self._bc(y, blk.branch3x3dbl_3a, out=out.slice(1088, 384))
        self._bc(y, blk.branch3x3dbl_3b, out=out.slice(1472, 384))
        self._bc(self._avg3(x), blk.branch_pool, out=out.slice(1856, 192))
        return out


def stem_of(arch: str, model: nn.Module):
    """(conv, bn) of the architecture's first layer when it is the shared
    conv7x7/s2 + BN + ReLU stem of the ResNet / ResNeXt / DenseNet families."""
    if arch.startswith("resnet") or arch.startswith("resnext"):
        return model.conv1, model.bn1
    if arch.startswith("densenet"):
        return model.features.conv0, model.features.norm0
    return None


def grouped_stem(eng: Engine, image: TRef, stems) -> list[TRef]:
    """One launch for the identical stems of several members (north star: "where members
    share an input layout, their first layers run as a grouped launch"): their folded
    weights are concatenated along Cout, the output is one NHWC tensor, and member i
    reads its channel slice.  Runs before the lanes fork."""
    ws, bs, couts = [], [], []
    c0 = stems[0][0]
    for conv, bn in stems:
        w, b = fold_bn(conv.weight.detach().float(), None, bn)
        ws.append(w)
        bs.append(b)
        couts.append(conv.out_channels)
    w = torch.cat(ws, 0)
    b = torch.cat(bs, 0)
    kh, kw = c0.kernel_size
    sh, sw = c0.stride
    ph, pw = c0.padding
    ho = (image.h + 2 * ph - kh) // sh + 1
    wo = (image.w + 2 * pw - kw) // sw + 1
    out = eng.tensor(ho, wo, sum(couts))
    meta = {"name": "conv", "flops": 2 * ho * wo * sum(couts) * w.shape[1] * kh * kw,
            "shape": (ho, wo, sum(couts), kh, kw, sh, image.c), "weight_bytes": 2 * w[0].numel() * len(w),
            "grouped_members": len(stems)}
    eng.op(_lib.EB_OP_CONV, image, out, cout=sum(couts), kh=kh, kw=kw, sh=sh, sw=sw, ph=ph, pw=pw,
           relu=True, lane=0,
           w_off=eng.weight(pack_conv_weight_f32(w, cin_pad=image.c) if eng.f32 else
                            pack_conv_weight(w, conv_mode(kh, kw, sh, sw, ph, pw, 8, True))),
           b_off=eng.weight(b.contiguous()), meta=meta, prefork=True)
    slices, off = [], 0
    for c in couts:
        slices.append(out.slice(off, c))
        off += c
    return slices


def lower(eng: Engine, arch: str, model: nn.Module, logits: TRef, lane: int,
          image: TRef | None = None, stem_out: TRef | None = None) -> None:
    """Declare the ops of one member; its logits land in ``logits`` (fp32 slice).

    ``image`` is the member's K1 input (the engine image, or a resized copy when the
    member's native resolution differs from the request's).
    """
    lw = Lowering(eng, lane)
    x = image if image is not None else eng.image
    if arch.startswith("resnet") or arch.startswith("resnext"):
        lw.resnet(model, x, logits, stem_out)
    elif arch.startswith("densenet"):
        lw.densenet(model, x, logits, stem_out)
    elif arch.startswith("vgg"):
        lw.vgg(model, x, logits)
    elif arch == "inception_v3":
        lw.inception(model, x, logits)
    else:
        raise ValueError(f"unsupported arch {arch!r}")


def packed_parameter_bytes(model: nn.Module) -> int:
    """Device bytes of the member: bf16 conv/linear weights + fp32 biases / BN affines."""
    total = 0
    for mod in model.modules():
        if isinstance(mod, (nn.Conv2d, nn.Linear)):
            total += 2 * mod.weight.numel() + 4 * mod.weight.shape[0]
        elif isinstance(mod, nn.BatchNorm2d):
            total += 8 * mod.num_features
    return total


def resized_image(eng: Engine, size: tuple[int, int], cache: dict) -> TRef:
    """The K1 image at another resolution (bilinear, align_corners=False), shared by
    every member of that native size."""
    if (eng.H, eng.W) == tuple(size):
        return eng.image
    if size not in cache:
        t = eng.tensor(size[0], size[1], 8)
        eng.op(_lib.EB_OP_RESIZE, eng.image, t, lane=0, meta={"name": "resize"})
        cache[size] = t
    return cache[size]
