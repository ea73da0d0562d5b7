"""The fused grouped stem + max-pools (csrc/stem_pool.cu: the 7x7/2 stem shared by two
members and both members' 3x3/2 max-pools in one kernel, the 112 x 112 stem output never
written) computes bitwise what the unfused launches compute -- same MMA order, same
rounding, max exact in any order.  Compared through whole ResNet-50 + DenseNet-121 members
(logits) at batch sizes below the fusion threshold and with 7- and 14-row bands."""

from __future__ import annotations

import os

import numpy as np
import pytest

from helpers import IMAGENET_MEAN, IMAGENET_STD, build, cnn1_doc
from paper_2003_01538_b200 import _lib
from paper_2003_01538_b200 import ensemble as E
from paper_2003_01538_b200 import synth
from paper_2003_01538_b200.ensemble import engine_for

pytestmark = pytest.mark.gpu


def _ensemble(tmp_path, fused: bool, name: str):
    old = os.environ.get("EB_STEM_POOL")
    os.environ["EB_STEM_POOL"] = "1" if fused else "0"
    try:
        d = tmp_path / name
        d.mkdir()
        ens = build(d, [cnn1_doc("resnet50_3", "resnet50", 3), cnn1_doc("densenet121_2", "densenet121", 2)],
                    max_batch=160, mean=IMAGENET_MEAN, std=IMAGENET_STD)
        engine_for(ens)  # finalized (and the fusion decided) while EB_STEM_POOL is set
        return ens
    finally:
        if old is None:
            os.environ.pop("EB_STEM_POOL")
        else:
            os.environ["EB_STEM_POOL"] = old


def test_fused_stem_pools_bitwise_equal_unfused(tmp_path):
    fused = _ensemble(tmp_path, True, "fused")
    plain = _ensemble(tmp_path, False, "plain")
    px = synth.images_fast(160, 224, 224, 3, seed0=9090)
    for b in (4, 19, 40, 129, 160):  # unfused below ~19 images; 7- and 14-row bands
        _, _, f = E.predict_u8(fused, px[:b], topk=5, want_logits=True)
        _, _, u = E.predict_u8(plain, px[:b], topk=5, want_logits=True)
        assert np.array_equal(f["logits"], u["logits"]), f"B={b}: fused stem + pools differ"
        assert np.array_equal(f["topk_idx"], u["topk_idx"])
    for ens in (fused, plain):
        E.predict_u8(ens, px[:64])
    ef, eu = engine_for(fused), engine_for(plain)
    # one stem launch either way; the two pool launches are gone
    assert ef.launch_count(_lib.EB_IN_U8_HWC, 64) == eu.launch_count(_lib.EB_IN_U8_HWC, 64) - 2
    assert ef.launch_count(_lib.EB_IN_U8_HWC, 4) == eu.launch_count(_lib.EB_IN_U8_HWC, 4)


def test_fusions_bitwise_in_the_c5_mix(tmp_path):
    """C5's mix (ResNet-152 + DenseNet-201 share a fused stem + pools, ResNeXt-50's own stem
    + pool is fused too, VGG-19 runs the fused block 1, Inception-v3 at 299 stays unfused) with both fusions on
    and off: the same logits, bit for bit, at a batch where both fusions run."""
    docs = [cnn1_doc("resnet152_6", "resnet152", 6), cnn1_doc("densenet201_7", "densenet201", 7),
            cnn1_doc("vgg19_8", "vgg19", 8), cnn1_doc("inception_v3_5", "inception_v3", 5, size=299),
            cnn1_doc("resnext50_32x4d_9", "resnext50_32x4d", 9)]
    ens = {}
    for flag in ("1", "0"):
        saved = {k: os.environ.get(k) for k in ("EB_STEM_POOL", "EB_BLOCK1")}
        os.environ["EB_STEM_POOL"] = os.environ["EB_BLOCK1"] = flag
        try:
            d = tmp_path / f"c5_{flag}"
            d.mkdir()
            ens[flag] = build(d, docs, max_batch=32, mean=IMAGENET_MEAN, std=IMAGENET_STD)
            engine_for(ens[flag])
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    px = synth.images_fast(32, 299, 299, 3, seed0=5151)
    _, _, f = E.predict_u8(ens["1"], px, topk=5, want_logits=True)
    _, _, u = E.predict_u8(ens["0"], px, topk=5, want_logits=True)
    assert np.array_equal(f["logits"], u["logits"])
    kind = _lib.EB_IN_U8_HWC
    # the fused C5 step: three pools (the grouped pair's two, ResNeXt's own) and one VGG conv fewer
    assert engine_for(ens["1"]).launch_count(kind, 32) == engine_for(ens["0"]).launch_count(kind, 32) - 4


def test_single_member_stem_pool_bitwise(tmp_path):
    """A lone ResNet-50 (its own 64-channel stem, no grouped launch) with the stem + pool
    fusion on and off."""
    ens = {}
    for flag in ("1", "0"):
        saved = os.environ.get("EB_STEM_POOL")
        os.environ["EB_STEM_POOL"] = flag
        try:
            d = tmp_path / f"r50_{flag}"
            d.mkdir()
            ens[flag] = build(d, [cnn1_doc("resnet50_3", "resnet50", 3)], max_batch=64, mean=IMAGENET_MEAN,
                              std=IMAGENET_STD)
            engine_for(ens[flag])
        finally:
            if saved is None:
                os.environ.pop("EB_STEM_POOL", None)
            else:
                os.environ["EB_STEM_POOL"] = saved
    px = synth.images_fast(64, 224, 224, 3, seed0=6262)
    for b in (4, 40, 64):
        _, _, f = E.predict_u8(ens["1"], px[:b], topk=5, want_logits=True)
        _, _, u = E.predict_u8(ens["0"], px[:b], topk=5, want_logits=True)
        assert np.array_equal(f["logits"], u["logits"]), f"B={b}"
    kind = _lib.EB_IN_U8_HWC
    assert engine_for(ens["1"]).launch_count(kind, 64) == engine_for(ens["0"]).launch_count(kind, 64) - 1
