"""The fused VGG block 1 (csrc/block1.cu: conv1_1 + conv1_2 + pool1 in one kernel, the
64-channel intermediate kept in shared memory) computes bitwise what the unfused pair
computes (the stem rows-mode conv, then the taps-in-N conv with its fused max-pool) --
same MMA K order, same fp32 bias / tap / pool order, same rounding.  Compared through the
whole VGG-16 member (logits), at batch sizes that select each band height (28 / 56 / 112
rows) and strip counts that do not divide the grid, and below the fusion threshold."""

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
    old = os.environ.get("EB_BLOCK1")
    os.environ["EB_BLOCK1"] = "1" if fused else "0"
    try:
        d = tmp_path / name
        d.mkdir()
        ens = build(d, [cnn1_doc("vgg16_4", "vgg16", 4)], max_batch=160, mean=IMAGENET_MEAN,
                    std=IMAGENET_STD)
        engine_for(ens)  # finalized (and the fusion decided) while EB_BLOCK1 is set
        return ens
    finally:
        if old is None:
            os.environ.pop("EB_BLOCK1")
        else:
            os.environ["EB_BLOCK1"] = old


def test_fused_block1_bitwise_equals_unfused(tmp_path):
    fused = _ensemble(tmp_path, True, "fused")
    plain = _ensemble(tmp_path, False, "plain")
    px = synth.images_fast(160, 224, 224, 3, seed0=8080)
    for b in (4, 12, 40, 129, 160):  # unfused below ~10 images; band heights 28 / 56 / 112
        _, _, f = E.predict_u8(fused, px[:b], topk=5, want_logits=True)
        _, _, u = E.predict_u8(plain, px[:b], topk=5, want_logits=True)
        assert np.array_equal(f["logits"], u["logits"]), f"B={b}: fused block 1 differs"
        assert np.array_equal(f["topk_idx"], u["topk_idx"])
    # the fused path is the one that ran: one launch fewer per forward (no conv1_1)
    for ens in (fused, plain):
        E.predict_u8(ens, px[:64])
    ef, eu = engine_for(fused), engine_for(plain)
    assert ef.launch_count(_lib.EB_IN_U8_HWC, 64) == eu.launch_count(_lib.EB_IN_U8_HWC, 64) - 1
    assert ef.launch_count(_lib.EB_IN_U8_HWC, 4) == eu.launch_count(_lib.EB_IN_U8_HWC, 4)
