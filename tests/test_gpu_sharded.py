"""GPU: the single-process sharded forward (load_ensemble(..., devices=...),
shard.ShardedEngine) equals the single-GPU forward bitwise.  The round-end box has one
GPU, so both replicas live on device 0 -- the host logic (contiguous shards, one thread
and stream per replica, reassembly in shard order) is the same as on 8 devices."""

from __future__ import annotations

import numpy as np
import pytest

from helpers import IMAGENET_MEAN, IMAGENET_STD, cnn1_doc, write_manifest
from paper_2003_01538_b200 import ensemble as E
from paper_2003_01538_b200 import synth
from paper_2003_01538_b200.policy import SensitivityPolicy

pytestmark = pytest.mark.gpu


def test_sharded_equals_single_gpu_bitwise(tmp_path):
    docs = [cnn1_doc("r18", "resnet18", 1, labels=["absent", "present"]),
            cnn1_doc("d121", "densenet121", 2, labels=["absent", "present"])]
    mp = write_manifest(tmp_path, docs, max_batch=16, mean=IMAGENET_MEAN, std=IMAGENET_STD)
    one = E.load_ensemble(E.load_manifest_file(mp))
    two = E.load_ensemble(E.load_manifest_file(mp), devices=(0, 0))
    assert two.devices == (0, 0) and two.max_batch == 16
    eng = E.engine_for(two)
    assert [e.max_batch for e in eng.engines] == [8, 8]
    px = synth.images(16, 224, 224, 3, seed0=55)
    for b in (1, 7, 16):
        o1, c1, r1 = E.predict_u8(one, px[:b], policy=SensitivityPolicy("at_least", 2), topk=2,
                                  want_logits=True)
        o2, c2, r2 = E.predict_u8(two, px[:b], policy=SensitivityPolicy("at_least", 2), topk=2,
                                  want_logits=True)
        assert o1 == o2 and c1 == c2
        for k in ("labels", "logits", "topk_idx", "topk_prob"):
            assert np.array_equal(r1[k], r2[k]), (b, k)
    with pytest.raises(E.errors.BatchTooLarge):
        E.predict_u8(two, synth.images(17, 224, 224, 3, seed0=1))
