"""A sample's result does not depend on the batch it arrives in (GPU).

The reference pins this for its own member kind: a batch equals its concatenated
single-sample forwards, bitwise (eg/models.py:273-274, /root/reference/pkg/tests/
test_ensemble.py:250-264) and internal parallelism must not change
values.  For CNN members that means every choice that changes the
order in which a layer's K dimension is summed (split-K count, tall vs plain
taps-in-N) is a function of the layer shape only (runtime.cu plan_conv), so the
logits -- not only the labels -- must be bitwise equal for every B, and for a
sample at any position of its batch.
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import IMAGENET_MEAN, IMAGENET_STD, build, cnn1_doc
from paper_2003_01538_b200 import ensemble as E
from paper_2003_01538_b200 import synth

pytestmark = pytest.mark.gpu

CONFIGS = {
    "c1": [("resnet18", 1), ("densenet121", 2)],
    "c2": [("resnet50", 3), ("densenet121", 2), ("vgg16", 4)],
}


@pytest.mark.parametrize("name", ["c2", "c1"])
def test_logits_bitwise_independent_of_batch(tmp_path, name):
    docs = [cnn1_doc(f"{a}_{s}", a, s) for a, s in CONFIGS[name]]
    ens = build(tmp_path, docs, max_batch=256, mean=IMAGENET_MEAN, std=IMAGENET_STD)
    px = synth.images_fast(256, 224, 224, 3, seed0=4242)
    _, _, full = E.predict_u8(ens, px, topk=5, want_logits=True)
    ref = full["logits"]
    checked = 0
    # prefixes (B = 1, 7, 128, 129: every tile-count / split-K / 2-SM boundary of C2)
    for b in (1, 7, 128, 129):
        _, _, part = E.predict_u8(ens, px[:b], topk=5, want_logits=True)
        assert np.array_equal(part["logits"], ref[:, :b]), f"B={b}: logits differ from B=256"
        assert np.array_equal(part["labels"], full["labels"][:, :b])
        assert np.array_equal(part["topk_idx"], full["topk_idx"][:, :b])
        checked += b
    # the same samples at other positions of a smaller batch, and singly
    for lo, hi in ((100, 107), (250, 256)):
        _, _, part = E.predict_u8(ens, px[lo:hi], want_logits=True)
        assert np.array_equal(part["logits"], ref[:, lo:hi]), f"rows {lo}:{hi} moved to 0: differ"
    for i in (0, 127, 128, 255):
        _, _, one = E.predict_u8(ens, px[i:i + 1], want_logits=True)
        assert np.array_equal(one["logits"][:, 0], ref[:, i]), f"sample {i} alone differs"
    print(f"{name}: {checked} prefix samples + 13 moved/single samples bitwise equal to B=256")
