"""GPU: execution contexts (engine.ContextPool, eb_engine_clone) and the batch-size
bucketed graph cache (runtime.cu bucket_of).

The reference re-enters forward concurrently from its gateway worker threads on one
shared ensemble (eg/gateway.py:222-257; tests/test_gateway.py:360-372) and requires the
responses to equal a sequential replay (tests/test_acceptance.py:208-238)."""

from __future__ import annotations

import concurrent.futures as cf

import numpy as np
import pytest

from helpers import IMAGENET_MEAN, IMAGENET_STD, cnn1_doc, write_manifest
from paper_2003_01538_b200 import _lib
from paper_2003_01538_b200 import ensemble as E
from paper_2003_01538_b200 import synth
from paper_2003_01538_b200.engine import ContextPool

pytestmark = pytest.mark.gpu


def _ens(tmp_path, contexts, max_batch=48):
    docs = [cnn1_doc("r18", "resnet18", 1), cnn1_doc("d121", "densenet121", 2)]
    mp = write_manifest(tmp_path, docs, max_batch=max_batch, mean=IMAGENET_MEAN, std=IMAGENET_STD)
    return E.load_ensemble(E.load_manifest_file(mp), contexts=contexts)


def test_concurrent_contexts_equal_sequential(tmp_path):
    ens = _ens(tmp_path, contexts=3)
    eng = E.engine_for(ens)
    assert isinstance(eng, ContextPool) and len(eng.contexts) == 3
    sizes = [1, 5, 17, 33, 48, 2, 9, 40, 3, 21, 48, 12]
    reqs = [synth.images(b, 224, 224, 3, seed0=1000 + 50 * i) for i, b in enumerate(sizes)]
    seq = [E.predict_u8(ens, x, topk=3, want_logits=True)[2] for x in reqs]
    with cf.ThreadPoolExecutor(8) as ex:
        par = list(ex.map(lambda x: E.predict_u8(ens, x, topk=3, want_logits=True)[2], reqs * 2))
    for a, b in zip(seq * 2, par):
        for k in ("labels", "logits", "topk_idx"):
            assert np.array_equal(a[k], b[k]), k


def test_bucketed_graphs_equal_exact_sizes(tmp_path):
    """A batch of B runs through the graph of its bucket (e.g. 33 -> 48): its rows are
    bitwise those of the same samples evaluated alone, and warmup pre-captures every
    bucket so no request pays a capture."""
    ens = _ens(tmp_path, contexts=1)
    eng = E.engine_for(ens)
    eng.warmup(_lib.EB_IN_U8_HWC)
    px = synth.images(48, 224, 224, 3, seed0=31)
    _, _, full = E.predict_u8(ens, px, want_logits=True)
    for b in (9, 17, 33, 47):
        _, _, part = E.predict_u8(ens, px[:b], want_logits=True)
        assert np.array_equal(part["logits"], full["logits"][:, :b]), b
    for i in (0, 30):
        _, _, one = E.predict_u8(ens, px[i:i + 1], want_logits=True)
        assert np.array_equal(one["logits"][:, 0], full["logits"][:, i])
