"""GPU parity of the LIN1 path (Track R): the B200 forward against the reference's
own outputs (golden vectors) and its own test cases, through the drop-in API."""

from __future__ import annotations

import json
import threading
from pathlib import Path

import numpy as np
import pytest

from helpers import build, lin1_doc
from oracle import lin1 as O
from paper_2003_01538_b200 import ensemble as E
from paper_2003_01538_b200 import models as M
from paper_2003_01538_b200 import policy as P
from paper_2003_01538_b200.errors import BadK, BatchTooLarge, EmptyBatch, PolicyUnavailable, ShapeMismatch

pytestmark = pytest.mark.gpu
GOLD = json.loads((Path(__file__).parent / "golden" / "reference_lin1.json").read_text())


def batch(values, dims=None):
    arr = np.asarray(values, dtype=np.float32)
    if arr.ndim == 1:
        arr = arr.reshape(1, -1)
    return M.SampleBatch(M.InputShape(tuple(dims) if dims else (arr.shape[1],)), arr)


@pytest.mark.parametrize("rec", GOLD["forward"], ids=lambda r: f"{r['case']}-b{r['batch']}")
def test_forward_matches_reference_goldens(tmp_path, rec):
    k = 2 if rec["classes"] == "binary" else rec["classes"]
    labels = ["absent", "present"] if k == 2 else [f"class_{i}" for i in range(k)]
    d = int(np.prod(rec["shape"]))
    docs = []
    for s in rec["seeds"]:
        w, b = O.gen_model_arrays(s, k, d)
        docs.append(lin1_doc(f"m{s}", rec["shape"], labels, w, b))
    ens = build(tmp_path, docs, mean=rec["mean"], std=rec["std"])
    x = O.unit_floats(rec["x_seed"], rec["batch"] * d).reshape(rec["batch"], d)
    out = E.forward(ens, M.SampleBatch(ens.shared_shape, x))
    assert [list(r) for r in out.per_model] == rec["labels"]


def test_known_answers_identity_swapped_tie(tmp_path):
    ens = build(tmp_path, [lin1_doc("m1"), lin1_doc("m2", weights=((0, 1), (1, 0)))])
    out = E.forward(ens, batch([[0.2, 0.9], [0.5, 0.5]]))
    assert out.per_model == ((1, 0), (0, 0))
    _, comb, _ = E.predict(ens, batch([[0.2, 0.9]]), policy=P.SensitivityPolicy("any"))
    assert comb == [1]


def test_three_class_dot_product(tmp_path):
    ens = build(tmp_path, [lin1_doc(labels=("a", "b", "c"), weights=((1, 2), (3, 4), (0, 0)),
                                    bias=(0, 0, 1))])
    assert E.forward(ens, batch([1.0, 1.0])).per_model == ((1,),)


def test_preprocess_bitwise(tmp_path):
    out = M.preprocess(batch(np.arange(12), dims=(3, 2, 2)), M.PreprocessSpec((0.0, 1.0, 2.0), (1.0, 1.0, 1.0)))
    assert out.data[0].tolist() == GOLD["known"]["preprocess_12"]
    rng = np.random.default_rng(0)
    x = rng.random((5, 3 * 7 * 9), dtype=np.float32)
    spec = M.PreprocessSpec((0.485, 0.456, 0.406), (0.229, 0.224, 0.225))
    got = M.preprocess(batch(x, dims=(3, 7, 9)), spec).data
    ref = O.preprocess(x, 3, spec.mean, spec.std)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_linear_predict_tie_break_totality():
    rng = np.random.default_rng(3)
    for _ in range(50):
        k = int(rng.integers(2, 7))
        logits = (rng.integers(-64, 65, size=k) / 16.0).astype(np.float32)
        for pos in rng.choice(k, size=int(rng.integers(0, 3)), replace=False):
            logits[pos] = logits.max()
        m = M.LinearModel("probe", M.InputShape((k,)), tuple(f"c{i}" for i in range(k)),
                          np.eye(k, dtype=np.float32), np.zeros(k, np.float32))
        assert M.linear_predict(m, batch(logits)) == [int(np.argmax(logits))]


def test_every_batch_size_and_errors(tmp_path):
    ens = build(tmp_path, [lin1_doc("m1"), lin1_doc("m2", weights=((0, 1), (1, 0)))], max_batch=16)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((16, 2)).astype(np.float32)
    for b in range(1, 17):
        out = E.forward(ens, batch(x[:b]))
        assert out.batch_size == b
        assert list(out.per_model[0]) == np.argmax(x[:b], axis=1).tolist()
    with pytest.raises(BatchTooLarge):
        E.forward(ens, batch(np.zeros((17, 2))))
    with pytest.raises(EmptyBatch):
        E.forward(ens, M.SampleBatch(M.InputShape((2,)), np.zeros((0, 2), np.float32)))
    with pytest.raises(ShapeMismatch):
        E.forward(ens, batch([[1.0, 2.0, 3.0]]))
    with pytest.raises(BadK):
        E.predict(ens, batch(x[:2]), policy=P.SensitivityPolicy("at_least", 3))


def test_batch_equals_concatenated_singles_at_full_size(tmp_path):
    d = 3 * 224 * 224
    docs = []
    for s in (11, 13, 14):
        w, b = O.gen_model_arrays(s, 2, d)
        docs.append(lin1_doc(f"m{s}", (3, 224, 224), ("absent", "present"), w, b))
    ens = build(tmp_path, docs, mean=(0.485, 0.456, 0.406), std=(0.229, 0.224, 0.225))
    x = O.unit_floats(77, 6 * d).reshape(6, d)
    full = E.forward(ens, M.SampleBatch(ens.shared_shape, x))
    singles = [E.forward(ens, M.SampleBatch(ens.shared_shape, x[i:i + 1])) for i in range(6)]
    for mi in range(3):
        assert list(full.per_model[mi]) == [s.per_model[mi][0] for s in singles]
    ref = O.forward([O.gen_model_arrays(s, 2, d) for s in (11, 13, 14)], x, 3,
                    (0.485, 0.456, 0.406), (0.229, 0.224, 0.225))
    assert [list(r) for r in full.per_model] == ref


def test_single_preprocess_invocation_for_any_n(tmp_path):
    docs = [lin1_doc(f"m{i}") for i in range(5)]
    ens = build(tmp_path, docs)
    before = M.preprocess_call_count()
    E.forward(ens, batch([[0.1, 0.2]]))
    assert M.preprocess_call_count() == before + 1


def test_policy_truth_tables_fused_and_standalone(tmp_path):
    for rec in GOLD["policy"]:
        votes = np.asarray(rec["votes"]).reshape(-1, 1)
        assert P.apply_policy(P.SensitivityPolicy("any"), votes) == [rec["any"]]
        assert P.apply_policy(P.SensitivityPolicy("all"), votes) == [rec["all"]]
        for k, want in enumerate(rec["at_least"], start=1):
            assert P.apply_policy(P.SensitivityPolicy("at_least", k), votes) == [want]
    # fused: N=3 identity/swapped members produce a vote matrix; K5 combines on device
    docs = [lin1_doc("a"), lin1_doc("b", weights=((0, 1), (1, 0))), lin1_doc("c")]
    ens = build(tmp_path, docs)
    x = np.asarray([[0.2, 0.9], [0.9, 0.2]], np.float32)
    out, comb, _ = E.predict(ens, batch(x), policy=P.SensitivityPolicy("at_least", 2))
    votes = np.asarray(out.per_model)
    assert comb == O.apply_policy("at_least", 2, votes)


def test_policy_unavailable_on_non_binary(tmp_path):
    ens = build(tmp_path, [lin1_doc(labels=("a", "b"))])
    with pytest.raises(PolicyUnavailable):
        E.predict(ens, batch([[0.1, 0.2]]), policy=P.SensitivityPolicy("any"))


def test_concurrent_forward_equals_sequential(tmp_path):
    d = 64
    docs = []
    for s in (1, 2, 3):
        w, b = O.gen_model_arrays(s, 4, d)
        docs.append(lin1_doc(f"m{s}", (d,), [f"c{i}" for i in range(4)], w, b))
    ens = build(tmp_path, docs)
    xs = [O.unit_floats(100 + i, (1 + i % 7) * d).reshape(-1, d) for i in range(32)]
    seq = [E.forward(ens, batch(x)).per_model for x in xs]
    got = [None] * len(xs)

    def work(i):
        got[i] = E.forward(ens, batch(xs[i])).per_model

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(xs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert got == seq


def test_lin1_logits_returned(tmp_path):
    """want_logits returns every member's scores: LIN1 members' fp64 scores narrowed to
    fp32 (eg/models.py:275-278 computes them in fp64), CNN members' fp32 logits."""
    d, k = 3 * 4 * 4, 3
    members = [O.gen_model_arrays(s, k, d) for s in (41, 42)]
    docs = [lin1_doc(f"m{i}", (3, 4, 4), ("a", "b", "c"), w, b) for i, (w, b) in enumerate(members)]
    mean, std = (0.1, 0.2, 0.3), (0.5, 1.0, 2.0)
    ens = build(tmp_path, docs, mean=mean, std=std)
    x = O.unit_floats(77, 6 * d).reshape(6, d)
    _, _, res = E.predict(ens, M.SampleBatch(ens.shared_shape, x), want_logits=True)
    xp = O.preprocess(x, 3, mean, std)
    for i, (w, b) in enumerate(members):
        want = O.linear_scores(xp, w, b).astype(np.float32)
        np.testing.assert_allclose(res["logits"][i, :, :k], want, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_mixed_lin1_and_cnn_members(tmp_path, precision):
    """An ensemble mixing the reference's LIN1 kind with a CNN member (same [3, 224, 224]
    shape, as the reference's uniform-shape rule requires): one forward evaluates both;
    each member's labels equal those of an ensemble holding it alone."""
    from helpers import IMAGENET_MEAN, IMAGENET_STD, cnn1_doc, write_manifest

    d = 3 * 224 * 224
    w, b = O.gen_model_arrays(61, 4, d)
    lin = lin1_doc("lin", (3, 224, 224), ("a", "b", "c", "d"), w, b)
    cnn = cnn1_doc("r18", "resnet18", 1)
    x = O.unit_floats(62, 5 * d).reshape(5, d)

    def run(docs, sub):
        sub.mkdir()
        mp = write_manifest(sub, docs, max_batch=8, mean=IMAGENET_MEAN, std=IMAGENET_STD)
        ens = E.load_ensemble(E.load_manifest_file(mp), precision=precision)
        return E.forward(ens, M.SampleBatch(ens.shared_shape, x)).per_model

    both = run([lin, cnn], tmp_path / "both")
    assert both[0] == run([lin], tmp_path / "lin")[0]
    assert both[1] == run([cnn], tmp_path / "cnn")[0]
    assert list(both[0]) == O.forward([(w, b)], x, 3, IMAGENET_MEAN, IMAGENET_STD)[0]
