"""CPU: the host-side mirror agrees with the reference's own loader semantics, and the
seam rebinds the reference's forward path (no device work here)."""

from __future__ import annotations

import json

import numpy as np

import pytest

from helpers import cnn1_doc, lin1_doc, write_manifest
from reference_import import import_reference

eg = import_reference()
pytestmark = pytest.mark.skipif(eg is None, reason="reference package not importable")


def _load_both(tmp_path, docs, **kw):
    from paper_2003_01538_b200 import ensemble as ours

    mp = write_manifest(tmp_path, docs, **kw)
    res = []
    for mod in (eg, ours):
        try:
            e = mod.load_ensemble(mod.load_manifest_file(mp))
            res.append(("ok", e.bytes_used, e.binary_compatible, e.max_batch, tuple(e.shared_shape.dims)))
        except Exception as exc:  # noqa: BLE001
            res.append(("err", type(exc).__name__, getattr(exc, "code", None)))
    return res


CASES = {
    "identity": ([lin1_doc()], {}),
    "two_models": ([lin1_doc("m1"), lin1_doc("m2", weights=((0, 1), (1, 0)))], {}),
    "budget_boundary_fail": ([lin1_doc()], {"budget": 23}),
    "budget_boundary_ok": ([lin1_doc()], {"budget": 24}),
    "shape_disagreement": ([lin1_doc("a"), lin1_doc("b", input_shape=(3,), weights=((1, 0, 0), (0, 1, 0)))], {}),
    "non_binary": ([lin1_doc(labels=("x", "y"))], {}),
    "bad_mean_len": ([lin1_doc(input_shape=(3, 1, 1), weights=((1, 0, 0), (0, 1, 0)))], {"mean": (0.0, 1.0)}),
    "per_channel_ok": ([lin1_doc(input_shape=(3, 1, 1), weights=((1, 0, 0), (0, 1, 0)))], {"mean": (0.0, 1.0, 2.0), "std": (1.0, 1.0, 2.0)}),
}


@pytest.mark.parametrize("name", list(CASES))
def test_loader_matches_reference(tmp_path, name):
    docs, kw = CASES[name]
    ref, ours = _load_both(tmp_path, docs, **kw)
    assert ours == ref


@pytest.mark.parametrize("doc_patch", [
    {"format": "lin2"}, {"id": "_hidden"}, {"labels": ["a"]}, {"labels": ["a", "a"]},
    {"weights": [[1.0, 0.0]]}, {"bias": [0.0]}, {"extra": 1}, {"input_shape": []},
])
def test_malformed_models_rejected_like_reference(tmp_path, doc_patch):
    from paper_2003_01538_b200 import models as ours

    doc = dict(lin1_doc(), **doc_patch)
    data = json.dumps(doc).encode()
    errs = []
    for mod in (eg.models, ours):
        try:
            mod.parse_model_file(data)
            errs.append("ok")
        except Exception as exc:  # noqa: BLE001
            errs.append(getattr(exc, "code", type(exc).__name__))
    assert errs[0] == errs[1] == "malformed_model"


def test_manifest_errors_like_reference():
    from paper_2003_01538_b200 import ensemble as ours

    bad = [b"{", b"[]", b'{"models": []}',
           json.dumps({"memory_budget_bytes": 1, "max_batch": 0, "preprocess": {"mean": [0], "std": [1]},
                       "models": [{"id": "a", "path": "a"}]}).encode(),
           json.dumps({"memory_budget_bytes": 1, "max_batch": 1, "preprocess": {"mean": [0], "std": [1]},
                       "models": [{"id": "a", "path": "a"}, {"id": "a", "path": "b"}]}).encode()]
    for data in bad:
        codes = []
        for mod in (eg.ensemble, ours):
            try:
                mod.load_manifest(data)
                codes.append("ok")
            except Exception as exc:  # noqa: BLE001
                codes.append(getattr(exc, "code", type(exc).__name__))
        assert codes[0] == codes[1] == "malformed_manifest", data


def test_cnn1_member_format(tmp_path):
    from paper_2003_01538_b200 import ensemble as ours

    mp = write_manifest(tmp_path, [cnn1_doc("r18", "resnet18", 1)], budget=10**9)
    ens = ours.load_ensemble(ours.load_manifest_file(mp))
    assert ens.shared_shape.dims == (3, 224, 224)
    assert len(ens.models[0].labels) == 1000
    # budget counts the real device bytes of the packed member (bf16 weights)
    assert 2 * 11_000_000 < ens.bytes_used < 2 * 12_500_000


@pytest.mark.parametrize("order", [0, 1])
def test_mixed_lin1_cnn1_shapes_rejected_in_any_order(tmp_path, order):
    """With any LIN1 member the reference's uniform-shape rule holds for every member
    (eg/ensemble.py:202-208), whatever the manifest order."""
    from paper_2003_01538_b200 import ensemble as ours
    from paper_2003_01538_b200 import errors

    docs = [lin1_doc("l1", (3, 8, 8), weights=np.zeros((2, 192)), bias=(0.0, 0.0)),
            cnn1_doc("r18", "resnet18", 1)]
    if order:
        docs = docs[::-1]
    mp = write_manifest(tmp_path, docs, budget=10**9)
    with pytest.raises(errors.ShapeMismatch):
        ours.load_ensemble(ours.load_manifest_file(mp))


def test_install_rebinds_and_restores():
    import ensemblegate.ensemble as eg_ens
    import ensemblegate.gateway as eg_gw
    import ensemblegate.models as eg_models

    from paper_2003_01538_b200 import ensemble as ours
    from paper_2003_01538_b200 import errors as our_err
    from paper_2003_01538_b200 import seam

    before = (eg_ens.forward, eg_gw.forward, eg_models.preprocess, eg_gw.GatewayApp._predict)
    seam.install()
    try:
        assert eg_ens.forward is ours.forward and eg_gw.forward is ours.forward
        assert our_err.BatchTooLarge is eg.errors.BatchTooLarge
        assert eg_gw.load_ensemble is ours.load_ensemble
    finally:
        seam.uninstall()
    assert (eg_ens.forward, eg_gw.forward, eg_models.preprocess, eg_gw.GatewayApp._predict) == before
