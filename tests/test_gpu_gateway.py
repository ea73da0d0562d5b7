"""GPU: the reference's unchanged REST gateway, with the seam installed, answers
byte-for-byte like the reference itself (config 3's endpoint path)."""

from __future__ import annotations

import base64
import concurrent.futures as cf
import json
import threading
import urllib.request
from pathlib import Path

import numpy as np
import pytest

from helpers import IMAGENET_MEAN, IMAGENET_STD, cnn1_doc, lin1_doc, write_manifest
from oracle import lin1 as O
from reference_import import import_reference

eg = import_reference()
pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).parent / "golden"


@pytest.fixture(autouse=True)
def _reference_present():
    # these tests serve the reference's own GatewayApp: its absence is a failure, not a
    # skip (__graft_entry__.build() installs it under baseline/_ref, which travels)
    if eg is None:
        pytest.fail("the reference package is not importable (baseline/_ref missing): "
                    "run __graft_entry__.build() in the build container")


def _requests(d, rng):
    from ensemblegate.wire import encode_request, f32le_sample

    reqs = []
    for b in (1, 2, 5, 16):
        x = rng.standard_normal((b, d)).astype(np.float32)
        reqs.append(encode_request([f32le_sample(r, (d,)) for r in x]))
        reqs.append(encode_request([f32le_sample(r, (d,)) for r in x], {"kind": "any"}))
        reqs.append(encode_request([f32le_sample(r, (d,)) for r in x], {"kind": "at_least", "k": 2}))
        reqs.append(encode_request([f32le_sample(r, (d,)) for r in x], {"kind": "at_least", "k": 9}))
    reqs.append(encode_request([f32le_sample(np.zeros(d + 1), (d + 1,))]))  # shape mismatch
    reqs.append(b'{"samples": []}')
    reqs.append(encode_request([f32le_sample(np.zeros(d), (d,))] * 17))  # > max_batch
    return reqs


def _ensemble_docs(d, binary=True):
    docs = []
    for s in (31, 32, 33):
        w, b = O.gen_model_arrays(s, 2 if binary else 4, d)
        labels = ("absent", "present") if binary else ("a", "b", "c", "d")
        docs.append(lin1_doc(f"m{s}", (d,), labels, w, b))
    return docs


@pytest.mark.parametrize("binary", [True, False])
def test_gateway_bytes_match_reference(tmp_path, binary):
    from ensemblegate.gateway import GatewayApp

    from paper_2003_01538_b200 import seam

    d = 96
    mp = write_manifest(tmp_path, _ensemble_docs(d, binary), max_batch=16)
    reqs = _requests(d, np.random.default_rng(4))
    ref_app = GatewayApp(eg.load_ensemble(eg.load_manifest_file(mp)))
    expected = [ref_app.handle("POST", "/v1/predict", r) for r in reqs]
    seam.install()
    try:
        app = GatewayApp(eg.gateway.load_ensemble(eg.load_manifest_file(mp)))
        got = [app.handle("POST", "/v1/predict", r) for r in reqs]
        assert got == expected
        assert app.handle("GET", "/v1/models") == ref_app.handle("GET", "/v1/models")
    finally:
        seam.uninstall()


def test_known_answer_body(tmp_path):
    from ensemblegate.gateway import GatewayApp
    from ensemblegate.wire import encode_request, f32le_sample

    from paper_2003_01538_b200 import seam

    mp = write_manifest(tmp_path, [lin1_doc()])
    seam.install()
    try:
        app = GatewayApp(eg.gateway.load_ensemble(eg.load_manifest_file(mp)))
        body = encode_request([f32le_sample([0.2, 0.9], (2,)), f32le_sample([0.9, 0.2], (2,))])
        assert app.handle("POST", "/v1/predict", body) == (
            200, b'{"_batch_size":2,"m1":["present","absent"]}')
    finally:
        seam.uninstall()


def test_live_server_concurrent_equals_sequential(tmp_path):
    from ensemblegate.gateway import GatewayApp, GatewayServer

    from paper_2003_01538_b200 import seam

    d = 64
    mp = write_manifest(tmp_path, _ensemble_docs(d), max_batch=16)
    reqs = _requests(d, np.random.default_rng(9))[:16]
    seam.install()
    try:
        app = GatewayApp(eg.gateway.load_ensemble(eg.load_manifest_file(mp)))
        seq = [app.handle("POST", "/v1/predict", r) for r in reqs]
        server = GatewayServer(("127.0.0.1", 0), app, 8)
        t = threading.Thread(target=server.serve_forever, kwargs={"poll_interval": 0.05}, daemon=True)
        t.start()
        url = f"http://127.0.0.1:{server.port}/v1/predict"

        def post(body):
            req = urllib.request.Request(url, data=body, method="POST",
                                         headers={"Content-Type": "application/json"})
            try:
                with urllib.request.urlopen(req, timeout=30) as r:
                    return r.status, r.read()
            except urllib.error.HTTPError as e:
                return e.code, e.read()

        with cf.ThreadPoolExecutor(8) as ex:
            got = list(ex.map(post, reqs * 2))
        server.shutdown()
        t.join(5)
        server.server_close()
        assert got == seq * 2
    finally:
        seam.uninstall()


def test_cnn_ensemble_through_endpoint(tmp_path):
    """A cnn1 ensemble served by the reference gateway (f32le RGB samples)."""
    from ensemblegate.gateway import GatewayApp
    from ensemblegate.wire import encode_request, f32le_sample

    from paper_2003_01538_b200 import ensemble as E
    from paper_2003_01538_b200 import seam, synth

    mp = write_manifest(tmp_path, [cnn1_doc("r18", "resnet18", 1)], max_batch=8,
                        mean=IMAGENET_MEAN, std=IMAGENET_STD)
    px = synth.images(3, 224, 224, 3, seed0=77)
    f32 = px.transpose(0, 3, 1, 2).astype(np.float32) / np.float32(255.0)
    seam.install()
    try:
        ens = eg.gateway.load_ensemble(eg.load_manifest_file(mp))
        app = GatewayApp(ens)
        body = encode_request([f32le_sample(x.reshape(-1), (3, 224, 224)) for x in f32])
        status, out = app.handle("POST", "/v1/predict", body)
        assert status == 200
        labels = json.loads(out)["r18"]
        res, _, _ = E.predict_u8(ens, px)
        assert labels == [ens.models[0].labels[i] for i in res.per_model[0]]
    finally:
        seam.uninstall()


def test_gateway_bytes_match_frozen_reference_output(tmp_path):
    """The seam-served gateway against the reference's response bytes frozen by
    oracle/gen_golden.py --gateway (tests/golden/gateway_bytes.json)."""
    from ensemblegate.gateway import GatewayApp

    from paper_2003_01538_b200 import seam

    gold = json.loads((GOLDEN / "gateway_bytes.json").read_text())
    seam.install()
    try:
        for case in gold["cases"]:
            sub = tmp_path / f"b{int(case['binary'])}"
            sub.mkdir()
            mp = write_manifest(sub, _ensemble_docs(case["d"], case["binary"]),
                                max_batch=case["max_batch"])
            app = GatewayApp(eg.gateway.load_ensemble(eg.load_manifest_file(mp)))
            for req, (status, body) in zip(case["requests"], case["responses"]):
                got = app.handle("POST", "/v1/predict", base64.b64decode(req))
                assert got == (status, body.encode()), (status, body[:200])
            st, body = case["models"]
            assert app.handle("GET", "/v1/models") == (st, body.encode())
    finally:
        seam.uninstall()


def test_pgm_requests_bytes_match_reference(tmp_path):
    """Grayscale [1, H, W] ensembles take "pgm" samples (eg/wire.py:60-72); with the seam
    they go through the native decoder (P5 parsed as eg/pgm.py does) -- same bytes as the
    reference's own gateway, including its errors for malformed documents."""
    from ensemblegate.gateway import GatewayApp

    from paper_2003_01538_b200 import seam

    h, w = 6, 9
    docs = []
    for s in (51, 52):
        wt, b = O.gen_model_arrays(s, 2, h * w)
        docs.append(lin1_doc(f"g{s}", (1, h, w), ("absent", "present"), wt, b))
    mp = write_manifest(tmp_path, docs, max_batch=16, mean=(0.5,), std=(0.25,), pixel_scale=200.0)
    rng = np.random.default_rng(8)

    def body(docs_):
        return json.dumps({"samples": [{"encoding": "pgm", "data": base64.b64encode(d).decode()}
                                       for d in docs_]}).encode()

    good = [b"P5\n%d %d\n255\n" % (w, h) + rng.integers(0, 256, h * w, dtype=np.uint8).tobytes()
            for _ in range(12)]
    reqs = [body(good[:b]) for b in (1, 3, 12)]
    reqs.append(body([b"P5\n%d %d\n9\n" % (w, h) + bytes([10] * (h * w))]))  # pixel > maxval
    reqs.append(body([b"P5\n%d %d\n255\n" % (w + 1, h) + bytes((w + 1) * h)]))  # other shape
    ref_app = GatewayApp(eg.load_ensemble(eg.load_manifest_file(mp)))
    expected = [ref_app.handle("POST", "/v1/predict", r) for r in reqs]
    assert [e[0] for e in expected[:3]] == [200, 200, 200]
    seam.install()
    try:
        app = GatewayApp(eg.gateway.load_ensemble(eg.load_manifest_file(mp)))
        assert [app.handle("POST", "/v1/predict", r) for r in reqs] == expected
    finally:
        seam.uninstall()
