"""CPU: the native f32le request decoder (F1) returns exactly what the reference's
decode_request returns, and declines everything else (so errors stay the reference's)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from reference_import import import_reference

eg = import_reference()
pytestmark = pytest.mark.skipif(eg is None, reason="reference package not importable")


def _check_same(body, dims, max_batch=64):
    from ensemblegate.wire import decode_request

    from paper_2003_01538_b200.wire import fast_decode

    got = fast_decode(body, dims, max_batch, pinned=False)
    assert got is not None
    ref_batch, ref_policy = decode_request(body)
    assert np.array_equal(got[0].view(np.uint32), ref_batch.data.view(np.uint32))
    if ref_policy is None:
        assert got[1] is None
    else:
        assert eg.parse_policy(json.loads(got[1])) == ref_policy


@pytest.mark.parametrize("dims,b", [((2,), 1), ((6,), 5), ((3, 8, 8), 7), ((3, 224, 224), 3)])
def test_matches_reference_decode(dims, b):
    from ensemblegate.wire import encode_request, f32le_sample

    rng = np.random.default_rng(b)
    x = rng.standard_normal((b, int(np.prod(dims)))).astype(np.float32)
    _check_same(encode_request([f32le_sample(r, dims) for r in x]), dims)
    _check_same(encode_request([f32le_sample(r, dims) for r in x], {"kind": "at_least", "k": 2}), dims)


def test_whitespace_and_key_order():
    from ensemblegate.wire import f32le_sample

    s = f32le_sample([1.5, -2.0], (2,))
    body = ('{ "policy" : {"kind":"any"} ,\n "samples": [ {"shape": [ 2 ], "data": "%s",'
            ' "encoding":"f32le"} ] }' % s["data"]).encode()
    _check_same(body, (2,))


@pytest.mark.parametrize("body", [
    b'{"samples": []}',
    b'{"samples": [{"encoding": "pgm", "data": "UDUKMSAxCjI1NQoA"}]}',
    b'{"samples": [{"encoding": "f32le", "shape": [2], "data": "AAAA"}]}',
    b'{"samples": [{"encoding": "f32le", "shape": [3], "data": "AACAPwAAAEA="}]}',
    b'{"samples": [{"encoding": "f32le", "shape": [2], "data": "AACAPwAAAEA=", "x": 1}]}',
    b'{"samples": [{"encoding": "f32le", "shape": [2], "data": "AACAPwAAgH8="}]}',  # inf
    b'{"samples": [{"encoding": "f32le", "shape": [2], "data": "AACAPwAA\\nAEA="}]}',
    b'{"samples": [], "samples": []}',
    b'{"extra": 1, "samples": [{"encoding": "f32le", "shape": [2], "data": "AACAPwAAAEA="}]}',
    b'not json',
    # leading zeros / negative zero in a shape: the reference's strict JSON decides
    b'{"samples": [{"encoding": "f32le", "shape": [02], "data": "AACAPwAAAEA="}]}',
    b'{"samples": [{"encoding": "f32le", "shape": [002], "data": "AACAPwAAAEA="}]}',
    b'{"samples": [{"encoding": "f32le", "shape": [-0], "data": "AACAPwAAAEA="}]}',
])
def test_declines_everything_else(body):
    from paper_2003_01538_b200.wire import fast_decode

    assert fast_decode(body, (2,), 8, pinned=False) is None


def test_decode_speed_64_rgb():
    import time

    from ensemblegate.wire import encode_request, f32le_sample

    from paper_2003_01538_b200.wire import fast_decode

    x = np.random.default_rng(0).random((64, 3 * 224 * 224), dtype=np.float32)
    body = encode_request([f32le_sample(r, (3, 224, 224)) for r in x])
    t = time.perf_counter()
    got = fast_decode(body, (3, 224, 224), 64, pinned=False)
    dt = time.perf_counter() - t
    assert got is not None and np.array_equal(got[0], x)
    assert dt < 0.5, dt  # the reference takes ~0.4 s on 8 cores for this body


def _pgm_body(docs):
    import base64

    return json.dumps({"samples": [{"encoding": "pgm", "data": base64.b64encode(d).decode()}
                                   for d in docs]}).encode()


def _p5(h, w, px, maxval=255, header=None):
    head = header if header is not None else f"P5\n{w} {h}\n{maxval}\n".encode()
    return head + bytes(px)


@pytest.mark.parametrize("scale", [255.0, 100.0, 7.0])
def test_pgm_matches_reference_decode(scale):
    """eg/wire.py:60-72 + eg/pgm.py:16-59: P5 raster / pixel_scale, shape [1, H, W]."""
    from ensemblegate.wire import decode_request

    from paper_2003_01538_b200.wire import fast_decode

    rng = np.random.default_rng(3)
    docs = [_p5(5, 7, rng.integers(0, 256, 35, dtype=np.uint8)) for _ in range(4)]
    docs.append(_p5(5, 7, rng.integers(0, 100, 35, dtype=np.uint8), maxval=99))
    docs.append(_p5(5, 7, [3] * 35, header=b"P5 \t7\r\n5\x0b\x0c255 "))  # any header whitespace
    docs.append(_p5(5, 7, [9] * 35, header=b"P5\n007 05\n0255\n"))  # leading zeros: int() accepts
    body = _pgm_body(docs)
    got = fast_decode(body, (1, 5, 7), 16, pinned=False, pixel_scale=scale)
    assert got is not None
    ref, _ = decode_request(body, pixel_scale=scale)
    assert np.array_equal(got[0].view(np.uint32), ref.data.view(np.uint32))
    # without a pixel scale (the f32le-only entry point) pgm is declined
    assert fast_decode(body, (1, 5, 7), 16, pinned=False) is None


@pytest.mark.parametrize("doc", [
    b"P2\n7 5\n255\n" + bytes(35),               # ASCII PGM
    b"P5\n7 5\n0\n" + bytes(35),                 # maxval 0
    b"P5\n7 5\n256\n" + bytes(35),               # maxval > 255
    b"P5\n7 5\n10\n" + bytes([11] * 35),         # pixel > maxval
    b"P5\n7 5\n255\n\n" + bytes(35),             # two whitespace bytes before the raster
    b"P5\n7 5\n255\n" + bytes(34),               # short raster
    b"P5\n7 5\n255" + bytes(35),                 # no separator
    b"P5\n+7 5\n255\n" + bytes(35),              # non-digit token
    b"P5\n7 6\n255\n" + bytes(42),               # other shape than the ensemble's
    b"P5\n7 5\n255\n",                           # no raster
])
def test_pgm_declines_what_the_reference_rejects(doc):
    from paper_2003_01538_b200.wire import fast_decode

    assert fast_decode(_pgm_body([doc]), (1, 5, 7), 16, pinned=False, pixel_scale=255.0) is None


@pytest.mark.parametrize("with_policy", [False, True])
def test_native_render_matches_reference_bytes(with_policy):
    """F4: eb_render_prediction == dumps_canonical(render_prediction(...)) byte for byte,
    including label escaping (quotes, backslashes, control and non-ASCII characters) and
    key order around the reserved "_batch_size" / "_combined" keys."""
    from types import SimpleNamespace

    from ensemblegate.jsonio import dumps_canonical
    from ensemblegate.wire import render_prediction

    from paper_2003_01538_b200.wire import Renderer

    labels_a = ("absent", "present")
    labels_b = ('say "hi"', "back\\slash", "tab\there", "café", "\U0001f600", "ctl\x01", "plain")
    models = [SimpleNamespace(id=i, labels=l) for i, l in
              (("zeta", labels_b), ("A1", labels_a), ("m.2", labels_b), ("_x"[1:], labels_a))]
    ens = SimpleNamespace(models=tuple(models))
    rng = np.random.default_rng(5)
    r = Renderer(ens)
    for b in (1, 3, 40):
        idx = np.stack([rng.integers(0, len(m.labels), b) for m in models]).astype(np.int32)
        out = SimpleNamespace(batch_size=b, per_model=tuple(tuple(int(v) for v in row) for row in idx))
        comb = [int(v) for v in rng.integers(0, 2, b)] if with_policy else None
        assert r.render(idx, comb) == dumps_canonical(render_prediction(ens, out, comb))
