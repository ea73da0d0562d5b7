"""Generate the committed golden fixtures under tests/golden/ (build container only).

    PYTHONPATH=/root/reference/pkg/src python -m oracle.gen_golden --lin1
    python -m oracle.gen_golden --gateway
    python -m oracle.gen_golden --cnn

--lin1 imports the reference itself (/root/reference, read-only) and records
its outputs: SplitMix64 streams, gen_model arrays, forward labels for seeded
ensembles, known answers from the reference's own tests, policy truth tables.
--cnn records torchvision fp32 CPU logits (oracle.cnn) for the CNN configs.
"""

from __future__ import annotations

import argparse
import hashlib
import itertools
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_lin1() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    import ensemblegate as eg  # the reference, read-only
    from ensemblegate import fixtures as fx
    from ensemblegate.models import parse_model_file

    out: dict = {"reference": "ensemblegate " + eg.__version__, "splitmix64": {}, "gen_model": [],
                 "forward": [], "known": {}, "policy": []}
    for seed in (0, 1, 1234, 2**63 + 5):
        s = fx.splitmix64(seed)
        out["splitmix64"][str(seed)] = [str(next(s)) for _ in range(8)]
    # gen_model arrays (small ones verbatim, large ones by digest)
    for seed, shape, classes in [(100, (6,), "binary"), (101, (6,), "binary"), (7, (3, 4, 4), 3),
                                 (11, (3, 224, 224), "binary"), (12, (3, 224, 224), 10)]:
        m = parse_model_file(fx.gen_model(seed, shape, classes, f"g{seed}"))
        rec = {"seed": seed, "shape": list(shape), "classes": classes,
               "sha_w": _sha(m.weights), "sha_b": _sha(m.bias)}
        if m.weights.size <= 64:
            rec["weights"] = m.weights.tolist()
            rec["bias"] = m.bias.tolist()
        out["gen_model"].append(rec)
    # forward on seeded ensembles (reference forward, eg/ensemble.py:232-250)
    cases = [
        dict(name="bin6_n3", seeds=[100, 101, 102], shape=(6,), classes="binary", mean=(0.0,),
             std=(1.0,), batches=[1, 3, 8, 64]),
        dict(name="k3_chw", seeds=[7, 8], shape=(3, 4, 4), classes=3, mean=(0.1, 0.2, 0.3),
             std=(0.5, 1.0, 2.0), batches=[1, 5]),
        dict(name="rgb224_bin_n3", seeds=[11, 13, 14], shape=(3, 224, 224), classes="binary",
             mean=IMAGENET_MEAN, std=IMAGENET_STD, batches=[4]),
        dict(name="rgb224_k10", seeds=[12], shape=(3, 224, 224), classes=10,
             mean=IMAGENET_MEAN, std=IMAGENET_STD, batches=[3]),
    ]
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        for case in cases:
            paths = []
            for s in case["seeds"]:
                p = td / f"{case['name']}_{s}.json"
                p.write_bytes(fx.gen_model(s, case["shape"], case["classes"], f"m{s}"))
                paths.append(p)
            man = td / f"{case['name']}_manifest.json"
            man.write_bytes(fx.gen_manifest(paths, budget=10**10, max_batch=64, out_dir=td,
                                            mean=case["mean"], std=case["std"]))
            ens = eg.load_ensemble(eg.load_manifest_file(man))
            d = int(np.prod(case["shape"]))
            for bi, b in enumerate(case["batches"]):
                seed = 5000 + bi
                x = (np.asarray(list(itertools.islice(fx.unit_floats(seed), b * d)),
                                dtype=np.float32).reshape(b, d))
                res = eg.forward(ens, eg.SampleBatch(eg.InputShape(tuple(case["shape"])), x))
                out["forward"].append({"case": case["name"], "seeds": case["seeds"],
                                       "shape": list(case["shape"]), "classes": case["classes"],
                                       "mean": list(case["mean"]), "std": list(case["std"]),
                                       "x_seed": seed, "batch": b,
                                       "labels": [list(r) for r in res.per_model]})
    # known answers lifted from the reference's own tests (run through the reference)
    ident = eg.LinearModel("m1", eg.InputShape((2,)), ("absent", "present"),
                           np.eye(2, dtype=np.float32), np.zeros(2, np.float32))
    sw = eg.LinearModel("m2", eg.InputShape((2,)), ("absent", "present"),
                        np.array([[0, 1], [1, 0]], np.float32), np.zeros(2, np.float32))
    b2 = lambda v: eg.SampleBatch(eg.InputShape((2,)), np.asarray([v], np.float32))  # noqa: E731
    three = eg.LinearModel("m3", eg.InputShape((2,)), ("a", "b", "c"),
                           np.array([[1, 2], [3, 4], [0, 0]], np.float32),
                           np.array([0, 0, 1], np.float32))
    out["known"] = {
        "identity_0.2_0.9": eg.linear_predict(ident, b2([0.2, 0.9])),
        "identity_tie_0.5_0.5": eg.linear_predict(ident, b2([0.5, 0.5])),
        "swapped_0.2_0.9": eg.linear_predict(sw, b2([0.2, 0.9])),
        "three_class_1_1": eg.linear_predict(three, b2([1.0, 1.0])),
        "preprocess_12": eg.preprocess(
            eg.SampleBatch(eg.InputShape((3, 2, 2)), np.arange(12, dtype=np.float32)[None]),
            eg.PreprocessSpec((0.0, 1.0, 2.0), (1.0, 1.0, 1.0))).data[0].tolist(),
    }
    for n in range(1, 5):
        for votes in itertools.product((0, 1), repeat=n):
            v = np.asarray(votes, dtype=np.int64).reshape(n, 1)
            rec = {"votes": list(votes),
                   "any": eg.apply_policy(eg.SensitivityPolicy("any"), v)[0],
                   "all": eg.apply_policy(eg.SensitivityPolicy("all"), v)[0],
                   "at_least": [eg.apply_policy(eg.SensitivityPolicy("at_least", k), v)[0]
                                for k in range(1, n + 1)]}
            out["policy"].append(rec)
    GOLDEN.mkdir(parents=True, exist_ok=True)
    (GOLDEN / "reference_lin1.json").write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", GOLDEN / "reference_lin1.json")


CNN_SETS = {
    # name: (members [(arch, seed)], batch, size)
    "c1": ([("resnet18", 1), ("densenet121", 2)], 32, 224),
    "c2": ([("resnet50", 3), ("densenet121", 2), ("vgg16", 4)], 32, 224),
    "inception": ([("inception_v3", 5)], 32, 299),
    # config 5: requests at 299 (the largest member); 224 members see a bilinear resize
    "c5": ([("resnet152", 6), ("densenet201", 7), ("vgg19", 8), ("inception_v3", 5),
            ("resnext50_32x4d", 9)], 32, 299),
    "resnext": ([("resnext50_32x4d", 9)], 32, 224),
}
# the bench workload itself (bench.py: C2, B = 256, synth.images_fast(256, seed0=1234)):
# oracle logits of four of its rows
BENCH_ROWS = (0, 127, 128, 255)


def gen_cnn(names) -> None:
    import torch

    from oracle import cnn
    from paper_2003_01538_b200 import synth
    from paper_2003_01538_b200.zoo import NATIVE_SIZE, build_torch_model

    cnn.set_threads()
    for name in names:
        if name == "c2_bench":
            members, size = CNN_SETS["c2"][0], 224
            px = synth.images_fast(256, 224, 224, 3, seed0=1234)[list(BENCH_ROWS)]
        else:
            members, b, size = CNN_SETS[name]
            px = synth.images(b, size, size, 3, seed0=1234, kind="structured")
        x = cnn.preprocess_u8(px, IMAGENET_MEAN, IMAGENET_STD, 255.0)
        logits = []
        for arch, seed in members:
            model = build_torch_model(arch, seed)
            native = NATIVE_SIZE.get(arch, 224)
            xm = x if native == size else cnn.resize(x, native)
            logits.append(cnn.logits(model, xm))
            del model
        arr = np.stack(logits).astype(np.float32)
        np.savez_compressed(GOLDEN / f"cnn_{name}.npz", logits=arr,
                            archs=np.array([a for a, _ in members]),
                            seeds=np.array([s for _, s in members]),
                            size=size, batch=len(px), seed0=1234, torch=torch.__version__,
                            rows=np.array(BENCH_ROWS if name == "c2_bench" else range(len(px))))
        print("wrote", name, arr.shape, "distinct top1 per member",
              [len(set(r.tolist())) for r in arr.argmax(-1)])


def gen_gateway() -> None:
    """Response bytes of the reference's own GatewayApp (eg/gateway.py:76-142) for the
    request sets of tests/test_gpu_gateway.py, frozen so the GPU tests compare the seam
    against the reference's output even where only its gateway code is importable."""
    import base64

    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, str(ROOT / "tests"))
    import ensemblegate as eg
    from ensemblegate.gateway import GatewayApp
    from test_gpu_gateway import _ensemble_docs, _requests

    from helpers import write_manifest

    out = {"reference": "ensemblegate " + eg.__version__, "cases": []}
    for binary in (True, False):
        with tempfile.TemporaryDirectory() as td:
            d = 96
            mp = write_manifest(Path(td), _ensemble_docs(d, binary), max_batch=16)
            reqs = _requests(d, np.random.default_rng(4))
            app = GatewayApp(eg.load_ensemble(eg.load_manifest_file(mp)))
            resp = [app.handle("POST", "/v1/predict", r) for r in reqs]
            models = app.handle("GET", "/v1/models")
        out["cases"].append({
            "binary": binary, "d": d, "max_batch": 16,
            "requests": [base64.b64encode(r).decode() for r in reqs],
            "responses": [[st, body.decode()] for st, body in resp],
            "models": [models[0], models[1].decode()]})
    (GOLDEN / "gateway_bytes.json").write_text(json.dumps(out, indent=0) + "\n")
    print("wrote", GOLDEN / "gateway_bytes.json")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--lin1", action="store_true")
    ap.add_argument("--cnn", nargs="*")
    ap.add_argument("--gateway", action="store_true")
    a = ap.parse_args()
    sys.path.insert(0, str(ROOT))
    if a.lin1:
        gen_lin1()
    if a.gateway:
        gen_gateway()
    if a.cnn is not None:
        gen_cnn(a.cnn or list(CNN_SETS) + ["c2_bench"])
