"""Fixture builders for the parity tests (mirror the reference's tests/conftest.py builders)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def lin1_doc(model_id="m1", input_shape=(2,), labels=("absent", "present"),
             weights=((1.0, 0.0), (0.0, 1.0)), bias=(0.0, 0.0)) -> dict:
    return {"format": "lin1", "id": model_id, "input_shape": list(input_shape),
            "labels": list(labels), "weights": [list(map(float, r)) for r in np.asarray(weights)],
            "bias": list(map(float, bias))}


def cnn1_doc(model_id, arch, seed, size=224, labels=1000) -> dict:
    return {"format": "cnn1", "id": model_id, "arch": arch, "seed": seed,
            "input_shape": [3, size, size], "labels": labels}


def write_manifest(tmp: Path, docs, budget=10**12, max_batch=64, mean=(0.0,), std=(1.0,),
                   pixel_scale=255.0) -> Path:
    entries = []
    for i, doc in enumerate(docs):
        p = tmp / f"model_{i}_{doc['id']}.json"
        p.write_text(json.dumps(doc))
        entries.append({"id": doc["id"], "path": p.name})
    man = {"memory_budget_bytes": budget, "max_batch": max_batch,
           "preprocess": {"mean": list(mean), "std": list(std), "pixel_scale": pixel_scale},
           "models": entries}
    mp = tmp / "manifest.json"
    mp.write_text(json.dumps(man))
    return mp


def build(tmp: Path, docs, **kw):
    from paper_2003_01538_b200 import ensemble as E

    return E.load_ensemble(E.load_manifest_file(write_manifest(tmp, docs, **kw)))
