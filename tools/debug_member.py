"""Compare one CNN member's GPU logits with the live CPU oracle (debug helper).

    python tools/debug_member.py ARCH SEED [--request-size S] [--batch B]
"""
import argparse
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import cnn as OC  # noqa: E402
from paper_2003_01538_b200 import ensemble as E  # noqa: E402
from paper_2003_01538_b200 import synth  # noqa: E402
from paper_2003_01538_b200.zoo import NATIVE_SIZE, build_torch_model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("arch")
ap.add_argument("seed", type=int)
ap.add_argument("--request-size", type=int, default=0)
ap.add_argument("--batch", type=int, default=2)
ap.add_argument("--extra", default="", help="second member arch:seed (forces a mixed ensemble)")
a = ap.parse_args()
mean, std = (0.485, 0.456, 0.406), (0.229, 0.224, 0.225)
native = NATIVE_SIZE.get(a.arch, 224)
req = a.request_size or native
td = Path(tempfile.mkdtemp())
docs = [{"format": "cnn1", "id": "m0", "arch": a.arch, "seed": a.seed, "input_shape": [3, native, native], "labels": 1000}]
if a.extra:
    ea, es = a.extra.split(":")
    docs.append({"format": "cnn1", "id": "m1", "arch": ea, "seed": int(es),
                 "input_shape": [3, req, req], "labels": 1000})
entries = []
for d in docs:
    (td / f"{d['id']}.json").write_text(json.dumps(d))
    entries.append({"id": d["id"], "path": f"{d['id']}.json"})
(td / "m.json").write_text(json.dumps({"memory_budget_bytes": 1 << 40, "max_batch": 8,
                                       "preprocess": {"mean": list(mean), "std": list(std), "pixel_scale": 255.0},
                                       "models": entries}))
ens = E.load_ensemble(E.load_manifest_file(td / "m.json"))
px = synth.images(a.batch, req, req, 3, seed0=1234)
_, _, res = E.predict_u8(ens, px, want_logits=True)
x = OC.preprocess_u8(px, mean, std)
if native != req:
    x = OC.resize(x, native)
ref = OC.logits(build_torch_model(a.arch, a.seed), x)
got = res["logits"][0, :, :1000]
print("ref absmax", np.abs(ref).max(), "got absmax", np.nanmax(np.abs(got)), "nan", np.isnan(got).sum())
print("max rel err", np.nanmax(np.abs(got - ref)) / np.abs(ref).max())
print("top1 ref", ref.argmax(-1), "got", got.argmax(-1))
bad = np.argwhere(np.abs(got - ref) > 0.05 * np.abs(ref).max())
print("bad entries", len(bad), bad[:10].tolist())
if a.extra:
    g1 = res["logits"][1, :, :1000]
    print("member1 absmax", np.nanmax(np.abs(g1)))
