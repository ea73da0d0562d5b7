import json, sys, tempfile
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import cnn as OC
from paper_2003_01538_b200 import ensemble as E, synth, _lib
from paper_2003_01538_b200.engine import TRef
mean, std = (0.485, 0.456, 0.406), (0.229, 0.224, 0.225)
td = Path(tempfile.mkdtemp())
docs = [{"format": "cnn1", "id": "m0", "arch": "resnet18", "seed": 6, "input_shape": [3, 224, 224], "labels": 1000},
        {"format": "cnn1", "id": "m1", "arch": "resnet34", "seed": 5, "input_shape": [3, 299, 299], "labels": 1000}]
entries = []
for d in docs:
    (td / f"{d['id']}.json").write_text(json.dumps(d)); entries.append({"id": d["id"], "path": f"{d['id']}.json"})
(td / "m.json").write_text(json.dumps({"memory_budget_bytes": 1 << 40, "max_batch": 4,
    "preprocess": {"mean": list(mean), "std": list(std), "pixel_scale": 255.0}, "models": entries}))
ens = E.load_ensemble(E.load_manifest_file(td / "m.json"))
eng = E.engine_for(ens)
px = synth.images(1, 299, 299, 3, seed0=1234)
_, _, res = E.predict_u8(ens, px, want_logits=True)
torch.cuda.synchronize()
img = eng.tensor_view(eng.image, 1).float().cpu()
x = OC.preprocess_u8(px, mean, std).permute(0, 2, 3, 1)
print("image err", (img[..., :3] - x).abs().max().item(), "pad max", img[..., 3:].abs().max().item())
# tensor 2 onward: find the resized one
for op in eng.op_meta[:3]: print(op)
rz = eng.tensor_view(TRef(3, 0, 8, 224, 224, 8), 1).float().cpu()
xr = OC.resize(x.permute(0, 3, 1, 2), 224).permute(0, 2, 3, 1)
print("resized err", (rz[..., :3] - xr).abs().max().item(), rz.abs().max().item())
# stem conv output of member 0 vs torch on the GPU's own resized image
from paper_2003_01538_b200.zoo import build_torch_model
from paper_2003_01538_b200.packing import fold_bn
m = build_torch_model("resnet18", 6)
w, b = fold_bn(m.conv1.weight, None, m.bn1)
stem_dst = eng.op_meta[1]["dst"]
out = eng.tensor_view(TRef(stem_dst, 0, 64, 112, 112, 64), 1).float().cpu()
ref = torch.relu(torch.nn.functional.conv2d(rz[..., :3].permute(0, 3, 1, 2), w.to(torch.bfloat16).float(), b, stride=2, padding=3)).permute(0, 2, 3, 1)
print("stem err", (out - ref).abs().max().item(), "ref max", ref.abs().max().item(), "out max", out.abs().max().item())
bad = ((out - ref).abs() > 0.1).nonzero()
print("bad", bad.shape[0], bad[:8].tolist())
