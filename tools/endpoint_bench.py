"""Config 3: flexible-batching stream through the unchanged reference gateway.

Starts the reference's own `GatewayServer` (baseline/_ref or /root/reference) with
the seam installed and the C2 ensemble (ResNet-50 + DenseNet-121 + VGG-16), then
POSTs requests whose batch sizes are uniform in 1..MAX (SplitMix64, seed 2003) at
concurrency 1 and 8, and reports p50/p99 latency (nearest rank, as
`eg/flexctl.py:268-273`) next to the device time of the same batches.

The load generator runs in separate processes (one per concurrent client), each of
which builds its request bodies from per-sample JSON fragments prepared before timing
(as `flexctl` builds payloads before timing, eg/flexctl.py:321-326), so client-side
encoding never competes with the server for the GIL.  The server keeps the
reference's worker-thread pool; the engine has `--contexts` execution contexts
(engine.ContextPool) and every batch-size bucket's graph is captured before the run.

    python tools/endpoint_bench.py [--requests 200] [--max-batch 512] [--contexts 4]
"""

from __future__ import annotations

import argparse
import base64
import concurrent.futures as cf
import json
import math
import multiprocessing as mp
import sys
import tempfile
import threading
import time
import urllib.request
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def nearest_rank(values, q):
    v = sorted(values)
    return v[max(0, math.ceil(q / 100.0 * len(v)) - 1)]


_FRAGS: list = []
_URL = ""


def _client_init(url: str, max_batch: int) -> None:
    """Per client process: the f32le JSON fragment of every sample of the pool."""
    global _FRAGS, _URL
    from paper_2003_01538_b200 import synth

    _URL = url
    pool = synth.images_fast(max_batch, 224, 224, 3, seed0=99).transpose(0, 3, 1, 2)
    pool = (pool.astype(np.float32) / np.float32(255.0)).reshape(max_batch, -1)
    _FRAGS = [('{"encoding":"f32le","shape":[3,224,224],"data":"%s"}'
               % base64.b64encode(pool[i].astype("<f4").tobytes()).decode()).encode()
              for i in range(max_batch)]


def _post(b: int):
    data = b'{"samples":[' + b",".join(_FRAGS[:b]) + b"]}"
    req = urllib.request.Request(_URL, data=data, method="POST",
                                 headers={"Content-Type": "application/json"})
    t0 = time.perf_counter()
    with urllib.request.urlopen(req, timeout=600) as r:
        body = r.read()
        ok = r.status == 200
    return (time.perf_counter() - t0) * 1e3, ok, len(json.loads(body).get("resnet50", [])) == b


def main():
    from reference_import import import_reference

    eg = import_reference()
    if eg is None:
        print(json.dumps({"unavailable": "reference package not installed (baseline/_ref)"}))
        return
    from ensemblegate.gateway import GatewayApp, GatewayServer

    import bench
    from paper_2003_01538_b200 import _lib, seam, synth
    from paper_2003_01538_b200.ensemble import engine_for

    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=200)
    ap.add_argument("--max-batch", type=int, default=512)
    ap.add_argument("--contexts", type=int, default=4)
    ap.add_argument("--concurrency", type=int, nargs="*", default=[1, 8])
    a = ap.parse_args()

    import os

    os.environ["EB_CONTEXTS"] = str(a.contexts)
    seam.install()
    td = Path(tempfile.mkdtemp(prefix="c3_"))
    entries = []
    for doc in bench.cnn_docs():
        (td / f"{doc['id']}.json").write_text(json.dumps(doc))
        entries.append({"id": doc["id"], "path": f"{doc['id']}.json"})
    (td / "m.json").write_text(json.dumps({
        "memory_budget_bytes": 1 << 40, "max_batch": a.max_batch,
        "preprocess": {"mean": list(bench.MEAN), "std": list(bench.STD), "pixel_scale": 255.0},
        "models": entries}))
    ens = eg.gateway.load_ensemble(eg.load_manifest_file(td / "m.json"))
    eng = engine_for(ens)
    t0 = time.perf_counter()
    eng.warmup(_lib.EB_IN_F32_CHW)  # every bucket's graph, every context
    warm_s = time.perf_counter() - t0
    app = GatewayApp(ens)
    server = GatewayServer(("127.0.0.1", 0), app, max(a.concurrency))
    t = threading.Thread(target=server.serve_forever, kwargs={"poll_interval": 0.05}, daemon=True)
    t.start()
    url = f"http://127.0.0.1:{server.port}/v1/predict"

    sizes = [int(z % a.max_batch) + 1 for z in synth.splitmix64(2003, a.requests)]

    # device time of the same batch sizes (resident input, CUDA events, bucketed graphs)
    import torch

    ctx0 = getattr(eng, "contexts", [eng])[0]
    stream = torch.cuda.ExternalStream(ctx0.stream())
    dev = {}
    for b in sorted(set(sizes)):
        ctx0.forward_device(b, _lib.EB_IN_F32_CHW)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            s0.record(stream)
        ctx0.forward_device(b, _lib.EB_IN_F32_CHW)
        with torch.cuda.stream(stream):
            s1.record(stream)
        torch.cuda.synchronize()
        dev[b] = s0.elapsed_time(s1)
    out = {"config": "C3: C2 ensemble behind the unchanged ensemblegate GatewayServer (seam), "
                     "f32le samples (the reference's wire encoding)",
           "requests": a.requests, "batch_sizes": "uniform 1..%d (SplitMix64 seed 2003)" % a.max_batch,
           "mean_batch": float(np.mean(sizes)), "contexts": a.contexts,
           "graph_warmup_s": warm_s,
           "device_ms": {"p50": nearest_rank([dev[b] for b in sizes], 50),
                         "p99": nearest_rank([dev[b] for b in sizes], 99)},
           "latency": "client wall clock per request (nearest rank), bodies built before timing"}
    ctx = mp.get_context("spawn")
    for c in a.concurrency:
        with cf.ProcessPoolExecutor(c, mp_context=ctx, initializer=_client_init,
                                    initargs=(url, a.max_batch)) as ex:
            list(ex.map(_post, [1] * c))  # warm-up, one per client
            t0 = time.perf_counter()
            res = list(ex.map(_post, sizes))
            wall = time.perf_counter() - t0
        lat = [r[0] for r in res]
        out[f"concurrency_{c}"] = {"p50_ms": nearest_rank(lat, 50), "p99_ms": nearest_rank(lat, 99),
                                   "images_per_s": sum(sizes) / wall,
                                   "failed": sum(not (r[1] and r[2]) for r in res)}
    server.shutdown()
    t.join(5)
    server.server_close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
