#!/usr/bin/env python
"""Benchmark of the ensemble forward path (BASELINE.json metric) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): the 3-member ensemble ResNet-50 +
DenseNet-121 + VGG-16 (cnn1 members, seeded random init, bf16 tcgen05 path), one
step = one forward + combine of a batch of B = 256 synthetic 224x224 RGB u8
images per GPU (the top of the config's 1-256 range).  Under torchrun each rank
owns a full replica, evaluates its own 256-image shard and the logits are
gathered to rank 0 with NCCL inside the timed step (weak scaling).

Reported on one JSON line (rank 0):
  value      device-timed images/s, inputs resident in HBM (CUDA events on the
             engine stream, L2 flushed between steps, max over ranks)
  e2e        the same metric through the public C-ABI (eb_forward_batches) with
             pinned host input, H2D + forward + D2H of labels of every step inside the
             timing (the next step's H2D overlaps this step's forward); the one-call-
             per-step eb_forward figure is reported beside it
  roofline   the tcgen05 conv/GEMM kernel class: algorithmic FLOPs of every conv
             launch / its CUDA-event time (serialised per-op profile)
  hbm_kernels   achieved GB/s of the memory-bound kernels (K1 preprocess, K5 combine)
             against the measured HBM peak, timed alone through the kernel-level ABI
  cpu_baseline  the oracle (torchvision fp32 eager on all host cores) on a
             bounded sample of the same workload
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MEMBERS = [("resnet50", 3), ("densenet121", 2), ("vgg16", 4)]
GFLOP_PER_IMG = 44.787  # SURVEY.md §2.4 (conv + linear, 2*MAC, torchvision flop counter)
MEAN = (0.485, 0.456, 0.406)
STD = (0.229, 0.224, 0.225)
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def _event_time(fn, iters: int = 50) -> float:
    """Mean ms per call of fn() on the current stream (CUDA events, after warm-up).
    EB_PROBE_ITERS=n: n timed calls and one warm-up (short launch lists under ncu)."""
    import torch

    if os.environ.get("EB_PROBE_ITERS"):
        iters = int(os.environ["EB_PROBE_ITERS"])
    for _ in range(1 if os.environ.get("EB_PROBE_ITERS") else 5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def hbm_kernels(B: int, hbm_peak: float, src: str) -> dict:
    """Achieved HBM bandwidth of the two memory-bound kernels of the path, through the
    kernel-level C-ABI on device buffers (north_star: preprocess and combine vs HBM peak).

    K1 preprocess: u8 HWC (3 B/px) -> bf16 NHWC8 (16 B/px): 19 algorithmic bytes per pixel;
    and straight into the stem layouts (u8 read + the layout's bytes written).
    K5 combine: 3 members x 1000 fp32 logits per image read, labels + top-5 written; at the
    bench batch it is latency-bound (a few MB), so it is also reported at B = 4096 (C4).
    """
    import ctypes

    import torch

    from paper_2003_01538_b200 import _lib

    lib = _lib.load()
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    out = {}
    hw = 224 * 224
    x = torch.randint(0, 256, (B, hw * 3), dtype=torch.uint8, device="cuda")
    y = torch.empty(B * hw * 8, dtype=torch.bfloat16, device="cuda")
    lut = torch.rand(3 * 256, device="cuda")
    ms = _event_time(lambda: _lib.check(lib.eb_k_preprocess_u8_nhwc8(P(x), P(y), B, 3, hw, P(lut), None)))
    bytes_ = B * hw * (3 + 16)
    out["preprocess_k1"] = {"batch": B, "us": ms * 1e3, "bytes": bytes_, "achieved_gbs": bytes_ / ms / 1e6,
                            "frac_of_hbm": bytes_ / ms / 1e6 / hbm_peak}
    # K1 as the engine runs it for C2 (u8 request): straight into the two stem layouts
    # (VGG 3x3/s1 padded rows, the grouped 7x7/s2 stem's even/odd column planes)
    xr = x.view(B, 224, 224, 3)
    for name, (kh, st, pd) in () if not hasattr(lib, "eb_k_preprocess_u8_layout") else (("rows_3x3", (3, 1, 1)), ("planes_7x7s2", (7, 2, 3))):
        nb = ctypes.c_uint64(0)
        _lib.check(lib.eb_k_stem_layout(B, 224, 224, kh, kh, st, st, pd, pd, ctypes.byref(nb)))
        ly = torch.empty(nb.value // 2, dtype=torch.bfloat16, device="cuda")
        ms = _event_time(lambda: _lib.check(lib.eb_k_preprocess_u8_layout(
            P(xr), B, 3, 224, 224, P(lut), kh, kh, st, st, pd, pd, P(ly), None)))
        bytes_ = B * hw * 3 + nb.value
        out[f"preprocess_k1_{name}"] = {"batch": B, "us": ms * 1e3, "bytes": bytes_,
                                        "achieved_gbs": bytes_ / ms / 1e6,
                                        "frac_of_hbm": bytes_ / ms / 1e6 / hbm_peak}
        del ly
    for b in (B, 4096):
        K, n, tk = 1000, 3, 5
        l32 = torch.randn(b, n * K, device="cuda")
        l64 = torch.zeros(1, 1, dtype=torch.float64, device="cuda")
        kind = torch.zeros(n, dtype=torch.int32, device="cuda")
        koff = torch.arange(0, n * K, K, dtype=torch.int32, device="cuda")
        kcnt = torch.full((n,), K, dtype=torch.int32, device="cuda")
        lab = torch.empty(n, b, dtype=torch.int32, device="cuda")
        tki = torch.empty(n, b, tk, dtype=torch.int32, device="cuda")
        tkp = torch.empty(n, b, tk, dtype=torch.float32, device="cuda")
        comb = torch.empty(b, dtype=torch.int32, device="cuda")
        ms = _event_time(lambda: _lib.check(lib.eb_k_combine(
            P(l32), n * K, P(l64), 1, P(kind), P(koff), P(kcnt), n, b, P(lab), tk, P(tki), P(tkp), 0, 0,
            P(comb), None)))
        bytes_ = b * (n * K * 4 + n * 4 + n * tk * 8)
        out[f"combine_k5_b{b}"] = {"batch": b, "us": ms * 1e3, "bytes": bytes_,
                                   "achieved_gbs": bytes_ / ms / 1e6, "frac_of_hbm": bytes_ / ms / 1e6 / hbm_peak}
    out["peak_gbs"] = hbm_peak
    out["peak_source"] = f"{src} hbm_gbs"
    return out


def op_bounds(op_meta, ms, B: int, tc_peak_tflops: float, hbm_gbs: float) -> list:
    """Per conv/FC launch: its roofline bound max(algorithmic flops / tensor peak,
    algorithmic bytes / HBM) in ms beside its measured ms.  Bytes = the input read once
    (a stem's 3 image channels, not the 8-channel padding) + the output written once (+ the
    residual read) + the weights.  (tools/ops_roofline.py prints the breakdown.)"""
    out = []
    for m, t in zip(op_meta, ms):
        if m.get("name") != "conv":
            continue
        ho, wo, co, kh, kw, s, ci = m["shape"]
        cin = 3 if ci == 8 else ci
        nbytes = B * 2 * (ho * s * wo * s * cin + ho * wo * co * (2 if m.get("res", -1) >= 0 else 1)) \
            + m.get("weight_bytes", 0)
        t_tc = m["flops"] * B / (tc_peak_tflops * 1e12) * 1e3
        t_hbm = nbytes / (hbm_gbs * 1e9) * 1e3
        out.append({"meta": m, "ms": float(t), "tensor_ms": t_tc, "hbm_ms": t_hbm,
                    "bound_ms": max(t_tc, t_hbm), "bytes": nbytes})
    return out


def peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return dict(PEAKS_FALLBACK), "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region (NVML every ~10 ms,
    falling back to nvidia-smi when NVML is unavailable)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.sm: list[float] = []
        self.reasons: set[str] = set()
        self.sm_max = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.sm_max = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            masks = [(n, getattr(pynvml, a)) for n, a in self.REASONS]
            while not self._stop.is_set():
                self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.reasons.update(n for n, m in masks if r & m)
                self._stop.wait(0.01)
            return
        except Exception:
            pass
        while not self._stop.is_set():  # nvidia-smi fallback
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                row = [x.strip() for x in out.split(",")]
                if row and row[0].replace(".", "").isdigit():
                    self.sm.append(float(row[0]))
                    self.sm_max = float(row[1]) if row[1].replace(".", "").isdigit() else None
                    self.reasons.update(n for (n, _), v in zip(self.REASONS, row[2:]) if v.lower() == "active")
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.sm_max,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def cnn_docs(members=MEMBERS):
    """cnn1 documents of the members, each at its native input size (Inception-v3: 299;
    an ensemble mixing sizes takes requests at the largest, zoo.NATIVE_SIZE)."""
    from paper_2003_01538_b200.zoo import NATIVE_SIZE

    return [{"format": "cnn1", "id": f"{a}", "arch": a, "seed": s,
             "input_shape": [3, NATIVE_SIZE.get(a, 224), NATIVE_SIZE.get(a, 224)], "labels": 1000}
            for a, s in members]


def build_ensemble(batch: int, device: int, members=MEMBERS, precision: str = "bf16"):
    from paper_2003_01538_b200 import ensemble as E

    td = Path(tempfile.mkdtemp(prefix="bench_"))
    entries = []
    for doc in cnn_docs(members):
        (td / f"{doc['id']}.json").write_text(json.dumps(doc))
        entries.append({"id": doc["id"], "path": f"{doc['id']}.json"})
    man = {"memory_budget_bytes": 1 << 40, "max_batch": batch,
           "preprocess": {"mean": list(MEAN), "std": list(STD), "pixel_scale": 255.0},
           "models": entries}
    (td / "manifest.json").write_text(json.dumps(man))
    # one engine on this GPU, one execution context (whatever EB_DEVICES / EB_CONTEXTS say)
    return E.load_ensemble(E.load_manifest_file(td / "manifest.json"), device=device,
                           precision=precision, devices=(device,), contexts=1)


def cpu_oracle_rate(n_images: int = 64, seconds_cap: float = 25.0, chunk: int = 8) -> dict:
    """torchvision fp32 eager on all host cores, the same members and inputs, in batches
    of ``chunk`` images until ``seconds_cap``."""
    import torch

    from oracle import cnn as OC
    from paper_2003_01538_b200 import synth
    from paper_2003_01538_b200.zoo import build_torch_model

    cores = OC.set_threads()
    models = [build_torch_model(a, s) for a, s in MEMBERS]
    px = synth.images_fast(n_images, 224, 224, 3, seed0=4321)
    with torch.no_grad():
        x = OC.preprocess_u8(px[:chunk], MEAN, STD, 255.0)
        for m in models:  # warm-up
            m(x)
        t0 = time.perf_counter()
        done = 0
        while done + chunk <= n_images and time.perf_counter() - t0 < seconds_cap:
            x = OC.preprocess_u8(px[done:done + chunk], MEAN, STD, 255.0)
            logits = np.stack([m(x).numpy() for m in models])
            _ = logits.argmax(-1)
            done += chunk
        dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "images/s", "cores": cores, "kind": "port",
            "sample": f"{done} images in batches of {chunk} x {len(MEMBERS)} members, torchvision "
                      "fp32 eager (u8 -> reference fp32 preprocess -> logits -> argmax)"}


# ---------------------------------------------------------------------- Track R (LIN1)

TRACK_R = {"members": 3, "shape": (3, 224, 224), "batch": 256}


def _lin1_arrays(k: int, d: int, seed: int):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((k, d), dtype=np.float32)
    b = rng.standard_normal(k, dtype=np.float32)
    return w, b


def track_r_gpu(pk: dict, steps: int = 10) -> dict:
    """The reference's own member kind on the B200: LIN1 N = 3 at [3, 224, 224], binary and
    K = 1000, B = 256.  K1 (f32 preprocess) + K6 (fp64 scores) + K5,
    device-timed with the input resident; GB/s of the path against the HBM peak and
    K6's fp64 FLOP/s."""
    import torch

    from paper_2003_01538_b200 import _lib
    from paper_2003_01538_b200.ensemble import build_engine
    from paper_2003_01538_b200.models import InputShape, LinearModel, PreprocessSpec

    c, h, w = TRACK_R["shape"]
    d, B, n = c * h * w, TRACK_R["batch"], TRACK_R["members"]
    out = {}
    for name, k in (("binary", 2), ("k1000", 1000)):
        labels = ("absent", "present") if k == 2 else tuple(f"c{i}" for i in range(k))
        models = []
        for i in range(n):
            wt, bs = _lin1_arrays(k, d, 100 + i)
            models.append(LinearModel(f"m{i}", InputShape((c, h, w)), labels, wt, bs))
        eng = build_engine(models, InputShape((c, h, w)), PreprocessSpec(MEAN, STD, 255.0), B)
        x = np.random.default_rng(7).random((B, d), dtype=np.float32)
        eng.forward(x, _lib.EB_IN_F32_CHW)  # H2D into the engine's input buffer + warm-up
        stream = torch.cuda.ExternalStream(eng.stream())
        for _ in range(3):
            eng.forward_device(B, _lib.EB_IN_F32_CHW)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
        for _ in range(steps):
            eng.forward_device(B, _lib.EB_IN_F32_CHW)
        with torch.cuda.stream(stream):
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        # K1: x read + normalised x written; K6: normalised x + W read; bias; labels
        bytes_ = 4 * B * d * 3 + 4 * n * k * d + 4 * n * k + 4 * n * B
        flops = 2.0 * B * d * n * k
        out[name] = {"batch": B, "members": n, "K": k, "D": d, "ms": ms, "images_per_s": B / (ms / 1e3),
                     "bytes": bytes_, "achieved_gbs": bytes_ / ms / 1e6,
                     "frac_of_hbm": bytes_ / ms / 1e6 / pk["hbm_gbs"], "fp64_tflops": flops / ms / 1e9}
        eng.close()
        del eng
    out["peak_gbs"] = pk["hbm_gbs"]
    out["path"] = "K1 f32 preprocess + K6 fp64 scores (fixed d-slices) + K5 argmax, inputs resident"
    return out


def _reference_module():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "ensemblegate").is_dir() and str(p) not in sys.path:
            sys.path.append(str(p))
    try:
        import ensemblegate

        return ensemblegate, "reference"
    except ImportError:
        return None, "port"


def track_r_cpu(seconds_cap: float = 20.0) -> dict:
    """The reference's own forward (eg/ensemble.py:232-250: preprocess + fp64 einsum +
    argmax per member) on the host, same LIN1 configs; the restatement in oracle/lin1.py
    when the reference package is not importable."""
    eg, kind = _reference_module()
    from oracle import lin1 as OL

    c, h, w = TRACK_R["shape"]
    d, n = c * h * w, TRACK_R["members"]
    out = {"kind": kind, "cores": 1,
           "note": "the reference's einsum is single-threaded numpy (SURVEY.md §3.2)"}
    for name, k, b in (("binary", 2, 64), ("k1000", 1000, 2)):
        labels = ("absent", "present") if k == 2 else tuple(f"c{i}" for i in range(k))
        arrays = [_lin1_arrays(k, d, 100 + i) for i in range(n)]
        x = np.random.default_rng(7).random((b, d), dtype=np.float32)
        if eg is not None:
            shape = eg.InputShape((c, h, w))
            models = tuple(eg.LinearModel(f"m{i}", shape, labels, wt, bs) for i, (wt, bs) in enumerate(arrays))
            ens = eg.Ensemble(models, shape, eg.PreprocessSpec(MEAN, STD, 255.0),
                              sum(m.parameter_bytes for m in models), 1 << 40, b, k == 2)
            run = lambda: eg.forward(ens, eg.SampleBatch(shape, x))  # noqa: E731
        else:
            run = lambda: OL.forward(arrays, x, c, MEAN, STD)  # noqa: E731
        run()
        t0 = time.perf_counter()
        reps = 0
        while True:
            run()
            reps += 1
            if time.perf_counter() - t0 > seconds_cap / 2 or reps >= 5:
                break
        dt = (time.perf_counter() - t0) / reps
        out[name] = {"batch": b, "members": n, "K": k, "images_per_s": b / dt, "ms_per_call": dt * 1e3}
    return out


# ---------------------------------------------------------------------- reference arm


def run_reference(args) -> None:
    """The reference path's CPU implementation on the host cores (oracle port: torchvision
    fp32 eager -- the reference has no CNN code), C2's members, a bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch

    from oracle import cnn as OC
    from paper_2003_01538_b200 import synth
    from paper_2003_01538_b200.zoo import build_torch_model

    cores = OC.set_threads()
    per_step = args.ref_sample
    models = [build_torch_model(a, s) for a, s in MEMBERS]
    px = synth.images_fast(per_step, 224, 224, 3, seed0=4321)
    times = []
    with torch.no_grad():
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            x = OC.preprocess_u8(px, MEAN, STD, 255.0)
            logits = np.stack([m(x).numpy() for m in models])
            _ = np.argmax(logits, axis=-1)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
    total = sum(times)
    value = per_step * len(times) / total
    line = {
        "impl": "reference", "metric": "ensemble images/s (N-model fwd+combine)", "value": value,
        "unit": "images/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C2 ensemble resnet50+densenet121+vgg16, 224x224 RGB u8, "
                               f"{per_step} images per step (bounded CPU sample)",
                   "members": [f"{a}:seed{s}" for a, s in MEMBERS]},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "port",
                         "sample": f"{per_step} images per step through torchvision fp32 eager "
                                   "(oracle port of the path; the reference has no CNN code)"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- our arm


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) with torchrun
    and return its exit code (rank 0 prints the line)."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator / transport lines on stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py")] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def device_rate(eng, B: int, kind: int, stream, topk: int, iters: int = 10) -> float:
    """images/s of eng.forward_device(B) (+ K5 with top-k), CUDA events on the engine
    stream, after warm-up (graph captured)."""
    import torch

    for _ in range(3):
        eng.forward_device(B, kind, topk)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        s0.record(stream)
    for _ in range(iters):
        eng.forward_device(B, kind, topk)
    with torch.cuda.stream(stream):
        s1.record(stream)
    torch.cuda.synchronize()
    return B * iters / (s0.elapsed_time(s1) / 1e3)


def extra_configs(device: int) -> dict:
    """C1 (B = 8) and C5 (B = 128 per GPU, its 8-GPU shard size) on this GPU, device-timed;
    plus bs = 1 latency of each through eb_forward."""
    import torch

    from paper_2003_01538_b200 import _lib, synth
    from paper_2003_01538_b200.ensemble import engine_for

    sets = {"C1": ([("resnet18", 1), ("densenet121", 2)], 8, 224),
            "C5": ([("resnet152", 6), ("densenet201", 7), ("vgg19", 8), ("inception_v3", 5),
                    ("resnext50_32x4d", 9)], 128, 299)}
    gflop = {"C1": 9.296, "C5": 90.761}
    out = {}
    for name, (members, B, size) in sets.items():
        ens = build_ensemble(B, device, members=members)
        eng = engine_for(ens)
        stream = torch.cuda.ExternalStream(eng.stream(), device=torch.device("cuda", device))
        kind = _lib.EB_IN_U8_HWC
        px = synth.images_fast(B, size, size, 3, seed0=77)
        eng.forward(px, kind)  # resident input + graph capture
        rate = device_rate(eng, B, kind, stream, topk=5)
        lat = []
        for _ in range(20):
            t0 = time.perf_counter()
            eng.forward(px[:1], kind)
            lat.append((time.perf_counter() - t0) * 1e3)
        out[name] = {"members": [f"{a}:seed{s}" for a, s in members], "batch": B, "input": size,
                     "images_per_s": rate, "tflops": rate * gflop[name] / 1e3,
                     "latency_bs1_p50_ms": statistics.median(lat[5:])}
        eng.close()
        del eng, ens
    # the fp32-faithful parity mode (csrc/ref32.cu) on C2: how fast exact top-k costs
    B = 32
    ens = build_ensemble(B, device, precision="fp32")
    eng = engine_for(ens)
    stream = torch.cuda.ExternalStream(eng.stream(), device=torch.device("cuda", device))
    eng.forward(synth.images_fast(B, 224, 224, 3, seed0=77), _lib.EB_IN_U8_HWC)
    rate = device_rate(eng, B, _lib.EB_IN_U8_HWC, stream, topk=5, iters=3)
    out["C2_fp32_parity_mode"] = {"batch": B, "images_per_s": rate,
                                  "tflops_fp32": rate * GFLOP_PER_IMG / 1e3,
                                  "path": "fp32 CUDA-core kernels (csrc/ref32.cu), top-5 equal to the oracle"}
    eng.close()
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=256, help="per-GPU batch at N = 1 (C2)")
    ap.add_argument("--global-batch", type=int, default=4096, help="C4: global batch at N > 1")
    ap.add_argument("--ref-sample", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true",
                    help="headline only: no batch sweep / Track R / C1 / C5 / drop-in f32 extras")
    ap.add_argument("--profile-json", default="", help="write the per-op profile here")
    ap.add_argument("--minimal", action="store_true",
                    help="timed steps only (for ncu launch lists): no e2e / latency / profile / cpu")
    ap.add_argument("--c4", action="store_true",
                    help="run the C4 (sharded global batch + NCCL gather) path even at N = 1")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with torchrun "
                 f"--nproc-per-node {args.gpus}, or without torchrun to let bench.py spawn the ranks")
    torch.cuda.set_device(local)
    c4 = world > 1 or args.c4
    if c4:
        if "MASTER_ADDR" not in os.environ:  # --c4 at N = 1 without torchrun
            import socket

            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(so.getsockname()[1]),
                                  RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2003_01538_b200 import _lib, synth
    from paper_2003_01538_b200.ensemble import engine_for
    from paper_2003_01538_b200.shard import gather_rows, shard_bounds

    # N = 1: C2 at B = 256 (BASELINE configs[1]); N > 1: C4, a global batch of 4096 split
    # contiguously (2048 / 1024 / 512 per rank), logits gathered to rank 0 over NCCL.
    if c4:
        lo, hi = shard_bounds(args.global_batch, rank, world)
        B, global_b = hi - lo, args.global_batch
    else:
        lo, B, global_b = 0, args.batch, args.batch
    ens = build_ensemble(B, local)
    eng = engine_for(ens)
    stream = torch.cuda.ExternalStream(eng.stream(), device=torch.device("cuda", local))
    kind = _lib.EB_IN_U8_HWC
    TOPK = 5  # north_star's combine: per-member softmax + top-5, labels, in the timed step

    host = torch.from_numpy(synth.images_fast(B, 224, 224, 3, seed0=1234, first_row=lo)).pin_memory()
    dev_in = eng.input_buffer(kind)
    torch.cuda.synchronize()
    # resident input: one copy into the engine's staging buffer
    from paper_2003_01538_b200.engine import TRef, _wrap_device_ptr

    staging = _wrap_device_ptr(dev_in, B * 224 * 224 * 3, torch.uint8, local)
    staging.copy_(host.view(-1).cuda())
    lt = eng.members[0][1]
    kpad = max(m[2] + m[3] for m in eng.members)
    logits_t = eng.tensor_view(TRef(lt, 0, kpad, 1, 1, kpad), B).view(B, -1)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        eng.forward_device(B, kind, TOPK)
        if c4:  # every shard's logits to the serving rank, on the engine stream
            with torch.cuda.stream(stream):
                gather_rows(logits_t, global_b, dst=0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    n_launch = eng.launch_count(kind, B)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if c4:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush (256 MiB > 126 MB L2), outside the events
                ev[i][0].record(stream)
            step()
            with torch.cuda.stream(stream):
                ev[i][1].record(stream)
        torch.cuda.synchronize()
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    if c4:
        t = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
        dist.barrier()
    value = global_b * args.steps / (dev_ms / 1e3)

    # ---- roofline of the tcgen05 conv/GEMM kernel class (serialised per-op profile, taken
    # right after the timed region so that it runs at the same power-capped clocks)
    # per-op median of 3 serialised runs (an eager run's event times absorb any host-side
    # launch hiccup of the op that follows it)
    # (each op launched 5 times back to back per run: its own duration, not the host's
    # launch latency between serialised eager launches)
    ms = np.median(np.stack([eng.profile(B, kind, repeat=5) for _ in range(3)]), axis=0) if not args.minimal else np.zeros(eng.n_ops)
    conv_ms = conv_flops = 0.0
    top = None
    for m, t in zip(eng.op_meta, ms):
        if m.get("name") == "conv":
            conv_ms += float(t)
            conv_flops += m["flops"] * B
            if top is None or t > top[1]:
                top = (m, float(t))
    pk, pk_src = peaks()
    achieved = conv_flops / (conv_ms / 1e3) / 1e12 if conv_ms > 0 else 0.0
    # DRAM traffic of the top launch from the committed ncu capture of the same layer
    traffic = None
    for tl in sorted((ROOT / "profiles").glob("*/top_launch_ncu.json"), reverse=True):
        t = json.loads(tl.read_text())
        if top is not None and list(t["shape(ho,wo,cout,kh,kw,s,cin)"]) == list(top[0]["shape"]) and t["batch"] == B:
            traffic = {"dram_bytes_per_launch": t["dram_bytes_read"] + t["dram_bytes_write"],
                       "algorithmic_bytes_per_launch": t["algorithmic_bytes"], "source": t["source"]}
            break
    peak = pk["bf16_tflops_sustained"]
    bound_ms = sum(r["bound_ms"] for r in op_bounds(eng.op_meta, ms, B, peak, pk["hbm_gbs"]))
    if args.profile_json and rank == 0:
        Path(args.profile_json).write_text(json.dumps(
            [{"i": i, **{k: (list(v) if isinstance(v, tuple) else v) for k, v in m.items()}, "ms": float(t)}
             for i, (m, t) in enumerate(zip(eng.op_meta, ms))], indent=0))

    if args.minimal:
        if rank == 0:
            print(json.dumps({"minimal": True, "value": value, "ms_per_step": dev_ms / args.steps,
                              "launches_per_step": n_launch}), flush=True)
        if c4:
            dist.destroy_process_group()
        return
    # ---- e2e through the public C-ABI with pinned host buffers: every step copies its
    # inputs host->device and reads its labels back inside the timed region.
    #  pipelined: one eb_forward_batches call over all steps (step i+1's H2D overlaps
    #             step i's forward) -- the headline e2e;
    #  sequential: one eb_forward call per step (nothing overlaps).
    host_np = host.numpy()
    host2 = torch.from_numpy(synth.images_fast(B, 224, 224, 3, seed0=9999, first_row=lo)).pin_memory().numpy()
    step_inputs = [host_np if i % 2 == 0 else host2 for i in range(args.steps)]

    def timed(fn):
        if c4:
            dist.barrier()
        t0 = time.perf_counter()
        fn()
        el = time.perf_counter() - t0
        if c4:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        return el

    for _ in range(2):
        eng.forward(host_np, kind)
    eng.forward_batches(step_inputs[:2], kind)
    # (the headline pipelined run first, right after the device-timed region: under the
    # power cap a later run sees lower clocks)
    pipe_s = timed(lambda: eng.forward_batches(step_inputs, kind))
    seq_s = timed(lambda: [eng.forward(x, kind) for x in step_inputs])
    e2e = global_b * args.steps / pipe_s
    e2e_seq = global_b * args.steps / seq_s
    n_members = len(eng.members)

    extras = {}
    if not c4 and not args.quick:
        # the reference-shaped drop-in call: forward(ensemble, SampleBatch) with f32 CHW
        # samples from ordinary (pageable) numpy memory, 4x the H2D bytes of u8
        from paper_2003_01538_b200 import ensemble as E
        from paper_2003_01538_b200 import models as M

        try:
            f32 = (host_np.transpose(0, 3, 1, 2).astype(np.float32) / np.float32(255.0)).reshape(B, -1)
            sb = M.SampleBatch(ens.shared_shape, f32)
            E.forward(ens, sb)
            n_f = max(3, args.steps // 4)
            f_s = timed(lambda: [E.forward(ens, sb) for _ in range(n_f)])
            extras["dropin_f32_forward"] = {
                "images_per_s": B * n_f / f_s, "h2d_bytes_per_step": int(f32.nbytes),
                "path": "ensemble.forward(ensemble, SampleBatch) -- f32 CHW from pageable numpy "
                        "(pinned staging slots), labels back as EnsembleOutput (the reference's own "
                        "call, eg/ensemble.py:232)"}
        except Exception as exc:  # an extra, never fatal
            extras["dropin_f32_forward"] = {"error": str(exc)[:200]}

    # ---- p50 latency at bs=1 (e2e through eb_forward) and the batch sweep
    one = host_np[:1].copy()
    for _ in range(3):
        eng.forward(one, kind)
    lat = []
    for _ in range(30):
        t0 = time.perf_counter()
        eng.forward(one, kind)
        lat.append((time.perf_counter() - t0) * 1e3)
    sweep = {}
    if not c4 and not args.quick:
        for b in (1, 8, 32, 64, 128, 256):
            if b <= B:
                sweep[str(b)] = device_rate(eng, b, kind, stream, TOPK)

    hbm = hbm_kernels(B, pk["hbm_gbs"], pk_src) if rank == 0 and not c4 else None
    eng_dev = eng.device

    cpu = None
    if rank == 0 and not c4 and not args.no_cpu_baseline:
        try:
            cpu = cpu_oracle_rate()
        except Exception as exc:  # the baseline is reported, never fatal
            cpu = {"error": str(exc)[:200]}
    if not c4 and not args.quick:
        # free this engine before the extra configurations are built
        eng.close()
        del eng, ens, logits_t, staging
        torch.cuda.empty_cache()
        try:
            extras["configs"] = extra_configs(eng_dev)
        except Exception as exc:
            extras["configs"] = {"error": str(exc)[:300]}
        try:
            tr = {"gpu": track_r_gpu(pk)}
            if not args.no_cpu_baseline:
                tr["cpu"] = track_r_cpu()
            extras["track_r"] = tr
        except Exception as exc:
            extras["track_r"] = {"error": str(exc)[:300]}

    if rank == 0:
        line = {
            "metric": "ensemble images/s (N-model fwd+combine)",
            "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if c4 else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {
                "workload": (f"C4 (BASELINE configs[3]): resnet50+densenet121+vgg16, global batch "
                             f"{global_b} of synthetic 224x224 RGB u8 images split contiguously over "
                             f"{world} GPUs ({B} per rank)") if c4 else
                            ("C2 (BASELINE configs[1]): resnet50+densenet121+vgg16 cnn1 members, "
                             f"{B} synthetic 224x224 RGB u8 images per step"),
                "batch_per_gpu": B, "global_batch": global_b,
                "members": [f"{a}:seed{s}" for a, s in MEMBERS],
                "parallelism": (f"dp{world}: a replica per GPU, contiguous shards, NCCL gather of the "
                                "[B_r, 3000] fp32 logits to rank 0 in every timed step") if c4 else "single GPU",
                "step": "K1 preprocess + every member's layers + K5 combine (argmax, softmax, top-5)",
                "l2": "flushed between timed steps (256 MiB write), outside the events",
            },
            "e2e": {"value": e2e, "unit": "images/s", "h2d_bytes_per_step": int(host.numel()) * world,
                    "d2h_bytes_per_step": int(4 * n_members * B) * world,
                    "path": "eb_forward_batches (C-ABI): pinned host u8 input copied and labels read "
                            "back every step; step i+1's copy overlaps step i's forward",
                    "sequential_value": e2e_seq,
                    "sequential_path": "one eb_forward call per step (copies not overlapped)"},
            "latency_bs1_ms": {"p50": statistics.median(lat), "p99": sorted(lat)[int(0.99 * (len(lat) - 1))],
                               "path": "eb_forward, B=1, host buffers"},
            "gpu_launches": int(n_launch * args.steps),
            "roofline": {"bound": "tensor", "kernel": "conv_umma_kernel + block1_kernel (all conv/FC launches)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{pk_src} bf16_tflops_sustained",
                         "flops_per_step": conv_flops, "kernel_ms_per_step_serialised": conv_ms,
                         "step_frac_of_peak": GFLOP_PER_IMG * 1e9 * global_b / (dev_ms / args.steps / 1e3) / 1e12 / peak / world,
                         "top_launch": {"shape(ho,wo,cout,kh,kw,s,cin)": list(top[0]["shape"]), "ms": top[1]} if top else None,
                         # each conv/FC launch against its own roofline bound (tensor or HBM)
                         "per_op_bound_ms": bound_ms, "per_op_bound_frac": bound_ms / conv_ms if conv_ms else None},
            "clocks": clk.summary(),
            "hbm_kernels": hbm,
            "cpu_baseline": cpu,
        }
        if sweep:
            line["batch_sweep_images_per_s"] = sweep
        if extras:
            line["extras"] = extras
        print(json.dumps(line), flush=True)
    if c4:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
