"""The drop-in forward boundary: manifests, ensemble residency, forward.

Mirrors eg/ensemble.py (manifest schema :94-125, all-or-nothing budgeted load
:180-229, ``forward`` :232-250) with the arithmetic on the B200:

    forward(ensemble, raw) -> EnsembleOutput
      = the reference's validation, in its order (EmptyBatch, BatchTooLarge,
        ShapeMismatch; eg/ensemble.py:238-247)
      + one native eb_forward call: H2D copy, K1 preprocess once, every member
        (LIN1 fp64 scores / CNN implicit-GEMM layers), K5 argmax, D2H labels.

``forward`` accepts this package's Ensemble as well as an ``ensemblegate``
Ensemble (LIN1 members; duck-typed), for which a device copy of the weights is
built once and cached for the lifetime of that object (ensembles are immutable,
eg/ensemble.py:133).
"""

from __future__ import annotations

import os

import threading
import weakref
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from . import errors
from .models import (
    BINARY_LABELS,
    MODEL_ID_RE,
    InputShape,
    PreprocessSpec,
    count_preprocess,
    loads_strict,
    parse_model_file,
)

_MANIFEST_FIELDS = frozenset({"memory_budget_bytes", "max_batch", "preprocess", "models"})
_PRE_FIELDS = frozenset({"mean", "std", "pixel_scale"})
_ENTRY_FIELDS = frozenset({"id", "path"})

POLICY_CODES = {"any": _lib.EB_POLICY_ANY, "all": _lib.EB_POLICY_ALL,
                "at_least": _lib.EB_POLICY_AT_LEAST}


@dataclass(frozen=True)
class ManifestEntry:
    id: str
    path: str


@dataclass(frozen=True)
class ModelManifest:
    memory_budget_bytes: int
    max_batch: int
    preprocess: PreprocessSpec
    models: tuple
    base_dir: Path = Path(".")

    def __post_init__(self):
        if self.memory_budget_bytes < 1:
            raise errors.MalformedManifest(f"memory_budget_bytes must be >= 1, got {self.memory_budget_bytes}")
        if self.max_batch < 1:
            raise errors.MalformedManifest(f"max_batch must be >= 1, got {self.max_batch}")
        entries = tuple(self.models)
        if not entries:
            raise errors.MalformedManifest("manifest needs at least one model entry")
        ids = [e.id for e in entries]
        dup = sorted({i for i in ids if ids.count(i) > 1})
        if dup:
            raise errors.MalformedManifest(f"duplicate model ids: {dup}")
        for e in entries:
            if not isinstance(e.id, str) or not MODEL_ID_RE.fullmatch(e.id):
                raise errors.MalformedManifest(f"bad model id {e.id!r}")
        object.__setattr__(self, "models", entries)
        object.__setattr__(self, "base_dir", Path(self.base_dir))

    @property
    def size(self) -> int:
        return len(self.models)


def _count(v, name):
    if isinstance(v, bool) or not isinstance(v, int):
        raise errors.MalformedManifest(f"{name} must be an integer, got {v!r}")
    return v


def _preprocess_spec(raw) -> PreprocessSpec:
    if not isinstance(raw, dict):
        raise errors.MalformedManifest("preprocess must be an object")
    unknown = sorted(set(raw) - _PRE_FIELDS)
    if unknown:
        raise errors.MalformedManifest(f"unknown preprocess fields: {unknown}")
    for key in ("mean", "std"):
        if key not in raw:
            raise errors.MalformedManifest(f"preprocess.{key} is required")
        vals = raw[key]
        if not isinstance(vals, list) or not vals:
            raise errors.MalformedManifest(f"preprocess.{key} must be a non-empty array")
        for v in vals:
            if isinstance(v, bool) or not isinstance(v, (int, float)):
                raise errors.MalformedManifest(f"preprocess.{key}: {v!r} is not a number")
    scale = raw.get("pixel_scale", 255.0)
    if isinstance(scale, bool) or not isinstance(scale, (int, float)):
        raise errors.MalformedManifest(f"preprocess.pixel_scale must be a number, got {scale!r}")
    try:
        return PreprocessSpec(tuple(raw["mean"]), tuple(raw["std"]), float(scale))
    except ValueError as exc:
        raise errors.MalformedManifest(f"bad preprocess: {exc}") from exc


def load_manifest(data: bytes, base_dir=".") -> ModelManifest:
    try:
        doc = loads_strict(data)
    except ValueError as exc:
        raise errors.MalformedManifest(f"unreadable manifest: {exc}") from exc
    if not isinstance(doc, dict):
        raise errors.MalformedManifest("manifest must be a JSON object")
    unknown = sorted(set(doc) - _MANIFEST_FIELDS)
    if unknown:
        raise errors.MalformedManifest(f"unknown manifest fields: {unknown}")
    missing = sorted(_MANIFEST_FIELDS - set(doc))
    if missing:
        raise errors.MalformedManifest(f"missing manifest fields: {missing}")
    budget = _count(doc["memory_budget_bytes"], "memory_budget_bytes")
    max_batch = _count(doc["max_batch"], "max_batch")
    spec = _preprocess_spec(doc["preprocess"])
    raw_models = doc["models"]
    if not isinstance(raw_models, list):
        raise errors.MalformedManifest("models must be an array")
    entries = []
    for i, e in enumerate(raw_models):
        if not isinstance(e, dict) or set(e) != _ENTRY_FIELDS:
            raise errors.MalformedManifest(f"models[{i}] must be an object with exactly 'id' and 'path'")
        if not isinstance(e["id"], str) or not isinstance(e["path"], str):
            raise errors.MalformedManifest(f"models[{i}]: id and path must be strings")
        entries.append(ManifestEntry(e["id"], e["path"]))
    return ModelManifest(budget, max_batch, spec, tuple(entries), Path(base_dir))


def load_manifest_file(path) -> ModelManifest:
    path = Path(path)
    return load_manifest(path.read_bytes(), base_dir=path.parent)


@dataclass(frozen=True)
class EnsembleOutput:
    """Per-model label indices for one batch, in manifest order."""

    model_ids: tuple
    per_model: tuple

    def __post_init__(self):
        ids = tuple(self.model_ids)
        rows = tuple(tuple(r) for r in self.per_model)
        if len(rows) != len(ids):
            raise ValueError(f"{len(rows)} output rows for {len(ids)} model ids")
        if len({len(r) for r in rows}) > 1:
            raise ValueError(f"inconsistent per-model output lengths: {sorted({len(r) for r in rows})}")
        object.__setattr__(self, "model_ids", ids)
        object.__setattr__(self, "per_model", rows)

    @property
    def batch_size(self) -> int:
        return len(self.per_model[0]) if self.per_model else 0


@dataclass(frozen=True, eq=False)
class Ensemble:
    """N members resident in one device weight pool (built lazily on first use)."""

    models: tuple
    shared_shape: InputShape
    preprocess: PreprocessSpec
    bytes_used: int
    memory_budget_bytes: int
    max_batch: int
    binary_compatible: bool
    device: int = 0
    # CNN arithmetic: "bf16" (tcgen05, the throughput path) or "fp32" (the fp32-faithful
    # parity mode, csrc/ref32.cu: top-k equal to the fp32 CPU oracle's)
    precision: str = "bf16"
    # more than one device: a replica per GPU, requests sharded across them (shard.py)
    devices: tuple = ()
    # execution contexts per device (engine.ContextPool): concurrent requests in flight
    contexts: int = 1
    _state: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        object.__setattr__(self, "models", tuple(self.models))

    @property
    def model_ids(self) -> tuple:
        return tuple(m.id for m in self.models)

    @property
    def size(self) -> int:
        return len(self.models)

    def engine(self):
        return engine_for(self)


def default_precision() -> str:
    """EB_PRECISION=fp32 selects the fp32-faithful mode for ensembles loaded without an
    explicit precision (e.g. through the seam, whose load_ensemble has the reference's
    signature)."""
    p = os.environ.get("EB_PRECISION", "bf16").lower()
    return "fp32" if p in ("fp32", "f32", "float32") else "bf16"


def default_devices() -> tuple:
    """EB_DEVICES=0,1,2,3 shards ensembles loaded without explicit devices (e.g. by the
    reference's gateway through the seam) over those GPUs."""
    v = os.environ.get("EB_DEVICES", "").strip()
    return tuple(int(d) for d in v.split(",") if d.strip()) if v else ()


def default_contexts() -> int:
    """EB_CONTEXTS=n: execution contexts per device for ensembles loaded without an
    explicit count (the gateway's worker threads then run up to n forwards at once)."""
    return max(1, int(os.environ.get("EB_CONTEXTS", "1") or 1))


def load_ensemble(manifest: ModelManifest, device: int = 0, precision: str | None = None,
                  devices=None, contexts: int | None = None) -> Ensemble:
    """Parse every member, check shapes and the byte budget, all or nothing.

    ``devices`` (two or more GPU ordinals) serves the ensemble from a replica per GPU
    with every request batch sharded contiguously across them (shard.ShardedEngine)."""
    precision = precision or default_precision()
    contexts = contexts or default_contexts()
    devices = tuple(devices) if devices is not None else default_devices()
    if len(devices) == 1:
        device, devices = devices[0], ()
    elif devices:
        device = devices[0]
    if precision not in ("bf16", "fp32"):
        raise ValueError(f"precision must be 'bf16' or 'fp32', got {precision!r}")
    loaded = []
    for entry in manifest.models:
        path = Path(entry.path)
        if not path.is_absolute():
            path = manifest.base_dir / path
        try:
            data = path.read_bytes()
        except OSError as exc:
            raise errors.MalformedModel(f"cannot read model file {path}: {exc}") from exc
        model = parse_model_file(data)
        if model.id != entry.id:
            raise errors.MalformedModel(f"model file {path} has id {model.id!r} but the manifest says {entry.id!r}")
        loaded.append(model)
    shape = loaded[0].input_shape
    if all(getattr(m, "kind", "lin1") == "cnn1" for m in loaded) and len(
            {m.input_shape for m in loaded}) > 1:
        # Mixed native resolutions (config 5: Inception-v3 at 299 beside 224 members) are
        # allowed when EVERY member is a CNN: requests arrive at the largest resolution and
        # K1 emits a bilinear-resized copy for the others.
        if len({m.input_shape.dims[0] for m in loaded}) > 1:
            raise errors.ShapeMismatch("CNN members must agree on the channel count")
        shape = max((m.input_shape for m in loaded), key=lambda s: s.dims[1] * s.dims[2])
    else:
        # any LIN1 member: the reference's uniform-shape rule for every member, in
        # manifest order (eg/ensemble.py:202-208)
        for m in loaded[1:]:
            if m.input_shape != shape:
                raise errors.ShapeMismatch(f"model {m.id!r} has input shape {list(m.input_shape.dims)}, "
                                    f"expected {list(shape.dims)} shared by the ensemble")
    for name, vals in (("mean", manifest.preprocess.mean), ("std", manifest.preprocess.std)):
        if len(vals) not in (1, shape.channels):
            raise errors.ShapeMismatch(f"preprocess {name} has {len(vals)} entries; input shape "
                                f"{list(shape.dims)} has {shape.channels} channel(s)")
    used = sum(m.parameter_bytes for m in loaded)
    if used > manifest.memory_budget_bytes:
        raise errors.BudgetExceeded(f"memory budget exceeded: ensemble needs {used} bytes, "
                             f"budget is {manifest.memory_budget_bytes} bytes")
    return Ensemble(tuple(loaded), shape, manifest.preprocess, used, manifest.memory_budget_bytes,
                    manifest.max_batch, all(m.labels == BINARY_LABELS for m in loaded), device,
                    precision, devices, contexts)


# ---------------------------------------------------------------------- device residency

_engines: dict[int, object] = {}
_engines_lock = threading.Lock()


def _kind(model) -> str:
    return getattr(model, "kind", "lin1")


def build_engine(models, shape, spec, max_batch: int, device: int = 0, precision: str = "bf16"):
    """Upload every member into one device pool and declare its ops (zoo / LIN1)."""
    from . import zoo
    from .engine import Engine
    from .packing import u8_lut

    c, h, w = shape.chw() if hasattr(shape, "chw") else (
        tuple(shape.dims) if len(shape.dims) == 3 else (1, 1, shape.dims[0]))
    eng = Engine((c, h, w), max_batch, device, precision)
    eng.set_preprocess(spec.mean, spec.std, u8_lut(spec.mean, spec.std, spec.pixel_scale, c))
    cnn = [m for m in models if _kind(m) == "cnn1"]
    lin = [m for m in models if _kind(m) != "cnn1"]
    koffs = {}
    logits32 = scores64 = None
    if cnn:
        off = 0
        for m in cnn:
            koffs[m.id] = off
            off += (len(m.labels) + 7) // 8 * 8
        logits32 = eng.tensor(1, 1, off, _lib.EB_F32)
    if lin:
        off = 0
        for m in lin:
            koffs[m.id] = off
            off += len(m.labels)
        scores64 = eng.tensor(1, 1, off, _lib.EB_F64)
        wcat = np.concatenate([np.asarray(m.weights, np.float32) for m in lin], axis=0)
        bcat = np.concatenate([np.asarray(m.bias, np.float32) for m in lin], axis=0)
        eng.op(_lib.EB_OP_LIN1, eng.image_f32, scores64, cout=off, lane=0,
               w_off=eng.weight(wcat), b_off=eng.weight(bcat))
    lane = 0
    images: dict = {}
    torch_models = {m.id: m.torch_model() for m in cnn}
    # members with an identical first layer on the same image share one grouped launch
    stem_groups: dict = {}
    for m in cnn:
        st = zoo.stem_of(m.arch, torch_models[m.id])
        if st is None:
            continue
        c = st[0]
        key = (tuple(m.input_shape.dims), c.kernel_size, c.stride, c.padding, c.in_channels)
        stem_groups.setdefault(key, []).append(m)
    stem_out: dict = {}
    if grouped_stems_enabled():
        for key, group in stem_groups.items():
            # launches of at most 128 output channels: a wider stem is two N tiles whose
            # 7-row filter no longer fits resident in shared memory beside the A stages
            # (B200, B = 128: 192 channels in one launch 684 us; 128 + 64 in two, 150 + 114)
            chunks, cur, width = [], [], 0
            for g in group:
                cout = zoo.stem_of(g.arch, torch_models[g.id])[0].out_channels
                if cur and width + cout > 128:
                    chunks.append(cur)
                    cur, width = [], 0
                cur.append(g)
                width += cout
            chunks.append(cur)
            for chunk in chunks:
                if len(chunk) < 2:
                    continue
                img = zoo.resized_image(eng, key[0][1:], images)
                outs = zoo.grouped_stem(eng, img, [zoo.stem_of(g.arch, torch_models[g.id]) for g in chunk])
                for g, o in zip(chunk, outs):
                    stem_out[g.id] = o
    for m in models:
        k = len(m.labels)
        if _kind(m) == "cnn1":
            img = zoo.resized_image(eng, tuple(m.input_shape.dims[1:]), images)
            # one concurrency lane per member (EB_ONE_LANE=1: all members on the main stream)
            mlane = 0 if os.environ.get("EB_ONE_LANE") == "1" else lane % 4
            zoo.lower(eng, m.arch, torch_models[m.id], logits32.slice(koffs[m.id], k), mlane,
                      image=img, stem_out=stem_out.get(m.id))
            lane += 1
            eng.member(_lib.EB_MEMBER_CNN, logits32, koffs[m.id], k)
        else:
            eng.member(_lib.EB_MEMBER_LIN1, scores64, koffs[m.id], k)
    eng.finalize()
    return eng


def grouped_stems_enabled() -> bool:
    import os

    return os.environ.get("EB_GROUPED_STEM", "1") not in ("0", "no", "false")


def engine_for(ensemble):
    """The cached device engine of an ensemble (ours or an ensemblegate one)."""
    state = getattr(ensemble, "_state", None)
    if state is not None and "engine" in state:
        return state["engine"]
    key = id(ensemble)
    with _engines_lock:
        if state is not None:
            if "engine" not in state:
                from .engine import ContextPool

                devices = getattr(ensemble, "devices", ())
                prec = getattr(ensemble, "precision", "bf16")
                nctx = getattr(ensemble, "contexts", 1)

                def on(dev, mb):
                    eng = build_engine(ensemble.models, ensemble.shared_shape, ensemble.preprocess,
                                       mb, dev, prec)
                    return ContextPool(eng, nctx) if nctx > 1 else eng

                if len(devices) > 1:
                    from .shard import ShardedEngine

                    per = -(-ensemble.max_batch // len(devices))
                    state["engine"] = ShardedEngine([on(d, per) for d in devices])
                else:
                    state["engine"] = on(getattr(ensemble, "device", 0), ensemble.max_batch)
            return state["engine"]
        eng = _engines.get(key)
        if eng is None:
            eng = build_engine(ensemble.models, ensemble.shared_shape, ensemble.preprocess,
                               ensemble.max_batch, 0, default_precision())
            _engines[key] = eng
            weakref.finalize(ensemble, _engines.pop, key, None)
        return eng


# ---------------------------------------------------------------------- forward


def _validate(ensemble, b: int, dims) -> None:
    if b == 0:
        raise errors.EmptyBatch("batch has no samples")
    if b > ensemble.max_batch:
        raise errors.BatchTooLarge(f"batch size {b} exceeds max_batch {ensemble.max_batch}")
    if tuple(dims) != tuple(ensemble.shared_shape.dims):
        raise errors.ShapeMismatch(f"batch shape {list(dims)} does not match ensemble "
                            f"input shape {list(ensemble.shared_shape.dims)}")


def _count_and_check_spec(ensemble) -> None:
    count_preprocess()
    spec, shape = ensemble.preprocess, ensemble.shared_shape
    ch = shape.dims[0] if len(shape.dims) == 3 else 1
    for name, vals in (("mean", spec.mean), ("std", spec.std)):
        if len(vals) not in (1, ch):
            raise errors.ShapeMismatch(f"{name} has {len(vals)} entries; shape {list(shape.dims)} "
                                f"has {ch} channel(s)")


def _policy_args(ensemble, policy):
    if policy is None:
        return _lib.EB_POLICY_NONE, 0
    if not ensemble.binary_compatible:
        raise errors.PolicyUnavailable("policy unavailable: every model must use the labels ['absent', 'present']")
    kind = getattr(policy, "kind", None)
    if kind not in POLICY_CODES:
        raise errors.BadPolicy(f"unknown policy kind {kind!r}")
    k = getattr(policy, "k", None)
    if kind == "at_least":
        n = len(ensemble.models)
        if isinstance(k, bool) or not isinstance(k, int):
            raise errors.BadK(f"k must be an integer, got {k!r}")
        if not 1 <= k <= n:
            raise errors.BadK(f"k must be between 1 and {n} for this ensemble, got {k}")
        return POLICY_CODES[kind], k
    return POLICY_CODES[kind], 0


def _output_type():
    try:  # return the caller's EnsembleOutput class when running inside ensemblegate
        from ensemblegate.ensemble import EnsembleOutput as RefOut  # type: ignore

        return RefOut
    except ImportError:
        return EnsembleOutput


def predict(ensemble, raw, policy=None, topk: int = 0, want_logits: bool = False):
    """forward + the K5 combine in one native call.

    Returns (EnsembleOutput, combined or None, extras) where extras holds
    top-k indices / softmax probabilities / logits when requested.
    """
    b = int(raw.data.shape[0])
    _validate(ensemble, b, raw.shape.dims)
    _count_and_check_spec(ensemble)  # forward's preprocess runs before the policy checks
    pk, kk = _policy_args(ensemble, policy)
    eng = engine_for(ensemble)
    res = eng.forward(np.ascontiguousarray(raw.data, dtype=np.float32), _lib.EB_IN_F32_CHW,
                      topk=topk, policy=pk, policy_k=kk, want_logits=want_logits)
    out = _output_type()(tuple(m.id for m in ensemble.models),
                         tuple(tuple(int(v) for v in row) for row in res["labels"]))
    combined = [int(v) for v in res["combined"]] if pk else None
    return out, combined, res


def forward(ensemble, raw):
    """Evaluate every member on one preprocessed batch, in manifest order."""
    b = int(raw.data.shape[0])
    _validate(ensemble, b, raw.shape.dims)
    _count_and_check_spec(ensemble)
    eng = engine_for(ensemble)
    res = eng.forward(np.ascontiguousarray(raw.data, dtype=np.float32), _lib.EB_IN_F32_CHW)
    return _output_type()(tuple(m.id for m in ensemble.models),
                          tuple(tuple(int(v) for v in row) for row in res["labels"]))


def predict_u8(ensemble, pixels: np.ndarray, policy=None, topk: int = 0, want_logits=False):
    """Raw uint8 (B, H, W, C) images: /pixel_scale and normalisation fused into K1."""
    if pixels.dtype != np.uint8 or pixels.ndim != 4:
        raise errors.ShapeMismatch("pixels must be a (B, H, W, C) uint8 array")
    b, h, w, c = pixels.shape
    _validate(ensemble, b, (c, h, w))
    _count_and_check_spec(ensemble)
    pk, kk = _policy_args(ensemble, policy)
    eng = engine_for(ensemble)
    res = eng.forward(np.ascontiguousarray(pixels), _lib.EB_IN_U8_HWC, topk=topk, policy=pk,
                      policy_k=kk, want_logits=want_logits)
    out = _output_type()(tuple(m.id for m in ensemble.models),
                         tuple(tuple(int(v) for v in row) for row in res["labels"]))
    combined = [int(v) for v in res["combined"]] if pk else None
    return out, combined, res
