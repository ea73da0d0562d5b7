"""Drop-in: route an unchanged ``ensemblegate`` installation through the B200 path.

    import ensemblegate
    from paper_2003_01538_b200 import seam
    seam.install()          # ensemblegate now serves forward/predict on the GPU

What is rebound ("inner seams"):

* ``ensemblegate.ensemble.forward`` and the name the gateway imported
  (``ensemblegate.gateway.forward``, eg/gateway.py:20) -> ``ensemble.forward``;
* ``ensemblegate.models.preprocess`` / ``linear_predict`` -> the K1 / K6 GPU ops;
* ``ensemblegate.gateway.load_ensemble`` (eg/gateway.py:20, used by ``serve``) ->
  this package's loader, which also accepts ``cnn1`` members;
* ``ensemblegate.gateway.apply_policy`` -> the K5 policy kernel, and
  ``GatewayApp._predict`` (eg/gateway.py:133-142) -> one fused native call
  (forward + combine), preserving the reference's error order: forward errors,
  then PolicyUnavailable, then BadK.
* this package's error classes become the reference's own (so the unchanged
  gateway maps them to the same HTTP statuses, eg/gateway.py:49-56), and the
  preprocess counter the reference's tests read (``preprocess_call_count``) is
  the one that is incremented.

``uninstall()`` restores everything.  Nothing here is on the compute path: it only
changes which function objects the reference's modules point at.
"""

from __future__ import annotations

import threading

_saved: list[tuple[object, str, object]] = []
_lock = threading.Lock()


def _set(obj, name, value):
    _saved.append((obj, name, getattr(obj, name)))
    setattr(obj, name, value)


def install() -> None:
    import ensemblegate.ensemble as eg_ens
    import ensemblegate.errors as eg_err
    import ensemblegate.gateway as eg_gw
    import ensemblegate.models as eg_models
    import ensemblegate.wire as eg_wire

    from . import ensemble as ours
    from . import errors as our_err
    from . import models as our_models
    from . import policy as our_policy

    with _lock:
        if _saved:
            return
        for name in ("GatewayError", "MalformedModel", "MalformedManifest", "ShapeMismatch",
                     "BudgetExceeded", "BatchTooLarge", "BadRequest", "EmptyBatch", "BadPolicy",
                     "BadK", "NotBinary", "PolicyUnavailable"):
            _set(our_err, name, getattr(eg_err, name))

        def bump_reference_counter():
            with eg_models._preprocess_lock:
                eg_models._preprocess_calls += 1

        _set(our_models, "_external_counter", bump_reference_counter)
        _set(eg_ens, "forward", ours.forward)
        _set(eg_gw, "forward", ours.forward)
        _set(eg_models, "preprocess", our_models.preprocess)
        _set(eg_models, "linear_predict", our_models.linear_predict)
        _set(eg_gw, "load_ensemble", ours.load_ensemble)
        _set(eg_gw, "apply_policy", our_policy.apply_policy)

        reference_predict = eg_gw.GatewayApp._predict

        def _predict(self, body: bytes):
            if eg_gw.forward is not ours.forward:
                # someone rebound the gateway's forward after install (the reference's own
                # tests monkeypatch it, tests/test_gateway.py:109-118): honour it through the
                # reference's unfused _predict, which calls gateway.forward
                return reference_predict(self, body)
            ensemble = self._require_ensemble()
            if ensemble is None:
                return 503, eg_gw._error_body("loading", "ensemble is still loading")
            decoded = _fast_path(ensemble, body)
            if decoded is None:  # anything unusual: the reference decoder and its errors
                batch, policy = eg_gw.decode_request(body, pixel_scale=ensemble.preprocess.pixel_scale)
            else:
                batch, policy = decoded
            output, combined, res = ours.predict(ensemble, batch, policy)
            return 200, _renderer(ensemble).render(res["labels"], combined)

        def _renderer(ensemble):
            # F4: the native renderer, prepared once per ensemble (immutable)
            from .wire import Renderer

            state = getattr(ensemble, "_state", None)
            if state is None:
                return Renderer(ensemble)
            if "renderer" not in state:
                state["renderer"] = Renderer(ensemble)
            return state["renderer"]

        def _fast_path(ensemble, body):
            from types import SimpleNamespace

            from .wire import fast_decode

            got = fast_decode(body, ensemble.shared_shape.dims, ensemble.max_batch,
                              pixel_scale=float(ensemble.preprocess.pixel_scale))
            if got is None:
                return None
            data, policy_raw = got
            policy = None
            if policy_raw is not None:
                try:
                    policy_obj = eg_wire.loads_strict(policy_raw)
                except ValueError:
                    return None
                policy = eg_wire.parse_policy(policy_obj)
            # already validated (shape, finiteness) by the native decoder: a view, no copy
            return SimpleNamespace(data=data, shape=ensemble.shared_shape), policy

        _set(eg_gw.GatewayApp, "_predict", _predict)


def uninstall() -> None:
    with _lock:
        while _saved:
            obj, name, value = _saved.pop()
            setattr(obj, name, value)


def installed() -> bool:
    return bool(_saved)


# pytest plugin form:  pytest -p paper_2003_01538_b200.seam <reference tests>
def pytest_configure(config):  # pragma: no cover - exercised only with the reference suite
    install()
