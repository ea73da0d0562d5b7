"""The error contract of the forward path (mirrors eg/errors.py:8-77).

When the reference package ``ensemblegate`` is importable, its classes are used
directly, so the unchanged reference gateway maps our errors to the same HTTP
statuses (eg/gateway.py:49-56).  Otherwise an identical hierarchy (same names,
same ``code`` strings, same subclass relations) is defined here.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from ensemblegate.errors import (  # type: ignore
        BadK,
        BadPolicy,
        BadRequest,
        BatchTooLarge,
        BudgetExceeded,
        EmptyBatch,
        GatewayError,
        MalformedManifest,
        MalformedModel,
        NotBinary,
        PolicyUnavailable,
        ShapeMismatch,
    )

    SHARED_WITH_REFERENCE = True
except ImportError:
    SHARED_WITH_REFERENCE = False

    class GatewayError(Exception):
        code = "internal"

    class MalformedModel(GatewayError):
        code = "malformed_model"

    class MalformedManifest(GatewayError):
        code = "malformed_manifest"

    class ShapeMismatch(GatewayError):
        code = "shape_mismatch"

    class BudgetExceeded(GatewayError):
        code = "budget_exceeded"

    class BatchTooLarge(GatewayError):
        code = "batch_too_large"

    class BadRequest(GatewayError):
        code = "bad_request"

    class EmptyBatch(BadRequest):
        code = "empty_batch"

    class BadPolicy(GatewayError):
        code = "bad_policy"

    class BadK(BadPolicy):
        code = "bad_k"

    class NotBinary(GatewayError):
        code = "not_binary"

    class PolicyUnavailable(GatewayError):
        code = "policy_unavailable"


__all__ = [
    "BadK", "BadPolicy", "BadRequest", "BatchTooLarge", "BudgetExceeded", "EmptyBatch",
    "GatewayError", "MalformedManifest", "MalformedModel", "NotBinary", "PolicyUnavailable",
    "ShapeMismatch", "SHARED_WITH_REFERENCE",
]
