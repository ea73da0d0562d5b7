"""bench.op_bounds: the per-launch roofline bound bench.py reports (CPU only)."""
import pytest

bench = pytest.importorskip("bench")


def test_op_bounds_tensor_and_hbm_sides():
    B = 256
    # a compute-heavy 3x3 (tensor-bound) and a 1x1 with a residual (HBM-bound)
    conv3 = {"name": "conv", "shape": [28, 28, 512, 3, 3, 1, 512], "res": -1, "weight_bytes": 4718592,
             "flops": 2 * 28 * 28 * 512 * 512 * 9}
    conv1 = {"name": "conv", "shape": [56, 56, 256, 1, 1, 1, 64], "res": 3, "weight_bytes": 32768,
             "flops": 2 * 56 * 56 * 256 * 64}
    pool = {"name": None, "kind": 1}
    r = bench.op_bounds([conv3, pool, conv1], [0.6, 0.1, 0.2], B, 1000.0, 5000.0)
    assert len(r) == 2  # the pool is not a conv/FC launch
    t3 = conv3["flops"] * B / 1e15 * 1e3
    assert r[0]["tensor_ms"] == pytest.approx(t3) and r[0]["bound_ms"] == pytest.approx(t3)
    by = B * 2 * (56 * 56 * 64 + 2 * 56 * 56 * 256) + 32768  # input + output + residual + weights
    assert r[1]["bytes"] == by
    assert r[1]["bound_ms"] == pytest.approx(by / 5e12 * 1e3)
    assert r[1]["bound_ms"] > r[1]["tensor_ms"]
    # stems count the image's 3 channels, not the 8-channel padded layout
    stem = {"name": "conv", "shape": [224, 224, 64, 3, 3, 1, 8], "res": -1, "weight_bytes": 0, "flops": 1}
    assert bench.op_bounds([stem], [1.0], 1, 1.0, 1.0)[0]["bytes"] == 2 * (224 * 224 * 3 + 224 * 224 * 64)
