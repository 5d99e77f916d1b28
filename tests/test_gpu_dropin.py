"""The reference-shaped float64 API (delta_for_rows, adapter_delta,
apply_masked) running on the device, against the reference's golden outputs
and the reference's own unit-test expectations (tests/test_adapters.py)."""

import numpy as np
import pytest
import torch

import helpers
from paper_2605_14217_b200 import (
    AdapterKind,
    AdapterParams,
    PositionSchedule,
    ScalingRule,
    adapter_delta,
    apply_masked,
    delta_for_rows,
    init_zero_delta,
)
from paper_2605_14217_b200.errors import DomainError, ShapeError
from paper_2605_14217_b200.linalg import rng_from_seed

pytestmark = pytest.mark.gpu


def test_delta_for_rows_matches_reference_golden(cuda_device):
    for c in helpers.delta_cases():
        p = helpers.make_params(c)
        d = delta_for_rows(p, c["rows"])
        assert d.dtype == np.float64 and d.shape == c["delta"].shape
        helpers.check_close(d, np.zeros_like(d), c["delta"], "f64", f"{c['kind']} r={c['rank']} {c['dims']}")


def test_known_answers_exact(cuda_device):
    # tests/test_adapters.py:64-88, exact equality
    lora = AdapterParams(AdapterKind.LORA, 1, (2, 2), ScalingRule.constant(1.0), A=np.array([[0.0, 2.0]]),
                         B=np.array([[1.0], [0.0]]))
    assert np.array_equal(adapter_delta(lora, np.array([3.0, 4.0])), np.array([8.0, 0.0]))
    dire = AdapterParams(AdapterKind.DIREFT, 1, (2,), ScalingRule.constant(1.0), A=np.array([[0.0, 1.0]]),
                         B=np.array([[1.0, 0.0]]), b=np.array([0.0]))
    assert np.array_equal(adapter_delta(dire, np.array([5.0, 7.0])), np.array([7.0, 0.0]))


@pytest.mark.parametrize("kind", list(AdapterKind))
@pytest.mark.parametrize("rank", [1, 4, 16])
def test_zero_delta_init(cuda_device, kind, rank):
    # tests/test_adapters.py:126-136: exact 0 for LoRA/DiReFT, <= 1e-12 LoReFT (exact 0 here)
    d = 16
    params = init_zero_delta(kind, rank, (d, d) if kind is AdapterKind.LORA else (d,), seed=33)
    rows = rng_from_seed(44).normal(size=(100, d))
    deltas = delta_for_rows(params, rows)
    assert np.max(np.abs(deltas)) == 0.0


def test_prefactor_linearity(cuda_device):
    # tests/test_adapters.py:104-112
    d = 10
    base = init_zero_delta(AdapterKind.DIREFT, 2, (d,), seed=1, scaling=ScalingRule.constant(1.0))
    A = rng_from_seed(2).normal(size=(2, d))
    b = rng_from_seed(3).normal(size=2)
    one = AdapterParams(AdapterKind.DIREFT, 2, (d,), ScalingRule.constant(1.0), A=A, B=base.B, b=b)
    three = AdapterParams(AdapterKind.DIREFT, 2, (d,), ScalingRule.constant(3.0), A=A, B=base.B, b=b)
    h = rng_from_seed(4).normal(size=d)
    np.testing.assert_allclose(adapter_delta(three, h), 3.0 * adapter_delta(one, h), rtol=1e-12)


def test_apply_masked_matches_reference_golden(cuda_device):
    for c in helpers.masked_cases():
        p = helpers.make_params(c)
        sched = PositionSchedule.ALL_POSITIONS if c["sched_all"] else PositionSchedule.PREFILL_ONLY
        y = c["y"].copy()
        out = apply_masked(p, sched, y, c.get("x"), c["plen"])
        assert np.array_equal(y, c["y"])  # inputs never mutated (adapters.py:312)
        cut = y.shape[0] if c["sched_all"] else min(c["plen"], y.shape[0])
        assert np.array_equal(out[cut:], c["y"][cut:])  # tail bit-identical
        helpers.check_close(out, c["y"], c["out"], "f64", f"masked {c['kind']} p={c['plen']}")


def test_apply_masked_errors(cuda_device):
    p = init_zero_delta(AdapterKind.LORA, 2, (6, 6), seed=9)
    y = np.zeros((5, 6))
    with pytest.raises(ShapeError):
        apply_masked(p, PositionSchedule.PREFILL_ONLY, y, None, prompt_len=3)
    with pytest.raises(DomainError):
        apply_masked(p, PositionSchedule.PREFILL_ONLY, y, y, prompt_len=-1)
    with pytest.raises(ShapeError):
        delta_for_rows(p, np.zeros((2, 3, 6)))
    with pytest.raises(ShapeError):
        adapter_delta(init_zero_delta(AdapterKind.DIREFT, 2, (8,), seed=0), np.zeros(9))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_delta_for_rows_on_device_tensors(cuda_device, dtype):
    for c in helpers.delta_cases()[:20]:
        p = helpers.make_params(c)
        rows = torch.from_numpy(c["rows"]).to(cuda_device, dtype)
        d = delta_for_rows(p, rows)
        assert d.device == rows.device and d.dtype == dtype
        # oracle on the quantised rows/params the device saw
        from oracle import preft_oracle as O

        q = lambda a: torch.from_numpy(np.asarray(a)).to(dtype).double().numpy()  # noqa: E731
        prm = {k: q(v) for k, v in helpers.params_of(c).items()}
        if c["kind"] == "loreft":  # device folds W - R in f64 before rounding
            prm = dict(A=q(c["W"] - c["R"]), B=prm["R"], b=c["b"])
            ref = O.delta_rows("direft", c["s"], q(c["rows"]), **prm)
        else:
            if "b" in prm:
                prm["b"] = c["b"]
            ref = O.delta_rows(c["kind"], c["s"], q(c["rows"]), **prm)
        mode = "f32" if dtype == torch.float32 else "bf16"
        out = d.double().cpu().numpy()
        helpers.check_close(out, np.zeros_like(out), ref, mode, f"device {c['kind']}")
