"""API contracts the advisor flagged: the LoRA/ReFT slot split
baked into K1, plan-side validation, and the K2 launch-shape hint of plans
created before their metadata was first built."""

import numpy as np
import pytest
import torch

import gpu_util as U
import helpers
from paper_2605_14217_b200 import AdapterKind
from paper_2605_14217_b200.errors import BatchError, ConfigError, ShapeError, StateError

pytestmark = pytest.mark.gpu


def _mixed_pool(dev, dtype=torch.bfloat16):
    from paper_2605_14217_b200.pool import AdapterPool

    pool = AdapterPool(2, 256, lora_sites={"Wq": (256, 256)}, lora_capacity=4, lora_rank=1, reft_capacity=4,
                       reft_rank=8, dtype=dtype, device=dev)
    lo = pool.fill_synthetic_(4, AdapterKind.LORA, 1, seed=1, sigma=0.05)
    re = pool.fill_synthetic_(4, AdapterKind.DIREFT, 8, seed=2, first_id=100)
    return pool, lo, re


def test_meta_built_with_another_split_is_rejected(cuda_device):
    """A meta built without the pool's split (the public BatchMeta.build
    default) used to make the ReFT kernel silently apply nothing."""
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_, apply_reft_

    pool, lo, re = _mixed_pool(cuda_device)
    rng = np.random.default_rng(0)
    qsl, ids, flags = U.random_entries(rng, 12, lo + re, p_decode=0.2)
    slots = pool.entry_arrays(qsl, ids, flags)
    meta = BatchMeta(32, 1024, device=cuda_device)
    T = int(qsl[-1])
    h = U.rand_act(rng, T, 256, torch.bfloat16, cuda_device)
    with pytest.raises(StateError):
        apply_reft_(h, meta, pool, 0)  # never built
    meta.build_arrays(qsl, slots, flags)  # default split: all LoRA
    with pytest.raises(ConfigError):
        apply_reft_(h, meta, pool, 0)
    with pytest.raises(ConfigError):
        apply_lora_(h, h, meta, pool, 0, "Wq")
    meta.build_arrays(qsl, slots, flags, slot_split=pool.slot_split)
    meta.set_slot_split(0)  # changing it after the build is caught too
    with pytest.raises(ConfigError):
        apply_reft_(h, meta, pool, 0)
    meta.build_arrays(qsl, slots, flags, slot_split=pool.slot_split)
    h_in = U.to_np(h)
    apply_reft_(h, meta, pool, 0)
    ref = U.reft_oracle(h_in, qsl, slots, flags, pool, 0)
    helpers.check_close(U.to_np(h), h_in, ref, "bf16", "reft after a correct build")


def test_pool_build_meta_sets_split(cuda_device):
    from paper_2605_14217_b200 import Phase, PositionSchedule, SeqEntry, make_batch
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_

    pool, lo, re = _mixed_pool(cuda_device)
    b = make_batch([SeqEntry(0, tuple(range(5)), 5, Phase.PREFILL, re[0], PositionSchedule.PREFILL_ONLY),
                    SeqEntry(1, tuple(range(3)), 3, Phase.PREFILL, lo[1], PositionSchedule.PREFILL_ONLY)])
    meta = BatchMeta(8, 64, device=cuda_device)
    pool.build_meta(meta, b)
    h = torch.randn(8, 256, device=cuda_device).to(torch.bfloat16)
    h0 = h.clone()
    apply_reft_(h, meta, pool, 0)
    assert not torch.equal(h[:5], h0[:5]) and torch.equal(h[5:], h0[5:])


def test_raw_arrays_validated_on_host(cuda_device):
    from paper_2605_14217_b200.meta import BatchMeta

    meta = BatchMeta(8, 64, device=cuda_device)
    z = np.zeros(2, np.int32)
    for qsl, slots, flags in (
        (np.array([1, 3, 5], np.int32), z, z),  # does not start at 0
        (np.array([0, 3, 3], np.int32), z, z),  # empty entry
        (np.array([0, 3, 5], np.int32), z, np.array([0, 8], np.int32)),  # unknown flag bit
        (np.array([0, 3, 5], np.int32), np.array([0, -2], np.int32), z),  # bad slot
        (np.array([0, 3], np.int32), z, z),  # offsets / entries mismatch
    ):
        with pytest.raises(BatchError):
            meta.build_arrays(qsl, slots, flags)


def test_plan_validates_like_ops(cuda_device):
    from paper_2605_14217_b200 import shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.plan import StepPlan
    from paper_2605_14217_b200.pool import AdapterPool

    dims = {k: (n // 16, m // 16) for k, (n, m) in shapes.LLAMA_8B.site_dims().items()}
    tp_pool = AdapterPool(2, 256, lora_sites=dims, lora_capacity=4, lora_rank=16, dtype=torch.bfloat16,
                          device=cuda_device, tp_rank=0, tp_size=2)
    meta = BatchMeta(8, 64, device=cuda_device)
    plan = StepPlan(meta, tp_pool, max_tokens=64)
    x = torch.zeros(64, 128, device=cuda_device, dtype=torch.bfloat16)
    with pytest.raises(ConfigError):  # a TP shard needs the split path
        plan.add_lora_group([torch.zeros(64, 128, device=cuda_device, dtype=torch.bfloat16)], x, 0, ("Wq",))
    pool, _, _ = _mixed_pool(cuda_device)
    plan = StepPlan(meta, pool, max_tokens=64)
    x = torch.zeros(64, 256, device=cuda_device, dtype=torch.bfloat16)
    y = torch.zeros_like(x)
    for bad in (-1, 2):
        with pytest.raises(ShapeError):
            plan.add_lora_group([y], x, bad, ("Wq",))
        with pytest.raises(ShapeError):
            plan.add_reft(y, bad)
    with pytest.raises(ShapeError):
        plan.add_lora_group([y], x, 0, ("Wnope",))
    lora_only = AdapterPool(1, 256, lora_sites={"Wq": (256, 256)}, lora_capacity=2, lora_rank=1,
                            dtype=torch.bfloat16, device=cuda_device)
    with pytest.raises(ShapeError):  # no ReFT slots: ShapeError, not AttributeError
        StepPlan(meta, lora_only, max_tokens=64).add_reft(y, 0)


def test_plan_rows_hint_follows_meta(cuda_device):
    """A plan created before its meta's first build used to keep the K2 team
    size of 0 rows (single-warp teams) forever."""
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.plan import StepPlan

    pool, lo, re = _mixed_pool(cuda_device)
    meta = BatchMeta(32, 2048, device=cuda_device)
    plan = StepPlan(meta, pool, max_tokens=2048)
    assert plan.rows_hint == 2048  # not 0
    rng = np.random.default_rng(3)
    qsl, ids, flags = U.random_entries(rng, 20, lo, p_decode=0.0, max_len=30)
    meta.build_arrays(qsl, pool.entry_arrays(qsl, ids, flags), flags, slot_split=pool.slot_split)
    T = int(qsl[-1])
    x = U.rand_act(rng, 2048, 256, torch.bfloat16, cuda_device)
    y = U.rand_act(rng, 2048, 256, torch.bfloat16, cuda_device)
    plan.add_lora_group([y], x, 1, ("Wq",))
    y_in = U.to_np(y)
    plan.run(run_meta=False)
    assert plan.rows_hint == T
    slots = pool.entry_arrays(qsl, ids, flags)
    ref = U.lora_oracle(y_in[:T], U.to_np(x)[:T], qsl, slots, flags, pool, 1, "Wq")
    helpers.check_close(U.to_np(y)[:T], y_in[:T], ref, "bf16", "plan with the meta's hint")
    fixed = StepPlan(meta, pool, max_tokens=2048, rows_hint=700)
    fixed.add_lora_group([y], x, 1, ("Wq",))
    fixed.run(run_meta=False)
    assert fixed.rows_hint == 700
