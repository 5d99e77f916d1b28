"""Paging (paging.PagedAdapterPool) and the serving replay (serving.py) on the
GPU: LRU page-ins restore slots bit-exactly, and a replayed reference
schedule (decode-first mixed batches, adapter cap, LRU paging) produces the
oracle's outputs step after step."""

import numpy as np
import pytest
import torch

import gpu_util as U
import helpers
from paper_2605_14217_b200 import AdapterKind, _lib
from paper_2605_14217_b200.adapters import PositionSchedule

pytestmark = pytest.mark.gpu

SITES = {"Wq": (256, 256), "Wk": (64, 256)}


def _catalogue(rng, n, kind="lora"):
    out = {}
    for a in range(n):
        if kind == "lora":
            out[a] = U.random_lora_adapter(rng, a, 2, SITES, 4 if a % 2 else 2)
        else:
            out[a] = U.random_reft_adapter(rng, a, 2, 256, 16, AdapterKind.DIREFT)
    return out


def test_page_in_restores_slots_bit_exactly(cuda_device):
    from paper_2605_14217_b200.paging import PagedAdapterPool
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(0)
    cat = _catalogue(rng, 6)
    pool = AdapterPool(2, 256, lora_sites=SITES, lora_capacity=3, lora_rank=4, dtype=torch.bfloat16,
                       device=cuda_device)
    ref = AdapterPool(2, 256, lora_sites=SITES, lora_capacity=6, lora_rank=4, dtype=torch.bfloat16,
                      device=cuda_device)
    for a in cat.values():
        ref.register(a)
    paged = PagedAdapterPool(pool, cat)
    for needed in ([0, 1, 2], [3], [4, 0], [5, 1], [2, 3, 4], [0]):
        paged.ensure(needed)
        torch.cuda.synchronize()
        for aid in needed:
            mine = pool.slot_views(AdapterKind.LORA, pool.info(aid).slot)
            theirs = ref.slot_views(AdapterKind.LORA, ref.info(aid).slot)
            assert all(torch.equal(a, b) for a, b in zip(mine, theirs)), f"adapter {aid} slot differs"
    assert paged.page_ins > 6 and paged.evictions > 0
    assert set(paged.resident_ids) == set(aid for aid in cat if aid in pool)


@pytest.mark.parametrize("kind", ["lora", "reft"])
def test_serving_replay_matches_oracle(cuda_device, kind):
    """A small Punica stream under a 4-slot pool: every step's adapter outputs
    equal the oracle on the catalogue's (device-rounded) parameters."""
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_group_, apply_reft_
    from paper_2605_14217_b200.paging import PagedAdapterPool
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.serving import Scheduler, ServeConfig, generate_workload
    from paper_2605_14217_b200.workload import AdapterMix, WorkloadConfig

    rng = np.random.default_rng(1 if kind == "lora" else 2)
    cat = _catalogue(rng, 10, kind)
    if kind == "lora":
        pool = AdapterPool(2, 256, lora_sites=SITES, lora_capacity=4, lora_rank=4, dtype=torch.bfloat16,
                           device=cuda_device)
        full = AdapterPool(2, 256, lora_sites=SITES, lora_capacity=10, lora_rank=4, dtype=torch.bfloat16,
                           device=cuda_device)
    else:
        pool = AdapterPool(2, 256, reft_capacity=4, reft_rank=16, dtype=torch.bfloat16, device=cuda_device)
        full = AdapterPool(2, 256, reft_capacity=10, reft_rank=16, dtype=torch.bfloat16, device=cuda_device)
    for a in cat.values():
        full.register(a)
    paged = PagedAdapterPool(pool, cat)
    wl = generate_workload(WorkloadConfig(24, 10, AdapterMix.UNIFORM, seed=4, l_max=64))
    cfg = ServeConfig(max_batch=8, max_gpu_adapters=4, step_token_budget=96, chunk_size=32)
    meta = BatchMeta(64, 96, device=cuda_device)
    n_checked = 0
    for step in Scheduler(wl, cfg, PositionSchedule.PREFILL_ONLY):
        paged.ensure(step.workset)
        flags = (step.decode_flags * _lib.ENTRY_DECODE).astype(np.int32)
        slots = pool.entry_arrays(step.qsl, step.adapter_ids, flags)
        meta.set_slot_split(pool.slot_split)
        meta.build_arrays(step.qsl, slots, flags)
        T = int(step.qsl[-1])
        # the oracle runs on the unpaged pool: same adapters, same rounding
        full_slots = full.entry_arrays(step.qsl, step.adapter_ids, flags)
        mask = U.oracle_mask(step.qsl, full_slots, flags)
        assert np.array_equal(meta.mask_host(), mask)
        for layer in range(2):
            if kind == "lora":
                x = U.rand_act(rng, T, 256, torch.bfloat16, cuda_device)
                ys = [U.rand_act(rng, T, SITES[s][0], torch.bfloat16, cuda_device) for s in SITES]
                y_in = [U.to_np(y) for y in ys]
                apply_lora_group_(ys, x, meta, pool, layer, tuple(SITES))
                for name, y, yi in zip(SITES, ys, y_in):
                    ref = U.lora_oracle(yi, U.to_np(x), step.qsl, full_slots, flags, full, layer, name)
                    helpers.check_close(U.to_np(y), yi, ref, "bf16", f"step {step.index} {name}")
            else:
                h = U.rand_act(rng, T, 256, torch.bfloat16, cuda_device)
                h_in = U.to_np(h)
                apply_reft_(h, meta, pool, layer)
                ref = U.reft_oracle(h_in, step.qsl, full_slots, flags, full, layer)
                helpers.check_close(U.to_np(h), h_in, ref, "bf16", f"step {step.index} reft")
        n_checked += 1
    assert n_checked > 10 and paged.evictions > 0
