"""K3 (fused ReFT^P: DiReFT / LoReFT) vs the oracle."""

import numpy as np
import pytest
import torch

import gpu_util as U
import helpers
from paper_2605_14217_b200 import AdapterKind, PositionSchedule, build_adapter

pytestmark = pytest.mark.gpu

MODES = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}


@pytest.mark.parametrize("mode", ["f32", "bf16", "f64"])
@pytest.mark.parametrize("rank", [1, 4, 8, 16, 32])
@pytest.mark.parametrize("d", [256, 4096, 1000])
def test_random_batches(cuda_device, mode, rank, d):
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(rank + d)
    dtype = MODES[mode]
    pool = AdapterPool(2, d, reft_capacity=8, reft_rank=rank, dtype=dtype, device=cuda_device)
    for aid in range(8):
        kind = AdapterKind.DIREFT if aid % 2 else AdapterKind.LOREFT
        pool.register(U.random_reft_adapter(rng, aid, 2, d, max(1, rank // (1 + aid % 2)), kind))
    meta = BatchMeta(128, 8192, device=cuda_device)
    qsl, ids, flags = U.random_entries(rng, 60, list(range(8)), max_len=40)
    slots = U.stage(meta, pool, qsl, ids, flags)
    T = int(qsl[-1])
    h = U.rand_act(rng, T, d, dtype, cuda_device)
    h_in = U.to_np(h)
    apply_reft_(h, meta, pool, 1)
    out = U.to_np(h)
    mask = U.oracle_mask(qsl, slots, flags)
    assert np.array_equal(out[~mask], h_in[~mask])
    ref = U.reft_oracle(h_in, qsl, slots, flags, pool, 1)
    helpers.check_close(out, h_in, ref, mode, f"reft d={d} r={rank}")


@pytest.mark.parametrize("kind", [AdapterKind.DIREFT, AdapterKind.LOREFT])
def test_zero_delta_adapters_leave_stream_bit_identical(cuda_device, kind):
    """tests/test_adapters.py:126-136 / test_acceptance c01: untrained adapters
    are transparent.  LoReFT is exactly zero here (W - R folds to 0), tighter
    than the reference's 1e-12."""
    from paper_2605_14217_b200 import ModelConfig
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    cfg = ModelConfig(d_model=64, n_layers=2, vocab=31, seed=5)
    pool = AdapterPool(2, 64, reft_capacity=3, reft_rank=8, dtype=torch.float32, device=cuda_device)
    for aid in range(3):
        pool.register(build_adapter(cfg, aid, kind, 8, PositionSchedule.ALL_POSITIONS, seed=aid))
    rng = np.random.default_rng(0)
    meta = BatchMeta(32, 1024, device=cuda_device)
    qsl, ids, flags = U.random_entries(rng, 20, [0, 1, 2])
    U.stage(meta, pool, qsl, ids, flags)
    h = U.rand_act(rng, int(qsl[-1]), 64, torch.float32, cuda_device)
    h0 = h.clone()
    for layer in range(2):
        apply_reft_(h, meta, pool, layer)
    assert torch.equal(h, h0)


def test_long_segments_zipf(cuda_device):
    """Config-5-like shape at reduced size: few hot adapters, long prompts,
    LoReFT r=32, d=4096 bf16 (register-resident row path)."""
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(55)
    pool = AdapterPool(1, 4096, reft_capacity=16, reft_rank=32, dtype=torch.bfloat16, device=cuda_device)
    for aid in range(16):
        pool.register(U.random_reft_adapter(rng, aid, 1, 4096, 32, AdapterKind.LOREFT))
    weights = 1.0 / (np.arange(16) + 1.0)
    ids = list(rng.choice(16, size=6, p=weights / weights.sum()))
    lens = rng.integers(1000, 3000, size=6)
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    meta = BatchMeta(16, int(qsl[-1]), tile_tokens=128, device=cuda_device)
    slots = U.stage(meta, pool, qsl, [int(i) for i in ids], np.zeros(6, np.int32))
    h = U.rand_act(rng, int(qsl[-1]), 4096, torch.bfloat16, cuda_device)
    h_in = U.to_np(h)
    apply_reft_(h, meta, pool, 0)
    ref = U.reft_oracle(h_in, qsl, slots, np.zeros(6, np.int32), pool, 0)
    helpers.check_close(U.to_np(h), h_in, ref, "bf16", "zipf loreft r32")
