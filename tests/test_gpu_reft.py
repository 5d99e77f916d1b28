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


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
@pytest.mark.parametrize("rank", [16, 32])
@pytest.mark.parametrize("d", [128, 1024, 2048, 4096, 8192])
def test_tensor_core_and_simt_variants(cuda_device, variant, rank, d):
    """The tcgen05 kernels (1 automatic, 2 streaming, 3 resident) and the SIMT
    kernel (0) on the same mixed batch: short (partial-chunk) and multi-unit
    segments, decode and adapter-less entries, and LoRA-class tokens
    interleaved in the sorted list (the ReFT kernel must skip their units)."""
    if variant == 3 and not (d % 1024 == 0 and d // 1024 in ((1, 2, 4, 8) if rank == 16 else (1, 2, 4))):
        pytest.skip("the resident kernel covers d = 1024 * {1, 2, 4, 8} (r = 32: up to 4096)")
    from paper_2605_14217_b200 import _lib
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_, apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(d + rank + variant)
    sites = {"Wq": (d, d)}
    pool = AdapterPool(1, d, lora_sites=sites, lora_capacity=3, lora_rank=1, reft_capacity=6, reft_rank=rank,
                       dtype=torch.bfloat16, device=cuda_device)
    assert pool.reft_tc
    for aid in range(3):
        pool.register(U.random_lora_adapter(rng, 100 + aid, 1, sites, 1))
    for aid in range(6):
        kind = AdapterKind.DIREFT if aid % 2 else AdapterKind.LOREFT
        pool.register(U.random_reft_adapter(rng, aid, 1, d, rank if aid < 4 else rank // 2, kind))
    lens = [1] * 10 + list(rng.integers(1, 40, size=20)) + [300, 129, 128, 700]
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids, flags = [], []
    for i, n in enumerate(lens):
        pick = rng.integers(0, 10)
        ids.append(None if pick == 9 else (100 + pick % 3 if pick >= 6 else int(pick % 6)))
        flags.append(_lib.ENTRY_DECODE if n == 1 and i < 10 else 0)
    flags = np.asarray(flags, dtype=np.int32)
    meta = BatchMeta(64, int(qsl[-1]), device=cuda_device)
    slots = U.stage(meta, pool, qsl, ids, flags)
    T = int(qsl[-1])
    h = U.rand_act(rng, T, d, torch.bfloat16, cuda_device)
    x = U.rand_act(rng, T, d, torch.bfloat16, cuda_device)
    y = U.rand_act(rng, T, d, torch.bfloat16, cuda_device)
    h_in, y_in = U.to_np(h), U.to_np(y)
    lib = _lib.load()
    try:
        assert lib.preft_set_reft_variant(variant) == 0
        apply_lora_(y, x, meta, pool, 0, "Wq")
        apply_reft_(h, meta, pool, 0)
        torch.cuda.synchronize()
    finally:
        lib.preft_set_reft_variant(-1)
    mask = U.oracle_mask(qsl, slots, flags)
    out = U.to_np(h)
    assert np.array_equal(out[~mask], h_in[~mask])
    ref = U.reft_oracle(h_in, qsl, slots, flags, pool, 0)
    helpers.check_close(out, h_in, ref, "bf16", f"reft variant {variant} d={d} r={rank}")
    lora_rows = np.isin(slots, [pool.info(100 + a).slot for a in range(3)])
    assert lora_rows.any()
    yref = U.lora_oracle(y_in, U.to_np(x), qsl, slots, flags, pool, 0, "Wq")
    helpers.check_close(U.to_np(y), y_in, yref, "bf16", "lora alongside reft")


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


def test_tiled_bt_is_b_transposed(cuda_device):
    """The tensor-core copy of B (pool.reft_Bt, core-matrix tiled) is exactly
    B^T of the SIMT slab, for registered and synthetic adapters."""
    from paper_2605_14217_b200.pool import AdapterPool, untile_kmajor

    rng = np.random.default_rng(3)
    pool = AdapterPool(2, 256, reft_capacity=4, reft_rank=16, dtype=torch.bfloat16, device=cuda_device)
    pool.register(U.random_reft_adapter(rng, 7, 2, 256, 16, AdapterKind.DIREFT))
    pool.register(U.random_reft_adapter(rng, 8, 2, 256, 8, AdapterKind.LOREFT))
    pool.fill_synthetic_(2, AdapterKind.DIREFT, 16, first_id=20)
    assert torch.equal(untile_kmajor(pool.reft_Bt), pool.reft_B.transpose(-1, -2))


@pytest.mark.parametrize("flags", [39, 5, 45])
def test_tensor_core_pipeline_knobs_keep_results(cuda_device, flags):
    """The K3-TC pipeline knobs (reduce epilogue, unpaced shrink, early
    re-read) change scheduling only: same parity, unselected rows untouched."""
    from paper_2605_14217_b200 import _lib
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(flags)
    d = 2048
    pool = AdapterPool(1, d, reft_capacity=4, reft_rank=16, dtype=torch.bfloat16, device=cuda_device)
    for aid in range(4):
        pool.register(U.random_reft_adapter(rng, aid, 1, d, 16, AdapterKind.DIREFT if aid % 2 else AdapterKind.LOREFT))
    lens = [1] * 6 + list(rng.integers(1, 60, size=10)) + [300, 257]
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = [int(i) % 4 if i % 7 else None for i in range(len(lens))]
    flags_e = np.array([_lib.ENTRY_DECODE] * 6 + [0] * (len(lens) - 6), dtype=np.int32)
    meta = BatchMeta(32, int(qsl[-1]), device=cuda_device)
    slots = U.stage(meta, pool, qsl, ids, flags_e)
    h = U.rand_act(rng, int(qsl[-1]), d, torch.bfloat16, cuda_device)
    h[3, 5] = -0.0  # a negative zero in an unselected row must survive the reduce epilogue
    h_in = U.to_np(h)
    neg0 = h[3, 5].clone()
    lib = _lib.load()
    assert lib.preft_set_reft_tc_flags(flags, -1) == 0
    try:
        apply_reft_(h, meta, pool, 0)
        torch.cuda.synchronize()
    finally:
        lib.preft_set_reft_tc_flags(-1, -1)
    mask = U.oracle_mask(qsl, slots, flags_e)
    out = U.to_np(h)
    assert np.array_equal(out[~mask], h_in[~mask])
    assert torch.equal(h[3, 5].view(torch.int16), neg0.view(torch.int16))
    ref = U.reft_oracle(h_in, qsl, slots, flags_e, pool, 0)
    helpers.check_close(out, h_in, ref, "bf16", f"reft knobs {flags}")


def test_colaunch_eager_and_graph(cuda_device):
    """d = 4096, r = 16 runs the TMEM-parked kernel and the streaming kernel at
    once (forked stream, unit list split).  The result matches the oracle (and
    the streaming kernel alone within the same tolerance: the two sum the
    shrink partials in different orders), and a CUDA graph that captured the
    fork/join replays it bit for bit."""
    from paper_2605_14217_b200 import _lib
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(7)
    d = 4096
    pool = AdapterPool(1, d, reft_capacity=6, reft_rank=16, dtype=torch.bfloat16, device=cuda_device)
    for aid in range(6):
        pool.register(U.random_reft_adapter(rng, aid, 1, d, 16, AdapterKind.DIREFT if aid % 2 else AdapterKind.LOREFT))
    lens = [1] * 8 + list(rng.integers(1, 300, size=24)) + [2048, 1024]
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = [int(i) % 6 if i % 5 else None for i in range(len(lens))]
    flags = np.array([_lib.ENTRY_DECODE] * 8 + [0] * (len(lens) - 8), dtype=np.int32)
    meta = BatchMeta(64, int(qsl[-1]), device=cuda_device)
    slots = U.stage(meta, pool, qsl, ids, flags)
    h0 = U.rand_act(rng, int(qsl[-1]), d, torch.bfloat16, cuda_device)
    h_in = U.to_np(h0)
    mask = U.oracle_mask(qsl, slots, flags)
    ref = U.reft_oracle(h_in, qsl, slots, flags, pool, 0)
    lib = _lib.load()
    try:
        assert lib.preft_set_reft_variant(-1) == 0
        h_co = h0.clone()
        apply_reft_(h_co, meta, pool, 0)
        torch.cuda.synchronize()
        out = U.to_np(h_co)
        assert np.array_equal(out[~mask], h_in[~mask])
        helpers.check_close(out, h_in, ref, "bf16", "reft co-launch d=4096 r=16")
        h_g = h0.clone()
        s = torch.cuda.Stream(cuda_device)
        s.wait_stream(torch.cuda.current_stream(cuda_device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            apply_reft_(h_g, meta, pool, 0)
        for _ in range(2):
            h_g.copy_(h0)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(h_g.view(torch.int16), h_co.view(torch.int16))
    finally:
        lib.preft_set_reft_variant(-1)


@pytest.mark.parametrize("variant", [2, 3])
@pytest.mark.parametrize("kind", ["all_decode", "no_adapter", "one_long", "unit_edges"])
def test_tensor_core_edge_batches(cuda_device, variant, kind):
    """The streaming (2) and resident (3) tcgen05 ReFT kernels at d = 2048,
    r = 32 on edge batches: nothing selected, no adapter at all, one long
    prompt of one adapter (many units of the same adapter back to back), and
    prompt lengths around the chunk (16) and unit (64) boundaries.  Unselected
    rows bit-identical, selected rows against the oracle."""
    from paper_2605_14217_b200 import _lib
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    d, rank = 2048, 32
    D = _lib.ENTRY_DECODE
    if kind == "all_decode":
        lens, ids, fl = [1] * 24, [i % 6 for i in range(24)], [D] * 24
    elif kind == "no_adapter":
        lens, ids, fl = [7, 64, 1, 130], [None] * 4, [0, 0, D, 0]
    elif kind == "one_long":
        lens, ids, fl = [1, 1, 1000, 1], [3, 4, 3, 3], [D, D, 0, D]
    else:
        lens = [1, 15, 16, 17, 63, 64, 65, 128, 129, 1, 1]
        ids = [0, 0, 1, 1, 2, 2, 3, 4, 4, 5, None]
        fl = [0] * 9 + [D, 0]
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    flags = np.asarray(fl, dtype=np.int32)
    rng = np.random.default_rng(11)
    pool = AdapterPool(1, d, reft_capacity=6, reft_rank=rank, dtype=torch.bfloat16, device=cuda_device)
    for aid in range(6):
        kind_ = AdapterKind.DIREFT if aid % 2 else AdapterKind.LOREFT
        pool.register(U.random_reft_adapter(rng, aid, 1, d, rank, kind_))
    meta = BatchMeta(len(ids), int(qsl[-1]), device=cuda_device)
    slots = U.stage(meta, pool, qsl, ids, flags)
    T = int(qsl[-1])
    h = U.rand_act(rng, T, d, torch.bfloat16, cuda_device)
    h_in = U.to_np(h)
    lib = _lib.load()
    try:
        assert lib.preft_set_reft_variant(variant) == 0
        apply_reft_(h, meta, pool, 0)
        torch.cuda.synchronize()
    finally:
        lib.preft_set_reft_variant(-1)
    meta.check_errors()
    mask = U.oracle_mask(qsl, slots, flags)
    out = U.to_np(h)
    assert np.array_equal(out[~mask], h_in[~mask])
    if mask.any():
        ref = U.reft_oracle(h_in, qsl, slots, flags, pool, 0)
        helpers.check_close(out, h_in, ref, "bf16", f"reft {kind} variant {variant}")
