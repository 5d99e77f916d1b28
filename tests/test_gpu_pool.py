"""HBM adapter pool: registration (K4), weight sync semantics (engine.py:676-697),
graph safety."""

import numpy as np
import pytest
import torch

import gpu_util as U
import helpers
from paper_2605_14217_b200 import AdapterKind, ModelAdapter, PositionSchedule
from paper_2605_14217_b200.errors import InfeasibleBatchError, RankError, ShapeError, StateError, SyncError

pytestmark = pytest.mark.gpu

SITES = {"Wq": (64, 32), "Wk": (16, 32)}


def _pool(device, dtype=torch.float32, cap=4, rank=4):
    from paper_2605_14217_b200.pool import AdapterPool

    return AdapterPool(2, 32, lora_sites=SITES, lora_capacity=cap, lora_rank=rank, reft_capacity=2, reft_rank=4,
                       dtype=dtype, device=device)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64])
def test_upload_rounds_once_and_zero_pads(cuda_device, dtype):
    rng = np.random.default_rng(0)
    pool = _pool(cuda_device, dtype)
    ad = U.random_lora_adapter(rng, 7, 2, SITES, 3)
    slot = pool.register(ad)
    for (layer, name), p in ad.lora_sites.items():
        A = pool.lora_A[name][layer, slot]
        Bt = pool.lora_Bt[name][layer, slot]
        want_A = torch.from_numpy(p.A).to(dtype)  # torch's f64 -> dtype cast rounds to nearest even
        assert torch.equal(A[:3].cpu(), want_A)
        assert torch.equal(Bt[:3].cpu(), torch.from_numpy(np.ascontiguousarray(p.B.T)).to(dtype))
        assert not A[3:].any() and not Bt[3:].any()
        assert float(pool.lora_scale[name][layer, slot]) == pytest.approx(32.0 / 3, rel=1e-7)


def test_register_errors_and_capacity(cuda_device):
    rng = np.random.default_rng(1)
    pool = _pool(cuda_device, cap=2, rank=4)
    pool.register(U.random_lora_adapter(rng, 0, 2, SITES, 2))
    pool.register(U.random_lora_adapter(rng, 1, 2, SITES, 2))
    with pytest.raises(InfeasibleBatchError):
        pool.register(U.random_lora_adapter(rng, 2, 2, SITES, 2))
    with pytest.raises(RankError):
        pool.register(U.random_lora_adapter(rng, 0, 2, SITES, 8))
    with pytest.raises(ShapeError):
        pool.register(U.random_lora_adapter(rng, 0, 2, {"Wq": (64, 16)}, 2))
    pool.unregister(1)
    assert 1 not in pool
    pool.register(U.random_lora_adapter(rng, 2, 2, SITES, 2))
    with pytest.raises(StateError):
        pool.unregister(99)


def test_sync_is_validate_all_then_apply(cuda_device):
    rng = np.random.default_rng(2)
    pool = _pool(cuda_device)
    a0 = U.random_lora_adapter(rng, 0, 2, SITES, 2)
    a1 = U.random_lora_adapter(rng, 1, 2, SITES, 2)
    pool.register(a0)
    pool.register(a1)
    before = pool.lora_A["Wq"].clone()
    good = U.random_lora_adapter(rng, 0, 2, SITES, 2)
    bad_rank = U.random_lora_adapter(rng, 1, 2, SITES, 3)
    with pytest.raises(SyncError):
        pool.sync([(0, good), (1, bad_rank)])
    assert torch.equal(pool.lora_A["Wq"], before)  # nothing applied
    with pytest.raises(SyncError):
        pool.sync([(5, good)])
    sched = ModelAdapter(0, AdapterKind.LORA, 2, PositionSchedule.ALL_POSITIONS, lora_sites=good.lora_sites)
    with pytest.raises(SyncError):
        pool.sync([(0, sched)])
    pool.sync([(0, good)])
    assert pool.info(0).version == 1
    assert not torch.equal(pool.lora_A["Wq"], before)


def test_graph_replay_sees_synced_weights_and_new_batches(cuda_device):
    """Capture K1 + K2 once; replay after a weight sync and after staging a
    different batch into the same fixed-address workspace."""
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_

    rng = np.random.default_rng(3)
    pool = _pool(cuda_device)
    for aid in range(3):
        pool.register(U.random_lora_adapter(rng, aid, 2, SITES, 4))
    meta = BatchMeta(32, 512, device=cuda_device)
    T = 200
    x = U.rand_act(rng, T, 32, torch.float32, cuda_device)
    y = torch.zeros(T, 64, device=cuda_device)
    qsl, ids, flags = U.random_entries(rng, 12, [0, 1, 2], max_len=16)
    U.stage(meta, pool, qsl, ids, flags)
    s = torch.cuda.Stream(cuda_device)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside capture
        apply_lora_(y, x, meta, pool, 1, "Wq", stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        meta.launch(stream=s)
        apply_lora_(y, x, meta, pool, 1, "Wq", stream=s)

    def replay_and_check(qsl, ids, flags):
        slots = pool.entry_arrays(qsl, ids, flags)
        n = int(qsl[-1])
        y.zero_()
        meta.set_slot_split(pool.slot_split)
        meta.build_arrays(qsl, slots, flags)  # stages + runs K1 eagerly
        g.replay()  # K1 again (idempotent) + K2 from the graph
        torch.cuda.synchronize()
        ref = U.lora_oracle(np.zeros((T, 64)), U.to_np(x), np.append(qsl, T) if n < T else qsl, np.append(slots, -1) if n < T else slots,
                            np.append(flags, 0) if n < T else flags, pool, 1, "Wq")
        helpers.check_close(U.to_np(y), np.zeros((T, 64)), ref, "f32", "graph replay")

    replay_and_check(qsl, ids, flags)
    pool.sync([(1, U.random_lora_adapter(rng, 1, 2, SITES, 4))])
    replay_and_check(qsl, ids, flags)
    qsl2, ids2, flags2 = U.random_entries(rng, 9, [0, 1, 2], max_len=20)
    replay_and_check(qsl2, ids2, flags2)


def test_register_from_adp1_directory_matches_in_memory(cuda_device, tmp_path):
    """The ADP1 bulk loader fills the pool with exactly the bits of the
    in-memory bundle it was saved from (LoRA with the tiled tensor-core copy,
    and ReFT)."""
    import gpu_util as U
    from paper_2605_14217_b200 import AdapterKind
    from paper_2605_14217_b200.adapter_io import register_dir, save_model_adapter
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(4)
    sites = {"Wq": (256, 128), "Wk": (128, 128)}
    lora = U.random_lora_adapter(rng, 11, 2, sites, 16)
    reft = U.random_reft_adapter(rng, 12, 2, 128, 16, AdapterKind.DIREFT)
    pools = [AdapterPool(2, 128, lora_sites=sites, lora_capacity=2, lora_rank=16, reft_capacity=2, reft_rank=16,
                         dtype=torch.bfloat16, device=cuda_device) for _ in range(2)]
    for a in (lora, reft):
        pools[0].register(a)
        register_dir(pools[1], save_model_adapter(a, tmp_path / str(a.adapter_id)))
    torch.cuda.synchronize()
    for a in (lora, reft):
        va = pools[0].slot_views(a.kind, pools[0].info(a.adapter_id).slot)
        vb = pools[1].slot_views(a.kind, pools[1].info(a.adapter_id).slot)
        assert all(torch.equal(x, y) for x, y in zip(va, vb))
