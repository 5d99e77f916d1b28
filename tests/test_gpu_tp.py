"""K2 split at the rank-r intermediate (csrc/lora_split.cu) and tensor-parallel
LoRA^P (tp.py, BASELINE config 4) vs the oracle.

* tp_size 1: shrink -> expand equals the reference hook (adapters.py:284-288,
  model.py:449-451) for the tcgen05 and SIMT variants, every dtype;
* tp_size 4 emulated on one GPU: four pool shards registered from the same
  float64 bundles, per-rank shrinks summed (the all-reduce), per-rank expands
  into column / row slices — the assembled output equals the unsharded oracle;
* the NCCL all-reduce path itself through a world-size-1 process group.
"""

import numpy as np
import pytest
import torch

import gpu_util as U
import helpers
from paper_2605_14217_b200 import _lib

pytestmark = pytest.mark.gpu


def _sites(d, kv, f):
    return {"Wq": (d, d), "Wk": (kv, d), "Wv": (kv, d), "Wo": (d, d), "Wgate": (f, d), "Wup": (f, d), "Wdown": (d, f)}


GROUPS = (("Wq", "Wk", "Wv"), ("Wo",), ("Wgate", "Wup"), ("Wdown",))


def _batch(rng, pool, lora_ids, n_entries=24, long=(300, 129, 64)):
    lens = list(rng.integers(1, 40, size=n_entries)) + list(long)
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids, flags = [], []
    for i in range(len(lens)):
        pick = int(rng.integers(0, 10))
        ids.append(None if pick == 9 else int(lora_ids[pick % len(lora_ids)]))
        dec = i < 6 and lens[i] == 1
        flags.append(_lib.ENTRY_DECODE if dec else (_lib.ENTRY_ALL_POSITIONS if pick == 8 else 0))
    return qsl, ids, np.asarray(flags, np.int32)


def _pool(cuda_device, sites, rank, dtype, tp_rank=0, tp_size=1, reft=False):
    from paper_2605_14217_b200.pool import AdapterPool

    return AdapterPool(1, sites["Wq"][1], lora_sites=sites, lora_capacity=5, lora_rank=rank,
                       reft_capacity=2 if reft else 0, reft_rank=16, dtype=dtype, device=cuda_device,
                       tp_rank=tp_rank, tp_size=tp_size)


@pytest.mark.parametrize("variant", [-1, 0])
@pytest.mark.parametrize("rank,mode", [(16, "bf16"), (32, "bf16"), (16, "f32"), (8, "f64")])
def test_split_shrink_expand_matches_oracle(cuda_device, variant, rank, mode):
    """tp_size 1: shrink + expand over every group of a (small) Llama layer,
    with LoRA- and ReFT-class adapters in the same batch."""
    from paper_2605_14217_b200 import AdapterKind
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.tp import SplitWorkspace, apply_lora_group_tp_

    dtype = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[mode]
    rng = np.random.default_rng(rank * 7 + variant + 3)
    sites = _sites(512, 128, 1024)
    pool = _pool(cuda_device, sites, rank, dtype, reft=True)
    ids = [100 + a for a in range(5)]
    for a in ids:
        pool.register(U.random_lora_adapter(rng, a, 1, sites, rank if a % 2 else rank // 2))
    pool.register(U.random_reft_adapter(rng, 7, 1, 512, 16, AdapterKind.DIREFT))
    qsl, eids, flags = _batch(rng, pool, ids + [7])
    T = int(qsl[-1])
    meta = BatchMeta(64, T, device=cuda_device)
    slots = U.stage(meta, pool, qsl, eids, flags)
    ws = SplitWorkspace(meta, pool)
    lib = _lib.load()
    assert lib.preft_set_split_variant(variant) == 0
    try:
        for group in GROUPS:
            m = sites[group[0]][1]
            x = U.rand_act(rng, T, m, dtype, cuda_device)
            ys = [U.rand_act(rng, T, sites[s][0], dtype, cuda_device) for s in group]
            y_in = [U.to_np(y) for y in ys]
            apply_lora_group_tp_(ys, x, meta, pool, 0, group, workspace=ws)
            torch.cuda.synchronize()
            mask = U.oracle_mask(qsl, slots, flags)
            for name, y, yi in zip(group, ys, y_in):
                out = U.to_np(y)
                assert np.array_equal(out[~mask], yi[~mask]), f"{name}: unselected rows touched"
                ref = U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, pool, 0, name)
                helpers.check_close(out, yi, ref, mode, f"{name} r={rank} {mode} variant={variant}")
    finally:
        lib.preft_set_split_variant(-1)


def test_split_tc_forced_rejects_ineligible_shapes(cuda_device):
    """variant 1 (tensor cores only) refuses what tcgen05 cannot run (r = 8)."""
    from paper_2605_14217_b200.errors import ShapeError
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.tp import SplitWorkspace, apply_lora_group_tp_

    sites = {"Wq": (256, 256)}
    pool = _pool(cuda_device, sites, 8, torch.bfloat16)
    rng = np.random.default_rng(0)
    pool.register(U.random_lora_adapter(rng, 1, 1, sites, 8))
    meta = BatchMeta(4, 64, device=cuda_device)
    U.stage(meta, pool, np.array([0, 40], np.int32), [1], np.zeros(1, np.int32))
    lib = _lib.load()
    lib.preft_set_split_variant(1)
    try:
        x = torch.zeros(40, 256, dtype=torch.bfloat16, device=cuda_device)
        y = torch.zeros(40, 256, dtype=torch.bfloat16, device=cuda_device)
        with pytest.raises(ShapeError):
            apply_lora_group_tp_([y], x, meta, pool, 0, ["Wq"], workspace=SplitWorkspace(meta, pool))
    finally:
        lib.preft_set_split_variant(-1)


@pytest.mark.parametrize("tp,widths", [(2, (1024, 256, 2048)), (4, (1024, 256, 2048)), (8, (8192, 1024, 28672))])
def test_tensor_parallel_emulated_on_one_gpu(cuda_device, tp, widths):
    """tp shards of one pool: every rank's shrink partials summed (what the
    NCCL all-reduce does), every rank expands into its slice; the assembled
    result equals the unsharded oracle for column- and row-parallel sites.
    tp = 8 runs BASELINE config 4's own per-rank shapes: Llama-3.1-70B sites
    split 8 ways (k/v n_loc = 128, the tcgen05 expand's minimum width; Wdown
    m_loc = 3584)."""
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.tp import SplitWorkspace, lora_expand_tp_, lora_shrink_tp_

    rng = np.random.default_rng(tp)
    sites = _sites(*widths)
    full = _pool(cuda_device, sites, 16, torch.bfloat16)
    shards = [_pool(cuda_device, sites, 16, torch.bfloat16, tp_rank=r, tp_size=tp) for r in range(tp)]
    ids = [100 + a for a in range(5)]
    for a in ids:
        ad = U.random_lora_adapter(rng, a, 1, sites, 16)
        full.register(ad)
        for p in shards:
            p.register(ad)
    qsl, eids, flags = _batch(rng, full, ids)
    T = int(qsl[-1])
    metas = [BatchMeta(64, T, device=cuda_device) for _ in range(tp)]
    slots = None
    for p, m in zip(shards, metas):
        slots = U.stage(m, p, qsl, eids, flags)
    mask = U.oracle_mask(qsl, slots, flags)
    if tp == 8:
        assert shards[0].lora_shard["Wk"].n_loc == 128 and shards[0].lora_shard["Wdown"].m_loc == 3584
    for group in GROUPS:
        sh = [p.lora_shard[s] for s in group for p in shards[:1]][0]
        n_full = [sites[s][0] for s in group]
        x_full = U.rand_act(rng, T, sites[group[0]][1], torch.bfloat16, cuda_device)
        y_base = [U.rand_act(rng, T, n, torch.bfloat16, cuda_device) for n in n_full]
        # per-rank activations in the layout of the site's TP style
        xs, yss = [], []
        for r, p in enumerate(shards):
            s0 = p.lora_shard[group[0]]
            xs.append(x_full if s0.style == "column" else x_full[:, s0.m0 : s0.m0 + s0.m_loc].contiguous())
            ys = []
            for name, yb in zip(group, y_base):
                sr = p.lora_shard[name]
                if sr.style == "column":
                    ys.append(yb[:, sr.n0 : sr.n0 + sr.n_loc].contiguous())
                else:  # full-width partial output: base on rank 0, zeros elsewhere
                    ys.append(yb.clone() if r == 0 else torch.zeros_like(yb))
            yss.append(ys)
        wss = [SplitWorkspace(m, p) for m, p in zip(metas, shards)]
        Ps = [lora_shrink_tp_(yss[r], xs[r], metas[r], shards[r], 0, group, wss[r]) for r in range(tp)]
        total = sum(P.clone() for P in Ps)  # the all-reduce
        for r in range(tp):
            Ps[r].copy_(total)
            lora_expand_tp_(Ps[r], yss[r], xs[r], metas[r], shards[r], 0, group)
        torch.cuda.synchronize()
        for i, name in enumerate(group):
            if sh.style == "column":
                out = np.concatenate([U.to_np(yss[r][i]) for r in range(tp)], axis=1)
            else:
                out = sum(U.to_np(yss[r][i]) for r in range(tp))
            yi = U.to_np(y_base[i])
            ref = U.lora_oracle(yi, U.to_np(x_full), qsl, slots, flags, full, 0, name)
            assert np.array_equal(out[~mask], yi[~mask]), f"{name}: unselected rows touched"
            helpers.check_close(out, yi, ref, "bf16", f"tp={tp} {name}")


def test_nccl_all_reduce_path_world_size_one(cuda_device, tmp_path):
    """apply_lora_group_tp_'s collective on a real NCCL communicator (one rank)."""
    import torch.distributed as dist

    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.tp import SplitWorkspace, lora_expand_tp_, lora_shrink_tp_

    if dist.is_initialized():
        pytest.skip("a process group already exists")
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=cuda_device)
    try:
        rng = np.random.default_rng(5)
        sites = {"Wq": (512, 512), "Wk": (128, 512), "Wv": (128, 512)}
        pool = _pool(cuda_device, sites, 16, torch.bfloat16)
        for a in range(3):
            pool.register(U.random_lora_adapter(rng, a, 1, sites, 16))
        qsl, eids, flags = _batch(rng, pool, [0, 1, 2])
        T = int(qsl[-1])
        meta = BatchMeta(64, T, device=cuda_device)
        slots = U.stage(meta, pool, qsl, eids, flags)
        x = U.rand_act(rng, T, 512, torch.bfloat16, cuda_device)
        ys = [U.rand_act(rng, T, sites[s][0], torch.bfloat16, cuda_device) for s in sites]
        y_in = [U.to_np(y) for y in ys]
        ws = SplitWorkspace(meta, pool)
        P = lora_shrink_tp_(ys, x, meta, pool, 0, tuple(sites), ws)
        dist.all_reduce(P[:T], op=dist.ReduceOp.SUM)
        lora_expand_tp_(P, ys, x, meta, pool, 0, tuple(sites))
        torch.cuda.synchronize()
        for name, y, yi in zip(sites, ys, y_in):
            ref = U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, pool, 0, name)
            helpers.check_close(U.to_np(y), yi, ref, "bf16", f"nccl {name}")
    finally:
        dist.destroy_process_group()
