"""K2 (fused LoRA^P) vs the oracle and the reference's golden outputs."""

import numpy as np
import pytest
import torch

import gpu_util as U
import helpers
from paper_2605_14217_b200 import AdapterKind, AdapterParams, ModelAdapter, PositionSchedule, ScalingRule
from paper_2605_14217_b200.errors import BatchError, ShapeError

pytestmark = pytest.mark.gpu

MODES = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}


def _golden_pool(g, dtype, device):
    from paper_2605_14217_b200.pool import AdapterPool

    d = int(g["d"])
    pool = AdapterPool(1, d, lora_sites={"Wq": (d, d)}, lora_capacity=4, lora_rank=1, reft_capacity=5, reft_rank=8,
                       dtype=dtype, device=device)
    for aid in range(9):
        kind = AdapterKind(str(g[f"a{aid}_kind"]))
        rank = int(g[f"a{aid}_rank"])
        kw = {k: g[f"a{aid}_{k}"] for k in ("A", "B", "b", "R", "W") if f"a{aid}_{k}" in g.files}
        dims = (d, d) if kind is AdapterKind.LORA else (d,)
        p = AdapterParams(kind, rank, dims, ScalingRule.constant(float(g[f"a{aid}_s"])), **kw)
        if kind is AdapterKind.LORA:
            pool.register(ModelAdapter(aid, kind, rank, PositionSchedule.PREFILL_ONLY, lora_sites={(0, "Wq"): p}))
        else:
            pool.register(ModelAdapter(aid, kind, rank, PositionSchedule.PREFILL_ONLY, reft_sites=(p,)))
    return pool


@pytest.mark.parametrize("name", ["hooks_config1_small.npz", "hooks_config1_small_shuffled.npz"])
@pytest.mark.parametrize("mode", ["f64", "f32", "bf16"])
def test_config1_small_against_reference(cuda_device, name, mode):
    """Reduced BASELINE config 1 (mixed LoRA^P r=1 + DiReFT^P r=8 + LoReFT^P,
    decode entries first or shuffled) through both hook kernels."""
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_, apply_reft_

    g = helpers.load(name)
    dtype = MODES[mode]
    pool = _golden_pool(g, dtype, cuda_device)
    meta = BatchMeta(64, 4096, device=cuda_device)
    qsl = g["qsl"].astype(np.int32)
    ids = [None if a < 0 else int(a) for a in g["adapter"]]
    flags = (g["is_decode"].astype(np.int32) * 1 | g["all_pos"].astype(np.int32) * 2).astype(np.int32)
    slots = U.stage(meta, pool, qsl, ids, flags)
    assert np.array_equal(meta.mask_host(), g["mask"])

    x = torch.from_numpy(g["x"]).to(cuda_device, dtype)
    y = torch.from_numpy(g["y_base"]).to(cuda_device, dtype)
    h = torch.from_numpy(g["h"]).to(cuda_device, dtype)
    y_in, h_in = U.to_np(y), U.to_np(h)
    apply_lora_(y, x, meta, pool, 0, "Wq")
    apply_reft_(h, meta, pool, 0)
    y_out, h_out = U.to_np(y), U.to_np(h)
    mask = g["mask"]
    # untouched rows are bit-identical (tests/test_model.py:298-327 contract)
    assert np.array_equal(y_out[~mask], y_in[~mask])
    assert np.array_equal(h_out[~mask], h_in[~mask])
    if mode == "f64":
        helpers.check_close(y_out, y_in, g["y_ref"], "f64", "lora vs reference")
        helpers.check_close(h_out, h_in, g["h_ref"], "f64", "reft vs reference")
    # oracle on the exact (quantised) device inputs
    y_ref = U.lora_oracle(y_in, U.to_np(x), qsl, slots, flags, pool, 0, "Wq")
    h_ref = U.reft_oracle(h_in, qsl, slots, flags, pool, 0)
    helpers.check_close(y_out, y_in, y_ref, mode, "lora vs oracle")
    helpers.check_close(h_out, h_in, h_ref, mode, "reft vs oracle")


SITES = {"Wq": (256, 128), "Wk": (64, 128), "Wv": (64, 128), "Wo": (128, 256)}


@pytest.mark.parametrize("mode", ["f32", "bf16", "f64"])
@pytest.mark.parametrize("rank", [1, 2, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("group", [("Wq",), ("Wq", "Wk"), ("Wq", "Wk", "Wv"), ("Wo",)])
def test_random_batches_groups_ranks(cuda_device, mode, rank, group):
    """Groups wider than one launch (nsites * r > 64: rank-32 q/k/v, rank-64
    pairs) run as several launches over the same x (ops.lora_site_chunks)."""
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_group_
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(rank * 7 + len(group))
    dtype = MODES[mode]
    pool = AdapterPool(2, 128, lora_sites=SITES, lora_capacity=12, lora_rank=rank, dtype=dtype, device=cuda_device)
    for aid in range(10):
        r = rank if aid % 3 else max(1, rank // 2)  # mixed ranks in one pool
        pool.register(U.random_lora_adapter(rng, 100 + aid, 2, SITES, r))
    meta = BatchMeta(256, 8192, device=cuda_device)
    qsl, ids, flags = U.random_entries(rng, 120, [100 + a for a in range(10)], max_len=50)
    slots = U.stage(meta, pool, qsl, ids, flags)
    T = int(qsl[-1])
    m = SITES[group[0]][1]
    x = U.rand_act(rng, T, m, dtype, cuda_device)
    ys = [U.rand_act(rng, T, SITES[s][0], dtype, cuda_device) for s in group]
    y_in = [U.to_np(y) for y in ys]
    layer = 1
    apply_lora_group_(ys, x, meta, pool, layer, group)
    mask = U.oracle_mask(qsl, slots, flags)
    for s, y, yi in zip(group, ys, y_in):
        out = U.to_np(y)
        assert np.array_equal(out[~mask], yi[~mask])
        ref = U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, pool, layer, s)
        helpers.check_close(out, yi, ref, mode, f"{s} r={rank}")


@pytest.mark.parametrize("variant", [0, 1, 2, 4, 8, -1])
@pytest.mark.parametrize("mode", ["f32", "bf16"])
@pytest.mark.parametrize("rank", [1, 2, 4])
def test_team_and_warp_variants(cuda_device, variant, mode, rank):
    """Every K2 variant (warp-per-row kernel; team kernel with 1/2/4/8 warps
    per row; automatic) against the oracle on aligned widths."""
    from paper_2605_14217_b200 import _lib
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_group_
    from paper_2605_14217_b200.pool import AdapterPool

    sites = {"Wq": (2048, 2048), "Wk": (512, 2048), "Wv": (512, 2048), "Wgate": (6144, 2048), "Wup": (6144, 2048),
             "Wdown": (2048, 6144)}
    rng = np.random.default_rng(rank * 3 + variant)
    dtype = MODES[mode]
    pool = AdapterPool(1, 2048, lora_sites=sites, lora_capacity=6, lora_rank=rank, dtype=dtype, device=cuda_device)
    for aid in range(6):
        pool.register(U.random_lora_adapter(rng, aid, 1, sites, rank))
    meta = BatchMeta(128, 4096, device=cuda_device)
    qsl, ids, flags = U.random_entries(rng, 40, list(range(6)), max_len=24)
    slots = U.stage(meta, pool, qsl, ids, flags)
    T = int(qsl[-1])
    lib = _lib.load()
    try:
        assert lib.preft_set_lora_variant(variant) == 0
        for group in (("Wq", "Wk", "Wv"), ("Wgate", "Wup"), ("Wdown",)):
            x = U.rand_act(rng, T, sites[group[0]][1], dtype, cuda_device)
            ys = [U.rand_act(rng, T, sites[s][0], dtype, cuda_device) for s in group]
            y_in = [U.to_np(y) for y in ys]
            apply_lora_group_(ys, x, meta, pool, 0, group)
            mask = U.oracle_mask(qsl, slots, flags)
            for s, y, yi in zip(group, ys, y_in):
                out = U.to_np(y)
                assert np.array_equal(out[~mask], yi[~mask])
                ref = U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, pool, 0, s)
                helpers.check_close(out, yi, ref, mode, f"variant {variant} {s} r={rank}")
    finally:
        lib.preft_set_lora_variant(-1)


@pytest.mark.parametrize("mode", ["f32", "bf16"])
def test_odd_widths_use_scalar_path(cuda_device, mode):
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_group_
    from paper_2605_14217_b200.pool import AdapterPool

    sites = {"Wgate": (45, 37), "Wup": (45, 37)}
    rng = np.random.default_rng(5)
    dtype = MODES[mode]
    pool = AdapterPool(1, 37, lora_sites=sites, lora_capacity=4, lora_rank=4, dtype=dtype, device=cuda_device)
    for aid in range(4):
        pool.register(U.random_lora_adapter(rng, aid, 1, sites, 3))
    meta = BatchMeta(64, 4096, device=cuda_device)
    qsl, ids, flags = U.random_entries(rng, 30, list(range(4)))
    slots = U.stage(meta, pool, qsl, ids, flags)
    T = int(qsl[-1])
    x = U.rand_act(rng, T, 37, dtype, cuda_device)
    ys = [U.rand_act(rng, T, 45, dtype, cuda_device) for _ in sites]
    y_in = [U.to_np(y) for y in ys]
    apply_lora_group_(ys, x, meta, pool, 0, tuple(sites))
    for s, y, yi in zip(sites, ys, y_in):
        ref = U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, pool, 0, s)
        helpers.check_close(U.to_np(y), yi, ref, mode, s)


def test_llama8b_shapes_sampled_parity(cuda_device):
    """Full Llama-3.1-8B site widths (one layer, 64 adapters r=1, bf16):
    every unselected row bit-identical; a sample of selected rows against
    the oracle on the device's own values."""
    from paper_2605_14217_b200 import shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_group_
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(8)
    sites = shapes.LLAMA_8B.site_dims()
    pool = AdapterPool(1, 4096, lora_sites=sites, lora_capacity=64, lora_rank=1, dtype=torch.bfloat16,
                       device=cuda_device)
    ids = pool.fill_synthetic_(64, AdapterKind.LORA, 1, seed=3)
    meta = BatchMeta(256, 16384, device=cuda_device)
    qsl, eids, flags = U.random_entries(rng, 96, ids, max_len=64)
    slots = U.stage(meta, pool, qsl, eids, flags)
    T = int(qsl[-1])
    mask = U.oracle_mask(qsl, slots, flags)
    for group in (("Wq", "Wk", "Wv"), ("Wo",), ("Wgate", "Wup"), ("Wdown",)):
        m = sites[group[0]][1]
        x = U.rand_act(rng, T, m, torch.bfloat16, cuda_device)
        ys = [U.rand_act(rng, T, sites[s][0], torch.bfloat16, cuda_device) for s in group]
        y_in = [y.clone() for y in ys]
        apply_lora_group_(ys, x, meta, pool, 0, group)
        sample = rng.choice(np.flatnonzero(mask), size=min(24, int(mask.sum())), replace=False)
        keep = np.zeros(T, bool)
        keep[sample] = True
        for s, y, yi in zip(group, ys, y_in):
            assert torch.equal(y[torch.from_numpy(~mask).to(cuda_device)], yi[torch.from_numpy(~mask).to(cuda_device)])
            # oracle on the sampled rows only (other rows masked out of the check)
            yi_np, x_np, out = U.to_np(yi), U.to_np(x), U.to_np(y)
            sub_mask_flags = flags.copy()
            ref = U.lora_oracle(yi_np, x_np, qsl, slots, flags, pool, 0, s)
            helpers.check_close(out[keep], yi_np[keep], ref[keep], "bf16", f"8B {s}")


def test_errors_map_to_reference_exceptions(cuda_device):
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_
    from paper_2605_14217_b200.pool import AdapterPool

    pool = AdapterPool(1, 64, lora_sites={"Wq": (64, 64)}, lora_capacity=2, lora_rank=2, dtype=torch.float32,
                       device=cuda_device)
    meta = BatchMeta(8, 64, device=cuda_device)
    with pytest.raises(BatchError):  # unknown adapter id (model.py:470-472)
        U.stage(meta, pool, np.array([0, 3], np.int32), [5], np.zeros(1, np.int32))
    U.stage(meta, pool, np.array([0, 3], np.int32), [None], np.zeros(1, np.int32))
    x = torch.zeros(3, 64, device=cuda_device)
    with pytest.raises(ShapeError):
        apply_lora_(torch.zeros(3, 32, device=cuda_device), x, meta, pool, 0, "Wq")
    with pytest.raises(ShapeError):
        apply_lora_(torch.zeros(3, 64, device=cuda_device, dtype=torch.bfloat16), x, meta, pool, 0, "Wq")
    with pytest.raises(ShapeError):
        apply_lora_(torch.zeros(2, 64, device=cuda_device), x, meta, pool, 0, "Wq")


TC_SITES = {"Wq": (512, 512), "Wk": (128, 512), "Wv": (128, 512), "Wo": (512, 512), "Wgate": (1024, 512),
            "Wup": (1024, 512), "Wdown": (512, 1024)}


@pytest.mark.parametrize("variant", [-1, 0])
@pytest.mark.parametrize("rank", [16, 32])
def test_rank16_32_tensor_core_route(cuda_device, variant, rank):
    """bf16 LoRA^P at r = 16 / 32 through the standard apply API: the tcgen05
    split pair (shrink into the meta's workspace, then expand) when eligible
    (variant -1), the SIMT kernels when forced (variant 0); both against the
    oracle, with mixed ranks, decode entries and adapter-less entries, every
    group of a (narrow) Llama layer, and through a StepPlan + CUDA graph."""
    from paper_2605_14217_b200 import _lib, shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_group_
    from paper_2605_14217_b200.plan import StepPlan
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(rank + variant)
    pool = AdapterPool(2, 512, lora_sites=TC_SITES, lora_capacity=10, lora_rank=rank, dtype=torch.bfloat16,
                       device=cuda_device)
    for aid in range(10):
        pool.register(U.random_lora_adapter(rng, aid, 2, TC_SITES, rank if aid % 3 else rank // 2))
    meta = BatchMeta(128, 4096, device=cuda_device)
    qsl, ids, flags = U.random_entries(rng, 70, list(range(10)), max_len=90)
    slots = U.stage(meta, pool, qsl, ids, flags)
    T = int(qsl[-1])
    mask = U.oracle_mask(qsl, slots, flags)
    lib = _lib.load()
    assert lib.preft_set_lora_variant(variant) == 0
    try:
        acts = {}
        for group in shapes.SITE_GROUPS:
            x = U.rand_act(rng, T, TC_SITES[group[0]][1], torch.bfloat16, cuda_device)
            ys = [U.rand_act(rng, T, TC_SITES[s][0], torch.bfloat16, cuda_device) for s in group]
            acts[group] = (x, ys, [U.to_np(y) for y in ys])
            apply_lora_group_(ys, x, meta, pool, 1, group)
        torch.cuda.synchronize()
        assert meta.lora_part is not None  # the workspace the TC route uses
        for group, (x, ys, y_in) in acts.items():
            for s, y, yi in zip(group, ys, y_in):
                out = U.to_np(y)
                assert np.array_equal(out[~mask], yi[~mask])
                ref = U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, pool, 1, s)
                helpers.check_close(out, yi, ref, "bf16", f"r={rank} variant={variant} {s}")
        # the same through a plan replayed from a CUDA graph: equal to the per-call API bit for bit
        base = {g: [y.clone() for y in ys] for g, (x, ys, _) in acts.items()}
        plan = StepPlan(meta, pool, max_tokens=T)
        for group, (x, ys, _) in acts.items():
            plan.add_lora_group(ys, x, 0, group)
        graph = plan.capture(run_meta=False)
        for g, (x, ys, _) in acts.items():
            for y, b in zip(ys, base[g]):
                y.copy_(b)
        graph.replay()
        torch.cuda.synchronize()
        for group, (x, ys, _) in acts.items():
            want = [b.clone() for b in base[group]]
            apply_lora_group_(want, x, meta, pool, 0, group)
            for y, w in zip(ys, want):
                assert torch.equal(y, w)
    finally:
        lib.preft_set_lora_variant(-1)


def _edge_batch(kind):
    """(qsl, ids, flags) of the edge batches the tcgen05 routes must handle."""
    from paper_2605_14217_b200 import _lib

    D = _lib.ENTRY_DECODE
    if kind == "all_decode":  # nothing selected: every entry a decode token of a prefill-only adapter
        lens, ids, fl = [1] * 24, [i % 10 for i in range(24)], [D] * 24
    elif kind == "no_adapter":
        lens, ids, fl = [7, 64, 1, 130], [None] * 4, [0, 0, D, 0]
    elif kind == "one_long":  # one adapter, one long prompt: many units of the same adapter
        lens, ids, fl = [1, 1, 1000, 1], [3, 4, 3, 3], [D, D, 0, D]
    else:  # unit_edges: prompt lengths around the 16-row chunk and 64-row unit, repeated adapters
        lens = [1, 15, 16, 17, 63, 64, 65, 128, 129, 1, 1]
        ids = [0, 0, 1, 1, 2, 2, 3, 4, 4, 5, None]
        fl = [0] * 9 + [D, 0]
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    return qsl, ids, np.array(fl, np.int32)


@pytest.mark.parametrize("kind", ["all_decode", "no_adapter", "one_long", "unit_edges"])
def test_tensor_core_edge_batches(cuda_device, kind):
    """The r = 16 tcgen05 route (split pair, or the fused kernel / dynamic grabs
    in the subprocess reruns below) on edge batches: nothing selected, no
    adapter at all, one long prompt of one adapter, and prompt lengths around
    the chunk (16) and unit (64) boundaries.  Unselected rows bit-identical,
    selected rows against the oracle."""
    from paper_2605_14217_b200 import shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_group_
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(7)
    pool = AdapterPool(1, 512, lora_sites=TC_SITES, lora_capacity=10, lora_rank=16, dtype=torch.bfloat16,
                       device=cuda_device)
    for aid in range(10):
        pool.register(U.random_lora_adapter(rng, aid, 1, TC_SITES, 16))
    qsl, ids, flags = _edge_batch(kind)
    meta = BatchMeta(len(ids), int(qsl[-1]), device=cuda_device)
    slots = U.stage(meta, pool, qsl, ids, flags)
    T = int(qsl[-1])
    mask = U.oracle_mask(qsl, slots, flags)
    for group in shapes.SITE_GROUPS:
        x = U.rand_act(rng, T, TC_SITES[group[0]][1], torch.bfloat16, cuda_device)
        ys = [U.rand_act(rng, T, TC_SITES[s][0], torch.bfloat16, cuda_device) for s in group]
        y_in = [U.to_np(y) for y in ys]
        apply_lora_group_(ys, x, meta, pool, 0, group)
        torch.cuda.synchronize()
        for s, y, yi in zip(group, ys, y_in):
            out = U.to_np(y)
            assert np.array_equal(out[~mask], yi[~mask]), (kind, s)
            if mask.any():
                ref = U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, pool, 0, s)
                helpers.check_close(out, yi, ref, "bf16", f"{kind} {s}")
    meta.check_errors()


def test_tensor_core_route_with_dynamic_grabs_forced():
    """The dynamic expand (item grabs from a global counter) on every TC
    launch, not only the wide groups it is chosen for: the r = 16/32 route's
    parity and CUDA-graph checks rerun in a process with PREFT_SPLIT_DYN=1
    (the switch is read once per process)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, PREFT_SPLIT_DYN="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                        str(root / "tests" / "test_gpu_lora.py"), "-k", "rank16_32_tensor_core_route or tensor_core_edge"],
                       capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_tensor_core_route_through_the_fused_kernel():
    """preft_lora_apply's r >= 16 route through the fused kernel (one launch:
    shrink -> one-rank exchange -> expand) on every eligible launch: the
    route's parity and CUDA-graph checks rerun with PREFT_LORA_FUSED=1 (the
    automatic choice takes it only for inputs of >= 8192 columns)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, PREFT_LORA_FUSED="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                        str(root / "tests" / "test_gpu_lora.py"), "-k", "rank16_32_tensor_core_route or tensor_core_edge"],
                       capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
