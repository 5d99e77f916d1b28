"""Parity at the BASELINE configs' STATED sizes (VERDICT r01 "next" #1).

* config 1 exactly: d = 4096, 16 DiReFT^P r8 + 16 LoRA^P r1, 32 decode +
  32 x 128 prefill entries, decode-first and shuffled, in f64 / f32 / bf16,
  against the oracle on the device's own values AND (f64) against the rows
  the reference itself produced (tests/golden/config1_full*.npz);
* config 5's shape: Zipf-skewed adapters over 512 LoReFT^P r32 slots with
  8k-16k-token prompts (8B width), bf16, on every tensor-core variant;
* config 4's shard widths (70B sites split 8 ways): see
  test_gpu_tp.test_tensor_parallel_emulated_on_one_gpu[8-...].
"""

import numpy as np
import pytest
import torch

import gpu_util as U
import helpers
from paper_2605_14217_b200 import AdapterKind, ModelAdapter, PositionSchedule

pytestmark = pytest.mark.gpu

MODES = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}


def _cfg1_pool(params, dtype, dev):
    from paper_2605_14217_b200.pool import AdapterPool

    d = helpers.CFG1_D
    pool = AdapterPool(1, d, lora_sites={"Wq": (d, d)}, lora_capacity=16, lora_rank=1, reft_capacity=16,
                       reft_rank=8, dtype=dtype, device=dev)
    for a, p in params.items():
        if p.kind is AdapterKind.LORA:
            pool.register(ModelAdapter(a, p.kind, p.rank, PositionSchedule.PREFILL_ONLY, lora_sites={(0, "Wq"): p}))
        else:
            pool.register(ModelAdapter(a, p.kind, p.rank, PositionSchedule.PREFILL_ONLY, reft_sites=(p,)))
    return pool


@pytest.mark.parametrize("shuffle", [False, True])
@pytest.mark.parametrize("mode", ["f64", "f32", "bf16"])
def test_config1_stated_size(cuda_device, mode, shuffle):
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_, apply_reft_

    g, params, x_np, h_np = helpers.config1_full(shuffle)
    dtype = MODES[mode]
    pool = _cfg1_pool(params, dtype, cuda_device)
    qsl = g["qsl"].astype(np.int32)
    ids = [int(a) for a in g["adapter"]]
    flags = g["is_decode"].astype(np.int32)
    meta = BatchMeta(64, 4128, device=cuda_device)
    slots = U.stage(meta, pool, qsl, ids, flags)
    assert np.array_equal(meta.mask_host(), g["mask"])
    T = len(g["mask"])
    rng = np.random.default_rng(11)
    y_np = rng.normal(size=(T, helpers.CFG1_D))
    x = torch.from_numpy(x_np).to(cuda_device, dtype)
    y = torch.from_numpy(y_np).to(cuda_device, dtype)
    h = torch.from_numpy(h_np).to(cuda_device, dtype)
    y_in, h_in = U.to_np(y), U.to_np(h)
    apply_lora_(y, x, meta, pool, 0, "Wq")
    apply_reft_(h, meta, pool, 0)
    y_out, h_out = U.to_np(y), U.to_np(h)
    mask = g["mask"]
    assert np.array_equal(y_out[~mask], y_in[~mask]) and np.array_equal(h_out[~mask], h_in[~mask])
    helpers.check_close(y_out, y_in, U.lora_oracle(y_in, U.to_np(x), qsl, slots, flags, pool, 0, "Wq"), mode,
                        "cfg1 lora vs oracle")
    helpers.check_close(h_out, h_in, U.reft_oracle(h_in, qsl, slots, flags, pool, 0), mode, "cfg1 reft vs oracle")
    if mode == "f64":  # the reference's own rows (no input quantisation in f64)
        rows = g["rows"]
        helpers.check_close(y_out[rows], y_in[rows], y_in[rows] + g["delta_rows"], "f64", "cfg1 lora vs reference")
        helpers.check_close(h_out[rows], h_np[rows], g["h_rows"], "f64", "cfg1 reft vs reference")


def test_config1_through_step_plan_and_graph(cuda_device):
    """The same config-1 step issued by the native StepPlan and replayed from
    a CUDA graph equals the per-call API bit for bit (bf16)."""
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_, apply_reft_
    from paper_2605_14217_b200.plan import StepPlan

    g, params, x_np, h_np = helpers.config1_full(False)
    pool = _cfg1_pool(params, torch.bfloat16, cuda_device)
    qsl = g["qsl"].astype(np.int32)
    flags = g["is_decode"].astype(np.int32)
    meta = BatchMeta(64, 4128, device=cuda_device)
    U.stage(meta, pool, qsl, [int(a) for a in g["adapter"]], flags)
    T = len(g["mask"])
    x = torch.from_numpy(x_np).to(cuda_device, torch.bfloat16)
    y0 = torch.randn(T, helpers.CFG1_D, device=cuda_device).to(torch.bfloat16)
    h0 = torch.from_numpy(h_np).to(cuda_device, torch.bfloat16)
    y_a, h_a = y0.clone(), h0.clone()
    apply_lora_(y_a, x, meta, pool, 0, "Wq")
    apply_reft_(h_a, meta, pool, 0)
    y_b, h_b = y0.clone(), h0.clone()
    plan = StepPlan(meta, pool, max_tokens=T)
    plan.add_lora_group([y_b], x, 0, ("Wq",))
    plan.add_reft(h_b, 0)
    plan.run()
    torch.cuda.synchronize()
    assert torch.equal(y_a, y_b) and torch.equal(h_a, h_b)
    y_b.copy_(y0)
    h_b.copy_(h0)
    graph = plan.capture()
    y_b.copy_(y0)
    h_b.copy_(h0)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_a, y_b) and torch.equal(h_a, h_b)


@pytest.mark.parametrize("variant", [-1, 2, 3])
def test_config5_zipf_loreft_r32_long_prompts(cuda_device, variant):
    """Config 5's shape: 512 LoReFT^P r=32 slots (8B width, one layer), Zipf
    adapter popularity (workload.py:137-140), prompts of 8k-16k tokens plus
    decode entries, bf16 through K3 (automatic / streaming / TMEM-parked);
    every unselected row bit-identical, sampled selected rows of EVERY
    segment against the oracle on the device's own values."""
    from paper_2605_14217_b200 import _lib
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.workload import AdapterMix, WorkloadConfig, assign_adapters

    d, r = 4096, 32
    pool = AdapterPool(1, d, reft_capacity=512, reft_rank=r, dtype=torch.bfloat16, device=cuda_device)
    pool.fill_synthetic_(512, AdapterKind.LOREFT, r, seed=51)
    rng = np.random.default_rng(5)
    n_req = 6
    ids = [int(a) for a in assign_adapters(WorkloadConfig(n_req, 512, AdapterMix.SKEWED, seed=5))]
    lens = rng.integers(8192, 16385, size=n_req)
    n_dec = 16
    all_lens = np.concatenate([np.ones(n_dec, np.int64), lens])
    qsl = np.concatenate([[0], np.cumsum(all_lens)]).astype(np.int32)
    flags = np.array([1] * n_dec + [0] * n_req, np.int32)
    eids = [int(rng.integers(0, 512)) for _ in range(n_dec)] + ids
    T = int(qsl[-1])
    meta = BatchMeta(64, T, device=cuda_device)
    slots = U.stage(meta, pool, qsl, eids, flags)
    h = torch.randn(T, d, device=cuda_device).to(torch.bfloat16)
    h_in = h.clone()
    lib = _lib.load()
    try:
        assert lib.preft_set_reft_variant(variant) == 0
        apply_reft_(h, meta, pool, 0)
    finally:
        lib.preft_set_reft_variant(-1)
    torch.cuda.synchronize()
    mask = U.oracle_mask(qsl, slots, flags)
    mt = torch.from_numpy(~mask).to(cuda_device)
    assert torch.equal(h[mt], h_in[mt])
    # 48 sampled rows per prompt (first, last, random): every segment covered
    params = U.reft_slot_params(pool, 0)
    for i in range(n_dec, n_dec + n_req):
        b, e = int(qsl[i]), int(qsl[i + 1])
        pick = np.unique(np.concatenate([[b, b + 1, e - 2, e - 1], rng.integers(b, e, size=44)]))
        hi = U.to_np(h_in[torch.from_numpy(pick).to(cuda_device)])
        ho = U.to_np(h[torch.from_numpy(pick).to(cuda_device)])
        p = params[int(slots[i])]
        from oracle import preft_oracle as O

        ref = hi + O.delta_rows(p["kind"], p["s"], hi, A=p["A"], B=p["B"], b=p["b"])
        helpers.check_close(ho, hi, ref, "bf16", f"cfg5 prompt {i} ({e - b} tokens, slot {int(slots[i])})")


@pytest.mark.parametrize("rank", [16, 32])
def test_lora_tensor_core_route_cfg2_batch_8b_widths(cuda_device, rank):
    """LoRA^P r16/32 (tcgen05 split pair) at Llama-3.1-8B widths on the full
    cfg2 batch (~240 K1 units: several per CTA, 256-wide expand chunks), one
    launch per group, sampled rows vs the oracle.  This is the case that
    exposed a tcgen05.ld issued under a branch (stale D columns)."""
    import bench
    from paper_2605_14217_b200 import shapes
    from paper_2605_14217_b200.ops import apply_lora_group_

    args = bench.parse([])
    ctx = bench.build_step(args, 0, 1, cuda_device, 256, 256, lora_rank=rank)
    for layer in (0, 17):
        for group in shapes.SITE_GROUPS:
            if len(group) * rank > 64:
                continue  # split into several launches by apply_lora_group_; covered by the narrow-width tests
            x, ys = ctx["acts"][group]
            for y in ys:
                y.copy_(torch.randn(y.shape, device=cuda_device))
            snap = {group: [y.clone() for y in ys]}
            apply_lora_group_(ys, x, ctx["meta"], ctx["pool"], layer, group)
            torch.cuda.synchronize()
            r = bench.check_lora_accumulated(ctx["pool"], ctx["meta"], ctx["qsl"], ctx["slots"], {group: (x, ys)},
                                             snap, [layer], k=96, seed=layer)
            assert r["status"] == "pass", (layer, group, r)
