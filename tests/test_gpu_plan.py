"""StepPlan (csrc/plan.cu): the native executor that issues a whole step —
K1, then every layer's fused LoRA^P groups and ReFT^P site — in one C call
(the reference's `layer x entry` loop, model.py:504-546).  The plan must
produce exactly what the per-call API produces (same kernels, same order),
eagerly and when captured into a CUDA graph, and match the oracle."""

import numpy as np
import pytest
import torch

import gpu_util as U
import helpers
from paper_2605_14217_b200 import AdapterKind

pytestmark = pytest.mark.gpu


def _setup(cuda_device, rng, d=1024, n_layers=2):
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.pool import AdapterPool

    sites = {"Wq": (d, d), "Wk": (d // 4, d), "Wv": (d // 4, d), "Wo": (d, d)}
    pool = AdapterPool(n_layers, d, lora_sites=sites, lora_capacity=4, lora_rank=1, reft_capacity=4, reft_rank=16,
                       dtype=torch.bfloat16, device=cuda_device)
    for aid in range(4):
        pool.register(U.random_lora_adapter(rng, aid, n_layers, sites, 1))
        kind = AdapterKind.DIREFT if aid % 2 else AdapterKind.LOREFT
        pool.register(U.random_reft_adapter(rng, 10 + aid, n_layers, d, 16, kind))
    qsl, ids, flags = U.random_entries(rng, 24, [0, 1, 2, 3, 10, 11, 12, 13], max_len=200)
    meta = BatchMeta(32, int(qsl[-1]), device=cuda_device)
    slots = U.stage(meta, pool, qsl, ids, flags)
    T = int(qsl[-1])
    acts = []
    for _ in range(n_layers):
        x = U.rand_act(rng, T, d, torch.bfloat16, cuda_device)
        ys = [U.rand_act(rng, T, sites[s][0], torch.bfloat16, cuda_device) for s in ("Wq", "Wk", "Wv")]
        yo = U.rand_act(rng, T, d, torch.bfloat16, cuda_device)
        h = U.rand_act(rng, T, d, torch.bfloat16, cuda_device)
        acts.append((x, ys, yo, h))
    return pool, meta, qsl, slots, flags, acts


def _clone(acts):
    return [(x, [y.clone() for y in ys], yo.clone(), h.clone()) for x, ys, yo, h in acts]


def _direct(pool, meta, acts):
    from paper_2605_14217_b200.ops import apply_lora_group_, apply_reft_

    for layer, (x, ys, yo, h) in enumerate(acts):
        apply_lora_group_(ys, x, meta, pool, layer, ("Wq", "Wk", "Wv"))
        apply_lora_group_([yo], x, meta, pool, layer, ("Wo",))
        apply_reft_(h, meta, pool, layer)
    torch.cuda.synchronize()


def _plan(pool, meta, acts):
    from paper_2605_14217_b200.plan import StepPlan

    plan = StepPlan(meta, pool)
    for layer, (x, ys, yo, h) in enumerate(acts):
        plan.add_lora_group(ys, x, layer, ("Wq", "Wk", "Wv"))
        plan.add_lora_group([yo], x, layer, ("Wo",))
        plan.add_reft(h, layer)
    assert plan.launches_per_run == 2 + 3 * len(acts)
    return plan


def _same(a, b):
    for (_, ys_a, yo_a, h_a), (_, ys_b, yo_b, h_b) in zip(a, b):
        for ya, yb in zip(ys_a + [yo_a, h_a], ys_b + [yo_b, h_b]):
            assert torch.equal(ya.view(torch.int16), yb.view(torch.int16))


@pytest.mark.parametrize("run_meta", [True, False])
def test_plan_matches_per_call_api_and_oracle(cuda_device, run_meta):
    rng = np.random.default_rng(11 + run_meta)
    pool, meta, qsl, slots, flags, acts = _setup(cuda_device, rng)
    ref = _clone(acts)
    _direct(pool, meta, ref)
    got = _clone(acts)
    plan = _plan(pool, meta, got)
    plan.run(run_meta=run_meta)
    torch.cuda.synchronize()
    _same(got, ref)
    # and against the oracle, layer 0
    mask = U.oracle_mask(qsl, slots, flags)
    x, ys, yo, h = acts[0]
    for name, y_in, y_out in zip(("Wq", "Wk", "Wv"), ys, got[0][1]):
        yi = U.to_np(y_in)
        out = U.to_np(y_out)
        assert np.array_equal(out[~mask], yi[~mask])
        helpers.check_close(out, yi, U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, pool, 0, name), "bf16",
                            f"plan {name}")
    hi = U.to_np(h)
    helpers.check_close(U.to_np(got[0][3]), hi, U.reft_oracle(hi, qsl, slots, flags, pool, 0), "bf16", "plan reft")


@pytest.mark.parametrize("run_meta", [True, False])
def test_plan_graph_replay_is_bit_identical(cuda_device, run_meta):
    rng = np.random.default_rng(21 + run_meta)
    pool, meta, qsl, slots, flags, acts = _setup(cuda_device, rng)
    ref = _clone(acts)
    _direct(pool, meta, ref)
    got = _clone(acts)
    plan = _plan(pool, meta, got)
    g = plan.capture(run_meta=run_meta)  # includes one eager warm-up run: restore the inputs
    for _ in range(2):
        for (_, ys_g, yo_g, h_g), (_, ys0, yo0, h0) in zip(got, acts):
            for dst, src in zip(ys_g + [yo_g, h_g], ys0 + [yo0, h0]):
                dst.copy_(src)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        _same(got, ref)


def test_capture_steps_runs_k_steps_and_times_tagged_launches(cuda_device):
    """StepPlan.capture_steps: K consecutive steps in one graph equal K eager
    runs bit for bit, and the tagged launches' events (captured as external
    event-record nodes) come back from collect_timing() after a replay."""
    from paper_2605_14217_b200.plan import StepPlan

    rng = np.random.default_rng(31)
    pool, meta, qsl, slots, flags, acts = _setup(cuda_device, rng)
    k = 3
    eager = _clone(acts)
    plan_e = _plan(pool, meta, eager)
    for _ in range(k):
        plan_e.run()
    torch.cuda.synchronize()
    got = _clone(acts)
    plan = StepPlan(meta, pool)
    for layer, (x, ys, yo, h) in enumerate(got):
        plan.add_lora_group(ys, x, layer, ("Wq", "Wk", "Wv"), tag=1)
        plan.add_lora_group([yo], x, layer, ("Wo",))
        plan.add_reft(h, layer)
    g = plan.capture_steps(k, timing_tag=1)  # its warm-up run edits the inputs: restore them
    for (_, ys_g, yo_g, h_g), (_, ys0, yo0, h0) in zip(got, acts):
        for dst, src in zip(ys_g + [yo_g, h_g], ys0 + [yo0, h0]):
            dst.copy_(src)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    _same(got, eager)
    total, count = plan.collect_timing()
    assert count == k * len(acts) and total > 0
