"""serving.Scheduler + paging.LruResidency vs the reference engine's step
schedule (engine.py:200-244, 397-489, 528-569), on CPU.

The committed fixture (tests/golden/serving_trace.npz, made by
tests/golden/make_serving_golden.py from the reference itself) pins the
scheduled request ids, worksets, LRU residency and page-ins of every step;
when /root/reference is mounted the same comparison also runs live on fresh
workloads.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

import helpers
from paper_2605_14217_b200.adapters import PositionSchedule
from paper_2605_14217_b200.errors import ConfigError, InfeasibleBatchError
from paper_2605_14217_b200.paging import LruResidency
from paper_2605_14217_b200.serving import RequestSpec, Scheduler, ServeConfig, generate_workload
from paper_2605_14217_b200.workload import AdapterMix, WorkloadConfig

CASES = {
    "uniform": dict(wl=dict(n_requests=120, n_adapters=48, mix=AdapterMix.UNIFORM, seed=3, l_max=256),
                    eng=dict(max_batch=16, max_gpu_adapters=8, step_token_budget=256, chunk_size=None)),
    "skewed_chunked": dict(wl=dict(n_requests=90, n_adapters=30, mix=AdapterMix.SKEWED, seed=5, l_max=200),
                           eng=dict(max_batch=12, max_gpu_adapters=6, step_token_budget=128, chunk_size=40)),
}


def _replay(workload, eng, schedule):
    """Our scheduler + LRU residency, recorded like the reference's StepRecords."""
    cfg = ServeConfig(**eng)
    lru = LruResidency(cfg.max_gpu_adapters)
    rec = {"scheduled": [], "workset": [], "resident": [], "paged_in": [], "prefill_tokens": [], "decode_tokens": []}
    for step in Scheduler(workload, cfg, schedule):
        paged, _, _ = lru.ensure(step.workset, {a: 1 for a in step.workset})
        rec["scheduled"].append(step.decode + [rid for rid, _ in step.prefill])
        rec["workset"].append(list(step.workset))
        rec["resident"].append(list(lru.resident_ids))
        rec["paged_in"].append(paged)
        rec["prefill_tokens"].append(step.prefill_tokens)
        rec["decode_tokens"].append(len(step.decode))
        # the entries K1 will see: decode first (1 token), then prefill chunks
        assert list(np.diff(step.qsl)) == [1] * len(step.decode) + [c for _, c in step.prefill]
    return rec


def _unflatten(g, key):
    flat, off = g[key], g[key + "_off"]
    return [list(flat[off[i]: off[i + 1]]) for i in range(len(off) - 1)]


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("sched", [PositionSchedule.PREFILL_ONLY, PositionSchedule.ALL_POSITIONS])
def test_schedule_matches_reference_golden(name, sched):
    g = helpers.load("serving_trace.npz")
    c = CASES[name]
    tag = f"{name}_{sched.value}"
    rec = _replay(generate_workload(WorkloadConfig(**c["wl"])), c["eng"], sched)
    assert len(rec["scheduled"]) == int(g[f"{tag}_n_steps"])
    for field in ("scheduled", "workset", "resident", "paged_in"):
        assert rec[field] == _unflatten(g, f"{tag}_{field}"), field
    assert rec["prefill_tokens"] == list(g[f"{tag}_prefill_tokens"])
    assert rec["decode_tokens"] == list(g[f"{tag}_decode_tokens"])


def test_prefill_only_adapters_need_no_slot_at_decode():
    """engine.py:521-526: a decode-only step of PREFILL_ONLY requests has an
    empty workset (tests/test_engine.py:193-201)."""
    wl = [RequestSpec(0, 3, 3, 7), RequestSpec(1, 2, 4, 9)]
    steps = list(Scheduler(wl, ServeConfig(max_batch=2, max_gpu_adapters=1, step_token_budget=8)))
    assert steps[0].workset == [7] and steps[0].prefill == [(0, 3)]  # adapter cap 1: request 1 waits
    decode_only = [s for s in steps if not s.prefill]
    assert decode_only and all(s.workset == [] for s in decode_only)


def test_lru_hand_trace_and_capacity():
    """tests/test_engine.py:127-137 and the InfeasibleBatchError rule."""
    lru = LruResidency(2)
    paged, evicted = [], []
    for aid in (1, 2, 3, 1):
        p, e, _ = lru.ensure([aid], {1: 10, 2: 10, 3: 10})
        paged += p
        evicted += e
    assert paged == [1, 2, 3, 1] and evicted == [1, 2]
    with pytest.raises(InfeasibleBatchError):
        lru.ensure([1, 2, 3], {1: 1, 2: 1, 3: 1})
    with pytest.raises(ConfigError):
        ServeConfig(max_batch=8, step_token_budget=4)


REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
@pytest.mark.parametrize("seed", [11, 12, 13])
def test_schedule_matches_live_reference(seed):
    sys.path.insert(0, str(REF))
    from prefillsim.adapters import AdapterKind as RK
    from prefillsim.adapters import PositionSchedule as RS
    from prefillsim.engine import AdapterSetup, EngineConfig, simulate
    from prefillsim.workload import AdapterMix as RMix
    from prefillsim.workload import WorkloadConfig as RW
    from prefillsim.workload import generate_workload as rgen

    rng = np.random.default_rng(seed)
    mix = [AdapterMix.UNIFORM, AdapterMix.SKEWED, AdapterMix.DISTINCT][seed % 3]
    wl_kw = dict(n_requests=int(rng.integers(20, 80)), n_adapters=int(rng.integers(4, 40)), seed=seed,
                 l_max=int(rng.integers(64, 300)))
    eng = dict(max_batch=int(rng.integers(2, 20)), max_gpu_adapters=int(rng.integers(1, 10)),
               chunk_size=None if seed % 2 else int(rng.integers(8, 64)))
    eng["step_token_budget"] = int(rng.integers(eng["max_batch"], 400))
    res = simulate(rgen(RW(mix=RMix(mix.value), **wl_kw)), EngineConfig(warmup=False, **eng),
                   AdapterSetup(kind=RK.LORA, rank=1, schedule=RS.PREFILL_ONLY))
    rec = _replay(generate_workload(WorkloadConfig(mix=mix, **wl_kw)), eng, PositionSchedule.PREFILL_ONLY)
    assert rec["scheduled"] == [list(s.scheduled) for s in res.steps]
    assert rec["workset"] == [list(s.workset) for s in res.steps]
    assert rec["resident"] == [list(s.resident) for s in res.steps]
    assert rec["paged_in"] == [list(s.paged_in) for s in res.steps]


def test_step_entry_flags_follow_the_scheduler_schedule():
    """The K1 flags of a step come from the Scheduler's own schedule map, so
    an ALL_POSITIONS adapter's decode tokens are both in the workset and
    selected by the device mask (model.py:316)."""
    from oracle import preft_oracle as O
    from paper_2605_14217_b200 import _lib

    wl = generate_workload(WorkloadConfig(40, 6, AdapterMix.UNIFORM, seed=2, l_max=48))
    sched_of = {a: (PositionSchedule.ALL_POSITIONS if a % 2 else PositionSchedule.PREFILL_ONLY) for a in range(6)}
    n_dec_selected = 0
    for step in Scheduler(wl, ServeConfig(max_batch=8, max_gpu_adapters=6, step_token_budget=64),
                          lambda a: sched_of[a]):
        flags = step.entry_flags()
        dec = (flags & _lib.ENTRY_DECODE) != 0
        allp = (flags & _lib.ENTRY_ALL_POSITIONS) != 0
        slots = np.array([-1 if a is None else a for a in step.adapter_ids], np.int32)
        mask = O.position_mask(step.qsl, slots, dec, allp)
        for i, a in enumerate(step.adapter_ids):
            sel = bool(mask[step.qsl[i]])
            assert sel == (a is not None and (not dec[i] or sched_of[a] is PositionSchedule.ALL_POSITIONS))
            if sel:
                assert a in step.workset  # every selected token's adapter is resident
            n_dec_selected += int(sel and dec[i])
    assert n_dec_selected > 0
