"""Oracle and host API vs the LIVE reference, on fresh random inputs.

Runs only where /root/reference is mounted (the build container); the GPU
box relies on the committed golden vectors instead.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference not mounted")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(REF))
    import prefillsim.adapters as RA
    import prefillsim.model as RM

    return RA, RM


def test_masks_fuzz(ref):
    RA, RM = ref
    from oracle import preft_oracle as O

    rng = np.random.default_rng(123)
    for _ in range(300):
        entries = []
        for i in range(int(rng.integers(1, 30))):
            dec = bool(rng.random() < 0.4)
            n = 1 if dec else int(rng.integers(1, 50))
            has = rng.random() < 0.8
            sched = RA.PositionSchedule.ALL_POSITIONS if rng.random() < 0.5 else RA.PositionSchedule.PREFILL_ONLY
            entries.append(RM.SeqEntry(i, tuple(range(n)), n + 3, RM.Phase.DECODE if dec else RM.Phase.PREFILL,
                                       int(rng.integers(0, 5)) if has else None, sched if has else None))
        b = RM.make_batch(entries)
        want = RM.compute_position_mask(b).values
        ad = [-1 if e.adapter_id is None else e.adapter_id for e in entries]
        dec = [e.phase is RM.Phase.DECODE for e in entries]
        allp = [e.schedule is RA.PositionSchedule.ALL_POSITIONS for e in entries]
        assert np.array_equal(O.position_mask(b.query_start_loc, ad, dec, allp), want)


@pytest.mark.parametrize("kind", ["lora", "direft", "loreft"])
def test_deltas_fuzz(ref, kind):
    RA, RM = ref
    from oracle import preft_oracle as O

    rng = np.random.default_rng({"lora": 1, "direft": 2, "loreft": 3}[kind])
    K = RA.AdapterKind(kind)
    for r in (1, 2, 5, 8, 16, 32):
        dims = (64, 96) if K is RA.AdapterKind.LORA else (96,)
        p = RM._perturbed_params(RA.init_zero_delta(K, r, dims, int(rng.integers(1, 1000))), 5, 0.4)
        rows = rng.normal(size=(29, dims[-1]))
        want = RA.delta_for_rows(p, rows)
        got = O.delta_rows(kind, p.prefactor, rows, **{k: getattr(p, k) for k in "A B b R W".split()
                                                        if getattr(p, k) is not None})
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_host_constructors_match_live_reference(ref):
    RA, RM = ref
    from paper_2605_14217_b200 import AdapterKind, ModelConfig, PositionSchedule, build_adapter, perturb_adapter

    cfg_r = RM.ModelConfig(d_model=24, n_layers=3, vocab=31, seed=5)
    cfg_m = ModelConfig(d_model=24, n_layers=3, vocab=31, seed=5)
    for kind in ("lora", "direft", "loreft"):
        a = RM.perturb_adapter(RM.build_adapter(cfg_r, 1, RA.AdapterKind(kind), 4, RA.PositionSchedule.ALL_POSITIONS,
                                                seed=9), seed=10)
        b = perturb_adapter(build_adapter(cfg_m, 1, AdapterKind(kind), 4, PositionSchedule.ALL_POSITIONS, seed=9),
                            seed=10)
        if kind == "lora":
            for key in a.lora_sites:
                for t1, t2 in zip(a.lora_sites[key].tensors, b.lora_sites[key].tensors):
                    assert np.array_equal(t1, t2)
        else:
            for p1, p2 in zip(a.reft_sites, b.reft_sites):
                for t1, t2 in zip(p1.tensors, p2.tensors):
                    assert np.array_equal(t1, t2)
