"""Pin the CPU oracle to the reference's own outputs (golden vectors).

The oracle (oracle/preft_oracle.py) is the checker for every GPU parity test;
these CPU tests prove it reproduces the reference (tests/golden/ was produced
by prefillsim itself, see tests/golden/make_golden.py).
"""

import numpy as np
import pytest

import helpers
from oracle import preft_oracle as O


def test_masks_bit_exact_against_reference():
    batches = helpers.mask_batches()
    assert len(batches) >= 400
    for b in batches:
        m = O.position_mask(b["qsl"], b["adapter"], b["is_decode"], b["all_pos"])
        assert m.dtype == bool
        assert np.array_equal(m, b["mask"])
        assert O.uniform(m) is b["uniform"]


def test_enumeration_oracle_agrees_with_reference():
    # tests/test_model.py:143-193: the independent per-token walk agrees
    for b in helpers.mask_batches():
        m = O.enumerate_mask(b["qsl"], b["adapter"], b["is_decode"], b["all_pos"], b["prompt_len"], b["cache_start"])
        assert np.array_equal(m, b["mask"])


def test_group_by_slot_contract():
    for b in helpers.mask_batches():
        qsl = b["qsl"]
        slot = b["adapter"]
        tokens, segs, tiles, offs, split = O.group_by_slot(qsl, slot, b["is_decode"], b["all_pos"], tile_tokens=4)
        mask = b["mask"]
        # every selected token exactly once, nothing else
        assert sorted(tokens[:, 0].tolist()) == np.flatnonzero(mask).tolist()
        # sorted by slot, ties in batch order (stable)
        keys = list(zip(tokens[:, 1].tolist(), tokens[:, 0].tolist()))
        assert keys == sorted(keys)
        # segments are maximal runs of one slot and tile them exactly
        assert segs[:, 2].sum() == len(tokens)
        assert len(set(segs[:, 0].tolist())) == len(segs)
        assert tiles[:, 2].sum() == len(tokens)
        assert (tiles[:, 2] <= 4).all() and (tiles[:, 2] >= 1).all()
        assert split == len(tokens)


def test_deltas_match_reference():
    cases = helpers.delta_cases()
    assert len(cases) >= 40
    for c in cases:
        d = O.delta_rows(c["kind"], c["s"], c["rows"], **helpers.params_of(c))
        ref = c["delta"]
        assert d.shape == ref.shape
        np.testing.assert_allclose(d, ref, rtol=1e-12, atol=1e-12 * max(1.0, np.max(np.abs(ref))))


def test_known_answers():
    # tests/test_adapters.py:64-88
    g = helpers.load("deltas.npz")
    d = O.delta_rows("lora", 1.0, np.array([[3.0, 4.0]]), A=np.array([[0.0, 2.0]]), B=np.array([[1.0], [0.0]]))
    assert np.array_equal(d[0], g["ka_lora_delta"]) and np.array_equal(d[0], [8.0, 0.0])
    d = O.delta_rows("direft", 1.0, np.array([[5.0, 7.0]]), A=np.array([[0.0, 1.0]]), B=np.array([[1.0, 0.0]]),
                     b=np.array([0.0]))
    assert np.array_equal(d[0], g["ka_direft_delta"]) and np.array_equal(d[0], [7.0, 0.0])


def test_apply_masked_matches_reference():
    for c in helpers.masked_cases():
        out = O.apply_masked(c["kind"], c["s"], c["sched_all"], c["y"], c.get("x"), c["plen"], **helpers.params_of(c))
        ref = c["out"]
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-13)
        cut = c["y"].shape[0] if c["sched_all"] else min(c["plen"], c["y"].shape[0])
        assert np.array_equal(out[cut:], c["y"][cut:])  # tail bit-identical (adapters.py:318-333)


@pytest.mark.parametrize("name", ["hooks_config1_small.npz", "hooks_config1_small_shuffled.npz"])
def test_forward_hooks_match_reference(name):
    g = helpers.load(name)
    qsl, adapter = g["qsl"], g["adapter"]
    mask = O.position_mask(qsl, adapter, g["is_decode"], g["all_pos"])
    assert np.array_equal(mask, g["mask"])
    params = {}
    for aid in range(9):
        p = {k: g[f"a{aid}_{k}"] for k in ("A", "B", "b", "R", "W") if f"a{aid}_{k}" in g.files}
        p["kind"] = str(g[f"a{aid}_kind"])
        p["s"] = float(g[f"a{aid}_s"])
        params[aid] = p
    lora_slot = np.where([a >= 0 and params[a]["kind"] == "lora" for a in adapter], adapter, -1)
    reft_slot = np.where([a >= 0 and params[a]["kind"] != "lora" for a in adapter], adapter, -1)
    y = O.lora_hook(g["y_base"], g["x"], qsl, mask, lora_slot, params)
    np.testing.assert_allclose(y, g["y_ref"], rtol=1e-12, atol=1e-12)
    h = O.reft_hook(g["h"], qsl, mask, reft_slot, params)
    np.testing.assert_allclose(h, g["h_ref"], rtol=1e-12, atol=1e-12)
    # decode / adapter-less rows untouched, bit for bit
    assert np.array_equal(y[~mask], g["y_base"][~mask])
    assert np.array_equal(h[~mask], g["h"][~mask])


@pytest.mark.parametrize("shuffle", [False, True])
def test_config1_full_size_bit_exact_against_reference(shuffle):
    """BASELINE configs[0] at its stated size (d = 4096, 32 decode + 32 x 128
    prefill, 16 DiReFT^P r8 + 16 LoRA^P r1): the oracle reproduces the
    reference's hook outputs BIT FOR BIT (sha256 of the full f64 arrays, made
    by make_golden.gen_config1_full through _project / the residual hook)."""
    import hashlib

    g, params, x, h = helpers.config1_full(shuffle)
    qsl, ad = g["qsl"], g["adapter"]
    mask = O.position_mask(qsl, ad, g["is_decode"], g["all_pos"])
    assert np.array_equal(mask, g["mask"]) and int(mask.sum()) == 4096 and len(mask) == 4128
    lora = {a: helpers.oracle_params(p) for a, p in params.items() if a >= 16}
    reft = {a: helpers.oracle_params(p) for a, p in params.items() if a < 16}
    delta = O.lora_hook(np.zeros_like(x), x, qsl, mask, np.where(ad >= 16, ad, -1), lora)
    h_out = O.reft_hook(h, qsl, mask, np.where((ad >= 0) & (ad < 16), ad, -1), reft)
    assert hashlib.sha256(delta.tobytes()).hexdigest() == str(g["delta_sha256"])
    assert hashlib.sha256(h_out.tobytes()).hexdigest() == str(g["h_sha256"])
    assert np.array_equal(delta[g["rows"]], g["delta_rows"]) and np.array_equal(h_out[g["rows"]], g["h_rows"])
