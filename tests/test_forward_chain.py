"""CPU: pin the chained forward restatement (tests/chain_forward.py) with the
oracle's hooks against the reference's own forward_chunk outputs
(tests/golden/forward_chain.npz, made by make_golden.gen_forward_chain), so
the GPU chain test (test_gpu_forward_chain.py) compares the device hooks
against a forward that is itself pinned to the reference."""

import numpy as np
import pytest

import chain_forward as C


@pytest.mark.parametrize("case,prefix", [("a", "a_"), ("b", "b_"), ("b", "bbase_")])
def test_oracle_chain_matches_reference_forward(case, prefix):
    g = C.fixture()
    cat = C.adapters(g, case)
    logits, hidden = C.forward(g, case, prefix, C.OracleHooks(g, prefix, cat))
    ref = g[prefix + "hidden"]
    for l, h in enumerate(hidden):
        err = np.max(np.abs(h.numpy() - ref[l])) / np.max(np.abs(ref[l]))
        assert err <= 1e-12, f"layer {l}: rel err {err:.3e}"
    err = np.max(np.abs(logits.numpy() - g[prefix + "logits"])) / np.max(np.abs(g[prefix + "logits"]))
    assert err <= 1e-12


def test_fixture_mask_is_the_oracle_mask():
    g = C.fixture()
    for prefix in ("a_", "b_", "bbase_"):
        h = C.OracleHooks(g, prefix, C.adapters(g, prefix[0]))
        assert np.array_equal(h.mask, g[prefix + "mask"])
