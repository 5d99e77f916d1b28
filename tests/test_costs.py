"""a14: the bench's byte/flop accounting (paper_2605_14217_b200/costs.py)
reconciled with the reference's own cost model of this path
(costmodel.py:139-249: site_params, adapter_total_params,
adapter_step_cost, lora_down_intensity).

Where the two agree by construction (square sites: flops and weight bytes)
the test demands equality; where they differ on purpose (GQA site widths,
the per-adapter masked-scan activation term, the dispatch-overhead bytes)
the test pins the exact size of the difference, as documented in costs.py.
"""

import sys
from pathlib import Path

import pytest

from paper_2605_14217_b200 import costs, shapes

REF = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def cm():
    if not REF.exists():
        pytest.skip("reference not mounted")
    sys.path.insert(0, str(REF))
    import prefillsim.costmodel as CM

    return CM


def square_dims(d):
    return {"Wq": (d, d)}


def test_lora_square_site_flops_equal_costmodel(cm):
    from prefillsim.adapters import AdapterKind, PositionSchedule
    from prefillsim.model import Phase

    hw = cm.HardwareProfile(peak_flops=1e15, hbm_bandwidth=1e12, link_bandwidth=1e9, bytes_per_param=2,
                            ridge=1000.0, adapter_op_overhead_s=0.0)
    for d, r, toks in ((4096, 1, [24, 7, 100]), (4096, 16, [2048]), (8192, 16, [5, 5, 5, 5])):
        c = cm.adapter_step_cost(AdapterKind.LORA, r, d, PositionSchedule.PREFILL_ONLY, Phase.PREFILL, len(toks),
                                 toks, hw)
        assert costs.lora_group_flops(square_dims(d), ("Wq",), sum(toks), r) == c.flops
        # weight bytes: costmodel's params * bpp per distinct adapter == our D * e * r * (m + n)
        act_ref = len(toks) * 2.0 * sum(toks) * d * 2  # the masked-scan term (costmodel.py:244)
        weights_ref = c.hbm_bytes - act_ref
        ours = costs.lora_group_bytes(square_dims(d), ("Wq",), sum(toks), len(toks), r)
        act_ours = sum(toks) * 2 * (d + 2 * d)
        assert ours - act_ours == weights_ref
        # activations: theirs scale with D (a pass over the whole step per adapter), ours do not
        assert act_ref / act_ours == pytest.approx(len(toks) * 2 / 3)


def test_prefill_only_decode_costs_nothing(cm):
    from prefillsim.adapters import AdapterKind, PositionSchedule
    from prefillsim.model import Phase

    c = cm.adapter_step_cost(AdapterKind.LORA, 1, 4096, PositionSchedule.PREFILL_ONLY, Phase.DECODE, 5, 1,
                             cm.H100_PROFILE)
    assert c.flops == 0 and c.hbm_bytes == 0
    # ours: decode tokens of PREFILL_ONLY adapters are unselected -> T_p = 0, D = 0
    assert costs.lora_group_bytes(square_dims(4096), ("Wq",), 0, 0, 1) == 0


def test_site_params_and_total_params(cm):
    from prefillsim.adapters import AdapterKind

    for r in (1, 8, 16, 32):
        assert costs.reft_layer_params(4096, r) == cm.site_params(AdapterKind.DIREFT, r, 4096)
        assert costs.lora_weight_bytes(square_dims(4096), ("Wq",), r, 1) == cm.site_params(AdapterKind.LORA, r, 4096)
    for shape, ref_shape in ((shapes.LLAMA_8B, cm.SHAPE_8B), (shapes.LLAMA_70B, cm.SHAPE_70B)):
        for r in (1, 16):
            ref_total = cm.adapter_total_params(AdapterKind.LORA, r, ref_shape)
            dims = shape.site_dims()
            ours = shape.n_layers * costs.lora_layer_params(dims, r)
            # GQA: k and v project d -> kv_dim, not d -> d (costmodel.py:163-169 square approximation)
            gqa = shape.n_layers * 2 * r * (shape.d_model - shape.kv_dim)
            assert ours + gqa == ref_total
            square = {k: (shape.d_model if k in ("Wk", "Wv") else n, m) for k, (n, m) in dims.items()}
            assert shape.n_layers * costs.lora_layer_params(square, r) == ref_total
            assert shape.n_layers * costs.reft_layer_params(shape.d_model, r) == cm.adapter_total_params(
                AdapterKind.DIREFT, r, ref_shape)


def test_reft_flops_match_costmodel_up_to_bias(cm):
    from prefillsim.adapters import AdapterKind, PositionSchedule
    from prefillsim.model import Phase

    hw = cm.HardwareProfile(peak_flops=1e15, hbm_bandwidth=1e12, link_bandwidth=1e9, bytes_per_param=2,
                            ridge=1000.0, adapter_op_overhead_s=0.0)
    for kind in (AdapterKind.DIREFT, AdapterKind.LOREFT):
        for r, toks in ((8, [128] * 16), (16, [2048] * 4), (32, [9000, 12000])):
            c = cm.adapter_step_cost(kind, r, 4096, PositionSchedule.PREFILL_ONLY, Phase.PREFILL, len(toks), toks, hw)
            # costmodel: 2 * (2 r d + r) per token; ours 4 r d (bias folded into the intermediate)
            assert c.flops - costs.reft_flops(4096, sum(toks), r) == 2 * r * sum(toks)


def test_intensities_classify_like_costmodel(cm):
    """The whole path is HBM-bound by the reference's own classifier too."""
    from prefillsim.adapters import AdapterKind

    d = 4096
    for r in (1, 16):
        dims = shapes.LLAMA_8B.site_dims()
        for group in shapes.SITE_GROUPS:
            T = 6264
            inten = costs.lora_group_flops(dims, group, T, r) / costs.lora_group_bytes(dims, group, T, 512, r)
            assert not cm.is_compute_bound(inten, cm.H100_PROFILE)
            # and below the rank-r down-projection bound lora_down_intensity (costmodel.py:142-154)
            assert inten <= cm.lora_down_intensity(T, d, r) * len(group) * 2
    inten = costs.reft_flops(d, 65536, 32) / costs.reft_bytes(d, 65536, 512, 32)
    assert not cm.is_compute_bound(inten, cm.H100_PROFILE)
    assert AdapterKind.LORA  # imported from the reference, not restated


def test_closed_forms_without_reference():
    """SURVEY.md 8(d) per-token numbers (runs with or without the reference)."""
    dims = shapes.LLAMA_8B.site_dims()
    unfused = sum(costs.lora_group_bytes(dims, (s,), 1, 0, 1) for s in dims)
    assert unfused == 249_856  # 7 separate sites, 8B, bf16, per selected token
    assert unfused * shapes.LLAMA_8B.n_layers == 7_995_392
    fused = sum(costs.lora_group_bytes(dims, g, 1, 0, 1) for g in shapes.SITE_GROUPS)
    assert fused == unfused - 2 * (2 * 4096 + 4096)  # q/k/v and gate/up read x once
    assert costs.reft_bytes(4096, 1, 0, 16) * 32 == 524_288
    assert costs.split_group_bytes(512, [512, 128, 128], 10, 0, 16) == 10 * 2 * (512 + 2 * 768) + 2 * 10 * 4 * 16 * 3
