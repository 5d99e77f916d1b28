"""Host-side API mirror vs the reference (CPU only): constructors, validation,
errors, ADP1 serialization, batch metadata validation, workload sampler."""

import numpy as np
import pytest

import helpers
from paper_2605_14217_b200 import (
    AdapterKind,
    AdapterParams,
    ForwardBatch,
    ModelConfig,
    Phase,
    PositionSchedule,
    ScalingRule,
    SeqEntry,
    adapter_byte_size,
    build_adapter,
    init_zero_delta,
    load_adapter,
    make_batch,
    mask_uniform,
    perturb_adapter,
    save_adapter,
    scaling_prefactor,
)
from paper_2605_14217_b200.batch import _perturbed_params
from paper_2605_14217_b200.errors import BatchError, ConfigError, DomainError, RankError, ShapeError

K, P = AdapterKind, PositionSchedule


def test_prefactor_values_and_errors():
    # tests/test_adapters.py:36-51
    assert scaling_prefactor(ScalingRule.constant(2.0), 64) == 2.0
    assert scaling_prefactor(ScalingRule.alpha_over_r(32.0), 32) == 1.0
    assert scaling_prefactor(ScalingRule.alpha_over_r(32.0), 8) == 4.0
    assert scaling_prefactor(ScalingRule.inv_sqrt_r(), 16) == 0.25
    with pytest.raises(RankError):
        scaling_prefactor(ScalingRule.inv_sqrt_r(), 0)
    with pytest.raises(DomainError):
        ScalingRule.constant(0.0)
    with pytest.raises(DomainError):
        ScalingRule.alpha_over_r(-1.0)
    with pytest.raises(DomainError):
        ScalingRule("bogus")


def test_init_zero_delta_bit_exact_with_reference():
    g = helpers.load("init_io.npz")
    for key, (kind, rank, dims, seed) in {
        "lora": (K.LORA, 4, (8, 6), 2),
        "direft": (K.DIREFT, 5, (32,), 3),
        "loreft": (K.LOREFT, 3, (16,), 4),
    }.items():
        p = init_zero_delta(kind, rank, dims, seed)
        for name in ("A", "B", "b", "R", "W"):
            if f"init_{key}_{name}" in g.files:
                assert np.array_equal(getattr(p, name).view(np.uint64), g[f"init_{key}_{name}"].view(np.uint64))


def test_build_and_perturb_bit_exact_with_reference():
    g = helpers.load("init_io.npz")
    cfg = ModelConfig(d_model=16, n_layers=2, vocab=31, seed=5, max_seq=64)
    for key, (kind, rank) in {"lora": (K.LORA, 2), "direft": (K.DIREFT, 4), "loreft": (K.LOREFT, 3)}.items():
        ad = perturb_adapter(build_adapter(cfg, 7, kind, rank, P.PREFILL_ONLY, seed=11), seed=12, sigma=0.2)
        if kind is K.LORA:
            for (layer, name), p in sorted(ad.lora_sites.items()):
                assert np.array_equal(p.A, g[f"build_{key}_{layer}_{name}_A"])
                assert np.array_equal(p.B, g[f"build_{key}_{layer}_{name}_B"])
        else:
            for layer, p in enumerate(ad.reft_sites):
                for name in ("A", "B", "b", "R", "W"):
                    if f"build_{key}_{layer}_{name}" in g.files:
                        assert np.array_equal(getattr(p, name), g[f"build_{key}_{layer}_{name}"])


@pytest.mark.parametrize("key,kind,rank,dims,seed", [
    ("lora", K.LORA, 4, (8, 6), 2), ("direft", K.DIREFT, 5, (32,), 3), ("loreft", K.LOREFT, 3, (16,), 4)])
def test_adp1_bytes_identical_to_reference(tmp_path, key, kind, rank, dims, seed):
    g = helpers.load("init_io.npz")
    ref_bytes = g[f"adp1_{key}"].tobytes()
    p = _perturbed_params(init_zero_delta(kind, rank, dims, seed), seed + 1000, 0.3)
    path = tmp_path / "a.bin"
    save_adapter(p, path)
    assert path.read_bytes() == ref_bytes
    (tmp_path / "r.bin").write_bytes(ref_bytes)
    back = load_adapter(tmp_path / "r.bin")
    assert back.kind is kind and back.rank == rank and back.dims == dims and back.scaling == p.scaling
    for a, b in zip(back.tensors, p.tensors):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_load_rejects_garbage_and_truncation(tmp_path):
    (tmp_path / "junk.bin").write_bytes(b"not an adapter")
    with pytest.raises(ShapeError):
        load_adapter(tmp_path / "junk.bin")
    g = helpers.load("init_io.npz")
    (tmp_path / "t.bin").write_bytes(g["adp1_lora"].tobytes()[:-3])
    with pytest.raises(ShapeError):
        load_adapter(tmp_path / "t.bin")


def test_params_validation_and_write_protection():
    with pytest.raises(ShapeError):
        AdapterParams(K.LORA, 2, (4, 4), ScalingRule.constant(1.0), A=np.zeros((2, 5)), B=np.zeros((4, 2)))
    with pytest.raises(ShapeError):
        AdapterParams(K.DIREFT, 2, (4,), ScalingRule.constant(1.0), A=np.zeros((2, 4)), B=np.zeros((2, 4)))
    with pytest.raises(RankError):
        init_zero_delta(K.DIREFT, 17, (16,), seed=0)
    with pytest.raises(RankError):
        init_zero_delta(K.LORA, 9, (8, 32), seed=0)
    p = init_zero_delta(K.DIREFT, 2, (8,), seed=0)
    with pytest.raises(ValueError):
        p.B[0, 0] = 1.0
    assert adapter_byte_size(init_zero_delta(K.DIREFT, 8, (64,), seed=0), 2) == 2064
    assert adapter_byte_size(init_zero_delta(K.LORA, 1, (64, 64), seed=0), 2) == 256


def test_loreft_device_fold_is_exact_algebra():
    p = _perturbed_params(init_zero_delta(K.LOREFT, 3, (12,), 4), 9, 0.3)
    shrink, expand, bias = p.device_operands()
    h = np.random.default_rng(0).normal(size=(5, 12))
    ref = p.prefactor * ((h @ p.W.T + p.b - h @ p.R.T) @ p.R)
    got = p.prefactor * ((h @ shrink.T + bias) @ expand)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-13)
    z = init_zero_delta(K.LOREFT, 3, (12,), 4)
    assert not z.device_operands()[0].any()  # W - R == 0 exactly at zero init


def test_batch_validation():
    # tests/test_model.py:88-108
    e = SeqEntry(0, (1, 2, 3), 3, Phase.PREFILL)
    with pytest.raises(BatchError):
        ForwardBatch((e,), (0, 2))
    with pytest.raises(BatchError):
        ForwardBatch((e,), (1, 4))
    b = make_batch([e])
    assert b.query_start_loc == (0, 3) and b.total_tokens == 3
    with pytest.raises(BatchError):
        SeqEntry(0, (1, 2), 4, Phase.DECODE)
    with pytest.raises(BatchError):
        make_batch([SeqEntry(0, (1,), 1, Phase.PREFILL), SeqEntry(0, (2,), 1, Phase.PREFILL)])
    with pytest.raises(BatchError):
        SeqEntry(0, (1,), 1, Phase.PREFILL, adapter_id=3)
    with pytest.raises(BatchError):
        make_batch([])
    with pytest.raises(ConfigError):
        ModelConfig(8, 1, 10, seed=0, lora_targets=("Wx",))


def test_host_uniform_flag_matches_reference():
    for b in helpers.mask_batches():
        entries = []
        for i in range(len(b["adapter"])):
            n = int(b["qsl"][i + 1] - b["qsl"][i])
            aid = int(b["adapter"][i])
            entries.append(SeqEntry(i, tuple(range(n)), int(b["prompt_len"][i]),
                                    Phase.DECODE if b["is_decode"][i] else Phase.PREFILL,
                                    None if aid < 0 else aid,
                                    None if aid < 0 else (P.ALL_POSITIONS if b["all_pos"][i] else P.PREFILL_ONLY)))
        assert mask_uniform(make_batch(entries)) is b["uniform"]


def test_workload_sampler_bit_exact_with_reference():
    from paper_2605_14217_b200.workload import (AdapterMix, WorkloadConfig, assign_adapters, sample_prompt_lens,
                                                sample_total_lens)

    g = helpers.load("workload.npz")
    for mix in AdapterMix:
        cfg = WorkloadConfig(1000, 512, mix, seed=3, l_max=2048)
        p = sample_prompt_lens(cfg)
        assert np.array_equal(p, g[f"{mix.value}_prompt"])
        assert np.array_equal(sample_total_lens(cfg, p), g[f"{mix.value}_total"])
        assert np.array_equal(np.asarray(assign_adapters(cfg)), g[f"{mix.value}_adapters"])


def test_routing_covers_every_request_once():
    from paper_2605_14217_b200.workload import hot_replicas, owner_of, route_requests, shard_adapters

    rng = np.random.default_rng(0)
    w = 1.0 / (np.arange(512) + 1.0)
    ids = list(rng.choice(512, size=2000, p=w / w.sum())) + [None] * 10
    for world in (1, 2, 4, 8):
        shards = [shard_adapters(512, r, world) for r in range(world)]
        assert sorted(sum(shards, [])) == list(range(512))
        reps = hot_replicas(ids, world)
        routed = route_requests(ids, world, reps)
        flat = sorted(sum(routed, []))
        assert flat == list(range(len(ids)))
        for r, reqs in enumerate(routed):
            for i in reqs:
                a = ids[i]
                if a is not None and a not in reps:
                    assert owner_of(a, world) == r
        if world == 8:
            assert 0 in reps  # adapter 0 carries ~14.7% > 1/8 of the Zipf load


def test_adapter_directory_round_trip_bit_exact(tmp_path):
    """ADP1 directories (adapter_io.py): every bundle of a LoRA and a ReFT
    ModelAdapter survives save/load bit for bit (adapters.py:391-436)."""
    import gpu_util as U
    from paper_2605_14217_b200 import AdapterKind
    from paper_2605_14217_b200.adapter_io import load_catalogue, load_model_adapter, save_model_adapter

    rng = np.random.default_rng(9)
    lora = U.random_lora_adapter(rng, 3, 2, {"Wq": (16, 8), "Wdown": (8, 24)}, 4)
    reft = U.random_reft_adapter(rng, 5, 3, 8, 2, AdapterKind.LOREFT)
    for a in (lora, reft):
        save_model_adapter(a, tmp_path / f"a{a.adapter_id}")
        b = load_model_adapter(tmp_path / f"a{a.adapter_id}")
        assert (b.adapter_id, b.kind, b.rank, b.schedule) == (a.adapter_id, a.kind, a.rank, a.schedule)
        pa = sorted(a.lora_sites.items()) if a.kind is AdapterKind.LORA else list(enumerate(a.reft_sites))
        pb = sorted(b.lora_sites.items()) if b.kind is AdapterKind.LORA else list(enumerate(b.reft_sites))
        assert [k for k, _ in pa] == [k for k, _ in pb]
        for (_, x), (_, y) in zip(pa, pb):
            assert x.dims == y.dims and x.scaling == y.scaling
            for tx, ty in zip(x.tensors, y.tensors):
                assert tx.tobytes() == ty.tobytes()
    assert sorted(load_catalogue(tmp_path)) == [3, 5]


def test_adapter_directory_rejects_corruption(tmp_path):
    import gpu_util as U
    from paper_2605_14217_b200.adapter_io import load_model_adapter, save_model_adapter
    from paper_2605_14217_b200.errors import ShapeError

    rng = np.random.default_rng(1)
    d = save_model_adapter(U.random_lora_adapter(rng, 1, 1, {"Wq": (8, 8)}, 2), tmp_path / "a")
    f = d / "L0_Wq.adp1"
    f.write_bytes(f.read_bytes()[:-3])
    with pytest.raises(ShapeError):
        load_model_adapter(d)
    with pytest.raises(ShapeError):
        load_model_adapter(tmp_path / "missing")


def test_lora_site_chunks_respect_kernel_limit():
    """nsites * r_max <= 64 and <= 3 sites per launch (include/preft.h)."""
    from paper_2605_14217_b200.ops import lora_site_chunks

    sites = ("Wq", "Wk", "Wv")
    assert lora_site_chunks(sites, 1) == [(0, 3)]
    assert lora_site_chunks(sites, 16) == [(0, 3)]
    assert lora_site_chunks(sites, 32) == [(0, 2), (2, 3)]
    assert lora_site_chunks(sites, 64) == [(0, 1), (1, 2), (2, 3)]
    assert lora_site_chunks(("Wgate", "Wup"), 64) == [(0, 1), (1, 2)]


def test_validate_arrays_matches_make_batch_rules():
    from paper_2605_14217_b200.errors import BatchError
    from paper_2605_14217_b200.meta import validate_arrays

    ok = (np.array([0, 2, 5], np.int32), np.array([0, -1], np.int32), np.array([1, 2], np.int32))
    validate_arrays(*ok)
    for bad in ((np.array([0, 2, 2], np.int32), ok[1], ok[2]), (np.array([1, 2, 5], np.int32), ok[1], ok[2]),
                (ok[0], ok[1], np.array([0, 4], np.int32)), (ok[0], np.array([0, -3], np.int32), ok[2])):
        with pytest.raises(BatchError):
            validate_arrays(*bad)
