"""Generate the golden vectors that pin the oracle (and the device kernels).

Run in the build container, where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every expected output below is produced by the REFERENCE implementation
(`prefillsim`, /root/reference/pkg/src) — compute_position_mask
(model.py:305-319), delta_for_rows (adapters.py:278-295), apply_masked
(adapters.py:298-333), _project (model.py:442-452), init_zero_delta /
build_adapter / perturb_adapter (adapters.py:212-262, model.py:346-413) and
save_adapter (adapters.py:391-401).  The vectors are small (< 2 MB total) and
committed; /root/reference is never read at test time on the GPU box.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import prefillsim  # noqa: E402
from prefillsim import adapters as RA  # noqa: E402
from prefillsim import model as RM  # noqa: E402
from prefillsim.linalg import rng_from_seed  # noqa: E402

OUT = Path(__file__).resolve().parent


def ref_digest() -> str:
    h = hashlib.sha256()
    for name in ("adapters.py", "model.py", "linalg.py"):
        h.update((REF / "prefillsim" / name).read_bytes())
    return h.hexdigest()


def entry_arrays(entries):
    adapter = np.array([-1 if e.adapter_id is None else e.adapter_id for e in entries], dtype=np.int64)
    is_dec = np.array([e.phase is RM.Phase.DECODE for e in entries], dtype=bool)
    allp = np.array([e.schedule is RA.PositionSchedule.ALL_POSITIONS for e in entries], dtype=bool)
    plen = np.array([e.prompt_len for e in entries], dtype=np.int64)
    return adapter, is_dec, allp, plen


def gen_masks():
    """Random mixed batches in the style of tests/test_model.py:160-193 and
    tests/test_acceptance.py:324-364, plus the hand cases of
    tests/test_model.py:113-140 and some long-span batches."""
    rng = rng_from_seed(2024, 7)
    batches = []
    for trial in range(400):
        entries, starts = [], []
        n = int(rng.integers(1, 12 if trial % 4 else 40))
        for seq in range(n):
            p = int(rng.integers(1, 9 if trial % 3 else 300))
            phase = RM.Phase.PREFILL if rng.random() < 0.5 else RM.Phase.DECODE
            if phase is RM.Phase.PREFILL:
                start = int(rng.integers(0, p))
                span = int(rng.integers(1, p - start + 1))
            else:
                start = p + int(rng.integers(0, 4))
                span = 1
            has = rng.random() < 0.8
            sched = RA.PositionSchedule.ALL_POSITIONS if rng.random() < 0.5 else RA.PositionSchedule.PREFILL_ONLY
            aid = int(rng.integers(0, 6)) if (has and trial % 2) else (seq if has else None)
            entries.append(
                RM.SeqEntry(seq, tuple(int(t) for t in rng.integers(0, 10, size=span)), p, phase,
                            adapter_id=aid, schedule=sched if has else None)
            )
            starts.append(start)
        batches.append((entries, starts))
    P = RA.PositionSchedule
    hand = [
        [RM.SeqEntry(i, (1,), 4, RM.Phase.DECODE, adapter_id=i, schedule=P.PREFILL_ONLY) for i in range(3)],
        [RM.SeqEntry(0, (5, 6), 2, RM.Phase.PREFILL, adapter_id=1, schedule=P.PREFILL_ONLY),
         RM.SeqEntry(1, (7,), 3, RM.Phase.DECODE, adapter_id=2, schedule=P.ALL_POSITIONS)],
        [RM.SeqEntry(0, (5, 6), 4, RM.Phase.PREFILL),
         RM.SeqEntry(1, (7,), 2, RM.Phase.DECODE, adapter_id=2, schedule=P.ALL_POSITIONS)],
    ]
    for h in hand:
        batches.append((h, [0 if e.phase is RM.Phase.PREFILL else e.prompt_len for e in h]))
    qsl, ad, dec, allp, plen, start, mask, uni = [], [], [], [], [], [], [], []
    e_off, t_off = [0], [0]
    for entries, starts in batches:
        b = RM.make_batch(entries)
        m = RM.compute_position_mask(b)
        a, d_, al, pl = entry_arrays(entries)
        qsl.append(np.asarray(b.query_start_loc, dtype=np.int64))
        ad.append(a)
        dec.append(d_)
        allp.append(al)
        plen.append(pl)
        start.append(np.asarray(starts, dtype=np.int64))
        mask.append(m.values.astype(bool))
        uni.append({True: 1, False: 0, None: -1}[m.uniform])
        e_off.append(e_off[-1] + len(entries))
        t_off.append(t_off[-1] + b.total_tokens)
    np.savez_compressed(
        OUT / "masks.npz",
        qsl=np.concatenate(qsl), adapter=np.concatenate(ad), is_decode=np.concatenate(dec),
        all_pos=np.concatenate(allp), prompt_len=np.concatenate(plen), cache_start=np.concatenate(start),
        mask=np.concatenate(mask), uniform=np.asarray(uni), e_off=np.asarray(e_off), t_off=np.asarray(t_off),
    )
    return len(batches)


def trained(kind, rank, dims, seed):
    p = RA.init_zero_delta(kind, rank, dims, seed)
    return RM._perturbed_params(p, seed + 1000, 0.3)


def gen_deltas():
    cases = {}
    K = RA.AdapterKind
    i = 0
    for kind in (K.LORA, K.DIREFT, K.LOREFT):
        for rank in (1, 2, 3, 4, 8, 16):
            for dims in (((48, 40), (16, 64), (7, 5)) if kind is K.LORA else ((64,), (40,), (17,))):
                if rank > min(dims):
                    continue
                p = trained(kind, rank, dims, seed=100 + i)
                width = dims[1] if kind is K.LORA else dims[0]
                rows = rng_from_seed(500 + i).normal(size=(37, width))
                delta = RA.delta_for_rows(p, rows)
                key = f"c{i:03d}"
                cases[key + "_kind"] = np.array(kind.value)
                cases[key + "_rank"] = np.array(rank)
                cases[key + "_dims"] = np.asarray(dims)
                cases[key + "_scaling"] = np.array([p.scaling.kind, repr(p.scaling.value)])
                cases[key + "_s"] = np.array(p.prefactor)
                for name in ("A", "B", "b", "R", "W"):
                    arr = getattr(p, name)
                    if arr is not None:
                        cases[key + "_" + name] = arr
                cases[key + "_rows"] = rows
                cases[key + "_delta"] = delta
                i += 1
    # known answers, tests/test_adapters.py:64-88
    lora = RA.AdapterParams(K.LORA, 1, (2, 2), RA.ScalingRule.constant(1.0), A=np.array([[0.0, 2.0]]),
                            B=np.array([[1.0], [0.0]]))
    cases["ka_lora_delta"] = RA.adapter_delta(lora, np.array([3.0, 4.0]))
    dire = RA.AdapterParams(K.DIREFT, 1, (2,), RA.ScalingRule.constant(1.0), A=np.array([[0.0, 1.0]]),
                            B=np.array([[1.0, 0.0]]), b=np.array([0.0]))
    cases["ka_direft_delta"] = RA.adapter_delta(dire, np.array([5.0, 7.0]))
    cases["n_cases"] = np.array(i)
    np.savez_compressed(OUT / "deltas.npz", **cases)
    return i


def gen_masked():
    K, P = RA.AdapterKind, RA.PositionSchedule
    cases = {}
    i = 0
    for kind in (K.LORA, K.DIREFT, K.LOREFT):
        dims = (10, 12) if kind is K.LORA else (12,)
        p = trained(kind, 3, dims, seed=77 + i)
        for sched in (P.PREFILL_ONLY, P.ALL_POSITIONS):
            for plen in (0, 1, 4, 12, 20):
                total = 12
                y = rng_from_seed(900 + i).normal(size=(total, dims[0]))
                x = rng_from_seed(950 + i).normal(size=(total, dims[1])) if kind is K.LORA else None
                out = RA.apply_masked(p, sched, y, x, plen)
                key = f"m{i:03d}"
                cases[key + "_kind"] = np.array(kind.value)
                cases[key + "_sched_all"] = np.array(sched is P.ALL_POSITIONS)
                cases[key + "_plen"] = np.array(plen)
                cases[key + "_s"] = np.array(p.prefactor)
                cases[key + "_rank"] = np.array(p.rank)
                cases[key + "_dims"] = np.asarray(dims)
                for name in ("A", "B", "b", "R", "W"):
                    arr = getattr(p, name)
                    if arr is not None:
                        cases[key + "_" + name] = arr
                cases[key + "_y"] = y
                if x is not None:
                    cases[key + "_x"] = x
                cases[key + "_out"] = out
                i += 1
    cases["n_cases"] = np.array(i)
    np.savez_compressed(OUT / "masked.npz", **cases)
    return i


def gen_hooks(shuffle: bool):
    """A reduced config-1 batch through the reference's own hook code.

    BASELINE config 1 at d = 128 instead of 4096 (same structure): 8 decode
    entries (PREFILL_ONLY, unselected) and 8 prefill entries of 16 tokens;
    prefill entry i uses LoRA^P r=1 (ids 0-3, site Wq) or DiReFT^P r=8
    (ids 4-7); plus one LoReFT^P r=4 entry (id 8) and one adapter-less
    prefill entry.  LoRA goes through `_project` (model.py:442-452) and ReFT
    through the residual hook (model.py:543-546), with rows taken from
    compute_position_mask exactly as forward_chunk does (model.py:509,538).
    """
    K, P = RA.AdapterKind, RA.PositionSchedule
    d = 128
    rng = rng_from_seed(31337, 1 if shuffle else 0)
    params, kinds = {}, {}
    for aid in range(9):
        if aid < 4:
            params[aid] = trained(K.LORA, 1, (d, d), seed=2000 + aid)
        elif aid < 8:
            params[aid] = trained(K.DIREFT, 8, (d,), seed=2000 + aid)
        else:
            params[aid] = trained(K.LOREFT, 4, (d,), seed=2000 + aid)
        kinds[aid] = params[aid].kind.value
    entries = []
    for i in range(8):
        entries.append(RM.SeqEntry(100 + i, (1,), 5, RM.Phase.DECODE, adapter_id=i % 9, schedule=P.PREFILL_ONLY))
    for i in range(9):
        entries.append(RM.SeqEntry(i, tuple(range(16)), 16, RM.Phase.PREFILL, adapter_id=i, schedule=P.PREFILL_ONLY))
    entries.append(RM.SeqEntry(50, tuple(range(7)), 9, RM.Phase.PREFILL))
    if shuffle:
        order = rng.permutation(len(entries))
        entries = [entries[j] for j in order]
    b = RM.make_batch(entries)
    T = b.total_tokens
    mask = RM.compute_position_mask(b).values
    x = rng.normal(size=(T, d))
    W = rng.normal(size=(d, d)) / np.sqrt(d)
    h = rng.normal(size=(T, d))
    y_base = x @ W.T
    y_ref = np.empty_like(y_base)
    h_ref = h.copy()
    for i, e in enumerate(entries):
        sp = b.span(i)
        rows = mask[sp]
        site = params[e.adapter_id] if (e.adapter_id is not None and params[e.adapter_id].kind is K.LORA) else None
        y_ref[sp] = RM._project(x[sp], W, site, rows)
        if e.adapter_id is not None and params[e.adapter_id].kind is not K.LORA and rows.any():
            blk = h_ref[sp]
            blk[rows] += RA.delta_for_rows(params[e.adapter_id], blk[rows])
            h_ref[sp] = blk
    a, dec, allp, plen = entry_arrays(entries)
    out = dict(qsl=np.asarray(b.query_start_loc), adapter=a, is_decode=dec, all_pos=allp, prompt_len=plen,
               mask=mask, x=x, W=W, y_base=y_base, y_ref=y_ref, h=h, h_ref=h_ref, d=np.array(d))
    for aid, p in params.items():
        out[f"a{aid}_kind"] = np.array(p.kind.value)
        out[f"a{aid}_rank"] = np.array(p.rank)
        out[f"a{aid}_s"] = np.array(p.prefactor)
        for name in ("A", "B", "b", "R", "W"):
            arr = getattr(p, name)
            if arr is not None:
                out[f"a{aid}_{name}"] = arr
    np.savez_compressed(OUT / f"hooks_config1_small{'_shuffled' if shuffle else ''}.npz", **out)


CFG1_D = 4096


def config1_entries(shuffle: bool):
    """BASELINE configs[0] exactly (SURVEY 8(d) cfg 1): 32 decode entries
    (PREFILL_ONLY adapters, unselected) then 32 prefill entries x 128 tokens;
    prefill entry i -> adapter i: ids 0-15 DiReFT^P r=8 (residual site),
    ids 16-31 LoRA^P r=1 (one 4096 -> 4096 site).  `shuffle` permutes the
    entries with rng_from_seed(0, 7)."""
    P = RA.PositionSchedule
    entries = [RM.SeqEntry(100 + i, (1,), 129, RM.Phase.DECODE, adapter_id=i, schedule=P.PREFILL_ONLY)
               for i in range(32)]
    entries += [RM.SeqEntry(i, tuple(range(128)), 128, RM.Phase.PREFILL, adapter_id=i, schedule=P.PREFILL_ONLY)
                for i in range(32)]
    if shuffle:
        order = rng_from_seed(0, 7).permutation(len(entries))
        entries = [entries[j] for j in order]
    return entries


def config1_params():
    """init_zero_delta(kind, r, dims, seed=a) then _perturbed_params(seed=a+1000, sigma=0.1) (model.py:383-397)."""
    K = RA.AdapterKind
    out = {}
    for a in range(32):
        kind, r, dims = (K.DIREFT, 8, (CFG1_D,)) if a < 16 else (K.LORA, 1, (CFG1_D, CFG1_D))
        out[a] = RM._perturbed_params(RA.init_zero_delta(kind, r, dims, a), a + 1000, 0.1)
    return out


def gen_config1_full(shuffle: bool):
    """BASELINE configs[0] at its stated size through the reference's own hook
    code: LoRA via _project (model.py:442-452, with W = 0 so its output is the
    delta alone), ReFT via the residual hook (model.py:543-546).  Inputs come
    from rng_from_seed(0, 1) in the order x, h; the full outputs are pinned by
    sha256 and a sample of rows is stored (the arrays are 135 MB each)."""
    K = RA.AdapterKind
    d = CFG1_D
    entries = config1_entries(shuffle)
    params = config1_params()
    b = RM.make_batch(entries)
    T = b.total_tokens
    mask = RM.compute_position_mask(b).values
    rng = rng_from_seed(0, 1)
    x = rng.normal(size=(T, d))
    h = rng.normal(size=(T, d))
    W0 = np.zeros((d, d))
    delta = np.zeros((T, d))
    h_ref = h.copy()
    for i, e in enumerate(entries):
        sp = b.span(i)
        rows = mask[sp]
        p = params[e.adapter_id]
        if p.kind is K.LORA:
            delta[sp] = RM._project(x[sp], W0, p, rows)
        elif rows.any():
            blk = h_ref[sp]
            blk[rows] += RA.delta_for_rows(p, blk[rows])
            h_ref[sp] = blk
    sel = np.flatnonzero(mask)
    pick = np.sort(np.concatenate([rng_from_seed(0, 9).choice(sel, size=24, replace=False),
                                   np.flatnonzero(~mask)[:4]]))
    a, dec, allp, plen = entry_arrays(entries)
    out = dict(qsl=np.asarray(b.query_start_loc), adapter=a, is_decode=dec, all_pos=allp, prompt_len=plen,
               mask=mask, rows=pick, delta_rows=delta[pick], h_rows=h_ref[pick],
               delta_sha256=np.array(hashlib.sha256(np.ascontiguousarray(delta).tobytes()).hexdigest()),
               h_sha256=np.array(hashlib.sha256(np.ascontiguousarray(h_ref).tobytes()).hexdigest()),
               d=np.array(d))
    np.savez_compressed(OUT / f"config1_full{'_shuffled' if shuffle else ''}.npz", **out)


def gen_init_and_io():
    K, P = RA.AdapterKind, RA.PositionSchedule
    out = {}
    for key, (kind, rank, dims, seed) in {
        "lora": (K.LORA, 4, (8, 6), 2),
        "direft": (K.DIREFT, 5, (32,), 3),
        "loreft": (K.LOREFT, 3, (16,), 4),
    }.items():
        p = RA.init_zero_delta(kind, rank, dims, seed)
        for name in ("A", "B", "b", "R", "W"):
            arr = getattr(p, name)
            if arr is not None:
                out[f"init_{key}_{name}"] = arr
        import tempfile

        with tempfile.TemporaryDirectory() as tmp:
            path = Path(tmp) / "a.bin"
            RA.save_adapter(trained(kind, rank, dims, seed), path)
            out[f"adp1_{key}"] = np.frombuffer(path.read_bytes(), dtype=np.uint8)
    cfg = RM.ModelConfig(d_model=16, n_layers=2, vocab=31, seed=5, max_seq=64)
    for key, (kind, rank) in {"lora": (K.LORA, 2), "direft": (K.DIREFT, 4), "loreft": (K.LOREFT, 3)}.items():
        ad = RM.perturb_adapter(RM.build_adapter(cfg, 7, kind, rank, P.PREFILL_ONLY, seed=11), seed=12, sigma=0.2)
        if kind is K.LORA:
            for (layer, name), p in sorted(ad.lora_sites.items()):
                out[f"build_{key}_{layer}_{name}_A"] = p.A
                out[f"build_{key}_{layer}_{name}_B"] = p.B
        else:
            for layer, p in enumerate(ad.reft_sites):
                for name in ("A", "B", "b", "R", "W"):
                    arr = getattr(p, name)
                    if arr is not None:
                        out[f"build_{key}_{layer}_{name}"] = arr
    np.savez_compressed(OUT / "init_io.npz", **out)


def gen_workload():
    """Punica request streams (workload.py:110-156) for every mix."""
    from prefillsim import workload as W

    out = {}
    for mix in W.AdapterMix:
        cfg = W.WorkloadConfig(1000, 512, mix, seed=3, l_max=2048)
        p = W.sample_prompt_lens(cfg)
        out[f"{mix.value}_prompt"] = p
        out[f"{mix.value}_total"] = W.sample_total_lens(cfg, p)
        out[f"{mix.value}_adapters"] = np.asarray(W.assign_adapters(cfg), dtype=np.int64)
    np.savez_compressed(OUT / "workload.npz", **out)


CHAIN_ADAPTERS = (  # id, kind, rank, schedule, build seed, perturb seed
    (1, "LORA", 4, "PREFILL_ONLY", 11, 111),
    (2, "DIREFT", 4, "PREFILL_ONLY", 12, 112),
    (3, "LOREFT", 4, "PREFILL_ONLY", 13, 113),
    (4, "LORA", 2, "ALL_POSITIONS", 14, 114),
    (5, "DIREFT", 2, "ALL_POSITIONS", 15, 115),
)
CHAIN_SIGMA = 0.3


def chain_adapters(cfg, zero: bool = False):
    K, P = RA.AdapterKind, RA.PositionSchedule
    out = {}
    for aid, kind, rank, sched, s0, s1 in CHAIN_ADAPTERS:
        a = RM.build_adapter(cfg, aid, K[kind], rank, P[sched], seed=s0)
        out[aid] = a if zero else RM.perturb_adapter(a, seed=s1, sigma=CHAIN_SIGMA)
    return out


def _chain_record(out, prefix, w, batch, adapters, cache):
    """Run the reference forward_chunk (model.py:455-552) and record its
    inputs (h0 = embed + pos, model.py:481-488) and outputs."""
    starts = {e.seq_id: cache.length(e.seq_id) for e in batch.entries}
    tokens = np.concatenate([np.asarray(e.tokens, dtype=np.intp) for e in batch.entries])
    positions = np.concatenate([np.arange(starts[e.seq_id], starts[e.seq_id] + len(e.tokens))
                                for e in batch.entries])
    a, dec, allp, plen = entry_arrays(batch.entries)
    out[prefix + "qsl"] = np.asarray(batch.query_start_loc)
    out[prefix + "tokens"] = tokens
    out[prefix + "seq"] = np.array([e.seq_id for e in batch.entries])
    out[prefix + "adapter"], out[prefix + "is_decode"], out[prefix + "all_pos"] = a, dec, allp
    out[prefix + "prompt_len"] = plen
    out[prefix + "h0"] = w.embed[tokens] + w.pos[positions]
    out[prefix + "mask"] = RM.compute_position_mask(batch).values
    logits, hidden = RM.forward_chunk(w, batch, adapters, cache, collect_hidden=True)
    out[prefix + "logits"] = logits
    out[prefix + "hidden"] = np.stack(hidden)


def gen_forward_chain():
    """End-to-end forward semantics through the hooks (VERDICT r01 missing #6):
    the reference's forward_chunk on a 2-layer toy model, where every layer's
    LoRA^P deltas feed attention / the MLP and the ReFT^P residual edit feeds
    the next layer's projections (model.py:504-546).

    case a: attention on, a fresh all-prefill batch (LoRA, DiReFT, LoReFT,
            adapter-less, and ALL_POSITIONS entries);
    case b: ablate_attention, a mixed step after a prefill: decode tokens of
            PREFILL_ONLY adapters (unselected) and ALL_POSITIONS adapters
            (selected) next to a partial prefill chunk and an adapter-less one,
            plus the same step with no adapters (the bitwise-decode property of
            tests/test_model.py:298-327)."""
    P = RA.PositionSchedule
    out = {}
    g = rng_from_seed(3, 4)
    cfg_a = RM.ModelConfig(d_model=64, n_layers=2, vocab=40, seed=5, max_seq=64)
    w = RM.build_model(cfg_a)
    adapters = chain_adapters(cfg_a)
    sched = {aid: P[s] for aid, _, _, s, _, _ in CHAIN_ADAPTERS}
    entries = []
    for sid, (aid, n) in enumerate(zip([1, 2, 3, None, 4, 5], [5, 7, 3, 4, 6, 8])):
        toks = tuple(int(t) for t in g.integers(0, cfg_a.vocab, size=n))
        entries.append(RM.SeqEntry(sid, toks, n, RM.Phase.PREFILL, aid, sched.get(aid)))
    _chain_record(out, "a_", w, RM.make_batch(entries), adapters, RM.KvCache(cfg_a.n_layers))
    out["a_cfg"] = np.array([cfg_a.d_model, cfg_a.n_layers, cfg_a.vocab, cfg_a.seed, cfg_a.max_seq, 0])
    for i, lw in enumerate(w.layers):
        for name in ("Wq", "Wk", "Wv", "Wo", "Wgate", "Wup", "Wdown"):
            out[f"a_L{i}_{name}"] = getattr(lw, name)
    out["a_unembed"] = w.unembed

    cfg_b = RM.ModelConfig(d_model=64, n_layers=2, vocab=40, seed=6, max_seq=64, ablate_attention=True)
    w = RM.build_model(cfg_b)
    adapters = chain_adapters(cfg_b)
    cache = RM.KvCache(cfg_b.n_layers)
    prompts = {sid: tuple(int(t) for t in g.integers(0, cfg_b.vocab, size=n)) for sid, n in enumerate([4, 6, 5, 3])}
    first = [RM.SeqEntry(sid, prompts[sid], len(prompts[sid]), RM.Phase.PREFILL, aid, sched[aid])
             for sid, aid in zip(range(4), [1, 2, 4, 5])]
    RM.prefill(w, RM.make_batch(first), adapters, cache)
    p6 = tuple(int(t) for t in g.integers(0, cfg_b.vocab, size=10))
    p7 = tuple(int(t) for t in g.integers(0, cfg_b.vocab, size=4))

    def step_entries(with_adapters):
        es = []
        for sid, aid in zip(range(4), [1, 2, 4, 5]):
            tok = (int(g2.integers(0, cfg_b.vocab)),)
            es.append(RM.SeqEntry(sid, tok, len(prompts[sid]), RM.Phase.DECODE,
                                  aid if with_adapters else None, sched[aid] if with_adapters else None))
        es.insert(2, RM.SeqEntry(6, p6[:6], 10, RM.Phase.PREFILL, 3 if with_adapters else None,
                                 sched[3] if with_adapters else None))
        es.append(RM.SeqEntry(7, p7, 4, RM.Phase.PREFILL))
        return es

    import copy

    base_cache = copy.deepcopy(cache)
    g2 = rng_from_seed(3, 5)
    _chain_record(out, "b_", w, RM.make_batch(step_entries(True)), adapters, cache)
    g2 = rng_from_seed(3, 5)
    _chain_record(out, "bbase_", w, RM.make_batch(step_entries(False)), adapters, base_cache)
    out["b_cfg"] = np.array([cfg_b.d_model, cfg_b.n_layers, cfg_b.vocab, cfg_b.seed, cfg_b.max_seq, 1])
    for i, lw in enumerate(w.layers):
        for name in ("Wq", "Wk", "Wv", "Wo", "Wgate", "Wup", "Wdown"):
            out[f"b_L{i}_{name}"] = getattr(lw, name)
    out["b_unembed"] = w.unembed
    np.savez_compressed(OUT / "forward_chain.npz", **out)


def main():
    if len(sys.argv) > 1:  # regenerate selected fixtures only, e.g. `make_golden.py forward_chain`
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        return
    gen_forward_chain()
    gen_workload()
    nb = gen_masks()
    nd = gen_deltas()
    nm = gen_masked()
    gen_hooks(False)
    gen_hooks(True)
    gen_config1_full(False)
    gen_config1_full(True)
    gen_init_and_io()
    (OUT / "REFERENCE_DIGEST.txt").write_text(
        f"prefillsim {prefillsim.__version__}\nsha256(adapters.py+model.py+linalg.py) {ref_digest()}\n"
        f"numpy {np.__version__}\nmask batches {nb}, delta cases {nd}, apply_masked cases {nm}\n"
    )
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
