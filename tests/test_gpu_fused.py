"""K2f, the fused shrink -> exchange -> expand kernel (csrc/lora_fused.cu),
vs the oracle (adapters.py:284-288, model.py:449-451).

* one rank (FusedExchange.local): every Llama site group, K-split pieces
  1/2/4, ranks 16/32, LoRA- and ReFT-class slots in one batch; repeated
  launches alternate the exchange parity; CUDA-graph replay is bit-identical;
* tp ranks EMULATED on one GPU (FusedExchange.emulated): each rank's launch
  runs concurrently on its own stream with a small grid and stores its
  partials into every rank's region — the real exchange protocol, with local
  HBM standing in for the peers' — and the assembled outputs equal the
  unsharded oracle; every rank's V is the same sum in the same order, so
  column slices agree bit for bit with a single-rank run on the same shards;
* a rank whose peer never arrives gives up after spin_ns and reports it.
"""

import numpy as np
import pytest
import torch

import gpu_util as U
import helpers
from paper_2605_14217_b200 import _lib

pytestmark = pytest.mark.gpu

GROUPS = (("Wq", "Wk", "Wv"), ("Wo",), ("Wgate", "Wup"), ("Wdown",))


def _sites(d, kv, f):
    return {"Wq": (d, d), "Wk": (kv, d), "Wv": (kv, d), "Wo": (d, d), "Wgate": (f, d), "Wup": (f, d), "Wdown": (d, f)}


def _batch(rng, lora_ids, n_entries=24, long=(300, 129, 64)):
    lens = list(rng.integers(1, 40, size=n_entries)) + list(long)
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids, flags = [], []
    for i in range(len(lens)):
        pick = int(rng.integers(0, 10))
        ids.append(None if pick == 9 else int(lora_ids[pick % len(lora_ids)]))
        dec = i < 6 and lens[i] == 1
        flags.append(_lib.ENTRY_DECODE if dec else (_lib.ENTRY_ALL_POSITIONS if pick == 8 else 0))
    return qsl, ids, np.asarray(flags, np.int32)


def _pool(dev, sites, rank, tp_rank=0, tp_size=1, reft=False):
    from paper_2605_14217_b200.pool import AdapterPool

    return AdapterPool(1, sites["Wq"][1], lora_sites=sites, lora_capacity=5, lora_rank=rank,
                       reft_capacity=2 if reft else 0, reft_rank=16, dtype=torch.bfloat16, device=dev,
                       tp_rank=tp_rank, tp_size=tp_size)


@pytest.mark.parametrize("planes", [1, 2, 4])
@pytest.mark.parametrize("rank", [16, 32])
def test_fused_single_rank_matches_oracle(cuda_device, planes, rank):
    from paper_2605_14217_b200 import AdapterKind
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.tp import FusedExchange, apply_lora_group_tp_

    rng = np.random.default_rng(rank + planes)
    sites = _sites(1024, 128, 2048)
    pool = _pool(cuda_device, sites, rank, reft=True)
    ids = [100 + a for a in range(5)]
    for a in ids:
        pool.register(U.random_lora_adapter(rng, a, 1, sites, rank if a % 2 else rank // 2))
    pool.register(U.random_reft_adapter(rng, 7, 1, 1024, 16, AdapterKind.DIREFT))
    qsl, eids, flags = _batch(rng, ids + [7])
    T = int(qsl[-1])
    meta = BatchMeta(64, T, device=cuda_device)
    slots = U.stage(meta, pool, qsl, eids, flags)
    ex = FusedExchange.local(meta, pool, planes=planes)
    mask = U.oracle_mask(qsl, slots, flags)
    for rep in range(2):  # the second pass runs on the other parity
        for group in GROUPS:
            m = sites[group[0]][1]
            x = U.rand_act(rng, T, m, torch.bfloat16, cuda_device)
            ys = [U.rand_act(rng, T, sites[s][0], torch.bfloat16, cuda_device) for s in group]
            y_in = [U.to_np(y) for y in ys]
            apply_lora_group_tp_(ys, x, meta, pool, 0, group, exchange=ex)
            torch.cuda.synchronize()
            for name, y, yi in zip(group, ys, y_in):
                out = U.to_np(y)
                assert np.array_equal(out[~mask], yi[~mask]), f"{name}: unselected rows touched"
                ref = U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, pool, 0, name)
                helpers.check_close(out, yi, ref, "bf16", f"fused {name} r={rank} planes={planes} pass {rep}")
    assert ex.errors() == 0


def test_fused_graph_replay_bitwise(cuda_device):
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.tp import FusedExchange, apply_lora_group_tp_

    rng = np.random.default_rng(11)
    sites = _sites(1024, 128, 2048)
    pool = _pool(cuda_device, sites, 16)
    ids = [100 + a for a in range(5)]
    for a in ids:
        pool.register(U.random_lora_adapter(rng, a, 1, sites, 16))
    qsl, eids, flags = _batch(rng, ids)
    T = int(qsl[-1])
    meta = BatchMeta(64, T, device=cuda_device)
    U.stage(meta, pool, qsl, eids, flags)
    ex = FusedExchange.local(meta, pool, planes=4)
    acts = {g: (U.rand_act(rng, T, sites[g[0]][1], torch.bfloat16, cuda_device),
                [U.rand_act(rng, T, sites[s][0], torch.bfloat16, cuda_device) for s in g]) for g in GROUPS}
    base = {g: [y.clone() for y in ys] for g, (x, ys) in acts.items()}

    def step(s):
        for g, (x, ys) in acts.items():
            apply_lora_group_tp_(ys, x, meta, pool, 0, g, exchange=ex, stream=s)

    s = torch.cuda.current_stream()
    step(s)
    torch.cuda.synchronize()
    eager = {g: [y.clone() for y in ys] for g, (x, ys) in acts.items()}
    graph = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(s)
    with torch.cuda.stream(cs), torch.cuda.graph(graph, stream=cs):
        step(cs)
    s.wait_stream(cs)
    for rep in range(3):  # 4 launches per replay: the parities keep alternating
        for g, (x, ys) in acts.items():
            for y, b in zip(ys, base[g]):
                y.copy_(b)
        graph.replay()
        torch.cuda.synchronize()
        for g, (x, ys) in acts.items():
            for y, e in zip(ys, eager[g]):
                assert torch.equal(y, e), f"graph replay {rep} differs for {g}"
    assert ex.errors() == 0


def _tp_setup(cuda_device, tp, widths, seed, batch=None):
    from paper_2605_14217_b200.meta import BatchMeta

    rng = np.random.default_rng(seed)
    sites = _sites(*widths)
    full = _pool(cuda_device, sites, 16)
    shards = [_pool(cuda_device, sites, 16, tp_rank=r, tp_size=tp) for r in range(tp)]
    ids = [100 + a for a in range(5)]
    for a in ids:
        ad = U.random_lora_adapter(rng, a, 1, sites, 16)
        full.register(ad)
        for p in shards:
            p.register(ad)
    qsl, eids, flags = _batch(rng, ids) if batch is None else batch(ids)
    T = int(qsl[-1])
    metas = [BatchMeta(64, T, device=cuda_device) for _ in range(tp)]
    slots = None
    for p, m in zip(shards, metas):
        slots = U.stage(m, p, qsl, eids, flags)
    return rng, sites, full, shards, metas, qsl, slots, flags, T


def _rank_acts(shards, group, x_full, y_base):
    xs, yss = [], []
    for r, p in enumerate(shards):
        s0 = p.lora_shard[group[0]]
        xs.append(x_full if s0.style == "column" else x_full[:, s0.m0: s0.m0 + s0.m_loc].contiguous())
        ys = []
        for name, yb in zip(group, y_base):
            sr = p.lora_shard[name]
            if sr.style == "column":
                ys.append(yb[:, sr.n0: sr.n0 + sr.n_loc].contiguous())
            else:
                ys.append(yb.clone() if r == 0 else torch.zeros_like(yb))
        yss.append(ys)
    return xs, yss


@pytest.mark.parametrize("tp,widths,planes", [(2, (1024, 256, 2048), 1), (2, (1024, 256, 2048), 2),
                                              (4, (1024, 512, 2048), 1), (8, (8192, 1024, 28672), 1)])
def test_fused_tensor_parallel_emulated(cuda_device, tp, widths, planes):
    """tp concurrent rank launches exchange their partials through each
    other's regions; tp = 8 at Llama-3.1-70B widths is config 4's own shape."""
    from paper_2605_14217_b200.tp import FusedExchange, apply_lora_group_tp_

    rng, sites, full, shards, metas, qsl, slots, flags, T = _tp_setup(cuda_device, tp, widths, 40 + tp)
    mask = U.oracle_mask(qsl, slots, flags)
    grid = 12  # tp x 12 CTAs co-resident on one B200
    exs = FusedExchange.emulated(metas[0], shards[0], tp, planes=planes, grid=grid)
    streams = [torch.cuda.Stream() for _ in range(tp)]
    for group in GROUPS:
        n_full = [sites[s][0] for s in group]
        x_full = U.rand_act(rng, T, sites[group[0]][1], torch.bfloat16, cuda_device)
        y_base = [U.rand_act(rng, T, n, torch.bfloat16, cuda_device) for n in n_full]
        xs, yss = _rank_acts(shards, group, x_full, y_base)
        torch.cuda.synchronize()
        for r in range(tp):
            apply_lora_group_tp_(yss[r], xs[r], metas[r], shards[r], 0, group, exchange=exs[r], stream=streams[r])
        torch.cuda.synchronize()
        sh = shards[0].lora_shard[group[0]]
        for i, name in enumerate(group):
            if sh.style == "column":
                out = np.concatenate([U.to_np(yss[r][i]) for r in range(tp)], axis=1)
            else:
                out = sum(U.to_np(yss[r][i]) for r in range(tp))
            yi = U.to_np(y_base[i])
            ref = U.lora_oracle(yi, U.to_np(x_full), qsl, slots, flags, full, 0, name)
            assert np.array_equal(out[~mask], yi[~mask]), f"{name}: unselected rows touched"
            helpers.check_close(out, yi, ref, "bf16", f"fused tp={tp} planes={planes} {name}")
    for r in range(tp):
        assert exs[r].errors() == 0, f"rank {r} timed out waiting for a peer"


def test_fused_missing_peer_times_out(cuda_device):
    """Only rank 0 of a 2-rank exchange launches: its waits give up after
    spin_ns (error bit set) instead of hanging the device."""
    from paper_2605_14217_b200.tp import FusedExchange, apply_lora_group_tp_

    rng, sites, full, shards, metas, qsl, slots, flags, T = _tp_setup(cuda_device, 2, (1024, 256, 2048), 3)
    exs = FusedExchange.emulated(metas[0], shards[0], 2, planes=1, grid=8)
    exs[0].c.spin_ns = 5_000_000  # 5 ms
    x = U.rand_act(rng, T, 1024, torch.bfloat16, cuda_device)
    y = U.rand_act(rng, T, 512, torch.bfloat16, cuda_device)
    apply_lora_group_tp_([y], x, metas[0], shards[0], 0, ("Wq",), exchange=exs[0])
    torch.cuda.synchronize()
    assert exs[0].errors() & 1


def test_fused_group_exchange_world_size_one(cuda_device, tmp_path):
    """FusedExchange.group over a real process group (one rank): the region is
    a cudaMalloc allocation whose IPC handle goes through all_gather_object."""
    import torch.distributed as dist

    from paper_2605_14217_b200.tp import FusedExchange, apply_lora_group_tp_

    if dist.is_initialized():
        pytest.skip("a process group already exists")
    dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    try:
        rng, sites, full, shards, metas, qsl, slots, flags, T = _tp_setup(cuda_device, 1, (1024, 256, 2048), 9)
        ex = FusedExchange.group(metas[0], shards[0])
        mask = U.oracle_mask(qsl, slots, flags)
        x = U.rand_act(rng, T, 1024, torch.bfloat16, cuda_device)
        ys = [U.rand_act(rng, T, n, torch.bfloat16, cuda_device) for n in (1024, 256, 256)]
        y_in = [U.to_np(y) for y in ys]
        apply_lora_group_tp_(ys, x, metas[0], shards[0], 0, ("Wq", "Wk", "Wv"), exchange=ex)
        torch.cuda.synchronize()
        for name, y, yi in zip(("Wq", "Wk", "Wv"), ys, y_in):
            ref = U.lora_oracle(yi, U.to_np(x), qsl, slots, flags, full, 0, name)
            helpers.check_close(U.to_np(y), yi, ref, "bf16", f"group exchange {name}")
        assert ex.errors() == 0
        ex.close()
    finally:
        dist.destroy_process_group()


_IPC_WORKER = r"""
import sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[3]); sys.path.insert(0, sys.argv[3] + "/tests")
rank, path = int(sys.argv[1]), sys.argv[2]
dist.init_process_group("gloo", init_method=f"file://{path}/pg", rank=rank, world_size=2)
import gpu_util as U
from paper_2605_14217_b200.meta import BatchMeta
from paper_2605_14217_b200.pool import AdapterPool
from paper_2605_14217_b200.tp import FusedExchange, apply_lora_group_tp_
dev = torch.device("cuda", 0)
rng = np.random.default_rng(5)
sites = {"Wq": (1024, 1024), "Wk": (256, 1024), "Wv": (256, 1024)}
pool = AdapterPool(1, 1024, lora_sites=sites, lora_capacity=5, lora_rank=16, dtype=torch.bfloat16, device=dev,
                   tp_rank=rank, tp_size=2)
for a in range(5):
    pool.register(U.random_lora_adapter(rng, 100 + a, 1, sites, 16))
lens = [37, 5, 64, 90, 1, 200]
qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
ids = [100, 101, 102, 103, None, 104]
flags = np.zeros(len(lens), np.int32)
meta = BatchMeta(16, int(qsl[-1]), device=dev)
U.stage(meta, pool, qsl, ids, flags)
ex = FusedExchange.group(meta, pool, planes=1, grid=8)
ex.c.spin_ns = 20_000_000_000  # the two processes' kernels time-slice on one GPU
T = int(qsl[-1])
g = torch.Generator().manual_seed(7)
x = torch.randn(T, 1024, generator=g).to(torch.bfloat16).to(dev)
ys = [torch.randn(T, n // 2, generator=g).to(torch.bfloat16).to(dev) for n in (1024, 256, 256)]
apply_lora_group_tp_(ys, x, meta, pool, 0, ("Wq", "Wk", "Wv"), exchange=ex)
torch.cuda.synchronize()
err = ex.errors()
out = [y.float().cpu().numpy() for y in ys]
np.savez(f"{path}/out{rank}.npz", *out, err=np.array(err))
dist.barrier()
ex.close()
dist.destroy_process_group()
"""


def test_fused_ipc_exchange_two_processes(cuda_device, tmp_path):
    """The real multi-process exchange: two processes (tp = 2) map each
    other's regions through cudaIpc and store partials into them.  Both run
    on the one GPU here (their kernels time-slice; a generous spin bound).
    Rank r's column slices must equal the unsharded oracle's."""
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    script = tmp_path / "worker.py"
    script.write_text(_IPC_WORKER)
    procs = [subprocess.Popen([sys.executable, str(script), str(r), str(tmp_path), root]) for r in range(2)]
    try:
        rcs = [p.wait(timeout=240) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert rcs == [0, 0]
    outs = [np.load(tmp_path / f"out{r}.npz") for r in range(2)]
    assert all(int(o["err"]) == 0 for o in outs)
    # the reference: one unsharded rank on the same inputs
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.pool import AdapterPool

    rng = np.random.default_rng(5)
    sites = {"Wq": (1024, 1024), "Wk": (256, 1024), "Wv": (256, 1024)}
    full = AdapterPool(1, 1024, lora_sites=sites, lora_capacity=5, lora_rank=16, dtype=torch.bfloat16,
                       device=cuda_device)
    for a in range(5):
        full.register(U.random_lora_adapter(rng, 100 + a, 1, sites, 16))
    lens = [37, 5, 64, 90, 1, 200]
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = [100, 101, 102, 103, None, 104]
    flags = np.zeros(len(lens), np.int32)
    meta = BatchMeta(16, int(qsl[-1]), device=cuda_device)
    slots = U.stage(meta, full, qsl, ids, flags)
    T = int(qsl[-1])
    g = torch.Generator().manual_seed(7)
    x = torch.randn(T, 1024, generator=g).to(torch.bfloat16)
    y0 = [torch.randn(T, n // 2, generator=g).to(torch.bfloat16) for n in (1024, 256, 256)]
    # both ranks drew the same x and the same (half-width) y slices: rank r's
    # slice r of the full output starts from that slice
    for i, (name, n) in enumerate(zip(("Wq", "Wk", "Wv"), (1024, 256, 256))):
        yi = np.concatenate([y0[i].double().numpy()] * 2, axis=1)
        ref = U.lora_oracle(yi, x.double().numpy(), qsl, slots, flags, full, 0, name)
        out = np.concatenate([outs[r][f"arr_{i}"] for r in range(2)], axis=1)
        helpers.check_close(out, yi, ref, "bf16", f"ipc tp=2 {name}")


def _edge(kind):
    def make(ids):
        D = _lib.ENTRY_DECODE
        if kind == "all_decode":
            lens, e, fl = [1] * 24, [ids[i % len(ids)] for i in range(24)], [D] * 24
        elif kind == "no_adapter":
            lens, e, fl = [7, 64, 1, 130], [None] * 4, [0, 0, D, 0]
        elif kind == "one_long":
            lens, e, fl = [1, 1, 1000, 1], [ids[3], ids[4], ids[3], ids[3]], [D, D, 0, D]
        else:
            lens = [1, 15, 16, 17, 63, 64, 65, 128, 129, 1, 1]
            e = [ids[i] for i in (0, 0, 1, 1, 2, 2, 3, 4, 4, 0)] + [None]
            fl = [0] * 9 + [D, 0]
        return np.concatenate([[0], np.cumsum(lens)]).astype(np.int32), e, np.asarray(fl, np.int32)
    return make


@pytest.mark.parametrize("planes", [1, 2])
@pytest.mark.parametrize("kind", ["all_decode", "no_adapter", "one_long", "unit_edges"])
def test_fused_tensor_parallel_edge_batches(cuda_device, kind, planes):
    """Two emulated ranks through the fused kernel on edge batches: nothing
    selected (every rank still publishes its flags and the launch tags stay in
    step), no adapter at all, one long prompt of one adapter, and prompt
    lengths around the chunk / unit boundaries."""
    from paper_2605_14217_b200.tp import FusedExchange, apply_lora_group_tp_

    tp = 2
    rng, sites, full, shards, metas, qsl, slots, flags, T = _tp_setup(cuda_device, tp, (1024, 256, 2048), 77,
                                                                     batch=_edge(kind))
    mask = U.oracle_mask(qsl, slots, flags)
    exs = FusedExchange.emulated(metas[0], shards[0], tp, planes=planes, grid=12)
    streams = [torch.cuda.Stream() for _ in range(tp)]
    for rep in range(2):  # both exchange parities
        for group in GROUPS:
            x_full = U.rand_act(rng, T, sites[group[0]][1], torch.bfloat16, cuda_device)
            y_base = [U.rand_act(rng, T, sites[s][0], torch.bfloat16, cuda_device) for s in group]
            xs, yss = _rank_acts(shards, group, x_full, y_base)
            torch.cuda.synchronize()
            for r in range(tp):
                apply_lora_group_tp_(yss[r], xs[r], metas[r], shards[r], 0, group, exchange=exs[r],
                                     stream=streams[r])
            torch.cuda.synchronize()
            sh = shards[0].lora_shard[group[0]]
            for i, name in enumerate(group):
                if sh.style == "column":
                    out = np.concatenate([U.to_np(yss[r][i]) for r in range(tp)], axis=1)
                else:
                    out = sum(U.to_np(yss[r][i]) for r in range(tp))
                yi = U.to_np(y_base[i])
                assert np.array_equal(out[~mask], yi[~mask]), f"{kind} {name}: unselected rows touched"
                if mask.any():
                    ref = U.lora_oracle(yi, U.to_np(x_full), qsl, slots, flags, full, 0, name)
                    helpers.check_close(out, yi, ref, "bf16", f"fused edge {kind} planes={planes} {name}")
    for r in range(tp):
        assert exs[r].errors() == 0, f"rank {r} timed out waiting for a peer"
