"""Multi-GPU layout logic on CPU: world_size-2 gloo processes.

The path shards by adapter: each rank owns a disjoint slice
of the pool and receives exactly the requests routed to its adapters; there
is no collective on the data path.  These checks run the host side of that
layout (bench.py's per-rank batches, workload routing) with the CPU oracle
standing in for the kernels, and use gloo only for the bookkeeping the
benchmark does (token sums, max-over-ranks timing, gathering results).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _params(aid: int, d: int):
    rng = np.random.default_rng(1000 + aid)
    return dict(kind="lora", s=32.0, A=rng.normal(size=(1, d)), B=rng.normal(size=(d, 1)))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from oracle import preft_oracle as O
        from paper_2605_14217_b200.workload import owner_of, route_requests

        # 1) bench's per-rank batches: adapters owned by this rank only
        qsl, ids, flags, lens, owned = bench.step_entries(rank, world, 64, 16)
        assert all(owner_of(a, world) == rank for a in ids)
        mine = torch.tensor([len(owned), int(lens.sum())], dtype=torch.float64)
        tot = mine.clone()
        dist.all_reduce(tot)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)

        # 2) sharded == unsharded: route a global request stream, apply the
        # hook per rank, gather, compare with the single-process result
        d = 32
        rng = np.random.default_rng(7)
        n_req = 40
        req_adapter = [int(a) for a in rng.integers(0, 16, size=n_req)]
        req_len = [int(v) for v in rng.integers(1, 9, size=n_req)]
        x_all = [rng.normal(size=(n, d)) for n in req_len]
        y_all = [rng.normal(size=(n, d)) for n in req_len]
        routed = route_requests(req_adapter, world, lens=req_len)[rank]
        out = {}
        if routed:
            q_ = np.concatenate([[0], np.cumsum([req_len[i] for i in routed])])
            slots = np.array([req_adapter[i] for i in routed])
            dec = np.zeros(len(routed), bool)
            mask = O.position_mask(q_, slots, dec, dec)
            prm = {a: _params(a, d) for a in set(slots.tolist())}
            y = O.lora_hook(np.concatenate([y_all[i] for i in routed]), np.concatenate([x_all[i] for i in routed]),
                            q_, mask, slots, prm)
            for j, i in enumerate(routed):
                out[i] = y[q_[j]:q_[j + 1]]
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            merged = {}
            for g in gathered:
                assert not (set(g) & set(merged)), "a request was processed on two ranks"
                merged.update(g)
            assert sorted(merged) == list(range(n_req))
            q_ = np.concatenate([[0], np.cumsum(req_len)])
            slots = np.array(req_adapter)
            dec = np.zeros(n_req, bool)
            mask = O.position_mask(q_, slots, dec, dec)
            full = O.lora_hook(np.concatenate(y_all), np.concatenate(x_all), q_, mask, slots,
                               {a: _params(a, d) for a in range(16)})
            for i in range(n_req):
                assert np.array_equal(merged[i], full[q_[i]:q_[i + 1]])
            q.put(("ok", tot.tolist(), float(t.item())))
    except Exception as exc:  # surface failures to the parent
        q.put(("error", repr(exc), rank))
        raise
    finally:
        dist.destroy_process_group()


def test_adapter_sharded_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    ok = [m for m in msgs if m[0] == "ok"]
    assert ok, msgs
    _, tot, tmax = ok[0]
    assert tot[0] == 512  # the two shards cover the 512-adapter catalogue
    assert tmax == 2.0  # max over ranks
