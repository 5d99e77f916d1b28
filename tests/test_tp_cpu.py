"""Tensor-parallel LoRA^P decomposition on CPU (BASELINE config 4, tp.py).

world_size-2 gloo processes stand in for two GPUs of a TP group: each rank
holds its shard of every site (A sliced along the input dim, B along the
output dim, via tp.site_shard), computes its partial shrink with the numpy
oracle, all-reduces the rank-r partials (the collective the GPU path issues
through NCCL), expands into its slice, and the gathered result must equal the
unsharded reference hook (adapters.py:284-288) for column- and row-parallel
sites.  The device kernels are covered by tests/test_gpu_tp.py.
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


SITES = {"Wq": (64, 64), "Wk": (16, 64), "Wv": (16, 64), "Wo": (64, 64), "Wgate": (96, 64), "Wup": (96, 64),
         "Wdown": (64, 96)}
GROUPS = (("Wq", "Wk", "Wv"), ("Wo",), ("Wgate", "Wup"), ("Wdown",))


def _adapter(name, r=4, seed=0):
    n, m = SITES[name]
    rng = np.random.default_rng(seed + list(SITES).index(name))
    return rng.normal(size=(r, m)), rng.normal(size=(n, r)), 32.0 / r


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_14217_b200.tp import site_shard

        rng = np.random.default_rng(11)
        T = 23
        errs = {}
        for group in GROUPS:
            m = SITES[group[0]][1]
            x = rng.normal(size=(T, m))
            y0 = {s: rng.normal(size=(T, SITES[s][0])) for s in group}
            sh = {s: site_shard(s, *SITES[s], rank, world) for s in group}
            style = sh[group[0]].style
            # this rank's activations, laid out as the base TP model holds them
            x_loc = x if style == "column" else x[:, sh[group[0]].m0 : sh[group[0]].m0 + sh[group[0]].m_loc]
            P = []
            for s in group:
                A, B, sc = _adapter(s)
                a = sh[s]
                xs = x_loc[:, a.x_offset : a.x_offset + a.m_loc]
                P.append(xs @ A[:, a.m0 : a.m0 + a.m_loc].T)  # partial shrink
            Pt = torch.from_numpy(np.concatenate(P, axis=1))
            dist.all_reduce(Pt)  # the rank-r all-reduce
            Pf = Pt.numpy()
            r = P[0].shape[1]
            for i, s in enumerate(group):
                A, B, sc = _adapter(s)
                a = sh[s]
                delta = sc * (Pf[:, i * r : (i + 1) * r] @ B[a.n0 : a.n0 + a.n_loc].T)
                if style == "column":
                    y_loc = y0[s][:, a.n0 : a.n0 + a.n_loc] + delta
                    parts = [None] * world
                    dist.all_gather_object(parts, y_loc)
                    out = np.concatenate(parts, axis=1)
                else:
                    y_part = (y0[s] if rank == 0 else np.zeros_like(y0[s])).copy()
                    y_part[:, a.y_offset : a.y_offset + a.n_loc] += delta
                    t = torch.from_numpy(y_part)
                    dist.all_reduce(t)  # the base model's own row-parallel all-reduce
                    out = t.numpy()
                ref = y0[s] + sc * ((x @ A.T) @ B.T)
                errs[s] = float(np.max(np.abs(out - ref)) / np.max(np.abs(ref)))
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


def test_tp_decomposition_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errs in res:
        assert set(errs) == set(SITES)
        for s, e in errs.items():
            assert e < 1e-12, (rank, s, e)


def test_site_shard_arithmetic():
    from paper_2605_14217_b200.errors import ShapeError
    from paper_2605_14217_b200.tp import shard_range, site_shard

    assert shard_range(8192, 3, 8) == (3072, 1024)
    q = site_shard("Wq", 8192, 8192, 2, 8)
    assert (q.style, q.x_offset, q.x_width, q.y_offset, q.y_width) == ("column", 2048, 8192, 0, 1024)
    d = site_shard("Wdown", 8192, 28672, 5, 8)
    assert (d.style, d.x_offset, d.x_width, d.y_offset, d.y_width) == ("row", 0, 3584, 5 * 1024, 8192)
    k = site_shard("Wk", 1024, 8192, 7, 8)
    assert (k.n0, k.n_loc, k.m0, k.m_loc) == (896, 128, 7168, 1024)
    with pytest.raises(ShapeError):
        shard_range(100, 0, 8)
