#!/usr/bin/env python
"""Phase breakdown of the tensor-core ReFT kernel (diagnostic, one GPU).

Runs one cfg3-shaped launch (8B d=4096, DiReFT r=16 or LoReFT r=32, long
prompts) with CTA 0's clock64() stamps enabled and prints the average cycles
per phase: load, shrink, partials+cluster sync, DSMEM reduce+sync, expand,
epilogue, store.  Also prints the launch's cluster count and the event time.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rank", type=int, default=16)
    p.add_argument("--kind", default="direft")
    p.add_argument("--tokens", type=int, default=65536)
    args = p.parse_args()
    import torch

    from paper_2605_14217_b200 import AdapterKind, _lib
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    dev = torch.device("cuda", 0)
    d = 4096
    pool = AdapterPool(1, d, reft_capacity=64, reft_rank=args.rank, dtype=torch.bfloat16, device=dev)
    ids = pool.fill_synthetic_(64, AdapterKind(args.kind), args.rank, seed=1)
    n_req = args.tokens // 2048
    lens = [2048] * n_req
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    rng = np.random.default_rng(0)
    eids = [int(ids[i]) for i in rng.integers(0, 64, size=n_req)]
    slots = pool.entry_arrays(qsl, eids, np.zeros(n_req, np.int32))
    meta = BatchMeta(n_req, int(qsl[-1]), device=dev)
    meta.set_slot_split(pool.slot_split)
    meta.build_arrays(qsl, slots, np.zeros(n_req, np.int32))
    h = torch.randn(int(qsl[-1]), d, device=dev).to(torch.bfloat16)
    lib = _lib.load()
    buf = torch.zeros(16 * 8, dtype=torch.int64, device=dev)
    for _ in range(3):
        apply_reft_(h, meta, pool, 0)
    torch.cuda.synchronize()
    lib.preft_diag_reft_tc(ctypes.c_void_p(buf.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    apply_reft_(h, meta, pool, 0)
    e1.record()
    torch.cuda.synchronize()
    clusters = lib.preft_diag_reft_tc(None)
    st = buf.view(16, 8).cpu().numpy()
    st = st[st[:, 7] > 0]
    names = ["load", "shrink", "partials+sync", "reduce+sync", "expand", "epilogue", "store"]
    phases = {n: float(np.mean(st[:, i + 1] - st[:, i])) for i, n in enumerate(names)}
    tile_cyc = float(np.mean(st[1:, 0] - st[:-1, 0])) if len(st) > 1 else None
    print(json.dumps({"rank": args.rank, "kind": args.kind, "tokens": int(qsl[-1]), "clusters": clusters,
                      "launch_us": round(e0.elapsed_time(e1) * 1e3, 1), "tiles_profiled": int(len(st)),
                      "cycles_per_phase": {k: round(v) for k, v in phases.items()},
                      "cycles_per_tile": round(tile_cyc) if tile_cyc else None}))


if __name__ == "__main__":
    main()
