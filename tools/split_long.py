#!/usr/bin/env python
"""Throughput of the split shrink / expand kernels on long prompts (full
64-row units): one 4096 -> 4096 LoRA site, r=16, 32 x 2048-token prompts."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2605_14217_b200 import AdapterKind
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.tp import SplitWorkspace, lora_expand_tp_, lora_shrink_tp_

    dev = torch.device("cuda", 0)
    d, r = 4096, 16
    pool = AdapterPool(1, d, lora_sites={"Wq": (d, d)}, lora_capacity=64, lora_rank=r, dtype=torch.bfloat16, device=dev)
    pool.fill_synthetic_(64, AdapterKind.LORA, r, seed=1)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    lens = [2048] * n
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ids = [int(i) % 64 for i in range(n)]
    slots = pool.entry_arrays(qsl, ids, np.zeros(n, np.int32))
    T = int(qsl[-1])
    meta = BatchMeta(n, T, device=dev)
    meta.set_slot_split(pool.slot_split)
    meta.build_arrays(qsl, slots, np.zeros(n, np.int32))
    ws = SplitWorkspace(meta, pool)
    xs = [torch.randn(T, d, device=dev).to(torch.bfloat16) for _ in range(2)]
    ys = [torch.randn(T, d, device=dev).to(torch.bfloat16) for _ in range(2)]
    s = torch.cuda.current_stream(dev)
    for i in range(3):
        P = lora_shrink_tp_([ys[i % 2]], xs[i % 2], meta, pool, 0, ("Wq",), ws)
        lora_expand_tp_(P, [ys[i % 2]], xs[i % 2], meta, pool, 0, ("Wq",))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tot = {"shrink": 0.0, "expand": 0.0}
    reps = 10
    for i in range(reps):
        ev[0].record(s)
        P = lora_shrink_tp_([ys[i % 2]], xs[i % 2], meta, pool, 0, ("Wq",), ws)
        ev[1].record(s)
        lora_expand_tp_(P, [ys[i % 2]], xs[i % 2], meta, pool, 0, ("Wq",))
        ev[2].record(s)
        torch.cuda.synchronize()
        tot["shrink"] += ev[0].elapsed_time(ev[1])
        tot["expand"] += ev[1].elapsed_time(ev[2])
    peak = 6650.0
    sb = T * d * 2
    eb = 2 * T * d * 2
    out = {k: round(v / reps * 1e3, 1) for k, v in tot.items()}
    out["shrink_frac"] = round(sb / (out["shrink"] * 1e-6) / 1e9 / peak, 3)
    out["expand_frac"] = round(eb / (out["expand"] * 1e-6) / 1e9 / peak, 3)
    out["tokens"] = T
    print(json.dumps(out))


if __name__ == "__main__":
    main()
