#!/usr/bin/env python
"""Per-CTA timeline (globaltimer, CTAs 0-127) of one fused shrink -> exchange
-> expand launch (csrc/lora_fused.cu) at config-4 shapes (rank 0's shard,
one rank): start after the PDL wait, end of the shrink phase, first unit's
partials ready for the expand, end.  GROUP=qkv|o|gu|down, PLANES=1|2|4."""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_2605_14217_b200 import AdapterKind, _lib, shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.tp import FusedExchange, lora_fused_tp_

    dev = torch.device("cuda", 0)
    shape = shapes.LLAMA_70B if os.environ.get("SHAPE", "70b") == "70b" else shapes.LLAMA_8B
    tp = 8 if shape is shapes.LLAMA_70B else 1
    pool = AdapterPool(1, shape.d_model, lora_sites=shape.site_dims(), lora_capacity=512, lora_rank=16,
                       dtype=torch.bfloat16, device=dev, tp_rank=0, tp_size=tp)
    pool.fill_synthetic_(512, AdapterKind.LORA, 16, seed=1)
    qsl, ids, flags, lens, _ = bench.step_entries(0, 1, 256, 256, seed=3)
    slots = pool.entry_arrays(qsl, ids, flags)
    T = int(qsl[-1])
    meta = BatchMeta(len(ids), T, device=dev)
    meta.build_arrays(qsl, slots, flags, slot_split=pool.slot_split)
    meta.ensure_lora_part()
    ex = FusedExchange.local(meta, pool, planes=int(os.environ.get("PLANES", "1")))
    groups = {"qkv": ("Wq", "Wk", "Wv"), "o": ("Wo",), "gu": ("Wgate", "Wup"), "down": ("Wdown",)}
    group = groups[os.environ.get("GROUP", "qkv")]
    x = torch.randn(T, pool.lora_shard[group[0]].x_width, device=dev).to(torch.bfloat16)
    ys = [torch.randn(T, pool.lora_shard[s].y_width, device=dev).to(torch.bfloat16) for s in group]
    lib = _lib.load()
    for _ in range(3):
        lora_fused_tp_(ys, x, meta, pool, 0, group, ex)
    buf = torch.zeros(2048, dtype=torch.int64, device=dev)
    lib.preft_diag_split(ctypes.c_void_p(buf.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lora_fused_tp_(ys, x, meta, pool, 0, group, ex)
    e1.record()
    torch.cuda.synchronize()
    lib.preft_diag_split(None)
    b = buf.cpu().numpy()
    start, p1end = b[1536:1792:2], b[1537:1792:2]
    vready, end = b[1793:2048:2], b[1280:1408]
    t0 = start.min()
    print(f"group {group} units {meta.units_host().shape[0]} launch {e0.elapsed_time(e1) * 1e3:.1f} us")
    for name, t in (("phase-1 end", p1end), ("first V ready", vready), ("end", end)):
        v = np.where(t > 0, t - t0, 0)
        print(f"{name:14s} ns: min {v[v > 0].min() if (v > 0).any() else 0} mean {v[v > 0].mean() if (v > 0).any() else 0:.0f} max {v.max()}")
    print("phase-1 busy per CTA:", " ".join(str(int(a - s)) for a, s in zip(p1end, start)))
    print("wait for first V  :", " ".join(str(int(v - a)) if v else "-" for v, a in zip(vready, p1end)))
    print("phase-2 busy      :", " ".join(str(int(e - a)) for e, a in zip(end, p1end)))


if __name__ == "__main__":
    main()
