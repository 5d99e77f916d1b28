#!/usr/bin/env python
"""Timelines (clock64, CTA 0) of one tensor-core shrink and expand launch at
config-4 shapes; GROUP=qkv|o|gu|down picks the site group (default qkv)."""
import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import os

    import torch

    import bench
    from paper_2605_14217_b200 import AdapterKind, _lib, shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.tp import SplitWorkspace, apply_lora_group_tp_

    dev = torch.device("cuda", 0)
    shape = shapes.LLAMA_70B
    pool = AdapterPool(1, shape.d_model, lora_sites=shape.site_dims(), lora_capacity=512, lora_rank=16,
                       dtype=torch.bfloat16, device=dev, tp_rank=0, tp_size=8)
    pool.fill_synthetic_(512, AdapterKind.LORA, 16, seed=1)
    if os.environ.get("LONG"):
        lens = [2048] * 32
        qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        ids = [int(i) * 7 % 512 for i in range(32)]
        flags = np.zeros(32, np.int32)
    else:
        qsl, ids, flags, lens, _ = bench.step_entries(0, 1, 256, 256, seed=3)
    slots = pool.entry_arrays(qsl, ids, flags)
    T = int(qsl[-1])
    meta = BatchMeta(len(ids), T, device=dev)
    meta.set_slot_split(pool.slot_split)
    meta.build_arrays(qsl, slots, flags)
    print("units", meta.units_host().shape[0], "chunks", meta.chunks_host().shape[0], file=sys.stderr)
    ws = SplitWorkspace(meta, pool)
    groups = {"qkv": ("Wq", "Wk", "Wv"), "o": ("Wo",), "gu": ("Wgate", "Wup"), "down": ("Wdown",)}
    group = ("Wo",) if os.environ.get("LONG") else groups[os.environ.get("GROUP", "qkv")]
    x = torch.randn(T, pool.lora_shard[group[0]].x_width, device=dev).to(torch.bfloat16)
    ys = [torch.randn(T, pool.lora_shard[s].y_width, device=dev).to(torch.bfloat16) for s in group]
    lib = _lib.load()
    for _ in range(3):
        apply_lora_group_tp_(ys, x, meta, pool, 0, group, workspace=ws, collective=False)
    buf = torch.zeros(2048, dtype=torch.int64, device=dev)
    lib.preft_diag_split(ctypes.c_void_p(buf.data_ptr()))
    apply_lora_group_tp_(ys, x, meta, pool, 0, group, workspace=ws, collective=False)
    torch.cuda.synchronize()
    lib.preft_diag_split(None)
    st = buf.view(512, 4).cpu().numpy()
    ctas = buf.cpu().numpy()[1536:].reshape(2, 128, 2)
    t0 = st[0, 0]
    print("shrink stage: producer_issue mma_consume | unit: s_full")
    for i in range(128):
        if st[i, 0] or st[i, 1] or st[i, 2]:
            print(i, *(int(v - t0) if v else 0 for v in st[i, :3]))
    e = st[128:256]
    x = st[256:384]
    e0 = e[0, 0]
    print("expand item: producer_issue mma_issue epi_start epi_end | first_ld_done rmw_done stores_issued (cycles from the first issue)")
    for i in range(128):
        if e[i].any():
            print(i, *(int(v - e0) if v else 0 for v in e[i]), "|", *(int(v - e0) if v else 0 for v in x[i, [2, 0, 1]]))
    for name, t in zip(("shrink", "expand"), ctas):
        t0 = t[:, 0].min()
        print(f"{name} CTA work windows (ns from the first start; CTAs 0-127):")
        print("  start", " ".join(str(int(v - t0)) for v in t[:, 0]))
        print("  end  ", " ".join(str(int(v - t0)) for v in t[:, 1]))
        d = t[:, 1] - t[:, 0]
        print(f"  busy ns: min {d.min()} mean {d.mean():.0f} max {d.max()} (argmax CTA {d.argmax()}), last end {t[:, 1].max() - t0}")


if __name__ == "__main__":
    main()
