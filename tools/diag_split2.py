#!/usr/bin/env python
"""Diagnostic: compare the tcgen05 and SIMT halves of the LoRA split pair
separately on the cfg2 r=16 batch (shrink P, then expand from the same P)."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    from paper_2605_14217_b200 import _lib, shapes
    from paper_2605_14217_b200.ops import lora_site_array, row_stride

    dev = torch.device("cuda", 0)
    args = bench.parse([])
    n_req = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ctx = bench.build_step(args, 0, 1, dev, n_req, n_req, lora_rank=16)
    pool, meta = ctx["pool"], ctx["meta"]
    lib = _lib.load()
    T = ctx["T"]
    mask = torch.from_numpy(meta.mask_host()).to(dev)
    for group in shapes.SITE_GROUPS:
        x, ys = ctx["acts"][group]
        arr = lora_site_array(ys, pool, 3, group)
        ldp = len(group) * 16
        Ps = {}
        for v in (1, 0):
            lib.preft_set_split_variant(v)
            P = torch.zeros(T, ldp, device=dev)
            st = lib.preft_lora_shrink(ctypes.byref(meta.c), ctypes.c_void_p(x.data_ptr()), T, row_stride(x),
                                       x.shape[1], arr, len(group), 16, pool.dtype_code, ctypes.c_void_p(P.data_ptr()),
                                       ldp, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            Ps[v] = P
            print(group, "shrink variant", v, "status", st)
        d = (Ps[1] - Ps[0])[mask.bool()]
        print(group, "P tc vs simt: max abs diff", float(d.abs().max()), "max |P|", float(Ps[0].abs().max()))
        bad = (Ps[1] - Ps[0]).abs().max(dim=1).values > 1e-2 * float(Ps[0].abs().max())
        rows = torch.nonzero(bad & mask.bool()).flatten()
        print("  bad rows", len(rows), rows[:20].tolist())
        outs = {}
        for v in (1, 0):
            lib.preft_set_split_variant(v)
            y2 = [torch.zeros_like(y) for y in ys]
            arr2 = lora_site_array(y2, pool, 3, group)
            st = lib.preft_lora_expand(ctypes.byref(meta.c), ctypes.c_void_p(Ps[0].data_ptr()), ldp, T, arr2,
                                       len(group), 16, pool.dtype_code,
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            outs[v] = y2
        for s, a, b in zip(group, outs[1], outs[0]):
            dd = (a.float() - b.float()).abs().max(dim=1).values
            rows = torch.nonzero(dd > 0.02 * float(b.float().abs().max())).flatten()
            print("  expand", s, "max diff", float(dd.max()), "max", float(b.float().abs().max()), "bad rows", len(rows),
                  rows[:10].tolist())
            qsl = ctx["qsl"]
            chunks = meta.chunks_host()
            units = meta.units_host()
            for r in rows[:12].tolist():
                e = int(np.searchsorted(qsl, r, side="right") - 1)
                cols = torch.nonzero((a[r].float() - b[r].float()).abs() > 0.02 * float(b.float().abs().max())).flatten()
                ci = int(np.flatnonzero((chunks[:, 0] <= r) & (r < chunks[:, 0] + chunks[:, 1]))[0])
                ui = int(np.flatnonzero((units[:, 1] <= ci) & (ci < units[:, 1] + units[:, 2]))[0])
                print(f"    row {r} entry {e} [{qsl[e]},{qsl[e+1]}) chunk {ci} {chunks[ci].tolist()} unit {ui} "
                      f"{units[ui].tolist()} cols {cols.min().item()}..{cols.max().item()} n={len(cols)} "
                      f"dev {a[r, cols[0]].item():.4f} ref {b[r, cols[0]].item():.4f}")
    lib.preft_set_split_variant(-1)


if __name__ == "__main__":
    main()
