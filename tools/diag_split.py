#!/usr/bin/env python
"""Diagnostic: the tcgen05 LoRA split pair on a full cfg2-sized batch (many
K1 units per CTA), one launch per group, vs the oracle on sampled rows —
and the same batch on the SIMT kernels.  Prints per-group errors."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    from paper_2605_14217_b200 import _lib, shapes
    from paper_2605_14217_b200.ops import apply_lora_group_

    dev = torch.device("cuda", 0)
    args = bench.parse([])
    n_req = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ctx = bench.build_step(args, 0, 1, dev, n_req, n_req, lora_rank=16)
    pool, meta, qsl, slots = ctx["pool"], ctx["meta"], ctx["qsl"], ctx["slots"]
    print("units", int(meta.counters_host()[_lib.CTR_UNITS]), "tokens", ctx["sel"])
    lib = _lib.load()
    for variant in (-1, 0):
        lib.preft_set_lora_variant(variant)
        for layer in (0, 5):
            for group in shapes.SITE_GROUPS:
                x, ys = ctx["acts"][group]
                for y in ys:
                    y.copy_(torch.randn(y.shape, device=dev))
                snap = {group: [y.clone() for y in ys]}
                apply_lora_group_(ys, x, meta, pool, layer, group)
                torch.cuda.synchronize()
                r = bench.check_lora_accumulated(pool, meta, qsl, slots, {group: (x, ys)}, snap, [layer], k=64)
                print("variant", variant, "layer", layer, group, r["status"], r["max_rel_err"], r["output_rel_err"])
    lib.preft_set_lora_variant(-1)


if __name__ == "__main__":
    main()
