#!/usr/bin/env python
"""Per-launch sweep of the K2 variants on the bench workload (one GPU).

For each site group of a Llama-3.1-8B layer and each kernel variant (warp
kernel, team kernel with 1/2/4/8 warps per row, automatic), time `--reps`
launches with CUDA events on the launching stream (layers rotate so adapter
weights and activations are not L2-resident from the previous launch) and
report average us, achieved GB/s of algorithmic bytes and the fraction of
the measured HBM peak.  Prints one JSON object.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--requests", type=int, default=256)
    p.add_argument("--decodes", type=int, default=256)
    p.add_argument("--reps", type=int, default=32)
    p.add_argument("--variants", default="0,1,2,4,8,-1")
    p.add_argument("--t1cfgs", default="0", help="PREFT_LORA_T1CFG values to sweep for variant 1")
    args = p.parse_args()
    import os

    import torch

    from paper_2605_14217_b200 import _lib, shapes
    from paper_2605_14217_b200.ops import apply_lora_group_

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    ctx = bench.build_step(args, 0, 1, dev, args.requests, args.decodes)
    peak, _ = bench.measured_peak_gbs()
    lib = _lib.load()
    out = {"tokens": ctx["sel"], "distinct": ctx["distinct"], "peak_gbs": peak, "groups": {}}
    s = torch.cuda.current_stream(dev)
    flush = torch.empty(512 * 2**20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    configs = []
    for v in [int(t) for t in args.variants.split(",")]:
        if v == 1:
            configs += [(1, c) for c in args.t1cfgs.split(",")]
        else:
            configs.append((v, "0"))
    for group in shapes.SITE_GROUPS:
        x, ys = ctx["acts"][group]
        nbytes = bench.group_bytes(ctx["shape"], group, ctx["sel"], ctx["distinct"])
        res = {}
        for v, cfg in configs:
            os.environ["PREFT_LORA_T1CFG"] = cfg
            assert lib.preft_set_lora_variant(v) == 0
            for layer in range(4):  # warm-up
                apply_lora_group_(ys, x, ctx["meta"], ctx["pool"], layer, group, stream=s)
            torch.cuda.synchronize()
            evs = []
            for r in range(args.reps):
                flush.zero_()  # evict activations/weights of the previous launch from L2
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                apply_lora_group_(ys, x, ctx["meta"], ctx["pool"], r % bench.N_LAYERS, group, stream=s)
                e1.record(s)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            us = sum(a.elapsed_time(b) for a, b in evs) * 1e3 / args.reps
            gbs = nbytes / (us * 1e-6) / 1e9
            key = str(v) if v != 1 else f"1.{cfg}"
            res[key] = {"us": round(us, 2), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
        lib.preft_set_lora_variant(-1)
        out["groups"]["/".join(group)] = {"bytes": nbytes, "variants": res}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
