#!/usr/bin/env python
"""Determinism check of the tensor-core split pair / fused kernel: the same
group launch repeated from the same inputs must give bit-identical outputs
(whole-unit schedules sum in a fixed order).  Prints, per group, how many of
N repeats differ from the first and the max |difference|.
env: PREFT_SPLIT_EPI=rm selects the read-modify-write expand epilogue."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_2605_14217_b200 import AdapterKind, shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.tp import FusedExchange, SplitWorkspace, apply_lora_group_tp_

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
    ws = SplitWorkspace(meta, pool)
    ex = FusedExchange.local(meta, pool, planes=1) if os.environ.get("FUSED") == "1" else None
    n = int(os.environ.get("REPEATS", "20"))
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    if os.environ.get("CHAIN"):
        # the bench's step: every layer x group, two activation sets, one CUDA graph
        L = int(os.environ.get("CHAIN"))
        pool = AdapterPool(L, shape.d_model, lora_sites=shape.site_dims(), lora_capacity=512, lora_rank=16,
                           dtype=torch.bfloat16, device=dev, tp_rank=0, tp_size=tp)
        pool.fill_synthetic_(512, AdapterKind.LORA, 16, seed=1)
        sets = []
        for _ in range(2):
            acts = {}
            for group in shapes.SITE_GROUPS:
                x = torch.randn(T, pool.lora_shard[group[0]].x_width, generator=g, device=dev).to(torch.bfloat16)
                ys = [torch.randn(T, pool.lora_shard[s].y_width, generator=g, device=dev).to(torch.bfloat16)
                      for s in group]
                acts[group] = (x, ys)
            sets.append(acts)
        init = [{gp: [y.clone() for y in ys] for gp, (x, ys) in acts.items()} for acts in sets]

        def step(st):
            for layer in range(L):
                for group in shapes.SITE_GROUPS:
                    x, ys = sets[layer % 2][group]
                    apply_lora_group_tp_(ys, x, meta, pool, layer, group, workspace=ws, stream=st, collective=False,
                                         exchange=ex)

        s0 = torch.cuda.current_stream()
        step(s0)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(s0)
        with torch.cuda.stream(cs), torch.cuda.graph(graph, stream=cs):
            step(cs)
        s0.wait_stream(cs)
        first, bad, worst = None, 0, 0.0
        for _ in range(n):
            for acts, ini in zip(sets, init):
                for gp, (x, ys) in acts.items():
                    for y, y0 in zip(ys, ini[gp]):
                        y.copy_(y0)
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            out = [y.clone() for acts in sets for gp, (x, ys) in acts.items() for y in ys]
            if first is None:
                first = out
                continue
            diff = max(float((a.float() - b.float()).abs().max()) for a, b in zip(out, first))
            if diff > 0:
                bad += 1
                worst = max(worst, diff)
        print(f"chain of {L} layers: {bad} of {n - 1} graph replays differ, max |diff| {worst}", flush=True)
        return
    for group in shapes.SITE_GROUPS:
        x = torch.randn(T, pool.lora_shard[group[0]].x_width, generator=g, device=dev).to(torch.bfloat16)
        y0 = [torch.randn(T, pool.lora_shard[s].y_width, generator=g, device=dev).to(torch.bfloat16) for s in group]
        first, bad, worst = None, 0, 0.0
        for _ in range(n):
            ys = [y.clone() for y in y0]
            apply_lora_group_tp_(ys, x, meta, pool, 0, group, workspace=ws, collective=False, exchange=ex)
            torch.cuda.synchronize()
            if first is None:
                first = ys
                continue
            diff = max(float((a.float() - b.float()).abs().max()) for a, b in zip(ys, first))
            if diff > 0:
                bad += 1
                worst = max(worst, diff)
        print(f"{'/'.join(group)}: {bad} of {n - 1} repeats differ, max |diff| {worst}", flush=True)


if __name__ == "__main__":
    main()
