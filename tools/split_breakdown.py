#!/usr/bin/env python
"""Where the config-4 (and 8B r16) split step spends its time: CUDA-graph
replays of the full step, of the shrinks alone, of the expands alone and of
each site group alone, over all layers (rank 0's shard on one GPU, no
collective).  Prints one JSON line per measurement.

usage: python tools/split_breakdown.py [--shape 70b|8b] [--tp 8] [--rank 16]"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="70b")
    ap.add_argument("--tp", type=int, default=8)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--quick", action="store_true", help="whole steps only (no per-group / per-half lines)")
    ap.add_argument("--empty", action="store_true", help="a batch of decode tokens only: the launches' fixed cost")
    ap.add_argument("--fused", default="", help="comma list of K-split pieces: also time the fused kernel")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2605_14217_b200 import AdapterKind, costs, shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.tp import FusedExchange, SplitWorkspace, lora_expand_tp_, lora_fused_tp_, lora_shrink_tp_

    dev = torch.device("cuda", 0)
    shape = shapes.LLAMA_70B if args.shape == "70b" else shapes.LLAMA_8B
    r = args.rank
    pool = AdapterPool(shape.n_layers, shape.d_model, lora_sites=shape.site_dims(), lora_capacity=512, lora_rank=r,
                       dtype=torch.bfloat16, device=dev, tp_rank=0, tp_size=args.tp)
    pool.fill_synthetic_(512, AdapterKind.LORA, r, seed=23, sigma=0.01)
    qsl, ids, flags, lens, _ = bench.step_entries(0, 1, 256, 256, seed=bench.SEED + 3)
    if args.empty:
        flags = flags | 1  # every entry a decode token of a prefill-only adapter: nothing selected
    slots = pool.entry_arrays(qsl, ids, flags)
    T = int(qsl[-1])
    meta = BatchMeta(len(ids), T, tile_tokens=128, device=dev)
    meta.build_arrays(qsl, slots, flags, slot_split=pool.slot_split)
    ws = SplitWorkspace(meta, pool)
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    sets = []
    for _ in range(2):
        acts = {}
        for group in shapes.SITE_GROUPS:
            sh = pool.lora_shard[group[0]]
            x = torch.randn(T, sh.x_width, generator=g, device=dev).to(torch.bfloat16)
            ys = [torch.randn(T, pool.lora_shard[s].y_width, generator=g, device=dev).to(torch.bfloat16) for s in group]
            acts[group] = (x, ys)
        sets.append(acts)
    per = max(1, 64 // r)

    def chunks(group):
        return [group[i:i + per] for i in range(0, len(group), per)]

    def run(groups, do_shrink, do_expand):
        def step(s):
            for layer in range(shape.n_layers):
                acts = sets[layer % 2]
                for group in groups:
                    x, ys = acts[group]
                    for sub in chunks(group):
                        sys_ = [ys[group.index(t)] for t in sub]
                        if ex is not None and do_shrink and do_expand:
                            lora_fused_tp_(sys_, x, meta, pool, layer, sub, ex, s)
                            continue
                        if do_shrink:
                            P = lora_shrink_tp_(sys_, x, meta, pool, layer, sub, ws, s)
                        else:
                            P = ws.view(T, len(sub) * r)
                        if do_expand:
                            lora_expand_tp_(P, sys_, x, meta, pool, layer, sub, s)
        s = torch.cuda.current_stream(dev)
        step(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(s)
        with torch.cuda.stream(cs):
            with torch.cuda.graph(graph, stream=cs):
                step(cs)
        s.wait_stream(cs)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.steps):
            graph.replay()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps

    sel = int(lens.sum())
    distinct = len({ids[i] for i in range(len(ids)) if not (flags[i] & 1)})
    peak, _ = bench.measured_peak_gbs()
    G = shapes.SITE_GROUPS

    def gbytes(groups):
        b = 0
        for group in groups:
            m_loc = pool.lora_shard[group[0]].m_loc
            b += costs.split_group_bytes(m_loc, [pool.lora_shard[t].n_loc for t in group], sel, distinct, r)
        return b * shape.n_layers

    cases = [("step", G, True, True, None)]
    if not args.quick:
        cases += [("shrink_only", G, True, False, None), ("expand_only", G, False, True, None)]
        cases += [("group " + "/".join(gp), [gp], True, True, None) for gp in G]
    for planes in [int(v) for v in args.fused.split(",") if v]:
        exf = FusedExchange.local(meta, pool, planes=planes)
        cases += [(f"fused{planes} step", G, True, True, exf)]
        if not args.quick:
            cases += [(f"fused{planes} group " + "/".join(gp), [gp], True, True, exf) for gp in G]
    out = []
    for name, groups, sh, ex_, exf in cases:
        ex = exf
        ms = run(groups, sh, ex_)
        nl = 1 if ex is not None else int(sh) + int(ex_)
        rec = {"what": name, "ms": round(ms, 4), "launches": shape.n_layers * sum(len(chunks(gp)) for gp in groups) * nl}
        if sh and ex_:
            rec["frac"] = round(gbytes(groups) / (ms / 1e3) / 1e9 / peak, 4)
        rec["us_per_launch"] = round(ms * 1e3 / rec["launches"], 2)
        print(json.dumps(rec), flush=True)
        out.append(rec)


if __name__ == "__main__":
    main()
