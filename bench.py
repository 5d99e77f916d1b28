#!/usr/bin/env python
"""bench.py — PreFT hot path on B200: prefill adapter tokens/s @512 adapters
(Llama-3.1-8B shapes) and % of HBM roofline.

Workload (BASELINE.json configs[1], "cfg2"): Llama-3.1-8B projection shapes,
32 layers x 7 LoRA^P sites (q/k/v, o, gate/up, down; sites that share an
input run as one fused launch), 512 LoRA^P rank-1 adapters (A, B ~ N(0,
0.01^2)) held in the HBM pool, Uniform Punica batch:
per GPU 256 prefill requests with Punica prompt lengths (lognormal, mean
~24, workload.py:110-116) and adapters uniform over the GPU's adapter shard,
plus 256 decode tokens (PREFILL_ONLY adapters -> skipped) listed first as
the reference engine does (engine.py:618-648).

One step = K1 (device metadata from the resident entry buffer) + 128 fused
LoRA launches (4 groups x 32 layers), issued by the native step plan.
`value` counts SELECTED prefill tokens through all 32 layers x 7 sites per
second of device time (CUDA events, max over ranks).  `e2e` is the same
metric through the reference-shaped host-buffer path: every step uploads the
entries and every layer's site activations from pinned host memory and
reads every updated output back.

Every timed line is followed (outside the timed region) by a parity check of
sampled rows against the CPU oracle on the device's own operands
(`"parity": {...}`); a failed check makes the line say so.

--gpus N without torchrun re-launches itself under torch.distributed.run
(one NCCL rank per GPU).  --impl reference times the UNMODIFIED reference
(prefillsim, installed into oracle/_ref by oracle/build_ref.py) on all host
cores over the same cfg2 batch, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "prefill adapter tokens/s @512 adapters (Llama-3.1-8B shapes); % HBM roofline"
UNIT = "tokens/s"
N_ADAPTERS = 512
RANK = 1
N_LAYERS = 32
SEED = 0


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--requests", type=int, default=256, help="prefill requests per GPU per step")
    p.add_argument("--decodes", type=int, default=256, help="decode tokens per GPU per step")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-punica-step", action="store_true")
    p.add_argument("--no-secondary", action="store_true", help="skip the config-1/3/5 secondary lines")
    p.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded CPU baseline sample length")
    p.add_argument("--ref-cores", type=int, default=0, help="reference arm: processes (0 = every host core)")
    p.add_argument("--no-parity", action="store_true", help="skip the post-timing parity checks")
    p.add_argument("--only", default="", help="comma list of secondary lines to run alone: "
                   "cfg1,cfg3,cfg5,cfg5s,cfg4,serving,punica,lora16 (skips the headline)")
    p.add_argument("--tp-exchange", choices=["fused", "nccl"], default="fused",
                   help="config 4 on a real TP group: the fused kernel's P2P exchange (default) or "
                        "shrink + NCCL all-reduce + expand")
    p.add_argument("--share-gpu", action="store_true",
                   help="functional check of the multi-rank path on a 1-GPU box: every rank on cuda:0, gloo "
                        "for the bookkeeping collectives; the ranks time-share the GPU, so the numbers are not "
                        "scaling measurements")
    p.add_argument("--eager", action="store_true",
                   help="issue the timed steps from the host (default: the K steps replayed as one CUDA graph)")
    p.add_argument("--dry-run", action="store_true",
                   help="CPU/gloo launcher check: routing + collectives + the JSON line, no kernels")
    return p.parse_args(argv)


# ---------------------------------------------------------------- workload


def step_entries(rank: int, world: int, n_prefill: int, n_decode: int, seed: int = SEED):
    """(qsl, adapter ids, flags, prompt lens) of one mixed step on one GPU.

    Prompt lengths: Punica lognormal (the reference's sampler); adapters
    uniform over the adapters this GPU owns (pool sharded by id, requests
    routed to the owner: SURVEY.md 8(e)).  Decode entries first.
    """
    from paper_2605_14217_b200 import _lib
    from paper_2605_14217_b200.workload import AdapterMix, WorkloadConfig, sample_prompt_lens, shard_adapters

    owned = shard_adapters(N_ADAPTERS, rank, world)
    cfg = WorkloadConfig(n_prefill + n_decode, N_ADAPTERS, AdapterMix.UNIFORM, seed + rank)
    lens = sample_prompt_lens(cfg)[:n_prefill]
    rng = np.random.default_rng(seed * 1000 + rank)
    ids = [int(owned[i]) for i in rng.integers(0, len(owned), size=n_prefill + n_decode)]
    all_lens = np.concatenate([np.ones(n_decode, dtype=np.int64), lens])
    qsl = np.concatenate([[0], np.cumsum(all_lens)]).astype(np.int32)
    flags = np.array([_lib.ENTRY_DECODE] * n_decode + [0] * n_prefill, dtype=np.int32)
    adapter_ids = ids[n_prefill:] + ids[:n_prefill]  # decode ids, then prefill ids
    return qsl, adapter_ids, flags, lens, owned


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = Path(tempfile.mkstemp(prefix="clocks_", suffix=".csv")[1])

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.3)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        self.path.unlink(missing_ok=True)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "samples": len(sm),
            "reasons": sorted(reasons),
        }


# ---------------------------------------------------------------- roofline helpers


def measured_peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except (KeyError, ValueError):
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def group_bytes(shape, group, n_tokens: int, distinct: int, rank: int = RANK, elem: int = 2) -> int:
    """Algorithmic bytes of one fused launch: x read once,
    every y read + written, each distinct adapter's A/Bt rows once."""
    from paper_2605_14217_b200 import costs

    return costs.lora_group_bytes(shape.site_dims(), group, n_tokens, distinct, rank, elem)


def ncu_traffic(kernel_hint: str):
    """dram bytes per launch of the dominant kernel from the committed ncu summary, if any."""
    for f in sorted((ROOT / "profiles").glob("ncu_summary_*.json"), reverse=True):
        try:
            d = json.loads(f.read_text())
            v = d.get("kernels", {}).get(kernel_hint, {}).get("dram_bytes_per_launch")
            if v:
                return float(v), f.name
        except (ValueError, OSError):
            continue
    return None, None


# ---------------------------------------------------------------- distributed


def _free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def maybe_self_launch(args) -> None:
    """`bench.py --gpus N` outside torchrun: re-run this script under
    torch.distributed.run with N ranks (one per GPU, NCCL; gloo for
    --dry-run) and exit with its status.  Rank 0 prints the JSON line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "4"))
    sys.stdout.flush()
    sys.exit(subprocess.call(cmd, env=env))


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


_BACKEND = {"name": None}


def dist_init(world, local, backend: str = "nccl"):
    import torch

    if backend == "nccl":
        torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        _BACKEND["name"] = backend


def _reduce_device():
    import torch

    return torch.device("cuda") if _BACKEND["name"] == "nccl" else torch.device("cpu")


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def all_max(value: float, world: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=_reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_sum(value: float, world: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=_reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def all_gather_floats(value: float, world: int) -> list[float]:
    if world == 1:
        return [value]
    import torch
    import torch.distributed as dist

    t = torch.zeros(world, dtype=torch.float64, device=_reduce_device())
    t[int(os.environ.get("RANK", "0"))] = value
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]


# ---------------------------------------------------------------- parity (checker, never timed)


def _np(t):
    import torch

    return t.detach().to(torch.float64).cpu().numpy()


def _row_entries(qsl: np.ndarray, rows: np.ndarray) -> np.ndarray:
    return np.searchsorted(np.asarray(qsl), rows, side="right") - 1


def class_mask(mask: np.ndarray, qsl, slots, pool, lora: bool) -> np.ndarray:
    """Rows a LoRA (or ReFT) launch adds to: selected rows whose slot is of
    that class (slots below pool.slot_split are LoRA adapters)."""
    row_slot = np.asarray(slots)[_row_entries(qsl, np.arange(len(mask)))]
    return mask & ((row_slot < pool.slot_split) if lora else (row_slot >= pool.slot_split))


def sample_rows(mask: np.ndarray, qsl, k: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """(selected rows, unselected rows): k selected rows spread over the
    entries (first/last rows of the longest entries included) + up to 8
    unselected ones."""
    rng = np.random.default_rng(seed)
    sel = np.flatnonzero(mask)
    uns = np.flatnonzero(~mask)
    pick = rng.choice(sel, size=min(k, len(sel)), replace=False) if len(sel) else sel
    lens = np.diff(np.asarray(qsl))
    edge = []
    for e in np.argsort(-lens)[:2]:
        b, en = int(qsl[e]), int(qsl[e + 1])
        edge += [b, en - 1] if mask[b] else []
    pick = np.unique(np.concatenate([pick, np.asarray(edge, dtype=np.int64)])).astype(np.int64)
    u = rng.choice(uns, size=min(8, len(uns)), replace=False) if len(uns) else uns
    return pick, np.sort(u).astype(np.int64)


def _verdict(errs: list[float], n_rows: int, tol: float, extra: dict | None = None) -> dict:
    worst = max(errs) if errs else 0.0
    out = {"status": "pass" if worst <= tol else "FAIL", "rows_checked": int(n_rows),
           "max_rel_err": float(f"{worst:.3e}"), "tol": tol,
           "vs": "oracle/preft_oracle.py (float64) on the device's own operands, sampled rows"}
    if extra:
        out.update(extra)
    return out


BF16_METRIC = ("max|dy_dev - dy_ref| / max|dy_ref| over sampled rows (dy = y - y0, the oracle replaying "
               "y <- bf16(y + delta_L)), less 2 bf16 ulps of max|y| for rounding ties the f32 and f64 deltas "
               "resolve differently")


def _bf16_ulp(v: float) -> float:
    return 2.0 ** (np.floor(np.log2(max(v, 1e-30))) - 7)


def _excess(d_out: np.ndarray, d_ref: np.ndarray, y_ref: np.ndarray) -> float:
    """Relative error of an accumulated bf16 update beyond 2 output ulps."""
    den = float(np.max(np.abs(d_ref))) if d_ref.size else 0.0
    err = float(np.max(np.abs(d_out - d_ref), initial=0.0))
    err = max(0.0, err - 2 * _bf16_ulp(float(np.max(np.abs(y_ref), initial=0.0))))
    return err / den if den > 0 else err


def _rel(out: np.ndarray, ref: np.ndarray) -> float:
    den = float(np.max(np.abs(ref))) if ref.size else 0.0
    return float(np.max(np.abs(out - ref))) / den if den > 0 else float(np.max(np.abs(out - ref), initial=0.0))


BF16_METRIC_TC = ("max|dy_dev - dy_ref| / max|dy_ref| over sampled rows (dy = y - y0, the oracle replaying "
                  "y <- bf16(y + bf16(delta_L)): the tcgen05 expand adds the bf16-rounded delta into y by TMA "
                  "reduce-add in L2), less 2 bf16 ulps of max|y|")


def lora_rows_delta(pool, layers, site: str, row_slots: np.ndarray, x_rows: np.ndarray, shard=None,
                    base: np.ndarray | None = None, delta_bf16: bool = False) -> np.ndarray:
    """The LoRA delta of each row (adapters.py:284-288) with the pool's stored
    operands (for a TP shard: its own A / B slices and the matching slice of
    x), summed over `layers`.  With `base`, returns instead the chain the
    device computes when every layer adds into the same bf16 output:
    y <- bf16(y + delta_L) layer after layer, or with delta_bf16 (the tcgen05
    expand's reduce-add epilogue: the delta is stored in bf16 and the L2 adds
    it to y) y <- bf16(y + bf16(delta_L)).  Over 40 chained layers whose
    deltas are ~1-3 ulps of y, the two models differ by several ulps of y."""
    import torch

    from oracle import preft_oracle as O

    idx = torch.as_tensor(row_slots, device=pool.device, dtype=torch.long)
    n = pool.lora_shard[site].n_loc if shard else pool.lora_sites[site][0]
    def bf16(v):
        return torch.from_numpy(v).to(torch.bfloat16).double().numpy()

    out = np.zeros((len(row_slots), n)) if base is None else base.copy()
    for L in layers:
        A = _np(pool.lora_A[site][L].index_select(0, idx))
        Bt = _np(pool.lora_Bt[site][L].index_select(0, idx))
        sc = _np(pool.lora_scale[site][L].index_select(0, idx))
        d = np.stack([O.delta_rows("lora", float(sc[j]), x_rows[j:j + 1], A=A[j], B=Bt[j].T)[0]
                      for j in range(len(row_slots))]) if len(row_slots) else np.zeros((0, n))
        if base is None:
            out += d
        else:
            out = bf16(out + (bf16(d) if delta_bf16 else d))
    return out


def check_lora_accumulated(pool, meta, qsl, slots, groups_acts, snapshot, layers, k=48, seed=0,
                           n_updates: int = 1, delta_bf16: bool = False) -> dict:
    """After one more run of a timed plan: y_s[rows] must equal y0 plus every
    layer's delta, each rounded into the bf16 output as the device stores it
    (the oracle replays y <- bf16(y + delta_L)); unselected rows untouched
    bit for bit.  `groups_acts` {group: (x, ys)}, `snapshot` {group: [y0 per
    site]} taken just before the run."""
    import torch

    mask = class_mask(meta.mask_host(), qsl, slots, pool, lora=True)
    sel, uns = sample_rows(mask, qsl, k, seed)
    ent = _row_entries(qsl, sel)
    row_slots = np.asarray(slots)[ent]
    errs, dlt = [], []
    for group, (x, ys) in groups_acts.items():
        xr = _np(x[torch.as_tensor(sel, device=x.device)])
        for s, y, y0 in zip(group, ys, snapshot[group]):
            if len(uns):
                ui = torch.as_tensor(uns, device=y.device)
                if not torch.equal(y[ui], y0[ui]):
                    return _verdict([float("inf")], len(sel), 2e-2, {"error": f"{s}: unselected rows modified"})
            si = torch.as_tensor(sel, device=y.device)
            out, base = _np(y[si]), _np(y0[si])
            ref = lora_rows_delta(pool, layers, s, row_slots, xr, base=base, delta_bf16=delta_bf16)
            errs.append(_excess(out - base, ref - base, ref))
            dlt.append(_rel(out, ref))
    return _verdict(errs, len(sel), 2e-2, {"output_rel_err": float(f"{max(dlt):.3e}"), "layers": len(layers),
                                           "metric": BF16_METRIC_TC if delta_bf16 else BF16_METRIC})


def check_reft_chain(pool, meta, qsl, slots, h, h0_rows, sel, layers, kind_label: str) -> dict:
    """A ReFT plan applies the residual edit layer after layer to the same h
    (model.py:543-546 once per layer): the oracle replays the chain on the
    sampled rows in float64, rounding to bf16 between layers as the stored
    activation is."""
    import torch

    from oracle import preft_oracle as O

    ent = _row_entries(qsl, sel)
    js = np.asarray(slots)[ent] - pool.slot_split
    idx = torch.as_tensor(js, device=pool.device, dtype=torch.long)
    ref = h0_rows.copy()
    for L in layers:
        A = _np(pool.reft_A[L].index_select(0, idx))
        B = _np(pool.reft_B[L].index_select(0, idx))
        b = _np(pool.reft_bias[L].index_select(0, idx))
        sc = _np(pool.reft_scale[L].index_select(0, idx))
        for j in range(len(sel)):
            ref[j] = ref[j] + O.delta_rows("direft", float(sc[j]), ref[j:j + 1], A=A[j], B=B[j], b=b[j])[0]
        ref = torch.from_numpy(ref).to(torch.bfloat16).double().numpy()
    out = _np(h[torch.as_tensor(sel, device=h.device)])
    return _verdict([_rel(out, ref)], len(sel), 2e-2, {"layers": len(layers), "chain": kind_label})


def check_reft_single(pool, meta, qsl, slots, h, layer: int, k=48, seed=0) -> dict:
    """One apply_reft_ launch on a copy of h: the delta itself to tolerance."""
    import torch

    from oracle import preft_oracle as O
    from paper_2605_14217_b200.ops import apply_reft_

    mask = class_mask(meta.mask_host(), qsl, slots, pool, lora=False)
    sel, uns = sample_rows(mask, qsl, k, seed)
    hc = h.clone()
    apply_reft_(hc, meta, pool, layer)
    torch.cuda.synchronize()
    si = torch.as_tensor(sel, device=h.device)
    base, out = _np(h[si]), _np(hc[si])
    if len(uns):
        ui = torch.as_tensor(uns, device=h.device)
        if not torch.equal(hc[ui], h[ui]):
            return _verdict([float("inf")], len(sel), 2e-2, {"error": "unselected rows modified"})
    js = np.asarray(slots)[_row_entries(qsl, sel)] - pool.slot_split
    d_ref = np.zeros_like(base)
    for j in range(len(sel)):
        jj = int(js[j])
        d_ref[j] = O.delta_rows("direft", float(_np(pool.reft_scale[layer][jj])), base[j:j + 1],
                                A=_np(pool.reft_A[layer][jj]), B=_np(pool.reft_B[layer][jj]),
                                b=_np(pool.reft_bias[layer][jj]))[0]
    # the stored output adds one bf16 rounding of |h| on top of the delta
    ulp = float(np.max(np.abs(base + d_ref))) * 2.0 ** -8
    err = float(np.max(np.abs((out - base) - d_ref)))
    rel = err / max(float(np.max(np.abs(d_ref))), 1e-30)
    ok = err <= 2e-2 * float(np.max(np.abs(d_ref))) + ulp
    return {"status": "pass" if ok else "FAIL", "rows_checked": int(len(sel)), "delta_rel_err": float(f"{rel:.3e}"),
            "tol": "2e-2 x max|delta| + 1 bf16 ulp of the output", "layer": layer,
            "vs": "oracle/preft_oracle.py (float64) on the device's own operands, sampled rows"}


# ---------------------------------------------------------------- our arm


def build_step(args, rank, world, device, n_prefill, n_decode, seed=SEED, lora_rank: int = RANK):
    import torch

    from paper_2605_14217_b200 import AdapterKind, shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.plan import StepPlan
    from paper_2605_14217_b200.pool import AdapterPool

    shape = shapes.LLAMA_8B
    qsl, ids, flags, lens, owned = step_entries(rank, world, n_prefill, n_decode, seed)
    pool = AdapterPool(N_LAYERS, shape.d_model, lora_sites=shape.site_dims(), lora_capacity=len(owned),
                       lora_rank=lora_rank, dtype=torch.bfloat16, device=device)
    pool.fill_synthetic_(0, AdapterKind.LORA, lora_rank, seed=seed + 17 * rank, sigma=0.01, ids=owned)
    slots = pool.entry_arrays(qsl, ids, flags)
    E, T = len(ids), int(qsl[-1])
    meta = BatchMeta(E, T, tile_tokens=128, device=device)
    meta.build_arrays(qsl, slots, flags, slot_split=pool.slot_split)  # entries now resident in HBM
    dims = shape.site_dims()
    g = torch.Generator(device=device)
    g.manual_seed(1234 + rank)
    acts = {}
    for group in shapes.SITE_GROUPS:
        m = dims[group[0]][1]
        x = torch.randn(T, m, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
        ys = [torch.randn(T, dims[s][0], generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
              for s in group]
        acts[group] = (x, ys)
    plan = StepPlan(meta, pool, max_tokens=T)
    for layer in range(N_LAYERS):
        for group in shapes.SITE_GROUPS:
            x, ys = acts[group]
            # the roofline's per-launch time comes from CUDA events around tagged launches
            # inside the timed steps; an event between two launches breaks their PDL
            # overlap, so only every TIMED_EVERY-th layer's gate/up launch is tagged
            timed = group == ("Wgate", "Wup") and layer % TIMED_EVERY == 0
            plan.add_lora_group(ys, x, layer, group, tag=1 if timed else 0)
    sel_prefill = int(lens.sum())
    distinct = len({ids[i] for i in range(len(ids)) if not (flags[i] & 1)})
    return dict(shape=shape, pool=pool, meta=meta, plan=plan, acts=acts, qsl=qsl, ids=ids, flags=flags, slots=slots,
                lens=lens, T=T, E=E, sel=sel_prefill, distinct=distinct, owned=owned, rank=lora_rank)


TIMED_EVERY = int(os.environ.get("PREFT_BENCH_TIMED_EVERY", "32"))


def time_steps(ctx, args, world, device, timing_tag=None):
    import torch

    plan = ctx["plan"]
    s = torch.cuda.current_stream(device)
    for _ in range(args.warmup):
        plan.run(s)
    torch.cuda.synchronize()
    graph = None
    if not args.eager:
        # the K timed steps as ONE CUDA graph (K1 + every site launch of every
        # step; the tagged launches' events as external event nodes), replayed
        # once untimed and once timed
        graph = plan.capture_steps(args.steps, timing_tag=timing_tag)
        graph.replay()
        torch.cuda.synchronize()
    elif timing_tag is not None:
        plan.set_timing(timing_tag, args.steps * N_LAYERS + 8)
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    if graph is not None:
        graph.replay()
    else:
        for _ in range(args.steps):
            plan.run(s)
    e1.record(s)
    torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    kernel = None
    if timing_tag is not None:
        total, count = plan.collect_timing()
        plan.set_timing(-1, 0)
        kernel = (total, count)
    del graph
    return ms, kernel


def parity_lora_plan(ctx, run_once, seed: int = 0, delta_bf16: bool = False) -> dict:
    """One more run of the timed plan (every layer adds into the same y):
    sampled rows of every site == y0 + sum of 32 layers' deltas (oracle)."""
    import torch

    # the timed steps added the same deltas into y again and again (|y| grows
    # until bf16 cannot resolve one delta): restart from fresh N(0, 1) outputs
    gen = torch.Generator(device=ctx["pool"].device)
    gen.manual_seed(4242 + seed)
    for x, ys in ctx["acts"].values():
        for y in ys:
            y.copy_(torch.randn(y.shape, generator=gen, device=y.device))
    snap = {g: [y.clone() for y in ys] for g, (x, ys) in ctx["acts"].items()}
    run_once()
    torch.cuda.synchronize()
    out = check_lora_accumulated(ctx["pool"], ctx["meta"], ctx["qsl"], ctx["slots"], ctx["acts"], snap,
                                 range(N_LAYERS), seed=seed, n_updates=N_LAYERS, delta_bf16=delta_bf16)
    del snap
    return out


def run_e2e(ctx, args, world, device):
    """Host-buffer path: per step H2D of the entries + every layer's site
    activations from pinned memory, the kernels, D2H of every updated output.
    Copies run on their own streams, double-buffered against compute.  The
    last layer's host outputs are checked against the oracle afterwards."""
    import torch

    from paper_2605_14217_b200 import shapes
    from paper_2605_14217_b200.ops import apply_lora_group_

    pool, meta, T = ctx["pool"], ctx["meta"], ctx["T"]
    dims = ctx["shape"].site_dims()
    host_in, dev = {}, [{}, {}]
    g = torch.Generator()
    g.manual_seed(99)
    h2d_bytes = d2h_bytes = 0
    host_out = [{}, {}]
    for group in shapes.SITE_GROUPS:
        m = dims[group[0]][1]
        xs = torch.randn(T, m, generator=g).to(torch.bfloat16).pin_memory()
        ys = [torch.randn(T, dims[s][0], generator=g).to(torch.bfloat16).pin_memory() for s in group]
        host_in[group] = (xs, ys)
        for b in range(2):
            dev[b][group] = (torch.empty_like(xs, device=device), [torch.empty_like(y, device=device) for y in ys])
            host_out[b][group] = [torch.empty_like(y).pin_memory() for y in ys]
        h2d_bytes += xs.numel() * 2 + sum(y.numel() * 2 for y in ys)
        d2h_bytes += sum(y.numel() * 2 for y in ys)
    comp = torch.cuda.current_stream(device)
    up, down = torch.cuda.Stream(device), torch.cuda.Stream(device)
    h2d_done = [torch.cuda.Event(), torch.cuda.Event()]
    comp_done = [torch.cuda.Event(), torch.cuda.Event()]
    d2h_done = [torch.cuda.Event(), torch.cuda.Event()]
    qsl, slots, flags = ctx["qsl"], ctx["slots"], ctx["flags"]

    def one_step():
        meta.build_arrays(qsl, slots, flags, stream=comp, slot_split=pool.slot_split)  # entries H2D + K1
        for layer in range(N_LAYERS):
            b = layer % 2
            with torch.cuda.stream(up):
                if layer >= 2:
                    up.wait_event(d2h_done[b])
                for group in shapes.SITE_GROUPS:
                    xs, ys = host_in[group]
                    xd, yds = dev[b][group]
                    xd.copy_(xs, non_blocking=True)
                    for yd, yh in zip(yds, ys):
                        yd.copy_(yh, non_blocking=True)
                h2d_done[b].record(up)
            comp.wait_event(h2d_done[b])
            for group in shapes.SITE_GROUPS:
                xd, yds = dev[b][group]
                apply_lora_group_(yds, xd, meta, pool, layer, group, stream=comp)
            comp_done[b].record(comp)
            with torch.cuda.stream(down):
                down.wait_event(comp_done[b])
                for group in shapes.SITE_GROUPS:
                    for yh, yd in zip(host_out[b][group], dev[b][group][1]):
                        yh.copy_(yd, non_blocking=True)
                d2h_done[b].record(down)
        comp.wait_stream(up)
        comp.wait_stream(down)

    for _ in range(max(1, min(args.warmup, 2))):
        one_step()
    torch.cuda.synchronize()
    barrier(world)
    n = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for _ in range(n):
        one_step()
    e1.record(comp)
    torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1) / n
    parity = None
    if not args.no_parity:
        # host_out[1] holds layer 31's outputs: host y + layer 31's delta of host x
        last = N_LAYERS - 1
        acts = {gp: (host_in[gp][0], host_out[last % 2][gp]) for gp in shapes.SITE_GROUPS}
        snap = {gp: host_in[gp][1] for gp in shapes.SITE_GROUPS}
        parity = check_lora_accumulated(pool, meta, qsl, slots, acts, snap, [last], seed=3)
        parity["what"] = "host outputs of layer 31 (last step) vs host inputs + oracle delta"
    return ms, N_LAYERS * h2d_bytes + meta.h2d_bytes, N_LAYERS * d2h_bytes, n, parity


def punica_step(args, rank, world, device):
    """Secondary point: a Punica-sized step (32 prefill requests + 32 decode
    tokens, max_batch 32, engine.py:101-112), CUDA-graph replayed."""
    import torch

    ctx = build_step(args, rank, world, device, 32, 32, seed=SEED + 7)
    g = ctx["plan"].capture()
    s = torch.cuda.current_stream(device)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record(s)
    for _ in range(n):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    out = {"workload": "Punica-sized step: 32 prefill requests + 32 decode tokens (engine.py:101-112), cfg2 shapes",
           "prefill_tokens": ctx["sel"], "ms_per_step": round(ms, 4),
           "value": round(ctx["sel"] / (ms / 1e3), 1), "unit": UNIT, "launch": "cuda graph",
           "rows_hint": ctx["plan"].rows_hint}
    if not args.no_parity:
        out["parity"] = parity_lora_plan(ctx, g.replay, seed=7)
    del ctx, g
    torch.cuda.empty_cache()
    return out


def lora_rank_config(args, device, rank_r: int = 16) -> dict:
    """LoRA^P at rank 16 on one GPU through the standard apply path (8B shapes,
    the cfg2 batch): where r makes the LoRA a contraction (~10.5 FLOP/B)."""
    import torch

    from paper_2605_14217_b200 import costs, shapes

    ctx = build_step(args, 0, 1, device, args.requests, args.decodes, lora_rank=rank_r)
    steps = max(3, min(args.steps, 10))
    a2 = argparse.Namespace(**{**vars(args), "steps": steps, "warmup": 2})
    ms, kernel = time_steps(ctx, a2, 1, device, timing_tag=1)
    k_ms, k_n = kernel
    dims = ctx["shape"].site_dims()
    step_bytes = N_LAYERS * sum(costs.lora_group_bytes(dims, g, ctx["sel"], ctx["distinct"], rank_r)
                                for g in shapes.SITE_GROUPS)
    gu = costs.lora_group_bytes(dims, ("Wgate", "Wup"), ctx["sel"], ctx["distinct"], rank_r)
    peak, _ = measured_peak_gbs()
    out = {"workload": f"8B shapes, 512 LoRA^P r{rank_r} adapters, cfg2 batch ({ctx['sel']} prefill tokens), 1 GPU",
           "prefill_tokens": ctx["sel"], "ms_per_step": round(ms / steps, 4),
           "value": round(ctx["sel"] * steps / (ms / 1e3), 1), "unit": UNIT,
           "step_frac_of_hbm_peak": round(step_bytes / (ms / steps / 1e3) / 1e9 / peak, 4),
           "gate_up_frac_of_hbm_peak": round(gu / (k_ms / k_n / 1e3) / 1e9 / peak, 4),
           "gate_up_avg_launch_us": round(k_ms / k_n * 1e3, 2)}
    if not args.no_parity:
        out["parity"] = parity_lora_plan(ctx, lambda: ctx["plan"].run(), seed=16, delta_bf16=True)
    # the same step through the fused kernel (one launch per group: shrink ->
    # one-rank exchange -> expand, csrc/lora_fused.cu)
    from paper_2605_14217_b200.tp import FusedExchange, lora_fused_tp_

    ex = FusedExchange.local(ctx["meta"], ctx["pool"])

    def fstep(st):
        for layer in range(N_LAYERS):
            for group in shapes.SITE_GROUPS:
                x, ys = ctx["acts"][group]
                lora_fused_tp_(ys, x, ctx["meta"], ctx["pool"], layer, group, ex, st)

    s = torch.cuda.current_stream(device)
    fstep(s)
    torch.cuda.synchronize()
    fg = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(device)
    cs.wait_stream(s)
    with torch.cuda.stream(cs), torch.cuda.graph(fg, stream=cs):
        fstep(cs)
    s.wait_stream(cs)
    fg.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        fg.replay()
    e1.record(s)
    torch.cuda.synchronize()
    fms = e0.elapsed_time(e1) / steps
    out["fused_kernel"] = {"ms_per_step": round(fms, 4),
                           "step_frac_of_hbm_peak": round(step_bytes / (fms / 1e3) / 1e9 / peak, 4),
                           "launches_per_step": N_LAYERS * len(shapes.SITE_GROUPS), "errors": ex.errors(),
                           "note": "one launch per site group: shrink -> one-rank exchange -> expand"}
    del ctx, fg, ex
    torch.cuda.empty_cache()
    return out


def reft_config(args, device, kind_name: str, rank: int, lens, ids, label: str, steps: int = 5,
                world: int = 1, grank: int = 0, owned=None, strong: dict | None = None) -> dict:
    """A ReFT^P residual site x 32 layers (8B shapes) over one batch of long
    prompts, one fused launch per layer (BASELINE configs 3/5).

    Weak scaling (default): each rank holds its 512/world shard of the pool
    (adapter a on GPU a mod world) and serves prompts routed to it, the
    prompt set per rank fixed.  `owned` / `strong`: the caller routed one
    global request stream (strong scaling) and passes this rank's adapters
    (its shard plus hot replicas) and its requests."""
    import torch

    from paper_2605_14217_b200 import AdapterKind, costs, shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.plan import StepPlan
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.workload import shard_adapters

    d = shapes.LLAMA_8B.d_model
    kind = AdapterKind(kind_name)
    if owned is None:
        owned = shard_adapters(N_ADAPTERS, grank, world)
        ids = [int(owned[int(a) % len(owned)]) for a in ids]  # requests routed to this GPU's adapters
    pool = AdapterPool(N_LAYERS, d, reft_capacity=len(owned), reft_rank=rank, dtype=torch.bfloat16, device=device)
    pool.fill_synthetic_(0, kind, rank, seed=5 + grank, ids=owned)
    n_dec = 64
    all_lens = np.concatenate([np.ones(n_dec, dtype=np.int64), np.asarray(lens, dtype=np.int64)])
    qsl = np.concatenate([[0], np.cumsum(all_lens)]).astype(np.int32)
    flags = np.array([1] * n_dec + [0] * len(lens), dtype=np.int32)
    eids = [int(owned[i % len(owned)]) for i in range(n_dec)] + [int(a) for a in ids]
    slots = pool.entry_arrays(qsl, eids, flags)
    T = int(qsl[-1])
    meta = BatchMeta(len(eids), T, tile_tokens=128, device=device)
    meta.build_arrays(qsl, slots, flags, slot_split=pool.slot_split)
    h = torch.randn(T, d, device=device, dtype=torch.float32).to(torch.bfloat16)
    plan = StepPlan(meta, pool, max_tokens=T)
    for layer in range(N_LAYERS):
        plan.add_reft(h, layer, tag=1 if layer % 8 == 0 else 0)  # sampled launch timing (see TIMED_EVERY)
    s = torch.cuda.current_stream(device)
    for _ in range(2):
        plan.run(s)
    plan.set_timing(1, steps * N_LAYERS)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        plan.run(s)
    e1.record(s)
    torch.cuda.synchronize()
    my_ms = e0.elapsed_time(e1) / steps
    ms = all_max(my_ms, world)
    k_ms, k_n = plan.collect_timing()
    sel = int(np.sum(lens))
    per_rank_sel = all_gather_floats(sel, world)
    sel_all = int(sum(per_rank_sel))
    distinct = len(set(int(a) for a in ids))
    per_launch = costs.reft_bytes(d, sel, distinct, rank)
    peak, _ = measured_peak_gbs()
    frac = per_launch / (k_ms / k_n / 1e3) / 1e9 / peak
    frac = all_sum(frac, world) / world
    tag = ""
    if strong:
        tag = f" [{world} GPUs, one global stream routed to adapter owners + hot replicas, strong scaling]"
    elif world > 1:
        tag = f" [{world} GPUs, adapter-sharded, weak scaling]"
    out = {"workload": label + tag, "prefill_tokens": sel_all, "ms_per_step": round(ms, 3),
           "value": round(sel_all / (ms / 1e3), 1), "unit": UNIT, "kernel_frac_of_hbm_peak": round(frac, 4),
           "avg_launch_us": round(k_ms / k_n * 1e3, 2), "n_gpus": world,
           "scaling": "strong" if strong else "weak"}
    if world > 1:
        mean = sel_all / world
        out["per_rank_prefill_tokens"] = [int(v) for v in per_rank_sel]
        out["token_imbalance_max_over_mean"] = round(max(per_rank_sel) / mean, 3) if mean else None
    if strong:
        out.update(strong)
    if not args.no_parity:
        h.copy_(torch.randn(h.shape, device=device))  # fresh activations (the timed steps edited h 32 x steps times)
        mask = class_mask(meta.mask_host(), qsl, slots, pool, lora=False)
        sel_rows, _ = sample_rows(mask, qsl, 32, seed=5)
        h0 = _np(h[torch.as_tensor(sel_rows, device=device)])
        plan.run(s)
        torch.cuda.synchronize()
        par = {"plan_32_layers": check_reft_chain(pool, meta, qsl, slots, h, h0, sel_rows, range(N_LAYERS),
                                                  "h <- bf16(h + delta_L(h)), L = 0..31"),
               "single_launch": check_reft_single(pool, meta, qsl, slots, h, 0, seed=6)}
        par["status"] = "pass" if all(v["status"] == "pass" for v in par.values()) else "FAIL"
        if world > 1:
            oks = all_sum(1.0 if par["status"] == "pass" else 0.0, world)
            par["ranks_passed"] = int(oks)
        out["parity"] = par
    del pool, meta, plan, h
    torch.cuda.empty_cache()
    return out


def cfg5_strong(args, device, world: int, grank: int) -> dict:
    """BASELINE config 5 as a multi-GPU serving problem: ONE global Zipf
    request stream (workload.py:137-140) over 512 LoReFT^P r32 adapters,
    prompts U[8k, 16k]; hot adapters (share > 0.5/world, e.g. adapter 0 with
    ~15%) are replicated on every GPU (workload.hot_replicas) and every
    request is routed to a GPU holding its adapter, least-loaded replica
    first (workload.route_requests).  Total work is fixed as world grows."""
    from paper_2605_14217_b200.workload import (AdapterMix, WorkloadConfig, assign_adapters, hot_replicas,
                                                route_requests, shard_adapters)

    n_req = 16
    ids = [int(a) for a in assign_adapters(WorkloadConfig(n_req, N_ADAPTERS, AdapterMix.SKEWED, seed=11))]
    lens = np.random.default_rng(12).integers(8192, 16385, size=n_req)
    hot = hot_replicas(ids, world)
    routes = route_requests(ids, world, hot, lens)
    mine = routes[grank]
    owned = sorted(set(shard_adapters(N_ADAPTERS, grank, world)) | {a for a, hs in hot.items() if grank in hs})
    info = {"global_requests": n_req, "global_prefill_tokens": int(lens.sum()),
            "hot_replicated_adapters": sorted(hot), "requests_per_rank": [len(r) for r in routes]}
    if not mine:  # nothing routed here: still take part in the collectives with an idle step
        mine_lens, mine_ids = [1], [owned[0]]
    else:
        mine_lens, mine_ids = [int(lens[i]) for i in mine], [ids[i] for i in mine]
    return reft_config(args, device, "loreft", 32, mine_lens, mine_ids,
                       "cfg5 strong: one Zipf stream of 16 prompts U[8k,16k] over 512 LoReFT^P r32 adapters x 32 layers",
                       world=world, grank=grank, owned=owned, strong=info)


def lora_reft_mix_config(args, device) -> dict:
    """Config 1 on the GPU: one layer, d = 4096, 16 DiReFT^P r=8 + 16 LoRA^P r=1
    (one 4096->4096 site), 32 prefill x 128 + 32 decode tokens."""
    import torch

    from paper_2605_14217_b200 import AdapterKind
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_, apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    d = 4096
    pool = AdapterPool(1, d, lora_sites={"Wq": (d, d)}, lora_capacity=16, lora_rank=1, reft_capacity=16,
                       reft_rank=8, dtype=torch.bfloat16, device=device)
    pool.fill_synthetic_(16, AdapterKind.LORA, 1, seed=1, ids=list(range(16, 32)))
    pool.fill_synthetic_(16, AdapterKind.DIREFT, 8, seed=2, ids=list(range(16)))
    lens = [1] * 32 + [128] * 32
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    flags = np.array([1] * 32 + [0] * 32, dtype=np.int32)
    eids = [i % 32 for i in range(32)] + list(range(32))
    slots = pool.entry_arrays(qsl, eids, flags)
    meta = BatchMeta(64, int(qsl[-1]), device=device)
    meta.build_arrays(qsl, slots, flags, slot_split=pool.slot_split)
    T = int(qsl[-1])
    x = torch.randn(T, d, device=device).to(torch.bfloat16)
    y = torch.randn(T, d, device=device).to(torch.bfloat16)
    h = torch.randn(T, d, device=device).to(torch.bfloat16)
    s = torch.cuda.current_stream(device)
    for _ in range(3):
        apply_lora_(y, x, meta, pool, 0, "Wq")
        apply_reft_(h, meta, pool, 0)
    torch.cuda.synchronize()
    n = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        meta.launch(s)
        apply_lora_(y, x, meta, pool, 0, "Wq")
        apply_reft_(h, meta, pool, 0)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    out = {"workload": "cfg1: 1 layer d=4096, 16 DiReFT^P r8 + 16 LoRA^P r1, 32x128 prefill + 32 decode",
           "prefill_tokens": 4096, "ms_per_step": round(ms, 4),
           "value": round(4096 / (ms / 1e3), 1), "unit": "tokens/s per (layer, site pair)"}
    if not args.no_parity:
        y.copy_(torch.randn(y.shape, device=device))  # fresh: the timed loop added the same delta 53 times
        h.copy_(torch.randn(h.shape, device=device))
        y0 = y.clone()
        meta.launch(s)
        apply_lora_(y, x, meta, pool, 0, "Wq")
        torch.cuda.synchronize()
        lora = check_lora_accumulated(pool, meta, qsl, slots, {("Wq",): (x, [y])}, {("Wq",): [y0]}, [0], seed=1)
        reft = check_reft_single(pool, meta, qsl, slots, h, 0, seed=2)
        out["parity"] = {"status": "pass" if lora["status"] == reft["status"] == "pass" else "FAIL",
                         "lora": lora, "reft": reft}
    del pool, meta
    torch.cuda.empty_cache()
    return out


def tp_config(args, device, world: int, rank: int, steps: int = 5) -> dict | None:
    """BASELINE config 4: Llama-3.1-70B shapes (80 layers, 7 LoRA^P sites), 512
    LoRA^P r=16 adapters, 8-way tensor parallelism with the pool sharded along
    m (A) and n (B) and the rank-r shrink partials all-reduced over NCCL
    (tp.py).  At 8 GPUs the real TP group runs; on 1 GPU rank 0's share of the
    work runs without the collective (its 26.5 GB shard of the pool, the same
    batch).  Each step is CUDA-graph replayed (shrink, all-reduce, expand per
    group and layer)."""
    import torch

    from paper_2605_14217_b200 import AdapterKind, costs, shapes
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.tp import FusedExchange, SplitWorkspace, apply_lora_group_tp_

    tp = 8
    if world not in (1, tp):
        return None
    real = world == tp
    shape = shapes.LLAMA_70B
    r = 16
    dims = shape.site_dims()
    pool = AdapterPool(shape.n_layers, shape.d_model, lora_sites=dims, lora_capacity=N_ADAPTERS, lora_rank=r,
                       dtype=torch.bfloat16, device=device, tp_rank=rank if real else 0, tp_size=tp)
    pool.fill_synthetic_(N_ADAPTERS, AdapterKind.LORA, r, seed=23, sigma=0.01)
    qsl, ids, flags, lens, _ = step_entries(0, 1, args.requests, args.decodes, seed=SEED + 3)
    slots = pool.entry_arrays(qsl, ids, flags)
    T = int(qsl[-1])
    meta = BatchMeta(len(ids), T, tile_tokens=128, device=device)
    meta.build_arrays(qsl, slots, flags, slot_split=pool.slot_split)
    ws = SplitWorkspace(meta, pool)
    g = torch.Generator(device=device)
    g.manual_seed(77 + rank)
    sets = []
    for _ in range(2):  # two activation sets alternate across layers (> L2 between reuses)
        acts = {}
        for group in shapes.SITE_GROUPS:
            sh = pool.lora_shard[group[0]]
            x = torch.randn(T, sh.x_width, generator=g, device=device).to(torch.bfloat16)
            ys = [torch.randn(T, pool.lora_shard[s].y_width, generator=g, device=device).to(torch.bfloat16)
                  for s in group]
            acts[group] = (x, ys)
        sets.append(acts)

    # on a real TP group the partials travel through the fused kernel's
    # cudaIpc exchange (no NCCL call on the data path) unless --tp-exchange nccl
    ex, exchange = None, "NCCL all-reduce of the rank-r partials between the shrink and expand kernels"
    if real and args.tp_exchange == "fused":
        try:
            ex = FusedExchange.group(meta, pool)
            exchange = "fused kernel: partials stored into every rank's exchange region over NVLink (cudaIpc)"
        except Exception as exc:  # keep the NCCL path measurable
            exchange += f" (fused exchange unavailable: {type(exc).__name__}: {exc})"
    if not real:
        exchange = "omitted (1 GPU)"

    def step(s, fused_ex=None):
        for layer in range(shape.n_layers):
            acts = sets[layer % 2]
            for group in shapes.SITE_GROUPS:
                x, ys = acts[group]
                apply_lora_group_tp_(ys, x, meta, pool, layer, group, workspace=ws, stream=s, collective=real,
                                     exchange=fused_ex if fused_ex is not None else ex)

    s = torch.cuda.current_stream(device)
    if ex is not None:
        # the first real multi-GPU use of the exchange: a short wait bound, one
        # layer probed first, and the NCCL path if any rank's wait timed out
        ex.c.spin_ns = 200_000_000
        for group in shapes.SITE_GROUPS:
            x, ys = sets[0][group]
            apply_lora_group_tp_(ys, x, meta, pool, 0, group, workspace=ws, stream=s, collective=real, exchange=ex)
        bad = all_max(float(ex.errors()), world)
        if bad:
            exchange = "NCCL all-reduce (the fused exchange timed out on this group; fell back)"
            barrier(world)
            ex.close()
            ex = None
    for _ in range(2):
        step(s)
    torch.cuda.synchronize()
    launch = "cuda graph"
    graph = torch.cuda.CUDAGraph()
    try:
        cs = torch.cuda.Stream(device)
        cs.wait_stream(s)
        with torch.cuda.stream(cs):
            with torch.cuda.graph(graph, stream=cs):
                step(cs)
        s.wait_stream(cs)
        replay = graph.replay
    except Exception as exc:  # e.g. a collective that refuses capture: time the eager launches
        torch.cuda.synchronize()
        launch = f"eager (graph capture failed: {type(exc).__name__})"
        graph = None

        def replay():
            step(s)
    for _ in range(2):
        replay()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        replay()
    e1.record(s)
    torch.cuda.synchronize()
    ms = all_max(e0.elapsed_time(e1) / steps, world)
    sel = int(lens.sum())
    distinct = len({ids[i] for i in range(len(ids)) if not (flags[i] & 1)})
    per_layer = 0
    for group in shapes.SITE_GROUPS:
        m_loc = pool.lora_shard[group[0]].m_loc
        n_locs = [pool.lora_shard[t].n_loc for t in group]
        per_layer += costs.split_group_bytes(m_loc, n_locs, sel, distinct, r)
    step_bytes = shape.n_layers * per_layer
    peak, _ = measured_peak_gbs()
    frac = step_bytes / (ms / 1e3) / 1e9 / peak
    allreduce_bytes = shape.n_layers * sum(T * 4 * r * len(gp) for gp in shapes.SITE_GROUPS)
    out = {"workload": "cfg4: Llama-3.1-70B shapes, 80 layers x 7 LoRA^P sites, 512 LoRA^P r16, TP=8 "
                       + ("(8 GPUs, NCCL all-reduce of the rank-r partials)" if real else
                          "(1 GPU: rank 0's shard and work, all-reduce omitted)"),
           "prefill_tokens": sel, "ms_per_step": round(ms, 3), "value": round(sel / (ms / 1e3), 1), "unit": UNIT,
           "per_rank_frac_of_hbm_peak": round(frac, 4), "per_rank_algorithmic_bytes": int(step_bytes),
           "allreduce_bytes_per_rank_per_step": int(allreduce_bytes) if real else 0,
           "pool_gb_per_rank": round(pool.nbytes / 1e9, 2), "launch": launch, "exchange": exchange}
    if not real and os.environ.get("PREFT_BENCH_NO_FUSED") != "1":
        # the fused shrink -> exchange -> expand kernel that a real TP group
        # runs, on rank 0's shard with a one-rank exchange (its remote stores
        # and waits omitted like the all-reduce above)
        exl = FusedExchange.local(meta, pool, planes=1)
        fg = torch.cuda.CUDAGraph()
        step(s, exl)
        torch.cuda.synchronize()
        cs2 = torch.cuda.Stream(device)
        cs2.wait_stream(s)
        with torch.cuda.stream(cs2), torch.cuda.graph(fg, stream=cs2):
            step(cs2, exl)
        s.wait_stream(cs2)
        fg.replay()
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(steps):
            fg.replay()
        e1.record(s)
        torch.cuda.synchronize()
        fms = e0.elapsed_time(e1) / steps
        out["fused_kernel"] = {"ms_per_step": round(fms, 3), "per_rank_frac_of_hbm_peak":
                               round(step_bytes / (fms / 1e3) / 1e9 / peak, 4), "launches_per_step": 320,
                               "note": "the kernel a real TP group runs (one launch per group and layer), "
                                       "exchange stores to peers omitted on 1 GPU"}
        del fg, exl
    if not args.no_parity and not real:
        # one more replay: set 0 takes the even layers' deltas (rank 0's partial
        # shrink over its m-slice, its n-slice of B; no all-reduce on 1 GPU)
        import torch as _t

        acts0 = sets[0]
        for x, ys in acts0.values():
            for y in ys:
                y.copy_(_t.randn(y.shape, device=device))
        snap = {gp: [y.clone() for y in ys] for gp, (x, ys) in acts0.items()}
        replay()
        _t.cuda.synchronize()
        mask = class_mask(meta.mask_host(), qsl, slots, pool, lora=True)
        sel_rows, _ = sample_rows(mask, qsl, 24, seed=4)
        row_slots = np.asarray(slots)[_row_entries(qsl, sel_rows)]
        errs = []
        idx = _t.as_tensor(sel_rows, device=device)
        for gp, (x, ys) in acts0.items():
            sh0 = pool.lora_shard[gp[0]]
            xr = _np(x[idx])[:, sh0.x_offset: sh0.x_offset + sh0.m_loc]  # the m-slice this rank's A covers
            for sname, y, y0 in zip(gp, ys, snap[gp]):
                sh = pool.lora_shard[sname]
                cols = slice(sh.y_offset, sh.y_offset + sh.n_loc)  # the n-slice this rank adds into
                base, outr = _np(y0[idx]), _np(y[idx])
                ref = lora_rows_delta(pool, range(0, shape.n_layers, 2), sname, row_slots, xr, shard=True,
                                      base=base[:, cols], delta_bf16=True)
                errs.append(_excess(outr[:, cols] - base[:, cols], ref - base[:, cols], ref))
                rest = np.ones(outr.shape[1], bool)
                rest[cols] = False
                if rest.any() and not np.array_equal(outr[:, rest], base[:, rest]):
                    errs.append(float("inf"))  # columns outside the rank's slice must stay untouched
        out["parity"] = _verdict(errs, len(sel_rows), 2e-2, {"what": "rank 0 shard: y_slice <- bf16(y_slice + s "
                                                             "(x_mslice A_shard^T) B_shard^T) over its 40 layers",
                                                             "metric": BF16_METRIC_TC})
    elif real:
        out["parity"] = {"status": "not checked on the multi-rank run (the kernels' TP=8 parity is "
                                   "tests/test_gpu_tp.py at 70B shard widths)"}
    if ex is not None:
        out["exchange_errors"] = ex.errors()
        barrier(world)
        ex.close()
    del pool, meta, ws, sets, graph
    torch.cuda.empty_cache()
    return out


def serving_replay(args, device, n_requests: int = 128, l_max: int = 256) -> dict:
    """the reference engine's schedule replayed on the
    device — Uniform Punica requests over 512 LoRA^P r=1 adapters (8B shapes),
    max_batch 32, at most 32 adapters resident (paged with LRU from pinned
    host slot images), token budget 2048, decode-first mixed
    batches; per step: paging, K1 from the new entries, 32 layers x 4 fused
    LoRA groups through the native step plan.  Tokens/s counts every token
    the steps process (prompt + generated), device time of the whole run."""
    import torch

    from paper_2605_14217_b200 import AdapterKind, shapes
    from paper_2605_14217_b200.adapters import PositionSchedule
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.paging import PagedAdapterPool
    from paper_2605_14217_b200.plan import StepPlan
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.serving import Scheduler, ServeConfig, generate_workload
    from paper_2605_14217_b200.workload import AdapterMix, WorkloadConfig

    shape = shapes.LLAMA_8B
    slots_n = 32
    pool = AdapterPool(N_LAYERS, shape.d_model, lora_sites=shape.site_dims(), lora_capacity=slots_n, lora_rank=RANK,
                       dtype=torch.bfloat16, device=device)
    snaps = {}
    for first in range(0, N_ADAPTERS, slots_n):  # pinned host slot images of all 512 adapters
        ids = list(range(first, min(N_ADAPTERS, first + slots_n)))
        pool.fill_synthetic_(0, AdapterKind.LORA, RANK, seed=100 + first, sigma=0.01, ids=ids)
        for a in ids:
            snaps[a] = pool.export_slot(a)
        torch.cuda.synchronize()
        for a in ids:
            pool.unregister(a, zero=False)
    paged = PagedAdapterPool(pool, {}, snapshots=snaps)
    cfg = ServeConfig(max_batch=32, max_gpu_adapters=slots_n, step_token_budget=2048)
    meta = BatchMeta(cfg.max_batch, cfg.step_token_budget, tile_tokens=128, device=device)
    dims = shape.site_dims()
    g = torch.Generator(device=device)
    g.manual_seed(5)
    T = cfg.step_token_budget
    wl = generate_workload(WorkloadConfig(n_requests, N_ADAPTERS, AdapterMix.UNIFORM, seed=0, l_max=l_max))
    # the K2 launch shape baked into the captured graph: the mean selected
    # rows of this schedule's adapter-carrying steps (host-known up front)
    counts = [st.prefill_tokens for st in Scheduler(wl, cfg, PositionSchedule.PREFILL_ONLY) if st.prefill_tokens]
    hint = int(np.mean(counts)) if counts else T
    plan = StepPlan(meta, pool, max_tokens=T, rows_hint=hint)
    bufs = {}
    for layer in range(N_LAYERS):
        for group in shapes.SITE_GROUPS:
            x = torch.randn(T, dims[group[0]][1], generator=g, device=device).to(torch.bfloat16)
            ys = [torch.randn(T, dims[t][0], generator=g, device=device).to(torch.bfloat16) for t in group]
            plan.add_lora_group(ys, x, layer, group)
            bufs[(layer, group)] = (x, ys)
    s = torch.cuda.current_stream(device)

    # the 128 site launches of a step as one CUDA graph (a serving engine's
    # decode-graph practice); metadata is rebuilt eagerly before each replay
    graph = None
    try:
        graph = plan.capture(run_meta=False)
    except Exception:  # capture unsupported here: eager launches through the native plan
        graph = None
    last = {}

    def run(limit=None):
        steps = toks = pre = 0
        for step in Scheduler(wl, cfg, PositionSchedule.PREFILL_ONLY):
            paged.ensure(step.workset, stream=s)
            # all-unselected steps skip the adapter path, decided on the host
            # (forward_chunk's skip_adapters, model.py:475): decode-only steps
            # of prefill-only adapters launch nothing
            if step.workset:
                flags = step.entry_flags()
                slots = pool.entry_arrays(step.qsl, step.adapter_ids, flags)
                meta.build_arrays(step.qsl, slots, flags, stream=s, slot_split=pool.slot_split)
                if graph is not None:
                    graph.replay()
                else:
                    plan.run(s, run_meta=False)
                last.update(qsl=step.qsl, slots=slots, flags=flags)
            steps += 1
            toks += step.tokens
            pre += step.prefill_tokens
            if limit and steps >= limit:
                break
        return steps, toks, pre

    run(limit=5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0, b0 = paged.page_ins, paged.paged_bytes
    e0.record(s)
    steps, toks, pre = run()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out = {"workload": f"serving replay: Uniform Punica {n_requests} requests (l_max {l_max}) over 512 LoRA^P r1 "
                       f"adapters, 8B shapes x 32 layers, max_batch 32, 32 device slots (LRU paging), budget 2048",
           "steps": steps, "tokens": toks, "prefill_tokens": pre, "ms": round(ms, 2),
           "value": round(toks / (ms / 1e3), 1), "unit": "tokens/s (prompt + generated)",
           "page_ins": paged.page_ins - p0, "paged_gb": round((paged.paged_bytes - b0) / 1e9, 2),
           "launch": "cuda graph per step (site launches), eager paging + K1" if graph is not None else "eager",
           "rows_hint": hint}
    if not args.no_parity and last:
        # the last adapter-carrying step again (its adapters are still resident):
        # layers 0 and 31 of every group vs the oracle
        meta.build_arrays(last["qsl"], last["slots"], last["flags"], stream=s, slot_split=pool.slot_split)
        chk = {(L, gp): bufs[(L, gp)] for L in (0, N_LAYERS - 1) for gp in shapes.SITE_GROUPS}
        snap = {k: [y.clone() for y in v[1]] for k, v in chk.items()}
        graph.replay() if graph is not None else plan.run(s, run_meta=False)
        torch.cuda.synchronize()
        res = [check_lora_accumulated(pool, meta, last["qsl"], last["slots"], {k[1]: v}, {k[1]: snap[k]}, [k[0]],
                                      k=24, seed=9) for k, v in chk.items()]
        worst = max(r["max_rel_err"] for r in res)
        out["parity"] = {"status": "pass" if all(r["status"] == "pass" for r in res) else "FAIL",
                         "rows_checked": res[0]["rows_checked"], "max_rel_err": worst, "tol": 2e-2,
                         "what": "last scheduled step replayed: layers 0 and 31, every site, vs the oracle"}
    del graph, plan, pool, paged, snaps, bufs
    torch.cuda.empty_cache()
    return out


def cpu_baseline(ctx, seconds: float) -> dict:
    """The reference's CPU path (prefillsim from oracle/_ref, else the oracle
    port) on one host core, on a bounded sample of the same workload: the
    first 8 prefill requests (plus 8 decode entries) through all 32 layers."""
    from threadpoolctl import threadpool_limits

    from oracle import cpu_reference as CR

    with threadpool_limits(1):
        res = CR.time_sample(ctx["qsl"], ctx["ids"], ctx["flags"], n_requests=8, seconds=seconds, seed=SEED)
    return {"value": round(res["tokens_per_s"], 3), "unit": UNIT, "cores": 1, "kind": res["kind"],
            "sample": res["sample"]}


def cfg2_config(args, world: int, sel: int, T: int, E: int, distinct: int, tokens_all: int) -> dict:
    return {
        "workload": "cfg2 Uniform Punica saturating step: Llama-3.1-8B shapes, 32 layers x 7 LoRA^P sites "
                    "(4 fused groups), 512 LoRA^P r=1 adapters sharded by id, per GPU "
                    f"{args.requests} prefill requests (Punica lengths) + {args.decodes} decode tokens",
        "model": "Llama-3.1-8B projection shapes (GQA k/v 1024), random init",
        "adapters": N_ADAPTERS,
        "rank": RANK,
        "prefill_tokens_per_gpu": sel,
        "tokens_per_gpu": T,
        "entries_per_gpu": E,
        "distinct_adapters_per_gpu": distinct,
        "global_batch": int(tokens_all),
        "seq_len": "ragged (Punica lognormal prompts)",
        "parallelism": f"adapter-sharded replicas x{world} (requests routed to adapter owner, no collective)",
        "l2_policy": "inputs larger than L2: ~0.9 GB of per-layer activations stream between reuses (L2 126 MB)",
    }


SECONDARY = ("cfg1", "cfg3", "cfg5", "cfg5s", "lora16", "serving", "cfg4")


def secondary_lines(args, device, world: int, rank: int, only: set[str]) -> list:
    """Every BASELINE config that is not the headline, each with its parity.
    A failure in one line is recorded in that line, never loses the others."""
    import torch

    from paper_2605_14217_b200.workload import AdapterMix, WorkloadConfig, assign_adapters

    want = (lambda k: k in only) if only else (lambda k: True)
    rng = np.random.default_rng(3)
    ids3 = rng.integers(0, N_ADAPTERS, size=32)
    ids5 = assign_adapters(WorkloadConfig(8, N_ADAPTERS, AdapterMix.SKEWED, seed=5))
    lens5 = rng.integers(8192, 16385, size=8)
    jobs = [
        ("cfg1", world == 1, lambda: lora_reft_mix_config(args, device)),
        ("cfg3", True, lambda: reft_config(args, device, "direft", 16, [2048] * 32, ids3,
                                           "cfg3: 8B shapes, DiReFT^P r16 x 32 layers, 512 adapters, 32 x 2048-token "
                                           "prompts + 64 decode per GPU", world=world, grank=rank)),
        ("cfg5", True, lambda: reft_config(args, device, "loreft", 32, lens5, ids5,
                                           "cfg5: Zipf over 512 adapters, 8 prompts U[8k,16k] per GPU, LoReFT^P r32 "
                                           "x 32 layers", world=world, grank=rank)),
        ("cfg5s", True, lambda: cfg5_strong(args, device, world, rank)),
        ("lora16", world == 1, lambda: lora_rank_config(args, device, 16)),
        ("serving", world == 1, lambda: serving_replay(args, device)),
        ("cfg4", world in (1, 8), lambda: tp_config(args, device, world, rank)),
    ]
    out = []
    for key, ok, fn in jobs:
        if not (ok and want(key)):
            continue
        try:
            line = fn()
        except Exception as exc:  # never lose the headline line to a secondary config
            line = {"workload": key, "error": f"{type(exc).__name__}: {exc}"[:300]}
            torch.cuda.empty_cache()
        if line is not None:
            line["key"] = key
            out.append(line)
    return out


SHARED_NOTE = ("every rank on ONE GPU (--share-gpu): a functional run of the multi-rank path (launcher, "
               "adapter sharding, request routing, per-rank kernels, max-over-ranks timing); the ranks time-share "
               "the GPU, so the values are not scaling measurements")


def run_ours(args):
    import torch

    world, rank, local = dist_setup(args)
    if args.share_gpu and world > 1:
        local = 0
        torch.cuda.set_device(0)
        dist_init(world, local, backend="gloo")
    else:
        dist_init(world, local)
    device = torch.device("cuda", local)
    only = {k for k in args.only.split(",") if k}
    if only:
        others = []
        if "punica" in only and world == 1:
            others.append(punica_step(args, rank, world, device))
        others += secondary_lines(args, device, world, rank, only)
        if rank == 0:
            line = {"metric": METRIC, "only": sorted(only), "n_gpus": world, "other_configs": others}
            if args.share_gpu and world > 1:
                line["shared_gpu"] = SHARED_NOTE
            print(json.dumps(line))
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    ctx = build_step(args, rank, world, device, args.requests, args.decodes)
    clocks = ClockSampler(local)
    clocks.start()
    ms_total, kernel = time_steps(ctx, args, world, device, timing_tag=1)
    clk = clocks.stop()
    ms_max = all_max(ms_total, world)
    tokens_all = all_sum(ctx["sel"], world)
    value = tokens_all * args.steps / (ms_max / 1e3)
    peak, peak_src = measured_peak_gbs()
    shape = ctx["shape"]
    from paper_2605_14217_b200 import shapes

    gu = ("Wgate", "Wup")
    gu_bytes = group_bytes(shape, gu, ctx["sel"], ctx["distinct"])
    k_ms, k_count = kernel
    k_avg_s = (k_ms / max(k_count, 1)) / 1e3
    achieved = gu_bytes / k_avg_s / 1e9
    traffic, traffic_src = ncu_traffic("lora_gate_up")
    step_bytes = N_LAYERS * sum(group_bytes(shape, gp, ctx["sel"], ctx["distinct"]) for gp in shapes.SITE_GROUPS)
    step_s = ms_total / args.steps / 1e3
    gpu_launches = ctx["plan"].launches_per_run * args.steps
    parity = None
    if not args.no_parity:
        parity = parity_lora_plan(ctx, lambda: ctx["plan"].run(), seed=rank)
        if world > 1:
            parity["ranks_passed"] = int(all_sum(1.0 if parity["status"] == "pass" else 0.0, world))

    e2e = None
    if not args.no_e2e:
        e_ms, bi, bo, n, e_par = run_e2e(ctx, args, world, device)
        e_ms = all_max(e_ms, world)
        e2e = {"value": round(tokens_all / (e_ms / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": int(bi),
               "d2h_bytes_per_step": int(bo), "ms_per_step": round(e_ms, 3), "steps": n,
               "path": "pinned host x/y of every layer -> device -> fused kernels -> host, copy streams overlapped",
               "parity": e_par}
    punica = None
    if not args.no_punica_step and world == 1:
        punica = punica_step(args, rank, world, device)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(ctx, args.cpu_seconds)
    others = None
    if not args.no_secondary:
        del ctx["plan"], ctx["acts"]
        torch.cuda.empty_cache()
        others = secondary_lines(args, device, world, rank, set())
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 1),
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_max / args.steps, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random adapters N(0,0.01^2), random bf16 activations, Punica prompt lengths)",
            "config": cfg2_config(args, world, ctx["sel"], ctx["T"], ctx["E"], ctx["distinct"], tokens_all),
            "parity": parity,
            "roofline": {
                "bound": "hbm",
                "kernel": "lora_team_kernel<bf16,R=1,NS=2,U=4,TEAM=1> (K2, gate/up fused group)",
                "achieved": round(achieved, 1),
                "peak": peak,
                "peak_source": peak_src,
                "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "traffic": traffic,
                "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": gu_bytes,
                "avg_launch_us": round(k_avg_s * 1e6, 2),
                "launches_timed": k_count,
                "step_frac": round(step_bytes / step_s / 1e9 / peak, 4),
                "step_algorithmic_bytes": step_bytes,
            },
            "clocks": clk,
            "gpu_launches": gpu_launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "punica_step": punica,
            "other_configs": others,
        }
        if args.share_gpu and world > 1:
            line["shared_gpu"] = SHARED_NOTE
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# ---------------------------------------------------------------- reference arm


def run_reference(args):
    """The reference's own CPU implementation of this path (prefillsim,
    unmodified, from oracle/_ref; else the pinned oracle port) on every host
    core, over the SAME cfg2 batch as the GPU arm: each step is the whole
    batch through all 32 layers x 7 LoRA^P sites."""
    world, rank, local = dist_setup(args)
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    from oracle import cpu_reference as CR

    qsl, ids, flags, lens, owned = step_entries(0, 1, args.requests, args.decodes)
    cores = args.ref_cores or len(os.sched_getaffinity(0))
    steps, warmup = max(1, args.steps), max(1, min(args.warmup, 2))
    res = CR.time_parallel(qsl, ids, flags, cores=cores, steps=steps, warmup=warmup, seed=SEED)
    value = res["tokens_per_s"]
    distinct = len({ids[i] for i in range(len(ids)) if not (flags[i] & 1)})
    T, E, sel = int(qsl[-1]), len(ids), int(lens.sum())
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": round(res["ms_per_step"], 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (random adapters N(0,0.01^2), random activations, Punica prompt lengths), same batch as "
                "the GPU arm",
        "impl": "reference",
        "config": cfg2_config(args, 1, sel, T, E, distinct, sel),
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores, "kind": res["kind"],
                         "sample": res["sample"]},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------- launcher dry run (CPU, gloo)


def run_dry(args):
    """The multi-rank plumbing without kernels: rank/world from torchrun, a
    gloo process group, each rank's adapter shard and routed cfg2 batch, the
    cfg5 strong-scaling routing with hot replicas, and the max/sum
    collectives; rank 0 prints the line.  tests/test_bench_launcher.py runs
    `bench.py --gpus 2 --dry-run` through the same self-launch code."""
    from paper_2605_14217_b200.workload import (AdapterMix, WorkloadConfig, assign_adapters, hot_replicas,
                                                route_requests)

    world, rank, local = dist_setup(args)
    dist_init(world, local, backend="gloo")
    qsl, ids, flags, lens, owned = step_entries(rank, world, args.requests, args.decodes)
    assert all(a in set(owned) for a in ids), "a request routed to a GPU that does not own its adapter"
    sel = int(lens.sum())
    tok = all_gather_floats(sel, world)
    t0 = time.perf_counter()
    barrier(world)
    ms = all_max((time.perf_counter() - t0) * 1e3, world)
    n_req = 16
    zids = [int(a) for a in assign_adapters(WorkloadConfig(n_req, N_ADAPTERS, AdapterMix.SKEWED, seed=11))]
    zl = np.random.default_rng(12).integers(8192, 16385, size=n_req)
    hot = hot_replicas(zids, world)
    routes = route_requests(zids, world, hot, zl)
    mine = sum(int(zl[i]) for i in routes[rank])
    zt = all_gather_floats(mine, world)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "backend": "gloo",
                          "per_rank_prefill_tokens": [int(v) for v in tok], "global_prefill_tokens": int(sum(tok)),
                          "barrier_ms_max": round(ms, 3),
                          "cfg5_strong": {"hot_replicated_adapters": sorted(hot),
                                          "per_rank_prefill_tokens": [int(v) for v in zt],
                                          "global_prefill_tokens": int(zl.sum())}}))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        run_reference(args)  # rank 0's work only: no need to launch the other ranks
        return
    maybe_self_launch(args)
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
