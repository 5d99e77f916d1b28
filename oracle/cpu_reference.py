"""Timing harness for the CPU reference path — TEST/BENCH INFRASTRUCTURE ONLY.

Used by bench.py for (a) the `cpu_baseline` object of the GPU arm's JSON line
(one core) and (b) `bench.py --impl reference` (all host cores).  What is
timed is the reference's hot-path slice exactly as forward_chunk performs it
(model.py:474, 504-546): compute_position_mask over the step's entries, then
per site and per entry with selected rows `out[rows] += delta_for_rows(site,
x[rows])` in float64 numpy — via oracle/preft_oracle.py, the restatement
pinned to the reference by tests/test_oracle_golden.py.  (The reference
itself is pure Python and is not installed on the GPU box.)

The sample is bounded: a few requests through the 7 LoRA sites of one layer
per step (Llama-3.1-8B shapes), reported as tokens/s through all 32 layers,
i.e. sample tokens / (time per layer x 32).
"""

from __future__ import annotations

import multiprocessing as mp
import time

import numpy as np

from oracle import preft_oracle as O

N_LAYERS = 32
D, FFN, KV = 4096, 14336, 1024
SITES = {"Wq": (D, D), "Wk": (KV, D), "Wv": (KV, D), "Wo": (D, D), "Wgate": (FFN, D), "Wup": (FFN, D),
         "Wdown": (D, FFN)}
GROUP_INPUT = {"Wq": "xqkv", "Wk": "xqkv", "Wv": "xqkv", "Wo": "xo", "Wgate": "xgu", "Wup": "xgu", "Wdown": "xd"}
INPUT_WIDTH = {"xqkv": D, "xo": D, "xgu": D, "xd": FFN}
RANK = 1
LAYERS_RESIDENT = 2  # distinct per-layer parameter sets cycled through (weights differ per layer)


def _sub_batch(qsl, ids, flags, req_index):
    """Entries [all decode entries of the batch head] + the chosen prefill requests."""
    is_dec = (np.asarray(flags) & 1) != 0
    dec_entries = [i for i in range(len(ids)) if is_dec[i]]
    pre_entries = [i for i in range(len(ids)) if not is_dec[i]]
    chosen = [pre_entries[j % len(pre_entries)] for j in req_index]
    keep = dec_entries[: max(1, len(chosen))] + chosen
    lens = [int(qsl[i + 1] - qsl[i]) for i in keep]
    sq = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    sids = np.array([ids[i] if ids[i] is not None else -1 for i in keep], dtype=np.int64)
    sdec = np.array([is_dec[i] for i in keep], dtype=bool)
    sall = np.array([bool(flags[i] & 2) for i in keep], dtype=bool)
    return sq, sids, sdec, sall, int(sum(lens[len(keep) - len(chosen):]))


class Sample:
    """One worker's data: f64 activations and adapter params for its requests."""

    def __init__(self, qsl, ids, flags, req_index, seed):
        self.qsl, self.ids, self.dec, self.allp, self.prefill_tokens = _sub_batch(qsl, ids, flags, req_index)
        T = int(self.qsl[-1])
        rng = np.random.default_rng(seed)
        self.x = {k: rng.normal(size=(T, w)) for k, w in INPUT_WIDTH.items()}
        self.y = {s: rng.normal(size=(T, n)) for s, (n, m) in SITES.items()}
        used = sorted({int(a) for a in self.ids if a >= 0})
        self.params = []
        for layer in range(LAYERS_RESIDENT):
            per_site = {}
            for s, (n, m) in SITES.items():
                per_site[s] = {
                    a: dict(kind="lora", s=32.0 / RANK, A=rng.normal(0, 0.01, size=(RANK, m)),
                            B=rng.normal(0, 0.01, size=(n, RANK)))
                    for a in used
                }
            self.params.append(per_site)
        self.step = 0

    def run_layer(self) -> int:
        """compute_position_mask + the 7 LoRA hooks of one layer; returns prefill tokens."""
        mask = O.position_mask(self.qsl, self.ids, self.dec, self.allp)
        p = self.params[self.step % LAYERS_RESIDENT]
        self.step += 1
        for s in SITES:
            self.y[s] = O.lora_hook(self.y[s], self.x[GROUP_INPUT[s]], self.qsl, mask, self.ids, p[s])
        return self.prefill_tokens


def time_sample(qsl, ids, flags, n_requests: int, seconds: float, seed: int = 0) -> dict:
    """Single-process timing for the GPU arm's cpu_baseline (caller limits BLAS threads)."""
    smp = Sample(qsl, ids, flags, list(range(n_requests)), seed)
    smp.run_layer()  # warm-up
    t0 = time.perf_counter()
    toks = 0
    layers = 0
    while True:
        toks += smp.run_layer()
        layers += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    per_layer = el / layers
    return {
        "tokens_per_s": smp.prefill_tokens / (per_layer * N_LAYERS),
        "sample": f"{n_requests} Punica prefill requests ({smp.prefill_tokens} tokens) + decode entries, "
                  f"7 LoRA sites of 1 layer per iteration ({layers} iterations, {el:.1f} s), f64 numpy, scaled x32 layers",
    }


# ---------------------------------------------------------------- multi-process (all host cores)

_W: Sample | None = None
_LIM = None


def _init(qsl, ids, flags, per_worker, seed, counter):
    global _W, _LIM
    from threadpoolctl import threadpool_limits

    _LIM = threadpool_limits(1)
    with counter.get_lock():
        w = counter.value
        counter.value += 1
    _W = Sample(qsl, ids, flags, list(range(w * per_worker, (w + 1) * per_worker)), seed + w)


def _work(_):
    t0 = time.perf_counter()
    n = _W.run_layer()
    return n, time.perf_counter() - t0


def time_parallel(qsl, ids, flags, cores: int, per_worker_requests: int, steps: int, warmup: int, seed: int = 0):
    """All-core reference: one process per core over disjoint request sets."""
    ctx = mp.get_context("fork")
    counter = ctx.Value("i", 0)
    with ctx.Pool(cores, initializer=_init, initargs=(qsl, ids, flags, per_worker_requests, seed, counter)) as pool:
        for _ in range(max(1, warmup)):
            pool.map(_work, range(cores), chunksize=1)
        times, toks = [], 0
        for _ in range(steps):
            t0 = time.perf_counter()
            res = pool.map(_work, range(cores), chunksize=1)
            times.append(time.perf_counter() - t0)
            toks = sum(r[0] for r in res)
    per_layer = float(np.median(times))
    return {
        "tokens_per_s": toks / (per_layer * N_LAYERS),
        "ms_per_step": per_layer * N_LAYERS * 1e3,
        "sample": f"{cores} processes x {per_worker_requests} Punica prefill requests ({toks} tokens/step), "
                  f"7 LoRA sites of 1 layer per step, median of {steps} steps, f64 numpy 1 BLAS thread/process, "
                  "scaled x32 layers",
    }
