"""Timing harness for the reference's CPU path — TEST/BENCH INFRASTRUCTURE ONLY.

Used by bench.py for (a) `--impl reference` (all host cores) and (b) the
`cpu_baseline` object of the GPU arm's JSON line (one core, bounded sample).

What is timed is the reference's own hot-path slice exactly as forward_chunk
performs it (model.py:474, 504-546), through the UNMODIFIED reference
installed in oracle/_ref by oracle/build_ref.py:

    mask = compute_position_mask(make_batch(entries))        model.py:271, 305
    for layer in 32 layers, for site in the 7 LoRA targets,
        for entry with selected rows:                         model.py:509, 538
            out = y_site[span];  out[rows] += delta_for_rows(site_params, x[span][rows])
                                                              model.py:449-451

in float64 numpy, IN PLACE on the site outputs (no copy of y, as `_project`
adds into its own output).  The base GEMMs (`x @ W.T`) are the base model,
not the adapter path, and are not timed.  When oracle/_ref is missing (the
reference was never mounted where build() ran) the oracle port
(oracle/preft_oracle.delta_rows, pinned bit-exact to the reference) does the
same loop and the result says kind "port".

Weights: two per-layer parameter sets are cycled through the 32 layers
(all 32 would be 5 GB of float64 for the cfg2 batch; two sets already exceed
every cache level, so the memory behaviour is the same).
"""

from __future__ import annotations

import multiprocessing as mp
import time

import numpy as np

N_LAYERS = 32
D, FFN, KV = 4096, 14336, 1024
SITES = {"Wq": (D, D), "Wk": (KV, D), "Wv": (KV, D), "Wo": (D, D), "Wgate": (FFN, D), "Wup": (FFN, D),
         "Wdown": (D, FFN)}
GROUP_INPUT = {"Wq": "xqkv", "Wk": "xqkv", "Wv": "xqkv", "Wo": "xo", "Wgate": "xgu", "Wup": "xgu", "Wdown": "xd"}
INPUT_WIDTH = {"xqkv": D, "xo": D, "xgu": D, "xd": FFN}
RANK = 1
LAYER_SETS = 2


def reference_modules():
    """(prefillsim.adapters, prefillsim.model, kind) — the installed reference, else the port."""
    from oracle import build_ref

    mods = build_ref.import_reference()
    if mods is not None:
        return mods[0], mods[1], "reference"
    return None, None, "port"


def split_requests(qsl, flags, n_parts: int) -> list[list[int]]:
    """Entry indices per worker: prefill requests dealt round-robin by size
    (largest first) so the parts carry ~equal tokens; decode entries dealt
    the same way."""
    qsl = np.asarray(qsl)
    lens = np.diff(qsl)
    is_dec = (np.asarray(flags) & 1) != 0
    parts: list[list[int]] = [[] for _ in range(n_parts)]
    load = np.zeros(n_parts)
    for i in sorted(range(len(lens)), key=lambda i: (is_dec[i], -lens[i])):
        w = int(np.argmin(load))
        parts[w].append(i)
        load[w] += lens[i]
    return [sorted(p) for p in parts]


class Worker:
    """One process's share of the step: its entries, activations and weights."""

    def __init__(self, qsl, ids, flags, entries: list[int], seed: int):
        self.RA, self.RM, self.kind = reference_modules()
        qsl = np.asarray(qsl)
        lens = [int(qsl[i + 1] - qsl[i]) for i in entries]
        self.qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        self.ids = [ids[i] for i in entries]
        self.dec = [bool(flags[i] & 1) for i in entries]
        self.allp = [bool(flags[i] & 2) for i in entries]
        self.prefill_tokens = int(sum(n for n, d in zip(lens, self.dec) if not d))
        T = int(self.qsl[-1])
        rng = np.random.default_rng(seed)
        self.x = {k: rng.normal(size=(T, w)) for k, w in INPUT_WIDTH.items()}
        self.y = {s: rng.normal(size=(T, n)) for s, (n, m) in SITES.items()}
        used = sorted({int(a) for a in self.ids if a is not None})
        self.params = []
        for _ in range(LAYER_SETS):
            per_site = {}
            for s, (n, m) in SITES.items():
                per_site[s] = {a: self._lora(rng.normal(0, 0.01, size=(RANK, m)), rng.normal(0, 0.01, size=(n, RANK)))
                               for a in used}
            self.params.append(per_site)
        if self.RM is not None:
            P = self.RA.PositionSchedule
            self.entries = [
                self.RM.SeqEntry(k, tuple(range(n)), n if not d else n + 1,
                                 self.RM.Phase.DECODE if d else self.RM.Phase.PREFILL, a,
                                 None if a is None else (P.ALL_POSITIONS if ap else P.PREFILL_ONLY))
                for k, (n, d, a, ap) in enumerate(zip(lens, self.dec, self.ids, self.allp))
            ]

    def _lora(self, A, B):
        if self.RA is None:
            return dict(kind="lora", s=32.0 / RANK, A=A, B=B)
        return self.RA.AdapterParams(self.RA.AdapterKind.LORA, RANK, (B.shape[0], A.shape[1]),
                                     self.RA.ScalingRule.alpha_over_r(32.0), A=A, B=B)

    def mask(self) -> np.ndarray:
        if self.RM is not None:
            return self.RM.compute_position_mask(self.RM.make_batch(self.entries)).values
        from oracle import preft_oracle as O

        ad = np.array([-1 if a is None else a for a in self.ids])
        return O.position_mask(self.qsl, ad, np.array(self.dec), np.array(self.allp))

    def delta(self, p, rows):
        if self.RA is not None:
            return self.RA.delta_for_rows(p, rows)
        from oracle import preft_oracle as O

        return O.delta_rows("lora", p["s"], rows, A=p["A"], B=p["B"])

    def run(self, n_layers: int = N_LAYERS) -> int:
        """One step: the mask, then every layer's 7 LoRA hooks, in place."""
        mask = self.mask()
        spans = [(slice(int(self.qsl[i]), int(self.qsl[i + 1])), self.ids[i]) for i in range(len(self.ids))]
        for layer in range(n_layers):
            p = self.params[layer % LAYER_SETS]
            for s in SITES:
                x, y, ps = self.x[GROUP_INPUT[s]], self.y[s], p[s]
                for sp, a in spans:
                    if a is None:
                        continue
                    rows = mask[sp]
                    if not rows.any():
                        continue
                    out = y[sp]  # a view: the add lands in y, as in _project's own output
                    out[rows] += self.delta(ps[a], x[sp][rows])
        return self.prefill_tokens


def time_sample(qsl, ids, flags, n_requests: int, seconds: float, seed: int = 0) -> dict:
    """One process, one BLAS thread (the caller limits threads): the first
    `n_requests` prefill requests (plus decode entries) through all 32
    layers per iteration, for about `seconds`."""
    is_dec = (np.asarray(flags) & 1) != 0
    pre = [i for i in range(len(ids)) if not is_dec[i]][:n_requests]
    dec = [i for i in range(len(ids)) if is_dec[i]][:n_requests]
    w = Worker(qsl, ids, flags, sorted(dec + pre), seed)
    w.run(1)  # warm-up
    t0 = time.perf_counter()
    iters = 0
    while True:
        w.run()
        iters += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    per = el / iters
    return {
        "tokens_per_s": w.prefill_tokens / per,
        "kind": w.kind,
        "sample": f"{len(pre)} of the step's prefill requests ({w.prefill_tokens} tokens) + {len(dec)} decode entries "
                  f"through all 32 layers x 7 LoRA^P sites per iteration ({iters} iterations, {el:.1f} s), "
                  f"{'prefillsim (oracle/_ref)' if w.kind == 'reference' else 'oracle port'} delta_for_rows, "
                  "f64 numpy, in place",
    }


# ---------------------------------------------------------------- all host cores

_W: Worker | None = None


def _init(qsl, ids, flags, parts, seed, counter):
    global _W
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    with counter.get_lock():
        w = counter.value
        counter.value += 1
    _W = Worker(qsl, ids, flags, parts[w], seed + w)


def _work(_):
    t0 = time.perf_counter()
    n = _W.run()
    return n, time.perf_counter() - t0, _W.kind


def time_parallel(qsl, ids, flags, cores: int, steps: int, warmup: int, seed: int = 0) -> dict:
    """The WHOLE step (every request of the batch, all 32 layers) split over
    one process per core (disjoint entries, one BLAS thread each); a step ends
    when the slowest process finishes.  Returns per-step wall times."""
    parts = split_requests(qsl, flags, cores)
    ctx = mp.get_context("fork")
    counter = ctx.Value("i", 0)
    with ctx.Pool(cores, initializer=_init, initargs=(qsl, ids, flags, parts, seed, counter)) as pool:
        for _ in range(max(1, warmup)):
            pool.map(_work, range(cores), chunksize=1)
        times, toks, kind = [], 0, "port"
        for _ in range(steps):
            t0 = time.perf_counter()
            res = pool.map(_work, range(cores), chunksize=1)
            times.append(time.perf_counter() - t0)
            toks = sum(r[0] for r in res)
            kind = res[0][2]
    total = float(np.sum(times))
    return {
        "tokens_per_s": toks * steps / total,
        "ms_per_step": total / steps * 1e3,
        "prefill_tokens": toks,
        "kind": kind,
        "sample": f"the full step: {toks} prefill tokens over {cores} processes (1 BLAS thread each), all 32 layers "
                  f"x 7 LoRA^P sites per step, {steps} timed steps, "
                  f"{'prefillsim (oracle/_ref) compute_position_mask + delta_for_rows' if kind == 'reference' else 'oracle port'}"
                  ", f64 numpy, in place",
    }
