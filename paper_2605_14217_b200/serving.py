"""Serving-step replay: the reference engine's scheduler driving the device
hot path.

The reference engine (engine.py:335-489) admits requests FCFS up to
`max_batch`, then forms each step's batch: every running decode request
first (one token each), then prefill chunks under the token budget and the
adapter cap (`_form_batch`, engine.py:528-569); an adapter that does not run
in a phase (prefill-only adapters at decode, engine.py:521-526) needs no
device slot.  The functional step lists decode entries first, then prefill
chunks (engine.py:615-648).

`Scheduler` restates that loop exactly (same scheduled ids, chunks, worksets
and LRU page-ins as the reference's `StepRecord`s — checked against the live
reference in tests/test_serving_cpu.py).  `ServingLoop` replays it on the
GPU: per step the worksets are paged into the HBM pool (paging.py), K1 builds
the device metadata from the entries, and every layer's adapter sites run
(LoRA^P groups, ReFT^P residual) — the whole adapter path of a serving step,
without the base model (the caller's GEMMs).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Mapping, Sequence

import numpy as np

from .adapters import PositionSchedule
from .batch import Phase
from .errors import ConfigError, DomainError, StateError

__all__ = ["RequestSpec", "generate_workload", "ServeConfig", "Scheduler", "StepBatch", "ServingLoop"]


@dataclass(frozen=True)
class RequestSpec:
    """workload.py:85-103: prompt length, output length, adapter (None = base)."""

    request_id: int
    prompt_len: int
    output_len: int
    adapter_id: int | None

    def __post_init__(self) -> None:
        if self.prompt_len < 1:
            raise DomainError("prompt_len must be >= 1")
        if self.output_len < 2:
            raise DomainError("output_len must be >= 2")


def generate_workload(cfg) -> list[RequestSpec]:
    """workload.py:148-156 (the sub-streams are restated in workload.py)."""
    from .workload import assign_adapters, sample_prompt_lens, sample_total_lens

    prompts = sample_prompt_lens(cfg)
    totals = sample_total_lens(cfg, prompts)
    adapters = assign_adapters(cfg)
    return [RequestSpec(i, int(p), int(t - p), a) for i, (p, t, a) in enumerate(zip(prompts, totals, adapters))]


@dataclass(frozen=True)
class ServeConfig:
    """The scheduling fields of EngineConfig (engine.py:101-133)."""

    max_batch: int = 32
    max_gpu_adapters: int = 32
    chunk_size: int | None = None
    step_token_budget: int = 2048

    def __post_init__(self) -> None:
        if self.max_batch < 1:
            raise ConfigError("max_batch must be >= 1")
        if self.max_gpu_adapters < 1:
            raise ConfigError("max_gpu_adapters must be >= 1")
        if self.chunk_size is not None and self.chunk_size < 1:
            raise ConfigError("chunk_size must be >= 1")
        if self.step_token_budget < self.max_batch:
            raise ConfigError("step_token_budget must cover one decode token per slot")


class _Request:
    def __init__(self, spec: RequestSpec):
        self.spec = spec
        self.prefill_pos = 0
        self.tokens_out = 0

    @property
    def in_decode(self) -> bool:
        return self.prefill_pos >= self.spec.prompt_len

    @property
    def done(self) -> bool:
        return self.in_decode and self.tokens_out >= self.spec.output_len


@dataclass
class StepBatch:
    """One scheduled step: the entries K1 consumes plus the bookkeeping the
    reference records in StepRecord (engine.py:176-197)."""

    index: int
    decode: list[int]  # request ids, one token each (listed first)
    prefill: list[tuple[int, int]]  # (request id, chunk)
    workset: list[int]  # adapters that execute this step (need a device slot)
    qsl: np.ndarray = field(repr=False, default=None)  # int32 [E+1]
    adapter_ids: list = field(repr=False, default=None)  # per entry, None = base
    decode_flags: np.ndarray = field(repr=False, default=None)  # int32 [E], 1 = decode
    all_positions: np.ndarray = field(repr=False, default=None)  # int32 [E], 1 = ALL_POSITIONS adapter

    def entry_flags(self) -> np.ndarray:
        """K1 flag word per entry (PREFT_ENTRY_*), from the scheduler's own
        schedule map, so the device mask always agrees with the workset."""
        from . import _lib

        f = self.decode_flags.astype(np.int32) * _lib.ENTRY_DECODE
        if self.all_positions is not None:
            f = f | (self.all_positions.astype(np.int32) * _lib.ENTRY_ALL_POSITIONS)
        return f.astype(np.int32)

    @property
    def prefill_tokens(self) -> int:
        return sum(c for _, c in self.prefill)

    @property
    def tokens(self) -> int:
        return len(self.decode) + self.prefill_tokens


class Scheduler:
    """engine.py:397-489 without the model: FCFS admission, decode-first batch
    formation under the token budget and the adapter cap."""

    def __init__(self, workload: Sequence[RequestSpec], cfg: ServeConfig,
                 schedule_of: Callable[[int], PositionSchedule] | PositionSchedule = PositionSchedule.PREFILL_ONLY):
        self.cfg = cfg
        self._schedule_of = schedule_of if callable(schedule_of) else (lambda _aid, s=schedule_of: s)
        self.queue = [_Request(s) for s in workload]
        self.running: list[_Request] = []
        self.step_idx = 0

    def _executes(self, req: _Request, phase: Phase) -> bool:
        """engine.py:521-526"""
        if req.spec.adapter_id is None:
            return False
        if phase is Phase.DECODE and self._schedule_of(req.spec.adapter_id) is PositionSchedule.PREFILL_ONLY:
            return False
        return True

    def _form_batch(self):
        """engine.py:528-569"""
        cfg = self.cfg
        budget = cfg.step_token_budget
        workset: list[int] = []
        decode_sched: list[_Request] = []
        prefill_sched: list[tuple[_Request, int]] = []

        def fits(req: _Request, phase: Phase) -> bool:
            if not self._executes(req, phase):
                return True
            aid = req.spec.adapter_id
            if aid in workset:
                return True
            if len(workset) < cfg.max_gpu_adapters:
                workset.append(aid)
                return True
            return False

        for req in self.running:
            if req.in_decode and not req.done:
                if budget < 1:
                    break
                if fits(req, Phase.DECODE):
                    decode_sched.append(req)
                    budget -= 1
        for req in self.running:
            if req.in_decode:
                continue
            if budget < 1:
                break
            chunk = req.spec.prompt_len - req.prefill_pos
            if cfg.chunk_size is not None:
                chunk = min(chunk, cfg.chunk_size)
            chunk = min(chunk, budget)
            if chunk < 1:
                continue
            if fits(req, Phase.PREFILL):
                prefill_sched.append((req, chunk))
                budget -= chunk
        return decode_sched, prefill_sched, workset

    def __iter__(self):
        return self

    def __next__(self) -> StepBatch:
        if not (self.queue or self.running):
            raise StopIteration
        while self.queue and len(self.running) < self.cfg.max_batch:  # engine.py:399-406
            self.running.append(self.queue.pop(0))
        decode_sched, prefill_sched, workset = self._form_batch()
        if not decode_sched and not prefill_sched:
            raise StateError("no request could be scheduled; engine is stuck")
        # entries as _step_functional lists them (engine.py:618-648)
        lens = [1] * len(decode_sched) + [c for _, c in prefill_sched]
        qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        ids = [r.spec.adapter_id for r in decode_sched] + [r.spec.adapter_id for r, _ in prefill_sched]
        dec = np.array([1] * len(decode_sched) + [0] * len(prefill_sched), dtype=np.int32)
        allp = np.array([a is not None and self._schedule_of(a) is PositionSchedule.ALL_POSITIONS for a in ids],
                        dtype=np.int32)
        step = StepBatch(self.step_idx, [r.spec.request_id for r in decode_sched],
                         [(r.spec.request_id, c) for r, c in prefill_sched], list(workset), qsl, ids, dec, allp)
        # progress (engine.py:436-465)
        for req, chunk in prefill_sched:
            req.prefill_pos += chunk
        for req in decode_sched:
            req.tokens_out += 1
        self.running = [r for r in self.running if not r.done]
        self.step_idx += 1
        return step


class ServingLoop:
    """Replays a Scheduler on the device: paging + K1 + every layer's adapter
    sites per step, on one stream, timed with CUDA events."""

    def __init__(self, paged, meta, layer_ops: Callable[[object, int], None], n_layers: int):
        """Entry flags come from each StepBatch (the Scheduler's schedule map),
        so the loop cannot disagree with the scheduler about which decode
        tokens an ALL_POSITIONS adapter covers (model.py:316)."""
        self.paged = paged  # paging.PagedAdapterPool
        self.meta = meta  # meta.BatchMeta sized for the step token budget
        self.layer_ops = layer_ops  # (stream, layer) -> launches every adapter site of one layer
        self.n_layers = n_layers

    def run(self, scheduler: Scheduler, max_steps: int | None = None, stream=None) -> dict:
        import torch

        from . import _lib

        pool = self.paged.pool
        s = stream if stream is not None else torch.cuda.current_stream(pool.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = tokens = prefill = 0
        e0.record(s)
        for step in scheduler:
            self.paged.ensure(step.workset, stream=s)
            if not step.workset:
                # nothing executes (forward_chunk's skip_adapters, model.py:475)
                steps += 1
                tokens += step.tokens
                if max_steps is not None and steps >= max_steps:
                    break
                continue
            flags = step.entry_flags()  # the scheduler's schedules: mask == workset by construction
            slots = pool.entry_arrays(step.qsl, step.adapter_ids, flags)
            self.meta.build_arrays(step.qsl, slots, flags, stream=s, slot_split=pool.slot_split)
            for layer in range(self.n_layers):
                self.layer_ops(s, layer)
            steps += 1
            tokens += step.tokens
            prefill += step.prefill_tokens
            if max_steps is not None and steps >= max_steps:
                break
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        return {"steps": steps, "tokens": tokens, "prefill_tokens": prefill, "ms": ms,
                "page_ins": self.paged.page_ins, "evictions": self.paged.evictions,
                "paged_bytes": self.paged.paged_bytes}
