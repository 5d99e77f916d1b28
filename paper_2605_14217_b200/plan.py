"""StepPlan — one native call per step for the whole hot path.

The reference runs its adapter hooks inside a Python `layer x entry` loop
(model.py:504-546).  A StepPlan records, once, every launch a step needs
(K1 + one fused launch per LoRA site group or ReFT site per layer, all with
fixed pointers into the pool and the activation buffers) in the native
executor (csrc/plan.cu); `run()` then issues the step with a single C call.
The plan is CUDA-graph capturable (`capture()`), which removes the host from
the loop entirely for small, launch-bound batches.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import torch

from . import _lib
from .errors import ShapeError
from .meta import BatchMeta
from .ops import check_lora_group, check_reft, lora_site_array, lora_site_chunks, row_stride, wants_lora_part
from .pool import AdapterPool

__all__ = ["StepPlan"]


class StepPlan:
    def __init__(self, meta: BatchMeta, pool: AdapterPool, max_tokens: int | None = None,
                 rows_hint: int | None = None):
        """`rows_hint`: the expected selected-row count per step, which picks
        the K2 team size baked into the launches (and into a captured graph);
        default: the meta's last build, else `max_tokens`.  Never affects results."""
        self.lib = _lib.load()
        self.meta = meta
        self.pool = pool
        self.rows = max_tokens if max_tokens is not None else meta.T_cap
        meta.set_slot_split(pool.slot_split)
        self.handle = self.lib.preft_plan_create(ctypes.byref(meta.c))
        if not self.handle:
            raise ShapeError("could not create a step plan")
        self.lib.preft_plan_set_slot_split(self.handle, pool.slot_split)
        self.rows_hint = 0
        self.set_rows_hint(rows_hint if rows_hint is not None else (meta.c.rows_hint or self.rows))
        self._fixed_hint = rows_hint is not None
        self._keep: list = []  # tensors the plan points into
        self.n_ops = 0
        self.n_launches = 0
        self.graph: torch.cuda.CUDAGraph | None = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.preft_plan_destroy(h)
            self.handle = None

    def set_rows_hint(self, rows: int) -> None:
        self.rows_hint = int(rows)
        _lib.check(self.lib.preft_plan_set_rows_hint(self.handle, self.rows_hint), "plan_set_rows_hint")

    def add_lora_group(self, ys: Sequence[torch.Tensor], x: torch.Tensor, layer: int, sites: Sequence[str],
                       tag: int = -1) -> None:
        """Same contract and checks as ops.apply_lora_group_ (a group too wide
        for one launch becomes several)."""
        pool = self.pool
        m = check_lora_group(ys, x, self.rows, pool, layer, sites)
        if wants_lora_part(pool) and self.meta.lora_part is None:
            self.meta.ensure_lora_part()
            _lib.check(self.lib.preft_plan_refresh_meta(self.handle, ctypes.byref(self.meta.c)), "plan_refresh_meta")
        for lo, hi in lora_site_chunks(sites, pool.lora_rank):
            arr = lora_site_array(ys[lo:hi], pool, layer, sites[lo:hi])
            st = self.lib.preft_plan_add_lora(self.handle, ctypes.c_void_p(x.data_ptr()), row_stride(x), m, arr,
                                              hi - lo, pool.lora_rank, pool.dtype_code, tag)
            _lib.check(st, "plan_add_lora")
            self.n_launches += 1
        self._keep += [x, *ys]
        self.n_ops += 1

    def add_reft(self, h: torch.Tensor, layer: int, tag: int = -1) -> None:
        pool = self.pool
        check_reft(h, self.rows, pool, layer)
        st = self.lib.preft_plan_add_reft(
            self.handle, ctypes.c_void_p(h.data_ptr()), h.shape[0], row_stride(h), pool.d_model,
            ctypes.c_void_p(pool.reft_A[layer].data_ptr()), ctypes.c_void_p(pool.reft_B[layer].data_ptr()),
            ctypes.c_void_p(pool.reft_Bt[layer].data_ptr() if pool.reft_Bt is not None else None),
            ctypes.c_void_p(pool.reft_bias[layer].data_ptr()), ctypes.c_void_p(pool.reft_scale[layer].data_ptr()),
            pool.reft_rank, pool.dtype_code, tag
        )
        _lib.check(st, "plan_add_reft")
        self._keep.append(h)
        self.n_ops += 1
        self.n_launches += 1

    @property
    def launches_per_run(self) -> int:
        """Kernels one run() launches: K1 (2) + one per site launch (the
        co-launched ReFT pair counts once)."""
        return 2 + self.n_launches

    def set_timing(self, tag: int, reserve_pairs: int) -> None:
        _lib.check(self.lib.preft_plan_set_timing(self.handle, tag, reserve_pairs), "plan_set_timing")

    def collect_timing(self) -> tuple[float, int]:
        total = ctypes.c_double(0.0)
        count = ctypes.c_int32(0)
        _lib.check(self.lib.preft_plan_collect_timing(self.handle, ctypes.byref(total), ctypes.byref(count)),
                   "plan_collect_timing")
        return total.value, count.value

    def run(self, stream=None, run_meta: bool = True, _capturing: bool = False) -> None:
        """Issue the step.  run_meta=True re-runs K1 (with the pool's slot
        split) on the entries already staged in the meta; run_meta=False
        trusts the caller's build, which must have used the pool's split."""
        s = stream if stream is not None else torch.cuda.current_stream(self.pool.device)
        if not run_meta and not _capturing:
            self.meta.require_split(self.pool.slot_split)
        if not self._fixed_hint and self.meta.c.rows_hint > 0 and self.meta.c.rows_hint != self.rows_hint:
            self.set_rows_hint(self.meta.c.rows_hint)
        _lib.check(self.lib.preft_plan_run(self.handle, int(run_meta), ctypes.c_void_p(s.cuda_stream)), "plan_run")
        if run_meta:
            self.meta.built_split = int(self.pool.slot_split)

    def capture_steps(self, steps: int, stream=None, timing_tag: int | None = None) -> torch.cuda.CUDAGraph:
        """Capture `steps` consecutive runs (K1 included) into ONE CUDA graph.
        With a timing tag the tagged launches' events are captured as external
        event-record nodes, so collect_timing() after a replay returns that
        replay's per-launch times.  (`bench.py` times its K steps as one replay.)"""
        s = stream if stream is not None else torch.cuda.Stream(self.pool.device)
        s.wait_stream(torch.cuda.current_stream(self.pool.device))
        with torch.cuda.stream(s):
            self.run(s, True, _capturing=True)  # warm-up: occupancy queries, smem attributes
        torch.cuda.current_stream(self.pool.device).wait_stream(s)
        torch.cuda.synchronize(self.pool.device)
        if timing_tag is not None:
            self.set_timing(timing_tag, steps * max(1, self.n_ops) + 8)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(steps):
                self.run(s, True, _capturing=True)
        return g

    def capture(self, stream=None, run_meta: bool = True) -> torch.cuda.CUDAGraph:
        """Capture one run() into a CUDA graph (timing must be off).  With
        run_meta=False the graph holds only the site launches: the caller
        rebuilds the metadata (BatchMeta.build_arrays: H2D + K1) before each
        replay, and the kernels read the new token counts from device memory."""
        s = stream if stream is not None else torch.cuda.Stream(self.pool.device)
        s.wait_stream(torch.cuda.current_stream(self.pool.device))
        # the graph is replayed after later builds (run_meta=False: the caller's
        # build_arrays with slot_split=pool.slot_split before every replay)
        with torch.cuda.stream(s):
            self.run(s, run_meta, _capturing=True)  # warm-up: occupancy queries, smem attributes
        torch.cuda.current_stream(self.pool.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.run(s, run_meta, _capturing=True)
        self.graph = g
        return g
