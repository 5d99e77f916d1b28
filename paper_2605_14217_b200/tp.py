"""Tensor-parallel LoRA^P (BASELINE config 4: Llama-3.1-70B shapes, 8-way TP,
512 LoRA^P r=16 adapters, rank-r shrink partials combined by an NCCL
all-reduce over NVLink).

The reference has no parallelism; its LoRA hook is
`out[rows] += s * ((X A^T) B^T)` (model.py:449-451, adapters.py:284-288).
Under Megatron/vLLM-style tensor parallelism the base projections are split
two ways, and the adapter follows the same split so that every rank holds only
1/tp of the pool (212 GB of 70B r=16 adapters -> 26.5 GB per GPU):

  column-parallel sites (Wq, Wk, Wv, Wgate, Wup): x is replicated [T, m],
      y is this rank's output slice [T, n/tp];
  row-parallel sites (Wo, Wdown): x is this rank's input slice [T, m/tp],
      y is the full-width partial output [T, n] that the base model
      all-reduces afterwards.

Every site stores A sharded along the input dimension m and B along the
output dimension n.  Per group of sites sharing x:

  1. shrink  (K2a, csrc/lora_split.cu): P = x[:, m-slice] . A_shard^T  (T x r per site, f32)
  2. NCCL all-reduce(sum) of P over the TP group: the full X A^T on every rank
  3. expand  (K2b): y[:, n-slice] += s * P . B_shard^T

For row-parallel sites each rank adds only its n-slice of the delta into the
partial output, so the base model's own all-reduce delivers the full delta
exactly once.  The all-reduce moves T x nsites x r x 4 bytes (2,048 tokens x
3 sites x 16 x 4 = 384 KiB for q/k/v), independent of the model width.

The sharding arithmetic here is pure Python (tests/test_tp_cpu.py checks it
with gloo at world size 2 against the unsharded oracle); the device work is
`apply_lora_group_tp_`.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

from .errors import ConfigError, ShapeError

__all__ = [
    "TP_STYLE",
    "SiteShard",
    "shard_range",
    "site_shard",
    "SplitWorkspace",
    "lora_shrink_tp_",
    "lora_expand_tp_",
    "apply_lora_group_tp_",
]

# Llama projections: which side of the base GEMM is split across the TP group
TP_STYLE = {
    "Wq": "column",
    "Wk": "column",
    "Wv": "column",
    "Wgate": "column",
    "Wup": "column",
    "Wo": "row",
    "Wdown": "row",
}


def shard_range(width: int, tp_rank: int, tp_size: int) -> tuple[int, int]:
    """(first, count) of this rank's contiguous slice of `width` columns."""
    if tp_size < 1 or not 0 <= tp_rank < tp_size:
        raise ConfigError(f"tp_rank {tp_rank} out of range for tp_size {tp_size}")
    if width % tp_size:
        raise ShapeError(f"width {width} is not divisible by tp_size {tp_size}")
    n = width // tp_size
    return tp_rank * n, n


@dataclass(frozen=True)
class SiteShard:
    """One rank's slice of a LoRA site of full shape (n, m) (AdapterParams dims)."""

    name: str
    n: int  # full output width
    m: int  # full input width
    n0: int
    n_loc: int
    m0: int
    m_loc: int
    style: str  # "column" | "row"

    @property
    def x_offset(self) -> int:
        """Column of x where this rank's shrink input starts (x is full for
        column-parallel sites, already the rank's slice for row-parallel)."""
        return self.m0 if self.style == "column" else 0

    @property
    def x_width(self) -> int:
        return self.m if self.style == "column" else self.m_loc

    @property
    def y_offset(self) -> int:
        """Column of y where this rank's delta goes (y is the rank's output
        slice for column-parallel sites, the full partial output for row)."""
        return 0 if self.style == "column" else self.n0

    @property
    def y_width(self) -> int:
        return self.n_loc if self.style == "column" else self.n


def site_shard(name: str, n: int, m: int, tp_rank: int = 0, tp_size: int = 1) -> SiteShard:
    style = TP_STYLE.get(name)
    if style is None:
        raise ShapeError(f"unknown LoRA target {name}")
    m0, m_loc = shard_range(m, tp_rank, tp_size)
    n0, n_loc = shard_range(n, tp_rank, tp_size)
    return SiteShard(name, n, m, n0, n_loc, m0, m_loc, style)


class SplitWorkspace:
    """Per-(meta, pool) f32 buffer for the rank-r partials P [T_cap][3 * r]."""

    def __init__(self, meta, pool):
        import torch

        self.T_cap = meta.T_cap
        self.P = torch.empty(meta.T_cap * 3 * pool.lora_rank, dtype=pool.acc, device=pool.device)
        # the tensor-core shrink's partial planes and arrival counters
        meta.ensure_lora_part()

    def view(self, T: int, width: int):
        """Contiguous [T][width] view (the all-reduce moves exactly these bytes)."""
        return self.P[: T * width].view(T, width)


def _site_array(ys, x, meta, pool, layer, sites):
    from . import _lib
    from .ops import _check_act, row_stride

    if not 1 <= len(sites) <= 3 or len(ys) != len(sites):
        raise ShapeError("a LoRA group has 1 to 3 sites and one output per site")
    if not 0 <= layer < pool.n_layers:
        raise ShapeError(f"layer {layer} out of range")
    shards = [pool.lora_shard[s] for s in sites]
    if len({(sh.style, sh.x_offset, sh.x_width, sh.m_loc) for sh in shards}) != 1:
        raise ShapeError(f"sites {tuple(sites)} do not share an input slice")
    _check_act(x, "x", shards[0].x_width, meta.T, pool.dtype, pool.device)
    arr = (_lib.PreftLoraSite * 3)()
    esz = x.element_size()
    for i, (name, y, sh) in enumerate(zip(sites, ys, shards)):
        _check_act(y, f"y[{name}]", sh.y_width, meta.T, pool.dtype, pool.device)
        arr[i].A = pool.lora_A[name][layer].data_ptr()
        arr[i].Bt = pool.lora_Bt[name][layer].data_ptr()
        arr[i].scale = pool.lora_scale[name][layer].data_ptr()
        arr[i].bias = None
        arr[i].y = y.data_ptr() + sh.y_offset * esz
        arr[i].ldy = row_stride(y)
        arr[i].n = sh.n_loc
        tc = pool.lora_Bt_tc.get(name)
        arr[i].Bt_tc = tc[layer].data_ptr() if tc is not None else None
    rows = min(int(x.shape[0]), *(int(y.shape[0]) for y in ys))
    return arr, shards, rows


def lora_shrink_tp_(ys, x, meta, pool, layer: int, sites: Sequence[str], workspace: SplitWorkspace, stream=None):
    """Step 1: this rank's partial P = x[:, m-slice] . A_shard^T; returns the
    contiguous [T][nsites * r] view of the workspace that holds it."""
    import torch

    from . import _lib
    from .ops import row_stride

    arr, shards, rows = _site_array(ys, x, meta, pool, layer, sites)
    if workspace.T_cap < rows:
        raise ShapeError("split workspace too small for this batch")
    ldp = len(sites) * pool.lora_rank
    P = workspace.view(rows, ldp)
    s = stream if stream is not None else torch.cuda.current_stream(pool.device)
    meta.require_split(pool.slot_split)
    st = _lib.load().preft_lora_shrink(
        ctypes.byref(meta.c), ctypes.c_void_p(x.data_ptr() + shards[0].x_offset * x.element_size()), rows,
        row_stride(x), shards[0].m_loc, arr, len(sites), pool.lora_rank, pool.dtype_code,
        ctypes.c_void_p(P.data_ptr()), ldp, ctypes.c_void_p(s.cuda_stream),
    )
    _lib.check(st, "lora_shrink")
    return P


def lora_expand_tp_(P, ys, x, meta, pool, layer: int, sites: Sequence[str], stream=None):
    """Step 3: y[:, n-slice] += s * P . B_shard^T with the all-reduced P."""
    import torch

    from . import _lib

    arr, _, rows = _site_array(ys, x, meta, pool, layer, sites)
    s = stream if stream is not None else torch.cuda.current_stream(pool.device)
    meta.require_split(pool.slot_split)
    st = _lib.load().preft_lora_expand(
        ctypes.byref(meta.c), ctypes.c_void_p(P.data_ptr()), P.shape[1], rows, arr, len(sites), pool.lora_rank,
        pool.dtype_code, ctypes.c_void_p(s.cuda_stream),
    )
    _lib.check(st, "lora_expand")
    return ys


def apply_lora_group_tp_(
    ys: Sequence,
    x,
    meta,
    pool,
    layer: int,
    sites: Sequence[str],
    group=None,
    workspace: SplitWorkspace | None = None,
    stream=None,
    collective: bool = True,
):
    """Tensor-parallel y_s[rows] += s_a (x[rows] A_s,a^T) B_s,a^T for 1-3 sites
    sharing x, on this rank's shard of the pool (`pool.tp_rank` of
    `pool.tp_size`): shrink, NCCL all-reduce of the rank-r partials on the
    same stream, expand.  `x` and `ys` follow the site's TP style (see the
    module docstring); `group` is the torch.distributed process group of the
    TP ranks (None = default group; no collective when tp_size == 1).
    collective=False skips the all-reduce (single-GPU emulation of one rank's
    share of the work; the result is then this rank's partial only)."""
    import torch

    ws = workspace if workspace is not None else SplitWorkspace(meta, pool)
    s = stream if stream is not None else torch.cuda.current_stream(pool.device)
    per = max(1, 64 // pool.lora_rank)  # a launch carries <= 64 rank-r columns of P
    if len(sites) > per:
        for i in range(0, len(sites), per):
            apply_lora_group_tp_(ys[i : i + per], x, meta, pool, layer, sites[i : i + per], group, ws, s, collective)
        return ys
    P = lora_shrink_tp_(ys, x, meta, pool, layer, sites, ws, s)
    if pool.tp_size > 1 and collective:
        import torch.distributed as dist

        with torch.cuda.stream(s):
            dist.all_reduce(P[: meta.T], op=dist.ReduceOp.SUM, group=group)
    return lora_expand_tp_(P, ys, x, meta, pool, layer, sites, s)
