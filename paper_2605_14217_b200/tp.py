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
    "FusedExchange",
    "lora_fused_tp_",
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


class FusedExchange:
    """The exchange regions of the fused kernel (preft_lora_fused: shrink ->
    partials to every rank -> expand, one launch per group; see
    include/preft.h preft_xchg_t and csrc/lora_fused.cu).

    * `FusedExchange.local(meta, pool)`: one rank on one device — the
      single-GPU path, or one rank's share of a TP group with the exchange
      omitted (the 1-GPU config-4 measurement);
    * `FusedExchange.group(meta, pool, group)`: the real TP group — every
      rank allocates its region (cudaMalloc, zeroed), the 64-byte IPC handles
      are all-gathered over torch.distributed and every peer's region is
      mapped, so the kernel stores its partial rows straight into the peers'
      HBM over NVLink (no NCCL call on the data path);
    * `FusedExchange.emulated(meta, pool, tp)`: tp ranks' regions on ONE
      device (tests: the ranks run as concurrent launches on separate
      streams with a small grid).

    Every rank must issue the same sequence of fused launches on its
    exchange (the launch count is the flags' tag)."""

    def __init__(self, xg, keep, owned=(), opened=()):
        self.c = xg
        self._keep = keep
        self._owned = list(owned)
        self._opened = list(opened)

    @staticmethod
    def _make(meta, bases, tp, rank, planes, peer_sys, grid):
        from . import _lib

        xg = _lib.PreftXchg()
        arr = (ctypes.c_void_p * tp)(*bases)
        _lib.check(_lib.load().preft_xchg_init(ctypes.byref(xg), arr, tp, rank, planes, meta.T_cap, meta.chunk_cap,
                                               1 if peer_sys else 0), "xchg_init")
        xg.grid = grid
        return xg

    @classmethod
    def region_bytes(cls, meta, tp: int, planes: int) -> int:
        from . import _lib

        return int(_lib.load().preft_xchg_region_bytes(tp, planes, meta.T_cap, meta.chunk_cap))

    @classmethod
    def local(cls, meta, pool, planes: int = 1, grid: int = 0):
        import torch

        n = (cls.region_bytes(meta, 1, planes) + 15) // 16 * 4
        buf = torch.zeros(n, dtype=torch.float32, device=pool.device)
        return cls(cls._make(meta, [buf.data_ptr()], 1, 0, planes, False, grid), [buf])

    @classmethod
    def emulated(cls, meta, pool, tp: int, planes: int = 1, grid: int = 0):
        """tp exchanges sharing regions on one device (rank r's view is item r)."""
        import torch

        n = (cls.region_bytes(meta, tp, planes) + 15) // 16 * 4
        bufs = [torch.zeros(n, dtype=torch.float32, device=pool.device) for _ in range(tp)]
        bases = [b.data_ptr() for b in bufs]
        return [cls(cls._make(meta, bases, tp, r, planes, False, grid), bufs) for r in range(tp)]

    @classmethod
    def group(cls, meta, pool, group=None, planes: int = 1, grid: int = 0):
        import torch.distributed as dist

        from . import _lib

        lib = _lib.load()
        tp, rank = pool.tp_size, pool.tp_rank
        if dist.get_world_size(group) != tp or dist.get_rank(group) != rank:
            raise ConfigError("the process group does not match the pool's tensor-parallel layout")
        nbytes = cls.region_bytes(meta, tp, planes)
        mine = ctypes.c_void_p()
        _lib.check(lib.preft_dev_alloc(nbytes, ctypes.byref(mine)), "dev_alloc")
        handle = ctypes.create_string_buffer(64)
        _lib.check(lib.preft_ipc_handle(mine, handle), "ipc_handle")
        handles = [None] * tp
        dist.all_gather_object(handles, bytes(handle.raw), group=group)  # also: every region is zeroed by now
        bases, opened = [], []
        for r, h in enumerate(handles):
            if r == rank:
                bases.append(mine.value)
                continue
            p = ctypes.c_void_p()
            _lib.check(lib.preft_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)), "ipc_open")
            bases.append(p.value)
            opened.append(p.value)
        return cls(cls._make(meta, bases, tp, rank, planes, True, grid), [], owned=[mine.value], opened=opened)

    def errors(self, stream=None) -> int:
        """state[2] of this rank's region (bit 0: a wait timed out); syncs the stream."""
        import torch

        from . import _lib

        s = stream if stream is not None else torch.cuda.current_stream()
        out = ctypes.c_int32()
        _lib.check(_lib.load().preft_xchg_errors(ctypes.byref(self.c), ctypes.c_void_p(s.cuda_stream),
                                                 ctypes.byref(out)), "xchg_errors")
        return int(out.value)

    def close(self) -> None:
        from . import _lib

        lib = _lib.load()
        for p in self._opened:
            lib.preft_ipc_close(ctypes.c_void_p(p))
        for p in self._owned:
            lib.preft_dev_free(ctypes.c_void_p(p))
        self._opened, self._owned, self._keep = [], [], []


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


def lora_fused_tp_(ys, x, meta, pool, layer: int, sites: Sequence[str], exchange: FusedExchange, stream=None):
    """Shrink -> exchange -> expand in one launch (preft_lora_fused): y[:, n-slice]
    += s * (sum over the exchange's ranks of x[:, m-slice] A_shard^T) B_shard^T."""
    import torch

    from . import _lib
    from .ops import row_stride

    arr, shards, rows = _site_array(ys, x, meta, pool, layer, sites)
    s = stream if stream is not None else torch.cuda.current_stream(pool.device)
    meta.require_split(pool.slot_split)
    st = _lib.load().preft_lora_fused(
        ctypes.byref(meta.c), ctypes.c_void_p(x.data_ptr() + shards[0].x_offset * x.element_size()), rows,
        row_stride(x), shards[0].m_loc, arr, len(sites), pool.lora_rank, pool.dtype_code,
        ctypes.byref(exchange.c), ctypes.c_void_p(s.cuda_stream),
    )
    _lib.check(st, "lora_fused")
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
    exchange: FusedExchange | None = None,
):
    """Tensor-parallel y_s[rows] += s_a (x[rows] A_s,a^T) B_s,a^T for 1-3 sites
    sharing x, on this rank's shard of the pool (`pool.tp_rank` of
    `pool.tp_size`): shrink, NCCL all-reduce of the rank-r partials on the
    same stream, expand.  `x` and `ys` follow the site's TP style (see the
    module docstring); `group` is the torch.distributed process group of the
    TP ranks (None = default group; no collective when tp_size == 1).
    collective=False skips the all-reduce (single-GPU emulation of one rank's
    share of the work; the result is then this rank's partial only).
    With an `exchange` (FusedExchange) the group runs as ONE fused launch
    whose partials travel through the exchange instead of NCCL."""
    import torch

    ws = workspace if workspace is not None else SplitWorkspace(meta, pool)
    s = stream if stream is not None else torch.cuda.current_stream(pool.device)
    per = max(1, 64 // pool.lora_rank)  # a launch carries <= 64 rank-r columns of P
    if len(sites) > per:
        for i in range(0, len(sites), per):
            apply_lora_group_tp_(ys[i : i + per], x, meta, pool, layer, sites[i : i + per], group, ws, s, collective,
                                 exchange)
        return ys
    if exchange is not None:
        return lora_fused_tp_(ys, x, meta, pool, layer, sites, exchange, s)
    P = lora_shrink_tp_(ys, x, meta, pool, layer, sites, ws, s)
    if pool.tp_size > 1 and collective:
        import torch.distributed as dist

        with torch.cuda.stream(s):
            dist.all_reduce(P[: meta.T], op=dist.ReduceOp.SUM, group=group)
    return lora_expand_tp_(P, ys, x, meta, pool, layer, sites, s)
