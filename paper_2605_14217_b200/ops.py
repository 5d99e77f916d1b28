"""Hot-path operators: the B200 replacements for the two adapter hook sites of
forward_chunk (model.py:442-452 `_project`, model.py:543-546 ReFT hook).

    apply_lora_(y, x, meta, pool, layer, site)          y[rows] += delta(x[rows])
    apply_lora_group_([y_q, y_k, y_v], x, meta, pool, layer, ("Wq", "Wk", "Wv"))
    apply_reft_(h, meta, pool, layer)                   h[rows] += delta(h[rows])

`rows` are the tokens K1 selected (decode tokens of PREFILL_ONLY adapters and
adapter-less tokens are never read or written).  One call covers every entry
of the batch, whatever mix of adapters it carries — the reference's
`layer x entry` Python loop (model.py:504-546) becomes one launch per site
(or per group of sites sharing x).  All calls are stream-ordered and
CUDA-graph capturable; none synchronises the host.

Also here: the device implementations behind the reference-shaped
`adapters.delta_for_rows` / `apply_masked` (f64 mode).
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .adapters import AdapterKind, AdapterParams
from .errors import ConfigError, ShapeError
from .meta import BatchMeta, default_meta
from .pool import AdapterPool, _round_rank, acc_dtype, torch_dtype_code

__all__ = [
    "apply_lora_",
    "apply_lora_group_",
    "apply_reft_",
    "is_torch_tensor",
    "delta_rows_host",
    "delta_rows_device",
    "apply_masked_host",
]


def is_torch_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


def row_stride(t: torch.Tensor) -> int:
    """Leading-dimension stride in elements (a 1-row view may report stride 0)."""
    return t.stride(0) if t.shape[0] > 1 else t.shape[1]


def _stream(stream, device) -> torch.cuda.Stream:
    return stream if stream is not None else torch.cuda.current_stream(device)


def _check_act(t: torch.Tensor, name: str, width: int, rows: int, dtype: torch.dtype, device) -> None:
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise ShapeError(f"{name} must be a CUDA tensor")
    if t.device != device:
        raise ShapeError(f"{name} is on {t.device}, the pool on {device}")
    if t.dtype != dtype:
        raise ShapeError(f"{name} has dtype {t.dtype}, the pool holds {dtype}")
    if t.dim() != 2 or t.stride(1) != 1:
        raise ShapeError(f"{name} must be a 2-D row-major (stride(1) == 1) tensor")
    if t.shape[1] != width:
        raise ShapeError(f"{name} width {t.shape[1]}, expected {width}")
    if t.shape[0] < rows:
        raise ShapeError(f"{name} has {t.shape[0]} rows, the batch has {rows} tokens")


def lora_site_chunks(sites: Sequence[str], rank: int) -> list[tuple[int, int]]:
    """Split a group of sites sharing x into launches the kernel accepts:
    at most 3 sites and nsites * r_max <= 64 per launch (include/preft.h)."""
    per = max(1, min(3, 64 // max(1, rank)))
    return [(i, min(len(sites), i + per)) for i in range(0, len(sites), per)]


def check_lora_group(ys, x, meta_rows: int, pool: AdapterPool, layer: int, sites: Sequence[str]) -> int:
    """Shared validation of a LoRA group (ops and StepPlan); returns m."""
    if not 1 <= len(sites) <= 3 or len(ys) != len(sites):
        raise ShapeError("a LoRA group has 1 to 3 sites and one output per site")
    if not isinstance(layer, (int, np.integer)) or not 0 <= layer < pool.n_layers:
        raise ShapeError(f"layer {layer} out of range [0, {pool.n_layers})")
    if not pool.lora_capacity:
        raise ShapeError("the pool holds no LoRA adapters")
    if pool.tp_size > 1:
        raise ConfigError("a tensor-parallel pool shard needs tp.apply_lora_group_tp_ (shrink, all-reduce, expand)")
    unknown = [s for s in sites if s not in pool.lora_sites]
    if unknown:
        raise ShapeError(f"unknown LoRA site(s) {unknown}; the pool has {sorted(pool.lora_sites)}")
    ms = {pool.lora_sites[s][1] for s in sites}
    if len(ms) != 1:
        raise ShapeError(f"sites {tuple(sites)} do not share an input width")
    m = ms.pop()
    _check_act(x, "x", m, meta_rows, pool.dtype, pool.device)
    for name, y in zip(sites, ys):
        _check_act(y, f"y[{name}]", pool.lora_sites[name][0], meta_rows, pool.dtype, pool.device)
    return m


def check_reft(h, meta_rows: int, pool: AdapterPool, layer: int) -> None:
    if not pool.reft_capacity:
        raise ShapeError("the pool holds no ReFT adapters")
    if not isinstance(layer, (int, np.integer)) or not 0 <= layer < pool.n_layers:
        raise ShapeError(f"layer {layer} out of range [0, {pool.n_layers})")
    _check_act(h, "h", pool.d_model, meta_rows, pool.dtype, pool.device)


def wants_lora_part(pool: AdapterPool) -> bool:
    """bf16 pools of rank 16/32 run LoRA on tensor cores (preft_lora_apply's
    tcgen05 route), which needs the meta's rank-r workspace."""
    return pool.dtype == torch.bfloat16 and pool.lora_rank in (16, 32)


def lora_site_array(ys, pool: AdapterPool, layer: int, sites: Sequence[str]):
    arr = (_lib.PreftLoraSite * 3)()
    for i, (name, y) in enumerate(zip(sites, ys)):
        arr[i].A = pool.lora_A[name][layer].data_ptr()
        arr[i].Bt = pool.lora_Bt[name][layer].data_ptr()
        arr[i].scale = pool.lora_scale[name][layer].data_ptr()
        arr[i].bias = None
        arr[i].y = y.data_ptr()
        arr[i].ldy = row_stride(y)
        arr[i].n = pool.lora_sites[name][0]
        tc = pool.lora_Bt_tc.get(name)
        arr[i].Bt_tc = tc[layer].data_ptr() if tc is not None else None
    return arr


def apply_lora_group_(
    ys: Sequence[torch.Tensor],
    x: torch.Tensor,
    meta: BatchMeta,
    pool: AdapterPool,
    layer: int,
    sites: Sequence[str],
    stream=None,
) -> Sequence[torch.Tensor]:
    """y_s[rows] += s_a * (x[rows] A_s,a^T) B_s,a^T for 1-3 sites sharing x, in place.

    Groups whose fused rank would exceed the kernel's 64 rank-r lanes
    (e.g. rank-32 q/k/v) run as several launches over the same x."""
    m = check_lora_group(ys, x, meta.T, pool, layer, sites)
    s = _stream(stream, pool.device)
    meta.require_split(pool.slot_split)
    if wants_lora_part(pool):
        meta.ensure_lora_part()
    lib = _lib.load()
    for lo, hi in lora_site_chunks(sites, pool.lora_rank):
        arr = lora_site_array(ys[lo:hi], pool, layer, sites[lo:hi])
        st = lib.preft_lora_apply(
            ctypes.byref(meta.c), ctypes.c_void_p(x.data_ptr()), row_stride(x), m, arr, hi - lo, pool.lora_rank,
            pool.dtype_code, ctypes.c_void_p(s.cuda_stream)
        )
        _lib.check(st, "lora_apply")
    return ys


def apply_lora_(y: torch.Tensor, x: torch.Tensor, meta: BatchMeta, pool: AdapterPool, layer: int, site: str,
                stream=None) -> torch.Tensor:
    """`_project`'s delta (model.py:449-451): y[rows] += delta(x[rows]), in place."""
    apply_lora_group_([y], x, meta, pool, layer, [site], stream)
    return y


def apply_reft_(h: torch.Tensor, meta: BatchMeta, pool: AdapterPool, layer: int, stream=None) -> torch.Tensor:
    """ReFT residual hook (model.py:543-546): h[rows] += delta(h[rows]), in place."""
    check_reft(h, meta.T, pool, layer)
    s = _stream(stream, pool.device)
    meta.require_split(pool.slot_split)
    st = _lib.load().preft_reft_apply(
        ctypes.byref(meta.c), ctypes.c_void_p(h.data_ptr()), h.shape[0], row_stride(h), pool.d_model,
        ctypes.c_void_p(pool.reft_A[layer].data_ptr()), ctypes.c_void_p(pool.reft_B[layer].data_ptr()),
        ctypes.c_void_p(pool.reft_Bt[layer].data_ptr() if pool.reft_Bt is not None else None),
        ctypes.c_void_p(pool.reft_bias[layer].data_ptr()), ctypes.c_void_p(pool.reft_scale[layer].data_ptr()),
        pool.reft_rank, pool.dtype_code, ctypes.c_void_p(s.cuda_stream)
    )
    _lib.check(st, "reft_apply")
    return h


# ---------------------------------------------------------------- drop-in (reference-shaped) API


class _OneSlot:
    """Device operands of a single AdapterParams bundle (slot 0)."""

    def __init__(self, params: AdapterParams, dtype: torch.dtype, device):
        lib = _lib.load()
        self.R = _round_rank(params.rank)
        shrink, expand, bias = params.device_operands()
        self.width_in = shrink.shape[1]
        self.width_out = expand.shape[1]
        code = torch_dtype_code(dtype)
        acc = acc_dtype(dtype)
        self.A = torch.zeros(1, self.R, self.width_in, dtype=dtype, device=device)
        self.B = torch.zeros(1, self.R, self.width_out, dtype=dtype, device=device)
        src = torch.from_numpy(np.concatenate([shrink.ravel(), expand.ravel()])).to(device)
        s = torch.cuda.current_stream(device)
        r = params.rank
        for dst, off, cols in ((self.A, 0, self.width_in), (self.B, shrink.size, self.width_out)):
            st = lib.preft_convert_2d(
                ctypes.c_void_p(dst.data_ptr()), code, cols, ctypes.c_void_p(src.data_ptr() + 8 * off), cols, 1, r,
                self.R, cols, ctypes.c_void_p(s.cuda_stream)
            )
            _lib.check(st, "convert_2d")
        self.scale = torch.tensor([params.prefactor], dtype=acc, device=device)
        self.bias = None
        if bias is not None:
            b = np.zeros(self.R)
            b[:r] = bias
            self.bias = torch.from_numpy(b).to(device=device, dtype=acc)
        self._keep = src


def _one_entry_meta(n_sel: int, total: int, device, split: int) -> BatchMeta:
    """Batch of `total` rows whose first `n_sel` rows carry slot 0."""
    n_entries = 1 if n_sel in (0, total) else 2
    meta = default_meta(n_entries, total, device)
    if n_sel in (0, total):
        qsl = np.array([0, total], dtype=np.int32)
        slots = np.array([0 if n_sel else -1], dtype=np.int32)
    else:
        qsl = np.array([0, n_sel, total], dtype=np.int32)
        slots = np.array([0, -1], dtype=np.int32)
    flags = np.zeros(len(slots), dtype=np.int32)
    meta.set_slot_split(split)
    meta.build_arrays(qsl, slots, flags)
    return meta


def _lora_launch(meta: BatchMeta, ops: _OneSlot, x: torch.Tensor, y: torch.Tensor, code: int) -> None:
    arr = (_lib.PreftLoraSite * 1)()
    arr[0].A = ops.A.data_ptr()
    arr[0].Bt = ops.B.data_ptr()
    arr[0].scale = ops.scale.data_ptr()
    arr[0].bias = ops.bias.data_ptr() if ops.bias is not None else None
    arr[0].y = y.data_ptr()
    arr[0].ldy = row_stride(y)
    arr[0].n = y.shape[1]
    s = torch.cuda.current_stream(x.device)
    st = _lib.load().preft_lora_apply(
        ctypes.byref(meta.c), ctypes.c_void_p(x.data_ptr()), row_stride(x), x.shape[1], arr, 1, ops.R, code,
        ctypes.c_void_p(s.cuda_stream)
    )
    _lib.check(st, "lora_apply")


def delta_rows_device(params: AdapterParams, rows: torch.Tensor) -> torch.Tensor:
    """delta_for_rows on a CUDA tensor: one shrink/expand launch, out of place."""
    dev = _lib.require_cuda(rows.device)
    dtype = rows.dtype
    torch_dtype_code(dtype)
    rows = rows.contiguous()
    P = rows.shape[0]
    out_w = params.dims[0]
    y = torch.zeros(P, out_w, dtype=dtype, device=dev)
    if P == 0:
        return y
    ops = _OneSlot(params, dtype, dev)
    meta = _one_entry_meta(P, P, dev, _lib.SLOT_SPLIT_ALL_LORA)
    _lora_launch(meta, ops, rows, y, torch_dtype_code(dtype))
    return y


def delta_rows_host(params: AdapterParams, rows: np.ndarray) -> np.ndarray:
    """delta_for_rows on float64 host rows: computed on the GPU in f64 mode."""
    dev = _lib.require_cuda()
    x = torch.from_numpy(np.ascontiguousarray(rows)).to(dev)
    return delta_rows_device(params, x).cpu().numpy()


def apply_masked_host(params: AdapterParams, out: np.ndarray, src: np.ndarray | None, cut: int) -> np.ndarray:
    """apply_masked's masked add on the GPU (f64): rows < cut get the delta, rows >= cut are never touched."""
    dev = _lib.require_cuda()
    total = out.shape[0]
    y = torch.from_numpy(np.ascontiguousarray(out)).to(dev)
    ops = _OneSlot(params, torch.float64, dev)
    if params.kind is AdapterKind.LORA:
        x = torch.from_numpy(np.ascontiguousarray(src)).to(dev)
        meta = _one_entry_meta(cut, total, dev, _lib.SLOT_SPLIT_ALL_LORA)
        _lora_launch(meta, ops, x, y, _lib.DTYPE_F64)
    else:
        meta = _one_entry_meta(cut, total, dev, 0)  # slot 0 is a ReFT-class slot
        s = torch.cuda.current_stream(dev)
        st = _lib.load().preft_reft_apply(
            ctypes.byref(meta.c), ctypes.c_void_p(y.data_ptr()), y.shape[0], row_stride(y), y.shape[1],
            ctypes.c_void_p(ops.A.data_ptr()), ctypes.c_void_p(ops.B.data_ptr()), None,
            ctypes.c_void_p(ops.bias.data_ptr()),
            ctypes.c_void_p(ops.scale.data_ptr()), ops.R, _lib.DTYPE_F64, ctypes.c_void_p(s.cuda_stream)
        )
        _lib.check(st, "reft_apply")
    return y.cpu().numpy()
