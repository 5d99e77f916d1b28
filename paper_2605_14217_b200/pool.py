"""HBM-resident adapter pool (north-star subsystem 1).

Replaces the reference's in-memory catalogue `{adapter_id: ModelAdapter}`
(model.py:325-339, forward_chunk's `adapters` argument, model.py:458) and the
engine's weight sync (engine.py:676-697) with fixed-address device slabs.

HBM layout (one allocation per slab):

    LoRA, per target site t with (n_t, m_t):
        A_t   [L][S_lora][R_lora][m_t]     shrink rows (reference A, (r, m))
        Bt_t  [L][S_lora][R_lora][n_t]     expand rows (reference B^T; B is (n, r))
        scale_t [L][S_lora]                alpha / r etc. (adapters.py:109-117)
    ReFT (DiReFT / LoReFT), residual site:
        A     [L][S_reft][R_reft][d]       DiReFT A, or LoReFT W - R
        B     [L][S_reft][R_reft][d]       DiReFT B, or LoReFT R
        bias  [L][S_reft][R_reft]
        scale [L][S_reft]
        Bt    [L][S_reft][d/8][R_reft/8][8][8]   B^T in UMMA core-matrix order
                                           (tensor-core kernel only, bf16 r 16/32)

One slot's rows for one (layer, site) are contiguous (R * width elements), so
a warp working on a token fetches its adapter with coalesced 128-bit loads;
rows k >= rank are zero.  Slots are numbered LoRA first ([0, S_lora)) then
ReFT ([S_lora, S_lora + S_reft)); `slot_split = S_lora` tells K1 where the
ReFT class starts.  Slabs never move, so a captured CUDA graph stays valid
across registrations and weight syncs: those are
stream-ordered in-place slot overwrites.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable, Mapping, Sequence

import numpy as np
import torch

from . import _lib
from .adapters import AdapterKind, PositionSchedule
from .batch import LORA_TARGETS, ForwardBatch, ModelAdapter
from .errors import ConfigError, InfeasibleBatchError, RankError, ShapeError, StateError, SyncError

__all__ = ["AdapterPool", "SlotInfo", "SlotSnapshot", "torch_dtype_code", "acc_dtype", "tile_kmajor", "untile_kmajor"]

_POW2 = (1, 2, 4, 8, 16, 32, 64)


def torch_dtype_code(dtype: torch.dtype) -> int:
    if dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    if dtype == torch.float32:
        return _lib.DTYPE_F32
    if dtype == torch.float64:
        return _lib.DTYPE_F64
    raise ShapeError(f"unsupported element type {dtype}; use bfloat16, float32 or float64")


def tile_kmajor(bt: torch.Tensor) -> torch.Tensor:
    """[..., n, k] -> [..., n/8, k/8, 8, 8]: the UMMA K-major core-matrix order
    (8 rows x 16 B core matrices, the K-direction ones of a row group adjacent)
    that csrc/reft_tc.cu copies into shared memory with one bulk copy."""
    *lead, n, k = bt.shape
    return bt.reshape(*lead, n // 8, 8, k // 8, 8).transpose(-3, -2).contiguous()


def untile_kmajor(t: torch.Tensor) -> torch.Tensor:
    """Inverse of tile_kmajor: [..., n/8, k/8, 8, 8] -> [..., n, k]."""
    *lead, nb, kb, _, _ = t.shape
    return t.transpose(-3, -2).reshape(*lead, nb * 8, kb * 8)


def acc_dtype(dtype: torch.dtype) -> torch.dtype:
    """Accumulator / scale / bias type for a pool element type."""
    return torch.float64 if dtype == torch.float64 else torch.float32


def _round_rank(r: int) -> int:
    for p in _POW2:
        if r <= p:
            return p
    raise RankError(f"rank {r} exceeds the device limit 64")


@dataclass
class SlotSnapshot:
    """Pinned host copy of one adapter's device slot (AdapterPool.export_slot)."""

    info: "SlotInfo"
    host: list
    ready: object  # torch.cuda.Event recorded after the D2H copies

    @property
    def nbytes(self) -> int:
        return sum(h.numel() * h.element_size() for h in self.host)


@dataclass
class SlotInfo:
    adapter_id: int
    slot: int
    kind: AdapterKind
    rank: int
    schedule: PositionSchedule
    version: int = 0


class AdapterPool:
    """Fixed-capacity HBM pool for LoRA^P and ReFT^P adapters of one model."""

    def __init__(
        self,
        n_layers: int,
        d_model: int,
        lora_sites: Mapping[str, tuple[int, int]] | None = None,
        lora_capacity: int = 0,
        lora_rank: int = 16,
        reft_capacity: int = 0,
        reft_rank: int = 16,
        dtype: torch.dtype = torch.bfloat16,
        device=None,
        tp_rank: int = 0,
        tp_size: int = 1,
    ):
        from .tp import site_shard

        if n_layers < 1 or d_model < 1:
            raise ConfigError("n_layers and d_model must be >= 1")
        if lora_capacity < 0 or reft_capacity < 0 or lora_capacity + reft_capacity < 1:
            raise ConfigError("the pool needs at least one slot")
        self.device = _lib.require_cuda(device)
        self.dtype = dtype
        self.dtype_code = torch_dtype_code(dtype)
        self.acc = acc_dtype(dtype)
        self.n_layers = int(n_layers)
        self.d_model = int(d_model)
        self.lora_capacity = int(lora_capacity)
        self.reft_capacity = int(reft_capacity)
        self.slot_split = self.lora_capacity
        self.lora_sites: dict[str, tuple[int, int]] = dict(lora_sites or {})
        bad = set(self.lora_sites) - set(LORA_TARGETS)
        if bad:
            raise ConfigError(f"unknown lora targets: {sorted(bad)}")
        if self.lora_capacity and not self.lora_sites:
            raise ConfigError("a pool with LoRA slots needs lora_sites {name: (n, m)}")
        self.lora_rank = _round_rank(lora_rank) if self.lora_capacity else 0
        self.reft_rank = _round_rank(reft_rank) if self.reft_capacity else 0
        L, dev = self.n_layers, self.device
        z = dict(dtype=dtype, device=dev)
        za = dict(dtype=self.acc, device=dev)
        self.reft_Bt: torch.Tensor | None = None
        self.reft_tc = False
        self.lora_A: dict[str, torch.Tensor] = {}
        self.lora_Bt: dict[str, torch.Tensor] = {}
        self.lora_Bt_tc: dict[str, torch.Tensor] = {}
        self.lora_scale: dict[str, torch.Tensor] = {}
        # tensor parallelism (tp.py): every LoRA site keeps A sharded along its
        # input dim and B along its output dim; tp_size == 1 is the whole site
        self.tp_rank, self.tp_size = int(tp_rank), int(tp_size)
        self.lora_shard = {name: site_shard(name, n, m, self.tp_rank, self.tp_size)
                           for name, (n, m) in self.lora_sites.items()}
        lora_tc = dtype == torch.bfloat16 and self.lora_rank in (16, 32)
        for name, sh in self.lora_shard.items():
            if self.lora_capacity:
                self.lora_A[name] = torch.zeros(L, self.lora_capacity, self.lora_rank, sh.m_loc, **z)
                self.lora_Bt[name] = torch.zeros(L, self.lora_capacity, self.lora_rank, sh.n_loc, **z)
                self.lora_scale[name] = torch.zeros(L, self.lora_capacity, **za)
                if lora_tc and sh.n_loc % 128 == 0:
                    # B (= Bt^T) pre-tiled for the tensor-core expand (csrc/lora_split.cu)
                    self.lora_Bt_tc[name] = torch.zeros(L, self.lora_capacity, sh.n_loc // 8, self.lora_rank // 8,
                                                        8, 8, **z)
        if self.reft_capacity:
            S, R, d = self.reft_capacity, self.reft_rank, self.d_model
            self.reft_A = torch.zeros(L, S, R, d, **z)
            self.reft_B = torch.zeros(L, S, R, d, **z)
            # B^T pre-tiled in UMMA core-matrix order for the tcgen05 expand
            # (csrc/reft_tc.cu, include/preft.h): bf16, r 16/32, d % 128 == 0
            self.reft_tc = dtype == torch.bfloat16 and R in (16, 32) and d % 128 == 0
            self.reft_Bt = torch.zeros(L, S, d // 8, R // 8, 8, 8, **z) if self.reft_tc else None
            self.reft_bias = torch.zeros(L, S, R, **za)
            self.reft_scale = torch.zeros(L, S, **za)
        self._slots: dict[int, SlotInfo] = {}
        self._free_lora = list(range(self.lora_capacity))[::-1]
        self._free_reft = list(range(self.lora_capacity, self.lora_capacity + self.reft_capacity))[::-1]

    # ------------------------------------------------------------ catalogue
    @property
    def slot_of(self) -> dict[int, int]:
        return {aid: info.slot for aid, info in self._slots.items()}

    def info(self, adapter_id: int) -> SlotInfo:
        try:
            return self._slots[adapter_id]
        except KeyError:
            raise StateError(f"adapter {adapter_id} is not registered") from None

    def __contains__(self, adapter_id: int) -> bool:
        return adapter_id in self._slots

    def __len__(self) -> int:
        return len(self._slots)

    @property
    def nbytes(self) -> int:
        tensors: list[torch.Tensor] = [*self.lora_A.values(), *self.lora_Bt.values(), *self.lora_scale.values(),
                                       *self.lora_Bt_tc.values()]
        if self.reft_capacity:
            tensors += [self.reft_A, self.reft_B, self.reft_bias, self.reft_scale]
            if self.reft_Bt is not None:
                tensors.append(self.reft_Bt)
        return sum(t.numel() * t.element_size() for t in tensors)

    def _validate(self, adapter: ModelAdapter) -> None:
        if adapter.kind is AdapterKind.LORA:
            if not self.lora_capacity:
                raise ConfigError("this pool has no LoRA slots")
            if adapter.rank > self.lora_rank:
                raise RankError(f"rank {adapter.rank} exceeds the pool's LoRA rank {self.lora_rank}")
            for (layer, name), p in adapter.lora_sites.items():
                if not 0 <= layer < self.n_layers:
                    raise ShapeError(f"layer {layer} out of range for a {self.n_layers}-layer pool")
                if name not in self.lora_sites:
                    raise ShapeError(f"site {name} is not a target of this pool")
                if tuple(p.dims) != tuple(self.lora_sites[name]):
                    raise ShapeError(f"site {name} has dims {p.dims}, pool expects {self.lora_sites[name]}")
                if p.kind is not AdapterKind.LORA or p.rank != adapter.rank:
                    raise ShapeError("site bundle does not match the adapter's kind/rank")
        else:
            if not self.reft_capacity:
                raise ConfigError("this pool has no ReFT slots")
            if adapter.rank > self.reft_rank:
                raise RankError(f"rank {adapter.rank} exceeds the pool's ReFT rank {self.reft_rank}")
            if len(adapter.reft_sites) != self.n_layers:
                raise ShapeError(f"{len(adapter.reft_sites)} ReFT sites for a {self.n_layers}-layer pool")
            for p in adapter.reft_sites:
                if tuple(p.dims) != (self.d_model,):
                    raise ShapeError(f"ReFT site dims {p.dims}, pool expects ({self.d_model},)")
                if p.kind is not adapter.kind or p.rank != adapter.rank:
                    raise ShapeError("site bundle does not match the adapter's kind/rank")

    def register(self, adapter: ModelAdapter, stream=None) -> int:
        """Place an adapter in a free slot (or overwrite its own slot); returns the slot."""
        self._validate(adapter)
        cur = self._slots.get(adapter.adapter_id)
        if cur is not None:
            if (cur.kind is AdapterKind.LORA) != (adapter.kind is AdapterKind.LORA):
                raise StateError(f"adapter {adapter.adapter_id} cannot change family in place")
            slot = cur.slot
        else:
            free = self._free_lora if adapter.kind is AdapterKind.LORA else self._free_reft
            if not free:
                raise InfeasibleBatchError(f"no free {adapter.kind.value} slot (pool is full)")
            slot = free.pop()
        self._upload(adapter, slot, stream)
        version = 0 if cur is None else cur.version + 1
        self._slots[adapter.adapter_id] = SlotInfo(
            adapter.adapter_id, slot, adapter.kind, adapter.rank, adapter.schedule, version
        )
        return slot

    def register_many(self, adapters: Iterable[ModelAdapter], stream=None) -> list[int]:
        return [self.register(a, stream) for a in adapters]

    def unregister(self, adapter_id: int, zero: bool = True) -> None:
        """Free an adapter's slot (zero=False leaves the stale weights for a
        caller that overwrites the whole slot next, e.g. paging)."""
        info = self.info(adapter_id)
        del self._slots[adapter_id]
        if zero:
            self._zero_slot(info)
        (self._free_lora if info.kind is AdapterKind.LORA else self._free_reft).append(info.slot)

    # ------------------------------------------------------------ slot snapshots (paging)
    def slot_views(self, kind: AdapterKind, slot: int) -> list[torch.Tensor]:
        """Device views of every slab slice one slot owns, all layers."""
        if kind is AdapterKind.LORA:
            views = []
            for name in self.lora_sites:
                views += [self.lora_A[name][:, slot], self.lora_Bt[name][:, slot], self.lora_scale[name][:, slot]]
                if name in self.lora_Bt_tc:
                    views.append(self.lora_Bt_tc[name][:, slot])
            return views
        j = slot - self.slot_split
        views = [self.reft_A[:, j], self.reft_B[:, j], self.reft_bias[:, j], self.reft_scale[:, j]]
        if self.reft_Bt is not None:
            views.append(self.reft_Bt[:, j])
        return views

    def export_slot(self, adapter_id: int, stream=None) -> "SlotSnapshot":
        """Pinned host copy of an adapter's device slot (stream-ordered D2H)."""
        info = self.info(adapter_id)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        host = []
        with torch.cuda.stream(s):
            for v in self.slot_views(info.kind, info.slot):
                h = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
                h.copy_(v, non_blocking=True)
                host.append(h)
        ev = torch.cuda.Event()
        ev.record(s)
        return SlotSnapshot(SlotInfo(adapter_id, -1, info.kind, info.rank, info.schedule, info.version), host, ev)

    def import_slot(self, snap: "SlotSnapshot", stream=None) -> int:
        """Place a snapshot into a free slot (stream-ordered H2D); returns the slot."""
        info = snap.info
        if info.adapter_id in self._slots:
            raise StateError(f"adapter {info.adapter_id} is already resident")
        free = self._free_lora if info.kind is AdapterKind.LORA else self._free_reft
        if not free:
            raise InfeasibleBatchError(f"no free {info.kind.value} slot (pool is full)")
        slot = free.pop()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        snap.ready.synchronize()  # the D2H that filled the snapshot has landed
        with torch.cuda.stream(s):
            for v, h in zip(self.slot_views(info.kind, slot), snap.host):
                v.copy_(h, non_blocking=True)
        self._slots[info.adapter_id] = SlotInfo(info.adapter_id, slot, info.kind, info.rank, info.schedule,
                                                info.version)
        return slot

    @property
    def lora_slot_bytes(self) -> int:
        return sum(v.numel() * v.element_size() for v in self.slot_views(AdapterKind.LORA, 0)) if self.lora_capacity else 0

    @property
    def reft_slot_bytes(self) -> int:
        return (sum(v.numel() * v.element_size() for v in self.slot_views(AdapterKind.DIREFT, self.slot_split))
                if self.reft_capacity else 0)

    def sync(self, updates: Sequence[tuple[int, ModelAdapter]], stream=None) -> None:
        """Atomic weight sync at a step boundary (engine.py:676-697).

        Every update is validated before any slot is touched; a bad payload
        raises SyncError and leaves the pool unchanged.  The uploads are
        stream-ordered, so kernels already queued for the current step read
        the old weights and the next step reads the new ones.
        """
        for aid, payload in updates:
            if aid not in self._slots:
                raise SyncError(f"sync targets unknown adapter {aid}")
            if payload is None:
                raise SyncError("functional sync needs replacement weights")
            cur = self._slots[aid]
            if payload.adapter_id != aid or payload.kind is not cur.kind or payload.rank != cur.rank or (
                payload.schedule is not cur.schedule
            ):
                raise SyncError(f"replacement for adapter {aid} does not match")
            try:
                self._validate(payload)
            except (ShapeError, RankError, ConfigError) as exc:
                raise SyncError(f"replacement for adapter {aid} is malformed: {exc}") from None
        for aid, payload in updates:
            info = self._slots[aid]
            self._upload(payload, info.slot, stream)
            info.version += 1

    # ------------------------------------------------------------ K4 upload
    def _convert(self, dst: torch.Tensor, code: int, src_dev: torch.Tensor, off: int, srow: int, scol: int,
                 rows_valid: int, rows: int, cols: int, stream) -> None:
        lib = _lib.load()
        ptr = src_dev.data_ptr() + 8 * off
        st = lib.preft_convert_2d(
            ctypes.c_void_p(dst.data_ptr()), code, dst.stride(-2) if dst.dim() > 1 else 1, ctypes.c_void_p(ptr),
            srow, scol, rows_valid, rows, cols, ctypes.c_void_p(stream.cuda_stream)
        )
        _lib.check(st, "convert_2d")

    def _upload(self, adapter: ModelAdapter, slot: int, stream=None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):  # zeroing, H2D and conversions all ordered on s
            self._upload_on(adapter, slot, s)

    def _upload_on(self, adapter: ModelAdapter, slot: int, s) -> None:
        chunks: list[np.ndarray] = []
        plan = []  # (dst view, dtype code, offset, srow, scol, rows_valid, rows, cols)
        off = 0

        def add(arr: np.ndarray) -> int:
            nonlocal off
            a = np.ascontiguousarray(arr, dtype=np.float64).ravel()
            chunks.append(a)
            o = off
            off += a.size
            return o

        acc_code = torch_dtype_code(self.acc)
        if adapter.kind is AdapterKind.LORA:
            R = self.lora_rank
            for name in self.lora_sites:
                self.lora_A[name][:, slot].zero_()
                self.lora_Bt[name][:, slot].zero_()
                self.lora_scale[name][:, slot].zero_()
            scales: dict[str, np.ndarray] = {name: np.zeros(self.n_layers) for name in self.lora_sites}
            for (layer, name), p in adapter.lora_sites.items():
                sh = self.lora_shard[name]
                r = p.rank
                m, n = sh.m_loc, sh.n_loc
                # this rank's slice: A columns [m0, m0+m_loc), B rows [n0, n0+n_loc)
                A = np.asarray(p.A)[:, sh.m0 : sh.m0 + m]
                B = np.asarray(p.B)[sh.n0 : sh.n0 + n, :]
                plan.append((self.lora_A[name][layer, slot], self.dtype_code, add(A), m, 1, r, R, m))
                # B is (n, r) row-major: Bt[k][j] = B[j][k] -> src strides (1, r)
                plan.append((self.lora_Bt[name][layer, slot], self.dtype_code, add(B), 1, r, r, R, n))
                scales[name][layer] = p.prefactor
            for name, sc in scales.items():
                plan.append((self.lora_scale[name][:, slot].unsqueeze(1), acc_code, add(sc), 1, 1, self.n_layers,
                             self.n_layers, 1))
        else:
            R, d = self.reft_rank, self.d_model
            j = slot - self.slot_split
            if self.reft_Bt is not None:
                self.reft_Bt[:, j].zero_()  # columns >= rank stay zero
            sc = np.zeros(self.n_layers)
            for layer, p in enumerate(adapter.reft_sites):
                shrink, expand, bias = p.device_operands()
                r = p.rank
                plan.append((self.reft_A[layer, j], self.dtype_code, add(shrink), d, 1, r, R, d))
                o_exp = add(expand)
                plan.append((self.reft_B[layer, j], self.dtype_code, o_exp, d, 1, r, R, d))
                plan.append((self.reft_bias[layer, j].unsqueeze(1), acc_code, add(bias), 1, 1, r, R, 1))
                sc[layer] = p.prefactor
            plan.append((self.reft_scale[:, j].unsqueeze(1), acc_code, add(sc), 1, 1, self.n_layers, self.n_layers, 1))
        host = torch.from_numpy(np.concatenate(chunks) if chunks else np.zeros(1))
        dev = host.to(self.device, non_blocking=False)
        for dst, code, o, srow, scol, rv, rows, cols in plan:
            self._convert(dst, code, dev, o, srow, scol, rv, rows, cols, s)
        if adapter.kind is AdapterKind.LORA:
            for name, tc in self.lora_Bt_tc.items():
                tc[:, slot].copy_(tile_kmajor(self.lora_Bt[name][:, slot].transpose(-1, -2)))
        if adapter.kind is not AdapterKind.LORA and self.reft_Bt is not None:
            # the tensor-core copy is a pure permutation of the converted B slab
            j = slot - self.slot_split
            self.reft_Bt[:, j].copy_(tile_kmajor(self.reft_B[:, j].transpose(-1, -2)))
        dev.record_stream(s)

    def _zero_slot(self, info: SlotInfo) -> None:
        if info.kind is AdapterKind.LORA:
            for name in self.lora_sites:
                self.lora_A[name][:, info.slot].zero_()
                self.lora_Bt[name][:, info.slot].zero_()
                self.lora_scale[name][:, info.slot].zero_()
                if name in self.lora_Bt_tc:
                    self.lora_Bt_tc[name][:, info.slot].zero_()
        else:
            j = info.slot - self.slot_split
            self.reft_A[:, j].zero_()
            self.reft_B[:, j].zero_()
            if self.reft_Bt is not None:
                self.reft_Bt[:, j].zero_()
            self.reft_bias[:, j].zero_()
            self.reft_scale[:, j].zero_()

    # ------------------------------------------------------------ synthetic fill (benchmarks)
    def fill_synthetic_(
        self,
        n_adapters: int,
        kind: AdapterKind,
        rank: int,
        schedule: PositionSchedule = PositionSchedule.PREFILL_ONLY,
        seed: int = 0,
        sigma: float = 0.01,
        first_id: int = 0,
        ids: Sequence[int] | None = None,
    ) -> list[int]:
        """Register `n_adapters` random adapters directly on the device.

        The benchmark protocol materialises untrained random adapters
        (PAPER.md:843-849): LoRA A, B ~ N(0, sigma^2); ReFT: orthonormal-ish
        expand rows and N(0, sigma^2) shrink rows / bias.  Generating 512
        Llama-shaped adapters through float64 host bundles would take minutes
        and ~10 GB of host RAM, so the slabs are filled with torch's device
        RNG instead.  Correctness of registration itself is covered by tests
        through `register`.
        """
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        wanted = list(ids) if ids is not None else [first_id + i for i in range(n_adapters)]
        ids = []
        for aid in wanted:
            if aid in self._slots:
                raise StateError(f"adapter {aid} is already registered")
            free = self._free_lora if kind is AdapterKind.LORA else self._free_reft
            if not free:
                raise InfeasibleBatchError("pool is full")
            slot = free.pop()
            self._slots[aid] = SlotInfo(aid, slot, kind, rank, schedule, 0)
            ids.append(aid)
        if kind is AdapterKind.LORA:
            if rank > self.lora_rank:
                raise RankError(f"rank {rank} exceeds the pool's LoRA rank {self.lora_rank}")
            slots = torch.tensor([self._slots[a].slot for a in ids], device=self.device)
            for name, sh in self.lora_shard.items():
                n, m = sh.n_loc, sh.m_loc
                for layer in range(self.n_layers):
                    A = torch.randn(len(ids), rank, m, generator=g, device=self.device, dtype=torch.float32) * sigma
                    Bt = torch.randn(len(ids), rank, n, generator=g, device=self.device, dtype=torch.float32) * sigma
                    self.lora_A[name][layer].index_copy_(0, slots, torch.nn.functional.pad(A, (0, 0, 0, self.lora_rank - rank)).to(self.dtype))
                    Btp = torch.nn.functional.pad(Bt, (0, 0, 0, self.lora_rank - rank)).to(self.dtype)
                    self.lora_Bt[name][layer].index_copy_(0, slots, Btp)
                    if name in self.lora_Bt_tc:
                        self.lora_Bt_tc[name][layer].index_copy_(0, slots, tile_kmajor(Btp.transpose(1, 2)))
                self.lora_scale[name].index_fill_(1, slots, 32.0 / rank)
        else:
            if rank > self.reft_rank:
                raise RankError(f"rank {rank} exceeds the pool's ReFT rank {self.reft_rank}")
            js = torch.tensor([self._slots[a].slot - self.slot_split for a in ids], device=self.device)
            d = self.d_model
            for layer in range(self.n_layers):
                A = torch.randn(len(ids), rank, d, generator=g, device=self.device) * sigma
                B = torch.randn(len(ids), rank, d, generator=g, device=self.device) / np.sqrt(d)
                b = torch.randn(len(ids), rank, generator=g, device=self.device) * 0.1
                pad = self.reft_rank - rank
                self.reft_A[layer].index_copy_(0, js, torch.nn.functional.pad(A, (0, 0, 0, pad)).to(self.dtype))
                Bp = torch.nn.functional.pad(B, (0, 0, 0, pad)).to(self.dtype)
                self.reft_B[layer].index_copy_(0, js, Bp)
                if self.reft_Bt is not None:
                    self.reft_Bt[layer].index_copy_(0, js, tile_kmajor(Bp.transpose(1, 2)))
                self.reft_bias[layer].index_copy_(0, js, torch.nn.functional.pad(b, (0, pad)).to(self.acc))
            self.reft_scale.index_fill_(1, js, 1.0 / np.sqrt(rank))
        return ids

    # ------------------------------------------------------------ batches
    def build_meta(self, meta, batch: ForwardBatch, stream=None):
        """Stage a ForwardBatch into `meta` with this pool's slot mapping and launch K1."""
        meta.set_slot_split(self.slot_split)
        return meta.build(batch, self.slot_of, stream)

    def entry_arrays(self, qsl: np.ndarray, adapter_ids: Sequence[int | None], flags: np.ndarray) -> np.ndarray:
        """Slot per entry for raw-array staging.

        An adapter that runs in the entry's phase must be resident (else
        BatchError, as forward_chunk raises for ids missing from the catalogue,
        model.py:470-472).  A PREFILL_ONLY adapter of a decode entry never runs
        (engine.py:521-526), so it needs no slot: with paging it may well be
        evicted, and the entry stages as adapter-less (the same mask)."""
        from .errors import BatchError

        out = np.full(len(adapter_ids), -1, dtype=np.int32)
        flags = np.asarray(flags)
        for i, a in enumerate(adapter_ids):
            if a is not None:
                info = self._slots.get(a)
                if info is None:
                    runs = not (flags[i] & _lib.ENTRY_DECODE) or bool(flags[i] & _lib.ENTRY_ALL_POSITIONS)
                    if runs:
                        raise BatchError(f"adapter {a} not in catalogue")
                    continue
                out[i] = info.slot
        return out
