"""Device batch metadata (K1) — the B200 replacement for compute_position_mask
and the per-entry row selection of forward_chunk (model.py:305-319, 474-475,
509, 538).

`BatchMeta` owns a fixed-capacity, fixed-address device workspace (so the
step that uses it can be captured in a CUDA graph) plus a pinned host staging
buffer.  Per step the host packs (E, T, query_start_loc, slot, flags) into the
pinned buffer, issues ONE async H2D copy and launches `preft_meta_build`; the
kernels after it read everything they need (selected-token count, sorted
(token, slot) list, tiles) from device memory, so there is no host sync on
the hot path.  Reading results back (`mask_host`, `counters_host`, ...) is for
tests and the reference-shaped API only.
"""

from __future__ import annotations

import ctypes
from typing import Mapping

import numpy as np
import torch

from . import _lib
from .adapters import PositionSchedule
from .batch import ForwardBatch, Phase, mask_uniform
from .errors import BatchError, ConfigError, InfeasibleBatchError, StateError

__all__ = ["BatchMeta", "default_meta", "pack_entries", "validate_arrays"]


def validate_arrays(qsl: np.ndarray, slots: np.ndarray, flags: np.ndarray) -> None:
    """Host check of raw K1 arrays, the same rules K1 enforces on the device
    (query_start_loc a strictly increasing prefix sum from 0, model.py:250-258;
    one slot and one flag word per entry; known flag bits only)."""
    qsl = np.asarray(qsl)
    E = len(slots)
    if qsl.ndim != 1 or len(qsl) != E + 1 or len(flags) != E:
        raise BatchError(f"query_start_loc has {len(qsl)} offsets, slots {E}, flags {len(flags)}")
    if int(qsl[0]) != 0:
        raise BatchError("query_start_loc must start at 0")
    if E and not bool(np.all(np.diff(qsl.astype(np.int64)) > 0)):
        raise BatchError("query_start_loc must be strictly increasing (every entry has >= 1 token)")
    fl = np.asarray(flags)
    if E and int(np.bitwise_or.reduce(fl.astype(np.int64))) & ~(_lib.ENTRY_DECODE | _lib.ENTRY_ALL_POSITIONS):
        raise BatchError("unknown entry flag bits")
    if E and int(np.min(np.asarray(slots))) < -1:
        raise BatchError("slot must be >= 0, or -1 for an adapter-less entry")


def pack_entries(batch: ForwardBatch, slot_of: Mapping[int, int]) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(query_start_loc int32[E+1], slot int32[E], flags int32[E]) for K1.

    An entry whose adapter is not registered raises BatchError, as
    forward_chunk does for ids missing from the catalogue (model.py:470-472).
    """
    E = len(batch.entries)
    qsl = np.asarray(batch.query_start_loc, dtype=np.int32)
    slots = np.full(E, -1, dtype=np.int32)
    flags = np.zeros(E, dtype=np.int32)
    for i, e in enumerate(batch.entries):
        if e.adapter_id is not None:
            s = slot_of.get(e.adapter_id)
            if s is None:
                raise BatchError(f"adapter {e.adapter_id} not in catalogue")
            slots[i] = s
        f = 0
        if e.phase is Phase.DECODE:
            f |= _lib.ENTRY_DECODE
        if e.schedule is PositionSchedule.ALL_POSITIONS:
            f |= _lib.ENTRY_ALL_POSITIONS
        flags[i] = f
    return qsl, slots, flags


class BatchMeta:
    """Fixed-capacity device workspace for one in-flight step."""

    def __init__(self, max_entries: int, max_tokens: int, tile_tokens: int = 128, device=None):
        if not 1 <= max_entries <= _lib.MAX_ENTRIES:
            raise InfeasibleBatchError(f"max_entries must be in [1, {_lib.MAX_ENTRIES}], got {max_entries}")
        if max_tokens < 1 or tile_tokens < 1:
            raise InfeasibleBatchError("max_tokens and tile_tokens must be >= 1")
        self.device = _lib.require_cuda(device)
        lib = _lib.load()
        self.E_cap = int(max_entries)
        self.T_cap = int(max_tokens)
        self.tile_tokens = int(tile_tokens)
        self.tile_cap = self.E_cap + self.T_cap // self.tile_tokens + 1
        self.chunk_cap = self.E_cap + self.T_cap // _lib.CHUNK_ROWS + 1
        words = int(lib.preft_meta_entries_words(self.E_cap))
        i32 = dict(dtype=torch.int32, device=self.device)
        self.entries = torch.zeros(words, **i32)
        self.mask = torch.zeros(self.T_cap, dtype=torch.uint8, device=self.device)
        self.tokens = torch.zeros(2 * self.T_cap, **i32)
        self.segments = torch.zeros(3 * self.E_cap, **i32)
        self.tiles = torch.zeros(4 * self.tile_cap, **i32)
        self.entry_offset = torch.zeros(self.E_cap, **i32)
        self.chunks = torch.zeros(2 * self.chunk_cap, **i32)
        # 4 ints per unit + the LoRA units' size order that K1 appends (PREFT_META_UNIT_ORDER)
        self.units = torch.zeros(5 * self.chunk_cap, **i32)
        self.counters = torch.zeros(_lib.NUM_COUNTERS, **i32)
        self.host = torch.zeros(words, dtype=torch.int32, pin_memory=True)
        self._host_np = self.host.numpy()
        self._staged = None  # event: the last H2D from `host` has been consumed
        self.c = _lib.PreftMeta(
            self.entries.data_ptr(),
            self.mask.data_ptr(),
            self.tokens.data_ptr(),
            self.segments.data_ptr(),
            self.tiles.data_ptr(),
            self.entry_offset.data_ptr(),
            self.counters.data_ptr(),
            self.E_cap,
            self.T_cap,
            self.tile_cap,
            self.tile_tokens,
            _lib.SLOT_SPLIT_ALL_LORA,
            0,
            self.chunks.data_ptr(),
            self.units.data_ptr(),
            self.chunk_cap,
            _lib.META_UNIT_ORDER,
            None,
            0,
        )
        self.lora_part: torch.Tensor | None = None
        self.E = 0
        self.T = 0
        self.uniform: bool | None = None
        # slot_split in force when K1 last ran: K1 bakes the LoRA/ReFT token
        # split into counters[SPLIT], so every launch that consumes this
        # metadata must use a pool with the same split (require_split)
        self.built_split: int | None = None

    @property
    def h2d_bytes(self) -> int:
        return 4 * (2 + (self.E + 1) + 2 * self.E)

    def fits(self, n_entries: int, n_tokens: int) -> bool:
        return n_entries <= self.E_cap and n_tokens <= self.T_cap

    # ------------------------------------------------------------ build
    def build(self, batch: ForwardBatch, slot_of: Mapping[int, int], stream: torch.cuda.Stream | None = None,
              slot_split: int | None = None):
        """Stage a ForwardBatch and launch K1 on `stream` (default: current).
        `slot_split`: the pool's first ReFT slot (AdapterPool.slot_split)."""
        qsl, slots, flags = pack_entries(batch, slot_of)
        self.uniform = mask_uniform(batch)
        return self.build_arrays(qsl, slots, flags, stream, slot_split=slot_split)

    def ensure_lora_part(self) -> None:
        """Attach the zeroed f32 workspace of the tensor-core LoRA split: the
        rank-r intermediate P [T_cap][<= 64] and the shrink's partial planes
        and per-unit arrival counters (preft_lora_part_floats; allocated once,
        fixed address, so plans and captured graphs stay valid)."""
        if self.lora_part is None:
            n = int(_lib.load().preft_lora_part_floats(ctypes.byref(self.c)))
            self.lora_part = torch.zeros(max(n, self.T_cap * 64), dtype=torch.float32, device=self.device)
            self.c.lora_part = self.lora_part.data_ptr()
            self.c.lora_part_floats = self.lora_part.numel()

    def set_slot_split(self, split: int) -> None:
        """First ReFT-class slot (AdapterPool.slot_split) for the NEXT K1 run;
        LoRA slots lie below it.  Changing it after a build does not re-split
        the built metadata (require_split catches the mismatch)."""
        self.c.slot_split = int(split)

    def require_split(self, split: int) -> None:
        """Raise unless K1 last ran with this slot split (pool.slot_split)."""
        if self.built_split is None:
            raise StateError("batch metadata has not been built (BatchMeta.build / build_arrays)")
        if self.built_split != int(split) or int(self.c.slot_split) != self.built_split:
            raise ConfigError(
                f"batch metadata was built with slot_split {self.built_split}, the pool's is {split}: "
                "rebuild it with slot_split=pool.slot_split (or pool.build_meta)"
            )

    def build_arrays(self, qsl: np.ndarray, slots: np.ndarray, flags: np.ndarray, stream=None,
                     slot_split: int | None = None, validate: bool = True):
        """Stage raw int32 arrays (qsl[E+1], slot[E], flags[E]) and launch K1.

        With `validate` (the default) the arrays are checked on the host the
        way make_batch checks a ForwardBatch (model.py:250-261): a malformed
        batch raises BatchError here instead of reaching K1, whose device
        error bits would otherwise only surface at the next check_errors()."""
        E = int(len(slots))
        T = int(qsl[-1]) if E else 0
        if E < 1:
            raise BatchError("batch must contain at least one entry")
        if not self.fits(E, T):
            raise InfeasibleBatchError(
                f"batch of {E} entries / {T} tokens exceeds the workspace ({self.E_cap} / {self.T_cap})"
            )
        if validate:
            validate_arrays(qsl, slots, flags)
        if slot_split is not None:
            self.set_slot_split(slot_split)
        if self._staged is not None:
            self._staged.synchronize()  # never overwrite a pinned buffer still being copied
        h = self._host_np
        h[0] = E
        h[1] = T
        h[2 : 3 + E] = qsl
        h[3 + E : 3 + 2 * E] = slots
        h[3 + 2 * E : 3 + 3 * E] = flags
        n = 3 + 3 * E
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            self.entries[:n].copy_(self.host[:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s)
            self._staged = ev
        self.c.rows_hint = T  # launch-shape hint for K2 (team size); results never depend on it
        _lib.check(_lib.load().preft_meta_build(ctypes.byref(self.c), ctypes.c_void_p(s.cuda_stream)), "meta_build")
        self.built_split = int(self.c.slot_split)
        self.E, self.T = E, T
        return self

    def launch(self, stream=None):
        """Re-run K1 on whatever is in `entries` (graph replay helper)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.check(_lib.load().preft_meta_build(ctypes.byref(self.c), ctypes.c_void_p(s.cuda_stream)), "meta_build")
        self.built_split = int(self.c.slot_split)

    # ------------------------------------------------------------ readback (syncs)
    def counters_host(self) -> np.ndarray:
        return self.counters.cpu().numpy()

    def check_errors(self) -> None:
        err = int(self.counters_host()[_lib.CTR_ERR])
        if err & (_lib.META_ERR_E_RANGE | _lib.META_ERR_T_RANGE | _lib.META_ERR_QSL):
            raise BatchError(f"device rejected the batch metadata (error bits {err:#x})")
        if err & (_lib.META_ERR_TILES | _lib.META_ERR_UNITS):
            raise InfeasibleBatchError("work list exceeded the tile / chunk capacity")

    def mask_host(self) -> np.ndarray:
        self.check_errors()
        return self.mask[: self.T].cpu().numpy().astype(bool)

    def selected_tokens(self) -> int:
        return int(self.counters_host()[_lib.CTR_SEL_TOKENS])

    def tokens_host(self) -> np.ndarray:
        n = self.selected_tokens()
        return self.tokens[: 2 * n].view(n, 2).cpu().numpy()

    def segments_host(self) -> np.ndarray:
        n = int(self.counters_host()[_lib.CTR_SEGMENTS])
        return self.segments[: 3 * n].view(n, 3).cpu().numpy()

    def tiles_host(self) -> np.ndarray:
        n = int(self.counters_host()[_lib.CTR_TILES])
        return self.tiles[: 4 * n].view(n, 4).cpu().numpy()

    def chunks_host(self) -> np.ndarray:
        n = int(self.counters_host()[_lib.CTR_CHUNKS])
        return self.chunks[: 2 * n].view(n, 2).cpu().numpy()

    def unit_order_host(self) -> np.ndarray:
        """The LoRA-class units in size order (largest first), as K1 appends them."""
        n = int(self.counters_host()[_lib.CTR_LORA_UNITS])
        return self.units[4 * self.chunk_cap: 4 * self.chunk_cap + n].cpu().numpy()

    def units_host(self) -> np.ndarray:
        n = int(self.counters_host()[_lib.CTR_UNITS])
        return self.units[: 4 * n].view(n, 4).cpu().numpy()

    def entry_offset_host(self) -> np.ndarray:
        return self.entry_offset[: self.E].cpu().numpy()


_DEFAULT: dict[int, BatchMeta] = {}


def default_meta(n_entries: int, n_tokens: int, device=None) -> BatchMeta:
    """Per-device scratch workspace for the reference-shaped API (grows as needed)."""
    dev = _lib.require_cuda(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    cur = _DEFAULT.get(idx)
    if cur is None or not cur.fits(n_entries, n_tokens):
        E = max(n_entries, 64 if cur is None else cur.E_cap)
        T = max(n_tokens, 4096 if cur is None else cur.T_cap)
        if E > _lib.MAX_ENTRIES:
            raise InfeasibleBatchError(f"{n_entries} entries exceed the device limit {_lib.MAX_ENTRIES}")
        cur = BatchMeta(min(_lib.MAX_ENTRIES, max(E, 1)), T, device=torch.device("cuda", idx))
        _DEFAULT[idx] = cur
    return cur
