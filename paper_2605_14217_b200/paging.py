"""Host <-> device adapter paging with LRU eviction.

The reference engine keeps at most `max_gpu_adapters` adapters on the device
and pages the rest in on demand, evicting the least recently used adapter
that the current step does not need (`AdapterPool.ensure`,
engine.py:200-244; hand trace tests/test_engine.py:127-137).  Here:

* `LruResidency` restates that bookkeeping exactly (same order of page-ins
  and evictions, same InfeasibleBatchError when a step needs more adapters
  than there are slots); it is pure Python, so the CPU tests check it against
  the reference's own hand trace and against the live reference.
* `PagedAdapterPool` applies those decisions to the HBM pool.  The first
  page-in of an adapter registers it from its float64 bundle (K4 conversion)
  and keeps a pinned host snapshot of the converted slot; every later page-in
  is a plain stream-ordered H2D copy of that snapshot into a free slot, and an
  eviction just frees the slot (the next page-in overwrites all of it).  Slabs
  never move, so captured graphs stay valid across paging.

Each adapter family (LoRA, ReFT) pages within its own slots; `capacity`
defaults to the pool's slot count for that family.
"""

from __future__ import annotations

from collections import OrderedDict
from typing import Mapping, Sequence

from .adapters import AdapterKind
from .batch import ModelAdapter
from .errors import ConfigError, InfeasibleBatchError, StateError

__all__ = ["LruResidency", "PagedAdapterPool"]


class LruResidency:
    """engine.py:200-244: resident ids in LRU order, capacity-bounded."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ConfigError("pool capacity must be >= 1")
        self.capacity = int(capacity)
        self._resident: OrderedDict[int, int] = OrderedDict()

    @property
    def resident_ids(self) -> tuple[int, ...]:
        return tuple(self._resident)

    def __contains__(self, adapter_id: int) -> bool:
        return adapter_id in self._resident

    def ensure(self, needed: Sequence[int], byte_size: Mapping[int, int]) -> tuple[list[int], list[int], int]:
        """Make every id in `needed` resident; returns (paged, evicted, bytes).

        Ids are processed in the given order and all of them are protected
        from eviction for the duration of the call (engine.py:216-244).
        """
        needed = list(dict.fromkeys(needed))
        if len(needed) > self.capacity:
            raise InfeasibleBatchError(f"step needs {len(needed)} adapters but the device holds {self.capacity}")
        paged: list[int] = []
        evicted: list[int] = []
        moved = 0
        pinned = set(needed)
        for aid in needed:
            if aid in self._resident:
                self._resident.move_to_end(aid)
                continue
            while len(self._resident) >= self.capacity:
                victim = next(a for a in self._resident if a not in pinned)
                del self._resident[victim]
                evicted.append(victim)
            self._resident[aid] = byte_size[aid]
            moved += byte_size[aid]
            paged.append(aid)
        return paged, evicted, moved


class PagedAdapterPool:
    """An `AdapterPool` fronted by a host catalogue larger than its slots."""

    def __init__(self, pool, catalogue: Mapping[int, ModelAdapter], lora_capacity: int | None = None,
                 reft_capacity: int | None = None, snapshots: Mapping[int, object] | None = None):
        self.pool = pool
        self.catalogue = dict(catalogue)
        self._kinds = {aid: a.kind for aid, a in self.catalogue.items()}
        for aid, snap in (snapshots or {}).items():  # pre-converted slot images (SlotSnapshot)
            self._kinds[aid] = snap.info.kind
        lc = pool.lora_capacity if lora_capacity is None else int(lora_capacity)
        rc = pool.reft_capacity if reft_capacity is None else int(reft_capacity)
        if lc > pool.lora_capacity or rc > pool.reft_capacity:
            raise ConfigError("paging capacity exceeds the pool's slots")
        self._lru = {True: LruResidency(lc) if lc else None, False: LruResidency(rc) if rc else None}
        self._snap: dict[int, object] = dict(snapshots or {})  # adapter id -> pinned SlotSnapshot
        self.paged_bytes = 0
        self.page_ins = 0
        self.evictions = 0

    def byte_size(self, adapter_id: int) -> int:
        """Device bytes of one adapter's slot (what a page-in moves)."""
        lora = self._kinds[adapter_id] is AdapterKind.LORA
        return self.pool.lora_slot_bytes if lora else self.pool.reft_slot_bytes

    @property
    def resident_ids(self) -> tuple[int, ...]:
        out = ()
        for lru in self._lru.values():
            if lru is not None:
                out += lru.resident_ids
        return out

    def ensure(self, needed: Sequence[int], stream=None) -> tuple[list[int], list[int], int]:
        """Make every adapter of the step resident (engine.py:412-418)."""
        for aid in needed:
            if aid not in self._kinds:
                raise StateError(f"adapter {aid} is not in the catalogue")
        paged, evicted, moved = [], [], 0
        for lora in (True, False):
            ids = [a for a in needed if (self._kinds[a] is AdapterKind.LORA) == lora]
            if not ids:
                continue
            lru = self._lru[lora]
            if lru is None:
                raise InfeasibleBatchError("the pool has no slots for this adapter family")
            sizes = {a: self.byte_size(a) for a in ids}
            p, e, m = lru.ensure(ids, sizes)
            for aid in e:
                self.pool.unregister(aid, zero=False)
            for aid in p:
                snap = self._snap.get(aid)
                if snap is None:  # first touch: convert from float64, keep the slot image
                    self.pool.register(self.catalogue[aid], stream)
                    self._snap[aid] = self.pool.export_slot(aid, stream)
                else:
                    self.pool.import_slot(snap, stream)
            paged += p
            evicted += e
            moved += m
        self.paged_bytes += moved
        self.page_ins += len(paged)
        self.evictions += len(evicted)
        return paged, evicted, moved

    def update(self, adapter_id: int, adapter: ModelAdapter, stream=None) -> None:
        """Weight sync for a paged catalogue: resident adapters are overwritten
        in place (AdapterPool.sync), non-resident ones on their next page-in."""
        self.catalogue[adapter_id] = adapter
        self._kinds[adapter_id] = adapter.kind
        self._snap.pop(adapter_id, None)
        if adapter_id in self.pool:
            self.pool.sync([(adapter_id, adapter)], stream)
            self._snap[adapter_id] = self.pool.export_slot(adapter_id, stream)
