"""ADP1 adapter files -> HBM pool bulk loader.

The reference stores one `AdapterParams` bundle per ADP1 file: little-endian
float64 tensors behind a small header (adapters.py:15-26, 391-436; restated
bit-exactly in `adapters.save_adapter` / `load_adapter`).  A served adapter is
a `ModelAdapter` (model.py:325-339): one bundle per (layer, LoRA site), or
one per layer for ReFT.  This module gives that a directory layout:

    <dir>/adapter.json                      {"adapter_id", "kind", "rank", "schedule",
                                             "sites": [[layer, site, file], ...]}
    <dir>/L<layer>_<site>.adp1              one ADP1 bundle per hook site

and loads whole catalogues of them.  `register_dir` reads every bundle of an
adapter and registers it in one call, which stages all of its sites into one
pinned float64 buffer, one H2D copy and one K4 conversion per slab
(`AdapterPool._upload_on`).  Bit-exactness: the files round-trip the float64
values exactly, so an adapter loaded from disk fills the pool with the same
bits as the in-memory bundle it was saved from.
"""

from __future__ import annotations

import json
from pathlib import Path
from typing import Mapping

from .adapters import AdapterKind, PositionSchedule, load_adapter, save_adapter
from .batch import ModelAdapter
from .errors import ShapeError

__all__ = ["save_model_adapter", "load_model_adapter", "load_catalogue", "register_dir"]

MANIFEST = "adapter.json"


def save_model_adapter(adapter: ModelAdapter, directory: str | Path) -> Path:
    """Write an adapter as a directory of ADP1 files plus a manifest."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    sites = []
    if adapter.kind is AdapterKind.LORA:
        for (layer, name), p in sorted(adapter.lora_sites.items()):
            f = f"L{layer}_{name}.adp1"
            save_adapter(p, d / f)
            sites.append([int(layer), name, f])
    else:
        for layer, p in enumerate(adapter.reft_sites):
            f = f"L{layer}_reft.adp1"
            save_adapter(p, d / f)
            sites.append([layer, "reft", f])
    manifest = {"format": "ADP1-dir/1", "adapter_id": int(adapter.adapter_id), "kind": adapter.kind.value,
                "rank": int(adapter.rank), "schedule": adapter.schedule.value, "sites": sites}
    (d / MANIFEST).write_text(json.dumps(manifest, indent=1))
    return d


def load_model_adapter(directory: str | Path) -> ModelAdapter:
    """Read a directory written by save_model_adapter (validates every bundle)."""
    d = Path(directory)
    try:
        m = json.loads((d / MANIFEST).read_text())
        kind = AdapterKind(m["kind"])
        schedule = PositionSchedule(m["schedule"])
        aid, rank, sites = int(m["adapter_id"]), int(m["rank"]), m["sites"]
    except (OSError, ValueError, KeyError) as exc:
        raise ShapeError(f"{d} is not an adapter directory: {exc}") from None
    bundles = {}
    for layer, name, f in sites:
        p = load_adapter(d / f)
        if p.kind is not kind or p.rank != rank:
            raise ShapeError(f"{d / f}: bundle kind/rank does not match the manifest")
        bundles[(int(layer), str(name))] = p
    if kind is AdapterKind.LORA:
        return ModelAdapter(aid, kind, rank, schedule, lora_sites=bundles)
    layers = sorted(layer for layer, _ in bundles)
    if layers != list(range(len(layers))):
        raise ShapeError(f"{d}: ReFT layers are not 0..L-1")
    return ModelAdapter(aid, kind, rank, schedule, reft_sites=tuple(bundles[(i, "reft")] for i in layers))


def load_catalogue(root: str | Path) -> dict[int, ModelAdapter]:
    """Every adapter directory under `root` (e.g. a paging catalogue)."""
    out: dict[int, ModelAdapter] = {}
    for man in sorted(Path(root).glob(f"*/{MANIFEST}")):
        a = load_model_adapter(man.parent)
        if a.adapter_id in out:
            raise ShapeError(f"adapter id {a.adapter_id} appears twice under {root}")
        out[a.adapter_id] = a
    return out


def register_dir(pool, directory: str | Path, stream=None) -> int:
    """Load one adapter directory and register it in the pool; returns its slot."""
    return pool.register(load_model_adapter(directory), stream)


def register_catalogue(pool, catalogue: Mapping[int, ModelAdapter], stream=None) -> list[int]:
    """Bulk registration (one staged upload per adapter)."""
    return [pool.register(a, stream) for _, a in sorted(catalogue.items())]
