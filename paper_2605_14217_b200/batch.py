"""Batch metadata + adapter catalogue API — drop-in for the hot-path half of
pkg/src/prefillsim/model.py (model.py:62-67, 223-413).

`SeqEntry`, `ForwardBatch`, `make_batch`, `PositionMask`, `ModelAdapter`,
`build_adapter` and `perturb_adapter` keep the reference's fields, validation
and exceptions.  `compute_position_mask` runs K1 (the device metadata builder)
and reads its mask back, so its result is the device's, bit-exact with
model.py:305-319.  The toy transformer itself (attention/MLP, KvCache,
generate) is not part of the hot path and is not rebuilt here.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from .adapters import AdapterKind, AdapterParams, PositionSchedule, ScalingRule, init_zero_delta
from .errors import BatchError, ConfigError
from .linalg import rng_from_seed

__all__ = [
    "LORA_TARGETS",
    "Phase",
    "ModelConfig",
    "SeqEntry",
    "ForwardBatch",
    "PositionMask",
    "ModelAdapter",
    "make_batch",
    "compute_position_mask",
    "mask_uniform",
    "build_adapter",
    "perturb_adapter",
]

LORA_TARGETS = ("Wq", "Wk", "Wv", "Wo", "Wgate", "Wup", "Wdown")


class Phase(enum.Enum):
    """model.py:65-67"""

    PREFILL = "prefill"
    DECODE = "decode"


@dataclass(frozen=True)
class ModelConfig:
    """Toy-model shape used by build_adapter (model.py:70-93); ffn = 2 * d_model."""

    d_model: int
    n_layers: int
    vocab: int
    seed: int
    max_seq: int = 512
    ablate_attention: bool = False
    lora_targets: tuple[str, ...] = LORA_TARGETS

    def __post_init__(self) -> None:
        if self.d_model < 1 or self.n_layers < 1 or self.vocab < 2:
            raise ConfigError("d_model, n_layers >= 1 and vocab >= 2 required")
        if self.max_seq < 2:
            raise ConfigError("max_seq must be at least 2")
        bad = set(self.lora_targets) - set(LORA_TARGETS)
        if bad:
            raise ConfigError(f"unknown lora targets: {sorted(bad)}")

    @property
    def ffn_dim(self) -> int:
        return 2 * self.d_model

    def site_dims(self) -> dict[str, tuple[int, int]]:
        """(n, m) per LoRA target, model.py:358-366."""
        d, f = self.d_model, self.ffn_dim
        return {"Wq": (d, d), "Wk": (d, d), "Wv": (d, d), "Wo": (d, d), "Wgate": (f, d), "Wup": (f, d), "Wdown": (d, f)}


@dataclass(frozen=True)
class SeqEntry:
    """One sequence's contribution to a step (model.py:223-242)."""

    seq_id: int
    tokens: tuple[int, ...]
    prompt_len: int
    phase: Phase
    adapter_id: int | None = None
    schedule: PositionSchedule | None = None

    def __post_init__(self) -> None:
        if self.prompt_len < 1:
            raise BatchError(f"prompt_len must be >= 1, got {self.prompt_len}")
        if not self.tokens:
            raise BatchError("entry carries no tokens")
        if self.phase is Phase.DECODE and len(self.tokens) != 1:
            raise BatchError("decode entries carry exactly one token")
        if self.adapter_id is not None and self.schedule is None:
            raise BatchError("adapter without a position schedule")


@dataclass(frozen=True)
class ForwardBatch:
    """Entries + query_start_loc prefix sum (model.py:245-268)."""

    entries: tuple[SeqEntry, ...]
    query_start_loc: tuple[int, ...]

    def __post_init__(self) -> None:
        offs = self.query_start_loc
        if len(offs) != len(self.entries) + 1 or offs[0] != 0:
            raise BatchError("query_start_loc must be a prefix-sum starting at 0")
        for i, entry in enumerate(self.entries):
            if offs[i + 1] - offs[i] != len(entry.tokens):
                raise BatchError(f"offsets disagree with token span of entry {i}")
        if any(b <= a for a, b in zip(offs, offs[1:])):
            raise BatchError("query_start_loc must be strictly increasing")
        seqs = [e.seq_id for e in self.entries]
        if len(set(seqs)) != len(seqs):
            raise BatchError("a sequence may appear at most once per batch")

    @property
    def total_tokens(self) -> int:
        return self.query_start_loc[-1]

    def span(self, i: int) -> slice:
        return slice(self.query_start_loc[i], self.query_start_loc[i + 1])


def make_batch(entries: Sequence[SeqEntry]) -> ForwardBatch:
    """model.py:271-277"""
    if not entries:
        raise BatchError("batch must contain at least one entry")
    offs = [0]
    for e in entries:
        offs.append(offs[-1] + len(e.tokens))
    return ForwardBatch(tuple(entries), tuple(offs))


@dataclass(frozen=True)
class PositionMask:
    """Boolean mask over the flattened query tokens (model.py:280-302)."""

    values: np.ndarray

    def __post_init__(self) -> None:
        vals = np.asarray(self.values, dtype=bool)
        object.__setattr__(self, "values", vals)
        vals.flags.writeable = False

    @property
    def uniform(self) -> bool | None:
        if bool(self.values.all()):
            return True
        if not bool(self.values.any()):
            return False
        return None


def entry_selected(entry: SeqEntry) -> bool:
    """model.py:314-316 (the rule K1 evaluates per entry on the device)."""
    if entry.adapter_id is None:
        return False
    return entry.phase is Phase.PREFILL or entry.schedule is PositionSchedule.ALL_POSITIONS


def mask_uniform(batch: ForwardBatch) -> bool | None:
    """PositionMask.uniform decided on the host in O(E), without a device sync.

    The all-False case is the paper's decode fast path: the runner skips the
    adapter launches entirely (model.py:475).
    """
    sel = [entry_selected(e) for e in batch.entries]
    if all(sel):
        return True
    if not any(sel):
        return False
    return None


def compute_position_mask(batch: ForwardBatch) -> PositionMask:
    """Device-computed PositionMask (K1), bit-exact with model.py:305-319."""
    from .meta import default_meta

    ids = sorted({e.adapter_id for e in batch.entries if e.adapter_id is not None})
    slot_of = {a: i for i, a in enumerate(ids)}
    meta = default_meta(len(batch.entries), batch.total_tokens)
    meta.build(batch, slot_of)
    return PositionMask(meta.mask_host())


# --------------------------------------------------------------- catalogue


@dataclass(frozen=True)
class ModelAdapter:
    """Catalogue entry with per-site bundles (model.py:325-339)."""

    adapter_id: int
    kind: AdapterKind
    rank: int
    schedule: PositionSchedule
    lora_sites: Mapping[tuple[int, str], AdapterParams] = field(default_factory=dict)
    reft_sites: tuple[AdapterParams, ...] = ()


def _site_seed(seed: int, index: int) -> int:
    """model.py:342-343"""
    return int(np.random.SeedSequence((seed, index)).generate_state(1)[0])


def build_adapter(
    config,
    adapter_id: int,
    kind: AdapterKind,
    rank: int,
    schedule: PositionSchedule,
    seed: int,
    scaling: ScalingRule | None = None,
) -> ModelAdapter:
    """Zero-delta adapter for every hook site (model.py:346-380).

    `config` is a ModelConfig (toy shapes, as in the reference) or any object
    with `n_layers`, `d_model`, `lora_targets` and `site_dims()` — e.g.
    shapes.LLAMA_8B for the Llama-3.1 projection shapes.
    """
    d = config.d_model
    if kind is AdapterKind.LORA:
        shapes = config.site_dims()
        sites = {}
        idx = 0
        for layer in range(config.n_layers):
            for name in config.lora_targets:
                sites[(layer, name)] = init_zero_delta(kind, rank, shapes[name], _site_seed(seed, idx), scaling)
                idx += 1
        return ModelAdapter(adapter_id, kind, rank, schedule, lora_sites=sites)
    reft = tuple(
        init_zero_delta(kind, rank, (d,), _site_seed(seed, layer), scaling) for layer in range(config.n_layers)
    )
    return ModelAdapter(adapter_id, kind, rank, schedule, reft_sites=reft)


def _perturbed_params(params: AdapterParams, seed: int, sigma: float) -> AdapterParams:
    """model.py:383-398"""
    g = rng_from_seed(seed)
    kw: dict[str, np.ndarray] = {}
    if params.kind is AdapterKind.LORA:
        kw["A"] = params.A
        kw["B"] = params.B + g.normal(0.0, sigma, size=params.B.shape)
    elif params.kind is AdapterKind.DIREFT:
        kw["A"] = params.A + g.normal(0.0, sigma, size=params.A.shape)
        kw["B"] = params.B
        kw["b"] = params.b + g.normal(0.0, sigma, size=params.b.shape)
    else:
        kw["R"] = params.R
        kw["W"] = params.W + g.normal(0.0, sigma, size=params.W.shape)
        kw["b"] = params.b + g.normal(0.0, sigma, size=params.b.shape)
    return AdapterParams(params.kind, params.rank, params.dims, params.scaling, **kw)


def perturb_adapter(adapter: ModelAdapter, seed: int, sigma: float = 0.1) -> ModelAdapter:
    """model.py:401-413"""
    if adapter.kind is AdapterKind.LORA:
        sites = {
            key: _perturbed_params(p, _site_seed(seed, i), sigma)
            for i, (key, p) in enumerate(sorted(adapter.lora_sites.items()))
        }
        return ModelAdapter(adapter.adapter_id, adapter.kind, adapter.rank, adapter.schedule, lora_sites=sites)
    reft = tuple(_perturbed_params(p, _site_seed(seed, i), sigma) for i, p in enumerate(adapter.reft_sites))
    return ModelAdapter(adapter.adapter_id, adapter.kind, adapter.rank, adapter.schedule, reft_sites=reft)
