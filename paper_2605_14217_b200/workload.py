"""Synthetic request streams (host-side input generator, not the hot path).

Restates pkg/src/prefillsim/workload.py:47-156 so the benchmark configs use
the reference's own request distribution on the GPU box (where the reference
is not installed): Punica prompt lengths p = rint(loc + scale*exp(sigma*z)),
sigma = 0.8, loc = -1, scale = 18, clipped to [1, l_max - 2]
(workload.py:110-116), totals uniform on [p + 2, l_max] (:119-125), adapter
mixes identical / uniform / skewed (Zipf 1/(k+1)) / distinct (:128-145), each
from its own named PCG64 sub-stream of the master seed (:51-55).  Same seeds
give the same arrays as the reference (pinned in tests/test_host_api.py).

Also: request -> GPU routing for the adapter-sharded multi-GPU layout
(SURVEY.md 8(e)): the owner of adapter a is `a mod world` unless it is hot
enough to be replicated.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .errors import ConfigError, DomainError
from .linalg import rng_from_seed

PROMPT_SIGMA = 0.8
PROMPT_LOC = -1.0
PROMPT_SCALE = 18.0
_STREAM_PROMPT = 1
_STREAM_TOTAL = 2
_STREAM_ADAPTER = 3
_STREAM_SHUFFLE = 4


class AdapterMix(enum.Enum):
    IDENTICAL = "identical"
    UNIFORM = "uniform"
    SKEWED = "skewed"
    DISTINCT = "distinct"


@dataclass(frozen=True)
class WorkloadConfig:
    n_requests: int
    n_adapters: int
    mix: AdapterMix
    seed: int
    l_max: int = 2048

    def __post_init__(self) -> None:
        if self.n_requests < 0 or self.n_adapters < 0:
            raise ConfigError("n_requests and n_adapters must be >= 0")
        if self.l_max < 4:
            raise ConfigError(f"l_max must be >= 4, got {self.l_max}")
        if self.seed < 0:
            raise ConfigError("seed must be non-negative")


def sample_prompt_lens(cfg: WorkloadConfig, size: int | None = None) -> np.ndarray:
    """workload.py:110-116"""
    n = cfg.n_requests if size is None else size
    z = rng_from_seed(cfg.seed, _STREAM_PROMPT).normal(size=n)
    raw = PROMPT_LOC + PROMPT_SCALE * np.exp(PROMPT_SIGMA * z)
    return np.clip(np.rint(raw), 1, cfg.l_max - 2).astype(np.int64)


def sample_total_lens(cfg: WorkloadConfig, prompt_lens: np.ndarray) -> np.ndarray:
    """workload.py:119-125"""
    prompt_lens = np.asarray(prompt_lens, dtype=np.int64)
    if np.any(prompt_lens > cfg.l_max - 2):
        raise DomainError("prompt length leaves no room for two output tokens")
    return rng_from_seed(cfg.seed, _STREAM_TOTAL).integers(prompt_lens + 2, cfg.l_max + 1)


def assign_adapters(cfg: WorkloadConfig) -> list[int | None]:
    """workload.py:128-145"""
    n, na = cfg.n_requests, cfg.n_adapters
    if na == 0:
        return [None] * n
    if cfg.mix is AdapterMix.IDENTICAL:
        ids = np.zeros(n, dtype=np.int64)
    elif cfg.mix is AdapterMix.UNIFORM:
        ids = rng_from_seed(cfg.seed, _STREAM_ADAPTER).integers(0, na, size=n)
    elif cfg.mix is AdapterMix.SKEWED:
        w = 1.0 / (np.arange(na, dtype=np.float64) + 1.0)
        ids = rng_from_seed(cfg.seed, _STREAM_ADAPTER).choice(na, size=n, p=w / w.sum())
    else:
        ids = np.arange(n, dtype=np.int64) % na
        ids = ids[rng_from_seed(cfg.seed, _STREAM_SHUFFLE).permutation(n)]
    return [int(i) for i in ids]


# ---------------------------------------------------------------- multi-GPU routing


def owner_of(adapter_id: int, world: int) -> int:
    """Home GPU of an adapter's pool slot (pool sharded by id)."""
    return adapter_id % world


def shard_adapters(n_adapters: int, rank: int, world: int) -> list[int]:
    return [a for a in range(n_adapters) if owner_of(a, world) == rank]


def route_requests(adapter_ids: Sequence[int | None], world: int, replicas: dict[int, Sequence[int]] | None = None,
                   lens: Sequence[int] | None = None) -> list[list[int]]:
    """Request indices per rank: each request goes to a GPU holding its adapter.

    Adapters listed in `replicas` (hot adapters copied to several GPUs, e.g.
    the Zipf head) go to the least-loaded replica holder by token count;
    adapter-less requests go to the least-loaded rank overall.  Routing is
    host-side and needs no collective on the data path.
    """
    replicas = replicas or {}
    load = [0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for i, a in enumerate(adapter_ids):
        w = 1 if lens is None else int(lens[i])
        if a is None:
            r = int(np.argmin(load))
        elif a in replicas:
            holders = list(replicas[a])
            r = holders[int(np.argmin([load[h] for h in holders]))]
        else:
            r = owner_of(a, world)
        out[r].append(i)
        load[r] += w
    return out


def hot_replicas(adapter_ids: Sequence[int | None], world: int, threshold: float = 0.5) -> dict[int, list[int]]:
    """Replicate adapters whose request share exceeds threshold / world on every GPU."""
    ids = [a for a in adapter_ids if a is not None]
    if not ids or world == 1:
        return {}
    vals, counts = np.unique(np.asarray(ids), return_counts=True)
    share = counts / len(ids)
    return {int(a): list(range(world)) for a, s in zip(vals, share) if s > threshold / world}
