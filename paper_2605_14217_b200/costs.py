"""Algorithmic bytes and flops of the hot path — the accounting behind every
roofline fraction bench.py reports, written next to the
reference's own cost model so the two can be reconciled
(tests/test_costs.py against costmodel.py:139-249).

Per launch, with e = element bytes of the activations (2 bf16, 4 f32),
e_w = stored weight bytes, T_p = selected tokens, D = distinct adapters:

  LoRA^P group (sites s sharing x, m -> n_s):
      bytes = T_p e (m + 2 sum n_s)  +  D e_w r sum (m + n_s)
      flops = T_p sum 2 r (m + n_s)
  ReFT^P residual site (width d):
      bytes = T_p e 2 d  +  D (e_w 2 r d + 4 r)     (bias in fp32)
      flops = T_p 4 r d                              (DiReFT, and LoReFT after
                                                      the W - R fold)
  tensor-parallel split (config 4), per rank: the sharded widths m_loc /
      n_loc, plus the rank-r partials P written by the shrink and read by
      the expand, 2 T_p 4 r per site.

How this differs from costmodel.py (each difference is pinned by a test):
  * sites: costmodel uses the square-projection approximation
    site_params = 2 r d (costmodel.py:163-169); we use the real (n, m) of
    each Llama-3.1 site, GQA k/v included.  With square sites the weight
    bytes and the flops are identical.
  * activations: costmodel charges every distinct adapter a masked pass over
    the WHOLE step, 2 step_tokens d bpp per adapter (costmodel.py:17-19,
    241-246).  The segmented kernels read each selected token's x once and
    read + write its y once, independent of D: T_p e (m + 2n).  That is the
    inefficiency the grouping removes; for D = 1 ours is 3/2 of theirs (the
    y read of the in-place add, which costmodel does not count).
  * dispatch overhead: costmodel adds adapter_op_overhead_s * bandwidth per
    (adapter, site) (costmodel.py:246); one launch covers every adapter here,
    so no such term exists in the algorithmic bytes (launch cost shows up in
    the measured time instead).
  * ReFT bias: costmodel counts r bias parameters at bpp and 2 r flops per
    token for them; we store the bias in fp32 (4 r bytes) and fold it into
    the rank-r intermediate (no separate flops counted).
"""

from __future__ import annotations

from typing import Mapping, Sequence

__all__ = [
    "lora_group_bytes",
    "lora_group_flops",
    "lora_weight_bytes",
    "reft_bytes",
    "reft_flops",
    "split_group_bytes",
    "lora_layer_params",
    "reft_layer_params",
]


def lora_weight_bytes(dims: Mapping[str, tuple[int, int]], group: Sequence[str], rank: int, elem_w: int = 2) -> int:
    """One adapter's A and B rows for the sites of a group (read once per launch)."""
    m = dims[group[0]][1]
    return elem_w * rank * sum(m + dims[s][0] for s in group)


def lora_group_bytes(dims: Mapping[str, tuple[int, int]], group: Sequence[str], n_tokens: int, distinct: int,
                     rank: int, elem: int = 2, elem_w: int | None = None) -> int:
    """x read once, every y read + written, each distinct adapter's weights once."""
    m = dims[group[0]][1]
    act = n_tokens * elem * (m + 2 * sum(dims[s][0] for s in group))
    return act + distinct * lora_weight_bytes(dims, group, rank, elem if elem_w is None else elem_w)


def lora_group_flops(dims: Mapping[str, tuple[int, int]], group: Sequence[str], n_tokens: int, rank: int) -> int:
    m = dims[group[0]][1]
    return n_tokens * sum(2 * rank * (m + dims[s][0]) for s in group)


def reft_bytes(d: int, n_tokens: int, distinct: int, rank: int, elem: int = 2, elem_w: int | None = None) -> int:
    ew = elem if elem_w is None else elem_w
    return n_tokens * elem * 2 * d + distinct * (ew * 2 * rank * d + 4 * rank)


def reft_flops(d: int, n_tokens: int, rank: int) -> int:
    return n_tokens * 4 * rank * d


def split_group_bytes(m_loc: int, n_locs: Sequence[int], n_tokens: int, distinct: int, rank: int,
                      elem: int = 2) -> int:
    """Per rank, one shrink + expand pair of a tensor-parallel group."""
    act = n_tokens * elem * (m_loc + 2 * sum(n_locs))
    wts = distinct * elem * rank * sum(m_loc + n for n in n_locs)
    part = 2 * n_tokens * 4 * rank * len(n_locs)
    return act + wts + part


def lora_layer_params(dims: Mapping[str, tuple[int, int]], rank: int) -> int:
    """Parameters of one LoRA adapter in one layer over all 7 target sites."""
    return sum(rank * (n + m) for n, m in dims.values())


def reft_layer_params(d: int, rank: int) -> int:
    """DiReFT A (r, d), B (r, d), b (r) — adapters.py:159-179."""
    return 2 * rank * d + rank
