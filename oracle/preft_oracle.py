"""CPU ORACLE of the PreFT hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (its `cpu_baseline` leg and
`--impl reference`) may import this module, and only as the checker / the
timed CPU baseline.  The product package (paper_2605_14217_b200) never
imports it; its compute paths fail loudly without the CUDA library.

This is a numpy float64 restatement of the reference `prefillsim` hot path
(/root/reference is not available on the GPU box).  Every function cites the
reference lines it follows.  Parity is PINNED: tests/test_oracle_golden.py
checks it against golden vectors produced by the reference itself
(tests/golden/make_golden.py imports prefillsim from /root/reference and
records its outputs), and tests/test_reference_live.py re-checks against the
live reference whenever /root/reference is mounted.

Entry encoding used throughout (one element per SeqEntry, model.py:223-242):
    qsl        int[E+1]  query_start_loc (model.py:248, make_batch :271-277)
    adapter    int[E]    adapter id, -1 for None
    is_decode  bool[E]   phase is DECODE
    all_pos    bool[E]   schedule is ALL_POSITIONS
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "position_mask",
    "enumerate_mask",
    "group_by_slot",
    "delta_rows",
    "apply_masked",
    "lora_hook",
    "reft_hook",
    "scaling_prefactor",
]


# ---------------------------------------------------------------- masks


def position_mask(qsl, adapter, is_decode, all_pos) -> np.ndarray:
    """compute_position_mask, model.py:305-319.

    values[span(i)] = True iff entry i has an adapter and (it is a prefill
    chunk or its schedule is ALL_POSITIONS).
    """
    qsl = np.asarray(qsl)
    values = np.zeros(int(qsl[-1]), dtype=bool)
    for i in range(len(adapter)):
        if adapter[i] < 0:  # model.py:314-315
            continue
        covered = (not is_decode[i]) or bool(all_pos[i])  # model.py:316
        if covered:
            values[qsl[i] : qsl[i + 1]] = True  # model.py:317-318
    return values


def enumerate_mask(qsl, adapter, is_decode, all_pos, prompt_len, cache_start) -> np.ndarray:
    """Independent per-token oracle, tests/test_model.py:143-157.

    Walks every token, computes its absolute position from the cache length
    and tests schedule membership directly (pos < prompt_len for prompt-only
    schedules).  Agrees with position_mask on every valid batch.
    """
    out = []
    for i in range(len(adapter)):
        for j in range(int(qsl[i + 1] - qsl[i])):
            pos = cache_start[i] + j
            if adapter[i] < 0:
                out.append(False)
            elif all_pos[i]:
                out.append(True)
            else:
                out.append(pos < prompt_len[i])
    return np.asarray(out, dtype=bool)


def uniform(values: np.ndarray):
    """PositionMask.uniform, model.py:296-302."""
    if values.all():
        return True
    if not values.any():
        return False
    return None


# ---------------------------------------------------------------- grouping (K1 contract)


def group_by_slot(qsl, slot, is_decode, all_pos, tile_tokens: int, slot_split: int = 2**31 - 1):
    """Restatement of K1's grouping contract (no reference counterpart).

    The reference applies adapters entry by entry (model.py:506-546); the
    device groups the SELECTED tokens by adapter slot first.  Contract:
      tokens    (n_sel, 2) int: (token index, slot), entries stably sorted by
                slot (ties keep batch order), each entry's tokens in order
      segments  (nseg, 3) int: (slot, first sorted position, length), one per
                distinct slot
      tiles     (ntiles, 4) int: (slot, first position, n tokens <= tile_tokens,
                segment id), covering every segment in order
      offsets   (E,) int: sorted position of each entry's first token or -1
      split     number of selected tokens whose slot < slot_split
    """
    qsl = np.asarray(qsl, dtype=np.int64)
    E = len(slot)
    sel = [slot[i] >= 0 and ((not is_decode[i]) or bool(all_pos[i])) for i in range(E)]
    order = sorted((i for i in range(E) if sel[i]), key=lambda i: (int(slot[i]), i))
    tokens = []
    offsets = np.full(E, -1, dtype=np.int64)
    for i in order:
        offsets[i] = len(tokens)
        for t in range(qsl[i], qsl[i + 1]):
            tokens.append((int(t), int(slot[i])))
    tokens = np.asarray(tokens, dtype=np.int64).reshape(-1, 2)
    segments = []
    for pos, (t, s) in enumerate(tokens):
        if pos == 0 or tokens[pos - 1][1] != s:
            segments.append([s, pos, 0])
        segments[-1][2] += 1
    segments = np.asarray(segments, dtype=np.int64).reshape(-1, 3)
    tiles = []
    for sid, (s, b, n) in enumerate(segments):
        for k in range(0, n, tile_tokens):
            tiles.append((s, b + k, min(tile_tokens, n - k), sid))
    tiles = np.asarray(tiles, dtype=np.int64).reshape(-1, 4)
    split = int(sum(1 for _, s in tokens if s < slot_split))
    return tokens, segments, tiles, offsets, split


def chunk_units(qsl, slot, is_decode, all_pos, chunk_rows: int = 16, unit_chunks: int = 4):
    """Restatement of K1's chunk/unit contract for the tensor-core ReFT kernel.

      chunks  (nchunks, 2) int: (first row, n rows <= chunk_rows): each selected
              entry, in the stable slot order of group_by_slot, cut into runs of
              consecutive rows starting at the entry's first row
      units   (nunits, 4) int: (slot, first chunk, n chunks <= unit_chunks, 0):
              the chunks of each slot's segment taken unit_chunks at a time
    """
    qsl = np.asarray(qsl, dtype=np.int64)
    E = len(slot)
    sel = [slot[i] >= 0 and ((not is_decode[i]) or bool(all_pos[i])) for i in range(E)]
    order = sorted((i for i in range(E) if sel[i]), key=lambda i: (int(slot[i]), i))
    chunks, seg_first = [], []
    for j, i in enumerate(order):
        if j == 0 or slot[order[j - 1]] != slot[i]:
            seg_first.append((int(slot[i]), len(chunks)))
        for r in range(int(qsl[i]), int(qsl[i + 1]), chunk_rows):
            chunks.append((r, min(chunk_rows, int(qsl[i + 1]) - r)))
    units = []
    for k, (s, c0) in enumerate(seg_first):
        c1 = seg_first[k + 1][1] if k + 1 < len(seg_first) else len(chunks)
        for c in range(c0, c1, unit_chunks):
            units.append((s, c, min(unit_chunks, c1 - c), 0))
    return (np.asarray(chunks, dtype=np.int64).reshape(-1, 2), np.asarray(units, dtype=np.int64).reshape(-1, 4))


# ---------------------------------------------------------------- adapter math


def scaling_prefactor(kind: str, value: float, rank: int) -> float:
    """adapters.py:109-117"""
    if kind == "constant":
        return value
    if kind == "alpha_over_r":
        return value / rank
    return 1.0 / np.sqrt(rank)


def delta_rows(kind: str, s: float, rows, A=None, B=None, b=None, R=None, W=None) -> np.ndarray:
    """delta_for_rows, adapters.py:278-295 (float64, same operation order).

    lora   s * ((X A^T) B^T)            A (r, m), B (n, r)      :284-288
    direft s * ((H A^T + b) B)          A, B (r, d), b (r,)     :292-293
    loreft s * ((H W^T + b - H R^T) R)  R, W (r, d), b (r,)     :294-295
    """
    rows = np.asarray(rows, dtype=np.float64)
    if kind == "lora":
        return s * ((rows @ A.T) @ B.T)
    if kind == "direft":
        return s * ((rows @ A.T + b) @ B)
    proj = rows @ R.T
    return s * ((rows @ W.T + b - proj) @ R)


def apply_masked(kind, s, schedule_all: bool, outputs, inputs, prompt_len, **params) -> np.ndarray:
    """apply_masked, adapters.py:298-333: copy, cut = total or min(p, total),
    out[:cut] += delta(src[:cut]) with src = inputs (lora) or outputs (reft)."""
    out = np.array(outputs, dtype=np.float64, copy=True)
    total = out.shape[0]
    cut = total if schedule_all else min(prompt_len, total)
    if cut == 0:
        return out
    src = np.asarray(inputs, dtype=np.float64) if kind == "lora" else out
    out[:cut] += delta_rows(kind, s, src[:cut], **params)
    return out


def lora_hook(y, x, qsl, mask, entry_slot, slot_params) -> np.ndarray:
    """The LoRA hook of forward_chunk for one site: `_project` per entry,
    model.py:442-452 with rows = mask[span] (model.py:509), i.e.
    out[rows] += delta_for_rows(site, x[rows]) entry by entry.

    slot_params[slot] = dict(kind="lora", s=..., A=..., B=...)
    """
    out = np.array(y, dtype=np.float64, copy=True)
    x = np.asarray(x, dtype=np.float64)
    for i in range(len(entry_slot)):
        if entry_slot[i] < 0:
            continue
        sl = slice(int(qsl[i]), int(qsl[i + 1]))
        rows = mask[sl]
        if not rows.any():
            continue
        p = slot_params[int(entry_slot[i])]
        blk = out[sl]
        blk[rows] += delta_rows(p["kind"], p["s"], x[sl][rows], A=p["A"], B=p["B"])
        out[sl] = blk
    return out


def reft_hook(h, qsl, mask, entry_slot, slot_params) -> np.ndarray:
    """The residual-stream hook of forward_chunk, model.py:543-546:
    block[rows] += delta_for_rows(site, block[rows]) entry by entry."""
    out = np.array(h, dtype=np.float64, copy=True)
    for i in range(len(entry_slot)):
        if entry_slot[i] < 0:
            continue
        sl = slice(int(qsl[i]), int(qsl[i + 1]))
        rows = mask[sl]
        if not rows.any():
            continue
        p = slot_params[int(entry_slot[i])]
        blk = out[sl]
        kw = {k: p[k] for k in ("A", "B", "b", "R", "W") if k in p}
        blk[rows] += delta_rows(p["kind"], p["s"], blk[rows], **kw)
        out[sl] = blk
    return out
