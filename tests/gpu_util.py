"""Helpers for the GPU parity tests: random mixed batches, pools built from
golden/oracle parameters, and oracle evaluation on exactly the values that
sit in the device pool (so bf16/fp32 inputs are identical on both sides)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import preft_oracle as O
from paper_2605_14217_b200 import _lib
from paper_2605_14217_b200.adapters import AdapterKind, AdapterParams, PositionSchedule, ScalingRule
from paper_2605_14217_b200.batch import ModelAdapter

SCHED = PositionSchedule


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().to(torch.float64).cpu().numpy()


def random_entries(rng, n_entries, adapter_ids, max_len=40, p_decode=0.35, p_none=0.1, p_all=0.25, lens=None):
    """(qsl, adapter_ids list (None allowed), flags int32) of a random mixed batch."""
    qsl = [0]
    ids, flags = [], []
    for i in range(n_entries):
        dec = rng.random() < p_decode
        n = 1 if dec else (int(lens[i]) if lens is not None else int(rng.integers(1, max_len + 1)))
        aid = None if (rng.random() < p_none or not adapter_ids) else int(adapter_ids[int(rng.integers(0, len(adapter_ids)))])
        allp = rng.random() < p_all
        f = (_lib.ENTRY_DECODE if dec else 0) | (_lib.ENTRY_ALL_POSITIONS if allp else 0)
        qsl.append(qsl[-1] + n)
        ids.append(aid)
        flags.append(f)
    return np.asarray(qsl, dtype=np.int32), ids, np.asarray(flags, dtype=np.int32)


def oracle_mask(qsl, slots, flags):
    return O.position_mask(qsl, slots, (flags & _lib.ENTRY_DECODE) != 0, (flags & _lib.ENTRY_ALL_POSITIONS) != 0)


def stage(meta, pool, qsl, ids, flags):
    slots = pool.entry_arrays(qsl, ids, flags)
    meta.set_slot_split(pool.slot_split)
    meta.build_arrays(qsl, slots, flags)
    return slots


def lora_slot_params(pool, layer, name):
    """Oracle parameter dicts per LoRA slot, read back from the device slabs."""
    A = to_np(pool.lora_A[name][layer])
    Bt = to_np(pool.lora_Bt[name][layer])
    sc = to_np(pool.lora_scale[name][layer])
    return {a: dict(kind="lora", s=float(sc[a]), A=A[a], B=Bt[a].T) for a in range(pool.lora_capacity)}


def reft_slot_params(pool, layer):
    """Oracle dicts per ReFT slot (DiReFT form s((hA'^T + b)B) of the stored operands)."""
    A = to_np(pool.reft_A[layer])
    B = to_np(pool.reft_B[layer])
    b = to_np(pool.reft_bias[layer])
    sc = to_np(pool.reft_scale[layer])
    return {
        pool.slot_split + j: dict(kind="direft", s=float(sc[j]), A=A[j], B=B[j], b=b[j])
        for j in range(pool.reft_capacity)
    }


def lora_oracle(y_in, x, qsl, slots, flags, pool, layer, name):
    mask = oracle_mask(qsl, slots, flags)
    cls = np.where((slots >= 0) & (slots < pool.slot_split), slots, -1)
    return O.lora_hook(y_in, x, qsl, mask, cls, lora_slot_params(pool, layer, name))


def reft_oracle(h_in, qsl, slots, flags, pool, layer):
    mask = oracle_mask(qsl, slots, flags)
    cls = np.where(slots >= pool.slot_split, slots, -1)
    return O.reft_hook(h_in, qsl, mask, cls, reft_slot_params(pool, layer))


def random_lora_adapter(rng, aid, n_layers, sites: dict, rank, schedule=SCHED.PREFILL_ONLY, sigma=0.3):
    lora = {}
    for layer in range(n_layers):
        for name, (n, m) in sites.items():
            A = rng.normal(size=(rank, m)) / np.sqrt(m)
            B = rng.normal(size=(n, rank)) * sigma
            lora[(layer, name)] = AdapterParams(AdapterKind.LORA, rank, (n, m), ScalingRule.alpha_over_r(32.0), A=A, B=B)
    return ModelAdapter(aid, AdapterKind.LORA, rank, schedule, lora_sites=lora)


def random_reft_adapter(rng, aid, n_layers, d, rank, kind=AdapterKind.DIREFT, schedule=SCHED.PREFILL_ONLY):
    from paper_2605_14217_b200.adapters import init_zero_delta

    sites = []
    for layer in range(n_layers):
        p = init_zero_delta(kind, rank, (d,), int(rng.integers(0, 2**31)))
        if kind is AdapterKind.DIREFT:
            p = AdapterParams(kind, rank, (d,), p.scaling, A=rng.normal(size=(rank, d)) / np.sqrt(d), B=p.B,
                              b=rng.normal(size=rank) * 0.1)
        else:
            p = AdapterParams(kind, rank, (d,), p.scaling, R=p.R, W=p.W + rng.normal(size=(rank, d)) * 0.1,
                              b=rng.normal(size=rank) * 0.1)
        sites.append(p)
    return ModelAdapter(aid, kind, rank, schedule, reft_sites=tuple(sites))


def rand_act(rng, rows, width, dtype, device):
    t = torch.from_numpy(rng.normal(size=(rows, width))).to(device=device, dtype=dtype)
    return t
