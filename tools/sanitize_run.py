#!/usr/bin/env python
"""Small invocations of every kernel family for compute-sanitizer runs:
K1, K2 (team, warp, f64), K2 split (tcgen05 + SIMT), K2f (fused, one-rank exchange), K3 (SIMT + tcgen05 streaming +
tcgen05 TMEM-parked at d = 1024 / 2048), K4."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch

    import gpu_util as U
    from paper_2605_14217_b200 import AdapterKind, _lib
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_lora_group_, apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool
    from paper_2605_14217_b200.tp import SplitWorkspace, apply_lora_group_tp_

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    for dtype, lr, rr in ((torch.bfloat16, 1, 16), (torch.bfloat16, 16, 32), (torch.float64, 2, 4)):
        d = 256
        sites = {"Wq": (d, d), "Wk": (128, d), "Wv": (128, d)}
        pool = AdapterPool(1, d, lora_sites=sites, lora_capacity=3, lora_rank=lr, reft_capacity=3, reft_rank=rr,
                           dtype=dtype, device=dev)
        for a in range(3):
            pool.register(U.random_lora_adapter(rng, a, 1, sites, lr))
            pool.register(U.random_reft_adapter(rng, 10 + a, 1, d, rr, AdapterKind.DIREFT))
        lens = [1] * 4 + list(rng.integers(1, 70, size=8)) + [150]
        qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        ids = [[0, 1, 2, 10, 11, 12, None][int(i) % 7] for i in range(len(lens))]
        flags = np.array([_lib.ENTRY_DECODE] * 4 + [0] * (len(lens) - 4), np.int32)
        meta = BatchMeta(32, int(qsl[-1]), device=dev)
        U.stage(meta, pool, qsl, ids, flags)
        T = int(qsl[-1])
        x = U.rand_act(rng, T, d, dtype, dev)
        ys = [U.rand_act(rng, T, sites[s][0], dtype, dev) for s in sites]
        h = U.rand_act(rng, T, d, dtype, dev)
        apply_lora_group_(ys, x, meta, pool, 0, tuple(sites))
        if dtype == torch.bfloat16 and lr == 1:
            # every K2 variant: the warp kernel and teams of 1 / 2 / 4 / 8 warps
            lib = _lib.load()
            for v in (0, 1, 2, 4, 8):
                assert lib.preft_set_lora_variant(v) == 0
                try:
                    apply_lora_group_(ys, x, meta, pool, 0, tuple(sites))
                    apply_lora_group_(ys[:1], x, meta, pool, 0, ("Wq",))
                    torch.cuda.synchronize()
                finally:
                    lib.preft_set_lora_variant(-1)
        apply_lora_group_tp_(ys, x, meta, pool, 0, tuple(sites), workspace=SplitWorkspace(meta, pool))
        if dtype == torch.bfloat16 and lr == 16:
            # K2f, the fused shrink -> exchange -> expand kernel, one rank, whole and K-split units
            from paper_2605_14217_b200.tp import FusedExchange

            for planes in (1, 4):
                ex = FusedExchange.local(meta, pool, planes=planes)
                for _ in range(2):  # both parities
                    apply_lora_group_tp_(ys, x, meta, pool, 0, tuple(sites), exchange=ex)
                torch.cuda.synchronize()
                assert ex.errors() == 0
        apply_reft_(h, meta, pool, 0)
        torch.cuda.synchronize()
        print("ok", dtype, lr, rr)
    lib = _lib.load()
    for d, rr in ((1024, 16), (2048, 32)):
        pool = AdapterPool(1, d, reft_capacity=3, reft_rank=rr, dtype=torch.bfloat16, device=dev)
        for a in range(3):
            pool.register(U.random_reft_adapter(rng, a, 1, d, rr, AdapterKind.LOREFT))
        lens = [1] * 4 + list(rng.integers(1, 70, size=6)) + [130]
        qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        ids = [[0, 1, 2, None][int(i) % 4] for i in range(len(lens))]
        flags = np.array([_lib.ENTRY_DECODE] * 4 + [0] * (len(lens) - 4), np.int32)
        meta = BatchMeta(16, int(qsl[-1]), device=dev)
        U.stage(meta, pool, qsl, ids, flags)
        h = U.rand_act(rng, int(qsl[-1]), d, torch.bfloat16, dev)
        assert lib.preft_set_reft_variant(3) == 0
        try:
            apply_reft_(h, meta, pool, 0)
            torch.cuda.synchronize()
        finally:
            lib.preft_set_reft_variant(-1)
        print("ok resident", d, rr)


if __name__ == "__main__":
    main()
