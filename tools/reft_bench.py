#!/usr/bin/env python
"""Per-launch timing of the ReFT^P kernels (diagnostic, one GPU).

One 8B-shaped residual site (d = 4096, bf16): DiReFT r=16 over 2,048-token
prompts (config 3's shape) and LoReFT r=32 over long Zipf prompts (config 5's
shape), for the tensor-core kernel and the SIMT kernel.  Each launch works on
a fresh activation buffer (a ring larger than L2), timed with CUDA events on
the launching stream.  Prints one JSON line per case with the algorithmic
bytes (T_p*2*d*e + D*e*2*r*d) and the fraction of peak.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run(kind, rank, lens, ids, variant, peak, iters=10, prof=False, d=4096):
    import torch

    from paper_2605_14217_b200 import AdapterKind, _lib
    from paper_2605_14217_b200.meta import BatchMeta
    from paper_2605_14217_b200.ops import apply_reft_
    from paper_2605_14217_b200.pool import AdapterPool

    dev = torch.device("cuda", 0)
    n_ad = int(max(ids)) + 1
    pool = AdapterPool(1, d, reft_capacity=n_ad, reft_rank=rank, dtype=torch.bfloat16, device=dev)
    pool.fill_synthetic_(n_ad, AdapterKind(kind), rank, seed=1)
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(qsl[-1])
    slots = pool.entry_arrays(qsl, [int(i) for i in ids], np.zeros(len(lens), np.int32))
    meta = BatchMeta(len(lens), T, device=dev)
    meta.set_slot_split(pool.slot_split)
    meta.build_arrays(qsl, slots, np.zeros(len(lens), np.int32))
    nbuf = max(2, int(np.ceil(300e6 / (T * d * 2))))
    hs = [torch.randn(T, d, device=dev).to(torch.bfloat16) for _ in range(nbuf)]
    lib = _lib.load()
    lib.preft_set_reft_variant(variant)
    try:
        for i in range(3):
            apply_reft_(hs[i % nbuf], meta, pool, 0)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        for i in range(iters):
            ev[i][0].record()
            apply_reft_(hs[(i + 3) % nbuf], meta, pool, 0)
            ev[i][1].record()
        torch.cuda.synchronize()
    finally:
        lib.preft_set_reft_variant(-1)
    us = float(np.mean([a.elapsed_time(b) for a, b in ev]) * 1e3)
    grid = int(lib.preft_diag_reft_tc(None))
    if prof and variant == 3:
        import ctypes

        buf = torch.zeros(736, dtype=torch.int64, device=dev)
        lib.preft_set_reft_variant(3)
        lib.preft_diag_reft_tc(ctypes.c_void_p(buf.data_ptr()))
        apply_reft_(hs[0], meta, pool, 0)
        torch.cuda.synchronize()
        lib.preft_diag_reft_tc(None)
        lib.preft_set_reft_variant(-1)
        st = buf.cpu().numpy().astype(np.int64)
        un = st[:128].reshape(16, 8)
        ch = st[128:640].reshape(64, 8)
        t0 = int(un[0, 5])
        sx = st[640:704].reshape(16, 4)
        print("units: s_full p_full v_full | mma first last | prod first last | stash first(h_full, t_empty) last(h_full, t_empty)", file=sys.stderr)
        for u in range(16):
            if un[u, 5]:
                r = [int(un[u, k]) - t0 if un[u, k] else -1 for k in (0, 1, 2, 3, 4, 5, 6)]
                x = [int(v) - t0 if v else -1 for v in sx[u]]
                print(u, r[:3], "|", r[3:5], "|", r[5:7], "|", x, file=sys.stderr)
        print("stash panels: waits done, released", file=sys.stderr)
        for c in range(48):
            if ch[c, 6]:
                print("  p", c, int(ch[c, 6]) - t0, int(ch[c, 7]) - t0, file=sys.stderr)
        print("chunks: epi d_full rmw released | mma bt_full d_empty issued", file=sys.stderr)
        for c in range(48):
            if ch[c, 3]:
                r = [int(ch[c, k]) - t0 if ch[c, k] else -1 for k in (0, 1, 2, 3, 4, 5)]
                print(c, r[:3], "|", r[3:], file=sys.stderr)
    if prof and variant == 1:
        import ctypes

        buf = torch.zeros(736, dtype=torch.int64, device=dev)
        lib.preft_set_reft_variant(1)
        lib.preft_diag_reft_tc(ctypes.c_void_p(buf.data_ptr()))
        apply_reft_(hs[0], meta, pool, 0)
        torch.cuda.synchronize()
        lib.preft_diag_reft_tc(None)
        lib.preft_set_reft_variant(-1)
        st = buf.cpu().numpy()
        ch = st[:512].reshape(64, 8).astype(np.int64)
        un = st[512:576].reshape(16, 4).astype(np.int64)
        sh = st[576:608].reshape(16, 2).astype(np.int64)
        xp = st[608:736].reshape(16, 8).astype(np.int64)
        t0 = int(un[0, 0])
        names = ["mma_epi_full", "mma_d_empty", "mma_issued", "ep_d_full", "ep_epi_full", "ep_ldtm", "ep_rmw", "ep_released"]
        print("chunk timeline (cycles from unit 0 s_full), " + " ".join(names), file=sys.stderr)
        for c in range(len(ch)):
            print(c, " ".join(f"{int(v) - t0:8d}" for v in ch[c]), file=sys.stderr)
        print("units: s_full, S loaded, exchanged, v_full | shrink first panel, last panel", file=sys.stderr)
        for u in range(16):
            if un[u, 0]:
                print(u, " ".join(f"{int(v) - t0:8d}" for v in un[u]), "|",
                      " ".join(f"{int(v) - t0:8d}" for v in sh[u]), "| p_empty ok, pushed, p_full ok",
                      " ".join(f"{int(v) - t0:8d}" for v in xp[u, :3]), "| gt", int(xp[u, 4]), int(xp[u, 5]),
                      file=sys.stderr)
    distinct = len(set(int(i) for i in ids))
    alg = T * 2 * d * 2 + distinct * 2 * (2 * rank * d) + distinct * 4 * rank
    gbs = alg / us / 1e3
    return {"kind": kind, "rank": rank, "d": d, "tokens": T, "distinct": distinct, "variant": ["simt", "tc", "pass", "res"][variant],
            "us": round(us, 1), "grid": grid, "gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
            "tokens_per_s_32_layers": round(T / (us * 1e-6) / 32, 1)}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--peak", type=float, default=None)
    p.add_argument("--case", choices=["cfg3", "cfg5", "all"], default="all")
    p.add_argument("--variant", choices=["tc", "simt", "pass", "res", "all"], default="all")
    p.add_argument("--iters", type=int, default=10)
    p.add_argument("--prof", action="store_true")
    p.add_argument("--d", type=int, default=4096, help="hidden size (8B shape: 4096)")
    p.add_argument("--persist-mb", type=float, default=None, help="L2 set-aside for persisting (evict_last) lines")
    args = p.parse_args()
    if args.persist_mb is not None:
        import ctypes

        import torch

        torch.cuda.init()
        rt = ctypes.CDLL("libcudart.so.12")
        mx = ctypes.c_int()
        rt.cudaDeviceGetAttribute(ctypes.byref(mx), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
        want = min(int(args.persist_mb * 2**20), mx.value)
        rc = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(want))  # cudaLimitPersistingL2CacheSize
        got = ctypes.c_size_t()
        rt.cudaDeviceGetLimit(ctypes.byref(got), 6)
        print(f"persisting L2: max {mx.value >> 20} MB, set rc={rc}, now {got.value >> 20} MB", file=sys.stderr)
    peak = args.peak
    if peak is None:
        f = ROOT / "MEASURED_PEAKS.json"
        peak = float(json.loads(f.read_text())["hbm_gbs"]) if f.exists() else 6650.0
    rng = np.random.default_rng(0)
    cfg3 = ([2048] * 32, rng.integers(0, 512, size=32))
    w = 1.0 / (np.arange(512) + 1.0)
    cfg5 = (list(rng.integers(8192, 16385, size=8)), rng.choice(512, size=8, p=w / w.sum()))
    for variant in {"tc": (1,), "simt": (0,), "pass": (2,), "res": (3,), "all": (1, 0)}[args.variant]:
        if args.case in ("cfg3", "all"):
            print(json.dumps(run("direft", 16, *cfg3, variant, peak, args.iters, args.prof, args.d)), flush=True)
        if args.case in ("cfg5", "all"):
            print(json.dumps(run("loreft", 32, *cfg5, variant, peak, args.iters, args.prof, args.d)), flush=True)


if __name__ == "__main__":
    main()
