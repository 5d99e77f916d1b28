#!/usr/bin/env python
"""Record the reference engine's step schedule (engine.py:397-489, cost mode)
for two Punica workloads into tests/golden/serving_trace.npz.

Run in the build container (imports /root/reference/pkg/src):
    python tests/golden/make_serving_golden.py
The fixture pins serving.Scheduler + paging.LruResidency on hosts without
the reference (tests/test_serving_cpu.py).
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from prefillsim.adapters import AdapterKind, PositionSchedule  # noqa: E402
from prefillsim.engine import AdapterSetup, EngineConfig, simulate  # noqa: E402
from prefillsim.workload import AdapterMix, WorkloadConfig, generate_workload  # noqa: E402

CASES = {
    "uniform": dict(wl=dict(n_requests=120, n_adapters=48, mix=AdapterMix.UNIFORM, seed=3, l_max=256),
                    eng=dict(max_batch=16, max_gpu_adapters=8, step_token_budget=256, chunk_size=None)),
    "skewed_chunked": dict(wl=dict(n_requests=90, n_adapters=30, mix=AdapterMix.SKEWED, seed=5, l_max=200),
                           eng=dict(max_batch=12, max_gpu_adapters=6, step_token_budget=128, chunk_size=40)),
}


def main():
    out = {}
    for name, c in CASES.items():
        wl = generate_workload(WorkloadConfig(**c["wl"]))
        for sched in (PositionSchedule.PREFILL_ONLY, PositionSchedule.ALL_POSITIONS):
            tag = f"{name}_{sched.value}"
            res = simulate(wl, EngineConfig(warmup=False, **c["eng"]),
                           AdapterSetup(kind=AdapterKind.LORA, rank=1, schedule=sched))
            out[f"{tag}_n_steps"] = np.array(len(res.steps))
            for field in ("scheduled", "workset", "resident", "paged_in"):
                flat, offs = [], [0]
                for s in res.steps:
                    v = [(-1 if a is None else int(a)) for a in getattr(s, field)]
                    flat += v
                    offs.append(len(flat))
                out[f"{tag}_{field}"] = np.asarray(flat, dtype=np.int64)
                out[f"{tag}_{field}_off"] = np.asarray(offs, dtype=np.int64)
            out[f"{tag}_prefill_tokens"] = np.asarray([s.prefill_tokens for s in res.steps], dtype=np.int64)
            out[f"{tag}_decode_tokens"] = np.asarray([s.decode_tokens for s in res.steps], dtype=np.int64)
    path = Path(__file__).with_name("serving_trace.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
