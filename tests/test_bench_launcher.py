"""bench.py's multi-rank launcher and reference arm, on CPU.

* `bench.py --gpus 2 --dry-run` goes through the same self-launch code the
  driver's `bench.py --gpus N` form uses (re-exec under torch.distributed.run,
  one rank per GPU) with a gloo group instead of NCCL: rank 0 must print one
  line with n_gpus = 2, each rank's routed batch, and the config-5 strong-
  scaling routing (hot adapters replicated, requests on adapter holders).
* `bench.py --impl reference` at a tiny size: the unmodified reference
  (oracle/_ref) timed over the same cfg2 config dict as the GPU arm.
"""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_gpus_2_self_launches_two_ranks():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                       text=True, timeout=240, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["dry_run"] and line["n_gpus"] == 2 and line["backend"] == "gloo"
    assert len(line["per_rank_prefill_tokens"]) == 2 and all(v > 0 for v in line["per_rank_prefill_tokens"])
    strong = line["cfg5_strong"]
    assert strong["hot_replicated_adapters"] == [0]  # the Zipf head carries > 0.5/2 of the requests
    assert sum(strong["per_rank_prefill_tokens"]) == strong["global_prefill_tokens"]
    # least-loaded routing of the replicated head keeps the ranks within 25% of each other
    assert max(strong["per_rank_prefill_tokens"]) / (strong["global_prefill_tokens"] / 2) < 1.25


def test_reference_arm_same_config_as_ours(tmp_path):
    from oracle import build_ref

    if build_ref.build() is None:
        pytest.skip("reference neither mounted nor installed")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup",
                        "1", "--requests", "6", "--decodes", "4", "--ref-cores", "2"], capture_output=True, text=True,
                       timeout=240, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["cpu_baseline"]["cores"] == 2 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    sys.path.insert(0, str(ROOT))
    import bench

    qsl, ids, flags, lens, _ = bench.step_entries(0, 1, 6, 4)
    assert line["config"]["prefill_tokens_per_gpu"] == int(lens.sum())
    assert line["config"]["workload"].startswith("cfg2")


@pytest.mark.gpu
def test_gpus_2_on_one_gpu_runs_the_multi_rank_path():
    """The multi-rank path with real kernels on a 1-GPU box: `bench.py --gpus 2
    --share-gpu` self-launches two ranks on cuda:0 (gloo bookkeeping); the
    config-5 strong-scaling line routes one global Zipf stream to the adapter
    owners with the head adapter replicated, and its parity must pass."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--share-gpu", "--steps", "2",
                        "--warmup", "3", "--only", "cfg5s"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 2 and "shared_gpu" in line
    (c,) = line["other_configs"]
    assert c["n_gpus"] == 2 and c["parity"]["status"] == "pass"
    assert c["hot_replicated_adapters"] == [0] and len(c["requests_per_rank"]) == 2
