#!/usr/bin/env bash
# One GPU session: tests, smoke, bench, per-kernel sweep, ncu launch list and
# full capture of one step's K2 launches.  Outputs land in gpurun_out/<tag>_*.
# usage (under gpurun): bash tools/gpu_round.sh <tag> [skip-tests]
set -u
TAG=${1:-run}
SKIP_TESTS=${2:-}
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out
mkdir -p $O
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > $O/${TAG}_tests.log 2>&1
  tail -2 $O/${TAG}_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
  tail -1 $O/${TAG}_smoke.log
fi
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
python - "$O/${TAG}_bench.json" <<'EOF'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    r = d["roofline"]
    print("bench", d["value"], "frac", r["frac"], "step_frac", r["step_frac"], "e2e", (d.get("e2e") or {}).get("value"),
          "cpu", (d.get("cpu_baseline") or {}).get("value"), "punica", d.get("punica_step"), "clocks", d.get("clocks"))
except Exception as e:
    print("bench failed", e)
EOF
timeout 300 python tools/kbench.py > $O/${TAG}_kbench.json 2> $O/${TAG}_kbench.err
timeout 300 python tools/kbench.py --requests 32 --decodes 32 > $O/${TAG}_kbench_small.json 2>> $O/${TAG}_kbench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lora|meta|reft" -c 390 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-punica-step --no-secondary \
  > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:lora -s 2 -c 4 -o $O/${TAG}_prof \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-punica-step --no-secondary > $O/${TAG}_ncu.log 2>&1
ls $O | grep "^${TAG}_"
