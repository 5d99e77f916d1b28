#!/usr/bin/env bash
# One GPU session: tests, smoke, bench, per-kernel sweeps, ncu launch list and
# full captures of the top kernels.  Outputs land in gpurun_out/<tag>_*.
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
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
python - "$O/${TAG}_bench.json" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    r = d["roofline"]
    print("bench", d["value"], "frac", r["frac"], "step_frac", r["step_frac"], "e2e", (d.get("e2e") or {}).get("value"),
          "cpu", (d.get("cpu_baseline") or {}).get("value"), "punica", d.get("punica_step"), "clocks", d.get("clocks"))
    for c in d.get("other_configs") or []:
        print("  ", c)
except Exception as e:
    print("bench failed", e)
PY
timeout 300 python tools/kbench.py > $O/${TAG}_kbench.json 2> $O/${TAG}_kbench.err
timeout 300 python tools/kbench.py --requests 32 --decodes 32 > $O/${TAG}_kbench_small.json 2>> $O/${TAG}_kbench.err
timeout 300 python tools/reft_bench.py > $O/${TAG}_reft.json 2>> $O/${TAG}_kbench.err
for d in 2048 4096; do for v in pass res; do
  timeout 200 python tools/reft_bench.py --variant $v --d $d --iters 20 >> $O/${TAG}_reft_variants.json 2>> $O/${TAG}_kbench.err
done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lora|meta|reft" -c 390 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-punica-step --no-secondary \
  > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:lora -s 2 -c 4 -o $O/${TAG}_prof \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-punica-step --no-secondary > $O/${TAG}_ncu.log 2>&1
python tools/ncu_summary.py --rep $O/${TAG}_prof.ncu-rep --launches $O/${TAG}_launches.csv \
  --out $O/${TAG}_ncu_summary.json > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:reft_tc -s 3 -c 1 -o $O/${TAG}_reft_prof \
  python tools/reft_bench.py --case cfg3 --variant tc --iters 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none -k regex:"shrink_tc|expand_tc" -s 8 -c 8 -o $O/${TAG}_split_prof \
  python bench.py --only cfg4 --no-parity --steps 1 > /dev/null 2>&1
# config 5's K3-TC (LoReFT r32, the whole kernel on 148 SMs), config 3's parked half at d = 4096, and the
# fused TP kernel at config-4 shapes (q/k/v group, one-rank exchange)
timeout 300 ncu --set full --clock-control none -k regex:reft_tc -s 3 -c 1 -o $O/${TAG}_cfg5_prof \
  python tools/reft_bench.py --case cfg5 --variant tc --iters 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:reft_res -s 3 -c 1 -o $O/${TAG}_res4k_prof \
  python tools/reft_bench.py --case cfg3 --variant tc --iters 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:lora_fused -s 2 -c 1 -o $O/${TAG}_fused_prof \
  env GROUP=qkv python tools/fused_prof.py > /dev/null 2>&1
# full reports are large (the 64 MiB return limit): keep CSV exports of the secondary captures
timeout 300 ncu --set full --clock-control none --import-source on -k regex:reft_res -s 3 -c 1 -o $O/${TAG}_res_prof \
  python tools/reft_bench.py --case cfg3 --variant res --d 2048 --iters 1 > /dev/null 2>&1
for r in reft_prof split_prof res_prof cfg5_prof res4k_prof fused_prof; do
  ncu -i $O/${TAG}_${r}.ncu-rep --page raw --csv > $O/${TAG}_${r}_raw.csv 2>/dev/null
  python tools/ncu_metrics.py $O/${TAG}_${r}.ncu-rep > $O/${TAG}_${r}_metrics.txt 2>/dev/null
  rm -f $O/${TAG}_${r}.ncu-rep
done
ls $O | grep "^${TAG}_"
