#!/bin/bash
# One GPU call: default bench line, the other configs, the reference arm, and
# the C5 launch list (ncu, durations only).  Usage: tools/round_bench.sh TAG
TAG=${1:-vX}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; tail -1 gpurun_out/bench_$TAG.log > gpurun_out/bench_$TAG.jsonl
timeout 300 python bench.py --impl reference >> gpurun_out/bench_$TAG.jsonl 2>/dev/null
: > gpurun_out/bench_${TAG}_configs.jsonl
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --no-cpu 2>/dev/null | tail -1 >> gpurun_out/bench_${TAG}_configs.jsonl
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c5_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
for f in (f"gpurun_out/bench_{tag}.jsonl", f"gpurun_out/bench_{tag}_configs.jsonl"):
    for l in open(f):
        d = json.loads(l)
        print(d.get("impl", "ours"), d["config"]["workload"], round(d["value"]), round(d["ms_per_step"], 4),
              (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), d.get("clocks", {}).get("sm_mhz"))
PY
