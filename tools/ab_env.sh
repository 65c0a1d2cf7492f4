#!/bin/bash
# A/B an environment knob on the bench step time: tools/ab_env.sh VAR "v1 v2" "configs"
VAR=$1; VALS=${2:-"0 1"}; CONFIGS=${3:-"1 2 3 4 5"}
mkdir -p gpurun_out
for c in $CONFIGS; do for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --config $c --steps 10 --no-cpu --no-e2e > gpurun_out/ab_c${c}_$v.log 2>&1
  tail -1 gpurun_out/ab_c${c}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c $VAR=$v', round(d['ms_per_step'],4), 'ms/step', {k: round(v,4) for k,v in d['kernel_ms'].items() if isinstance(v, float)})" || tail -3 gpurun_out/ab_c${c}_$v.log
done; done
