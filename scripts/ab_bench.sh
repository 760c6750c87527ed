#!/bin/bash
# Interleaved A/B of whole bench steps: ab_bench.sh "ENV_A" "ENV_B" [reps] [bench args]
A="$1"; B="$2"; reps=${3:-3}; shift 3; args="$@"
for i in $(seq $reps); do
  for e in "$A" "$B"; do
    r=$(env $e timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 $args 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"]["sm_mhz"])')
    echo "[$e] $r"
  done
done
