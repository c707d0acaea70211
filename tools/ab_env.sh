#!/bin/bash
# Interleaved A/B of runtime switches on the K3 breakdown: tools/ab_env.sh ROUNDS "ENV1" "ENV2" ...
R=$1; shift
for r in $(seq $R); do
  for v in "$@"; do
    t=$(env $v timeout 300 python profiles/prefill_breakdown.py --reps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['k3_vs_ms'],2))")
    echo "$v $t"
  done
done
