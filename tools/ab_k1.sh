#!/bin/bash
# Interleaved A/B of K1 (gate_tc) across builds: tools/ab_k1.sh ROUNDS "ENV1" "ENV2" ...
R=$1; shift
for r in $(seq $R); do
  for v in "$@"; do
    t=$(env $v timeout 300 python profiles/prefill_breakdown.py --reps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['k1_gate_ms'],3), round(d['k3_vs_ms'],2))")
    echo "$v $t"
  done
done
