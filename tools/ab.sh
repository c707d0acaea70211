#!/bin/bash
# Interleaved A/B of K3 variants: tools/ab.sh ROUNDS name1 name2 ... (build/var/libwgkv_NAME.so)
R=$1; shift
for r in $(seq $R); do
  for v in "$@"; do
    t=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/prefill_breakdown.py --reps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['k3_vs_ms'],2))")
    echo "$v $t"
  done
done
