#!/bin/bash
# Interleaved A/B of decode variants: tools/ab_decode.sh ROUNDS "ARGS" name1 name2 ... (build/var/libwgkv_NAME.so)
R=$1; shift; A=$1; shift
for r in $(seq $R); do
  for v in "$@"; do
    t=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_breakdown.py $A --iters 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['k5_attn_us'],1), round(d['decode_layer_us'],1))")
    echo "$v $t"
  done
done
