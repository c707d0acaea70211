#!/bin/bash
# Interleaved A/B of the top-k decode chain: PDL launches (product) vs plain launches (WGKV_TOPK_NOPDL=1),
# printing K5-with-selection and whole-decode-layer microseconds from profiles/decode_breakdown.py.
for args in "--T 1048576 --batch 1 --hq 4 --hkv 1 --topk 256" "--topk 256" "--T 1048576 --batch 1 --hq 4 --hkv 1 --topk 256 --quest"; do
for r in 1 2; do
  for v in 0 1; do
    if [ $v = 1 ]; then export WGKV_TOPK_NOPDL=1; else unset WGKV_TOPK_NOPDL; fi
    t=$(timeout 300 python profiles/decode_breakdown.py $args --iters 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['k5_attn_us'],1), round(d['decode_layer_us'],1))" 2>&1 | tail -1)
    echo "[$args] nopdl=$v $t"
  done
done
done
