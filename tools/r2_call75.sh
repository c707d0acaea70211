for r in 1 2 3; do
  for v in base sc32 sc16; do
    echo "$v $(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_breakdown.py --T 1048576 --batch 1 --hq 4 --hkv 1 --topk 256 --iters 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['k5_attn_us'],1), round(d['decode_layer_us'],1))")"
  done
done
