for r in 1 2; do
for cfg in "--T 131072 --batch 4 --hq 16 --hkv 4" "--T 32768 --batch 2" "--T 32768 --batch 1 --hq 64 --hkv 8"; do
  for f in 0 148; do
      r=$(WGKV_DECODE_FUSED=$f timeout 300 python profiles/decode_layers.py $cfg --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['fp64_gate_graph_us_per_layer'],2), round(d['forced_gate_graph_us_per_layer'],2))")
      echo "$cfg fused=$f $r"
  done
done
done
