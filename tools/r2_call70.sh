for r in 1 2; do
  for v in base gu32 gu32f16; do
    for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4 --hq 8 --hkv 2" "--T 131072 --batch 4 --hq 16 --hkv 4" "--T 32768 --batch 2" "--T 131072 --batch 4"; do
      r=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py $cfg --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['fp64_gate_graph_us_per_layer'],2), round(d['forced_gate_graph_us_per_layer'],2))")
      echo "$cfg $v $r"
    done
  done
done
