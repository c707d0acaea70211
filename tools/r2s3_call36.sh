for r in 1 2; do
for v in cap24 cap16 cap36; do
  b=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 131072 --batch 4 --hq 16 --hkv 4 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  c=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 131072 --batch 4 --hq 4 --hkv 1 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  e=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 32768 --batch 1 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  f=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 131072 --batch 4 --hq 8 --hkv 2 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  echo "$v shard2=$b shard8=$c b1_32k=$e shard4=$f"
done
done
