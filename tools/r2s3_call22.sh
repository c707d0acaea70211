for r in 1 2; do
for v in ipc3 ipc2 ipc4; do
  a=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 131072 --batch 4 --hq 32 --hkv 8 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  b=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 131072 --batch 4 --hq 16 --hkv 4 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  c=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 131072 --batch 4 --hq 4 --hkv 1 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  e=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 65536 --batch 8 --hq 32 --hkv 8 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  echo "$v 128k4=$a shard2=$b shard8=$c 64k8=$e"
done
done
