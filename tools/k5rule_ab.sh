for v in v1 v2 v3; do
  a=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --steps 10 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  b=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_breakdown.py --T 131072 --batch 4 --topk 64 --iters 100 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['k5_attn_us'],1))")
  c=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_breakdown.py --T 1048576 --batch 1 --hq 4 --hkv 1 --iters 100 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['k5_attn_us'],1))")
  e=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_breakdown.py --T 1048576 --batch 1 --hq 4 --hkv 1 --topk 256 --iters 100 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['k5_attn_us'],1))")
  f=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_breakdown.py --T 131072 --batch 4 --iters 100 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['k5_attn_us'],1))")
  echo "$v b1_32k=$a 128k4_topk=$b 1m=$c 1m_topk=$e 128k4=$f"
done
