timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fuzz.py tests/test_gpu_peer.py -x -q > gpurun_out/r2s3_early_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/r2s3_early_tests.log
for r in 1 2 3; do
for v in noearly early; do
  a=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 131072 --batch 4 --hq 32 --hkv 8 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  b=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 131072 --batch 4 --hq 16 --hkv 4 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  c=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py --T 65536 --batch 16 --hq 32 --hkv 8 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  echo "$v 128k4=$a shard2=$b 64k16=$c"
done
done
