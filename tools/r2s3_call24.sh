timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fuzz.py tests/test_gpu_peer.py -x -q > gpurun_out/r2s3_ipc_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/r2s3_ipc_tests.log
for cfg in "--T 131072 --batch 4" "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 8 --hkv 2"; do
  a=$(timeout 300 python profiles/decode_layers.py $cfg --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  echo "$cfg -> $a us/layer"
done
