timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_waves.log 2>&1; echo gpu rc $?
tail -1 gpurun_out/r2_pytest_waves.log
for r in 1 2; do
  for v in nowaves waves; do
    for cfg in "--T 131072 --batch 4" "--T 131072 --batch 4 --hq 16 --hkv 4" "--T 32768 --batch 2" "--T 131072 --batch 4 --hq 8 --hkv 2" "--T 32768 --batch 1"; do
      r=$(WGKV_LIB=build/var/libwgkv_$v.so timeout 300 python profiles/decode_layers.py $cfg --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['fp64_gate_graph_us_per_layer'],2), round(d['forced_gate_graph_us_per_layer'],2))")
      echo "$cfg $v $r"
    done
  done
done
