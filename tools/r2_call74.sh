timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_cs.log 2>&1; echo gpu rc $?
tail -1 gpurun_out/r2_pytest_cs.log
for r in 1 2 3; do
  for v in base new; do
    L=build/var/libwgkv_base.so; [ $v = new ] && L=paper_2512_17452_b200/libwgkv_b200.so
    for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4"; do
      r=$(WGKV_LIB=$L timeout 300 python profiles/decode_layers.py $cfg --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['fp64_gate_graph_us_per_layer'],2), round(d['forced_gate_graph_us_per_layer'],2))")
      echo "$cfg $v $r"
    done
  done
done
