for r in 1 2; do
for v in default k5; do
  E=""; [ $v = k5 ] && E="WGKV_GATE_PLACE=k5"
  a=$(env $E timeout 300 python profiles/decode_layers.py --T 131072 --batch 4 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  b=$(env $E timeout 300 python profiles/decode_layers.py --T 65536 --batch 8 --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['fp64_gate_graph_us_per_layer'],1))")
  echo "$v 128k4=$a 64k8=$b"
done
done
