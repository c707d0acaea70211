for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1"; do
  for v in base pw ef pwef; do
    for f in 0 148; do
      r=$(WGKV_LIB=build/var/libwgkv_$v.so WGKV_DECODE_FUSED=$f timeout 300 python profiles/decode_layers.py $cfg --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['fp64_gate_graph_us_per_layer'],2), round(d['forced_gate_graph_us_per_layer'],2))")
      echo "$cfg $v fused=$f $r"
    done
  done
done
WGKV_LIB=build/var/libwgkv_tlpwef.so timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --forced --dump gpurun_out/tlf_32kf_pwef.npz > /dev/null 2>&1
WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --forced --dump gpurun_out/tlf_32kf.npz > /dev/null 2>&1
