timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_fused.log 2>&1; echo gpu rc $?
tail -3 gpurun_out/r2_pytest_fused.log
for r in 1 2; do
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4 --hq 8 --hkv 2"; do
    for f in 0 148; do
      r=$(WGKV_DECODE_FUSED=$f timeout 300 python profiles/decode_layers.py $cfg --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['fp64_gate_graph_us_per_layer'],2), round(d['forced_gate_graph_us_per_layer'],2))")
      echo "$cfg fused=$f $r"
    done
done
done
WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --dump gpurun_out/tlf_32k.npz > /dev/null 2>&1
WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 131072 --batch 4 --hq 4 --hkv 1 --dump gpurun_out/tlf_s8.npz > /dev/null 2>&1
