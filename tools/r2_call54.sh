timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_fused.log 2>&1; echo gpu rc $?
tail -3 gpurun_out/r2_pytest_fused.log
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4 --hq 8 --hkv 2"; do
  for v in base new; do
    for f in 0 148; do
      L=build/var/libwgkv_base.so; [ $v = new ] && L=paper_2512_17452_b200/libwgkv_b200.so
      r=$(WGKV_LIB=$L WGKV_DECODE_FUSED=$f timeout 300 python profiles/decode_layers.py $cfg --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['fp64_gate_graph_us_per_layer'],2), round(d['forced_gate_graph_us_per_layer'],2))")
      echo "$cfg $v fused=$f $r"
    done
  done
done
for v in base new; do
  L=build/var/libwgkv_base.so; [ $v = new ] && L=paper_2512_17452_b200/libwgkv_b200.so
  echo "prefill $v $(WGKV_LIB=$L timeout 300 python profiles/prefill_breakdown.py --reps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['k3_vs_ms'],2))")"
done
WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --forced --dump gpurun_out/tlf_32kf.npz > /dev/null 2>&1
WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --dump gpurun_out/tlf_32k.npz > /dev/null 2>&1
