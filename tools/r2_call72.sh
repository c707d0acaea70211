timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_comb.log 2>&1; echo gpu rc $?
tail -1 gpurun_out/r2_pytest_comb.log
for r in 1 2 3; do
  for v in base new; do
    L=build/var/libwgkv_base.so; [ $v = new ] && L=paper_2512_17452_b200/libwgkv_b200.so
    echo "$v $(WGKV_LIB=$L timeout 300 python profiles/decode_breakdown.py --T 1048576 --batch 1 --hq 4 --hkv 1 --topk 256 --iters 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['k5_attn_us'],1), round(d['decode_layer_us'],1))")"
  done
done
