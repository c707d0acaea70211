timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "topk or ragged" > gpurun_out/r2s3_union_tests.log 2>&1; echo topk tests rc $?; tail -2 gpurun_out/r2s3_union_tests.log
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_fuzz.py tests/test_gpu_peer.py -q -x > gpurun_out/r2s3_union_tests2.log 2>&1; echo other tests rc $?; tail -2 gpurun_out/r2s3_union_tests2.log
for r in 1 2 3; do
for v in two one; do
  E=""; [ $v = two ] && E="WGKV_TOPK_TWO_PASS=1"
  a=$(env $E timeout 300 python profiles/decode_breakdown.py --T 1048576 --batch 1 --hq 4 --hkv 1 --topk 256 --iters 100 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['k5_attn_us'],1), round(d['decode_layer_us'],1))")
  b=$(env $E timeout 300 python profiles/decode_breakdown.py --T 131072 --batch 4 --topk 256 --iters 100 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['k5_attn_us'],1), round(d['decode_layer_us'],1))")
  echo "$v 1m=$a 128k4_topk=$b"
done
done
