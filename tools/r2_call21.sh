mkdir -p gpurun_out
WGKV_GATE_PLACE=side timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider -k "session or ragged or decode or shard or many_pairs" > gpurun_out/r2_pytest_side.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/r2_pytest_side.log
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4"; do
  for env in "X=1" "WGKV_GATE_PLACE=side"; do
  echo "== $cfg $env"; env $env timeout 300 python profiles/decode_layers.py $cfg --steps 30
  done
done > gpurun_out/r2_decode_ab6.txt 2>&1
