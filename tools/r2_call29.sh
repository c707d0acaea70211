mkdir -p gpurun_out
for lib in k5p2s1 k5p2s2; do WGKV_LIB=build/var/libwgkv_$lib.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider -k "session or ragged or topk or many_pairs or shard or configs0" > gpurun_out/r2_pytest_$lib.log 2>&1; echo $lib pytest rc $?; tail -1 gpurun_out/r2_pytest_$lib.log; done
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4"; do
  for lib in k5b k5p2s1 k5p2s2 k5p2s1w8; do
  echo "== $cfg $lib"; WGKV_LIB=build/var/libwgkv_$lib.so timeout 300 python profiles/decode_layers.py $cfg --steps 30
  done
done > gpurun_out/r2_decode_ab7.txt 2>&1
