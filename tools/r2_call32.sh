mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/r2_pytest_gpu.log
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4"; do
  echo "== $cfg"; timeout 300 python profiles/decode_layers.py $cfg --steps 30
done > gpurun_out/r2_decode_ab8.txt 2>&1
