set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu.log 2>&1; echo pytest rc $?
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4"; do
  for env in "X=1" "WGKV_GATE_PLACE=k5" "WGKV_GATE_PLACE=finish" "WGKV_GATE_PLACE=finish WGKV_K5_NO_TRIGGER=1"; do
    echo "== $cfg $env"; env $env timeout 300 python profiles/decode_layers.py $cfg --steps 30
  done
done > gpurun_out/r2_decode_ab3.txt 2>&1
