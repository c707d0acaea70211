set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu.log 2>&1; echo pytest rc $?
timeout 600 ./oracle/_ref/dropin_session > gpurun_out/r2_dropin.log 2>&1; echo dropin rc $?
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4"; do
  for env in "X=1" "WGKV_GATE_IN_FINISH=1" "WGKV_K5_NO_TRIGGER=1" "WGKV_GATE_IN_FINISH=1 WGKV_K5_NO_TRIGGER=1"; do
    echo "== $cfg $env"; env $env timeout 300 python profiles/decode_layers.py $cfg --steps 30
  done
done > gpurun_out/r2_decode_ab.txt 2>&1
