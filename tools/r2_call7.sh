mkdir -p gpurun_out
WGKV_K3=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest_k3v2.log 2>&1; echo pytest rc $?
tail -15 gpurun_out/r2_pytest_k3v2.log
bash tools/ab_env.sh 2 "WGKV_K3=1" "WGKV_K3=2" > gpurun_out/r2_k3_ab2.txt 2>&1
cat gpurun_out/r2_k3_ab2.txt
