mkdir -p gpurun_out
WGKV_K3=3 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "tc_prefill or golden or gqa" > gpurun_out/r2_pytest_k3v3.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/r2_pytest_k3v3.log
bash tools/ab_env.sh 2 "WGKV_K3=1" "WGKV_K3=3" > gpurun_out/r2_k3_ab7.txt 2>&1
cat gpurun_out/r2_k3_ab7.txt | grep -v "^ \|Trace\|json"
