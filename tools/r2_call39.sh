mkdir -p gpurun_out
WGKV_K3=4 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider -k "tc_prefill or golden or gqa or fragmented" > gpurun_out/r2_pytest_k3v4.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/r2_pytest_k3v4.log
bash tools/ab_env.sh 2 "WGKV_K3=1" "WGKV_K3=4" > gpurun_out/r2_k3_ab11.txt 2>&1
cat gpurun_out/r2_k3_ab11.txt | grep -v "^ \|Trace\|json"
WGKV_K3=4 WGKV_TRACE_FN=wgkv_dbg_k3_trace4 WGKV_LIB=build/var/libwgkv_v4tr.so timeout 300 python profiles/prefill_breakdown.py --reps 1 --trace gpurun_out/k3v4_trace.npy > gpurun_out/r2_k3v4_trace.log 2>&1
