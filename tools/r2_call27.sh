mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider -k "tc_prefill or golden or gqa or configs2 or fragmented or shard" > gpurun_out/r2_pytest_rope.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/r2_pytest_rope.log
bash tools/ab_env.sh 3 "WGKV_LIB=build/var/libwgkv_base2.so" "X=1" > gpurun_out/r2_k3_ab10.txt 2>&1
cat gpurun_out/r2_k3_ab10.txt | grep -v "^ \|Trace\|json"
