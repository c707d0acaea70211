mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -p no:cacheprovider -k "gate_bits or golden or tc_prefill or configs or shard or fragmented" > gpurun_out/r2_pytest_k1hs.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/r2_pytest_k1hs.log
bash tools/ab_k1.sh 3 "WGKV_LIB=build/var/libwgkv_k1ts.so" "WGKV_LIB=build/var/libwgkv_k1hs.so" > gpurun_out/r2_k1_ab2.txt 2>&1; cat gpurun_out/r2_k1_ab2.txt | grep -v "^ \|Trace\|json"
ncu --set full --clock-control none -k regex:gate_tc_kernel -s 2 -c 1 -o gpurun_out/r2_k1c_full python profiles/prefill_breakdown.py --reps 1 > /dev/null 2>&1
