mkdir -p gpurun_out
bash tools/ab_env.sh 3 "WGKV_K3=1" "WGKV_K3=1 WGKV_LIB=build/var/libwgkv_m8.so" "WGKV_K3=2" > gpurun_out/r2_k3_ab4.txt 2>&1
WGKV_K3=2 WGKV_TRACE_V1=1 WGKV_LIB=build/var/libwgkv_v2tr.so timeout 300 python profiles/prefill_breakdown.py --reps 1 --trace gpurun_out/k3v2m8_trace.npy > gpurun_out/r2_k3v2_trace.log 2>&1
cat gpurun_out/r2_k3_ab4.txt
