mkdir -p gpurun_out
bash tools/ab_env.sh 2 "WGKV_K3=1" "WGKV_K3=2" "WGKV_K3=2 WGKV_LIB=build/var/libwgkv_v2sp0.so" "WGKV_K3=2 WGKV_LIB=build/var/libwgkv_v2sp3.so" "WGKV_K3=2 WGKV_LIB=build/var/libwgkv_v2e0.so" "WGKV_K3=2 WGKV_LIB=build/var/libwgkv_v2e516.so" > gpurun_out/r2_k3_ab5.txt 2>&1
WGKV_K3=2 WGKV_TRACE_V1=1 WGKV_LIB=build/var/libwgkv_v2sp1tr.so timeout 300 python profiles/prefill_breakdown.py --reps 1 --trace gpurun_out/k3v2sp_trace.npy > gpurun_out/r2_k3v2_trace.log 2>&1
cat gpurun_out/r2_k3_ab5.txt
