mkdir -p gpurun_out
bash tools/ab_env.sh 2 "WGKV_K3=1" "WGKV_K3=3 WGKV_LIB=build/var/libwgkv_v3a.so" "WGKV_K3=3 WGKV_LIB=build/var/libwgkv_v3b.so" "WGKV_K3=3 WGKV_LIB=build/var/libwgkv_v3c.so" > gpurun_out/r2_k3_ab9.txt 2>&1
WGKV_K3=3 WGKV_TRACE_FN=wgkv_dbg_k3_trace3 WGKV_LIB=build/var/libwgkv_v3atr.so timeout 300 python profiles/prefill_breakdown.py --reps 1 --trace gpurun_out/k3v3a_trace.npy > gpurun_out/r2_k3v3_trace.log 2>&1
cat gpurun_out/r2_k3_ab9.txt | grep -v "^ \|Trace\|json"
