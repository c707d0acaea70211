mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_fused.log 2>&1; echo gpu rc $?
tail -15 gpurun_out/r2_pytest_fused.log
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4 --hq 8 --hkv 2"; do
  for f in 0 148; do
    echo "== $cfg fused_max=$f"
    WGKV_DECODE_FUSED=$f timeout 300 python profiles/decode_layers.py $cfg --steps 10 2>&1 | tail -1
  done
done
export WGKV_LIB=build/var/libwgkv_tl.so
timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --dump gpurun_out/tlf_32k.npz > gpurun_out/tlf_32k.json 2>&1; echo rc $?
timeout 300 python profiles/decode_timeline.py --T 131072 --batch 4 --hq 4 --hkv 1 --dump gpurun_out/tlf_s8.npz > gpurun_out/tlf_s8.json 2>&1; echo rc $?
