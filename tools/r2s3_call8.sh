mkdir -p gpurun_out
for cfg in "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 32768 --batch 1 --hq 32 --hkv 8" "--T 131072 --batch 4 --hq 8 --hkv 2"; do
  echo "== $cfg"
  WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py $cfg 2>&1 | head -24
done
