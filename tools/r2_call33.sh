mkdir -p gpurun_out
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4 --hq 8 --hkv 2" "--T 131072 --batch 4"; do
  for lib in c24 c64 c96 c64d1 c128d1; do
  echo "== $cfg $lib"; WGKV_LIB=build/var/libwgkv_$lib.so timeout 300 python profiles/decode_layers.py $cfg --steps 30
  done
done > gpurun_out/r2_decode_ab9.txt 2>&1
