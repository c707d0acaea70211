mkdir -p gpurun_out
for cfg in "--T 32768 --batch 1" "--T 131072 --batch 4 --hq 4 --hkv 1" "--T 131072 --batch 4"; do
  for lib in d6s2c2 d8s3c1 d6s3c1 d8s2c1; do
  echo "== $cfg $lib"; WGKV_LIB=build/var/libwgkv_$lib.so timeout 300 python profiles/decode_layers.py $cfg --steps 30
  done
done > gpurun_out/r2_decode_ab10.txt 2>&1
