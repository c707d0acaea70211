for r in 1 2; do
for v in ipc3 ipc2; do
  WGKV_LIB=build/var/libwgkv_$v.so timeout 600 python bench.py --config serve --no-cpu-baseline > gpurun_out/r2s3_serve_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r2s3_serve_$v.json')); print('$v', [round(x['decode_tok_s_per_gpu']) for x in d['sweep']])"
done
done
