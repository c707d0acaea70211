mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s3_pytest_gpu7.log 2>&1; echo pytest rc $?
tail -2 gpurun_out/r2s3_pytest_gpu7.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke7.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/r2s3_bench_v12.json 2> gpurun_out/r2s3_bench_v12.err; echo bench rc $?
for n in 8 4 2; do
  timeout 900 python bench.py --emulate-shard $n --no-cpu-baseline > gpurun_out/r2s3_bench_shard${n}_v12.json 2> gpurun_out/r2s3_bench_shard${n}_v12.err; echo shard $n rc $?
done
timeout 1200 python bench.py --config 32k --no-cpu-baseline > gpurun_out/r2s3_bench_32k_v12.json 2> gpurun_out/r2s3_bench_32k_v12.err; echo 32k rc $?
for f in v11 shard8_v12 shard4_v12 shard2_v12 32k_v12; do
python -c "import json; d=json.load(open('gpurun_out/r2s3_bench_$f.json')); print('$f', round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['executed']['frac'],3), round(d['decode_tok_s_per_gpu'],1), round(d['decode_roofline']['frac'],3), round(d['e2e']['value']), round(d['e2e']['decode_tok_s_per_gpu'],1), d['decode_kernels_per_layer'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
