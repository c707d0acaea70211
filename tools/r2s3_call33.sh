mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s3_pytest_gpu8.log 2>&1; echo pytest rc $?
tail -2 gpurun_out/r2s3_pytest_gpu8.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke8.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/r2s3_smoke8.log
timeout 900 python bench.py > gpurun_out/r2s3_bench_v13.json 2> gpurun_out/r2s3_bench_v13.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/r2s3_bench_v13.json')); print(round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['executed']['frac'],3), round(d['decode_tok_s_per_gpu'],1), round(d['decode_roofline']['frac'],3), round(d['e2e']['value']), round(d['e2e']['decode_tok_s_per_gpu'],1), d['gpu_launches'], d['clocks'])"
