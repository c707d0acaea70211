mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s3_pytest_gpu5.log 2>&1; echo pytest rc $?
tail -2 gpurun_out/r2s3_pytest_gpu5.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke5.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/r2s3_bench_v10.json 2> gpurun_out/r2s3_bench_v10.err; echo bench rc $?
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2s3_bench_reference.json 2>/dev/null; echo ref rc $?
python -c "import json; d=json.load(open('gpurun_out/r2s3_bench_v10.json')); print(round(d['value']), d['roofline']['frac'], d['roofline']['executed'], round(d['decode_tok_s_per_gpu'],1), round(d['decode_roofline']['frac'],3), round(d['e2e']['value']), d['clocks'])"
