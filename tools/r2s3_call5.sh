mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s3_pytest_gpu2.log 2>&1; echo pytest rc $?
tail -5 gpurun_out/r2s3_pytest_gpu2.log
for n in 8 4 2; do
  timeout 900 python bench.py --emulate-shard $n --no-cpu-baseline > gpurun_out/r2s3_bench_shard$n.json 2> gpurun_out/r2s3_bench_shard$n.err; echo shard $n rc $?
  python -c "import json; d=json.load(open('gpurun_out/r2s3_bench_shard$n.json')); print($n, round(d['value']), round(d['decode_tok_s_per_gpu'],1), round(d['decode_roofline']['frac'],3), d['e2e']['decode_tok_s_per_gpu'], d['clocks'])"
done
