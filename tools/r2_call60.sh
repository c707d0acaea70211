mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench_v5.json 2> gpurun_out/r2_bench_v5.err; echo bench rc $?
for n in 8 4 2; do timeout 600 python bench.py --emulate-shard $n --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_shard${n}_v5.json 2>/dev/null; echo shard$n rc $?; done
timeout 600 python bench.py --config 32k --no-cpu-baseline > gpurun_out/r2_bench_32k_v5.json 2>/dev/null; echo 32k rc $?
for f in r2_bench_v5 r2_bench_shard8_v5 r2_bench_shard4_v5 r2_bench_shard2_v5 r2_bench_32k_v5; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['value']), d.get('decode_tok_s_per_gpu') and round(d['decode_tok_s_per_gpu']), d['roofline']['frac'] if 'roofline' in d else None, d.get('decode_roofline',{}).get('frac'), d.get('e2e',{}).get('value'))"; done
