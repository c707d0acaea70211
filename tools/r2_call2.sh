set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -p no:cacheprovider -k "topk or ragged" > gpurun_out/r2_topk_tests.log 2>&1; echo topk rc $?
for n in 2 4 8; do timeout 600 python bench.py --emulate-shard $n --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_shard$n.json 2>gpurun_out/r2_bench_shard$n.err; echo shard $n rc $?; done
timeout 600 python bench.py --config 32k --no-cpu-baseline > gpurun_out/r2_bench_32k.json 2>gpurun_out/r2_bench_32k.err; echo 32k rc $?
timeout 900 python tools/dense_attn_compare.py > gpurun_out/r2_dense.json 2> gpurun_out/r2_dense.err; echo dense rc $?
