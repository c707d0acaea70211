set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 3300 --csv --log-file gpurun_out/r2_launches_128k.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:vs_prefill_tc -s 2 -c 1 -o gpurun_out/r2_k3_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_k3_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn_mma -s 40 -c 1 -o gpurun_out/r2_k5_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_k5_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_finish -s 40 -c 1 -o gpurun_out/r2_fin_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_fin_run.log 2>&1
timeout 900 python bench.py --config serve > gpurun_out/r2_bench_serve.json 2>gpurun_out/r2_bench_serve.err
timeout 900 python bench.py --config 1m > gpurun_out/r2_bench_1m.json 2>gpurun_out/r2_bench_1m.err
ls -la gpurun_out
