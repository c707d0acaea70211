mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench_v3.json 2> gpurun_out/r2_bench_v3.err; echo bench rc $?
timeout 600 python bench.py --emulate-shard 8 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_shard8_v3.json 2>/dev/null; echo shard8 rc $?
timeout 600 python bench.py --emulate-shard 2 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_shard2_v3.json 2>/dev/null
timeout 600 python bench.py --emulate-shard 4 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_shard4_v3.json 2>/dev/null
timeout 600 python bench.py --config 32k --no-cpu-baseline > gpurun_out/r2_bench_32k_v3.json 2>/dev/null; echo 32k rc $?
timeout 900 python bench.py --config serve > gpurun_out/r2_bench_serve_v3.json 2>/dev/null; echo serve rc $?
timeout 900 python bench.py --config 1m > gpurun_out/r2_bench_1m_v3.json 2>/dev/null; echo 1m rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_128k.csv -k regex:"vs_prefill|gate|admit|decode|rope_table|combine|assemble|topk" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_launch_run.log 2>&1; echo ncu rc $?
