mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo bench rc $?
timeout 600 python bench.py --emulate-shard 8 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_shard8_final.json 2>/dev/null; echo shard8 rc $?
timeout 600 python bench.py --config 32k --no-cpu-baseline > gpurun_out/r2_bench_32k_final.json 2>/dev/null; echo 32k rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_final.csv -k regex:"vs_prefill|gate|admit|decode|rope_table|combine|assemble|topk" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_launch_final.log 2>&1; echo ncu rc $?
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2_bench_reference.json 2>/dev/null; echo ref rc $?
