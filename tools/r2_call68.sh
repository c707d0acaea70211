mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench_v6.json 2> gpurun_out/r2_bench_v6.err; echo bench rc $?
for n in 8 4 2; do timeout 600 python bench.py --emulate-shard $n --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_shard${n}_v6.json 2>/dev/null; echo shard$n rc $?; done
timeout 600 python bench.py --config 32k --no-cpu-baseline > gpurun_out/r2_bench_32k_v6.json 2>/dev/null; echo 32k rc $?
timeout 900 python bench.py --config serve > gpurun_out/r2_bench_serve_v6.json 2>gpurun_out/r2_bench_serve_v6.err; echo serve rc $?
timeout 900 python bench.py --config 1m > gpurun_out/r2_bench_1m_v6.json 2>gpurun_out/r2_bench_1m_v6.err; echo 1m rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3300 --csv --log-file gpurun_out/r2_launches_128k_v6.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_launch_run_v6.log 2>&1; echo ncu1 rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_launches_32k_v6.csv python bench.py --config 32k --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_launch_run32_v6.log 2>&1; echo ncu2 rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn_mma -s 40 -c 1 -o gpurun_out/r2_k5fused_full python bench.py --config 32k --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_k5f_run.log 2>&1; echo ncu3 rc $?
