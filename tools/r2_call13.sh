mkdir -p gpurun_out
timeout 600 python profiles/proj_breakdown.py > gpurun_out/r2_proj.json 2>&1; echo proj rc $?
timeout 900 python bench.py > gpurun_out/r2_bench_v2.json 2> gpurun_out/r2_bench_v2.err; echo bench rc $?
timeout 600 python bench.py --emulate-shard 8 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_shard8_v2.json 2>/dev/null; echo shard8 rc $?
timeout 600 python bench.py --config 32k --no-cpu-baseline > gpurun_out/r2_bench_32k_v2.json 2>/dev/null; echo 32k rc $?
timeout 600 ./oracle/_ref/dropin_session > gpurun_out/r2_dropin.log 2>&1; echo dropin rc $?
