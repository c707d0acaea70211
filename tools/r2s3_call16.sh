mkdir -p gpurun_out
timeout 1200 python bench.py --config serve --no-cpu-baseline > gpurun_out/r2s3_bench_serve_v9.json 2> gpurun_out/r2s3_bench_serve_v9.err; echo serve rc $?
timeout 1200 python bench.py --config 1m --no-cpu-baseline > gpurun_out/r2s3_bench_1m_v9.json 2> gpurun_out/r2s3_bench_1m_v9.err; echo 1m rc $?
