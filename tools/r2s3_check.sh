mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s3_pytest_gpu.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/r2s3_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/r2s3_bench.json 2> gpurun_out/r2s3_bench.err; echo bench rc $?
cat gpurun_out/r2s3_bench.json
