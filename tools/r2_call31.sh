mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -s -p no:cacheprovider -k "gate_proj" > gpurun_out/r2_f1b.log 2>&1; echo rc $?; grep -E "passed|failed|gate_proj dm" gpurun_out/r2_f1b.log
timeout 600 python profiles/proj_breakdown.py > gpurun_out/r2_proj_v2.json 2>&1; cat gpurun_out/r2_proj_v2.json
