timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_configs.py -x -q > gpurun_out/r2s3_trap_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/r2s3_trap_tests.log
timeout 900 python bench.py --emulate-shard 8 --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/r2s3_trap_s8.json 2>/dev/null; echo shard8 rc $?
python -c "import json; d=json.load(open('gpurun_out/r2s3_trap_s8.json')); print(round(d['value']), round(d['decode_tok_s_per_gpu'],1), round(d['decode_roofline']['frac'],3))"
