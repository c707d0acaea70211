mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q -x -k "not configs2_layer and not configs0 and not gate_proj_fused and not many_pairs and not fuzz" > gpurun_out/r2_memcheck2.log 2>&1; echo memcheck rc $?
tail -3 gpurun_out/r2_memcheck2.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -k "gqa4_two_seqs and bf16" > gpurun_out/r2_racecheck4.log 2>&1; echo racecheck rc $?
tail -3 gpurun_out/r2_racecheck4.log
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -q -k "gqa4_two_seqs and bf16" > gpurun_out/r2_synccheck.log 2>&1; echo synccheck rc $?
tail -3 gpurun_out/r2_synccheck.log
