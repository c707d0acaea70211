mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "graph" > gpurun_out/r2_graph_test.log 2>&1; echo graphtest rc $?; tail -3 gpurun_out/r2_graph_test.log
timeout 2400 compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q -p no:cacheprovider -k "not configs2_layer and not configs0 and not gate_proj_fused and not many_pairs" > gpurun_out/r2_memcheck.log 2>&1; echo memcheck rc $?; tail -4 gpurun_out/r2_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "gqa4_two_seqs and bf16" > gpurun_out/r2_racecheck1.log 2>&1; echo race1 rc $?; tail -3 gpurun_out/r2_racecheck1.log
timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_configs.py -q -p no:cacheprovider -k "gate_proj_fused and 512" > gpurun_out/r2_racecheck2.log 2>&1; echo race2 rc $?; tail -3 gpurun_out/r2_racecheck2.log
timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "ragged_batch_decode" > gpurun_out/r2_racecheck3.log 2>&1; echo race3 rc $?; tail -3 gpurun_out/r2_racecheck3.log
