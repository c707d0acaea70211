mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/r2s3_peer_tests.log 2>&1; echo peer tests rc $?
tail -30 gpurun_out/r2s3_peer_tests.log
for n in 8 4 2; do
 for x in peer nccl; do
  timeout 600 python bench.py --emulate-shard $n --decode-exchange $x --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/r2s3_shard${n}_$x.json 2> gpurun_out/r2s3_shard${n}_$x.err; echo shard $n $x rc $?
  python -c "import json; d=json.load(open('gpurun_out/r2s3_shard${n}_$x.json')); print('$n $x', round(d['decode_tok_s_per_gpu'],1), round(d['decode_roofline']['frac'],3), d['decode_kernels_per_layer'], d['clocks']['sm_mhz'])"
 done
done
