mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/r2s3_peer_tests.log 2>&1; echo peer tests rc $?
tail -4 gpurun_out/r2s3_peer_tests.log
for n in 8 4 2; do
 for x in peer nccl; do
  timeout 900 python bench.py --emulate-shard $n --prefill-exchange $x --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/r2s3_pf_s${n}_$x.json 2> gpurun_out/r2s3_pf_s${n}_$x.err; echo shard $n $x rc $?
  python -c "import json; d=json.load(open('gpurun_out/r2s3_pf_s${n}_$x.json')); print($n, '$x', round(d['value']), round(d['roofline']['k3_share_of_prefill'],3), round(d['decode_roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/r2s3_pf_s${n}_$x.err
 done
done
