mkdir -p gpurun_out
run() { # name, env, exchange
  env $2 timeout 600 python bench.py --emulate-shard 8 --decode-exchange $3 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/r2s3_x_$1.json 2>gpurun_out/r2s3_x_$1.err
  python -c "import json; d=json.load(open('gpurun_out/r2s3_x_$1.json')); print('$1', round(d['decode_tok_s_per_gpu'],1), round(d['decode_roofline']['frac'],3), d['decode_kernels_per_layer'], d['clocks']['sm_mhz'])"
}
for r in 1 2; do
run none X=1 none
run assemble X=1 nccl
run peer X=1 peer
run peer_notrig WGKV_PEER_TRIGGER=0 peer
run peer_gpu WGKV_PEER_SCOPE=gpu peer
run peer_one WGKV_PEER_ONE=1 peer
run peer_one_nopdl "WGKV_PEER_ONE=1 WGKV_PEER_PDL=0" peer
run peer_one_gpu "WGKV_PEER_ONE=1 WGKV_PEER_SCOPE=gpu" peer
done
