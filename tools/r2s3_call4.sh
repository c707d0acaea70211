mkdir -p gpurun_out


run() { # name, shards, exchange
  timeout 600 python bench.py --emulate-shard $2 --decode-exchange $3 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/r2s3_y_$1.json 2>gpurun_out/r2s3_y_$1.err
  python -c "import json; d=json.load(open('gpurun_out/r2s3_y_$1.json')); print('$1', round(d['decode_tok_s_per_gpu'],1), round(d['decode_roofline']['frac'],3), d['decode_kernels_per_layer'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/r2s3_y_$1.err
}
for n in 8 4 2; do
run s${n}_none $n none
run s${n}_nccl $n nccl
run s${n}_peer $n peer
done
