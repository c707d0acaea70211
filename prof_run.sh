set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 3300 --csv --log-file gpurun_out/launches_128k.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:vs_prefill_tc -s 2 -c 1 -o gpurun_out/k3_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/k3_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn_mma -s 40 -c 1 -o gpurun_out/k5_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/k5_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate_prefill -s 2 -c 1 -o gpurun_out/k1_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/k1_run.log 2>&1
ls -la gpurun_out
