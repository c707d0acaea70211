set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:gate_tc_kernel -s 2 -c 1 -o gpurun_out/r2_k1_full python profiles/prefill_breakdown.py --reps 1 > gpurun_out/r2_k1_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"admit_scatter|admit_plan|gate_recheck" -c 3 -o gpurun_out/r2_k2_full python profiles/prefill_breakdown.py --reps 0 > gpurun_out/r2_k2_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate_proj_kernel -c 1 -o gpurun_out/r2_f1_full python profiles/proj_breakdown.py --reps 1 > gpurun_out/r2_f1_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn_mma -s 40 -c 1 -o gpurun_out/r2_k5b_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_k5b_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_finish -s 40 -c 1 -o gpurun_out/r2_finb_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_finb_run.log 2>&1
ls -la gpurun_out/*.ncu-rep
