mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_topk_launches.csv -k regex:"topk|decode|combine|append" python profiles/decode_breakdown.py --T 1048576 --batch 1 --hq 4 --hkv 1 --topk 256 --iters 3 > gpurun_out/r2s3_topk_ncu.log 2>&1; echo ncu rc $?
timeout 300 python profiles/decode_breakdown.py --T 1048576 --batch 1 --hq 4 --hkv 1 --topk 256 --iters 100 2>&1 | tail -1
