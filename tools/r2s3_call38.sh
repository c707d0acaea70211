mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn_mma --launch-skip 200 --launch-count 1 -o gpurun_out/r2s3_k5_fused_32k -f python profiles/decode_layers.py --T 32768 --batch 1 --steps 4 > gpurun_out/r2s3_ncu_k5.log 2>&1; echo ncu rc $?
