mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_attn_mma -s 40 -c 1 -o gpurun_out/k5_fused_32k -f python profiles/decode_layers.py --T 32768 --batch 1 --steps 2 > gpurun_out/k5_fused_ncu.log 2>&1; echo ncu rc $?
tail -3 gpurun_out/k5_fused_ncu.log
