set -x
mkdir -p gpurun_out
timeout 300 python profiles/decode_layers.py --T 32768 --batch 1 > gpurun_out/r2_declayers_32k.json 2>&1
timeout 600 python profiles/decode_layers.py --T 131072 --batch 4 --hq 4 --hkv 1 > gpurun_out/r2_declayers_shard8.json 2>&1
timeout 600 python profiles/decode_layers.py --T 131072 --batch 4 > gpurun_out/r2_declayers_128k.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_dec32k.csv -k regex:"decode|finish|gate|route|combine|assemble" python profiles/decode_layers.py --T 32768 --batch 1 --layers 4 --steps 2 > gpurun_out/r2_ncu_dec32k.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_decshard8.csv -k regex:"decode|finish|gate|route|combine|assemble" python profiles/decode_layers.py --T 131072 --batch 4 --hq 4 --hkv 1 --layers 4 --steps 2 > gpurun_out/r2_ncu_decshard8.log 2>&1
