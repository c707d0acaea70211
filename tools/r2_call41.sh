mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/r2_fuzz.log 2>&1; echo fuzz rc $?
tail -5 gpurun_out/r2_fuzz.log
bash tools/ab_decode.sh 3 "" base qlo 2>&1 | tee gpurun_out/r2_ab_qlo.txt
bash tools/ab_decode.sh 2 "--T 32768 --batch 1" base qlo 2>&1 | tee gpurun_out/r2_ab_qlo32k.txt
