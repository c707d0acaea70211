mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/r2_fuzz.log 2>&1; echo fuzz rc $?
tail -3 gpurun_out/r2_fuzz.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo gpu rc $?
tail -3 gpurun_out/r2_pytest_gpu.log
bash tools/ab_decode.sh 3 "" base qrow 2>&1 | tee gpurun_out/r2_ab_qrow.txt
bash tools/ab_decode.sh 2 "--T 32768 --batch 1" base qrow 2>&1 | tee gpurun_out/r2_ab_qrow32k.txt
