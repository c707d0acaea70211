mkdir -p gpurun_out
export WGKV_LIB=build/var/libwgkv_tl.so
timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --dump gpurun_out/tl_32k.npz > gpurun_out/tl_32k.json 2>&1; echo rc $?
timeout 300 python profiles/decode_timeline.py --T 131072 --batch 4 --hq 4 --hkv 1 --dump gpurun_out/tl_s8.npz > gpurun_out/tl_s8.json 2>&1; echo rc $?
timeout 300 python profiles/decode_timeline.py --T 131072 --batch 4 --hq 4 --hkv 1 --forced --dump gpurun_out/tl_s8f.npz > gpurun_out/tl_s8f.json 2>&1; echo rc $?
timeout 600 python profiles/decode_timeline.py --T 131072 --batch 4 --dump gpurun_out/tl_128k.npz > gpurun_out/tl_128k.json 2>&1; echo rc $?
head -c 600 gpurun_out/tl_32k.json
