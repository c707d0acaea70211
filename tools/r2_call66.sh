WGKV_LIB=build/var/libwgkv_tl.so timeout 600 python profiles/decode_timeline.py --T 131072 --batch 4 --dump gpurun_out/tl2_128k.npz > gpurun_out/tl2_128k.json 2>&1; echo rc $?
WGKV_LIB=build/var/libwgkv_tl.so timeout 600 python profiles/decode_timeline.py --T 131072 --batch 4 --hq 16 --hkv 4 --dump gpurun_out/tl2_s2.npz > gpurun_out/tl2_s2.json 2>&1; echo rc $?
