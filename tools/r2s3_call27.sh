WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --dump gpurun_out/tl32k.npz 2>&1 | head -70
