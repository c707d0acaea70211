WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --dump gpurun_out/tl3_32k.npz > /dev/null 2>&1; echo $?
