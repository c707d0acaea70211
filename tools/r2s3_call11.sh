WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 131072 --batch 4 2>&1 | head -60
