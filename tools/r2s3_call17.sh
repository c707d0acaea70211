WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 2>&1 | head -90
WGKV_LIB=build/var/libwgkv_tl.so timeout 300 python profiles/decode_timeline.py --T 131072 --batch 4 --hq 4 --hkv 1 2>&1 | head -20
