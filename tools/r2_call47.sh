export WGKV_LIB=build/var/libwgkv_tl.so
timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --dump gpurun_out/tlf_32k.npz > gpurun_out/tlf_32k.json 2>&1; echo rc $?
timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --forced --dump gpurun_out/tlf_32kf.npz > gpurun_out/tlf_32kf.json 2>&1; echo rc $?
tail -3 gpurun_out/tlf_32k.json
