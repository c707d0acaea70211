export WGKV_LIB=build/var/libwgkv_tl.so
WGKV_K5_NO_TRIGGER=1 timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --forced --dump gpurun_out/tlf_32kf_nt.npz > gpurun_out/tlf_32kf_nt.json 2>&1; echo rc $?
timeout 300 python profiles/decode_timeline.py --T 32768 --batch 1 --layers 1 --forced --dump gpurun_out/tlf_32kf_l1.npz > gpurun_out/tlf_32kf_l1.json 2>&1; echo rc $?
tail -3 gpurun_out/tlf_32kf_l1.json
