#!/bin/bash
# Experiment build with the decode kernels' per-CTA %globaltimer timeline
# (csrc/timeline.cuh) -> build/var/libwgkv_tl.so; load with WGKV_LIB=build/var/libwgkv_tl.so
# and read with profiles/decode_timeline.py.  Not a product artefact.
set -e
cd "$(dirname "$0")/.."
make -s -j8 lib
mkdir -p build/var/tl
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -DWGKV_TIMELINE $*"
$NV -c paper_2512_17452_b200/csrc/decode_mma.cu -o build/var/tl/decode_mma.o
$NV -c paper_2512_17452_b200/csrc/decode_finish.cu -o build/var/tl/decode_finish.o
OBJ=$(ls build/*.o | grep -v -e '/decode_mma.o' -e '/decode_finish.o')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var/libwgkv_tl.so $OBJ build/var/tl/decode_mma.o build/var/tl/decode_finish.o -Xcompiler -fPIC -ldl
echo built build/var/libwgkv_tl.so
