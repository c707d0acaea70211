#!/bin/bash
# Whole-library experiment build with extra defines: tools/full_variant.sh NAME -DFOO=1 ...
# -> build/var/libwgkv_NAME.so (load with WGKV_LIB=...); not a product artefact.
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
mkdir -p build/var/$NAME
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr $*"
for f in paper_2512_17452_b200/csrc/*.cu; do b=$(basename $f .cu); $NV -c $f -o build/var/$NAME/$b.o & done; wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var/libwgkv_$NAME.so build/var/$NAME/*.o -Xcompiler -fPIC -ldl
echo built build/var/libwgkv_$NAME.so
