#!/bin/bash
# Build a variant libntdgpu.so with one source recompiled under extra -D flags (experiments).
#   tools/variant_lib.sh NAME SOURCE.cu "-DFOO=1 -DBAR=2"   ->  build/var/libntdgpu_NAME.so
set -e
cd "$(dirname "$0")/.."
python -m paper_1909_09771_b200.build > /dev/null
NAME=$1; SRC=$2; DEFS=$3
mkdir -p build/var
BASE=$(basename $SRC .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 -Iinclude $DEFS -c paper_1909_09771_b200/csrc/$SRC -o build/var/${BASE}_$NAME.o
OBJS=$(ls build/ntdgpu/*.o | grep -v "/${BASE}.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var/libntdgpu_$NAME.so $OBJS build/var/${BASE}_$NAME.o -lcudart
echo build/var/libntdgpu_$NAME.so
