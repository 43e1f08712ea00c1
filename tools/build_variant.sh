#!/bin/bash
# Build an experiment copy of the library with one object recompiled under
# extra -D flags:  tools/build_variant.sh TAG SRC.cu -DFOO=1 ...
# -> paper_2405_11353_b200/libntt_b200_TAG.so (load with NTT_LIB_PATH=...)
set -e
cd "$(dirname "$0")/.."
TAG=$1; SRC=$2; shift 2
OBJ=build/obj
mkdir -p build/var
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr --compress-mode=size -I include"
$NV "$@" -c paper_2405_11353_b200/csrc/$SRC -o build/var/${SRC%.cu}_$TAG.o
objs=$(ls $OBJ/*.o | grep -v "/${SRC%.cu}.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2405_11353_b200/libntt_b200_$TAG.so $objs build/var/${SRC%.cu}_$TAG.o -lcudart
echo built paper_2405_11353_b200/libntt_b200_$TAG.so
