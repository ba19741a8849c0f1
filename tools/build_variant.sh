#!/bin/bash
# Builds an A/B variant of the engine: tools/build_variant.sh NAME "-DFLAG ..." -> build_var/NAME/libtdpgpu.so
# (select it with TDPG_LIB=build_var/NAME/libtdpgpu.so; the in-tree library is untouched).
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2
out=build_var/$name; mkdir -p "$out/src"; [ -e build_var/include ] || ln -s ../include build_var/include
cp paper_2503_11674_b200/csrc/*.cu paper_2503_11674_b200/csrc/*.cuh paper_2503_11674_b200/csrc/Makefile "$out/src/"
make -s -C "$out/src" -j8 NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --expt-relaxed-constexpr -Xcompiler -fPIC,-O2,-fvisibility=hidden -I$PWD/include -Xptxas -v $flags" LIB=../libtdpgpu.so
echo "$out/libtdpgpu.so"
