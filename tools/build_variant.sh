#!/bin/bash
# Link a variant of librsvd_b200.so with one source recompiled under extra flags (experiments):
#   tools/build_variant.sh NAME SOURCE.cu "-DFLAG=1 ..."  ->  _variants/NAME/librsvd_b200.so (git-ignored; travels to the GPU box)
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; flags=$3
python -m paper_2110_03423_b200.build > /dev/null
out=_variants/$name
mkdir -p $out
obj=$out/$(basename $src .cu).o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
    -Iinclude -Ipaper_2110_03423_b200/csrc -Xptxas -warn-spills --expt-relaxed-constexpr $flags \
    -c paper_2110_03423_b200/csrc/$src -o $obj
objs=$(ls paper_2110_03423_b200/_lib/obj/*.o | grep -v "/$(basename $src .cu).o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/librsvd_b200.so $objs $obj -lcudart
echo $out/librsvd_b200.so
