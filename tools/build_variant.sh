#!/bin/bash
# build_variant.sh <name> <extra nvcc flags...>  -> paper_2311_02542_b200/lib/ab/<name>.so
# (A/B experiments: LUMI_CUDA_LIB=paper_2311_02542_b200/lib/ab/<name>.so)
name=$1; shift
d=/tmp/variant_$name; rm -rf $d; mkdir -p $d
cd "$(dirname "$0")/../paper_2311_02542_b200/csrc" || exit 1
mkdir -p ../lib/ab
for f in *.cu; do
  extra=""
  [ "$f" = train.cu ] && extra="-fmad=false"  # as in the Makefile: the training path rounds like the reference
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $extra \
    -I../../include "$@" -Xptxas -v -c $f -o $d/${f%.cu}.o 2> $d/${f%.cu}.ptxas.txt || { cat $d/${f%.cu}.ptxas.txt; exit 1; }
done
for f in *.cpp; do g++ -std=c++17 -O2 -fPIC -pthread -I../../include -I/usr/local/cuda/include -c $f -o $d/${f%.cpp}.o; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../lib/ab/$name.so $d/*.o -lcudart
grep -h -A2 "k_render_ws\|k_march" $d/*.ptxas.txt | grep -E "registers|spill" | head -4
