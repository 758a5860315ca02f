#!/bin/bash
# build_variant.sh <name> <extra nvcc flags...>  -> paper_2311_02542_b200/lib/ab/<name>.so
name=$1; shift
d=/tmp/variant_$name; mkdir -p $d
cd /root/repo/paper_2311_02542_b200/csrc
for f in lumi_api render_simt render_tc bake; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include "$@" -Xptxas -v -c $f.cu -o $d/$f.o 2> $d/$f.ptxas.txt || { cat $d/$f.ptxas.txt; exit 1; }
done
g++ -std=c++17 -O2 -fPIC -I../../include -c checkpoint.cpp -o $d/checkpoint.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../lib/ab/$name.so $d/*.o -lcudart
grep -A1 "k_render_tc" $d/render_tc.ptxas.txt | grep -E "registers|spill" | head -2
