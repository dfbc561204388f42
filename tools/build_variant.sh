#!/bin/bash
# Developer tool: build a variant of the library with extra -D defines for rm_fft.cu only, reusing the other
# objects of an RM_OBJ_CACHE build (python -m paper_1805_06688_b200.build with RM_OBJ_CACHE=/tmp/rmobj).
#   tools/build_variant.sh NAME -DRM_STAGE_NB=9 ...   ->  paper_1805_06688_b200/_lib/var_NAME.so  (use with RM_LIB=...)
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
cache=${RM_OBJ_CACHE:-/tmp/rmobj}/plain
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  -Xptxas -v "$@" -I "$root/include" -I "$root/paper_1805_06688_b200/csrc" -c "$root/paper_1805_06688_b200/csrc/rm_fft.cu" \
  -o "$cache/../var_$name.o" 2> "$cache/../var_$name.ptxas"
objs=$(ls "$cache"/*.o | grep -v rm_fft.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/paper_1805_06688_b200/_lib/var_$name.so" $objs "$cache/../var_$name.o" -lcudart
grep -A2 "chain_fft_kernelILi2" "$cache/../var_$name.ptxas" | grep -o "[0-9]* bytes spill stores, [0-9]* bytes spill loads\|Used [0-9]* registers" | tr '\n' ' '; echo " <- $name"
