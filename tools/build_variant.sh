#!/bin/bash
# Build a tuning variant of libvfmm.so into build/<name>/ with extra nvcc flags:
#   tools/build_variant.sh u4 -DVFMM_RING_UNROLL=4
# then select it at run time with VFMM_LIB=build/<name>/libvfmm.so.
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build/$name
mkdir -p "$out"
src=$root/paper_0809_1810_b200/csrc
objs=()
for f in capi tree upward subtree m2l downward p2p shard; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v "$@" -c "$src/$f.cu" -o "$out/$f.o" \
    2> "$out/$f.ptxas.log" &
  objs+=("$out/$f.o")
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libvfmm.so" "${objs[@]}"
echo "$out/libvfmm.so"
