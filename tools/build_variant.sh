#!/bin/bash
# Build libsfxb_cuda.so with extra -D flags into lib_variants/NAME/ (A/B runs via SFXB_LIB).
#   tools/build_variant.sh NAME -DFLAG=... [-DFLAG2=...]
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/lib_variants/$name
mkdir -p "$out"
nvcc=/usr/local/cuda/bin/nvcc
arch="-gencode arch=compute_100a,code=sm_100a"
$nvcc $arch -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr "$@" \
  -c "$root/paper_2504_03909_b200/csrc/sfxb_cuda.cu" -o "$out/sfxb_cuda.o" &&
$nvcc $arch -shared -o "$out/libsfxb_cuda.so" "$out/sfxb_cuda.o" "$root/paper_2504_03909_b200/build/imad_peak.o" -lcudart -ldl &&
rm -f "$out/sfxb_cuda.o" && echo "built $out"
