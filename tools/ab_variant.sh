#!/bin/bash
# Build a kernel variant from a git revision (or a csrc directory) into
# paper_2605_17923_b200/_lib/variants/<name>.so; select it at run time with AL_LIB_VARIANT=<name>.
# Extra nvcc flags via $AB_NVCC_FLAGS (e.g. -DAL_CTA_TRACE for the per-CTA timestamp build).
#   tools/ab_variant.sh <name> <git-rev | csrc-dir>
set -euo pipefail
name=$1; src=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
mkdir -p "$tmp/p/csrc" "$tmp/include"
if [ -d "$src" ]; then
  cp -r "$src"/. "$tmp/p/csrc/"; cp "$root/include/adaln_b200.h" "$tmp/include/"
else
  for f in adaln_capi.cu adaln_kernels.cuh bwd_steal.cuh block_kernels.cuh dtype.cuh ptx.cuh instances_extern.inc; do
    git -C "$root" show "$src:paper_2605_17923_b200/csrc/$f" > "$tmp/p/csrc/$f"; done
  git -C "$root" show "$src:include/adaln_b200.h" > "$tmp/include/adaln_b200.h"
fi
mkdir -p "$root/paper_2605_17923_b200/_lib/variants"
nvcc -gencode=arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -cudart static -DAL_MONOLITHIC ${AB_NVCC_FLAGS:-} \
  -o "$root/paper_2605_17923_b200/_lib/variants/$name.so" "$tmp/p/csrc/adaln_capi.cu"
rm -rf "$tmp"
echo "built variants/$name.so"
