#!/bin/bash
# Build the working tree's CUDA library with extra preprocessor defines as
# paper_2603_14371_b200/liboxygen_b200.<name>.so (OXY_LIB_VARIANT=<name> A/B runs).
#   tools/def_build.sh <name> "-DFOO -DBAR"
set -e
name=$1; defs=$2
tmp=$(mktemp -d)
mkdir -p "$tmp/paper_2603_14371_b200" "$tmp/include"
cp -r paper_2603_14371_b200/csrc "$tmp/paper_2603_14371_b200/csrc"; cp include/*.h "$tmp/include/"
rm -rf "$tmp/paper_2603_14371_b200/csrc/build"
make -s -j8 -C "$tmp/paper_2603_14371_b200/csrc" NVCC="nvcc $defs" \
    OUT="$(pwd)/paper_2603_14371_b200/liboxygen_b200.$name.so" > /dev/null
rm -rf "$tmp"
echo "built liboxygen_b200.$name.so ($defs)"
