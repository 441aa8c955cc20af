#!/bin/bash
# Timing build of the working tree (-DOXY_ATTN_PROF -DOXY_GEMM_PROF): paper_2603_14371_b200/liboxygen_b200.aprof.so
# (read by tools/attn_prof.py and tools/gemm_prof.py)
set -e
tmp=$(mktemp -d)
mkdir -p "$tmp/paper_2603_14371_b200" "$tmp/include"
cp -r paper_2603_14371_b200/csrc "$tmp/paper_2603_14371_b200/csrc"; cp include/*.h "$tmp/include/"
rm -rf "$tmp/paper_2603_14371_b200/csrc/build"
make -s -j8 -C "$tmp/paper_2603_14371_b200/csrc" NVCC="nvcc -DOXY_ATTN_PROF -DOXY_GEMM_PROF ${EXTRA_DEFS}" \
    OUT="$(pwd)/paper_2603_14371_b200/liboxygen_b200.aprof.so" > /dev/null
rm -rf "$tmp"
echo built liboxygen_b200.aprof.so
