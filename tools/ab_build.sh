#!/bin/bash
# Build the CUDA library of another commit (csrc + include) as
# paper_2603_14371_b200/liboxygen_b200.<name>.so for same-session A/B runs
# (OXY_LIB_VARIANT=<name>).  Usage: tools/ab_build.sh <commit> <name>
set -e
commit=$1; name=$2
tmp=$(mktemp -d)
git archive "$commit" paper_2603_14371_b200/csrc include | tar -x -C "$tmp"
sed -i "s#^OUT := ../liboxygen_b200.so#OUT := $(pwd)/paper_2603_14371_b200/liboxygen_b200.$name.so#" \
    "$tmp/paper_2603_14371_b200/csrc/Makefile"
make -s -j8 -C "$tmp/paper_2603_14371_b200/csrc" > /dev/null
rm -rf "$tmp"
echo "built paper_2603_14371_b200/liboxygen_b200.$name.so from $commit"
