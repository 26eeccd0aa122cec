#!/bin/bash
# tools/build_variant.sh NAME "-DFLAG ..." : build libotfgpu.so with extra nvcc flags into build/NAME/
# (A/B timing with tools/variants.sh; the in-tree library is untouched).
set -e
name=$1; shift
mkdir -p build/$name
make -s -C paper_2603_08417_b200/csrc EXTRA="$*" OUT=../../build/$name/libotfgpu.so ../../build/$name/libotfgpu.so
