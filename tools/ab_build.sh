#!/bin/bash
# Build a variant of libda_b200.so for A/B timing runs: tools/ab_build.sh NAME [EXTRA nvcc flags]
# Sources come from $AB_SRC (default: the package's csrc); the library lands in
# tools/ab/NAME/libda_b200.so (git-ignored, travels to the GPU box).  Run with
# DA_LIB_PATH=tools/ab/NAME/libda_b200.so.
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
NAME=$1; shift
SRC="${AB_SRC:-$ROOT/paper_1509_05194_b200/csrc}"
W=/tmp/ab_$NAME
rm -rf "$W"; mkdir -p "$W/pkg/csrc" "$W/include"
cp "$SRC"/*.cu "$SRC"/*.cuh "$SRC"/*.h "$SRC"/Makefile "$W/pkg/csrc/"
cp "$ROOT"/include/*.h "$W/include/"
make -s -C "$W/pkg/csrc" -j16 EXTRA="$*" > /dev/null
mkdir -p "$ROOT/tools/ab/$NAME"
cp "$W/pkg/libda_b200.so" "$ROOT/tools/ab/$NAME/"
grep -A2 "beam_fast_kernelIfLb1ELb1E" "$W/pkg/csrc/build/encode_fast.ptxas.log" | grep -E "registers|spill" | tr '\n' ' '; echo " <- $NAME"
