#!/bin/bash
# Builds an alternative libsvx_b200.so under variants/<name>/ with extra nvcc flags
# (kernel-variant A/B through SVX_LIB, scripts/ab_bench.sh).
# Usage: bash scripts/build_variant.sh <name> "<extra nvcc flags>"
set -e
name=$1; shift
out=$(cd "$(dirname "$0")/.." && pwd)/variants/$name
mkdir -p $out
make -s -C "$(dirname "$0")/../paper_2412_00291_b200/csrc" -j8 OUT=$out EXTRA="$*" $out/libsvx_b200.so
echo "built $out/libsvx_b200.so"
