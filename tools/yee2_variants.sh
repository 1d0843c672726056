#!/bin/bash
# Build alternative two-step-sweep configurations of the product library into
# tools/ab_libs/ (git-ignored *.so; they travel with gpurun) for A/B timing:
#   bash tools/yee2_variants.sh NAME "-DYEE2_TY=16 -DYEE2_NT=672 -DYEE2_MB64=1 -DYEE2_MB32=2"
# then on the GPU: SFEEC_B200_LIB=tools/ab_libs/libNAME.so python bench.py ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; defs=$2
B=$ROOT/build/ab_$name
mkdir -p $B $ROOT/tools/ab_libs
cd $ROOT/paper_2301_01753_b200/csrc
make -s BUILD=$B OUT=$ROOT/tools/ab_libs/lib$name.so NVFLAGS_EXTRA="$defs"
