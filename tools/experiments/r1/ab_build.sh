#!/bin/bash
# A/B experiment builds: tools/ab_build.sh NAME "-DFLAG=1 ..." -> tools/ab/NAME/libmvb200.so
# (run a variant with MV_LIB=tools/ab/NAME/libmvb200.so; the product build is untouched)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p tools/ab/$name/obj
MV_BUILD_OUT=tools/ab/$name/libmvb200.so MV_BUILD_OBJ=tools/ab/$name/obj MV_NVCC_EXTRA="$*" \
  python paper_2506_09991_b200/build.py
