#!/bin/bash
# Build a libcpd variant with extra nvcc defines into variants/libcpd_TAG.so (ships to
# the GPU box with the snapshot; git-ignored).  Usage: tools/build_variant.sh TAG "-DX=1 -DY=2"
TAG=$1
DEFS=$2
mkdir -p variants
CPD_LIB=$PWD/variants/libcpd_$TAG.so CPD_BUILD_TAG=_$TAG CPD_NVCC_DEFS="$DEFS" \
  python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > variants/build_$TAG.log 2>&1 \
  && echo "built variants/libcpd_$TAG.so" || { echo "build $TAG FAILED"; tail -20 variants/build_$TAG.log; }
