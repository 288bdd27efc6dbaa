#!/bin/bash
# Build libcpd variants with different stage-ring shared-memory budgets and time the hot kernels.
OUT=${OUT:-gpurun_out/tune}
mkdir -p $OUT
LIBS=""
for KB in ${KBS:-64 96 128 160 220}; do
  CPD_LIB=/tmp/libcpd_s$KB.so CPD_BUILD_TAG=_s$KB CPD_NVCC_DEFS="-DCPD_SMEM_KB=$KB $EXTRA_DEFS" \
    python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_s$KB.log 2>&1 || echo "build $KB failed"
  LIBS="$LIBS,/tmp/libcpd_s$KB.so"
done
python tools/kern_time.py --config ${CFG:-c5} --libs ${LIBS:1} --corner 1 2>&1 | tee $OUT/kern_time_${CFG:-c5}.txt
