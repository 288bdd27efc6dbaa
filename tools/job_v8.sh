set -x
OUT=gpurun_out/r1s3i; mkdir -p $OUT
LIBS=paper_2511_13894_b200/libcpd.so
for V in "sm512:-DCPD_SLAB_MIN=512" "sm2k:-DCPD_SLAB_MIN=2048" "sm8k:-DCPD_SLAB_MIN=8192"; do
  T=${V%%:*}; D=${V#*:}
  CPD_LIB=/tmp/libcpd_$T.so CPD_BUILD_TAG=_$T CPD_NVCC_DEFS="$D" python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_$T.log 2>&1
  LIBS=$LIBS,/tmp/libcpd_$T.so
done
timeout 1500 python tools/kern_time.py --config c5 --libs $LIBS 2>&1 | tee $OUT/kt_c5.txt
