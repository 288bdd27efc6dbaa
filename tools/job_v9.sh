set -x
OUT=gpurun_out/r1s3j; mkdir -p $OUT
LIBS=paper_2511_13894_b200/libcpd.so
for V in "s1m:-DCPD_SLAB_COLS=(1<<20)" "s2m:-DCPD_SLAB_COLS=(2<<20)" "s8m:-DCPD_SLAB_COLS=(8<<20)"; do
  T=${V%%:*}; D=${V#*:}
  CPD_LIB=/tmp/libcpd_$T.so CPD_BUILD_TAG=_$T CPD_NVCC_DEFS="$D" python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_$T.log 2>&1
  LIBS=$LIBS,/tmp/libcpd_$T.so
done
timeout 1500 python tools/kern_time.py --config c5 --libs $LIBS 2>&1 | tee $OUT/kt_c5.txt
