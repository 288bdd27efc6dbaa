set -x
OUT=gpurun_out/r1s3c; mkdir -p $OUT
LIBS=paper_2511_13894_b200/libcpd.so
for V in "u6:-DCPD_SELL_U=6" "u12:-DCPD_SELL_U=12" "u6m5:-DCPD_SELL_U=6 -DCPD_SELL_MINB=5" "u4:-DCPD_SELL_U=4"; do
  T=${V%%:*}; D=${V#*:}
  CPD_LIB=/tmp/libcpd_$T.so CPD_BUILD_TAG=_$T CPD_NVCC_DEFS="$D" python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_$T.log 2>&1
  LIBS=$LIBS,/tmp/libcpd_$T.so
done
timeout 1500 python tools/kern_time.py --config c5 --corner 1 --libs $LIBS 2>&1 | tee $OUT/kt_c5.txt
