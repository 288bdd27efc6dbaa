set -x
OUT=gpurun_out/r1s2k; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
LIBS=paper_2511_13894_b200/libcpd.so
for V in "w512:-DCPD_WCAP_LONG=512" "w1024:-DCPD_WCAP_LONG=1024" "mb3:-DCPD_SELL_MINB=3 -DCPD_W_MINB=3"; do
  T=${V%%:*}; D=${V#*:}
  CPD_LIB=/tmp/libcpd_$T.so CPD_BUILD_TAG=_$T CPD_NVCC_DEFS="$D" python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_$T.log 2>&1
  LIBS=$LIBS,/tmp/libcpd_$T.so
done
timeout 900 python tools/kern_time.py --config c5 --corner 1 --libs $LIBS 2>&1 | tee $OUT/kt_c5.txt
