set -x
OUT=gpurun_out/r1s2v; mkdir -p $OUT
LIBS=paper_2511_13894_b200/libcpd.so
for V in "na:-DCPD_NOALLOC=1" "pre:-DCPD_PRE=1 -DCPD_SELL_MINB=3"; do
  T=${V%%:*}; D=${V#*:}
  CPD_LIB=/tmp/libcpd_$T.so CPD_BUILD_TAG=_$T CPD_NVCC_DEFS="$D" python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_$T.log 2>&1
  LIBS=$LIBS,/tmp/libcpd_$T.so
done
timeout 900 python tools/kern_time.py --config c5 --libs $LIBS 2>&1 | tee $OUT/kt_c5.txt
timeout 600 python tools/kern_time.py --config c3 --libs $LIBS 2>&1 | tee $OUT/kt_c3.txt
timeout 600 python tools/kern_time.py --config c4 --libs $LIBS 2>&1 | tee $OUT/kt_c4.txt
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -k p2p > $OUT/pytest_p2p.log 2>&1; tail -15 $OUT/pytest_p2p.log
