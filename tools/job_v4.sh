set -x
OUT=gpurun_out/r1s2r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ineq.py -x -q > $OUT/pytest_ineq.log 2>&1; tail -15 $OUT/pytest_ineq.log
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
LIBS=paper_2511_13894_b200/libcpd.so
for V in "merge:-DCPD_SLAB_MERGE=1" "hb16:-DCPD_HB=16384" "du4:-DCPD_DU=4" "du16:-DCPD_DU=16"; do
  T=${V%%:*}; D=${V#*:}
  CPD_LIB=/tmp/libcpd_$T.so CPD_BUILD_TAG=_$T CPD_NVCC_DEFS="$D" python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_$T.log 2>&1
  LIBS=$LIBS,/tmp/libcpd_$T.so
done
timeout 1200 python tools/kern_time.py --config c5 --libs $LIBS 2>&1 | tee $OUT/kt_c5.txt
