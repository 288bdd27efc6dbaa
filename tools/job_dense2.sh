set -x
OUT=gpurun_out/r1s2j; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -5 $OUT/pytest_gpu.log
LIBS=paper_2511_13894_b200/libcpd.so
for V in "pre:-DCPD_PRE=1" "mb5:-DCPD_SELL_MINB=5 -DCPD_W_MINB=5"; do
  T=${V%%:*}; D=${V#*:}
  CPD_LIB=/tmp/libcpd_$T.so CPD_BUILD_TAG=_$T CPD_NVCC_DEFS="$D" python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_$T.log 2>&1
  LIBS=$LIBS,/tmp/libcpd_$T.so
done
timeout 900 python tools/kern_time.py --config c5 --corner 1 --libs $LIBS 2>&1 | tee $OUT/kt_c5.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --kernel-name-base demangled -k "regex:k_csrw|k_finish|k_sell|k_dense" -s 10 -c 16 python tools/prof_run.py --iters 3 > $OUT/ncu_seg.log 2>&1; grep -E "^  void|duration|bytes" $OUT/ncu_seg.log | tail -48
