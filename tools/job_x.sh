set -x
OUT=gpurun_out/r1s2n; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
CPD_LIB=/tmp/libcpd_x0.so CPD_BUILD_TAG=_x0 CPD_NVCC_DEFS="-DCPD_XLAST=0" python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_x0.log 2>&1
timeout 900 python tools/kern_time.py --config c5 --corner 1 --libs paper_2511_13894_b200/libcpd.so,/tmp/libcpd_x0.so 2>&1 | tee $OUT/kt_c5.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -5 $OUT/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --kernel-name-base demangled -k "regex:EpiDual|k_dense|k_sell" -s 14 -c 14 python tools/prof_run.py --iters 3 > $OUT/ncu_seg.log 2>&1; grep -E "^  void|duration|bytes" $OUT/ncu_seg.log | tail -56
