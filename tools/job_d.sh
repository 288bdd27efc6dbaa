set -x
OUT=gpurun_out/r1s3f; mkdir -p $OUT
git_prev=/tmp/libcpd_prev.so
timeout 900 python tools/kern_time.py --config c5 2>&1 | tee $OUT/kt_c5.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "c5 or format or push or fullsize" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --kernel-name-base demangled -k "regex:k_dense" -s 2 -c 2 python tools/prof_run.py --iters 3 > $OUT/ncu.log 2>&1; grep -E "^  void|duration|bytes" $OUT/ncu.log | tail -6
