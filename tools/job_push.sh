set -x
OUT=gpurun_out/r1s2u; mkdir -p $OUT
timeout 900 python tools/kern_time.py --config c5 --corner 1 --env "CPD_PUSH=1;CPD_PUSH=0" 2>&1 | tee $OUT/kt_c5.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -25 $OUT/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k "regex:EpiDual|k_dense|EpiPrimal" -s 6 -c 8 python tools/prof_run.py --iters 3 > $OUT/ncu.log 2>&1; grep -E "^  void|duration|bytes" $OUT/ncu.log | tail -32
