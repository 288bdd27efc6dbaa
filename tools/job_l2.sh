set -x
OUT=gpurun_out/r1s2w; mkdir -p $OUT
timeout 900 python tools/kern_time.py --config c5 --env "CPD_L2FETCH=0;CPD_L2FETCH=32;CPD_L2FETCH=64;CPD_L2FETCH=128" 2>&1 | tee $OUT/kt_c5.txt
CPD_L2FETCH=32 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k "regex:EpiDual|k_dense|EpiPrimal" -s 6 -c 8 python tools/prof_run.py --iters 3 > $OUT/ncu32.log 2>&1; grep -E "^  void|duration|bytes" $OUT/ncu32.log | tail -32
