set -x
OUT=gpurun_out/r1s3g; mkdir -p $OUT
timeout 900 python tools/kern_time.py --config c5 --corner 1 2>&1 | tee $OUT/kt_c5.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:k_finish" -s 4 -c 4 python tools/prof_run.py --iters 3 > $OUT/ncu.log 2>&1; grep -E "^  void|duration" $OUT/ncu.log | tail -8
