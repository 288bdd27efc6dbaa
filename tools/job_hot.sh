set -x
OUT=gpurun_out/r1s2z; mkdir -p $OUT
timeout 900 python tools/kern_time.py --config c5 --corner 1 --env "CPD_HOTROWS=0;CPD_HOTROWS=1" 2>&1 | tee $OUT/kt_c5.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -25 $OUT/pytest_gpu.log
