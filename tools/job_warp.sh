set -x
OUT=gpurun_out/r1s2d; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -15 $OUT/pytest_gpu.log
for c in c5 c3 c4 c2; do timeout 600 python tools/kern_time.py --config $c --corner 1 --env "CPD_WARP=0;CPD_WARP=1" 2>&1 | tee $OUT/kt_$c.txt; done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_sell|k_csrw" -s 4 -c 4 -o $OUT/warp python tools/prof_run.py --iters 3 > $OUT/ncu_warp.log 2>&1; tail -2 $OUT/ncu_warp.log
