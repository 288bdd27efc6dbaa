set -x
OUT=gpurun_out/r1s3d; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1800 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo rc=$?; wc -l $OUT/bench.json
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:EpiPrimalT|EpiDual|k_dense" -s 10 -c 12 -o $OUT/full python tools/prof_run.py --iters 3 > $OUT/ncu_full.log 2>&1; echo ncu rc=$?
