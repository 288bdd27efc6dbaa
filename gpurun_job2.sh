set -x
OUT=gpurun_out/r1s2b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > $OUT/pytest_dist.log 2>&1; tail -3 $OUT/pytest_dist.log
OUT=$OUT timeout 1500 bash tools/tune_smem.sh
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:EpiPrimal|EpiDual" -s 3 -c 3 -o $OUT/full python tools/prof_run.py --iters 3 > $OUT/ncu_full.log 2>&1; tail -2 $OUT/ncu_full.log
