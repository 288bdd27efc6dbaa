set -x
OUT=gpurun_out/r1last; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1800 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo rc=$?; wc -l $OUT/bench.json
timeout 1200 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo rc=$?; wc -l $OUT/bench_ref.json
