set -x
OUT=gpurun_out/r1s2y; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python bench.py --force-dist --steps 1 --warmup 1 --iters1 128 --iters2 128 --tte '' --no-cpu-baseline --no-e2e > $OUT/bench_dist.json 2> $OUT/bench_dist.err; echo rc=$?; head -c 300 $OUT/bench_dist.json; echo; wc -l $OUT/bench_dist.json
timeout 600 python bench.py --impl reference --config c2-s --steps 2 --warmup 1 > $OUT/bench_ref.json 2>$OUT/bench_ref.err; echo rc=$?; wc -l $OUT/bench_ref.json
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
