set -x
OUT=gpurun_out/r1s2o; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_scaling.py -x -q > $OUT/pytest_scaling.log 2>&1; tail -25 $OUT/pytest_scaling.log
timeout 900 python tools/kern_time.py --config c5 --corner 1 2>&1 | tee $OUT/kt_c5.txt
timeout 900 python -c "
import bench, json; print(json.dumps(bench.time_to_eps(['c2','c3','c4'], 0), indent=1))" 2>&1 | tee $OUT/tte.txt
