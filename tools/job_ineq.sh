set -x
OUT=gpurun_out/r1s2q; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_ineq.py tests/test_gpu_scaling.py -x -q > $OUT/pytest_ineq.log 2>&1; tail -30 $OUT/pytest_ineq.log
timeout 900 python -c "
import bench, json; print(json.dumps(bench.time_to_eps(['c4-ineq'], 0), indent=1))" 2>&1 | tee $OUT/tte.txt
