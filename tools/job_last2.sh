set -x
OUT=gpurun_out/r1last2; mkdir -p $OUT
bash tools/job_ct.sh 2>&1 | grep -E "create|plan|sell|renumber" | tail -9
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1800 python bench.py --tte '' --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo rc=$?; python -c "
import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'])"
