set -x
OUT=gpurun_out/r1s3b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
CPD_LIB=/tmp/libcpd_wl128.so CPD_BUILD_TAG=_wl128 CPD_NVCC_DEFS="-DCPD_WLONG=128" python -c "from paper_2511_13894_b200 import _build; _build.build(force=True)" > $OUT/build_wl128.log 2>&1
timeout 900 python tools/kern_time.py --config c5 --libs paper_2511_13894_b200/libcpd.so,/tmp/libcpd_wl128.so 2>&1 | tee $OUT/kt_c5.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 1200 python bench.py --steps 2 --warmup 1 --tte '' --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; python -c "
import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['e2e'], d['roofline']['frac'])"
