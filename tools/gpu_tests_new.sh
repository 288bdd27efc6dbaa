#!/bin/bash
# New-test session: build, then the given pytest selection (default: round-2 GPU test files).
TAG=${1:-new}
shift
SEL=${@:-tests/test_gpu_errors.py tests/test_gpu_fullpaths.py tests/test_gpu_fullsize.py}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 2400 python -m pytest $SEL -m gpu -q -rA --durations=30 > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -40 $OUT/pytest.log
