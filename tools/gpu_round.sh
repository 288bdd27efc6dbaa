#!/bin/bash
# Round deliverable session on one B200: build, gpu tests, smoke, bench (JSON line),
# ncu launch list of a short bench, ncu --set full of one iteration's hot kernels,
# corner study.  Usage: bash tools/gpu_round.sh TAG
TAG=${1:-round}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 1800 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 4000 $OUT/bench.json
if [ "${NCU:-1}" = "1" ]; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
     python bench.py --steps 1 --warmup 1 --iters1 256 --iters2 256 --no-e2e --no-cpu-baseline --tte '' > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
     -k "regex:EpiPrimalT|EpiDual|k_dense" -s 10 -c 12 -o $OUT/full python tools/prof_run.py --iters 3 > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
if [ "${STUDY:-1}" = "1" ]; then
  timeout 900 python tools/corner_study.py --out $OUT/corner_study > $OUT/corner_study.log 2>&1; echo "study rc=$?"
fi
