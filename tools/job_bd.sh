set -x
OUT=gpurun_out/r1s2x; mkdir -p $OUT
timeout 1200 python bench.py --force-dist --steps 1 --warmup 1 --iters1 256 --iters2 256 --tte '' --no-cpu-baseline > $OUT/bench_dist.json 2> $OUT/bench_dist.err; echo rc=$?; tail -c 1500 $OUT/bench_dist.json; tail -5 $OUT/bench_dist.err
timeout 1200 python bench.py --force-dist --partition 0 --steps 1 --warmup 1 --iters1 128 --iters2 128 --tte '' --no-cpu-baseline --no-e2e > $OUT/bench_dist0.json 2> $OUT/bench_dist0.err; echo rc=$?; tail -c 600 $OUT/bench_dist0.json; tail -5 $OUT/bench_dist0.err
timeout 900 python -c "
import lpgen, paper_2511_13894_b200 as cpd, json, time
lp = lpgen.config('c5'); P = cpd.Problem.from_lp(lp).scale(10, 1); S = cpd.Solver(P, max_iters=40000)
t = time.time(); r = S.solve(); print(json.dumps({k: r[k] for k in ('status','iterations','score','pobj','wall_s')}), lp.opt, time.time() - t)
" 2>&1 | tee $OUT/c5_scaled_tte.txt
