# Problem-creation timing on C5 through the public API (pinned host buffers), with
# the phase timer (CPD_TIMING=1); optional env variants as arguments ("CPD_SHORT=0").
OUT=gpurun_out/r1ct; mkdir -p $OUT
for V in "${@:-default}"; do
env $( [ "$V" = default ] || echo "$V" ) CPD_TIMING=1 timeout 600 python -c "
import time, lpgen, numpy as np, torch, paper_2511_13894_b200 as cpd
lp = lpgen.config('c5')
pin = {}
for k in ('ATp','ATj','ATx','b','c','lb','ub'):
    a = getattr(lp, k); t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True); t.numpy()[...] = a; pin[k] = t.numpy()
for rep in range(2):
    t0 = time.time()
    P = cpd.Problem(lp.m, lp.n, AT=(pin['ATp'], pin['ATj'], pin['ATx']), b=pin['b'], c=pin['c'], lb=pin['lb'], ub=pin['ub'])
    t1 = time.time(); S = cpd.Solver(P, max_iters=64); t2 = time.time()
    print('$V', 'create', round(t1-t0,3), 'solver', round(t2-t1,3), flush=True)
    S.close(); P.close()
" > $OUT/ct_${V//[=,]/_}.log 2>&1; cat $OUT/ct_${V//[=,]/_}.log
done
