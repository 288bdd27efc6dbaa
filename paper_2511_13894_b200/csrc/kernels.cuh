// kernels.cuh — sm_100a device code for the R-PDHG + corner-push hot path.
//
// One kernel template does all sparse work: k_spmv<NV, Epi> walks a precomputed
// nnz-balanced PLAN of a CSR matrix (A or A^T), forms NV row sums of gathered
// vectors, and hands every finished row to a fused epilogue (the PDHG primal or
// dual step, the restart-check evaluations, the power iteration, the corner-model
// setup).  Epilogues accumulate the scalars the method needs (norms, dots,
// counts) in registers; a deterministic block reduction and a last-block-done
// grid combine turn them into totals, and the last block runs the epilogue's
// `finalize` (termination / restart / step-size decisions) ON THE DEVICE, so the
// host never synchronises inside a batch of iterations.
//
// Paper mapping (PAPER.md lines):
//   EpiPrimal  a2 + a5 + a6(n-side): x+ = proj(x - tau (c - A^T y)), x_avg, c^T x,
//              ||r_D||^2, dual-objective bound terms           (BJ north_star)
//   EpiDual    a3 + a4 + a5 + a6(m-side): y+ = y + sigma (b - (2 A x+ - A x)), y_avg,
//              ||b - A x+||^2, b^T y+                           (BJ north_star)
//   EpiCheckN/M  a7: KKT of current and average, restart decision, omega update
//   EpiCorner  a8: z = c - A^T y, Algorithm 1 bound map, Uniform objective
//   k_stats    a10: off-bound / zero-reduced-cost / candidate counts
// Deterministic: every sum is taken in a fixed order for a fixed grid.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <math.h>

namespace cpd {

constexpr int TPB = 256;       // threads per CTA of every hot kernel
constexpr int CAP = 2048;      // nonzeros per plan entry (8 per thread)
constexpr int RMAX = 512;      // rows per stream entry
constexpr int NSMAX = 12;      // max scalars an epilogue reduces

enum { MODE_FULL = 0, MODE_PRIMAL_ONLY = 1, MODE_NONE = 2 };
enum { ST_RUNNING = -1, ST_CONVERGED = 0, ST_ITER_LIMIT = 1, ST_TIME_LIMIT = 2, ST_FAIL = 3 };
enum { GATE_ALWAYS = 0, GATE_K1 = 1, GATE_K2 = 2, GATE_CHECK = 3, GATE_RESTART = 4 };

// Plan entry: stream entry {row0, row1, log2(threads per row), -1}
//             long chunk  {row, chunk, -1, long_id}
struct PlanEntry { int32_t a, b, c, d; };

struct DevPlan {
    const PlanEntry* ent;
    int32_t nent;
    int32_t nlong;
    const int64_t* long_off;   // [nlong] first chunk slot of each long row
    int32_t* long_cnt;         // [nlong] arrival counters (reset by the last arriver)
    double* long_part;         // [chunks * 2] chunk partial sums (NV <= 2)
    double* long_acc;          // [nlong * NSMAX] epilogue scalars of long rows
};

struct DevCsr {
    const int32_t* __restrict__ p;
    const int32_t* __restrict__ j;
    const double* __restrict__ x;
    int32_t rows;
};

// Bounds: per-element arrays, or uniform scalars when the array pointer is null.
struct Bounds {
    const double* l;
    const double* u;
    double l0, u0;
    __device__ __forceinline__ double lo(int j) const { return l ? l[j] : l0; }
    __device__ __forceinline__ double hi(int j) const { return u ? u[j] : u0; }
};

// Device control block: run configuration + state, read by every gate.
struct Ctl {
    // configuration of the current run
    int32_t mode, restart_on, K, traj_on;
    int64_t k_stop, max_iters, min_iters;
    double eps_rel, eps_abs, target, nb, nc;
    double beta_suff, beta_nec, beta_art, theta;
    // run state
    int64_t k, t, restarts, iterations;
    int32_t done, status, returned_average, check_pending;
    int32_t restart_flag, use_avg, nonfinite_x, pad;
    double eta, omega, tau, sigma;
    double S_r, S_prev;
    double rp2_cur, bty_cur;     // ||b - A x_k||^2 and b^T y_k (from the last dual step)
    double last[8];              // rp, rd, pobj, dobj, r_p, r_d, r_g, score of the last evaluated point
    double en[NSMAX];            // totals of the check's A^T pass
    // power iteration
    double pw_inv, pw_nrm, sigma_hat, step_scale;
    // trajectory
    int64_t traj_len, traj_cap;
    int64_t* traj_k;
    int64_t* traj_off;
    double* traj_rp;
    // generic totals written by one-off kernels (norms, stats, score)
    double out[NSMAX];
};

struct Gate {
    int32_t kind, slot, node;
    int32_t* active;   // optional: active[node] = 1 when the launch does work
};

// A gathered vector: fixed, or one of a ping-pong pair chosen by the device k
// (mode 1: buffer of iterate k+1, mode 2: buffer of iterate k).
struct VecSel {
    const double* a;
    const double* b;
    int32_t mode;
    __device__ __forceinline__ const double* get(const Ctl* c) const;
};

__device__ __forceinline__ bool gate_open(const Gate& g, const Ctl* c)
{
    switch (g.kind) {
    case GATE_K1:
        return !c->done && !c->check_pending && (c->k % c->K) == g.slot;
    case GATE_K2:
        return !c->done && !c->check_pending && (c->k % c->K) == g.slot && c->k < c->k_stop;
    case GATE_CHECK:
        return !c->done && c->check_pending;
    case GATE_RESTART:
        return !c->done && c->restart_flag;
    default:
        return true;
    }
}

__device__ __forceinline__ const double* VecSel::get(const Ctl* c) const
{
    if (mode == 0) return a;
    const int64_t kk = c->k + (mode == 1 ? 1 : 0);
    return (kk & 1) ? b : a;
}

__device__ __forceinline__ double proj(double v, double lo, double hi)
{
    double r = v > lo ? v : lo;   // max(v, lo)
    return r < hi ? r : hi;       // min(., hi)
}

// Counter-based U[0,1): SplitMix64 finalizer of seed + (j+1) * golden gamma
// (the (j+1)-th output of a SplitMix64 stream; SURVEY §8(c) "U(seed, j)").
__device__ __forceinline__ double u01(uint64_t seed, int64_t j)
{
    uint64_t s = seed + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ULL;
    s = (s ^ (s >> 30)) * 0xBF58476D1CE4E5B9ULL;
    s = (s ^ (s >> 27)) * 0x94D049BB133111EBULL;
    s ^= s >> 31;
    return (double)(s >> 11) * (1.0 / 9007199254740992.0);
}

// KKT score terms (S-3): o = {rp, rd, pobj, dobj, r_p, r_d, r_g, score}
__device__ __forceinline__ void score8(double rp2, double rd2, double pobj, double dobj,
                                       double nb, double nc, double* o)
{
    o[0] = sqrt(rp2);
    o[1] = sqrt(rd2);
    o[2] = pobj;
    o[3] = dobj;
    o[4] = o[0] / (1.0 + nb);
    o[5] = o[1] / (1.0 + nc);
    o[6] = fabs(pobj - dobj) / (1.0 + fabs(pobj) + fabs(dobj));
    double s = o[4];
    if (o[5] > s) s = o[5];
    if (o[6] > s) s = o[6];
    o[7] = s;
}

// Dual-side terms of one column for z = c_j - (A^T y)_j (S-6 reading of P:109-131):
// r_D_j = z - [l>-inf] max(z,0) + [u<inf] max(-z,0); bound part of the dual objective.
__device__ __forceinline__ void dual_terms(double z, double lo, double hi, double& rd2, double& bnd)
{
    double zp = z > 0.0 ? z : 0.0;
    double zm = -z > 0.0 ? -z : 0.0;
    double rd = z;
    if (lo > -INFINITY) { rd -= zp; bnd += lo * zp; }
    if (hi < INFINITY) { rd += zm; bnd -= hi * zm; }
    rd2 += rd * rd;
}

// ------------------------------------------------------------ reductions
template <int NS>
__device__ __forceinline__ void warp_sum(double (&v)[NS])
{
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[s] += __shfl_down_sync(0xffffffffu, v[s], o);
}

// Deterministic block reduction; result valid in thread 0.
template <int NS>
__device__ __forceinline__ void block_sum(double (&v)[NS], double (*sw)[NS])
{
    warp_sum<NS>(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int s = 0; s < NS; ++s) sw[w][s] = v[s];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            double t = 0.0;
            for (int i = 0; i < TPB / 32; ++i) t += sw[i][s];
            v[s] = t;
        }
    }
}

// Block partials -> last-block-done grid combine -> fin(totals) in thread 0 of the
// last block.  `extra` (nextra x NS) are extra per-item partials (long rows).
template <int NS, class Fin>
__device__ __forceinline__ void grid_finalize(double (&acc)[NS], double* bpart, unsigned* ctr,
                                              const double* extra, int nextra, Fin fin)
{
    __shared__ double sw[TPB / 32][NS];
    __shared__ int s_last;
    block_sum<NS>(acc, sw);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) bpart[(size_t)blockIdx.x * NS + s] = acc[s];
        __threadfence();
        unsigned prev = atomicAdd(ctr, 1u);
        s_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double tot[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) tot[s] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += TPB)
#pragma unroll
        for (int s = 0; s < NS; ++s) tot[s] += __ldcg(&bpart[(size_t)b * NS + s]);
    for (int l = threadIdx.x; l < nextra; l += TPB)
#pragma unroll
        for (int s = 0; s < NS; ++s) tot[s] += __ldcg(&extra[(size_t)l * NSMAX + s]);
    block_sum<NS>(tot, sw);
    if (threadIdx.x == 0) {
        fin(tot);
        *ctr = 0u;
        __threadfence();
    }
}

// ------------------------------------------------------------ SpMV + epilogue
// Row sums s_v = sum_k M_rk * vec_v[col_k] (v < NV) for every row r of M, each
// handed to epi.row(r, s, acc).  Stream entries stage the products of up to CAP
// nonzeros in shared memory (coalesced loads of col/val, one gather each), then
// 2^lg threads reduce each row; long rows (> CAP nonzeros) are split into CAP
// chunks whose partials the last-arriving CTA sums in chunk order.
template <int NV, class Epi>
__global__ void __launch_bounds__(TPB)
k_spmv(DevCsr M, DevPlan P, VecSel vs0, VecSel vs1, Epi epi, Gate gate, Ctl* ctl, double* bpart,
       unsigned* ctr)
{
    constexpr int NS = Epi::NS;
    __shared__ double s_prod[NV][CAP];
    __shared__ int32_t s_rp[RMAX + 1];
    __shared__ double s_w[TPB / 32][NV];
    __shared__ int s_go;
    if (threadIdx.x == 0) {
        s_go = gate_open(gate, ctl);
        if (s_go && gate.active && blockIdx.x == 0) gate.active[gate.node] = 1;
    }
    __syncthreads();
    if (!s_go) return;
    const double* __restrict__ v0 = vs0.get(ctl);
    const double* __restrict__ v1 = vs1.get(ctl);
    Epi e = epi;
    e.load(ctl);
    double acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    const int tid = threadIdx.x;

    for (int ei = blockIdx.x; ei < P.nent; ei += gridDim.x) {
        const PlanEntry E = P.ent[ei];
        if (E.c >= 0) {
            // ---------------- stream entry: rows [r0, r1)
            const int r0 = E.a, nr = E.b - E.a;
            for (int q = tid; q <= nr; q += TPB) s_rp[q] = M.p[r0 + q];
            __syncthreads();
            const int p0 = s_rp[0];
            const int cnt = s_rp[nr] - p0;
#pragma unroll 4
            for (int q = tid; q < cnt; q += TPB) {
                const int col = __ldg(&M.j[p0 + q]);
                const double a = __ldg(&M.x[p0 + q]);
                s_prod[0][q] = a * __ldg(&v0[col]);
                if (NV > 1) s_prod[NV - 1][q] = a * __ldg(&v1[col]);
            }
            __syncthreads();
            const int lg = E.c, tpr = 1 << lg, lane = tid & (tpr - 1);
            const int per_round = TPB >> lg;
            for (int base = 0; base < nr; base += per_round) {
                const int g = base + (tid >> lg);
                double s[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) s[v] = 0.0;
                if (g < nr) {
                    const int qa = s_rp[g] - p0, qb = s_rp[g + 1] - p0;
                    for (int q = qa + lane; q < qb; q += tpr)
#pragma unroll
                        for (int v = 0; v < NV; ++v) s[v] += s_prod[v][q];
                }
                for (int o = tpr >> 1; o > 0; o >>= 1)
#pragma unroll
                    for (int v = 0; v < NV; ++v) s[v] += __shfl_xor_sync(0xffffffffu, s[v], o);
                if (g < nr && lane == 0) e.row(r0 + g, s, acc);
            }
            __syncthreads();
        } else {
            // ---------------- long-row chunk
            const int row = E.a, chunk = E.b, lid = E.d;
            const int rp0 = M.p[row], rp1 = M.p[row + 1];
            const int q0 = rp0 + chunk * CAP;
            const int q1 = min(q0 + CAP, rp1);
            double s[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) s[v] = 0.0;
#pragma unroll 4
            for (int q = q0 + tid; q < q1; q += TPB) {
                const int col = __ldg(&M.j[q]);
                const double a = __ldg(&M.x[q]);
                s[0] += a * __ldg(&v0[col]);
                if (NV > 1) s[NV - 1] += a * __ldg(&v1[col]);
            }
            block_sum<NV>(s, s_w);
            if (tid == 0) {
                const int64_t off = P.long_off[lid];
#pragma unroll
                for (int v = 0; v < NV; ++v) P.long_part[(off + chunk) * 2 + v] = s[v];
                __threadfence();
                const int nch = (rp1 - rp0 + CAP - 1) / CAP;
                const int prev = atomicAdd(&P.long_cnt[lid], 1);
                if (prev == nch - 1) {
                    __threadfence();
                    double full[NV];
#pragma unroll
                    for (int v = 0; v < NV; ++v) full[v] = 0.0;
                    for (int c = 0; c < nch; ++c)
#pragma unroll
                        for (int v = 0; v < NV; ++v) full[v] += __ldcg(&P.long_part[(off + c) * 2 + v]);
                    P.long_cnt[lid] = 0;
                    double la[NS];
#pragma unroll
                    for (int s2 = 0; s2 < NS; ++s2) la[s2] = 0.0;
                    e.row(row, full, la);
#pragma unroll
                    for (int s2 = 0; s2 < NS; ++s2) P.long_acc[(size_t)lid * NSMAX + s2] = la[s2];
                }
            }
            __syncthreads();
        }
    }
    grid_finalize<NS>(acc, bpart, ctr, P.long_acc, P.nlong, [&](double* tot) { e.finalize(tot, ctl); });
}

// Elementwise pass over [0, N) with reductions and a device-side finalize.
template <class Op>
__global__ void __launch_bounds__(TPB)
k_elem(int64_t N, Op op, Gate gate, Ctl* ctl, double* bpart, unsigned* ctr)
{
    constexpr int NS = Op::NS;
    __shared__ int s_go;
    if (threadIdx.x == 0) {
        s_go = gate_open(gate, ctl);
        if (s_go && gate.active && blockIdx.x == 0) gate.active[gate.node] = 1;
    }
    __syncthreads();
    if (!s_go) return;
    Op o = op;
    o.load(ctl);
    double acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < N; i += (int64_t)gridDim.x * TPB)
        o.elem(i, acc);
    grid_finalize<NS>(acc, bpart, ctr, nullptr, 0, [&](double* tot) { o.finalize(tot, ctl); });
}

// ------------------------------------------------------------ epilogues
// Selects the ping-pong buffer of iterate k.
struct PingPong {
    double* b[2];
    __device__ __forceinline__ double* at(int64_t k) const { return b[k & 1]; }
};

// a2 + a5 + n-side of a6, and the per-iteration termination decision F(k).
struct EpiPrimal {
    static constexpr int NS = 4;   // c^T x_k, ||r_D(y_k)||^2, bound terms, #nonfinite(x_{k+1})
    const double* c;
    Bounds bd;
    PingPong X, Xa;
    // loaded
    double tau, inv_t1;
    const double* xc;
    double* xn;
    const double* xac;
    double* xan;
    double t1;
    __device__ void load(const Ctl* ctl)
    {
        tau = ctl->tau;
        t1 = (double)(ctl->t + 1);
        xc = X.at(ctl->k);
        xn = X.at(ctl->k + 1);
        xac = Xa.at(ctl->k);
        xan = Xa.at(ctl->k + 1);
    }
    __device__ __forceinline__ void row(int j, const double* s, double* acc) const
    {
        const double cj = c[j];
        const double z = cj - s[0];
        const double x = xc[j];
        const double lo = bd.lo(j), hi = bd.hi(j);
        const double xp = proj(x - tau * z, lo, hi);
        xn[j] = xp;
        const double xa = xac[j];
        xan[j] = xa + (xp - xa) / t1;
        acc[0] += cj * x;
        dual_terms(z, lo, hi, acc[1], acc[2]);
        acc[3] += isfinite(xp) ? 0.0 : 1.0;
    }
    // F(k): termination of iterate k (k >= 1, not a check iteration), P:124-126 / P:391-395.
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        ctl->restart_flag = 0;
        ctl->nonfinite_x = tot[3] > 0.0;
        const int64_t k = ctl->k;
        if (k == 0 || (k % ctl->K) == 0 || ctl->mode == MODE_NONE) return;
        double o[8];
        score8(ctl->rp2_cur, tot[1], tot[0], ctl->bty_cur + tot[2], ctl->nb, ctl->nc, o);
        for (int i = 0; i < 8; ++i) ctl->last[i] = o[i];
        bool conv = false;
        if (ctl->mode == MODE_FULL) conv = o[7] <= ctl->eps_rel;
        else conv = k >= ctl->min_iters && o[0] <= ctl->target;
        if (conv) {
            ctl->done = 1; ctl->status = ST_CONVERGED; ctl->iterations = k;
        } else if (k == ctl->max_iters) {
            ctl->done = 1; ctl->status = ST_ITER_LIMIT; ctl->iterations = k;
        }
    }
};

// a3 + a4 + a5 + m-side of a6: y+ = y + sigma (b - (2 A x+ - A x)).
struct EpiDual {
    static constexpr int NS = 3;   // ||b - A x_{k+1}||^2, b^T y_{k+1}, #nonfinite(y_{k+1})
    const double* b;
    double *y, *ya, *ax;
    double sigma, t1;
    __device__ void load(const Ctl* ctl)
    {
        sigma = ctl->sigma;
        t1 = (double)(ctl->t + 1);
    }
    __device__ __forceinline__ void row(int i, const double* s, double* acc) const
    {
        const double axn = s[0];
        const double bi = b[i];
        const double yo = y[i];
        const double yp = yo + sigma * (bi - (2.0 * axn - ax[i]));
        y[i] = yp;
        ax[i] = axn;
        const double yav = ya[i];
        ya[i] = yav + (yp - yav) / t1;
        const double r = bi - axn;
        acc[0] += r * r;
        acc[1] += bi * yp;
        acc[2] += isfinite(yp) ? 0.0 : 1.0;
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        ctl->rp2_cur = tot[0];
        ctl->bty_cur = tot[1];
        if (tot[2] > 0.0 || ctl->nonfinite_x) {
            ctl->done = 1; ctl->status = ST_FAIL; ctl->iterations = ctl->k + 1;
            return;
        }
        ctl->k += 1;
        ctl->t += 1;
        if ((ctl->k % ctl->K) == 0 && (ctl->restart_on || ctl->mode != MODE_NONE))
            ctl->check_pending = 1;
    }
};

// a7, A^T pass of a check: (A^T y_k), (A^T y_avg) -> current & average n-side terms.
struct EpiCheckN {
    static constexpr int NS = 9;   // ctx_c, rd2_c, bnd_c, dx2_c, ctx_a, rd2_a, bnd_a, dx2_a, off_bound(x_k; M)
    const double* c;
    Bounds bd;       // bounds of the run's model
    Bounds orig;     // original bounds (trajectory count)
    PingPong X, Xa;
    const double* xr;
    int two;         // 1: average term computed (second gathered vector present)
    double eps_abs;
    const double *xc, *xac;
    int traj;
    __device__ void load(const Ctl* ctl)
    {
        xc = X.at(ctl->k);
        xac = Xa.at(ctl->k);
        traj = ctl->traj_on;
        eps_abs = ctl->eps_abs;
    }
    __device__ __forceinline__ void row(int j, const double* s, double* acc) const
    {
        const double cj = c[j];
        const double lo = bd.lo(j), hi = bd.hi(j);
        const double x = xc[j];
        const double xrj = xr[j];
        acc[0] += cj * x;
        dual_terms(cj - s[0], lo, hi, acc[1], acc[2]);
        acc[3] += (x - xrj) * (x - xrj);
        if (two) {
            const double xa = xac[j];
            acc[4] += cj * xa;
            dual_terms(cj - s[1], lo, hi, acc[5], acc[6]);
            acc[7] += (xa - xrj) * (xa - xrj);
        }
        if (traj) acc[8] += ((x - orig.lo(j) > eps_abs) && (orig.hi(j) - x > eps_abs)) ? 1.0 : 0.0;
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        for (int i = 0; i < NS; ++i) ctl->en[i] = tot[i];
    }
};

// a7, A pass of a check: A x_avg (kept for a restart to the average), m-side terms,
// then the check decision (termination of current / average, restart, omega).
struct EpiCheckM {
    static constexpr int NS = 4;   // rp2_a, bty_a, dy2_c, dy2_a
    const double *b, *y, *ya, *yr;
    double* axa;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int i, const double* s, double* acc) const
    {
        axa[i] = s[0];
        const double bi = b[i];
        const double r = bi - s[0];
        acc[0] += r * r;
        const double yav = ya[i], yo = y[i], yri = yr[i];
        acc[1] += bi * yav;
        acc[2] += (yo - yri) * (yo - yri);
        acc[3] += (yav - yri) * (yav - yri);
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        const double* en = ctl->en;
        const int64_t k = ctl->k;
        double oc[8], oa[8];
        score8(ctl->rp2_cur, en[1], en[0], ctl->bty_cur + en[2], ctl->nb, ctl->nc, oc);
        for (int i = 0; i < 8; ++i) ctl->last[i] = oc[i];
        if (ctl->traj_on && ctl->traj_len < ctl->traj_cap) {
            ctl->traj_k[ctl->traj_len] = k;
            ctl->traj_off[ctl->traj_len] = (int64_t)en[8];
            ctl->traj_rp[ctl->traj_len] = oc[0];
            ctl->traj_len += 1;
        }
        ctl->check_pending = 0;
        if (ctl->mode == MODE_FULL && oc[7] <= ctl->eps_rel) {
            ctl->done = 1; ctl->status = ST_CONVERGED; ctl->iterations = k;
            return;
        }
        if (ctl->mode == MODE_PRIMAL_ONLY && k >= ctl->min_iters && oc[0] <= ctl->target) {
            ctl->done = 1; ctl->status = ST_CONVERGED; ctl->iterations = k;
            return;
        }
        if (ctl->restart_on) {
            score8(tot[0], en[5], en[4], tot[1] + en[6], ctl->nb, ctl->nc, oa);
            const double S_c = oc[7], S_a = oa[7];
            if (ctl->mode == MODE_FULL && S_a <= ctl->eps_rel) {
                for (int i = 0; i < 8; ++i) ctl->last[i] = oa[i];
                ctl->done = 1; ctl->status = ST_CONVERGED; ctl->iterations = k;
                ctl->returned_average = 1;
                return;
            }
            const int use_avg = S_a < S_c;           // tie -> current (S-14)
            const double S = use_avg ? S_a : S_c;
            if (S <= ctl->beta_suff * ctl->S_r ||
                (S <= ctl->beta_nec * ctl->S_r && S > ctl->S_prev) ||
                (double)ctl->t >= ctl->beta_art * (double)k) {
                const double dx = sqrt(use_avg ? en[7] : en[3]);
                const double dy = sqrt(use_avg ? tot[3] : tot[2]);
                if (dx > 1e-10 && dy > 1e-10)
                    ctl->omega = exp(ctl->theta * log(dy / dx) + (1.0 - ctl->theta) * log(ctl->omega));
                ctl->tau = ctl->eta / ctl->omega;
                ctl->sigma = ctl->eta * ctl->omega;
                if (use_avg) {
                    ctl->rp2_cur = tot[0];
                    ctl->bty_cur = tot[1];
                }
                ctl->restart_flag = 1;
                ctl->use_avg = use_avg;
                ctl->S_r = S;
                ctl->S_prev = INFINITY;
                ctl->t = 0;
                ctl->restarts += 1;
            } else {
                ctl->S_prev = S;
            }
        }
        if (ctl->mode != MODE_NONE && k == ctl->max_iters) {
            ctl->done = 1; ctl->status = ST_ITER_LIMIT; ctl->iterations = k;
        }
    }
};

// Restart apply: (x, y, Ax) <- candidate; (x_r, y_r) <- (x, y); averages <- 0.
struct OpRestart {
    static constexpr int NS = 1;
    PingPong X, Xa;
    double *y, *ya, *ax, *axa, *xr, *yr;
    int32_t n, m;
    int use_avg;
    double *xc, *xac;
    __device__ void load(const Ctl* ctl)
    {
        use_avg = ctl->use_avg;
        xc = X.at(ctl->k);
        xac = Xa.at(ctl->k);
    }
    __device__ __forceinline__ void elem(int64_t i, double*) const
    {
        if (i < n) {
            double v = use_avg ? xac[i] : xc[i];
            xc[i] = v;
            xr[i] = v;
            xac[i] = 0.0;
        }
        if (i < m) {
            double v = use_avg ? ya[i] : y[i];
            if (use_avg) ax[i] = axa[i];
            y[i] = v;
            yr[i] = v;
            ya[i] = 0.0;
        }
    }
    __device__ void finalize(const double*, Ctl*) const {}
};

// Run start: x_0 = proj(x_init), y_0 = y_init (or 0), references, zero averages.
struct OpBegin {
    static constexpr int NS = 1;
    const double *xs, *ys;    // sources (may alias destinations elementwise)
    Bounds bd;
    double *x0, *xa0, *xa1, *xr, *y, *ya, *yr;
    int32_t n, m;
    int zero_y;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void elem(int64_t i, double*) const
    {
        if (i < n) {
            const double v = proj(xs[i], bd.lo((int)i), bd.hi((int)i));
            x0[i] = v;
            xr[i] = v;
            xa0[i] = 0.0;
            xa1[i] = 0.0;
        }
        if (i < m) {
            const double v = zero_y ? 0.0 : ys[i];
            y[i] = v;
            yr[i] = v;
            ya[i] = 0.0;
        }
    }
    __device__ void finalize(const double*, Ctl*) const {}
};

// ||b||^2, ||c||^2 -> nb, nc, omega0, tau, sigma (S-8).
struct OpNorms {
    static constexpr int NS = 2;
    const double *b, *c;
    int32_t n, m;
    double omega_in;   // > 0: given
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void elem(int64_t i, double* acc) const
    {
        if (i < m) acc[0] += b[i] * b[i];
        if (i < n) acc[1] += c[i] * c[i];
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        ctl->nb = sqrt(tot[0]);
        ctl->nc = sqrt(tot[1]);
        if (omega_in > 0.0) ctl->omega = omega_in;
        else ctl->omega = (ctl->nc > 1e-10 && ctl->nb > 1e-10) ? ctl->nc / ctl->nb : 1.0;
        ctl->tau = ctl->eta / ctl->omega;
        ctl->sigma = ctl->eta * ctl->omega;
        if (ctl->mode == MODE_PRIMAL_ONLY) ctl->target = ctl->eps_rel * (1.0 + ctl->nb);
    }
};

// Run-start evaluation: A x_0 -> Ax buffer, ||b - A x_0||^2, b^T y_0.
struct EpiInitM {
    static constexpr int NS = 2;
    const double *b, *y;
    double* ax;   // may be null (score only)
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int i, const double* s, double* acc) const
    {
        if (ax) ax[i] = s[0];
        const double r = b[i] - s[0];
        acc[0] += r * r;
        acc[1] += b[i] * y[i];
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        ctl->rp2_cur = tot[0];
        ctl->bty_cur = tot[1];
    }
};

// Run-start evaluation: A^T y_0 -> S_r = score(x_0, y_0); FULL: converged at k = 0?
struct EpiInitN {
    static constexpr int NS = 3;
    const double *c, *x;
    Bounds bd;
    int decide;   // 0: only store the score in ctl->last
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int j, const double* s, double* acc) const
    {
        const double cj = c[j];
        acc[0] += cj * x[j];
        dual_terms(cj - s[0], bd.lo(j), bd.hi(j), acc[1], acc[2]);
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        double o[8];
        score8(ctl->rp2_cur, tot[1], tot[0], ctl->bty_cur + tot[2], ctl->nb, ctl->nc, o);
        for (int i = 0; i < 8; ++i) ctl->last[i] = o[i];
        if (!decide) return;
        ctl->S_r = o[7];
        ctl->S_prev = INFINITY;
        if (ctl->mode == MODE_FULL && o[7] <= ctl->eps_rel) {
            ctl->done = 1; ctl->status = ST_CONVERGED; ctl->iterations = 0;
        }
    }
};

// Power iteration (S-2): v0 = U(seed, j) - 0.5; w = (A v) * inv; v = A^T w.
struct OpPowInit {
    static constexpr int NS = 1;
    double* v;
    uint64_t seed;
    int32_t n;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void elem(int64_t j, double* acc) const
    {
        const double x = u01(seed, j) - 0.5;
        v[j] = x;
        acc[0] += x * x;
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        ctl->pw_inv = 1.0 / sqrt(tot[0]);
    }
};
struct EpiPowM {
    static constexpr int NS = 1;
    double* w;
    double inv;
    __device__ void load(const Ctl* ctl) { inv = ctl->pw_inv; }
    __device__ __forceinline__ void row(int i, const double* s, double*) const { w[i] = s[0] * inv; }
    __device__ void finalize(const double*, Ctl*) const {}
};
struct EpiPowN {
    static constexpr int NS = 1;
    double* v;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int j, const double* s, double* acc) const
    {
        v[j] = s[0];
        acc[0] += s[0] * s[0];
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        const double nu = sqrt(tot[0]);
        ctl->pw_nrm = nu;
        ctl->pw_inv = 1.0 / nu;
        ctl->sigma_hat = sqrt(nu);
        ctl->eta = ctl->step_scale / ctl->sigma_hat;
    }
};

// a8: z = c - A^T y*, Algorithm 1 bound map, Uniform objective.
struct EpiCorner {
    static constexpr int NS = 2;   // fix_lb, fix_ub
    const double *c, *x;
    Bounds bd;
    double *z, *lhat, *uhat, *chat;
    const double* obj;   // caller objective (device copy) or null
    double eps_abs, obj_scale;
    uint64_t seed;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int j, const double* s, double* acc) const
    {
        const double zj = c[j] - s[0];
        z[j] = zj;
        const double xj = x[j];
        if (zj < -eps_abs) { lhat[j] = xj; acc[0] += 1.0; } else lhat[j] = bd.lo(j);
        if (zj > eps_abs) { uhat[j] = xj; acc[1] += 1.0; } else uhat[j] = bd.hi(j);
        chat[j] = obj ? obj[j] : obj_scale * u01(seed, j);
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        ctl->out[0] = tot[0];
        ctl->out[1] = tot[1];
    }
};

// a10 corner statistics: counts as exact fp64 sums (< 2^53).
struct OpStats {
    static constexpr int NS = 6;   // off, off_strict, off_model, zero_rc, candidates, (spare)
    const double *x, *z, *lh, *uh;
    Bounds bd;
    double eps;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ static bool off(double x, double lo, double hi, double tol)
    {
        return (x - lo > tol) && (hi - x > tol);
    }
    __device__ __forceinline__ void elem(int64_t jj, double* acc) const
    {
        const int j = (int)jj;
        const double xj = x[j];
        const bool o = off(xj, bd.lo(j), bd.hi(j), eps);
        acc[0] += o;
        acc[1] += off(xj, bd.lo(j), bd.hi(j), 0.0);
        if (lh) acc[2] += off(xj, lh[j], uh[j], eps);
        if (z) {
            const double az = fabs(z[j]);
            acc[3] += az <= eps;
            acc[4] += o && az < eps;
        }
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        for (int i = 0; i < NS; ++i) ctl->out[i] = tot[i];
    }
};

}  // namespace cpd
