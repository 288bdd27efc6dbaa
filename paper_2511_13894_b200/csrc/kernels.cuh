// kernels.cuh — sm_100a device code for the R-PDHG + corner-push hot path.
//
// Every sparse pass forms NV row sums of gathered vectors and hands each finished
// row to a fused epilogue (the PDHG primal or dual step, the restart-check
// evaluations, the power iteration, the corner-model setup, the split-product
// store).  Three engines stream the matrix:
//   k_sell   SELL-32 copy of a short-row layout (A^T): warp = 32 rows, lane = row,
//            coalesced streaming, L1 / shared-memory gathers;
//   k_csrw   warp items of a CSR plan (A with long rows): rows items via a segmented
//            warp scan, long-row pieces per column slab, k_dense for the heavy rows
//            by dense column blocks in shared memory, k_finish per long row;
//   k_spmv   the persistent TMA (cp.async.bulk + mbarrier) ring for other CSR plans.
// Epilogues accumulate the scalars the method needs (norms, dots, counts) in
// registers; a deterministic block reduction and a last-block-done grid combine
// turn them into totals, and the last block runs the epilogue's `finalize`
// (termination / restart / step-size decisions) ON THE DEVICE, so the host never
// synchronises inside a batch of iterations.
//
// Paper mapping (PAPER.md lines):
//   EpiPrimal  a2 + a5 + a6(n-side): x+ = proj(x - tau (c - A^T y)), x_avg, c^T x,
//              ||r_D||^2, dual-objective bound terms           (BJ north_star)
//   EpiDual    a3 + a4 + a5 + a6(m-side): y+ = y + sigma (b - (2 A x+ - A x)), y_avg,
//              ||b - A x+||^2, b^T y+                           (BJ north_star)
//   EpiCheckN/M  a7: KKT of current and average, restart decision, omega update
//   EpiCorner  a8: z = c - A^T y, Algorithm 1 bound map, Uniform objective
//   OpStats    a10: off-bound / zero-reduced-cost / candidate counts
// Deterministic: every sum is taken in a fixed order for a fixed grid (the opt-in
// short-row push, CPD_PUSH=1, is the one exception: fp64 atomics).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <math.h>
#include <type_traits>

namespace cpd {

constexpr int TPB = 256;       // threads per CTA of every hot kernel
constexpr int CAP = 2048;      // nonzeros per plan entry (one TMA stage)
constexpr int RMAX = 256;      // rows per rows-entry
constexpr int SINGLE_MIN = 256;  // a row with more nonzeros gets an entry of its own (block reduce)
constexpr int NSTAGE = 3;      // TMA pipeline depth (stages per CTA)
constexpr int NVECMAX = 5;     // staged per-row vectors per entry
constexpr int NSMAX = 12;      // max scalars an epilogue reduces
#ifndef CPD_WCAP_ROWS
#define CPD_WCAP_ROWS 1024
#endif
#ifndef CPD_WLONG
#define CPD_WLONG 128
#endif
constexpr int WCAP_ROWS = CPD_WCAP_ROWS;  // k_csrw: nonzeros per rows item (<= 32 rows)
constexpr int WLONG = CPD_WLONG;          // k_csrw: a longer row is cut into pieces
#ifndef CPD_WCAP_LONG
#define CPD_WCAP_LONG 512
#endif
constexpr int WCAP_LONG = CPD_WCAP_LONG;  // k_csrw: nonzeros per long-row piece
#ifndef CPD_HEAVY_MIN
#define CPD_HEAVY_MIN 131072
#endif
constexpr int HEAVY_MIN = CPD_HEAVY_MIN; // k_dense: rows with at least this many nonzeros
#ifndef CPD_HB
#define CPD_HB 8192
#endif
constexpr int HB = CPD_HB;       // k_dense: columns per dense block (64 KB of the vector in smem)
#ifndef CPD_DCHUNK
#define CPD_DCHUNK 512
#endif
constexpr int DCHUNK = CPD_DCHUNK;   // k_dense: entries per item (balances the Zipf head across warps)
#ifndef CPD_TPB_D
#define CPD_TPB_D 512
#endif
constexpr int TPB_D = CPD_TPB_D;
constexpr int FIN_SPLIT = 1024;
#ifndef CPD_FIN_G
#define CPD_FIN_G 8
#endif
constexpr int FIN_G = CPD_FIN_G;   // k_finish lanes per (non-heavy) long row
constexpr int TPB_F = 256;       // k_finish threads per CTA (1024 measured slower: 52 vs 45 us)
constexpr int HOT_ROWS = 4096;
#ifndef CPD_HOTY_FUSED
#define CPD_HOTY_FUSED 2048
#endif
constexpr int HOT_ROWS_FUSED = CPD_HOTY_FUSED;   // staged y entries of the fused primal step (smem budget)
#ifndef CPD_HOTY
#define CPD_HOTY 2048
#endif
// staged y entries of the other A^T SELL passes (C5: 4096 halves the two-vector check
// pass's occupancy, 1.90 vs 0.95 ms — profiles/r02_kernel_iterations.md)
constexpr int HOT_ROWS_STAGED = CPD_HOTY;   // y entries of the longest rows of A staged in k_sell's shared memory  // k_finish: rows with more partials get a CTA, the rest a warp

enum { MODE_FULL = 0, MODE_PRIMAL_ONLY = 1, MODE_NONE = 2, MODE_DUAL_ONLY = 3 };
enum { ST_RUNNING = -1, ST_CONVERGED = 0, ST_ITER_LIMIT = 1, ST_TIME_LIMIT = 2, ST_FAIL = 3 };
enum { GATE_ALWAYS = 0, GATE_K1 = 1, GATE_K2 = 2, GATE_CHECK = 3, GATE_RESTART = 4 };

// Plan entry (16 B):
//   rows entry  {r0, r1, p0, p1}: rows [r0, r1) whose nonzeros are [p0, p1) (<= CAP)
//   long piece  {slot, -1 - long_id, q0, q1}: nonzeros [q0, q1) of a long row, all inside
//               one column slab (SURVEY §7 "gather locality"); its GW warp partials go
//               to lpart[(slot * GW + wg) * 2 + v] (slots of one row are contiguous)
struct PlanEntry { int32_t a, b, p0, p1; };

struct DevPlan {
    const PlanEntry* ent;
    int32_t nent;
    int32_t nlong;
    int32_t pslot;             // warp partials per piece slot (GW: k_spmv, 1: k_csrw)
    int32_t nheavy, nhb;       // heavy rows / dense column blocks (k_dense)
    const PlanEntry* dense_ent;   // {slot, block, q0, q1}: <= DCHUNK entries of one heavy row in one block
    const int32_t* dense_ptr;     // [nhb + 1] items of each block
    const uint16_t* dense_col16;  // [nnz] heavy-row entries: column offset inside their HB block (12 -> 10 B/entry)
    int32_t dense_maxitems;       // most items in one block (k_dense item-sum smem)
    const int32_t* short_ptr;     // [nslab][rows + 1] short-row entries by slab (k_csrw slab mode)
    const int32_t* short_col;
    const double* short_val;
    double* short_part;           // [NV][rows] running sums across slab passes
    double* push_acc;             // short-row sums pushed by the primal step (k_csrw rows items read + zero)
    const int32_t* long_row;   // [nlong] row index of each long row
    const int32_t* long_ptr;   // [nlong + 1] piece slots of each long row (column order)
    const int32_t* long_ents;  // k_finish order: nfin_heavy rows (a CTA each), then the rest (a warp each)
    int32_t nfin_heavy;
    double* lpart;             // [pieces * GW * 2] warp partial sums (NV <= 2)
    // fused dual step (hot-row fusion): long rows l < hotd (= internal rows 0..hotd-1)
    // are summed from the primal step's per-warp partials hot_part[l * hot_stride + w]
    int32_t hotd = 0, hot_stride = 0;
    const double* hot_part = nullptr;
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
    // reflected restarted Halpern PDHG + PID primal weight (NEXT-1; H-1..H-4)
    int32_t method, pid;
    double rho, kp, ki, kd;
    double r0, r_prev, r_last;          // fixed-point residuals: at the anchor, last check, last iteration
    double pid_int, pid_eprev;
    double dx2_h, dxa2_h, dya2_h;       // ||xh - x||^2, ||xh - x_anchor||^2, ||yh - y_anchor||^2 (last iteration)
    double rp2_h, bty_h;                // ||b - A xh||^2, b^T yh of the last T(z)
};

// Primal-weight update at a restart from the anchor movement (dx, dy): theta smoothing
// (R-PDHG, S-1) or the PID controller on e = log(dy/dx) - log omega (reading H-3).
__device__ __forceinline__ void weight_update(Ctl* ctl, double dx, double dy)
{
    if (!(dx > 1e-10 && dy > 1e-10)) return;
    if (ctl->pid) {
        const double e = log(dy / dx) - log(ctl->omega);
        ctl->pid_int += e;
        const double lw = log(ctl->omega) + ctl->kp * e + ctl->ki * ctl->pid_int + ctl->kd * (e - ctl->pid_eprev);
        ctl->pid_eprev = e;
        ctl->omega = exp(lw);
    } else {
        ctl->omega = exp(ctl->theta * log(dy / dx) + (1.0 - ctl->theta) * log(ctl->omega));
    }
}

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

// L2 eviction-priority helpers: the primal iterate x+ (gathered by the next dual
// step) is written / gathered evict-last so it outlives the streamed matrix data
// in L2 (CPD_XLAST=0 disables, for A/B measurements).
#ifndef CPD_XLAST
#define CPD_XLAST 1
#endif
__device__ __forceinline__ void st_keep(double* p, double v)
{
#if CPD_XLAST
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#else
    *p = v;
#endif
}
__device__ __forceinline__ double ld_keep(const double* p)
{
#if CPD_XLAST
    uint64_t pol;
    double v;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
#else
    return __ldg(p);
#endif
}

// Streamed (read-once) loads of matrix indices / values: evict-first in L1 and L2
// (ld.global.cs), or with CPD_NOALLOC=1 not allocated in L1 at all.
#ifndef CPD_NOALLOC
#define CPD_NOALLOC 0
#endif
__device__ __forceinline__ int32_t ld_stream(const int32_t* p)
{
#if CPD_NOALLOC
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}
__device__ __forceinline__ int32_t ld_stream(const uint16_t* p)
{
    return (int32_t)__ldcs((const unsigned short*)p);
}
__device__ __forceinline__ double ld_stream(const double* p)
{
#if CPD_NOALLOC
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}
__device__ __forceinline__ int2 ld_stream(const int2* p)
{
#if CPD_NOALLOC
    int2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}
__device__ __forceinline__ double2 ld_stream(const double2* p)
{
#if CPD_NOALLOC
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}

// Bulk L2 prefetch of a byte range (cp.async.bulk.prefetch.L2, sm_90+): one
// instruction, no registers or shared memory held, fire and forget.  The streamed
// matrix ranges of the work item CPD_PF items ahead are pulled into L2 so the
// dependent index -> gather chain of the item pays L2 latency, not DRAM latency.
#ifndef CPD_PF
#define CPD_PF 0
#endif
__device__ __forceinline__ void l2_prefetch(const void* p, int64_t bytes)
{
    if (bytes <= 0) return;
    const uint64_t a = (uint64_t)p & ~15ull;
    const uint64_t e = ((uint64_t)p + (uint64_t)bytes + 15ull) & ~15ull;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a)) : "memory");
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
// w: 1 / s_j of a diagonally scaled problem (z = z^ / s_j in the original space, the
// violation scales the same way; the bound terms l^ z^+ = l z+ need no weight)
// Returns r_D_j (the dual corner push counts |r_D_j| > eps_abs, reading D-3).
__device__ __forceinline__ double dual_terms(double z, double lo, double hi, double& rd2, double& bnd,
                                             double w = 1.0)
{
    double zp = z > 0.0 ? z : 0.0;
    double zm = -z > 0.0 ? -z : 0.0;
    double rd = z;
    if (lo > -INFINITY) { rd -= zp; bnd += lo * zp; }
    if (hi < INFINITY) { rd += zm; bnd -= hi * zm; }
    rd *= w;
    rd2 += rd * rd;
    return rd;
}

// Implicit inequality rows: sense 0 '=', 1 '<=' (Ax <= b),
// 2 '>=' (Ax >= b).  r = b - Ax counts its violation only; the dual of L = c^T x +
// y^T (b - A x) is projected onto y >= 0 ('>=') / y <= 0 ('<=').
__device__ __forceinline__ double row_viol(const int8_t* sn, int i, double r)
{
    if (!sn) return r;
    const int s = sn[i];
    return s == 1 ? (r < 0.0 ? r : 0.0) : s == 2 ? (r > 0.0 ? r : 0.0) : r;
}
__device__ __forceinline__ double dual_proj(const int8_t* sn, int i, double v)
{
    if (!sn) return v;
    const int s = sn[i];
    return s == 1 ? (v < 0.0 ? v : 0.0) : s == 2 ? (v > 0.0 ? v : 0.0) : v;
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
template <int NS, int NT = TPB>
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
            for (int i = 0; i < NT / 32; ++i) t += sw[i][s];
            v[s] = t;
        }
    }
}

// Block partial of `acc` stored at bpart[(prev + blockIdx.x) * NS]; the last block
// to arrive sums bpart[0 .. prev + gridDim.x) in index order (deterministic) and
// runs fin(totals) in its thread 0.  `prev` = partials a preceding kernel left
// (the rows kernel of a plan with long rows), or 0.
template <int NS, int NT = TPB, class Fin>
__device__ __forceinline__ void grid_finalize(double (&acc)[NS], double* bpart, unsigned* ctr, int prev,
                                              double* red, Fin fin)
{
    __shared__ double sw[NT / 32][NS];
    __shared__ int s_last;
    block_sum<NS, NT>(acc, sw);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) bpart[(size_t)(prev + blockIdx.x) * NS + s] = acc[s];
        __threadfence();
        unsigned old = atomicAdd(ctr, 1u);
        s_last = (old == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double tot[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) tot[s] = 0.0;
    const int nb = prev + (int)gridDim.x;
    for (int b = threadIdx.x; b < nb; b += NT)
#pragma unroll
        for (int s = 0; s < NS; ++s) tot[s] += __ldcg(&bpart[(size_t)b * NS + s]);
    block_sum<NS, NT>(tot, sw);
    if (threadIdx.x == 0) {
        if (red) {   // distributed: this rank's totals; summed over ranks, then k_fin
#pragma unroll
            for (int s = 0; s < NS; ++s) red[s] = tot[s];
        } else {
            fin(tot);
        }
        *ctr = 0u;
        __threadfence();
    }
}

// Block partial only (no combine): the finishing kernel combines it.
template <int NS, int NT = TPB>
__device__ __forceinline__ void block_partial(double (&acc)[NS], double* bpart, int prev = 0)
{
    __shared__ double sw[NT / 32][NS];
    block_sum<NS, NT>(acc, sw);
    if (threadIdx.x == 0)
#pragma unroll
        for (int s = 0; s < NS; ++s) bpart[(size_t)(prev + blockIdx.x) * NS + s] = acc[s];
}

// ------------------------------------------------------------ TMA / mbarrier (sm_90+ PTX, used on sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`; the
// streamed bytes are marked evict-first in L2 so they do not push out the gathered
// vector (y, or the current column slab of x).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------------------ SpMV + epilogue
// Shared-memory stage of one plan entry, filled by the TMA engine: row pointers,
// column indices, values and up to NVEC per-row input vectors of the epilogue.
// Every array is copied as its 16-byte-aligned superset; consumers index with the
// element offset of the first wanted element (arrays are padded by >= 16 bytes).
template <int NVEC>
struct alignas(16) Stage {
    double val[CAP + 2];
    double vec[NVEC > 0 ? NVEC : 1][RMAX + 2];
    int32_t col[CAP + 4];
    int32_t rp[RMAX + 8];
};

constexpr int NCW = 16;                   // consumer warps per CTA of k_spmv (one CTA per SM)
constexpr int TPB_SP = (NCW + 1) * 32;    // + one TMA producer warp
constexpr int NGRP = 2;                   // long-row pieces rotate over NGRP groups of consumer warps
constexpr int GW = NCW / NGRP;            // warps per group
constexpr int WCHUNK = CAP / GW;          // nonzeros per warp share of a long-row piece (8 per lane)
#ifndef CPD_SMEM_KB
#define CPD_SMEM_KB 220
#endif
constexpr size_t SMEM_BUDGET = CPD_SMEM_KB * 1024;   // shared memory of the stage ring (rest is L1)

template <int NV, int NVEC>
struct StageSet {
    Stage<NVEC> st;
    double prod2[NV > 1 ? CAP : 2];   // second products (NV = 2)
};
// as many stages as fit one CTA per SM (<= 16)
constexpr size_t SEG_BYTES = (size_t)NCW * 3 * 2 * 32 * sizeof(double);   // per-warp segment scratch (NV <= 2)
template <int NV, int NVEC>
constexpr int nstage_of()
{
    return (int)((SMEM_BUDGET - SEG_BYTES) / sizeof(StageSet<NV, NVEC>)) > 16
               ? 16
               : (int)((SMEM_BUDGET - SEG_BYTES) / sizeof(StageSet<NV, NVEC>));
}

template <int NV, int NVEC>
struct alignas(16) SpmvSmem {
    static constexpr int NS_ = nstage_of<NV, NVEC>();
    StageSet<NV, NVEC> ss[NS_];
    double seg[NCW][3][NV * 32];   // per-warp head / tail / complete row partials
    uint64_t full[NS_];    // TMA -> consumers
    uint64_t empty[NS_];   // consumer warps -> producer
    PlanEntry ent[NS_];
};

__device__ __forceinline__ uint32_t al_dn16(uint64_t b) { return (uint32_t)(b & ~15ull); }

struct VSrc {
    const double* p[NVECMAX];
};

__device__ __forceinline__ uint32_t span_bytes(uint64_t esz, int64_t lo, int64_t hi)
{
    if (hi <= lo) return 0u;
    const uint64_t a0 = ((uint64_t)lo * esz) & ~15ull;
    const uint64_t a1 = ((uint64_t)hi * esz + 15ull) & ~15ull;
    return (uint32_t)(a1 - a0);
}

__device__ __forceinline__ void span_copy(void* dst, const void* base, uint64_t esz, int64_t lo, int64_t hi,
                                          uint64_t* bar)
{
    if (hi <= lo) return;
    const uint64_t a0 = ((uint64_t)lo * esz) & ~15ull;
    const uint64_t a1 = ((uint64_t)hi * esz + 15ull) & ~15ull;
    tma_load_1d(dst, (const char*)base + a0, (uint32_t)(a1 - a0), bar);
}

// Issue the bulk copies of entry E into stage `st` (one thread): expect_tx with
// the byte total first, then the copies.
template <int NVEC>
__device__ __forceinline__ void stage_issue(const PlanEntry& E, Stage<NVEC>& st, uint64_t* bar, const DevCsr& M,
                                            const VSrc& vs)
{
    const bool rows = E.b >= 0;
    uint32_t bytes = span_bytes(4, E.p0, E.p1) + span_bytes(8, E.p0, E.p1);
    if (rows) bytes += span_bytes(4, E.a, (int64_t)E.b + 1);
    if (rows)
#pragma unroll
        for (int v = 0; v < NVEC; ++v)
            if (vs.p[v]) bytes += span_bytes(8, E.a, E.b);
    mbar_arrive_expect_tx(bar, bytes);
    span_copy(st.col, M.j, 4, E.p0, E.p1, bar);
    span_copy(st.val, M.x, 8, E.p0, E.p1, bar);
    if (rows) span_copy(st.rp, M.p, 4, E.a, (int64_t)E.b + 1, bar);
    if (rows)
#pragma unroll
        for (int v = 0; v < NVEC; ++v)
            if (vs.p[v]) span_copy(st.vec[v], vs.p[v], 8, E.a, E.b, bar);
}

// One consumer warp's share of staged entry `s` (plan index ei).
//  rows entry: the warp owns the rows whose first nonzero lies in its 1/NCW share of
//    the entry's nonzeros; it gathers vec[col] for them (lane-strided, coalesced,
//    4 loads in flight per lane), forms the products in place in shared memory,
//    then lane = row: sums the row and applies the fused epilogue (all lanes busy).
//  long-row piece: consecutive pieces rotate over NGRP groups of GW warps (16 loads
//    in flight per lane); each warp of the group sums its WCHUNK nonzeros and lane 0
//    writes the warp partial to lpart[(ei * GW + wg) * 2 + v] for k_finish.
// Returns true if the warp already released the stage (arrived on empty[s]).
template <int NV, class Epi>
__device__ __forceinline__ bool consume_entry(SpmvSmem<NV, Epi::NVEC>& S, int s, int ei, const DevPlan& P,
                                              const Epi& e, const double* __restrict__ v0,
                                              const double* __restrict__ v1, double (&acc)[Epi::NS], int w,
                                              int lane, int& gbase, int& lbase)
{
    constexpr int NVEC = Epi::NVEC;
    constexpr int U = 8;
    const PlanEntry E = S.ent[s];
    Stage<NVEC>& st = S.ss[s].st;
    const int32_t* col = st.col + (E.p0 & 3);
    double* val = st.val + (E.p0 & 1);
    double* val2 = S.ss[s].prod2;
    const int cnt = E.p1 - E.p0;
    if (E.b >= 0) {
        // rows entry: 32-row chunks; chunk j of this entry belongs to warp (gbase + j) % NCW
        const int nr = E.b - E.a;
        const int32_t* rp = st.rp + (E.a & 3);
        const int p0 = E.p0;
        const int nch = (nr + 31) >> 5;
        int j = (w - gbase) % NCW;
        if (j < 0) j += NCW;
        gbase += nch;
        const double* vin[NVEC > 0 ? NVEC : 1];
#pragma unroll
        for (int v = 0; v < NVEC; ++v) vin[v] = st.vec[v] + (E.a & 1);
        for (; j < nch; j += NCW) {
            const int rb = j * 32, re = min(rb + 32, nr);
            const int qa = rp[rb] - p0, qb = rp[re] - p0;
            for (int q0 = qa; q0 < qb; q0 += 32 * U) {
                int c[U];
                double g[U], g2[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = q0 + lane + 32 * u;
                    c[u] = q < qb ? col[q] : -1;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    g[u] = c[u] >= 0 ? __ldg(&v0[c[u]]) : 0.0;
                    if (NV > 1) g2[u] = c[u] >= 0 ? __ldg(&v1[c[u]]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = q0 + lane + 32 * u;
                    if (q < qb) {
                        const double a = val[q];
                        val[q] = a * g[u];
                        if (NV > 1) val2[q] = a * g2[u];
                    }
                }
            }
            __syncwarp();
            // balanced segmented row sums: lane L sums the contiguous span
            // [qa + L k, qa + (L+1) k) of the chunk's products; a row inside one span
            // is complete there (cv), a row crossing spans is its start lane's tail (tv)
            // + the through lanes' tails + its end lane's head (hv) — fixed order.
            double* hv = S.seg[w][0];
            double* tv = S.seg[w][1];
            double* cv = S.seg[w][2];
            const int n = qb - qa, k = (n + 31) >> 5;
            const int s0 = qa + lane * k, s1 = min(s0 + k, qb);
            if (s0 < s1) {
                int lo = rb, hi = re - 1;   // last row with start <= s0
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (rp[mid] - p0 <= s0) lo = mid; else hi = mid - 1;
                }
                int r = lo;
                bool before = rp[r] - p0 < s0;
                double a[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) a[v] = 0.0;
                int q = s0;
                while (true) {
                    const int rend = rp[r + 1] - p0;
                    const int stop = min(rend, s1);
                    for (; q < stop; ++q) {
                        a[0] += val[q];
                        if (NV > 1) a[NV - 1] += val2[q];
                    }
                    if (rend > s1) {   // row continues into the next span
#pragma unroll
                        for (int v = 0; v < NV; ++v) tv[v * 32 + lane] = a[v];
                        break;
                    }
                    double* dst = before ? hv + lane : cv + (r - rb);
#pragma unroll
                    for (int v = 0; v < NV; ++v) dst[v * 32] = a[v];
                    ++r;
                    if (r >= re || q >= s1) break;
                    before = false;
#pragma unroll
                    for (int v = 0; v < NV; ++v) a[v] = 0.0;
                }
            }
            __syncwarp();
            const int i = rb + lane;
            if (i < re) {
                const int a0 = rp[i] - p0, a1 = rp[i + 1] - p0;
                double sm[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) sm[v] = 0.0;
                if (a1 > a0) {
                    const int La = (a0 - qa) / k, Lb = (a1 - 1 - qa) / k;
                    if (La == Lb) {
#pragma unroll
                        for (int v = 0; v < NV; ++v) sm[v] = cv[v * 32 + (i - rb)];
                    } else {
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            double t = tv[v * 32 + La];
                            for (int L = La + 1; L < Lb; ++L) t += tv[v * 32 + L];
                            sm[v] = t + hv[v * 32 + Lb];
                        }
                    }
                }
                e.row(E.a + i, sm, vin, i, acc);
            }
            __syncwarp();
        }
    } else {
        // long-row piece: group (lbase % NGRP) of GW warps, WCHUNK nonzeros per warp.
        // col/val are copied to registers and the stage is released before the gathers.
        const int grp = lbase % NGRP;
        ++lbase;
        if (w / GW != grp) return false;
        const int wg = w % GW;
        const int q0 = wg * WCHUNK;
        int c[WCHUNK / 32];
        double a[WCHUNK / 32];
#pragma unroll
        for (int u = 0; u < WCHUNK / 32; ++u) {
            const int q = q0 + lane + 32 * u;
            c[u] = q < cnt ? col[q] : -1;
            a[u] = q < cnt ? val[q] : 0.0;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
        double sm[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) sm[v] = 0.0;
        double g[WCHUNK / 32], g2[WCHUNK / 32];
#pragma unroll
        for (int u = 0; u < WCHUNK / 32; ++u) {
            g[u] = c[u] >= 0 ? __ldg(&v0[c[u]]) : 0.0;
            if (NV > 1) g2[u] = c[u] >= 0 ? __ldg(&v1[c[u]]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < WCHUNK / 32; ++u) {
            sm[0] += a[u] * g[u];
            if (NV > 1) sm[NV - 1] += a[u] * g2[u];
        }
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sm[v] += __shfl_xor_sync(0xffffffffu, sm[v], o);
        if (lane == 0)
#pragma unroll
            for (int v = 0; v < NV; ++v) P.lpart[((size_t)E.a * GW + wg) * 2 + v] = sm[v];
        return true;
    }
    return false;
}

// Row sums s_v = sum_k M_rk * vec_v[col_k] (v < NV) for every row r of M, each handed
// to the fused epilogue.  One persistent, warp-specialised CTA per SM walks the plan
// round-robin: a producer warp stages each entry with the TMA engine (col, val, row
// pointers and the epilogue's per-row inputs) into a ring of NS_ stages guarded by
// full/empty mbarriers, and NCW consumer warps each process their own share of every
// staged entry with no CTA-wide barrier.  Long-row pieces leave per-warp partials
// that k_finish completes.
template <int NV, class Epi>
__global__ void __launch_bounds__(TPB_SP, 1)
k_spmv(DevCsr M, DevPlan P, VecSel vs0, VecSel vs1, Epi epi, Gate gate, Ctl* ctl, double* bpart,
       unsigned* ctr, double* red)
{
    constexpr int NS = Epi::NS;
    constexpr int NVEC = Epi::NVEC;
    using Smem = SpmvSmem<NV, NVEC>;
    constexpr int NST = Smem::NS_;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto& S = *reinterpret_cast<Smem*>(smem_raw);
    __shared__ int s_go;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        s_go = gate_open(gate, ctl);
        if (s_go && gate.active && blockIdx.x == 0) gate.active[gate.node] = 1;
        if (s_go) {
#pragma unroll
            for (int s = 0; s < NST; ++s) {
                mbar_init(&S.full[s], 1);
                mbar_init(&S.empty[s], NCW);
            }
            fence_mbar_init();
        }
    }
    __syncthreads();
    if (!s_go) return;
    Epi e = epi;
    e.load(ctl);
    double acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    const int G = gridDim.x;
    if (w == NCW) {
        // ---------------- producer warp (one lane)
        if (lane == 0) {
            VSrc vsrc;
#pragma unroll
            for (int v = 0; v < NVECMAX; ++v) vsrc.p[v] = v < NVEC ? e.vec(v) : nullptr;
            uint32_t eph = 0;
            int s = 0, it = 0;
            for (int ei = blockIdx.x; ei < P.nent; ei += G, ++it) {
                const PlanEntry E = P.ent[ei];
                if (it >= NST) {
                    mbar_wait(&S.empty[s], (eph >> s) & 1u);
                    eph ^= 1u << s;
                    fence_proxy_async_smem();
                }
                S.ent[s] = E;
                stage_issue<NVEC>(E, S.ss[s].st, &S.full[s], M, vsrc);
                s = s + 1 == NST ? 0 : s + 1;
            }
        }
        __syncwarp();
    } else {
        // ---------------- consumer warps
        const double* __restrict__ v0 = vs0.get(ctl);
        const double* __restrict__ v1 = vs1.get(ctl);
        uint32_t fph = 0;
        int s = 0, gbase = 0, lbase = 0;
        for (int ei = blockIdx.x; ei < P.nent; ei += G) {
            mbar_wait(&S.full[s], (fph >> s) & 1u);
            fph ^= 1u << s;
            const bool released = consume_entry<NV, Epi>(S, s, ei, P, e, v0, v1, acc, w, lane, gbase, lbase);
            __syncwarp();
            if (lane == 0 && !released) mbar_arrive(&S.empty[s]);
            s = s + 1 == NST ? 0 : s + 1;
        }
    }
    if (P.nlong == 0)
        grid_finalize<NS, TPB_SP>(acc, bpart, ctr, 0, red, [e, ctl](double* tot) { e.finalize(tot, ctl); });
    else
        block_partial<NS, TPB_SP>(acc, bpart);
}

// Long rows: one CTA per long row sums the row's contiguous warp partials (fixed
// order: strided per thread, then the block tree), runs the epilogue on the full
// row sum, then combines this kernel's block partials with those k_spmv left
// (first `prev` slots) and finalizes.
template <int NV, class Epi>
__global__ void __launch_bounds__(TPB_F)
k_finish(DevPlan P, Epi epi, Gate gate, Ctl* ctl, double* bpart, unsigned* ctr, int prev, double* red)
{
    constexpr int NS = Epi::NS;
    constexpr int NVEC = Epi::NVEC;
    __shared__ int s_go;
    __shared__ double s_w[TPB_F / 32][NV];
    if (threadIdx.x == 0) s_go = gate_open(gate, ctl);
    __syncthreads();
    if (!s_go) return;
    Epi e = epi;
    e.load(ctl);
    const double* vin[NVEC > 0 ? NVEC : 1];
#pragma unroll
    for (int v = 0; v < NVEC; ++v) vin[v] = e.vec(v);
    double acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    // rows with many partials (heavy rows: tens of thousands): one CTA each, strided
    // per thread then the block tree; the others one warp each, lane-strided then the
    // xor tree (fixed order either way)
    for (int h = blockIdx.x; h < P.nfin_heavy; h += gridDim.x) {
        const int l = P.long_ents[h];
        double sm[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) sm[v] = 0.0;
        if (NV == 1 && l < P.hotd) {   // fused: the primal step's per-warp partials of this row
            double a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            const double* hp = P.hot_part + (int64_t)l * P.hot_stride;
            int t = threadIdx.x;
            for (; t + 7 * TPB_F < P.hot_stride; t += 8 * TPB_F)
#pragma unroll
                for (int u = 0; u < 8; ++u) a8[u] += __ldcg(hp + t + u * TPB_F);
            for (; t < P.hot_stride; t += TPB_F) a8[0] += __ldcg(hp + t);
#pragma unroll
            for (int q = 0; q < 8; ++q) sm[0] += a8[q];
            block_sum<NV, TPB_F>(sm, s_w);
            if (threadIdx.x == 0) {
                const int r = P.long_row[l];
                e.row(r, sm, vin, r, acc);
            }
            continue;
        }
        const int64_t t0 = (int64_t)P.long_ptr[l] * P.pslot, t1 = (int64_t)P.long_ptr[l + 1] * P.pslot;
        // 8 independent accumulators per thread (loads in flight), combined in fixed order
        double a8[8][NV];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int v = 0; v < NV; ++v) a8[u][v] = 0.0;
        int64_t t = t0 + threadIdx.x;
        for (; t + 7 * TPB_F < t1; t += 8 * TPB_F)
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int v = 0; v < NV; ++v) a8[u][v] += __ldcg(&P.lpart[(t + u * TPB_F) * 2 + v]);
        for (int u = 0; t < t1; t += TPB_F, ++u)
#pragma unroll
            for (int v = 0; v < NV; ++v) a8[u & 7][v] += __ldcg(&P.lpart[t * 2 + v]);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int v = 0; v < NV; ++v) sm[v] += a8[u][v];
        block_sum<NV, TPB_F>(sm, s_w);
        if (threadIdx.x == 0) {
            const int r = P.long_row[l];
            e.row(r, sm, vin, r, acc);
        }
    }
    {
        // the other long rows have few partials (< 131,072 nnz: at most ~70 pieces), so
        // FIN_G lanes sum one row (lane-strided, then the xor tree inside the group: a
        // fixed order) and a warp finishes 32 / FIN_G rows at once
        constexpr int G = FIN_G;
        const int lane = threadIdx.x & 31, sub = lane / G, sl = lane % G;
        const int nw = gridDim.x * (TPB_F / 32);
        for (int h0 = P.nfin_heavy + ((blockIdx.x * TPB_F + threadIdx.x) >> 5) * (32 / G); h0 < P.nlong;
             h0 += nw * (32 / G)) {
            const int h = h0 + sub;
            const bool ok = h < P.nlong;
            const int l = ok ? P.long_ents[h] : 0;
            double sm[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) sm[v] = 0.0;
            if (ok) {
                const int64_t t0 = (int64_t)P.long_ptr[l] * P.pslot, t1 = (int64_t)P.long_ptr[l + 1] * P.pslot;
                for (int64_t t = t0 + sl; t < t1; t += G)
#pragma unroll
                    for (int v = 0; v < NV; ++v) sm[v] += __ldcg(&P.lpart[t * 2 + v]);
            }
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) sm[v] += __shfl_xor_sync(0xffffffffu, sm[v], o);
            if (ok && sl == 0) {
                const int r = P.long_row[l];
                e.row(r, sm, vin, r, acc);
            }
        }
    }
    grid_finalize<NS, TPB_F>(acc, bpart, ctr, prev, red, [e, ctl](double* tot) { e.finalize(tot, ctl); });
}

// ------------------------------------------------------------ SELL-32 SpMV + epilogue
// For layouts whose rows are short and of similar length (A^T of every config):
// warp = slice of 32 consecutive rows, lane = row.  Column indices and values are
// streamed straight from HBM (coalesced: 128 B / 256 B per warp per k, evict-first),
// the gathered vector goes through L1 (no shared memory is used, so L1 keeps its
// full capacity for the reused entries), and the fused epilogue gets the row sum
// in the lane that owns the row.  Sum order = CSR order (k ascending).
// Short-row push: an A^T entry whose row of A is short carries
// PUSH_BIT in its SELL column index; after the primal epilogue of column j the
// warp adds a_ij x+_j to acc[i] (fp64 atomics, L2-resident m-vector), and the dual
// step takes those rows' sums from acc instead of gathering x+ again.
constexpr int32_t PUSH_BIT = 1 << 30;
constexpr int32_t COL_MASK = PUSH_BIT - 1;
template <class E, class = void>
struct PushRole { static constexpr int v = 0; };   // 1: produces acc (primal step), 2: consumes it (dual step)
template <class E>
struct PushRole<E, std::void_t<decltype(E::PUSH)>> { static constexpr int v = E::PUSH; };

struct DevSell {
    const int64_t* __restrict__ sp;
    const int32_t* __restrict__ col;
    const double* __restrict__ val;
    int32_t rows, nslice;
    double* push = nullptr;   // acc (m) when this pass pushes its short-row products
    int32_t hot = 0;          // gathered entries [0, hot) staged in shared memory (hot-row renumbering)
    int32_t r0 = 0;           // the slices hold rows [r0, r0 + rows) of the layout (short-row suffix of A)
    // column-split passes (short-row SELL by column half): the first pass stores its row
    // sums in part[v * rows + rl] and skips the epilogue; the second starts from init
    double* part = nullptr;
    const double* init = nullptr;
    // hot-row fusion (the primal step): each lane holds its padding first,
    // then its entries in DESCENDING row order, so the hot rows 0..hotd-1 are each lane's
    // last entries and sit in the slice's final round; a_hj x+_j is accumulated per lane
    // in shared memory and flushed as per-warp partials hot_part[h * hot_stride + warp]
    int32_t hotd = 0, hot_stride = 0;
    double* hot_part = nullptr;
};
template <class E, class = void>
struct FuseRole { static constexpr int v = 0; };   // 1: primal step (forms the hot sums), 2: dual step
template <class E>
struct FuseRole<E, std::void_t<decltype(E::FUSE)>> { static constexpr int v = E::FUSE; };

constexpr int TPB_SELL = 256;
// SELL entry layout inside a slice: SELL_PAIR = 1 stores entries k, k+1 of a lane next to
// each other ([k / 2][lane][k % 2], slice width even), so a lane streams them with one
// 8-byte (index) and one 16-byte (value) load: coalesced AND vectorised; 0 = [k][lane].
#ifndef CPD_SELL_PAIR
#define CPD_SELL_PAIR 1
#endif
constexpr int SELL_PAIR = CPD_SELL_PAIR;
__host__ __device__ __forceinline__ int64_t sell_pos(int64_t k, int64_t lane)
{
    return SELL_PAIR ? (k >> 1) * 64 + lane * 2 + (k & 1) : k * 32 + lane;
}
#ifndef CPD_PRE
#define CPD_PRE 0   // 1: epilogue inputs held in registers across the sum (more registers)
#endif
#ifndef CPD_SELL_U
#define CPD_SELL_U 6
#endif
constexpr int SELL_U = CPD_SELL_U;   // entries per lane in flight

#ifndef CPD_SELL_MINB
#define CPD_SELL_MINB 4
#endif
template <int NV, class Epi, int FZ = 0>   // FZ: the fused primal step (hot-row fusion)
__global__ void __launch_bounds__(TPB_SELL, CPD_SELL_MINB)
k_sell(DevSell M, VecSel vs0, VecSel vs1, Epi epi, Gate gate, Ctl* ctl, double* bpart, unsigned* ctr,
       double* red, int prev, int fin)
{
    constexpr int NS = Epi::NS;
    constexpr int NVEC = Epi::NVEC;
    __shared__ int s_go;
    if (threadIdx.x == 0) {
        s_go = gate_open(gate, ctl);
        if (s_go && gate.active && blockIdx.x == 0) gate.active[gate.node] = 1;
    }
    __syncthreads();
    if (!s_go) return;
    Epi e = epi;
    e.load(ctl);
    const double* vin[NVEC > 0 ? NVEC : 1];
#pragma unroll
    for (int v = 0; v < NVEC; ++v) vin[v] = e.vec(v);
    const double* __restrict__ v0 = vs0.get(ctl);
    const double* __restrict__ v1 = vs1.get(ctl);
    double acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (TPB_SELL / 32);
    __shared__ double vst[TPB_SELL / 32][(NVEC > 0 ? NVEC : 1) * 32];
    // the gathered vector's hot prefix (the longest rows of A, most of the gathers)
    extern __shared__ __align__(16) double yhot[];   // [NV][hot], then the fused rows' accumulators
    const int hot = M.hot;
    for (int t = threadIdx.x; t < hot; t += TPB_SELL) {
        yhot[t] = v0[t];
        if (NV > 1) yhot[hot + t] = v1[t];
    }
    // hot-row fusion: this warp's lane-private accumulators hacc[h][lane] (conflict-free,
    // fixed summation order: the warp's slices in order, then a fixed lane tree)
    constexpr bool FUSE = FZ && FuseRole<Epi>::v == 1 && NV == 1;
    const int hotd = FUSE ? M.hotd : 0;
    // (measured slower on C5, profiles/r02_kernel_iterations.md: the hottest rows'
    // accumulators in registers — spills at the 64-register cap; the last round's hot
    // entries parked in shared memory before the epilogue — less L1 for the gathers)
    double* hacc = yhot + NV * hot + (threadIdx.x >> 5) * (hotd * 32);
    for (int h = 0; h < hotd; ++h) hacc[h * 32 + lane] = 0.0;
    __syncthreads();
    // push only for an iteration the dual step will complete (k < k_stop)
    const bool push_on = M.push != nullptr && ctl->k < ctl->k_stop;
    for (int s = (blockIdx.x * TPB_SELL + threadIdx.x) >> 5; s < M.nslice; s += nw) {
        const int64_t b = M.sp[s];
        const int len = (int)((M.sp[s + 1] - b) >> 5);
        if (CPD_PF > 0 && lane == 0 && s + CPD_PF * nw < M.nslice) {
            const int64_t pb = M.sp[s + CPD_PF * nw], pe = M.sp[s + CPD_PF * nw + 1];
            l2_prefetch(M.col + pb, (pe - pb) * 4);
            l2_prefetch(M.val + pb, (pe - pb) * 8);
        }
        const int rl = s * 32 + lane;   // row of the slice layout; r = row of the matrix
        const int r = M.r0 + rl;
        // the epilogue's per-row inputs do not depend on the sum: load them now
        // (streamed, evict-first) into this warp's stage
        double* stg = vst[threadIdx.x >> 5];
#if CPD_PRE
        double pre[NVEC > 0 ? NVEC : 1];   // in registers until the sum is done (no wait here)
#pragma unroll
        for (int v = 0; v < NVEC; ++v) pre[v] = (rl < M.rows && vin[v]) ? __ldcs(vin[v] + r) : 0.0;
#else
        if (rl < M.rows && !M.part)
#pragma unroll
            for (int v = 0; v < NVEC; ++v) stg[v * 32 + lane] = vin[v] ? __ldcs(vin[v] + r) : 0.0;
#endif
        const int32_t* cb = M.col + b;
        const double* vb = M.val + b;
        double sm[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) sm[v] = (M.init && rl < M.rows) ? __ldcs(M.init + (int64_t)v * M.rows + rl) : 0.0;
        // two-stage software pipeline over rounds of SELL_U entries per lane
        auto ldround = [&](int (&cc)[SELL_U], double (&aa)[SELL_U], int k0) {
            if constexpr (SELL_PAIR) {
                static_assert(SELL_U % 2 == 0, "pair layout: even rounds");
#pragma unroll
                for (int u = 0; u < SELL_U; u += 2) {
                    const bool ok = k0 + u < len;   // len even: both of the pair
                    const int64_t q = sell_pos(k0 + u, lane);
                    const int2 c2 = ok ? ld_stream(reinterpret_cast<const int2*>(cb + q)) : make_int2(-1, -1);
                    const double2 a2 = ok ? ld_stream(reinterpret_cast<const double2*>(vb + q)) : make_double2(0.0, 0.0);
                    cc[u] = c2.x;
                    cc[u + 1] = c2.y;
                    aa[u] = a2.x;
                    aa[u + 1] = a2.y;
                }
            } else {
#pragma unroll
                for (int u = 0; u < SELL_U; ++u) {
                    const bool ok = k0 + u < len;
                    cc[u] = ok ? ld_stream(cb + sell_pos(k0 + u, lane)) : -1;
                    aa[u] = ok ? ld_stream(vb + sell_pos(k0 + u, lane)) : 0.0;
                }
            }
        };
        int c[SELL_U];
        double a[SELL_U];
        ldround(c, a, 0);
        auto round_sum = [&]() {   // this round's gathers and products
            double g[SELL_U], g2[SELL_U];
#pragma unroll
            for (int u = 0; u < SELL_U; ++u) {
                const int cc = c[u] & COL_MASK;
                g[u] = c[u] < 0 ? 0.0 : cc < hot ? yhot[cc] : __ldg(&v0[cc]);
                if (NV > 1) g2[u] = c[u] < 0 ? 0.0 : cc < hot ? yhot[hot + cc] : __ldg(&v1[cc]);
            }
            return [=, &sm](void) {
#pragma unroll
                for (int u = 0; u < SELL_U; ++u)
                    if (c[u] >= 0) {
                        sm[0] += a[u] * g[u];
                        if (NV > 1) sm[NV - 1] += a[u] * g2[u];
                    }
            };
        };
        // all but the last round: the next round's loads in flight during this round's
        // gathers; the last round's entries stay in c / a (the fused primal step uses them)
        int k0 = 0;
        for (; k0 + SELL_U < len; k0 += SELL_U) {
            auto fma = round_sum();
            int cn[SELL_U];
            double an[SELL_U];
            ldround(cn, an, k0 + SELL_U);
            fma();
#pragma unroll
            for (int u = 0; u < SELL_U; ++u) {
                c[u] = cn[u];
                a[u] = an[u];
            }
        }
        if (len > 0) round_sum()();
        if (M.part) {   // first column pass: running sums only
            if (rl < M.rows)
#pragma unroll
                for (int v = 0; v < NV; ++v) __stcs(M.part + (int64_t)v * M.rows + rl, sm[v]);
            continue;
        }
        if (rl < M.rows) {
            const double* vs[NVEC > 0 ? NVEC : 1];
#pragma unroll
            for (int v = 0; v < NVEC; ++v) {
#if CPD_PRE
                stg[v * 32 + lane] = pre[v];
#endif
                vs[v] = stg + v * 32;
            }
            if constexpr (FUSE) {
                const double xp = e.row(r, sm, vs, lane, acc);
                if (hotd > 0) {
                    // the last round holds the lane's last (= lowest-row) entries (padding
                    // comes first in a reversed slice)
                    bool more = len > SELL_U;
#pragma unroll
                    for (int u = 0; u < SELL_U; ++u) {
                        const int32_t cc = c[u] & COL_MASK;
                        const bool hit = c[u] >= 0 && cc < hotd;
                        if (hit) hacc[cc * 32 + lane] += a[u] * xp;
                        // an earlier hot entry only if the round starts with one
                        if (u == 0) more = more && hit;
                    }
                    if (__any_sync(__activemask(), more)) {   // rare: scan back from the last round
                        for (int k = len - SELL_U - 1; k >= 0; --k) {
                            const int32_t c0 = more ? __ldg(cb + sell_pos(k, lane)) : 0;
                            const int32_t cc = c0 & COL_MASK;
                            if (more) {
                                if (c0 >= 0 && cc < hotd) hacc[cc * 32 + lane] += __ldg(vb + sell_pos(k, lane)) * xp;
                                else more = false;   // padding or a colder row: no hot entry before it
                            }
                            if (!__any_sync(__activemask(), more)) break;
                        }
                    }
                }
            } else {
                e.row(r, sm, vs, lane, acc);
            }
            if constexpr (PushRole<Epi>::v == 1) {
                if (push_on) {   // a_ij x+_j into acc[i] for the short rows i of column j
                    const double xp = e.pushval(r);
                    for (int k = 0; k < len; ++k) {
                        const int32_t cc = cb[sell_pos(k, lane)];
                        if (cc >= 0 && (cc & PUSH_BIT)) atomicAdd(&M.push[cc & COL_MASK], vb[sell_pos(k, lane)] * xp);
                    }
                }
            }
        }
    }
    if constexpr (FUSE) {   // per-warp partials of the hot rows (fixed-order lane tree)
        const int gw = blockIdx.x * (TPB_SELL / 32) + (threadIdx.x >> 5);
        for (int h = 0; h < hotd; ++h) {
            double v = hacc[h * 32 + lane];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) M.hot_part[(int64_t)h * M.hot_stride + gw] = v;
        }
    }
    if (M.part) return;   // first column pass: no epilogue, no partials
    if (fin)
        grid_finalize<NS, TPB_SELL>(acc, bpart, ctr, 0, red, [e, ctl](double* tot) { e.finalize(tot, ctl); });
    else
        block_partial<NS, TPB_SELL>(acc, bpart, prev);   // k_finish combines (short-row SELL of A)
}

// ------------------------------------------------------------ warp-item CSR SpMV + epilogue
// For general CSR layouts (A): one warp per plan item, no shared memory.
//  rows item (<= 32 rows, <= WCAP_ROWS nonzeros): the item's nonzeros are streamed
//    coalesced (lane-strided, WU per lane in flight), each lane finds the row of its
//    element by a 5-step shuffle search over the row starts, a segmented warp scan
//    sums each row's run inside the 32-element round, and the lane that owns the
//    row (lane = row) adds the run's total; then lane = row runs the epilogue.
//  long-row piece (<= WCAP_LONG nonzeros inside one column slab): lane-strided sum,
//    warp xor-reduction, one partial per piece for k_finish.
// Slab mode (slab >= 0, the default for the warp plan's rows items when the vector
//   spans >= 2 slabs): the rows items sum only their entries in column slab `slab`
//   (slab-major copy P.short_*, items re-based per slab at create), so the pass
//   gathers from an L2-resident part of the
//   vector; running sums live in P.short_part, the last pass (spass bit 1) runs the
//   epilogue, the first (bit 0) starts the sums.
// Fixed order for a fixed plan: deterministic.
constexpr int TPB_W = 256;
constexpr int WU = 4;

#ifndef CPD_W_MINB
#define CPD_W_MINB 4
#endif
template <int NV, class Epi>
__global__ void __launch_bounds__(TPB_W, CPD_W_MINB)
k_csrw(DevCsr M, DevPlan P, VecSel vs0, VecSel vs1, Epi epi, Gate gate, Ctl* ctl, double* bpart, unsigned* ctr,
       double* red, int prev, int fin, int slab, int spass)
{
    constexpr int NS = Epi::NS;
    constexpr int NVEC = Epi::NVEC;
    __shared__ int s_go;
    if (threadIdx.x == 0) {
        s_go = gate_open(gate, ctl);
        if (s_go && gate.active && blockIdx.x == 0) gate.active[gate.node] = 1;
    }
    __syncthreads();
    if (!s_go) return;
    Epi e = epi;
    e.load(ctl);
    const double* vin[NVEC > 0 ? NVEC : 1];
#pragma unroll
    for (int v = 0; v < NVEC; ++v) vin[v] = e.vec(v);
    const double* __restrict__ v0 = vs0.get(ctl);
    const double* __restrict__ v1 = vs1.get(ctl);
    double acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (TPB_W / 32);
    // slab >= 0: rows items over the short-row copy of column slab `slab` (running
    // sums in P.short_part between passes; the last pass runs the epilogue)
    const bool sl_mode = slab >= 0;
    const bool sl_last = !sl_mode || (spass & 2);   // spass: bit 0 first pass, bit 1 last pass
    const int32_t* __restrict__ rptr = sl_mode ? P.short_ptr + (int64_t)slab * (M.rows + 1) : M.p;
    __shared__ double vst[TPB_W / 32][(NVEC > 0 ? NVEC : 1) * 32];
    for (int it = (blockIdx.x * TPB_W + threadIdx.x) >> 5; it < P.nent; it += nw) {
        const PlanEntry E = P.ent[it];
        const bool sl_item = sl_mode && E.b >= 0;
        if (CPD_PF > 0 && lane == 0 && it + CPD_PF * nw < P.nent) {
            const PlanEntry F = P.ent[it + CPD_PF * nw];
            const bool fs = sl_mode && F.b >= 0;
            l2_prefetch((fs ? P.short_col : M.j) + F.p0, (int64_t)(F.p1 - F.p0) * 4);
            l2_prefetch((fs ? P.short_val : M.x) + F.p0, (int64_t)(F.p1 - F.p0) * 8);
        }
        const int32_t* __restrict__ mj = sl_item ? P.short_col : M.j;
        const double* __restrict__ mx = sl_item ? P.short_val : M.x;
        const int p0 = E.p0, T = E.p1 - E.p0;   // (slab mode: P.ent = the slab's own items)
        // one round: WU lane-strided entries from `base` (streamed, evict-first)
        auto ldround = [&](int (&cc)[WU], double (&aa)[WU], int base) {
#pragma unroll
            for (int u = 0; u < WU; ++u) {
                const int q = base + 32 * u + lane;
                cc[u] = q < T ? ld_stream(mj + p0 + q) : -1;
                aa[u] = q < T ? ld_stream(mx + p0 + q) : 0.0;
            }
        };
        if (E.b >= 0) {
            const int r0 = E.a, nr = E.b - E.a;
            const int rs = lane < nr ? rptr[r0 + lane] - p0 : 0x7fffffff;   // start of row `lane`
            const int re = lane < nr ? rptr[r0 + lane + 1] - p0 : 0;         // its end
            double* stg = vst[threadIdx.x >> 5];
#if CPD_PRE
            double pre[NVEC > 0 ? NVEC : 1];
#pragma unroll
            for (int v = 0; v < NVEC; ++v) pre[v] = (sl_last && lane < nr && vin[v]) ? __ldcs(vin[v] + r0 + lane) : 0.0;
#else
            if (sl_last && lane < nr)
#pragma unroll
                for (int v = 0; v < NVEC; ++v) stg[v * 32 + lane] = vin[v] ? __ldcs(vin[v] + r0 + lane) : 0.0;
#endif
            double racc[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) racc[v] = (sl_mode && !(spass & 1) && lane < nr) ? P.short_part[v * (int64_t)M.rows + r0 + lane] : 0.0;
            if (PushRole<Epi>::v == 2 && P.push_acc) {   // sums pushed by the primal step
                if (lane < nr) {
                    racc[0] = P.push_acc[r0 + lane];
                    P.push_acc[r0 + lane] = 0.0;
                }
            } else {
            // two-stage software pipeline: the next round's indices / values are in
            // flight while this round's gathers are
            int c[WU];
            double a[WU];
            ldround(c, a, 0);
            for (int base = 0; base < T; base += 32 * WU) {
                double g[WU][NV];
#pragma unroll
                for (int u = 0; u < WU; ++u) {
                    g[u][0] = c[u] >= 0 ? ld_keep(&v0[c[u]]) : 0.0;
                    if (NV > 1) g[u][NV - 1] = c[u] >= 0 ? __ldg(&v1[c[u]]) : 0.0;
                }
                int cn[WU];
                double an[WU];
                ldround(cn, an, base + 32 * WU);
#pragma unroll
                for (int u = 0; u < WU; ++u) {
                    const int rb = base + 32 * u;
                    if (rb >= T) break;   // warp-uniform
                    const int q = rb + lane;
                    // row of element q: largest i < nr with rs_i <= q (invalid q: own key)
                    int lo = 0;
#pragma unroll
                    for (int st = 16; st > 0; st >>= 1) {
                        const int cand = lo + st;
                        const int rv = __shfl_sync(FULL, rs, cand & 31);
                        if (cand < nr && rv <= q) lo = cand;
                    }
                    const int key = q < T ? lo : 64 + lane;
                    double sv[NV];
#pragma unroll
                    for (int v = 0; v < NV; ++v) sv[v] = a[u] * g[u][v];
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const int kt = __shfl_up_sync(FULL, key, d);
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            const double t = __shfl_up_sync(FULL, sv[v], d);
                            if (lane >= d && kt == key) sv[v] += t;
                        }
                    }
                    // owner lane = row: its run in this round ends at min(re, rb + 32) - 1
                    const bool hit = lane < nr && rs < rb + 32 && re > rb && re > rs;
                    const int pos = hit ? min(re, rb + 32) - 1 - rb : 0;
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double t = __shfl_sync(FULL, sv[v], pos);
                        if (hit) racc[v] += t;
                    }
                }
#pragma unroll
                for (int u = 0; u < WU; ++u) {
                    c[u] = cn[u];
                    a[u] = an[u];
                }
            }
            }
            if (!sl_last) {
                if (lane < nr)
#pragma unroll
                    for (int v = 0; v < NV; ++v) P.short_part[v * (int64_t)M.rows + r0 + lane] = racc[v];
                continue;
            }
            if (lane < nr) {
                const double* vs[NVEC > 0 ? NVEC : 1];
#pragma unroll
                for (int v = 0; v < NVEC; ++v) {
#if CPD_PRE
                    stg[v * 32 + lane] = pre[v];
#endif
                    vs[v] = stg + v * 32;
                }
                e.row(r0 + lane, racc, vs, lane, acc);
            }
        } else {
            double sm[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) sm[v] = 0.0;
            int c[WU];
            double a[WU];
            ldround(c, a, 0);
            for (int base = 0; base < T; base += 32 * WU) {
                double g[WU][NV];
#pragma unroll
                for (int u = 0; u < WU; ++u) {
                    g[u][0] = c[u] >= 0 ? ld_keep(&v0[c[u]]) : 0.0;
                    if (NV > 1) g[u][NV - 1] = c[u] >= 0 ? __ldg(&v1[c[u]]) : 0.0;
                }
                int cn[WU];
                double an[WU];
                ldround(cn, an, base + 32 * WU);
#pragma unroll
                for (int u = 0; u < WU; ++u) {
                    if (c[u] >= 0) {
                        sm[0] += a[u] * g[u][0];
                        if (NV > 1) sm[NV - 1] += a[u] * g[u][NV - 1];
                    }
                    c[u] = cn[u];
                    a[u] = an[u];
                }
            }
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sm[v] += __shfl_xor_sync(FULL, sm[v], o);
            if (lane == 0)
#pragma unroll
                for (int v = 0; v < NV; ++v) P.lpart[(size_t)E.a * 2 + v] = sm[v];
        }
    }
    if (!sl_last) return;
    if (fin)
        grid_finalize<NS, TPB_W>(acc, bpart, ctr, 0, red, [e, ctl](double* tot) { e.finalize(tot, ctl); });
    else
        block_partial<NS, TPB_W>(acc, bpart, prev);
}

// ------------------------------------------------------------ heavy rows by dense column blocks
// The few rows holding most nonzeros (C5: Zipf head) touch a large fraction of the
// columns, so gathering their vector entries one 32-byte sector at a time costs
// 4x the bytes in L2.  Instead each CTA takes a block of HB columns, loads that
// block of the vector once (coalesced) into shared memory, and every warp sums the
// block's entries of its heavy rows from shared memory; one partial per (row,
// block) goes to the row's slot for k_finish (fixed order: deterministic).
template <int NV, bool C16 = false>   // C16: 16-bit in-block column offsets (P.dense_col16)
__global__ void __launch_bounds__(TPB_D)
k_dense(DevCsr M, DevPlan P, int32_t cols, VecSel vs0, VecSel vs1, Gate gate, Ctl* ctl)
{
    extern __shared__ __align__(16) double xs[];   // [NV][HB] vector block
    __shared__ int s_go;
    if (threadIdx.x == 0) s_go = gate_open(gate, ctl);
    __syncthreads();
    if (!s_go) return;
    const double* __restrict__ v0 = vs0.get(ctl);
    const double* __restrict__ v1 = vs1.get(ctl);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int NWD = TPB_D / 32;
#ifndef CPD_DU
#define CPD_DU 8
#endif
    constexpr int DU = CPD_DU;
    // balanced at item granularity: CTA c takes items [c I / G, (c + 1) I / G) (sorted by
    // column block) and loads each block of the vector its range touches
    const int64_t I = P.dense_ptr[P.nhb];
    const int ia = (int)(I * blockIdx.x / gridDim.x), ib = (int)(I * (blockIdx.x + 1) / gridDim.x);
    int blk = 0;
    {
        int lo = 0, hi = P.nhb;   // last block with dense_ptr[blk] <= ia
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (P.dense_ptr[mid] <= ia) lo = mid; else hi = mid;
        }
        blk = lo;
    }
    for (; blk < P.nhb && P.dense_ptr[blk] < ib; ++blk) {
        const int j0 = blk * HB, nj = min(HB, cols - j0);
        const int i0 = max(P.dense_ptr[blk], ia), i1 = min(P.dense_ptr[blk + 1], ib);
        if (i1 <= i0) continue;
        __syncthreads();
        for (int t = threadIdx.x; t < nj; t += TPB_D) {
            xs[t] = v0[j0 + t];
            if (NV > 1) xs[HB + t] = v1[j0 + t];
        }
        __syncthreads();
        for (int i = i0 + w; i < i1; i += NWD) {
            const PlanEntry E = P.dense_ent[i];
            if (CPD_PF > 0 && lane == 0 && i + CPD_PF * NWD < ib) {
                const PlanEntry F = P.dense_ent[i + CPD_PF * NWD];
                l2_prefetch(M.j + F.p0, (int64_t)(F.p1 - F.p0) * 4);
                l2_prefetch(M.x + F.p0, (int64_t)(F.p1 - F.p0) * 8);
            }
            double sm[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) sm[v] = 0.0;
            // <= DCHUNK entries: all of this lane's loads issued at once
            for (int q = E.p0 + lane; q < E.p1; q += 32 * DU) {
                int c[DU];
                double a[DU];
#pragma unroll
                for (int u = 0; u < DU; ++u) {
                    const int qq = q + 32 * u;
                    if constexpr (C16) c[u] = qq < E.p1 ? ld_stream(P.dense_col16 + qq) : -1;
                    else c[u] = qq < E.p1 ? ld_stream(M.j + qq) - j0 : -1;
                    a[u] = qq < E.p1 ? ld_stream(M.x + qq) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < DU; ++u)
                    if (c[u] >= 0) {
                        sm[0] += a[u] * xs[c[u]];
                        if (NV > 1) sm[NV - 1] += a[u] * xs[HB + c[u]];
                    }
            }
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sm[v] += __shfl_xor_sync(FULL, sm[v], o);
            if (lane == 0)
#pragma unroll
                for (int v = 0; v < NV; ++v) P.lpart[(size_t)E.a * 2 + v] = sm[v];
        }
    }
}

// Elementwise pass over [0, N) with reductions and a device-side finalize.
template <class Op>
__global__ void __launch_bounds__(TPB)
k_elem(int64_t N, Op op, Gate gate, Ctl* ctl, double* bpart, unsigned* ctr, double* red)
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
    grid_finalize<NS>(acc, bpart, ctr, 0, red, [o, ctl](double* tot) { o.finalize(tot, ctl); });
}

// ------------------------------------------------------------ distributed helpers
// Owned-slice epilogue of a split product: the row sums of rows [0, N) of this
// rank's slice arrive reduce-scattered in recv[v * L + i] (v < NV); each is handed
// to the same fused epilogue the single-GPU kernel applies.
template <int NV, class Epi>
__global__ void __launch_bounds__(TPB)
k_slice(int64_t N, int64_t L, const double* __restrict__ recv, Epi epi, Gate gate, Ctl* ctl, double* bpart,
        unsigned* ctr, double* red)
{
    constexpr int NS = Epi::NS;
    constexpr int NVEC = Epi::NVEC;
    __shared__ int s_go;
    if (threadIdx.x == 0) s_go = gate_open(gate, ctl);
    __syncthreads();
    if (!s_go) return;
    Epi e = epi;
    e.load(ctl);
    const double* vin[NVEC > 0 ? NVEC : 1];
#pragma unroll
    for (int v = 0; v < NVEC; ++v) vin[v] = e.vec(v);
    double acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < N; i += (int64_t)gridDim.x * TPB) {
        double sm[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) sm[v] = recv[v * L + i];
        e.row((int)i, sm, vin, (int)i, acc);
    }
    grid_finalize<NS>(acc, bpart, ctr, 0, red, [e, ctl](double* tot) { e.finalize(tot, ctl); });
}

// Device finalize of an epilogue on totals summed over ranks (red, after the
// scalar allreduce); same gate as the kernel whose totals these are.
template <class Epi>
__global__ void k_fin(Epi epi, Gate gate, Ctl* ctl, const double* red)
{
    if (!gate_open(gate, ctl)) return;
    double tot[Epi::NS];
#pragma unroll
    for (int s = 0; s < Epi::NS; ++s) tot[s] = red[s];
    epi.finalize(tot, ctl);
}

// Split product: row r's NV sums go to the reduce-scatter send buffer, laid out
// [owner q = r / L][v][r - q L] so that rank q receives [v][L].
template <int NV_>
struct EpiStore {
    static constexpr int NS = 1;
    static constexpr int NVEC = 0;
    double* part;
    int64_t L;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    __device__ __forceinline__ void row(int r, const double* s, const double* const*, int, double*) const
    {
        const int64_t q = r / L;
        double* d = part + q * NV_ * L + (r - q * L);
#pragma unroll
        for (int v = 0; v < NV_; ++v) d[v * L] = s[v];
    }
    __device__ void finalize(const double*, Ctl*) const {}
};

// Fused split product (CPD_P2P=1): row r's NV sums are stored straight into the
// owner rank's receive window over NVLink peer memory (NCCL symmetric window),
// slot [this rank][v][r - q L], while the SpMV streams; after a barrier the owner
// sums the world slots of each owned row in rank order (k_slice_p2p).
template <int NV_>
struct EpiStorePeer {
    static constexpr int NS = 1;
    static constexpr int NVEC = 0;
    double* const* peer;   // [world] base of every rank's receive window (device pointers)
    int64_t L;
    int32_t rank;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    __device__ __forceinline__ void row(int r, const double* s, const double* const*, int, double*) const
    {
        const int64_t q = r / L;
        double* d = peer[q] + ((int64_t)rank * NV_) * L + (r - q * L);
#pragma unroll
        for (int v = 0; v < NV_; ++v) d[v * L] = s[v];
    }
    __device__ void finalize(const double*, Ctl*) const {}
};

// Owned-slice epilogue of a fused split product: sum of the world ranks' slots.
template <int NV, class Epi>
__global__ void __launch_bounds__(TPB)
k_slice_p2p(int64_t N, int64_t L, int32_t world, const double* __restrict__ win, Epi epi, Gate gate, Ctl* ctl,
            double* bpart, unsigned* ctr, double* red)
{
    constexpr int NS = Epi::NS;
    constexpr int NVEC = Epi::NVEC;
    __shared__ int s_go;
    if (threadIdx.x == 0) s_go = gate_open(gate, ctl);
    __syncthreads();
    if (!s_go) return;
    Epi e = epi;
    e.load(ctl);
    const double* vin[NVEC > 0 ? NVEC : 1];
#pragma unroll
    for (int v = 0; v < NVEC; ++v) vin[v] = e.vec(v);
    double acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < N; i += (int64_t)gridDim.x * TPB) {
        double sm[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) sm[v] = 0.0;
        for (int p = 0; p < world; ++p)
#pragma unroll
            for (int v = 0; v < NV; ++v) sm[v] += win[((int64_t)p * NV + v) * L + i];
        e.row((int)i, sm, vin, (int)i, acc);
    }
    grid_finalize<NS>(acc, bpart, ctr, 0, red, [e, ctl](double* tot) { e.finalize(tot, ctl); });
}

// Replica refresh: dst[i] = src(k)[i] for i < N (the owned slice, copied into its
// place in the all-gather buffer).
static __global__ void __launch_bounds__(TPB) k_copy_sel(int64_t N, double* dst, VecSel src, Gate gate, Ctl* ctl)
{
    __shared__ int s_go;
    if (threadIdx.x == 0) s_go = gate_open(gate, ctl);
    __syncthreads();
    if (!s_go) return;
    const double* s = src.get(ctl);
    for (int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x; i < N; i += (int64_t)gridDim.x * TPB) dst[i] = s[i];
}

// ------------------------------------------------------------ epilogues
// Selects the ping-pong buffer of iterate k.
struct PingPong {
    double* b[2];
    // a select, not b[k & 1]: a dynamic index would put the epilogue struct in local memory
    __device__ __forceinline__ double* at(int64_t k) const { return (k & 1) ? b[1] : b[0]; }
};

// a2 + a5 + n-side of a6, and the per-iteration termination decision F(k).
// Staged per-row inputs: 0 c, 1 x_k, 2 x_avg, 3 lb, 4 ub (3-4 only with per-element
// bounds, PE = true: the corner model, or an LP with non-uniform bounds).
template <bool PE>
struct EpiPrimalT {
    static constexpr int NS = 5;   // c^T x_k, ||r_D(y_k)||^2, bound terms, #nonfinite(x_{k+1}), #{|r_D_j| > eps}
    static constexpr int NVEC = PE ? 5 : 3;
    static constexpr int PUSH = 1;
    static constexpr int FUSE = 1;
    __device__ __forceinline__ double pushval(int j) const { return xn[j]; }
    const double* c;
    Bounds bd;
    PingPong X, Xa;
    // loaded
    double tau, inv_t, eps_dual;
    const double* xc;
    double* xn;
    const double* xac;
    double* xan;
    const double* w = nullptr;   // 1/s (scaled problem): ||r_D|| in the original space
    __device__ void load(const Ctl* ctl)
    {
        tau = ctl->tau;
        eps_dual = ctl->eps_abs;
        inv_t = 1.0 / (double)(ctl->t + 1);
        xc = X.at(ctl->k);
        xn = X.at(ctl->k + 1);
        xac = Xa.at(ctl->k);
        xan = Xa.at(ctl->k + 1);
    }
    __device__ __forceinline__ const double* vec(int v) const
    {
        return v == 0 ? c : v == 1 ? xc : v == 2 ? xac : v == 3 ? bd.l : bd.u;
    }
    // row j of A^T; vin[v][li] = staged (or global, li = j) input v of row j
    __device__ __forceinline__ double row(int j, const double* s, const double* const* vin, int li,
                                          double* acc) const
    {
        const double cj = vin[0][li];
        const double z = cj - s[0];
        const double x = vin[1][li];
        double lo = bd.l0, hi = bd.u0;
        if constexpr (PE) {
            lo = vin[3][li];
            hi = vin[4][li];
        }
        const double xp = proj(x - tau * z, lo, hi);
        st_keep(&xn[j], xp);
        const double xa = vin[2][li];
        // averages are read once per iteration: streamed (evict-first) so L2 keeps x+
        __stcs(&xan[j], xa + (xp - xa) * inv_t);   // (x+ - x_avg)/t as a multiply (<= 1 ulp)
        acc[0] += cj * x;
        const double rd = dual_terms(z, lo, hi, acc[1], acc[2], w ? w[j] : 1.0);
        acc[3] += isfinite(xp) ? 0.0 : 1.0;
        acc[4] += fabs(rd) > eps_dual ? 1.0 : 0.0;
        return xp;
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
        else if (ctl->mode == MODE_DUAL_ONLY) conv = k >= ctl->min_iters && tot[4] == 0.0;   // reading D-3
        else conv = k >= ctl->min_iters && o[0] <= ctl->target;
        if (conv) {
            ctl->done = 1; ctl->status = ST_CONVERGED; ctl->iterations = k;
        } else if (k == ctl->max_iters) {
            ctl->done = 1; ctl->status = ST_ITER_LIMIT; ctl->iterations = k;
        }
    }
};

using EpiPrimal = EpiPrimalT<true>;

// a3 + a4 + a5 + m-side of a6: y+ = y + sigma (b - (2 A x+ - A x)).
// Staged per-row inputs: 0 b, 1 y_k, 2 (A x_k), 3 y_avg.
struct EpiDual {
    static constexpr int NS = 3;   // ||b - A x_{k+1}||^2, b^T y_{k+1}, #nonfinite(y_{k+1})
    static constexpr int NVEC = 4;
    static constexpr int PUSH = 2;
    static constexpr int FUSE = 2;
    const double* b;
    double *y, *ya, *ax;
    double sigma, inv_t;
    const double* w = nullptr;   // 1/r (scaled problem): ||r_P|| in the original space
    const int8_t* sn = nullptr;  // row senses (null: all equality rows)
    __device__ void load(const Ctl* ctl)
    {
        sigma = ctl->sigma;
        inv_t = 1.0 / (double)(ctl->t + 1);
    }
    __device__ __forceinline__ const double* vec(int v) const
    {
        return v == 0 ? b : v == 1 ? y : v == 2 ? ax : ya;
    }
    __device__ __forceinline__ void row(int i, const double* s, const double* const* vin, int li,
                                        double* acc) const
    {
        const double axn = s[0];
        const double bi = vin[0][li];
        const double yo = vin[1][li];
        const double yp = dual_proj(sn, i, yo + sigma * (bi - (2.0 * axn - vin[2][li])));
        y[i] = yp;
        ax[i] = axn;
        const double yav = vin[3][li];
        __stcs(&ya[i], yav + (yp - yav) * inv_t);
        const double r = row_viol(sn, i, bi - axn) * (w ? w[i] : 1.0);
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
    static constexpr int NS = 11;  // ctx_c, rd2_c, bnd_c, dx2_c, ctx_a, rd2_a, bnd_a, dx2_a, off_bound(x_k; M),
                                   // #{|r_D_j(y_k)| > eps}, off_bound(x_avg; M)
    static constexpr int NVEC = 0;
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    const double* c;
    Bounds bd;       // bounds of the run's model
    Bounds orig;     // original bounds (trajectory count)
    PingPong X, Xa;
    const double* xr;
    int two;         // 1: average term computed (second gathered vector present)
    double eps_abs;
    const double *xc, *xac;
    int traj;
    const double* w = nullptr;    // 1/s (scaled problem)
    const double* sx = nullptr;   // s: the trajectory count tests x = s x^ against orig
    __device__ void load(const Ctl* ctl)
    {
        xc = X.at(ctl->k);
        xac = Xa.at(ctl->k);
        traj = ctl->traj_on;
        eps_abs = ctl->eps_abs;
    }
    __device__ __forceinline__ void row(int j, const double* s, const double* const*, int, double* acc) const
    {
        const double cj = c[j];
        const double lo = bd.lo(j), hi = bd.hi(j);
        const double x = xc[j];
        const double xrj = xr[j];
        const double wj = w ? w[j] : 1.0;
        acc[0] += cj * x;
        const double rd = dual_terms(cj - s[0], lo, hi, acc[1], acc[2], wj);
        acc[9] += fabs(rd) > eps_abs ? 1.0 : 0.0;
        acc[3] += (x - xrj) * (x - xrj);
        if (two) {
            const double xa = xac[j];
            acc[4] += cj * xa;
            dual_terms(cj - s[1], lo, hi, acc[5], acc[6], wj);
            acc[7] += (xa - xrj) * (xa - xrj);
        }
        if (traj) {
            const double xo = sx ? x * sx[j] : x;
            acc[8] += ((xo - orig.lo(j) > eps_abs) && (orig.hi(j) - xo > eps_abs)) ? 1.0 : 0.0;
            if (two) {
                const double xa = sx ? xac[j] * sx[j] : xac[j];
                acc[10] += ((xa - orig.lo(j) > eps_abs) && (orig.hi(j) - xa > eps_abs)) ? 1.0 : 0.0;
            }
        }
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
    static constexpr int NVEC = 0;
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    const double *b, *y, *ya, *yr;
    double* axa;
    const double* w = nullptr;   // 1/r (scaled problem)
    const int8_t* sn = nullptr;  // row senses
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int i, const double* s, const double* const*, int, double* acc) const
    {
        axa[i] = s[0];
        const double bi = b[i];
        const double r = row_viol(sn, i, bi - s[0]) * (w ? w[i] : 1.0);
        acc[0] += r * r;
        const double yav = ya[i], yo = y[i], yri = yr[i];
        acc[1] += bi * yav;
        acc[2] += (yo - yri) * (yo - yri);
        acc[3] += (yav - yri) * (yav - yri);
    }
    // Fig. 1 trajectory: the off-bound count and ||b - A x|| of the iterate
    // the check leaves (the average when it restarts or returns there, else the current)
    __device__ static void record(Ctl* ctl, int64_t k, double off, double rp)
    {
        if (ctl->traj_on && ctl->traj_len < ctl->traj_cap) {
            ctl->traj_k[ctl->traj_len] = k;
            ctl->traj_off[ctl->traj_len] = (int64_t)off;
            ctl->traj_rp[ctl->traj_len] = rp;
            ctl->traj_len += 1;
        }
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        const double* en = ctl->en;
        const int64_t k = ctl->k;
        double oc[8], oa[8];
        score8(ctl->rp2_cur, en[1], en[0], ctl->bty_cur + en[2], ctl->nb, ctl->nc, oc);
        for (int i = 0; i < 8; ++i) ctl->last[i] = oc[i];
        const double off_c = en[8], off_a = en[10], rp_a = sqrt(tot[0]);
        ctl->check_pending = 0;
        if ((ctl->mode == MODE_FULL && oc[7] <= ctl->eps_rel) ||
            (ctl->mode == MODE_PRIMAL_ONLY && k >= ctl->min_iters && oc[0] <= ctl->target) ||
            (ctl->mode == MODE_DUAL_ONLY && k >= ctl->min_iters && en[9] == 0.0)) {
            record(ctl, k, off_c, oc[0]);
            ctl->done = 1; ctl->status = ST_CONVERGED; ctl->iterations = k;
            return;
        }
        if (!ctl->restart_on) record(ctl, k, off_c, oc[0]);
        if (ctl->restart_on) {
            score8(tot[0], en[5], en[4], tot[1] + en[6], ctl->nb, ctl->nc, oa);
            const double S_c = oc[7], S_a = oa[7];
            if (ctl->mode == MODE_FULL && S_a <= ctl->eps_rel) {
                for (int i = 0; i < 8; ++i) ctl->last[i] = oa[i];
                record(ctl, k, off_a, rp_a);
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
                weight_update(ctl, dx, dy);
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
                if (use_avg) record(ctl, k, off_a, rp_a);
                else record(ctl, k, off_c, oc[0]);
            } else {
                ctl->S_prev = S;
                record(ctl, k, off_c, oc[0]);
            }
        }
        if (ctl->mode != MODE_NONE && k == ctl->max_iters) {
            ctl->done = 1; ctl->status = ST_ITER_LIMIT; ctl->iterations = k;
        }
    }
};

// ------------------------------------------------------------ reflected restarted Halpern PDHG
// (the cuPDLP+ lineage of P:412-414; readings H-1..H-4).
// z = (x, y) is the Halpern sequence, zh = T(z) the PDHG map's output (the in-box point
// every test is made on and the point a run returns), z_a the anchor, t the iterations
// since the last restart, lambda = (t+1)/(t+2):
//   K1: xh = proj(x - tau (c - A^T y));  x+ = lambda((1+rho) xh - rho x) + (1-lambda) x_a
//   K2: yh = y + sigma (b - (2 A xh - A x));  y+ = lambda((1+rho) yh - rho y) + (1-lambda) y_a
//       A x+ = lambda((1+rho) A xh - rho A x) + (1-lambda) A x_a   (kept per row: no extra SpMV)
//       r^2 = ||xh-x||^2/tau + ||yh-y||^2/sigma + 2 <yh-y, A xh - A x>   (fixed-point residual)
//   every K: score(zh) (one A^T pass over yh), restart on r, weight from the anchor movement.

// K1: staged per-row inputs 0 c, 1 x_k, 2 x_anchor (3 lb, 4 ub with per-element bounds).
template <bool PE>
struct EpiPrimalH {
    static constexpr int NS = 3;   // ||xh - x||^2, ||xh - x_a||^2, #nonfinite(xh)
    static constexpr int NVEC = PE ? 5 : 3;
    static constexpr int FUSE = 1;   // hot-row fusion: row() returns xh_j, the dual step's gathered value
    const double* c;
    Bounds bd;
    PingPong X;
    const double* xa;
    double* xh;
    double tau, lam, rho;
    const double* xc;
    double* xn;
    __device__ void load(const Ctl* ctl)
    {
        tau = ctl->tau;
        rho = ctl->rho;
        lam = (double)(ctl->t + 1) / (double)(ctl->t + 2);
        xc = X.at(ctl->k);
        xn = X.at(ctl->k + 1);
    }
    __device__ __forceinline__ const double* vec(int v) const
    {
        return v == 0 ? c : v == 1 ? xc : v == 2 ? xa : v == 3 ? bd.l : bd.u;
    }
    __device__ __forceinline__ double row(int j, const double* s, const double* const* vin, int li,
                                          double* acc) const
    {
        const double x = vin[1][li];
        double lo = bd.l0, hi = bd.u0;
        if constexpr (PE) {
            lo = vin[3][li];
            hi = vin[4][li];
        }
        const double h = proj(x - tau * (vin[0][li] - s[0]), lo, hi);
        st_keep(&xh[j], h);   // gathered by the dual step
        const double a = vin[2][li];
        __stcs(&xn[j], lam * ((1.0 + rho) * h - rho * x) + (1.0 - lam) * a);
        acc[0] += (h - x) * (h - x);
        acc[1] += (h - a) * (h - a);
        acc[2] += isfinite(h) ? 0.0 : 1.0;
        return h;
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        ctl->restart_flag = 0;
        ctl->dx2_h = tot[0];
        ctl->dxa2_h = tot[1];
        ctl->nonfinite_x = tot[2] > 0.0;
    }
};

// K2: staged per-row inputs 0 b, 1 y_k, 2 (A x_k), 3 y_anchor, 4 (A x_anchor).
struct EpiDualH {
    static constexpr int NS = 6;   // ||b - A xh||^2, b^T yh, ||yh - y||^2, <yh - y, A xh - A x>, ||yh - y_a||^2, #nonfinite
    static constexpr int NVEC = 5;
    static constexpr int FUSE = 2;   // the fused rows' sums come from the primal step's partials
    const double* b;
    double *y, *ax, *yh, *axh;
    const double *ya, *axa;
    double sigma, lam, rho;
    const double* w = nullptr;   // 1/r (scaled problem): ||r_P|| in the original space
    const int8_t* sn = nullptr;
    __device__ void load(const Ctl* ctl)
    {
        sigma = ctl->sigma;
        rho = ctl->rho;
        lam = (double)(ctl->t + 1) / (double)(ctl->t + 2);
    }
    __device__ __forceinline__ const double* vec(int v) const
    {
        return v == 0 ? b : v == 1 ? y : v == 2 ? ax : v == 3 ? ya : axa;
    }
    __device__ __forceinline__ void row(int i, const double* s, const double* const* vin, int li,
                                        double* acc) const
    {
        const double sh = s[0];   // (A xh)_i
        const double bi = vin[0][li], yo = vin[1][li], axo = vin[2][li];
        const double h = dual_proj(sn, i, yo + sigma * (bi - (2.0 * sh - axo)));
        y[i] = lam * ((1.0 + rho) * h - rho * yo) + (1.0 - lam) * vin[3][li];
        ax[i] = lam * ((1.0 + rho) * sh - rho * axo) + (1.0 - lam) * vin[4][li];
        yh[i] = h;
        axh[i] = sh;
        const double r = row_viol(sn, i, bi - sh) * (w ? w[i] : 1.0);
        acc[0] += r * r;
        acc[1] += bi * h;
        acc[2] += (h - yo) * (h - yo);
        acc[3] += (h - yo) * (sh - axo);
        acc[4] += (h - vin[3][li]) * (h - vin[3][li]);
        acc[5] += isfinite(h) ? 0.0 : 1.0;
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        if (tot[5] > 0.0 || ctl->nonfinite_x) {
            ctl->done = 1; ctl->status = ST_FAIL; ctl->iterations = ctl->k + 1;
            return;
        }
        const double r2 = ctl->dx2_h / ctl->tau + tot[2] / ctl->sigma + 2.0 * tot[3];
        const double r = sqrt(r2 > 0.0 ? r2 : 0.0);
        if (ctl->t == 0) ctl->r0 = r;   // the residual at the anchor
        ctl->r_last = r;
        ctl->rp2_h = tot[0];
        ctl->bty_h = tot[1];
        ctl->dya2_h = tot[4];
        ctl->k += 1;
        ctl->t += 1;
        const int64_t k = ctl->k;
        if (ctl->mode == MODE_PRIMAL_ONLY && k >= ctl->min_iters && sqrt(tot[0]) <= ctl->target) {
            ctl->done = 1; ctl->status = ST_CONVERGED; ctl->iterations = k;
            return;
        }
        if ((k % ctl->K) == 0 && (ctl->restart_on || ctl->mode != MODE_NONE)) {
            ctl->check_pending = 1;
        } else if (ctl->mode != MODE_NONE && k == ctl->max_iters) {
            ctl->done = 1; ctl->status = ST_ITER_LIMIT; ctl->iterations = k;
        }
    }
};

// Check of a Halpern run (every K): A^T yh -> score(zh), trajectory, restart
// on the fixed-point residual, weight update from the anchor movement.
struct EpiCheckH {
    static constexpr int NS = 5;   // c^T xh, ||r_D(yh)||^2, bound terms, off-bound(xh; M), #{|r_D_j(yh)| > eps}
    static constexpr int NVEC = 0;
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    const double* c;
    const double* xh;
    Bounds bd, orig;
    double eps_abs;
    int traj;
    const double* w = nullptr;    // 1/s (scaled problem)
    const double* sx = nullptr;   // s: the trajectory count tests x = s x^ against orig
    __device__ void load(const Ctl* ctl)
    {
        traj = ctl->traj_on;
        eps_abs = ctl->eps_abs;
    }
    __device__ __forceinline__ void row(int j, const double* s, const double* const*, int, double* acc) const
    {
        const double cj = c[j], x = xh[j];
        acc[0] += cj * x;
        const double rd = dual_terms(cj - s[0], bd.lo(j), bd.hi(j), acc[1], acc[2], w ? w[j] : 1.0);
        acc[4] += fabs(rd) > eps_abs ? 1.0 : 0.0;
        if (traj) {
            const double xo = sx ? x * sx[j] : x;
            acc[3] += ((xo - orig.lo(j) > eps_abs) && (orig.hi(j) - xo > eps_abs)) ? 1.0 : 0.0;
        }
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        const int64_t k = ctl->k;
        double o[8];
        score8(ctl->rp2_h, tot[1], tot[0], ctl->bty_h + tot[2], ctl->nb, ctl->nc, o);
        for (int i = 0; i < 8; ++i) ctl->last[i] = o[i];
        if (ctl->traj_on && ctl->traj_len < ctl->traj_cap) {
            ctl->traj_k[ctl->traj_len] = k;
            ctl->traj_off[ctl->traj_len] = (int64_t)tot[3];
            ctl->traj_rp[ctl->traj_len] = o[0];
            ctl->traj_len += 1;
        }
        ctl->check_pending = 0;
        if ((ctl->mode == MODE_FULL && o[7] <= ctl->eps_rel) ||
            (ctl->mode == MODE_DUAL_ONLY && k >= ctl->min_iters && tot[4] == 0.0)) {
            ctl->done = 1; ctl->status = ST_CONVERGED; ctl->iterations = k;
            return;
        }
        if (ctl->restart_on) {
            const double r = ctl->r_last;
            if (r <= ctl->beta_suff * ctl->r0 || (r <= ctl->beta_nec * ctl->r0 && r > ctl->r_prev) ||
                (double)ctl->t >= ctl->beta_art * (double)k) {
                weight_update(ctl, sqrt(ctl->dxa2_h), sqrt(ctl->dya2_h));
                ctl->tau = ctl->eta / ctl->omega;
                ctl->sigma = ctl->eta * ctl->omega;
                ctl->restart_flag = 1;
                ctl->r_prev = INFINITY;
                ctl->t = 0;
                ctl->restarts += 1;
            } else {
                ctl->r_prev = r;
            }
        }
        if (ctl->mode != MODE_NONE && k == ctl->max_iters) {
            ctl->done = 1; ctl->status = ST_ITER_LIMIT; ctl->iterations = k;
        }
    }
};

// Halpern restart apply: z = z_anchor = zh (and their A x), the iterate of k.
struct OpRestartH {
    static constexpr int NS = 1;
    PingPong X;
    double *xa, *y, *ya, *ax, *axa;
    const double *xh, *yh, *axh;
    int32_t n, m;
    double* xc;
    __device__ void load(const Ctl* ctl) { xc = X.at(ctl->k); }
    __device__ __forceinline__ void elem(int64_t i, double*) const
    {
        if (i < n) {
            const double v = xh[i];
            xc[i] = v;
            xa[i] = v;
        }
        if (i < m) {
            const double v = yh[i], a = axh[i];
            y[i] = v;
            ya[i] = v;
            ax[i] = a;
            axa[i] = a;
        }
    }
    __device__ void finalize(const double*, Ctl*) const {}
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
    static constexpr int NS = 4;
    const double *b, *c;
    int32_t n, m;
    double omega_in;   // > 0: given
    // scaled problem (1/r, 1/s): the relative criteria use the ORIGINAL norms
    // ||b|| = ||b^ / r||, ||c|| = ||c^ / s||; omega0 uses the scaled ones (cuPDLP)
    const double* wm = nullptr;
    const double* wn = nullptr;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void elem(int64_t i, double* acc) const
    {
        if (i < m) {
            acc[0] += b[i] * b[i];
            const double bo = wm ? b[i] * wm[i] : b[i];
            acc[2] += bo * bo;
        }
        if (i < n) {
            acc[1] += c[i] * c[i];
            const double co = wn ? c[i] * wn[i] : c[i];
            acc[3] += co * co;
        }
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        const double nbs = sqrt(tot[0]), ncs = sqrt(tot[1]);
        ctl->nb = sqrt(tot[2]);
        ctl->nc = sqrt(tot[3]);
        if (omega_in > 0.0) ctl->omega = omega_in;
        else ctl->omega = (ncs > 1e-10 && nbs > 1e-10) ? ncs / nbs : 1.0;
        ctl->tau = ctl->eta / ctl->omega;
        ctl->sigma = ctl->eta * ctl->omega;
        if (ctl->mode == MODE_PRIMAL_ONLY) ctl->target = ctl->eps_rel * (1.0 + ctl->nb);
    }
};

// Run-start evaluation: A x_0 -> Ax buffer, ||b - A x_0||^2, b^T y_0.
struct EpiInitM {
    static constexpr int NS = 2;
    static constexpr int NVEC = 0;
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    const double *b, *y;
    double* ax;   // may be null (score only)
    const double* w = nullptr;   // 1/r (scaled problem)
    const int8_t* sn = nullptr;  // row senses
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int i, const double* s, const double* const*, int, double* acc) const
    {
        if (ax) ax[i] = s[0];
        const double r = row_viol(sn, i, b[i] - s[0]) * (w ? w[i] : 1.0);
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
    static constexpr int NVEC = 0;
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    const double *c, *x;
    Bounds bd;
    int decide;   // 0: only store the score in ctl->last
    const double* w = nullptr;   // 1/s (scaled problem)
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int j, const double* s, const double* const*, int, double* acc) const
    {
        const double cj = c[j];
        acc[0] += cj * x[j];
        dual_terms(cj - s[0], bd.lo(j), bd.hi(j), acc[1], acc[2], w ? w[j] : 1.0);
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
    int64_t jbase = 0;   // global index of local column 0 (distributed problems)
    const int32_t* jmap = nullptr;   // user index of internal column j (column renumbering)
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void elem(int64_t j, double* acc) const
    {
        const double x = u01(seed, jmap ? (int64_t)jmap[j] : jbase + j) - 0.5;
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
    static constexpr int NVEC = 0;
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    double* w;
    double inv;
    __device__ void load(const Ctl* ctl) { inv = ctl->pw_inv; }
    __device__ __forceinline__ void row(int i, const double* s, const double* const*, int, double*) const { w[i] = s[0] * inv; }
    __device__ void finalize(const double*, Ctl*) const {}
};
struct EpiPowN {
    static constexpr int NS = 1;
    static constexpr int NVEC = 0;
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    double* v;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int j, const double* s, const double* const*, int, double* acc) const
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
    static constexpr int NVEC = 0;
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    const double *c, *x;
    Bounds bd;
    double *z, *lhat, *uhat, *chat;
    const double* obj;   // caller objective (device copy) or null
    double eps_abs, obj_scale;
    uint64_t seed;
    int64_t jbase = 0;   // global index of local column 0 (distributed problems)
    const int32_t* jmap = nullptr;   // user index of internal column j (column renumbering)
    const double* w = nullptr;    // 1/s (scaled problem): the bound map tests z = z^ / s
    const double* sx = nullptr;   // s: objective of the corner model in the scaled space
    double* lho = nullptr;        // scaled problem: the model bounds in the original space
    double* uho = nullptr;        //   (x* = s x^* where fixed, else the original bound)
    Bounds ob{};
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void row(int j, const double* s, const double* const*, int, double* acc) const
    {
        const double zj = c[j] - s[0];
        z[j] = zj;
        const double zo = w ? zj * w[j] : zj;
        const double xj = x[j];
        if (zo < -eps_abs) { lhat[j] = xj; acc[0] += 1.0; } else lhat[j] = bd.lo(j);
        if (zo > eps_abs) { uhat[j] = xj; acc[1] += 1.0; } else uhat[j] = bd.hi(j);
        if (lho) {
            lho[j] = zo < -eps_abs ? xj * sx[j] : ob.lo(j);
            uho[j] = zo > eps_abs ? xj * sx[j] : ob.hi(j);
        }
        const double oj = obj ? obj[j] : obj_scale * u01(seed, jmap ? (int64_t)jmap[j] : jbase + j);
        chat[j] = sx ? oj * sx[j] : oj;
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        ctl->out[0] = tot[0];
        ctl->out[1] = tot[1];
    }
};

// Corner-model row senses: an inequality row whose slack has a
// non-trivial reduced cost (|y*_i| > eps_abs, y* in the original space) becomes an
// equality; counts the changed rows.
struct OpSense {
    static constexpr int NS = 1;
    const int8_t* sn;
    const double* y;
    const double* sy;   // r (scaled problem): y = r y^
    int8_t* shat;
    double eps;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void elem(int64_t ii, double* acc) const
    {
        const int i = (int)ii;
        const int s = sn[i];
        const double yo = sy ? y[i] * sy[i] : y[i];
        const bool eq = s != 0 && fabs(yo) > eps;
        shat[i] = eq ? (int8_t)0 : (int8_t)s;
        acc[0] += eq ? 1.0 : 0.0;
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const { ctl->out[2] = tot[0]; }
};

// Dual corner model (NEXT-4, reading D-1): bounds that free the off-bound columns of the
// phase-1 x (z_j = 0), keep z_j >= 0 at a lower bound and z_j <= 0 at an upper bound.
struct OpDualModel {
    static constexpr int NS = 3;   // off, lower, upper
    const double* x;
    Bounds bd;
    double *lh, *uh;
    double eps;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ void elem(int64_t jj, double* acc) const
    {
        const int j = (int)jj;
        const double xj = x[j], lo = bd.lo(j), hi = bd.hi(j);
        if (xj - lo > eps && hi - xj > eps) {
            lh[j] = -INFINITY; uh[j] = INFINITY; acc[0] += 1.0;
        } else if (xj - lo <= eps && lo > -INFINITY) {
            lh[j] = lo; uh[j] = INFINITY; acc[1] += 1.0;
        } else {
            lh[j] = -INFINITY; uh[j] = hi; acc[2] += 1.0;
        }
    }
    __device__ void finalize(const double* tot, Ctl* ctl) const
    {
        for (int i = 0; i < NS; ++i) ctl->out[i] = tot[i];
    }
};

// a10 corner statistics: counts as exact fp64 sums (< 2^53).
struct OpStats {
    static constexpr int NS = 6;   // off, off_strict, off_model, zero_rc, candidates, (spare)
    const double *x, *z, *lh, *uh;
    Bounds bd;
    double eps;
    // scaled problem: x = s x^, z = z^ / s; bd and lh/uh are ORIGINAL-space bounds
    const double* sx = nullptr;
    const double* wz = nullptr;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ static bool off(double x, double lo, double hi, double tol)
    {
        return (x - lo > tol) && (hi - x > tol);
    }
    __device__ __forceinline__ void elem(int64_t jj, double* acc) const
    {
        const int j = (int)jj;
        const double sj = sx ? sx[j] : 1.0;
        const double xj = sx ? x[j] * sj : x[j];
        const bool o = off(xj, bd.lo(j), bd.hi(j), eps);
        acc[0] += o;
        acc[1] += off(xj, bd.lo(j), bd.hi(j), 0.0);
        if (lh) acc[2] += off(xj, lh[j], uh[j], eps);   // lh/uh: model bounds in the original space
        if (z) {
            const double az = fabs(wz ? z[j] * wz[j] : z[j]);
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
