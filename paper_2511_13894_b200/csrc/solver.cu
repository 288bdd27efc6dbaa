// solver.cu — the R-PDHG run state machine (DESIGN.md §6 "Schedule"),
// Algorithm 1 orchestration, statistics, stand-alone entry points and
// the extern "C" ABI of include/cpd.h.
//
// One run = begin (power iteration, norms, projected start, initial KKT) + batches.
// A batch is the fixed node sequence
//     [check A^T pass] [check A pass + decision] [restart apply] (K1_s, K2_s) s = 0..K-1
// launched as ONE CUDA graph; every node reads the device control block and
// either does its work or returns at once (gates), so the same graph serves every
// batch and the host synchronises once per K iterations.
//
// Distributed problems: every pass goes through pass<NV>(side, ...):
// the side whose rows are split runs the SpMV into a partial buffer, reduce-
// scatters it and applies the same fused epilogue to the owned slice; scalar
// totals are allreduced and the device decision (k_fin) runs on the sums, so all
// ranks take identical decisions.  With one GPU (split < 0) pass<> is exactly
// the single fused kernel with its last-CTA finalize.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "internal.cuh"

namespace cpd {

// ------------------------------------------------------------------ Ctx
Ctx::Ctx(const cpd_problem* p) : P(p)
{
    CPD_CUDA(cudaSetDevice(p->device));
    // L2 fetch granularity for the random gathers (CPD_L2FETCH=32/64/128 bytes; device-wide)
    if (const char* lf = getenv("CPD_L2FETCH")) {
        const int g = atoi(lf);
        if (g > 0) CPD_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)g));
    }
    CPD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CPD_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    CPD_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    CPD_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    if (const char* e = getenv("CPD_CONC")) conc = e[0] != '0';
    if (const char* e = getenv("CPD_DGRID")) dense_frac = std::min(1.0, std::max(0.05, atof(e)));
    ctl_main.alloc(1);
    ctl_aux.alloc(1);
    CPD_CUDA(cudaMemset(ctl_main.p, 0, sizeof(Ctl)));
    CPD_CUDA(cudaMemset(ctl_aux.p, 0, sizeof(Ctl)));
    CPD_CUDA(cudaMallocHost(&h_main, sizeof(Ctl)));
    CPD_CUDA(cudaMallocHost(&h_aux, sizeof(Ctl)));
    std::memset(h_main, 0, sizeof(Ctl));
    std::memset(h_aux, 0, sizeof(Ctl));
    ctl = ctl_main.p;
    h_ctl = h_main;
    // block partials: every segment launch of a warp plan (<= 8 blocks/SM each) + k_finish
    const size_t nseg = std::max(p->A.plan.seg.size(), p->AT.plan.seg.size());
    bpart.alloc((size_t)p->num_sms * (8 * (nseg + 1) + 16) * NSMAX);
    ctr.alloc(1);
    CPD_CUDA(cudaMemset(ctr.p, 0, sizeof(unsigned)));
    const Plan& pa = p->A.plan;
    const Plan& pt = p->AT.plan;
    lpartA.alloc((size_t)std::max<int64_t>(1, pa.long_pieces) * GW * 2);
    lpartAT.alloc((size_t)std::max<int64_t>(1, pt.long_pieces) * GW * 2);
    if (pa.short_on) shortA.alloc((size_t)2 * p->A.rows);
    if (p->A.sell_half[0].on) sshortA.alloc((size_t)2 * p->A.sell_half[0].rows);
    if (fuse_ok(p)) {   // per-warp partials of the fused hot rows; slots never written stay 0
        hot_stride = 64 * p->num_sms;   // >= the primal step's warps (<= 64 resident per SM)
        hotpart.alloc((size_t)pa.hotd * hot_stride);
        CPD_CUDA(cudaMemset(hotpart.p, 0, sizeof(double) * (size_t)pa.hotd * hot_stride));
    }
    if (pt.short_on) shortAT.alloc((size_t)2 * p->AT.rows);
    red.alloc(NSMAX);
    CPD_CUDA(cudaMemset(red.p, 0, sizeof(double) * NSMAX));
    if (p->split >= 0) {
        part.alloc((size_t)p->world * 2 * p->L);
        recv.alloc((size_t)2 * p->L);
        CPD_CUDA(cudaMemset(part.p, 0, sizeof(double) * p->world * 2 * p->L));
        CPD_CUDA(cudaMemset(recv.p, 0, sizeof(double) * 2 * p->L));
    }
    grid_elem = p->num_sms * 4;
    p2p_setup();
}

Ctx::~Ctx()
{
    p2p_teardown();
    if (h_main) cudaFreeHost(h_main);
    if (h_aux) cudaFreeHost(h_aux);
    if (st) cudaStreamDestroy(st);
    if (side) cudaStreamDestroy(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
}

DevPlan Ctx::planA() const
{
    const Plan& pl = P->A.plan;
    return DevPlan{pl.ent.p, pl.nent, pl.nlong, pl.warp ? 1 : GW, pl.nheavy, pl.nhb, pl.dense_ent.p,
                   pl.dense_ptr.p, pl.dense_col16.p, pl.dense_maxitems, pl.short_ptr.p, pl.short_col.p, pl.short_val.p, shortA.p, nullptr,
                   pl.long_row.p,
                   pl.long_ptr.p, pl.long_ents.p, pl.nfin_heavy, lpartA.p};
}

// Hot-row fusion applies to single-GPU problems whose A^T passes run on a reversed
// SELL-32 and whose plan fused rows; not with the short-row push.
// CPD_FUSE=0 disables it at solve time.
bool fuse_ok(const cpd_problem* P)
{
    const char* e = getenv("CPD_FUSE");
    return P->A.plan.hotd > 0 && P->AT.sell.on && P->AT.sell.rev && !P->push_on && P->split < 0 &&
           !(e && e[0] == '0');
}

DevPlan Ctx::planA_fused() const
{
    DevPlan d = planA();
    const Plan& pl = P->A.plan;
    d.dense_ent = pl.dense_ent_f.p;
    d.dense_ptr = pl.dense_ptr_f.p;
    d.dense_maxitems = pl.dense_maxitems_f;
    d.hotd = pl.hotd;
    d.hot_stride = hot_stride;
    d.hot_part = hotpart.p;
    return d;
}

DevPlan Ctx::planAT() const
{
    const Plan& pl = P->AT.plan;
    return DevPlan{pl.ent.p, pl.nent, pl.nlong, pl.warp ? 1 : GW, pl.nheavy, pl.nhb, pl.dense_ent.p,
                   pl.dense_ptr.p, pl.dense_col16.p, pl.dense_maxitems, pl.short_ptr.p, pl.short_col.p, pl.short_val.p, shortAT.p, nullptr,
                   pl.long_row.p,
                   pl.long_ptr.p, pl.long_ents.p, pl.nfin_heavy, lpartAT.p};
}

void Ctx::pull_ctl()
{
    CPD_CUDA(cudaMemcpyAsync(h_ctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CPD_CUDA(cudaStreamSynchronize(st));
}

void Ctx::push_ctl(const Ctl& h)
{
    *h_ctl = h;
    CPD_CUDA(cudaMemcpyAsync(ctl, h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    CPD_CUDA(cudaStreamSynchronize(st));
}

__global__ void k_set_i64(int64_t* f, int64_t v) { *f = v; }
__global__ void k_set_i32(int32_t* f, int32_t v) { *f = v; }

void Ctx::set_i64(int64_t* f, int64_t v)
{
    k_set_i64<<<1, 1, 0, st>>>(f, v);
    CPD_CUDA(cudaGetLastError());
    ++launches;
}

void Ctx::set_i32(int32_t* f, int32_t v)
{
    k_set_i32<<<1, 1, 0, st>>>(f, v);
    CPD_CUDA(cudaGetLastError());
    ++launches;
}

void Ctx::sync() { CPD_CUDA(cudaStreamSynchronize(st)); }

static std::mutex g_grid_mu;

// Resident-CTA grid of `kernel` at (threads, dynamic smem) on the CURRENT device,
// cached per (device, kernel, smem).  The max-dynamic-smem attribute is per device,
// so it is set on every device a kernel runs on (raised to the largest size seen).
static int occ_grid(const void* kernel, int threads, size_t smem, int num_sms, int cap_per_sm = 0)
{
    int dev = 0;
    CPD_CUDA(cudaGetDevice(&dev));
    static std::map<std::tuple<int, const void*, size_t, int>, int> cache;
    std::lock_guard<std::mutex> lk(g_grid_mu);
    const auto key = std::make_tuple(dev, kernel, smem, threads);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    // the attribute only ever grows (a launch of an earlier, larger size stays valid)
    static std::map<std::pair<int, const void*>, size_t> attr;
    size_t& cur = attr.try_emplace(std::make_pair(dev, kernel), (size_t)0).first->second;
    if (smem > cur) {
        CPD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cur = smem;
    }
    int nb = 0;
    CPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem));
    nb = std::max(1, nb);
    if (cap_per_sm > 0) nb = std::min(nb, cap_per_sm);
    const int g = nb * num_sms;
    cache[key] = g;
    return g;
}
#ifndef CPD_SLAB_MERGE
#define CPD_SLAB_MERGE 1
#endif

template <int NV, class Epi>
void launch_spmv(Ctx& cx, const Matrix& M, const DevPlan& dp, VecSel v0, VecSel v1, const Epi& epi,
                 Gate g, double* red)
{
    if (M.sell.on) {
        // A^T gathers y: its hot prefix (hot-row renumbering) is staged in shared memory
        // fused primal step: per-lane accumulators of the hot rows after the staged y
        constexpr bool FZ = FuseRole<Epi>::v == 1 && NV == 1;
        const bool fz = FZ && cx.fuse && &M == &cx.P->AT;
        const int hotd = fz ? cx.P->A.plan.hotd : 0;
        const int hot = (&M == &cx.P->AT) ? std::min(cx.P->hot, fz ? HOT_ROWS_FUSED : HOT_ROWS_STAGED) : 0;
        const size_t hsm = (size_t)NV * hot * sizeof(double) + (size_t)(TPB_SELL / 32) * hotd * 32 * sizeof(double);
        const void* kfn = fz ? (const void*)k_sell<NV, Epi, FZ ? 1 : 0> : (const void*)k_sell<NV, Epi, 0>;
        const int sgrid = occ_grid(kfn, TPB_SELL, hsm, cx.P->num_sms);
        const int gr = std::max(1, std::min<int>(sgrid, (M.sell.nslice + 7) / 8));
        DevSell ds = M.dsell();
        ds.hot = hot;
        if (fz) {
            ds.hotd = hotd;
            ds.hot_stride = cx.hot_stride;
            ds.hot_part = cx.hotpart.p;
        }
        if (PushRole<Epi>::v == 1) ds.push = cx.push_acc;
        if (fz)
            k_sell<NV, Epi, FZ ? 1 : 0><<<gr, TPB_SELL, hsm, cx.st>>>(ds, v0, v1, epi, g, cx.ctl, cx.bpart.p, cx.ctr.p,
                                                                    red, 0, 1);
        else
            k_sell<NV, Epi, 0><<<gr, TPB_SELL, hsm, cx.st>>>(ds, v0, v1, epi, g, cx.ctl, cx.bpart.p, cx.ctr.p, red, 0, 1);
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
        return;
    }
    if (dp.pslot == 1) {   // warp-item plan
        const int wgrid = occ_grid((const void*)k_csrw<NV, Epi>, TPB_W, 0, cx.P->num_sms);
        Gate g0 = g;
        g0.active = nullptr;
        // one launch per item segment (rows items, then each column slab's pieces), so
        // all warps sweep one slab of the gathered vector at a time (L2-resident)
        const std::vector<int32_t>& seg = M.plan.seg;
        const bool single = dp.nlong == 0;
        int prev = 0;
        Gate gs = g;
        auto launch_dense = [&](bool concurrent = false) {
            if (dp.nheavy > 0) {   // heavy rows by dense column blocks (their slots, then k_finish)
                const size_t DSM = (size_t)NV * HB * sizeof(double);
                const bool c16 = dp.dense_col16 != nullptr;
                const void* kd = c16 ? (const void*)k_dense<NV, true> : (const void*)k_dense<NV, false>;
                const int dgrid = occ_grid(kd, TPB_D, DSM, cx.P->num_sms);
                // item-balanced: every CTA busy; concurrent: a share of the machine
                const int grd = std::max(1, concurrent ? (int)(dgrid * cx.dense_frac) : dgrid);
                cudaStream_t ss = concurrent ? cx.side : cx.st;
                if (c16) k_dense<NV, true><<<grd, TPB_D, DSM, ss>>>(M.dev(), dp, M.cols, v0, v1, g0, cx.ctl);
                else k_dense<NV, false><<<grd, TPB_D, DSM, ss>>>(M.dev(), dp, M.cols, v0, v1, g0, cx.ctl);
                CPD_CUDA(cudaGetLastError());
                ++cx.launches;
            }
        };
        const bool conc = cx.conc && dp.nheavy > 0;
        auto fork = [&]() {
            CPD_CUDA(cudaEventRecord(cx.ev_fork, cx.st));
            CPD_CUDA(cudaStreamWaitEvent(cx.side, cx.ev_fork, 0));
        };
        auto join = [&]() {
            CPD_CUDA(cudaEventRecord(cx.ev_join, cx.side));
            CPD_CUDA(cudaStreamWaitEvent(cx.st, cx.ev_join, 0));
        };
        auto launch_items = [&](int a, int b, int fin, int slab = -1, int spass = 0) {
            DevPlan ds = dp;
            if (PushRole<Epi>::v == 2) ds.push_acc = cx.push_acc;
            ds.ent = (slab >= 0 ? M.plan.short_ent.p + (size_t)slab * M.plan.seg[1] : dp.ent) + a;
            ds.nent = b - a;
            const int gr = std::max(1, std::min<int>(wgrid, (ds.nent + 7) / 8));
            k_csrw<NV, Epi><<<gr, TPB_W, 0, cx.st>>>(M.dev(), ds, v0, v1, epi, gs, cx.ctl, cx.bpart.p, cx.ctr.p,
                                                     red, prev, fin, slab, spass);
            CPD_CUDA(cudaGetLastError());
            ++cx.launches;
            gs.active = nullptr;
            if (slab < 0 || (spass & 2)) prev += gr;   // only the last slab pass leaves partials
        };
        // (the short-row push, when on, already summed the rows items' products in K1)
        if ((M.sell_short.on || M.sell_half[0].on) && !(PushRole<Epi>::v == 2 && cx.push_acc)) {
            // short-row suffix as SELL-32 passes (lane = row): one pass, or one per
            // column half (running sums between them), then the heavy rows' dense blocks
            // and every long piece; k_finish combines and finalizes
            const int sgrid = occ_grid((const void*)k_sell<NV, Epi>, TPB_SELL, 0, cx.P->num_sms);
            auto sell_pass = [&](const DevSell& ds, int nslice, int fin) {
                const int gr = std::max(1, std::min<int>(sgrid, (nslice + 7) / 8));
                k_sell<NV, Epi><<<gr, TPB_SELL, 0, cx.st>>>(ds, v0, v1, epi, gs, cx.ctl, cx.bpart.p, cx.ctr.p, red,
                                                            prev, fin);
                CPD_CUDA(cudaGetLastError());
                ++cx.launches;
                gs.active = nullptr;
                return gr;
            };
            if (conc) {   // heavy rows' dense blocks on the side stream, next to everything below
                fork();
                launch_dense(true);
            }
            if (M.sell_half[0].on) {
                static_assert(NV <= 2, "short_part holds two vectors");
                sell_pass(M.dsell_half(0, cx.sshortA.p), M.sell_half[0].nslice, 0);   // no partials
                prev += sell_pass(M.dsell_half(1, cx.sshortA.p), M.sell_half[1].nslice, single ? 1 : 0);
            } else {
                prev += sell_pass(M.dsell_short(), M.sell_short.nslice, single ? 1 : 0);
            }
            if (!conc) launch_dense();
            if (!single && seg.back() > seg[1]) launch_items(seg[1], seg.back(), 0);
            if (conc) join();
        } else if (M.plan.short_on && !(PushRole<Epi>::v == 2 && cx.push_acc)) {
            launch_dense();
            // the short rows' items once per column slab (each pass gathers from one
            // L2-resident slab of the vector), then every long piece
            const int nsl = M.plan.short_nslab;
            for (int i = 0; i < nsl; ++i) {
                const int sl = i;   // (reverse order, or the dense blocks after the passes: no different, v40)
                const int sp = (i == 0 ? 1 : 0) | (i == nsl - 1 ? 2 : 0);
                launch_items(seg[0], seg[1], (i == nsl - 1 && single) ? 1 : 0, sl, sp);
                if (M.plan.short_ilv && !single && (size_t)sl + 2 < seg.size() && seg[sl + 2] > seg[sl + 1])
                    launch_items(seg[sl + 1], seg[sl + 2], 0);   // this slab's long pieces
            }
            if (M.plan.short_ilv) {
                for (size_t k = nsl + 1; !single && k + 1 < seg.size(); ++k)
                    if (seg[k + 1] > seg[k]) launch_items(seg[k], seg[k + 1], 0);
            } else
            if (!single && seg.back() > seg[1]) launch_items(seg[1], seg.back(), 0);
        } else {
            // rows items first (x+ just written by the primal step is still in L2), then
            // the heavy rows' dense blocks, then each slab's long pieces
            for (size_t k = 0; k + 1 < seg.size(); ++k) {
                if (k == 1) launch_dense();
#if CPD_SLAB_MERGE
                if (k == 1 && !single) {   // every slab's pieces in one launch
                    if (seg.back() > seg[1]) launch_items(seg[1], seg.back(), 0);
                    break;
                }
#endif
                if (seg[k + 1] <= seg[k] && !single) continue;
                launch_items(seg[k], seg[k + 1], single ? 1 : 0);
                if (single) break;
            }
            if (seg.size() < 3) launch_dense();
        }
        if (dp.nlong > 0) {
            const int gf = std::max(1, std::min(cx.P->num_sms * 8, std::max(dp.nfin_heavy, (dp.nlong + TPB_F / 32 - 1) / (TPB_F / 32))));
            Gate g2 = g;
            g2.active = nullptr;
            k_finish<NV, Epi><<<gf, TPB_F, 0, cx.st>>>(dp, epi, g2, cx.ctl, cx.bpart.p, cx.ctr.p, prev, red);
            CPD_CUDA(cudaGetLastError());
            ++cx.launches;
        }
        return;
    }
    constexpr size_t SMEM = sizeof(SpmvSmem<NV, Epi::NVEC>);
    const int grid = occ_grid((const void*)k_spmv<NV, Epi>, TPB_SP, SMEM, cx.P->num_sms, 8);
    const int gr = std::max(1, std::min(grid, dp.nent));
    k_spmv<NV, Epi><<<gr, TPB_SP, SMEM, cx.st>>>(M.dev(), dp, v0, v1, epi, g, cx.ctl, cx.bpart.p, cx.ctr.p,
                                                 red);
    CPD_CUDA(cudaGetLastError());
    ++cx.launches;
    if (dp.nlong > 0) {
        const int gf = std::max(1, std::min(cx.P->num_sms * 8, std::max(dp.nfin_heavy, (dp.nlong + TPB_F / 32 - 1) / (TPB_F / 32))));
        Gate g2 = g;
        g2.active = nullptr;
        k_finish<NV, Epi><<<gf, TPB_F, 0, cx.st>>>(dp, epi, g2, cx.ctl, cx.bpart.p, cx.ctr.p, gr, red);
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
    }
}

template <class Op>
void launch_elem(Ctx& cx, int64_t N, const Op& op, Gate g, double* red)
{
    const int64_t need = (N + TPB - 1) / TPB;
    const int gr = (int)std::max<int64_t>(1, std::min<int64_t>(need, cx.grid_elem));
    k_elem<Op><<<gr, TPB, 0, cx.st>>>(N, op, g, cx.ctl, cx.bpart.p, cx.ctr.p, red);
    CPD_CUDA(cudaGetLastError());
    ++cx.launches;
}

template <class Epi>
static void launch_fin(Ctx& cx, const Epi& e, Gate g)
{
    g.active = nullptr;
    k_fin<Epi><<<1, 1, 0, cx.st>>>(e, g, cx.ctl, cx.red.p);
    CPD_CUDA(cudaGetLastError());
    ++cx.launches;
}

// One epilogue pass over side `side` (0: rows of A, m-side; 1: rows of A^T, n-side).
template <int NV, class Epi>
static void pass(Ctx& cx, int side, VecSel v0, VecSel v1, const Epi& epi, Gate g)
{
    const cpd_problem* P = cx.P;
    const Matrix& M = side ? P->AT : P->A;
    const DevPlan dp = side ? cx.planAT()
                            : ((FuseRole<Epi>::v == 2 && NV == 1 && cx.fuse) ? cx.planA_fused() : cx.planA());
    if (P->split < 0) {
        launch_spmv<NV>(cx, M, dp, v0, v1, epi, g, nullptr);
        return;
    }
    if (P->split == side && cx.p2p) {
        // fused: the SpMV stores each row sum into its owner's window (NVLink peer
        // memory); a one-scalar allreduce is the barrier before the owners' sums
        EpiStorePeer<NV> es{cx.peer.p, P->L, P->rank};
        launch_spmv<NV>(cx, M, dp, v0, v1, es, g, nullptr);
        cx.allreduce_sum(cx.red.p + NSMAX - 1, 1);
        const int64_t N = P->own_len[side];
        const int gr = (int)std::max<int64_t>(1, std::min<int64_t>((N + TPB - 1) / TPB, cx.grid_elem));
        Gate g2 = g;
        g2.active = nullptr;
        k_slice_p2p<NV, Epi><<<gr, TPB, 0, cx.st>>>(N, P->L, P->world, cx.winbuf, epi, g2, cx.ctl, cx.bpart.p,
                                                    cx.ctr.p, cx.red.p);
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
    } else if (P->split == side) {
        EpiStore<NV> es{cx.part.p, P->L};
        launch_spmv<NV>(cx, M, dp, v0, v1, es, g, nullptr);
        cx.reduce_scatter(cx.part.p, cx.recv.p, (int64_t)NV * P->L);
        const int64_t N = P->own_len[side];
        const int gr = (int)std::max<int64_t>(1, std::min<int64_t>((N + TPB - 1) / TPB, cx.grid_elem));
        Gate g2 = g;
        g2.active = nullptr;
        k_slice<NV, Epi><<<gr, TPB, 0, cx.st>>>(N, P->L, cx.recv.p, epi, g2, cx.ctl, cx.bpart.p, cx.ctr.p,
                                                cx.red.p);
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
    } else {
        launch_spmv<NV>(cx, M, dp, v0, v1, epi, g, cx.red.p);
    }
    cx.allreduce_sum(cx.red.p, Epi::NS);
    launch_fin(cx, epi, g);
}

// Elementwise pass over the owned parts; `reduce` = the op's totals matter.
template <class Op>
static void elem(Ctx& cx, int64_t N, const Op& op, Gate g, bool reduce)
{
    const cpd_problem* P = cx.P;
    if (P->split < 0) {
        launch_elem(cx, N, op, g, nullptr);
        return;
    }
    launch_elem(cx, N, op, g, cx.red.p);
    if (reduce) {
        cx.allreduce_sum(cx.red.p, Op::NS);
        launch_fin(cx, op, g);
    }
}

// Replica of a split-side vector for the other side's gathers: the owned slice
// is copied into its place of `rep` (world * L) and all-gathered in place.
static void refresh(Ctx& cx, int side, VecSel src, double* rep, Gate g)
{
    const cpd_problem* P = cx.P;
    if (P->split != side) return;
    const int64_t N = P->own_len[side];
    const int gr = (int)std::max<int64_t>(1, std::min<int64_t>((N + TPB - 1) / TPB, cx.grid_elem));
    g.active = nullptr;
    k_copy_sel<<<gr, TPB, 0, cx.st>>>(N, rep + (int64_t)P->rank * P->L, src, g, cx.ctl);
    CPD_CUDA(cudaGetLastError());
    ++cx.launches;
    cx.all_gather_inplace(rep, P->L);
}

static Gate always() { return Gate{GATE_ALWAYS, 0, 0, nullptr}; }
static VecSel fixed(const double* v) { return VecSel{v, v, 0}; }
static VecSel none() { return VecSel{nullptr, nullptr, 0}; }

// Replica of the split side for one-off evaluations: `ext` (world * L doubles)
// or a scratch allocation.
struct Reps {
    DBuf<double> own;
    double* r = nullptr;
    explicit Reps(const cpd_problem* P, double* ext = nullptr)
    {
        if (P->split < 0) return;
        if (ext) {
            r = ext;
            return;
        }
        own.alloc((size_t)P->world * P->L);
        CPD_CUDA(cudaMemset(own.p, 0, sizeof(double) * P->world * P->L));
        r = own.p;
    }
    // gathered view of an owned vector of `side` (refreshing the replica if split)
    const double* view(Ctx& cx, int side, const double* v)
    {
        if (cx.P->split != side) return v;
        refresh(cx, side, fixed(v), r, always());
        return r;
    }
};

// Standalone evaluations shared by the solver and the stand-alone ABI calls.
// score of (x, y) (owned parts) for objective c / bounds bd (owned parts)
static void eval_score(Ctx& cx, const double* x, const double* y, const double* c, Bounds bd,
                       double nb, double nc, double out[8], const int8_t* sn = nullptr)
{
    AuxScope aux(cx);
    const cpd_problem* P = cx.P;
    Reps rp(P);
    Ctl h{};
    h.nb = nb;
    h.nc = nc;
    h.K = 1;
    cx.push_ctl(h);
    EpiInitM em{P->b_own(), y, nullptr};
    em.w = P->w_m();
    em.sn = sn;
    pass<1>(cx, 0, fixed(rp.view(cx, 1, x)), none(), em, always());
    EpiInitN en{c, x, bd, 0};
    en.w = P->w_n();
    pass<1>(cx, 1, fixed(rp.view(cx, 0, y)), none(), en, always());
    cx.pull_ctl();
    for (int i = 0; i < 8; ++i) out[i] = cx.h_ctl->last[i];
}

static void eval_norms(Ctx& cx, const double* b, const double* c, double* nb, double* nc)
{
    AuxScope aux(cx);
    const cpd_problem* P = cx.P;
    Ctl h{};
    h.K = 1;
    h.mode = MODE_NONE;
    h.eta = 1.0;
    cx.push_ctl(h);
    OpNorms on{b, c, P->own_len[1], P->own_len[0], 1.0};
    on.wm = P->w_m();
    on.wn = P->w_n();
    elem(cx, std::max(P->own_len[1], P->own_len[0]), on, always(), true);
    cx.pull_ctl();
    *nb = cx.h_ctl->nb;
    *nc = cx.h_ctl->nc;
}

// internal: x, z are the solver's (scaled-space) vectors and lh/uh original-space
// model bounds; else every array is already in the original space
static void eval_stats(Ctx& cx, bool internal, const double* x, const double* z, const double* lh, const double* uh,
                       double eps, int64_t floor_, int64_t fix_lb, int64_t fix_ub, cpd_stats* out)
{
    AuxScope aux(cx);
    const cpd_problem* P = cx.P;
    Ctl h{};
    h.K = 1;
    cx.push_ctl(h);
    OpStats os{x, z, lh, uh, P->bounds_orig(), eps};
    if (internal) {
        os.sx = P->s_n();
        os.wz = P->w_n();
    }
    elem(cx, P->own_len[1], os, always(), true);
    cx.pull_ctl();
    const double* o = cx.h_ctl->out;
    std::memset(out, 0, sizeof(*out));
    out->off_bound = (int64_t)o[0];
    out->off_bound_strict = (int64_t)o[1];
    out->off_bound_model = lh ? (int64_t)o[2] : 0;
    out->zero_rc = z ? (int64_t)o[3] : 0;
    out->candidates = z ? (int64_t)o[4] : 0;
    out->fix_lb = fix_lb;
    out->fix_ub = fix_ub;
    out->rows_eq = 0;
    const int64_t m = P->m_glob;
    out->est_primal_pushes = std::max<int64_t>(out->off_bound - m, 0);
    out->est_dual_pushes = z ? std::max<int64_t>(m - out->zero_rc, 0) : 0;
    const int64_t thr = std::max<int64_t>(2 * m, floor_);
    out->is_candidate = z ? (out->candidates >= thr) : 0;
}

// sigma_hat by `iters` power iterations; v (n-side owned), w (m-side owned) scratch.
static void power_iterate(Ctx& cx, Reps& rp, int32_t iters, uint64_t seed, double* v, double* w)
{
    const cpd_problem* P = cx.P;
    OpPowInit pi{v, seed, P->own_len[1], P->gofs[1]};
    pi.jmap = P->cperm.p;   // U(seed, user column)
    elem(cx, P->own_len[1], pi, always(), true);
    for (int it = 0; it < iters; ++it) {
        EpiPowM pm{w, 0.0};
        pass<1>(cx, 0, fixed(rp.view(cx, 1, v)), none(), pm, always());
        EpiPowN pn{v};
        pass<1>(cx, 1, fixed(rp.view(cx, 0, w)), none(), pn, always());
    }
}

static double power_sigma(Ctx& cx, int32_t iters, uint64_t seed, double step_scale, double* v,
                          double* w)
{
    AuxScope aux(cx);
    Reps rp(cx.P);
    Ctl h{};
    h.K = 1;
    h.step_scale = step_scale;
    cx.push_ctl(h);
    power_iterate(cx, rp, iters, seed, v, w);
    cx.pull_ctl();
    return cx.h_ctl->sigma_hat;
}

__global__ void k_copy(int64_t N, double* dst, const double* src)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// op 0: dst = src / d (into the scaled space); op 1: dst = src * d (back to the original)
__global__ void k_scale_vec(int64_t N, double* dst, const double* src, const double* d, int op)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = op ? src[i] * d[i] : src[i] / d[i];
}

// internal row order <-> user order of y-side vectors (hot-row renumbering):
// mode 0 gather dst[k] = src[perm[k]] (user -> internal); mode 1 scatter dst[perm[k]] = src[k]
__global__ void k_perm_vec(int64_t N, double* dst, const double* src, const int32_t* perm, int mode)
{
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (mode) dst[perm[k]] = src[k];
        else dst[k] = src[perm[k]];
    }
}

__global__ void k_zero(int64_t N, double* dst)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = 0.0;
}

// z = c - A^T y
struct EpiZ {
    static constexpr int NS = 1;
    static constexpr int NVEC = 0;
    const double* c;
    double* z;
    __device__ void load(const Ctl*) {}
    __device__ __forceinline__ const double* vec(int) const { return nullptr; }
    __device__ __forceinline__ void row(int j, const double* s, const double* const*, int, double*) const
    {
        z[j] = c[j] - s[0];
    }
    __device__ void finalize(const double*, Ctl*) const {}
};

}  // namespace cpd

// ====================================================================== solver
using namespace cpd;

enum { NODE_CHECK_N = 0, NODE_CHECK_M = 1, NODE_RESTART = 2, NODE_K0 = 3 };
enum { KT_K1 = 0, KT_K2 = 1, KT_CN = 2, KT_CM = 3, KT_RS = 4, KT_N = 5 };
static const char* KT_NAMES[3][KT_N] = {
    {"primal_step_AT", "dual_step_A", "check_eval_AT", "check_eval_A", "restart_apply"},
    {"primal_step_AT:corner", "dual_step_A:corner", "check_eval_AT:corner", "check_eval_A:corner",
     "restart_apply:corner"},
    {"primal_step_AT:dual", "dual_step_A:dual", "check_eval_AT:dual", "check_eval_A:dual", "restart_apply:dual"}};

struct RunCfg {
    int kind = 0;            // 0 original model, 1 corner model, 2 dual corner model (NEXT-4)
    int mode = MODE_FULL;
    int64_t max_iters = 0, min_iters = 0;
    double time_limit = 0.0;
    const double* xs = nullptr;
    const double* ys = nullptr;   // null => y = 0
    bool power = false;
    double eta = 0.0;
    double omega_in = 0.0;
    int traj = 0;
};

struct cpd_solver {
    const cpd_problem* P;
    cpd_params prm;
    Ctx cx;
    // state vectors: n-side (x-like) of length own_len[1], m-side (y-like) own_len[0]
    DBuf<double> X0, X1, Xa0, Xa1, Xr, Y, Ya, Yr, AX, AXa, Ystar, Z, lhat, uhat, chat, objd, SN, SM;
    DBuf<double> LHo, UHo, TX, TY, TY2, TX2;   // scaled problems: original-space model bounds; unscale scratch
    DBuf<double> XH, YH, AXH;         // Halpern: T(z) = (xh, yh) of the last iteration and A xh
    DBuf<double> LHD, UHD, XS;        // dual corner model bounds; the phase-1 x it keeps
    DBuf<int8_t> shat;                // corner-model row senses
    DBuf<double> ACC;                 // short-row push sums (m), zero between iterations
    int64_t rows_eq = 0;
    // replicas of the split side (world * L): current vector / its average
    DBuf<double> RV, RA;
    DBuf<int64_t> trk, troff;
    DBuf<double> trrp;
    DBuf<int32_t> active;
    int32_t* h_active = nullptr;
    int cur_par = 0;            // parity of the buffer holding the current x
    bool run_active = false;
    int run_kind = 0;
    int64_t run_k_base = 0;
    bool have_corner = false;
    double eta_phase1 = 0.0;
    bool eta_known = false;
    int64_t fix_lb = 0, fix_ub = 0;
    double corner_eps = 1e-6;
    cudaGraphExec_t gexec[3] = {nullptr, nullptr, nullptr};
    cudaGraph_t graph[3] = {nullptr, nullptr, nullptr};
    std::vector<cudaEvent_t> ev0, ev1;
    double kt_ms[3][KT_N] = {};
    int64_t kt_n[3][KT_N] = {};
    int nnodes = 0;
    const int64_t traj_cap = 1 << 16;
    int64_t graph_kernels[3] = {0, 0, 0};
    int64_t graph_launches = 0;

    cpd_solver(const cpd_problem* p, const cpd_params& pr) : P(p), prm(pr), cx(p)
    {
        const size_t n = p->own_len[1], m = p->own_len[0];
        for (auto* b : {&X0, &X1, &Xa0, &Xa1, &Xr, &Z, &lhat, &uhat, &chat, &objd, &SN}) b->alloc(n);
        for (auto* b : {&Y, &Ya, &Yr, &AX, &AXa, &Ystar, &SM}) b->alloc(m);
        for (auto* b : {&X0, &X1, &Xa0, &Xa1, &Xr, &Z}) CPD_CUDA(cudaMemset(b->p, 0, sizeof(double) * n));
        for (auto* b : {&Y, &Ya, &Yr, &AX, &AXa, &Ystar}) CPD_CUDA(cudaMemset(b->p, 0, sizeof(double) * m));
        if (pr.method == 1) {
            XH.alloc(n);
            YH.alloc(m);
            AXH.alloc(m);
        }
        if (p->push_on) {
            ACC.alloc(std::max<int32_t>(p->m, 1));
            CPD_CUDA(cudaMemset(ACC.p, 0, sizeof(double) * p->m));
        }
        if (p->split >= 0) {
            const size_t R = (size_t)p->world * p->L;
            RV.alloc(R);
            RA.alloc(R);
            CPD_CUDA(cudaMemset(RV.p, 0, sizeof(double) * R));
            CPD_CUDA(cudaMemset(RA.p, 0, sizeof(double) * R));
        }
        trk.alloc(traj_cap);
        troff.alloc(traj_cap);
        trrp.alloc(traj_cap);
        nnodes = NODE_K0 + 2 * prm.check_every;
        active.alloc(nnodes);
        CPD_CUDA(cudaMallocHost(&h_active, sizeof(int32_t) * nnodes));
        if (prm.profile) {
            ev0.resize(nnodes);
            ev1.resize(nnodes);
            for (int i = 0; i < nnodes; ++i) {
                CPD_CUDA(cudaEventCreate(&ev0[i]));
                CPD_CUDA(cudaEventCreate(&ev1[i]));
            }
        }
        CPD_CUDA(cudaDeviceSynchronize());
    }
    ~cpd_solver()
    {
        for (int k = 0; k < 3; ++k) {
            if (gexec[k]) cudaGraphExecDestroy(gexec[k]);
            if (graph[k]) cudaGraphDestroy(graph[k]);
        }
        for (auto e : ev0) cudaEventDestroy(e);
        for (auto e : ev1) cudaEventDestroy(e);
        if (h_active) cudaFreeHost(h_active);
    }
    const int8_t* sense_of(int kind) const
    {
        return kind == 1 ? (P->has_sense ? shat.p : nullptr) : P->sense_own();
    }
    const double* lh_orig() const { return P->scaled ? LHo.p : lhat.p; }
    const double* uh_orig() const { return P->scaled ? UHo.p : uhat.p; }
    int32_t nO() const { return P->own_len[1]; }
    int32_t mO() const { return P->own_len[0]; }
    double* Xp(int par) { return par ? X1.p : X0.p; }

    const double* obj_of(int kind) const { return kind == 1 ? chat.p : P->c_own(); }
    Bounds bounds_of(int kind) const
    {
        if (kind == 1) return Bounds{lhat.p, uhat.p, 0.0, 0.0};
        if (kind == 2) return Bounds{LHD.p, UHD.p, 0.0, 0.0};
        return P->bounds_own();
    }
    // gather source of an owned vector of `side`: the replica when that side is split
    VecSel gsrc(int side, VecSel own, double* rep) const { return P->split == side ? fixed(rep) : own; }

    // ---------------------------------------------------------- begin
    void begin(const RunCfg& rc)
    {
        const int32_t n = nO(), m = mO();
        Ctl h{};
        h.mode = rc.mode;
        h.restart_on = prm.restart ? 1 : 0;
        h.K = prm.check_every;
        h.traj_on = rc.traj;
        h.k_stop = 0;
        h.max_iters = rc.max_iters;
        h.min_iters = rc.min_iters;
        h.eps_rel = prm.eps_rel;
        h.eps_abs = corner_eps;
        h.beta_suff = prm.beta_suff;
        h.beta_nec = prm.beta_nec;
        h.beta_art = prm.beta_art;
        h.theta = prm.theta;
        h.status = ST_RUNNING;
        h.eta = rc.eta;
        h.step_scale = prm.step_scale;
        h.S_prev = INFINITY;
        h.traj_cap = traj_cap;
        h.traj_k = trk.p;
        h.traj_off = troff.p;
        h.traj_rp = trrp.p;
        h.method = prm.method;
        h.pid = prm.pid;
        h.rho = prm.reflection;
        h.kp = prm.kp;
        h.ki = prm.ki;
        h.kd = prm.kd;
        h.r0 = h.r_prev = h.r_last = INFINITY;
        cx.push_ctl(h);
        if (ACC.p) CPD_CUDA(cudaMemsetAsync(ACC.p, 0, sizeof(double) * P->m, cx.st));   // no stale pushes
        Reps rp(P, RV.p);
        if (rc.power) power_iterate(cx, rp, prm.power_iters, prm.seed, SN.p, SM.p);   // writes ctl->eta
        const double* c = obj_of(rc.kind);
        const Bounds bd = bounds_of(rc.kind);
        OpNorms on{P->b_own(), c, n, m, rc.omega_in};
        on.wm = P->w_m();
        on.wn = P->w_n();
        elem(cx, std::max(n, m), on, always(), true);
        OpBegin ob{rc.xs, rc.ys, bd, X0.p, Xa0.p, Xa1.p, Xr.p, Y.p, Ya.p, Yr.p, n, m, rc.ys ? 0 : 1};
        elem(cx, std::max(n, m), ob, always(), false);
        EpiInitM em{P->b_own(), Y.p, AX.p};
        em.w = P->w_m();
        em.sn = sense_of(rc.kind);
        pass<1>(cx, 0, fixed(rp.view(cx, 1, X0.p)), none(), em, always());
        EpiInitN en{c, X0.p, bd, 1};
        en.w = P->w_n();
        // the batch's K1 gathers the y replica: refresh it here (split m-side)
        refresh(cx, 0, fixed(Y.p), RV.p, always());
        pass<1>(cx, 1, gsrc(0, fixed(Y.p), RV.p), none(), en, always());
        if (prm.method == 1) {   // Halpern: anchor z_a = z_0 (and A x_a), T(z) "so far" = z_0
            const int g = std::min<int64_t>(cx.grid_elem, ((int64_t)std::max(n, m) + 255) / 256 + 1);
            k_copy<<<g, 256, 0, cx.st>>>(n, Xa0.p, X0.p);
            k_copy<<<g, 256, 0, cx.st>>>(n, XH.p, X0.p);
            k_copy<<<g, 256, 0, cx.st>>>(m, Ya.p, Y.p);
            k_copy<<<g, 256, 0, cx.st>>>(m, YH.p, Y.p);
            k_copy<<<g, 256, 0, cx.st>>>(m, AXa.p, AX.p);
            k_copy<<<g, 256, 0, cx.st>>>(m, AXH.p, AX.p);
            CPD_CUDA(cudaGetLastError());
            cx.launches += 6;
        }
        cx.pull_ctl();
        cur_par = 0;
        run_active = true;
        run_kind = rc.kind;
        if (!std::isfinite(cx.h_ctl->eta) || !(cx.h_ctl->eta > 0.0))
            throw Error(CPD_E_ARG, "step size is not positive and finite (zero matrix?)");
    }

    // ---------------------------------------------------------- one Halpern batch
    // [check: A^T yh -> score(zh), restart test] [restart apply] (K1_s, K2_s)_{s<K}
    template <class Rec>
    void enqueue_batch_halpern(int kind, bool, Rec& rec)
    {
        const int32_t n = nO(), m = mO();
        const int K = prm.check_every;
        const double* c = obj_of(kind);
        const Bounds bd = bounds_of(kind);
        const PingPong X{{X0.p, X1.p}};
        {
            EpiCheckH e{c, XH.p, bd, P->bounds_orig(), 0.0, 0};
            e.w = P->w_n();
            e.sx = P->s_n();
            Gate g{GATE_CHECK, 0, NODE_CHECK_N, active.p};
            rec(ev0, NODE_CHECK_N);
            pass<1>(cx, 1, fixed(YH.p), none(), e, g);
            rec(ev1, NODE_CHECK_N);
            OpRestartH orr{X, Xa0.p, Y.p, Ya.p, AX.p, AXa.p, XH.p, YH.p, AXH.p, n, m, nullptr};
            Gate gr{GATE_RESTART, 0, NODE_RESTART, active.p};
            rec(ev0, NODE_RESTART);
            elem(cx, std::max(n, m), orr, gr, false);
            rec(ev1, NODE_RESTART);
        }
        cx.fuse = fuse_ok(P);   // primal step forms the hot rows' A xh products (as for R-PDHG)
        for (int s = 0; s < K; ++s) {
            const int n1 = NODE_K0 + 2 * s, n2 = n1 + 1;
            const Gate g1{GATE_K1, s, n1, active.p}, g2{GATE_K2, s, n2, active.p};
            rec(ev0, n1);
            if (kind == 0 && P->uniform_bounds) {
                EpiPrimalH<false> e1{c, bd, X, Xa0.p, XH.p, 0.0, 0.0, 0.0, nullptr, nullptr};
                pass<1>(cx, 1, fixed(Y.p), none(), e1, g1);
            } else {
                EpiPrimalH<true> e1{c, bd, X, Xa0.p, XH.p, 0.0, 0.0, 0.0, nullptr, nullptr};
                pass<1>(cx, 1, fixed(Y.p), none(), e1, g1);
            }
            rec(ev1, n1);
            EpiDualH e2{P->b_own(), Y.p, AX.p, YH.p, AXH.p, Ya.p, AXa.p, 0.0, 0.0, 0.0};
            e2.w = P->w_m();
            e2.sn = sense_of(kind);
            rec(ev0, n2);
            pass<1>(cx, 0, fixed(XH.p), none(), e2, g2);
            rec(ev1, n2);
        }
        cx.fuse = false;
    }

    // ---------------------------------------------------------- one batch
    void enqueue_batch(int kind, bool capture)
    {
        const int64_t l0 = cx.launches;
        const int32_t n = nO(), m = mO();
        const int K = prm.check_every;
        const double* c = obj_of(kind);
        const Bounds bd = bounds_of(kind);
        const Bounds orig = P->bounds_orig();
        const PingPong X{{X0.p, X1.p}}, Xa{{Xa0.p, Xa1.p}};
        auto rec = [&](std::vector<cudaEvent_t>& ev, int node) {
            if (!prm.profile) return;
            if (capture) CPD_CUDA(cudaEventRecordWithFlags(ev[node], cx.st, cudaEventRecordExternal));
            else CPD_CUDA(cudaEventRecord(ev[node], cx.st));
        };
        CPD_CUDA(cudaMemsetAsync(active.p, 0, sizeof(int32_t) * nnodes, cx.st));
        if (prm.method == 1) {   // reflected restarted Halpern PDHG (NEXT-1)
            enqueue_batch_halpern(kind, capture, rec);
            if (capture) graph_kernels[kind] = cx.launches - l0;
            CPD_CUDA(cudaMemcpyAsync(h_active, active.p, sizeof(int32_t) * nnodes, cudaMemcpyDeviceToHost, cx.st));
            CPD_CUDA(cudaMemcpyAsync(cx.h_ctl, cx.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, cx.st));
            return;
        }
        // restart check: A^T pass (current y and average y) + A pass (A x_avg) + decision
        {
            EpiCheckN e{c, bd, orig, X, Xa, Xr.p, prm.restart ? 1 : 0, 0.0, nullptr, nullptr, 0};
            e.w = P->w_n();
            e.sx = P->s_n();
            Gate g{GATE_CHECK, 0, NODE_CHECK_N, active.p};
            rec(ev0, NODE_CHECK_N);
            // RV holds y_k (refreshed after every dual step); RA <- average of y
            if (prm.restart) {
                refresh(cx, 0, fixed(Ya.p), RA.p, g);
                pass<2>(cx, 1, gsrc(0, fixed(Y.p), RV.p), gsrc(0, fixed(Ya.p), RA.p), e, g);
            } else {
                pass<1>(cx, 1, gsrc(0, fixed(Y.p), RV.p), none(), e, g);
            }
            rec(ev1, NODE_CHECK_N);
            EpiCheckM em{P->b_own(), Y.p, Ya.p, Yr.p, AXa.p};
            em.w = P->w_m();
            em.sn = sense_of(kind);
            Gate gm{GATE_CHECK, 0, NODE_CHECK_M, active.p};
            rec(ev0, NODE_CHECK_M);
            refresh(cx, 1, VecSel{Xa0.p, Xa1.p, 2}, RA.p, gm);
            pass<1>(cx, 0, gsrc(1, VecSel{Xa0.p, Xa1.p, 2}, RA.p), none(), em, gm);
            rec(ev1, NODE_CHECK_M);
            OpRestart orr{X, Xa, Y.p, Ya.p, AX.p, AXa.p, Xr.p, Yr.p, n, m, 0, nullptr, nullptr};
            Gate gr{GATE_RESTART, 0, NODE_RESTART, active.p};
            rec(ev0, NODE_RESTART);
            elem(cx, std::max(n, m), orr, gr, false);
            refresh(cx, 0, fixed(Y.p), RV.p, gr);   // y may have changed
            rec(ev1, NODE_RESTART);
        }
        cx.push_acc = ACC.p;   // primal step pushes short-row products, dual step consumes them
        cx.fuse = fuse_ok(P);  // primal step forms the hot rows' dual-step products
        for (int s = 0; s < K; ++s) {
            const int n1 = NODE_K0 + 2 * s, n2 = n1 + 1;
            const Gate g1{GATE_K1, s, n1, active.p}, g2{GATE_K2, s, n2, active.p};
            rec(ev0, n1);
            const VecSel ysrc = gsrc(0, fixed(Y.p), RV.p);
            if (kind == 0 && P->uniform_bounds) {   // scalar bounds: 3 staged per-row inputs
                EpiPrimalT<false> e1{c, bd, X, Xa, 0.0, 0.0, 0.0, nullptr, nullptr, nullptr, nullptr};
                e1.w = P->w_n();
                pass<1>(cx, 1, ysrc, none(), e1, g1);
            } else {
                EpiPrimalT<true> e1{c, bd, X, Xa, 0.0, 0.0, 0.0, nullptr, nullptr, nullptr, nullptr};
                e1.w = P->w_n();
                pass<1>(cx, 1, ysrc, none(), e1, g1);
            }
            // x_{k+1} replica for the dual step's gathers (split n-side); the
            // gate is the dual step's: it runs exactly when the dual step does
            refresh(cx, 1, VecSel{X0.p, X1.p, 1}, RV.p, g2);
            rec(ev1, n1);
            EpiDual e2{P->b_own(), Y.p, Ya.p, AX.p, 0.0, 0.0};
            e2.w = P->w_m();
            e2.sn = sense_of(kind);
            rec(ev0, n2);
            pass<1>(cx, 0, gsrc(1, VecSel{X0.p, X1.p, 1}, RV.p), none(), e2, g2);
            // y_{k+1} replica for the next primal step (split m-side); k already advanced
            refresh(cx, 0, fixed(Y.p), RV.p, always());
            rec(ev1, n2);
        }
        cx.push_acc = nullptr;
        cx.fuse = false;
        if (capture) graph_kernels[kind] = cx.launches - l0;
        CPD_CUDA(cudaMemcpyAsync(h_active, active.p, sizeof(int32_t) * nnodes, cudaMemcpyDeviceToHost, cx.st));
        CPD_CUDA(cudaMemcpyAsync(cx.h_ctl, cx.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, cx.st));
    }

    void run_batch()
    {
        const int kind = run_kind;
        if (prm.use_graph) {
            if (!gexec[kind]) {
                CPD_CUDA(cudaStreamBeginCapture(cx.st, cudaStreamCaptureModeThreadLocal));
                try {
                    enqueue_batch(kind, true);
                } catch (...) {
                    cudaGraph_t g;
                    cudaStreamEndCapture(cx.st, &g);
                    if (g) cudaGraphDestroy(g);
                    throw;
                }
                CPD_CUDA(cudaStreamEndCapture(cx.st, &graph[kind]));
                CPD_CUDA(cudaGraphInstantiate(&gexec[kind], graph[kind], 0));
                cx.launches -= graph_kernels[kind];   // capture counted them; launches count below
            }
            CPD_CUDA(cudaGraphLaunch(gexec[kind], cx.st));
            cx.launches += graph_kernels[kind];
            graph_launches += 1;
        } else {
            enqueue_batch(kind, false);
        }
        CPD_CUDA(cudaStreamSynchronize(cx.st));
        if (prm.profile) account_times(kind);
    }

    void account_times(int kind)
    {
        for (int node = 0; node < nnodes; ++node) {
            if (!h_active[node]) continue;
            float ms = 0.f;
            CPD_CUDA(cudaEventElapsedTime(&ms, ev0[node], ev1[node]));
            int kt;
            if (node == NODE_CHECK_N) kt = KT_CN;
            else if (node == NODE_CHECK_M) kt = KT_CM;
            else if (node == NODE_RESTART) kt = KT_RS;
            else kt = ((node - NODE_K0) & 1) ? KT_K2 : KT_K1;
            kt_ms[kind][kt] += ms;
            kt_n[kind][kt] += 1;
        }
    }

    // Advance the run until it terminates or reaches iteration k_stop.
    void advance(int64_t k_stop, double time_limit)
    {
        cx.set_i64(&cx.ctl->k_stop, k_stop);
        cx.pull_ctl();
        const auto t0 = std::chrono::steady_clock::now();
        while (true) {
            const Ctl& h = *cx.h_ctl;
            if (h.done) break;
            if (h.k >= k_stop && !h.check_pending) break;
            run_batch();
            if (time_limit > 0.0 && !cx.h_ctl->done) {
                double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                cx.allreduce_max_host(&el);   // distributed: one decision for all ranks
                if (el > time_limit) {
                    cx.set_i32(&cx.ctl->status, ST_TIME_LIMIT);
                    cx.set_i64(&cx.ctl->iterations, cx.h_ctl->k);
                    cx.set_i32(&cx.ctl->done, 1);
                    cx.pull_ctl();
                    break;
                }
            }
        }
        cur_par = (int)(cx.h_ctl->k & 1);
    }

    // After a terminated run: make (X[cur_par], Y) the returned point.
    void commit()
    {
        const Ctl& h = *cx.h_ctl;
        const int64_t k = h.k;
        cur_par = (int)(k & 1);
        if (prm.method == 1 && k > 0) {   // Halpern: the run returns T(z) of its last iteration
            const int g = std::min<int64_t>(cx.grid_elem, ((int64_t)std::max(nO(), mO()) + 255) / 256 + 1);
            k_copy<<<g, 256, 0, cx.st>>>(nO(), Xp(cur_par), XH.p);
            k_copy<<<g, 256, 0, cx.st>>>(mO(), Y.p, YH.p);
            CPD_CUDA(cudaGetLastError());
            cx.launches += 2;
        } else if (h.returned_average) {
            const int g = std::min<int64_t>(cx.grid_elem, ((int64_t)std::max(nO(), mO()) + 255) / 256 + 1);
            k_copy<<<g, 256, 0, cx.st>>>(nO(), Xp(cur_par), (k & 1) ? Xa1.p : Xa0.p);
            k_copy<<<g, 256, 0, cx.st>>>(mO(), Y.p, Ya.p);
            CPD_CUDA(cudaGetLastError());
            cx.launches += 2;
        }
        run_active = false;
    }

    void fill_result(cpd_result* r, int kind, double wall)
    {
        const Ctl h = *cx.h_ctl;   // state at termination
        double o[8];
        eval_score(cx, Xp(cur_par), Y.p, obj_of(kind), bounds_of(kind), h.nb, h.nc, o, sense_of(kind));
        r->status = h.status;
        r->returned_average = h.returned_average;
        r->iterations = (h.status == ST_RUNNING) ? h.k : h.iterations;
        r->restarts = h.restarts;
        r->pobj = o[2];
        r->dobj = o[3];
        r->gap = std::fabs(o[2] - o[3]);
        r->rp_norm = o[0];
        r->rd_norm = o[1];
        r->score = o[7];
        r->step_size = h.eta;
        r->primal_weight = h.omega;
        r->wall_s = wall;
    }

    void solve(cpd_result* out)
    {
        const auto t0 = std::chrono::steady_clock::now();
        RunCfg rc;
        rc.kind = 0;
        rc.mode = MODE_FULL;
        rc.max_iters = prm.max_iters;
        rc.xs = Xp(cur_par);
        rc.ys = Y.p;
        rc.power = !(prm.step_size > 0.0);
        rc.eta = prm.step_size;
        rc.omega_in = prm.primal_weight;
        begin(rc);
        eta_phase1 = cx.h_ctl->eta;
        eta_known = true;
        advance(prm.max_iters, prm.time_limit_s);
        commit();
        cx.sync();
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (out) fill_result(out, 0, wall);
    }

    void step(int64_t k)
    {
        if (!run_active || run_kind != 0) {
            RunCfg rc;
            rc.kind = 0;
            rc.mode = MODE_NONE;
            rc.max_iters = INT64_MAX;
            rc.xs = Xp(cur_par);
            rc.ys = Y.p;
            rc.power = !(prm.step_size > 0.0);
            rc.eta = prm.step_size;
            rc.omega_in = prm.primal_weight;
            begin(rc);
            run_k_base = 0;
        }
        advance(cx.h_ctl->k + k, 0.0);
    }

    void corner_push(const cpd_corner_params& cp, cpd_result* out, cpd_stats* before, cpd_stats* after)
    {
        const auto t0 = std::chrono::steady_clock::now();
        if (run_active) commit();
        const int32_t n = nO(), m = mO();
        corner_eps = cp.eps_abs;
        const int g = std::min<int64_t>(cx.grid_elem, ((int64_t)std::max(n, m) + 255) / 256 + 1);
        // phase-1 solution (x*, y*): x* stays in X[cur_par]; y* saved in Ystar
        k_copy<<<g, 256, 0, cx.st>>>(m, Ystar.p, Y.p);
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
        const double* obj = nullptr;
        if (cp.obj) {
            if (n > 0)
                CPD_CUDA(cudaMemcpyAsync(objd.p, cp.obj + P->gofs[1], sizeof(double) * n,
                                         cp.obj_mem == CPD_DEVICE ? cudaMemcpyDeviceToDevice
                                                                  : cudaMemcpyHostToDevice,
                                         cx.st));
            if (P->cperm.p) {   // user column order -> internal
                ensure_tmp();
                CPD_CUDA(cudaMemcpyAsync(TX.p, objd.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, cx.st));
                perm_cols(objd.p, TX.p, 0);
            }
            obj = objd.p;
        }
        // Algorithm 1 line 2: z*, bound map, objective
        {
            AuxScope aux(cx);
            Reps rp(P, RV.p);
            Ctl h{};
            h.K = 1;
            cx.push_ctl(h);
            EpiCorner ec{P->c_own(), Xp(cur_par), P->bounds_own(), Z.p, lhat.p, uhat.p, chat.p, obj, cp.eps_abs,
                         cp.obj_scale, cp.seed, P->gofs[1]};
            ec.jmap = P->cperm.p;   // Uniform objective by user column
            if (P->scaled) {   // bound map on z = z^/s; objective s * obj; model bounds also in the original space
                if (!LHo.p) {
                    LHo.alloc(n);
                    UHo.alloc(n);
                }
                ec.w = P->w_n();
                ec.sx = P->s_n();
                ec.lho = LHo.p;
                ec.uho = UHo.p;
                ec.ob = P->bounds_orig();
            }
            pass<1>(cx, 1, fixed(rp.view(cx, 0, Ystar.p)), none(), ec, always());
            rows_eq = 0;
            if (P->has_sense) {   // inequality rows with |y*_i| > eps_abs become '='
                if (!shat.p) shat.alloc(std::max(m, 1));
                OpSense os{P->sense_own(), Ystar.p, P->scaled ? P->sr.p : nullptr, shat.p, cp.eps_abs};
                elem(cx, m, os, always(), true);
            }
            cx.pull_ctl();
            fix_lb = (int64_t)cx.h_ctl->out[0];
            fix_ub = (int64_t)cx.h_ctl->out[1];
            if (P->has_sense) rows_eq = (int64_t)cx.h_ctl->out[2];
        }
        have_corner = true;
        if (before) {
            eval_stats(cx, true, Xp(cur_par), Z.p, lh_orig(), uh_orig(), cp.eps_abs, cp.candidate_floor, fix_lb,
                       fix_ub, before);
            before->rows_eq = rows_eq;
        }
        if (!eta_known) {
            // no phase 1 on this solver: step size as phase 1 would have chosen it
            if (prm.step_size > 0.0) eta_phase1 = prm.step_size;
            else eta_phase1 = prm.step_scale / power_sigma(cx, prm.power_iters, prm.seed, 1.0, SN.p, SM.p);
            eta_known = true;
        }
        RunCfg rc;
        rc.kind = 1;
        rc.mode = MODE_PRIMAL_ONLY;
        rc.max_iters = cp.max_iters;
        rc.min_iters = cp.min_iters;
        rc.xs = Xp(cur_par);
        rc.ys = nullptr;   // Algorithm 1 line 3: start from (x, 0)
        rc.power = false;
        rc.eta = eta_phase1;
        rc.omega_in = 0.0;   // fresh primal weight from ||c^|| / ||b|| (S-8)
        rc.traj = cp.traj_every > 0 ? 1 : 0;
        begin(rc);
        advance(cp.max_iters, cp.time_limit_s);
        commit();
        cx.sync();
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (out) fill_result(out, 1, wall);
        // y, z returned are phase 1's
        k_copy<<<g, 256, 0, cx.st>>>(m, Y.p, Ystar.p);
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
        if (after) {
            eval_stats(cx, true, Xp(cur_par), Z.p, lh_orig(), uh_orig(), cp.eps_abs, cp.candidate_floor, fix_lb,
                       fix_ub, after);
            after->rows_eq = rows_eq;
        }
    }

    // NEXT-4 dual corner push (readings D-1..D-3): PDHG on (A, b, c, lhat_D, uhat_D)
    // from the current (x, y), stopped at k >= min_iters once every dual violation is
    // <= eps_abs; returns (x, yhat, zhat) with x unchanged (phase 1's).
    void dual_corner_push(const cpd_corner_params& cp, cpd_result* out, cpd_stats* before, cpd_stats* after)
    {
        const auto t0 = std::chrono::steady_clock::now();
        if (run_active) commit();
        const int32_t n = nO(), m = mO();
        corner_eps = cp.eps_abs;
        if (!LHD.p) {
            LHD.alloc(std::max(n, 1));
            UHD.alloc(std::max(n, 1));
            XS.alloc(std::max(n, 1));
        }
        const int g = std::min<int64_t>(cx.grid_elem, ((int64_t)std::max(n, m) + 255) / 256 + 1);
        k_copy<<<g, 256, 0, cx.st>>>(n, XS.p, Xp(cur_par));   // the phase-1 x the push keeps
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
        if (before) {
            compute_z();
            eval_stats(cx, true, XS.p, Z.p, nullptr, nullptr, cp.eps_abs, cp.candidate_floor, 0, 0, before);
        }
        {   // D-1 bound map
            AuxScope aux(cx);
            Ctl h{};
            h.K = 1;
            cx.push_ctl(h);
            OpDualModel od{XS.p, P->bounds_own(), LHD.p, UHD.p, cp.eps_abs};
            elem(cx, n, od, always(), true);
            cx.pull_ctl();
            dual_counts[0] = (int64_t)cx.h_ctl->out[0];
            dual_counts[1] = (int64_t)cx.h_ctl->out[1];
            dual_counts[2] = (int64_t)cx.h_ctl->out[2];
        }
        if (!eta_known) {
            if (prm.step_size > 0.0) eta_phase1 = prm.step_size;
            else eta_phase1 = prm.step_scale / power_sigma(cx, prm.power_iters, prm.seed, 1.0, SN.p, SM.p);
            eta_known = true;
        }
        RunCfg rc;
        rc.kind = 2;
        rc.mode = MODE_DUAL_ONLY;
        rc.max_iters = cp.max_iters;
        rc.min_iters = cp.min_iters;
        rc.xs = XS.p;
        rc.ys = Y.p;   // from (x*, y*)
        rc.power = false;
        rc.eta = eta_phase1;
        rc.omega_in = 0.0;
        begin(rc);
        advance(cp.max_iters, cp.time_limit_s);
        commit();
        cx.sync();
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (out) fill_result(out, 2, wall);
        k_copy<<<g, 256, 0, cx.st>>>(n, Xp(cur_par), XS.p);   // x stays phase 1's
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
        if (after) {
            compute_z();
            eval_stats(cx, true, XS.p, Z.p, nullptr, nullptr, cp.eps_abs, cp.candidate_floor, 0, 0, after);
        }
        run_active = false;
    }
    int64_t dual_counts[3] = {0, 0, 0};

    // x: n-side vector, y: m-side vector, both GLOBAL length; each rank takes its part.
    void set_iterate(const double* x, const double* y, int mem)
    {
        const auto kind = mem == CPD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        if (nO() > 0) {
            if (x && P->cperm.p) {   // user column order -> internal
                ensure_tmp();
                CPD_CUDA(cudaMemcpyAsync(TX.p, x, sizeof(double) * nO(), kind, cx.st));
                perm_cols(X0.p, TX.p, 0);
            } else if (x) {
                CPD_CUDA(cudaMemcpyAsync(X0.p, x + P->gofs[1], sizeof(double) * nO(), kind, cx.st));
            } else {
                CPD_CUDA(cudaMemsetAsync(X0.p, 0, sizeof(double) * nO(), cx.st));
            }
        }
        if (mO() > 0) {
            if (y && P->hot) {   // user order -> internal row order
                ensure_tmp();
                CPD_CUDA(cudaMemcpyAsync(TY.p, y, sizeof(double) * mO(), kind, cx.st));
                perm_vec(Y.p, TY.p, 0);
            } else if (y) {
                CPD_CUDA(cudaMemcpyAsync(Y.p, y + P->gofs[0], sizeof(double) * mO(), kind, cx.st));
            } else {
                CPD_CUDA(cudaMemsetAsync(Y.p, 0, sizeof(double) * mO(), cx.st));
            }
        }
        if (P->scaled) {   // original-space input: x^ = x / s, y^ = y / r
            scale_vec(nO(), X0.p, X0.p, P->ss.p, 0);
            scale_vec(mO(), Y.p, Y.p, P->sr.p, 0);
        }
        cx.sync();
        cur_par = 0;
        run_active = false;
        have_corner = false;
        eta_known = false;
    }

    void ensure_tmp()
    {
        if (!TX.p) {
            TX.alloc(std::max(nO(), 1));
            TY.alloc(std::max(mO(), 1));
        }
        if (P->hot && !TY2.p) TY2.alloc(std::max(mO(), 1));
        if (P->cperm.p && !TX2.p) TX2.alloc(std::max(nO(), 1));
    }

    void perm_vec(double* dst, const double* src, int mode)
    {
        const int64_t N = mO();
        if (N <= 0) return;
        const int g = (int)std::min<int64_t>(cx.grid_elem, (N + 255) / 256);
        k_perm_vec<<<g, 256, 0, cx.st>>>(N, dst, src, P->rperm.p, mode);
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
    }

    // n-side vectors between the user's column order and the internal one (mode 0:
    // user -> internal, 1: internal -> user); no-op copy when there is no renumbering
    void perm_cols(double* dst, const double* src, int mode)
    {
        const int64_t N = nO();
        if (N <= 0) return;
        const int g = (int)std::min<int64_t>(cx.grid_elem, (N + 255) / 256);
        k_perm_vec<<<g, 256, 0, cx.st>>>(N, dst, src, P->cperm.p, mode);
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
    }

    void scale_vec(int64_t N, double* dst, const double* src, const double* d, int op)
    {
        if (N <= 0) return;
        const int g = (int)std::min<int64_t>(cx.grid_elem, (N + 255) / 256);
        k_scale_vec<<<g, 256, 0, cx.st>>>(N, dst, src, d, op);
        CPD_CUDA(cudaGetLastError());
        ++cx.launches;
    }

    void compute_z()
    {
        AuxScope aux(cx);
        Reps rp(P, RV.p);
        Ctl h{};
        h.K = 1;
        cx.push_ctl(h);
        EpiZ ez{P->c_own(), Z.p};
        pass<1>(cx, 1, fixed(rp.view(cx, 0, Y.p)), none(), ez, always());
        cx.sync();
    }

    // Full (global) vector of `side` from every rank's owned part.
    void gather_full(int side, const double* own, double* out, int mem)
    {
        const auto kind = mem == CPD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        if (P->world == 1 && P->split < 0) {
            CPD_CUDA(cudaMemcpyAsync(out, own, sizeof(double) * P->own_len[side], kind, cx.st));
            return;
        }
        int64_t Lmax = 1;
        for (int64_t l : P->rank_len[side]) Lmax = std::max(Lmax, l);
        DBuf<double> send(Lmax), all((size_t)Lmax * P->world);
        if (P->own_len[side] > 0)
            CPD_CUDA(cudaMemcpyAsync(send.p, own, sizeof(double) * P->own_len[side], cudaMemcpyDeviceToDevice,
                                     cx.st));
        cx.all_gather(send.p, all.p, Lmax);
        for (int q = 0; q < P->world; ++q)
            if (P->rank_len[side][q] > 0)
                CPD_CUDA(cudaMemcpyAsync(out + P->rank_gofs[side][q], all.p + (int64_t)q * Lmax,
                                         sizeof(double) * P->rank_len[side][q], kind, cx.st));
        cx.sync();
    }

    // Original-space iterate: x = s x^, y = r y^, z = z^ / s (scaled problems).
    void get_iterate(double* x, double* y, double* z, int mem)
    {
        if (z) compute_z();
        const double *xs = Xp(cur_par), *ys = Y.p, *zs = Z.p;
        if (P->scaled || P->hot || P->cperm.p) {
            ensure_tmp();
            if (x) {
                if (P->scaled) scale_vec(nO(), TX.p, xs, P->ss.p, 1), xs = TX.p;
                if (P->cperm.p) perm_cols(TX2.p, xs, 1), xs = TX2.p;   // internal -> user column order
                gather_full(1, xs, x, mem);
            }
            if (y) {
                if (P->scaled) scale_vec(mO(), TY.p, ys, P->sr.p, 1), ys = TY.p;
                if (P->hot) perm_vec(TY2.p, ys, 1), ys = TY2.p;   // internal -> user row order
                gather_full(0, ys, y, mem);
            }
            if (z) {
                cx.sync();   // TX, TX2 reused
                if (P->scaled) scale_vec(nO(), TX.p, zs, P->is.p, 1), zs = TX.p;
                if (P->cperm.p) perm_cols(TX2.p, zs, 1), zs = TX2.p;
                gather_full(1, zs, z, mem);
            }
            cx.sync();
            return;
        }
        if (x) gather_full(1, xs, x, mem);
        if (y) gather_full(0, ys, y, mem);
        if (z) gather_full(1, zs, z, mem);
        cx.sync();
    }

    double kernel_bytes(const std::string& name) const
    {
        // local (this rank's) algorithmic bytes: matrix block + owned vectors + gathered vector
        const double nnz = (double)P->nnz, nr = P->n, mr = P->m, n = nO(), m = mO();
        const bool corner = name.find(":corner") != std::string::npos || name.find(":dual") != std::string::npos;
        const std::string base = name.substr(0, name.find(':'));
        const double bnd = (corner || !P->uniform_bounds) ? 16.0 * n : 0.0;
        // short-row push: their entries are read again by K1 (12 B) and not by K2; K2
        // reads and zeroes acc (16 B per row)
        const double pz = P->push_on ? (double)P->push_nnz : 0.0;
        if (prm.method == 1) {
            // Halpern: K1 reads c, x, x_anchor, writes xh, x+ (40 B per column, as R-PDHG);
            // K2 reads b, y, Ax, y_anchor, Ax_anchor and writes y+, Ax+, yh, A xh (72 B per row);
            // the check is one A^T pass over yh reading c, xh; restart copies 3 n- and 6 m-vectors
            if (base == "primal_step_AT") return 12 * nnz + 4 * (nr + 1) + 8 * mr + 40 * n + bnd;
            if (base == "dual_step_A") return 12 * nnz + 4 * (mr + 1) + 8 * nr + 72 * m;
            if (base == "check_eval_AT") return 12 * nnz + 4 * (nr + 1) + 8 * mr + 16 * n + bnd;
            if (base == "restart_apply") return 24 * n + 48 * m;
            return -1.0;
        }
        // SURVEY §8(d) per-unit figures: one A^T y product + primal update, one A x+
        // product + dual update.  (Hot-row fusion forms part of the A x+ product inside
        // the primal step's stream — the dual step then reads plan_info fused_nnz entries
        // fewer; the figure stays the product's, and bench.py also reports the K1+K2 pair.)
        if (base == "primal_step_AT") return 12 * nnz + 4 * (nr + 1) + 8 * mr + 40 * n + bnd + 12 * pz;
        if (base == "dual_step_A")
            return 12 * (nnz - pz) + 4 * (mr + 1) + 8 * nr + 56 * m + (P->push_on ? 16.0 * mr : 0.0);
        if (base == "check_eval_AT")
            return 12 * nnz + 4 * (nr + 1) + (prm.restart ? 16 : 8) * mr + 32 * n + bnd + (corner ? 16 * n : 0);
        if (base == "check_eval_A") return 12 * nnz + 4 * (mr + 1) + 8 * nr + 40 * m;
        if (base == "restart_apply") return 32 * n + 48 * m;
        return -1.0;
    }
};
// ====================================================================== ABI
static thread_local std::string g_err;

static int fail(int code, const std::string& msg)
{
    g_err = msg;
    return code;
}

#define ABI_BEGIN try {
#define ABI_END                                                                 \
    }                                                                           \
    catch (const cpd::Error& e) { return fail(e.code, e.what()); }              \
    catch (const std::bad_alloc&) { return fail(CPD_E_NOMEM, "host allocation failed"); } \
    catch (const std::exception& e) { return fail(CPD_E_CUDA, e.what()); }      \
    catch (...) { return fail(CPD_E_CUDA, "unknown error"); }                   \
    return CPD_OK;

cpd_problem* cpd_problem_create_impl(int32_t m, int32_t n, int64_t nnz, const int32_t* Ap,
                                     const int32_t* Aj, const double* Ax, const int32_t* ATp,
                                     const int32_t* ATj, const double* ATx, const double* b,
                                     const double* c, const double* lb, const double* ub,
                                     int32_t mem, int32_t device);

cpd_problem* cpd_problem_create_dist_impl(int32_t rank, int32_t world, const char id[128], int32_t partition,
                                          int32_t m, int32_t n, int64_t nnz, const int32_t* ATp,
                                          const int32_t* ATj, const double* ATx, const double* b,
                                          const double* c, const double* lb, const double* ub, int32_t device);

extern "C" {

const char* cpd_last_error(void) { return g_err.c_str(); }

int cpd_problem_create_dist(int32_t rank, int32_t world, const char id[128], int32_t partition, int32_t m,
                            int32_t n, int64_t nnz, const int32_t* AT_rowptr, const int32_t* AT_col,
                            const double* AT_val, const double* b, const double* c, const double* lb,
                            const double* ub, int32_t device, cpd_problem** out)
{
    ABI_BEGIN
    if (!out) return fail(CPD_E_ARG, "out is NULL");
    *out = cpd_problem_create_dist_impl(rank, world, id, partition, m, n, nnz, AT_rowptr, AT_col, AT_val, b, c,
                                        lb, ub, device);
    ABI_END
}

int cpd_problem_set_senses(cpd_problem* p, const int8_t* sense, int32_t mem)
{
    ABI_BEGIN
    if (!p || !sense) return fail(CPD_E_ARG, "NULL argument");
    if (p->live_solvers.load() > 0)
        return fail(CPD_E_STATE, "set_senses after a solver was created on this problem (destroy it first)");
    // this rank's local rows of A: all m (single GPU, col-block) or rows R_p (row-block)
    const int64_t off = p->split == 1 ? p->gofs[0] : 0;
    std::vector<int8_t> h((size_t)p->m);
    if (mem == CPD_DEVICE) CPD_CUDA(cudaMemcpy(h.data(), sense + off, (size_t)p->m, cudaMemcpyDeviceToHost));
    else std::memcpy(h.data(), sense + off, (size_t)p->m);
    for (int64_t i = 0; i < p->m; ++i)
        if (h[i] < 0 || h[i] > 2) return fail(CPD_E_ARG, "row sense must be 0, 1 or 2 (row " + std::to_string(i + off) + ")");
    if (p->hot) {   // user -> internal row order
        std::vector<int8_t> t(h);
        for (int64_t k = 0; k < p->m; ++k) h[k] = t[p->h_rperm[k]];
    }
    CPD_CUDA(cudaSetDevice(p->device));
    p->sense.alloc(std::max<int32_t>(p->m, 1));
    CPD_CUDA(cudaMemcpy(p->sense.p, h.data(), (size_t)p->m, cudaMemcpyHostToDevice));
    p->has_sense = true;
    ABI_END
}

int cpd_problem_scale(cpd_problem* p, int32_t ruiz_iters, int32_t pock_chambolle)
{
    ABI_BEGIN
    if (!p || ruiz_iters < 0 || ruiz_iters > 1000) return fail(CPD_E_ARG, "bad argument");
    if (p->split >= 0) return fail(CPD_E_ARG, "scaling of distributed problems is not supported");
    if (p->scaled) return fail(CPD_E_STATE, "problem is already scaled");
    if (p->live_solvers.load() > 0)
        return fail(CPD_E_STATE, "scale after a solver was created on this problem (destroy it first)");
    CPD_CUDA(cudaSetDevice(p->device));
    cpd::scale_problem(p, ruiz_iters, pock_chambolle ? 1 : 0);
    ABI_END
}

int cpd_problem_get_scaling(const cpd_problem* p, double* r, double* s)
{
    ABI_BEGIN
    if (!p) return fail(CPD_E_ARG, "NULL problem");
    if (!p->scaled) return fail(CPD_E_STATE, "problem is not scaled");
    CPD_CUDA(cudaSetDevice(p->device));
    if (r) {
        CPD_CUDA(cudaMemcpy(r, p->sr.p, sizeof(double) * p->m, cudaMemcpyDeviceToHost));
        if (p->hot) {   // internal -> user row order
            std::vector<double> t(r, r + p->m);
            for (int64_t k = 0; k < p->m; ++k) r[p->h_rperm[k]] = t[k];
        }
    }
    if (s) {
        CPD_CUDA(cudaMemcpy(s, p->ss.p, sizeof(double) * p->n, cudaMemcpyDeviceToHost));
        if (p->cperm.p) {   // internal -> user column order
            std::vector<int32_t> cp((size_t)p->n);
            CPD_CUDA(cudaMemcpy(cp.data(), p->cperm.p, sizeof(int32_t) * p->n, cudaMemcpyDeviceToHost));
            std::vector<double> t(s, s + p->n);
            for (int64_t k = 0; k < p->n; ++k) s[cp[k]] = t[k];
        }
    }
    ABI_END
}

int cpd_problem_dist_info(const cpd_problem* p, int64_t info[10])
{
    ABI_BEGIN
    if (!p || !info) return fail(CPD_E_ARG, "NULL argument");
    info[0] = p->world;
    info[1] = p->rank;
    info[2] = p->split < 0 ? -1 : (p->split == 1 ? 0 : 1);   // partition
    info[3] = p->L;
    info[4] = p->own_len[0];
    info[5] = p->own_len[1];
    info[6] = p->gofs[0];
    info[7] = p->gofs[1];
    info[8] = p->m;
    info[9] = p->n;
    ABI_END
}
int cpd_version(void) { return CPD_VERSION; }

int cpd_problem_create(int32_t m, int32_t n, int64_t nnz, const int32_t* A_rowptr, const int32_t* A_col,
                       const double* A_val, const int32_t* AT_rowptr, const int32_t* AT_col,
                       const double* AT_val, const double* b, const double* c, const double* lb,
                       const double* ub, int32_t mem, int32_t device, cpd_problem** out)
{
    ABI_BEGIN
    if (!out) return fail(CPD_E_ARG, "out is NULL");
    *out = cpd_problem_create_impl(m, n, nnz, A_rowptr, A_col, A_val, AT_rowptr, AT_col, AT_val, b, c, lb,
                                   ub, mem, device);
    ABI_END
}

int cpd_problem_destroy(cpd_problem* p)
{
    ABI_BEGIN
    if (p) {
        if (p->live_solvers.load() > 0)   // their graphs and buffers point into the problem
            return fail(CPD_E_STATE, "problem still has live solvers (destroy them first)");
        cudaSetDevice(p->device);
        delete p;
        (void)cudaGetLastError();   // an error of the teardown is not the next call's error
    }
    ABI_END
}

int cpd_problem_info(const cpd_problem* p, int64_t info[8])
{
    ABI_BEGIN
    if (!p || !info) return fail(CPD_E_ARG, "NULL argument");
    info[0] = p->m_glob;
    info[1] = p->n_glob;
    info[2] = p->nnz;
    info[3] = p->A.plan.nlong;
    info[4] = p->AT.plan.nlong;
    info[5] = p->A.plan.nent;
    info[6] = p->AT.plan.nent;
    info[7] = p->uniform_bounds ? 1 : 0;
    ABI_END
}

int cpd_problem_plan_info(const cpd_problem* p, int64_t out[16])
{
    ABI_BEGIN
    if (!p || !out) return fail(CPD_E_ARG, "NULL argument");
    const cpd::Plan& pl = p->A.plan;
    out[0] = pl.warp;
    out[1] = pl.nheavy;
    out[2] = pl.nheavy > 0 ? pl.nhb : 0;
    out[3] = pl.nslab;
    out[4] = pl.short_on ? pl.short_nslab : 0;
    out[5] = pl.nlong;
    out[6] = pl.long_pieces;
    out[7] = pl.rows_entries;
    out[8] = p->AT.sell.on ? 1 : 0;
    out[9] = p->hot;
    out[10] = pl.warp ? 0 : pl.nent;
    out[11] = p->cperm.p ? 1 : 0;
    out[12] = cpd::fuse_ok(p) ? pl.hotd : 0;
    out[13] = cpd::fuse_ok(p) ? pl.hot_nnz : 0;   // entries of the fused rows (the dual step skips them)
    out[14] = out[15] = 0;
    ABI_END
}

void cpd_params_default(cpd_params* p)
{
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->eps_rel = 1e-4;
    p->eps_abs = 1e-6;
    p->max_iters = 100000;
    p->time_limit_s = 0.0;
    p->check_every = 64;
    p->step_scale = 0.9;
    p->step_size = 0.0;
    p->power_iters = 128;
    p->seed = 7;
    p->primal_weight = 0.0;
    p->restart = 1;
    p->beta_suff = 0.2;
    p->beta_nec = 0.8;
    p->beta_art = 0.36;
    p->theta = 0.5;
    p->use_graph = 1;
    p->profile = 0;
    p->method = 0;
    p->reflection = 1.0;
    p->pid = 0;
    p->kp = 0.99;
    p->ki = 0.01;
    p->kd = 0.0;
}

void cpd_corner_params_default(cpd_corner_params* p)
{
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->eps_abs = 1e-6;
    p->obj_scale = 1.0;
    p->seed = 1001;
    p->obj = nullptr;
    p->obj_mem = CPD_HOST;
    p->min_iters = 100;
    p->max_iters = 100000;
    p->time_limit_s = 0.0;
    p->traj_every = 64;
    p->candidate_floor = 100000;
}

int cpd_solver_create(const cpd_problem* p, const cpd_params* prm, cpd_solver** out)
{
    ABI_BEGIN
    if (!p || !out) return fail(CPD_E_ARG, "NULL argument");
    cpd_params d;
    cpd_params_default(&d);
    const cpd_params& pr = prm ? *prm : d;
    if (pr.check_every < 1 || pr.check_every > 1024) return fail(CPD_E_ARG, "check_every must be in [1, 1024]");
    if (!(pr.eps_rel > 0.0) || !(pr.step_scale > 0.0) || pr.power_iters < 1 || pr.max_iters < 0 ||
        pr.restart < 0 || pr.restart > 1 || pr.method < 0 || pr.method > 1 || !(pr.reflection >= 0.0) ||
        pr.pid < 0 || pr.pid > 1 || !std::isfinite(pr.kp) || !std::isfinite(pr.ki) || !std::isfinite(pr.kd))
        return fail(CPD_E_ARG, "invalid parameter");
    if (pr.method == 1 && p->split >= 0)
        return fail(CPD_E_ARG, "the Halpern method (method = 1) is single-GPU only");
    CPD_CUDA(cudaSetDevice(p->device));
    *out = new cpd_solver(p, pr);
    p->live_solvers.fetch_add(1);
    ABI_END
}

int cpd_solver_destroy(cpd_solver* s)
{
    ABI_BEGIN
    if (s) {
        cudaSetDevice(s->P->device);
        const cpd_problem* p = s->P;
        delete s;
        p->live_solvers.fetch_sub(1);
        (void)cudaGetLastError();
    }
    ABI_END
}

int cpd_solve(cpd_solver* s, cpd_result* out)
{
    ABI_BEGIN
    if (!s) return fail(CPD_E_ARG, "NULL solver");
    CPD_CUDA(cudaSetDevice(s->P->device));
    s->solve(out);
    ABI_END
}

int cpd_corner_push(cpd_solver* s, const cpd_corner_params* cp, cpd_result* out, cpd_stats* before,
                    cpd_stats* after)
{
    ABI_BEGIN
    if (!s) return fail(CPD_E_ARG, "NULL solver");
    cpd_corner_params d;
    cpd_corner_params_default(&d);
    const cpd_corner_params& c = cp ? *cp : d;
    if (!(c.eps_abs >= 0.0) || c.min_iters < 0 || c.max_iters < 0) return fail(CPD_E_ARG, "invalid corner parameter");
    CPD_CUDA(cudaSetDevice(s->P->device));
    s->corner_push(c, out, before, after);
    ABI_END
}

int cpd_dual_corner_push(cpd_solver* s, const cpd_corner_params* cp, cpd_result* out, cpd_stats* before,
                         cpd_stats* after)
{
    ABI_BEGIN
    if (!s) return fail(CPD_E_ARG, "NULL solver");
    cpd_corner_params d;
    cpd_corner_params_default(&d);
    const cpd_corner_params& c = cp ? *cp : d;
    if (!(c.eps_abs >= 0.0) || c.min_iters < 0 || c.max_iters < 0) return fail(CPD_E_ARG, "invalid corner parameter");
    if (s->P->split >= 0 || s->P->scaled)
        return fail(CPD_E_STATE, "the dual corner push needs an unscaled single-GPU problem");
    CPD_CUDA(cudaSetDevice(s->P->device));
    s->dual_corner_push(c, out, before, after);
    ABI_END
}

int cpd_corner_decide(const cpd_stats* st, int32_t m, int32_t* primal, int32_t* dual)
{
    if (!st || !primal || !dual || m < 0) return fail(CPD_E_ARG, "NULL argument");
    *primal = st->is_candidate ? 1 : 0;
    *dual = (st->est_dual_pushes > 0 && std::min<int64_t>(m, st->off_bound) > st->zero_rc) ? 1 : 0;
    return CPD_OK;
}

int cpd_step(cpd_solver* s, int64_t k)
{
    ABI_BEGIN
    if (!s || k < 0) return fail(CPD_E_ARG, "NULL solver or k < 0");
    CPD_CUDA(cudaSetDevice(s->P->device));
    s->step(k);
    ABI_END
}

int cpd_get_iterate(const cpd_solver* s, double* x, double* y, double* z, int32_t mem)
{
    ABI_BEGIN
    if (!s) return fail(CPD_E_ARG, "NULL solver");
    CPD_CUDA(cudaSetDevice(s->P->device));
    const_cast<cpd_solver*>(s)->get_iterate(x, y, z, mem);
    ABI_END
}

int cpd_set_iterate(cpd_solver* s, const double* x, const double* y, int32_t mem)
{
    ABI_BEGIN
    if (!s) return fail(CPD_E_ARG, "NULL solver");
    CPD_CUDA(cudaSetDevice(s->P->device));
    s->set_iterate(x, y, mem);
    ABI_END
}

int cpd_get_stats(const cpd_solver* cs, int64_t candidate_floor, cpd_stats* out)
{
    ABI_BEGIN
    if (!cs || !out) return fail(CPD_E_ARG, "NULL argument");
    auto* s = const_cast<cpd_solver*>(cs);
    CPD_CUDA(cudaSetDevice(s->P->device));
    s->compute_z();
    eval_stats(s->cx, true, s->Xp(s->cur_par), s->Z.p, s->have_corner ? s->lh_orig() : nullptr,
               s->have_corner ? s->uh_orig() : nullptr, s->have_corner ? s->corner_eps : s->prm.eps_abs,
               candidate_floor, s->have_corner ? s->fix_lb : 0, s->have_corner ? s->fix_ub : 0, out);
    out->rows_eq = s->have_corner ? s->rows_eq : 0;
    ABI_END
}

int cpd_get_trajectory(const cpd_solver* s, int64_t* k, int64_t* off_bound, double* rp, int64_t cap,
                       int64_t* len)
{
    ABI_BEGIN
    if (!s || !len) return fail(CPD_E_ARG, "NULL argument");
    CPD_CUDA(cudaSetDevice(s->P->device));
    Ctl h;
    CPD_CUDA(cudaMemcpy(&h, s->cx.ctl_main.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
    const int64_t L = std::min<int64_t>(h.traj_len, std::max<int64_t>(cap, 0));
    if (L > 0) {
        if (k) CPD_CUDA(cudaMemcpy(k, s->trk.p, sizeof(int64_t) * L, cudaMemcpyDeviceToHost));
        if (off_bound) CPD_CUDA(cudaMemcpy(off_bound, s->troff.p, sizeof(int64_t) * L, cudaMemcpyDeviceToHost));
        if (rp) CPD_CUDA(cudaMemcpy(rp, s->trrp.p, sizeof(double) * L, cudaMemcpyDeviceToHost));
    }
    *len = h.traj_len;
    ABI_END
}

int cpd_power_sigma(const cpd_problem* p, int32_t iters, uint64_t seed, double* sigma)
{
    ABI_BEGIN
    if (!p || !sigma || iters < 1) return fail(CPD_E_ARG, "bad argument");
    CPD_CUDA(cudaSetDevice(p->device));
    Ctx cx(p);
    DBuf<double> v(std::max(p->own_len[1], 1)), w(std::max(p->own_len[0], 1));
    *sigma = power_sigma(cx, iters, seed, 1.0, v.p, w.p);
    ABI_END
}

int cpd_problem_score(const cpd_problem* p, const double* x, const double* y, int32_t mem, double out[8])
{
    ABI_BEGIN
    if (!p || !x || !y || !out) return fail(CPD_E_ARG, "NULL argument");
    CPD_CUDA(cudaSetDevice(p->device));
    Ctx cx(p);
    // owned parts of the (global) x and y
    const int64_t nO = p->own_len[1], mO = p->own_len[0];
    DBuf<double> dx(std::max<int64_t>(nO, 1)), dy(std::max<int64_t>(mO, 1));
    const auto kind = mem == CPD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    // every copy on the context's (non-blocking) stream, ordered with its kernels
    if (nO) CPD_CUDA(cudaMemcpyAsync(dx.p, x + p->gofs[1], sizeof(double) * nO, kind, cx.st));
    if (mO) CPD_CUDA(cudaMemcpyAsync(dy.p, y + p->gofs[0], sizeof(double) * mO, kind, cx.st));
    cx.sync();
    if (p->cperm.p && nO) {   // user column order -> internal
        DBuf<double> t(nO);
        CPD_CUDA(cudaMemcpyAsync(t.p, dx.p, sizeof(double) * nO, cudaMemcpyDeviceToDevice, cx.st));
        k_perm_vec<<<(int)std::min<int64_t>(4096, (nO + 255) / 256), 256, 0, cx.st>>>(nO, dx.p, t.p, p->cperm.p, 0);
        CPD_CUDA(cudaGetLastError());
        cx.sync();
    }
    if (p->hot && mO) {   // user row order -> internal
        DBuf<double> t(mO);
        CPD_CUDA(cudaMemcpyAsync(t.p, dy.p, sizeof(double) * mO, cudaMemcpyDeviceToDevice, cx.st));
        k_perm_vec<<<(int)std::min<int64_t>(4096, (mO + 255) / 256), 256, 0, cx.st>>>(mO, dy.p, t.p, p->rperm.p, 0);
        CPD_CUDA(cudaGetLastError());
        cx.sync();
    }
    if (p->scaled) {   // original-space point -> scaled
        if (nO) k_scale_vec<<<(int)std::min<int64_t>(4096, (nO + 255) / 256), 256, 0, cx.st>>>(nO, dx.p, dx.p, p->ss.p, 0);
        if (mO) k_scale_vec<<<(int)std::min<int64_t>(4096, (mO + 255) / 256), 256, 0, cx.st>>>(mO, dy.p, dy.p, p->sr.p, 0);
        CPD_CUDA(cudaGetLastError());
        cx.sync();
    }
    double nb, nc;
    eval_norms(cx, p->b_own(), p->c_own(), &nb, &nc);
    eval_score(cx, dx.p, dy.p, p->c_own(), p->bounds_own(), nb, nc, out, p->sense_own());
    ABI_END
}

int cpd_compute_stats(const cpd_problem* p, const double* x, const double* z, const double* lhat,
                      const double* uhat, double eps_abs, int64_t candidate_floor, int32_t mem,
                      cpd_stats* out)
{
    ABI_BEGIN
    if (!p || !x || !out || ((lhat == nullptr) != (uhat == nullptr))) return fail(CPD_E_ARG, "bad argument");
    CPD_CUDA(cudaSetDevice(p->device));
    Ctx cx(p);
    // owned parts of the (global) n-vectors
    DBuf<double> b[4];
    const double* src[4] = {x, z, lhat, uhat};
    const double* dev[4] = {nullptr, nullptr, nullptr, nullptr};
    const int64_t nO = p->own_len[1];
    const auto kind = mem == CPD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (int i = 0; i < 4; ++i)
        if (src[i]) {
            b[i].alloc(std::max<int64_t>(nO, 1));
            if (nO) CPD_CUDA(cudaMemcpyAsync(b[i].p, src[i] + p->gofs[1], sizeof(double) * nO, kind, cx.st));
            if (p->cperm.p && nO) {   // user column order -> internal
                DBuf<double> t(nO);
                CPD_CUDA(cudaMemcpyAsync(t.p, b[i].p, sizeof(double) * nO, cudaMemcpyDeviceToDevice, cx.st));
                k_perm_vec<<<(int)std::min<int64_t>(4096, (nO + 255) / 256), 256, 0, cx.st>>>(nO, b[i].p, t.p,
                                                                                            p->cperm.p, 0);
                CPD_CUDA(cudaGetLastError());
                cx.sync();
            }
            dev[i] = b[i].p;
        }
    cx.sync();
    eval_stats(cx, false, dev[0], dev[1], dev[2], dev[3], eps_abs, candidate_floor, 0, 0, out);
    ABI_END
}

int cpd_get_kernel_times(cpd_solver* s, const char** names, double* ms, int64_t* launches, int32_t cap,
                         int32_t* len, int32_t reset)
{
    ABI_BEGIN
    if (!s || !len) return fail(CPD_E_ARG, "NULL argument");
    int32_t L = 0;
    for (int kind = 0; kind < 3; ++kind)
        for (int k = 0; k < KT_N; ++k) {
            if (L < cap) {
                if (names) names[L] = KT_NAMES[kind][k];
                if (ms) ms[L] = s->kt_ms[kind][k];
                if (launches) launches[L] = s->kt_n[kind][k];
            }
            ++L;
        }
    *len = std::min(L, std::max(cap, 0));
    if (reset) {
        std::memset(s->kt_ms, 0, sizeof(s->kt_ms));
        std::memset(s->kt_n, 0, sizeof(s->kt_n));
    }
    ABI_END
}

int cpd_solver_counters(const cpd_solver* s, int64_t out[4])
{
    ABI_BEGIN
    if (!s || !out) return fail(CPD_E_ARG, "NULL argument");
    out[0] = s->cx.launches;
    out[1] = s->graph_launches;
    out[2] = s->graph_kernels[0];
    out[3] = s->graph_kernels[1];
    ABI_END
}

int cpd_memcache_info(int32_t device, int64_t* cached_bytes)
{
    ABI_BEGIN
    int ndev = 0;
    CPD_CUDA(cudaGetDeviceCount(&ndev));
    if (!cached_bytes || device < 0 || device >= ndev) return fail(CPD_E_ARG, "bad device or NULL argument");
    CPD_CUDA(cudaSetDevice(device));
    *cached_bytes = (int64_t)cpd::dev_cached_bytes();
    ABI_END
}

int cpd_memcache_release(int32_t device)
{
    ABI_BEGIN
    int ndev = 0;
    CPD_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(CPD_E_ARG, "bad device ordinal");
    CPD_CUDA(cudaSetDevice(device));
    cpd::dev_trim();
    ABI_END
}

int cpd_kernel_bytes(const cpd_solver* s, const char* name, double* bytes)
{
    ABI_BEGIN
    if (!s || !name || !bytes) return fail(CPD_E_ARG, "NULL argument");
    *bytes = s->kernel_bytes(name);
    if (*bytes < 0) return fail(CPD_E_ARG, std::string("unknown kernel ") + name);
    ABI_END
}

}  // extern "C"
