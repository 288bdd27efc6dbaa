// problem.cu — cpd_problem: device copies, device-side validation, device
// transpose (stable radix sort by column), uniform-bound detection, SpMV plans.
// The problem statement is P:64-92 (A m x n, b, c, bounds handled implicitly).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <functional>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

namespace cpd {

// ------------------------------------------------------------------ plans
// Column slab width for long-row pieces: 4M columns = 32 MB of the gathered fp64
// vector, so the slab being swept stays resident in the 126 MB L2.
#ifndef CPD_SLAB_COLS
#define CPD_SLAB_COLS (4 << 20)
#endif
constexpr int64_t SLAB_COLS = CPD_SLAB_COLS;
// Runtime overrides of the plan thresholds (env CPD_SLAB_COLS, CPD_HEAVY_MIN), read at
// plan build: the parity tests use them to route reduced LPs through the engine paths
// that only the full-size configs reach by default (multi-slab long pieces, k_dense).
static int64_t env_i64(const char* name, int64_t dflt)
{
    const char* e = getenv(name);
    return (e && *e) ? std::max<int64_t>(1, atoll(e)) : dflt;
}
static int64_t slab_cols() { return env_i64("CPD_SLAB_COLS", SLAB_COLS); }
static int64_t heavy_min() { return env_i64("CPD_HEAVY_MIN", HEAVY_MIN); }
#ifndef CPD_SLAB_MIN
#define CPD_SLAB_MIN 0   // long rows shorter than this are not cut at column-slab boundaries
#endif
#ifndef CPD_HOTD_DEFAULT
#define CPD_HOTD_DEFAULT 6   // hot-row fusion: the longest rows whose dual-step product the primal step forms
#endif
#ifndef CPD_SHORT_SLABS
#define CPD_SHORT_SLABS 2   // short rows (CPD_SHORT=1): column slabs of n / 2 (80 MB of C5's x each)
#endif

// pos[l * nb + s - 1] = first position q of long row l with col[q] >= s * SLAB_COLS.
__global__ void k_slab_pos(int32_t nl, int32_t nb, const int32_t* lrows, const int32_t* p,
                           const int32_t* col, int32_t* pos, int64_t width = SLAB_COLS, int64_t first = 1)
{
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)nl * nb;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int32_t l = (int32_t)(idx / nb);
        const int64_t target = (idx % nb + first) * width;
        const int32_t r = lrows[l];
        int32_t lo = p[r], hi = p[r + 1];
        while (lo < hi) {
            const int32_t mid = lo + (hi - lo) / 2;
            if ((int64_t)col[mid] < target) lo = mid + 1; else hi = mid;
        }
        pos[idx] = lo;
    }
}

// col16[q] = col[q] mod HB for the entries q of heavy row rows[blockIdx.x]
// (grid: blockIdx.y = heavy row, blockIdx.x strides its entries: the Zipf head's rows
// hold millions of entries each)
__global__ void k_col16(const int32_t* rows, const int32_t* p, const int32_t* col, uint16_t* col16)
{
    const int32_t r = rows[blockIdx.y];
    for (int64_t q = p[r] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < p[r + 1];
         q += (int64_t)gridDim.x * blockDim.x)
        col16[q] = (uint16_t)(col[q] & (HB - 1));
}

// Short rows (<= long_min entries) split by column slab: cnt[s * rows + r] = entries of
// row r in slab s (0 for long rows); a row's columns are ascending, so the slab
// boundaries are found by binary search.
__global__ void k_short_count(int32_t rows, int32_t nslab, int64_t long_min, const int32_t* p, const int32_t* col,
                              int32_t* cnt, int64_t width)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = p[r], b = p[r + 1];
        const bool sh = b - a <= long_min;
        int32_t prev = a;
        for (int32_t s = 0; s < nslab; ++s) {
            int32_t end = b;
            if (s + 1 < nslab) {   // first q in [prev, b) with col[q] >= (s + 1) * width
                int32_t lo = prev, hi = b;
                const int64_t key = (int64_t)(s + 1) * width;
                while (lo < hi) {
                    const int32_t mid = lo + (hi - lo) / 2;
                    if (col[mid] < key) lo = mid + 1; else hi = mid;
                }
                end = lo;
            }
            cnt[(int64_t)s * rows + r] = sh ? end - prev : 0;
            prev = end;
        }
    }
}

// slab pointers from the slab-major exclusive scan: sp[s][r] = flat[s * rows + r],
// sp[s][rows] = start of slab s + 1 (the total for the last slab)
__global__ void k_short_ptr(int32_t rows, int32_t nslab, const int32_t* flat, const int32_t* cnt, int32_t* sp)
{
    const int64_t N = (int64_t)nslab * (rows + 1);
    const int64_t tot = (int64_t)nslab * rows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / (rows + 1), r = i % (rows + 1);
        sp[i] = r < rows ? flat[s * rows + r] : (s + 1 < nslab ? flat[(s + 1) * rows] : flat[tot - 1] + cnt[tot - 1]);
    }
}

// the rows items re-based per slab: {a, b, sp[s][a], sp[s][b]} (k_csrw slab mode
// reads the item's entry range directly, one dependent load less per item)
__global__ void k_short_ents(int32_t ni, int32_t nslab, int32_t rows, const PlanEntry* ent, const int32_t* sp,
                             PlanEntry* out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)nslab * ni;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / ni;
        const PlanEntry E = ent[i % ni];
        const int32_t* p = sp + s * (rows + 1);
        out[i] = PlanEntry{E.a, E.b, p[E.a], p[E.b]};
    }
}

// entries copied slab-major (row order, then column order inside each slab): a warp
// per row, lane-strided (coalesced) over the row's entries
__global__ void k_short_fill(int32_t rows, int32_t nslab, int64_t long_min, const int32_t* p, const int32_t* col,
                             const double* val, const int32_t* sp, int32_t* scol, double* sval, int64_t width)
{
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t a = p[r], b = p[r + 1];
        if (b - a > long_min) continue;
        for (int32_t q = a + lane; q < b; q += 32) {
            const int32_t c = col[q];
            const int64_t s64 = c / width;
            const int32_t s = s64 < nslab - 1 ? (int32_t)s64 : nslab - 1;
            int32_t off = 0;   // entries of this row in slabs before s
            for (int32_t t = 0; t < s; ++t) off += sp[(int64_t)t * (rows + 1) + r + 1] - sp[(int64_t)t * (rows + 1) + r];
            const int32_t d = sp[(int64_t)s * (rows + 1) + r] + (q - a - off);
            scol[d] = c;
            sval[d] = val[q];
        }
    }
}

// Rows entries: maximal runs of consecutive rows with <= CAP nonzeros and <= RMAX
// rows.  A row with more than SINGLE_MIN nonzeros is LONG: cut at column-slab
// boundaries and into CAP pieces, pieces ordered slab-major after all rows entries
// (while the CTAs sweep one slab, that slab of the gathered vector stays in L2);
// k_finish sums its pieces and applies its epilogue.
void build_plan(int32_t rows, int32_t cols, const std::vector<int32_t>& rp, const int32_t* d_p,
                const int32_t* d_col, const double* d_val, Plan& plan, bool warp, int32_t hotd_req)
{
    // TMA plan: <= RMAX rows / CAP nnz per entry, rows > SINGLE_MIN long, CAP pieces.
    // warp plan (k_csrw): <= 32 rows / WCAP_ROWS nnz per item, rows > WLONG long, WCAP_LONG pieces.
    const int64_t cap_rows = warp ? WCAP_ROWS : CAP, max_rows = warp ? 32 : RMAX;
    const int64_t long_min = warp ? WLONG : SINGLE_MIN, piece = warp ? WCAP_LONG : CAP;
    plan.warp = warp ? 1 : 0;
    std::vector<PlanEntry> ent;
    std::vector<int32_t> lrows;
    int64_t nrows_e = 0;
    int32_t r0 = 0;
    int64_t cur = 0;
    auto flush = [&](int32_t r1) {
        if (r1 > r0) {
            ent.push_back(PlanEntry{r0, r1, rp[r0], rp[r1]});
            ++nrows_e;
        }
    };
    for (int32_t r = 0; r < rows; ++r) {
        const int64_t len = (int64_t)rp[r + 1] - rp[r];
        if (len > long_min) {
            // long row: pieces (any length > SINGLE_MIN; k_finish applies its epilogue)
            flush(r);
            lrows.push_back(r);
            r0 = r + 1;
            cur = 0;
            continue;
        }
        if (cur + len > cap_rows || (r - r0) >= max_rows) {
            flush(r);
            r0 = r;
            cur = 0;
        }
        cur += len;
    }
    flush(rows);
    // long rows: slab boundaries (device binary search), pieces
    const int32_t nl = (int32_t)lrows.size();
    const int64_t SLABW = slab_cols();
    const int32_t nslab = (int32_t)std::max<int64_t>(1, ((int64_t)cols + SLABW - 1) / SLABW);
    const int32_t nb = nslab - 1;
    std::vector<int32_t> pos((size_t)nl * std::max(nb, 0));
    if (nl > 0 && nb > 0) {
        DBuf<int32_t> dl(nl), dpos((size_t)nl * nb);
        CPD_CUDA(cudaMemcpy(dl.p, lrows.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice));
        const int64_t tot = (int64_t)nl * nb;
        k_slab_pos<<<(int)std::min<int64_t>((tot + 255) / 256, 4096), 256>>>(nl, nb, dl.p, d_p, d_col, dpos.p,
                                                                               SLABW);
        CPD_CUDA(cudaGetLastError());
        CPD_CUDA(cudaMemcpy(pos.data(), dpos.p, sizeof(int32_t) * tot, cudaMemcpyDeviceToHost));
    }
    // heavy rows (warp plan): >= HEAVY_MIN nonzeros; their product runs by dense
    // column blocks of HB columns (k_dense), one partial slot per block
    const int32_t nhb = (int32_t)(((int64_t)cols + HB - 1) / HB);
    std::vector<int32_t> heavy_l;
    std::vector<char> is_heavy(nl, 0);
    if (warp && (cols >= 2 * HB || getenv("CPD_HEAVY_MIN")))   // (env: tests force k_dense on small n)
        for (int32_t l = 0; l < nl; ++l)
            if ((int64_t)rp[lrows[l] + 1] - rp[lrows[l]] >= heavy_min()) {
                heavy_l.push_back(l);
                is_heavy[l] = 1;
            }
    // pieces[s] = list of (long id, q0, q1) in row order
    std::vector<std::vector<PlanEntry>> by_slab(nslab);
    for (int32_t l = 0; l < nl; ++l) {
        if (is_heavy[l]) continue;
        const int32_t r = lrows[l];
        int32_t a = rp[r];
        if ((int64_t)rp[r + 1] - rp[r] < CPD_SLAB_MIN) {
            // too short to profit from slab cuts (they would leave tiny pieces): plain
            // pieces, listed with the slab of the row's middle entry
            const int32_t mid = std::min<int32_t>(nslab - 1, nb > 0 ? (int32_t)(std::lower_bound(
                pos.begin() + (size_t)l * nb, pos.begin() + (size_t)(l + 1) * nb, (a + rp[r + 1]) / 2 + 1) -
                (pos.begin() + (size_t)l * nb)) : 0);
            for (int32_t q = a; q < rp[r + 1]; q += (int32_t)piece)
                by_slab[mid].push_back(PlanEntry{r, -1 - l, q, (int32_t)std::min<int64_t>((int64_t)q + piece, rp[r + 1])});
            continue;
        }
        for (int32_t s = 0; s < nslab; ++s) {
            const int32_t b = (s + 1 < nslab) ? pos[(size_t)l * nb + s] : rp[r + 1];
            for (int32_t q = a; q < b; q += (int32_t)piece)
                by_slab[s].push_back(PlanEntry{r, -1 - l, q, (int32_t)std::min<int64_t>((int64_t)q + piece, b)});
            a = b;
        }
    }
    // slots: the pieces of long row l occupy [lptr[l], lptr[l+1]) in column order
    std::vector<int32_t> lptr(nl + 1, 0);
    for (int32_t s = 0; s < nslab; ++s)
        for (const PlanEntry& E : by_slab[s]) lptr[-1 - E.b + 1]++;
    // heavy rows: block boundary positions (device binary search), then items of
    // <= DCHUNK entries grouped by column block; a heavy row's slots are its items
    // in column order
    const int32_t nh = (int32_t)heavy_l.size();
    std::vector<int32_t> hpos((size_t)nh * (nhb + 1));
    if (nh > 0) {
        std::vector<int32_t> hr(nh);
        for (int32_t h = 0; h < nh; ++h) hr[h] = lrows[heavy_l[h]];
        DBuf<int32_t> dhr(nh), dpos((size_t)nh * (nhb + 1));
        CPD_CUDA(cudaMemcpy(dhr.p, hr.data(), sizeof(int32_t) * nh, cudaMemcpyHostToDevice));
        const int64_t tot = (int64_t)nh * (nhb + 1);
        k_slab_pos<<<(int)std::min<int64_t>((tot + 255) / 256, 4096), 256>>>(nh, nhb + 1, dhr.p, d_p, d_col,
                                                                            dpos.p, HB, 0);
        CPD_CUDA(cudaGetLastError());
        CPD_CUDA(cudaMemcpy(hpos.data(), dpos.p, sizeof(int32_t) * tot, cudaMemcpyDeviceToHost));
        for (int32_t h = 0; h < nh; ++h) {
            int64_t cnt = 0;
            for (int32_t b = 0; b < nhb; ++b) {
                const int64_t len = (int64_t)hpos[(size_t)h * (nhb + 1) + b + 1] - hpos[(size_t)h * (nhb + 1) + b];
                cnt += (len + DCHUNK - 1) / DCHUNK;   // one partial slot per item
            }
            lptr[heavy_l[h] + 1] = (int32_t)cnt;
        }
    }
    for (int32_t l = 0; l < nl; ++l) lptr[l + 1] += lptr[l];
    plan.nheavy = nh;
    plan.nhb = nhb;
    if (nh > 0) {
        std::vector<std::vector<PlanEntry>> dl(nhb);
        for (int32_t h = 0; h < nh; ++h) {
            int32_t slot = lptr[heavy_l[h]];
            for (int32_t b = 0; b < nhb; ++b) {
                const int32_t q0 = hpos[(size_t)h * (nhb + 1) + b], q1 = hpos[(size_t)h * (nhb + 1) + b + 1];
                for (int32_t q = q0; q < q1; q += DCHUNK)
                    dl[b].push_back(PlanEntry{slot++, b, q, std::min(q + DCHUNK, q1)});
            }
        }
        std::vector<PlanEntry> dent;
        std::vector<int32_t> dptr(nhb + 1, 0);
        int32_t maxit = 1;
        for (int32_t b = 0; b < nhb; ++b) {
            dent.insert(dent.end(), dl[b].begin(), dl[b].end());
            dptr[b + 1] = (int32_t)dent.size();
            maxit = std::max<int32_t>(maxit, (int32_t)dl[b].size());
        }
        plan.dense_maxitems = maxit;
        // 16-bit column offsets of the heavy rows' entries (HB is a power of two <= 65536);
        // CPD_DENSE16=0 keeps the 32-bit column indices
        const char* d16 = getenv("CPD_DENSE16");
        if (!(d16 && d16[0] == '0') && (HB & (HB - 1)) == 0 && HB <= 65536) {
            plan.dense_col16.alloc((size_t)rp[rows]);
            std::vector<int32_t> hr(nh);
            for (int32_t h = 0; h < nh; ++h) hr[h] = lrows[heavy_l[h]];
            DBuf<int32_t> dhr2(nh);
            CPD_CUDA(cudaMemcpy(dhr2.p, hr.data(), sizeof(int32_t) * nh, cudaMemcpyHostToDevice));
            k_col16<<<dim3(64, std::max(1, nh)), 256>>>(dhr2.p, d_p, d_col, plan.dense_col16.p);
            CPD_CUDA(cudaGetLastError());
        }
        plan.dense_ent.alloc(std::max<size_t>(dent.size(), 1));
        plan.dense_ptr.alloc(nhb + 1);
        CPD_CUDA(cudaMemcpy(plan.dense_ent.p, dent.data(), sizeof(PlanEntry) * dent.size(), cudaMemcpyHostToDevice));
        CPD_CUDA(cudaMemcpy(plan.dense_ptr.p, dptr.data(), sizeof(int32_t) * (nhb + 1), cudaMemcpyHostToDevice));
        // hot-row fusion: rows 0..D-1 (the longest, heavy, long-row ids 0..D-1) take their
        // dual-step product from the primal step; the fused dual step's dense items skip them
        int32_t D = 0;
        while (D < hotd_req && D < nl && lrows[D] == D && is_heavy[D]) ++D;
        plan.hotd = D;
        plan.hot_nnz = D > 0 ? (int64_t)rp[D] - rp[0] : 0;
        if (D > 0) {
            std::vector<PlanEntry> fent;
            std::vector<int32_t> fptr(nhb + 1, 0);
            int32_t fmax = 1;
            const int32_t hot_slot_end = lptr[D];   // slots of long rows 0..D-1 come first
            for (int32_t b = 0; b < nhb; ++b) {
                int32_t c = 0;
                for (const PlanEntry& E : dl[b])
                    if (E.a >= hot_slot_end) { fent.push_back(E); ++c; }
                fptr[b + 1] = (int32_t)fent.size();
                fmax = std::max(fmax, c);
            }
            plan.dense_maxitems_f = fmax;
            plan.dense_ent_f.alloc(std::max<size_t>(fent.size(), 1));
            plan.dense_ptr_f.alloc(nhb + 1);
            if (!fent.empty())
                CPD_CUDA(cudaMemcpy(plan.dense_ent_f.p, fent.data(), sizeof(PlanEntry) * fent.size(),
                                    cudaMemcpyHostToDevice));
            CPD_CUDA(cudaMemcpy(plan.dense_ptr_f.p, fptr.data(), sizeof(int32_t) * (nhb + 1), cudaMemcpyHostToDevice));
        }
    }
    std::vector<int32_t> next(lptr.begin(), lptr.end() - 1);
    int64_t npieces = 0;
    plan.seg.assign(1, 0);
    plan.seg.push_back((int32_t)ent.size());
    for (int32_t s = 0; s < nslab; ++s) {
        plan.seg.push_back((int32_t)(ent.size() + by_slab[s].size()));   // seg[s + 1 .. s + 2) = slab s
        for (PlanEntry E : by_slab[s]) {
            E.a = next[-1 - E.b]++;   // slab-major visit == column order within each row
            ent.push_back(E);
            ++npieces;
        }
    }
    if (ent.size() > (size_t)INT32_MAX / 2) throw Error(CPD_E_DIM, "plan too large");
    plan.nent = (int32_t)ent.size();
    plan.nlong = nl;
    plan.rows_entries = nrows_e;
    plan.single_entries = 0;
    plan.long_pieces = (int64_t)lptr[nl];
    plan.nslab = nslab;
    // warp plan with >= 2 slabs: the short rows' items also run once per column slab
    // (k_csrw slab mode over a slab-major copy of their entries), so their gathers of
    // the vector hit an L2-resident half instead of DRAM.  On by default (C5: dual step
    // -1%, profiles/r01_kernel_iterations.md v35); CPD_SHORT=0 disables.  (A thread-
    // per-row version, v18, was latency-bound and slower.)
    plan.short_on = 0;
    const char* she = getenv("CPD_SHORT");
    // CPD_SHORT_SLABS (env, else the macro): number of short-row slabs; 0 = the long
    // pieces' slabs (SLAB_COLS wide), so a short pass and that slab's pieces run back to back
    const char* sse = getenv("CPD_SHORT_SLABS");
    const int64_t nreq = sse ? atoll(sse) : CPD_SHORT_SLABS;
    const int32_t nss = nreq <= 0 ? nslab : (int32_t)std::min<int64_t>(nreq, std::max<int64_t>(1, cols));
    const int64_t sw = nreq <= 0 ? slab_cols() : ((int64_t)cols + nss - 1) / nss;
    plan.short_ilv = nreq <= 0 ? 1 : 0;
    plan.short_nslab = nss;
    plan.short_width = sw;
    if (warp && rows > 0 && ((nslab >= 2 && !(she && she[0] == '0')) || (she && she[0] == '1'))) {   // =1: also small n (tests)
        const int32_t nslab = nss;   // the short rows' own column slabs (each x slab L2-resident)
        DBuf<int32_t> cnt((size_t)nslab * rows);
        const int g = (int)std::min<int64_t>(((int64_t)rows + 255) / 256, 8192);
        k_short_count<<<g, 256>>>(rows, nslab, long_min, d_p, d_col, cnt.p, sw);
        CPD_CUDA(cudaGetLastError());
        // sp[s][r] = exclusive prefix over (s, r) in slab-major order; sp[s][rows] = end of slab s
        plan.short_ptr.alloc((size_t)nslab * (rows + 1));
        DBuf<int32_t> flat((size_t)nslab * rows + 1);
        size_t tb = 0;
        CPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, flat.p, (int)((int64_t)nslab * rows)));
        DBuf<unsigned char> tmp(tb);
        CPD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, flat.p, (int)((int64_t)nslab * rows)));
        k_short_ptr<<<(int)std::min<int64_t>(((int64_t)nslab * (rows + 1) + 255) / 256, 65536), 256>>>(
            rows, nslab, flat.p, cnt.p, plan.short_ptr.p);
        CPD_CUDA(cudaGetLastError());
        int32_t htot = 0;
        CPD_CUDA(cudaMemcpy(&htot, plan.short_ptr.p + (size_t)nslab * (rows + 1) - 1, sizeof(int32_t),
                            cudaMemcpyDeviceToHost));
        const int64_t total = htot;
        plan.short_col.alloc(std::max<int64_t>(total, 1));
        plan.short_val.alloc(std::max<int64_t>(total, 1));
        const int gw = (int)std::min<int64_t>(((int64_t)rows * 32 + 255) / 256, 65536);
        k_short_fill<<<gw, 256>>>(rows, nslab, long_min, d_p, d_col, d_val, plan.short_ptr.p, plan.short_col.p,
                                  plan.short_val.p, sw);
        CPD_CUDA(cudaGetLastError());
        plan.short_nnz = total;
        plan.short_on = 1;
    }
    plan.ent.alloc(std::max<size_t>(ent.size(), 1));
    CPD_CUDA(cudaMemcpy(plan.ent.p, ent.data(), sizeof(PlanEntry) * ent.size(), cudaMemcpyHostToDevice));
    if (plan.short_on && plan.seg[1] > 0) {
        const int32_t ni = plan.seg[1];
        plan.short_ent.alloc((size_t)plan.short_nslab * ni);
        const int64_t tot = (int64_t)plan.short_nslab * ni;
        k_short_ents<<<(int)std::min<int64_t>((tot + 255) / 256, 65536), 256>>>(ni, plan.short_nslab, rows, plan.ent.p,
                                                                             plan.short_ptr.p, plan.short_ent.p);
        CPD_CUDA(cudaGetLastError());
    }
    plan.long_row.alloc(std::max(nl, 1));
    plan.long_ptr.alloc(nl + 1);
    // k_finish order: long rows with > FIN_SPLIT partials first (a CTA each), then the
    // rest (a warp each)
    {
        const int64_t ps = warp ? 1 : GW;
        std::vector<int32_t> order;
        // (the fused hot rows always get a CTA: their sums span the primal step's warps)
        auto cta = [&](int32_t l) { return l < plan.hotd || (int64_t)(lptr[l + 1] - lptr[l]) * ps > FIN_SPLIT; };
        for (int32_t l = 0; l < nl; ++l)
            if (cta(l)) order.push_back(l);
        plan.nfin_heavy = (int32_t)order.size();
        for (int32_t l = 0; l < nl; ++l)
            if (!cta(l)) order.push_back(l);
        plan.long_ents.alloc(std::max(nl, 1));
        if (nl) CPD_CUDA(cudaMemcpy(plan.long_ents.p, order.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice));
    }
    if (nl) CPD_CUDA(cudaMemcpy(plan.long_row.p, lrows.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice));
    CPD_CUDA(cudaMemcpy(plan.long_ptr.p, lptr.data(), sizeof(int32_t) * (nl + 1), cudaMemcpyHostToDevice));
}

// ------------------------------------------------------------ SELL-32
// entries [a, b) of row r with columns in [c0, c1) (columns ascending): [lo, hi)
__device__ __forceinline__ void col_range(const int32_t* j, int32_t a, int32_t b, int32_t c0, int32_t c1,
                                          int32_t& lo, int32_t& hi)
{
    int32_t l = a, h = b;
    while (l < h) {
        const int32_t mid = l + (h - l) / 2;
        if (j[mid] < c0) l = mid + 1; else h = mid;
    }
    lo = l;
    h = b;
    while (l < h) {
        const int32_t mid = l + (h - l) / 2;
        if (j[mid] < c1) l = mid + 1; else h = mid;
    }
    hi = l;
}

__global__ void k_sell_len(int32_t rows, int32_t nslice, const int32_t* p, int64_t* len, int32_t r0 = 0,
                           const int32_t* j = nullptr, int32_t c0 = 0, int32_t c1 = 0)
{
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nslice;
         s += (int64_t)gridDim.x * blockDim.x) {
        int32_t mx = 0;
        const int64_t r1 = std::min<int64_t>((s + 1) * 32, rows);
        for (int64_t r = s * 32; r < r1; ++r) {
            int32_t lo = p[r0 + r], hi = p[r0 + r + 1];
            if (j) col_range(j, lo, hi, c0, c1, lo, hi);
            mx = max(mx, hi - lo);
        }
        len[s] = (int64_t)((mx + SELL_PAIR) / (1 + SELL_PAIR) * (1 + SELL_PAIR)) * 32;   // pair layout: even width
    }
}

// one thread per (slice, lane): row r0 + r's entries, then padding (-1, 0.0); rev: the
// padding, then the row's entries in descending column order
__global__ void k_sell_fill(int32_t rows, int32_t nslice, const int32_t* p, const int32_t* j, const double* x,
                            const int64_t* sp, int32_t* scol, double* sval, int32_t r0 = 0, int32_t c0 = 0,
                            int32_t c1 = 0, bool rev = false)
{
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)nslice * 32;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t >> 5, lane = t & 31, r = t;
        const int64_t b = sp[s], len = (sp[s + 1] - b) >> 5;
        int32_t lo = r < rows ? p[r0 + r] : 0, hi = r < rows ? p[r0 + r + 1] : 0;
        if (c1 > c0 && r < rows) col_range(j, lo, hi, c0, c1, lo, hi);
        const int64_t q0 = lo, n = hi - lo;
        for (int64_t k = 0; k < len; ++k) {
            const int64_t d = b + sell_pos(k, lane);
            // rev: padding first, then the entries in reverse order (each lane's last
            // entries are its lowest columns, in the slice's last round)
            const int64_t kk = rev ? k - (len - n) : k;
            const bool ok = rev ? kk >= 0 : k < n;
            const int64_t q = q0 + (rev ? n - 1 - kk : k);
            scol[d] = ok ? j[q] : -1;
            sval[d] = ok ? x[q] : 0.0;
        }
    }
}

// Mark the SELL entries of A^T whose row of A is short (<= WLONG entries: the warp
// plan's rows items) with PUSH_BIT (short-row push).
__global__ void k_mark_push(int64_t N, int32_t* scol, const int32_t* Ap)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = scol[q];
        if (c >= 0 && Ap[c + 1] - Ap[c] <= WLONG) scol[q] = c | PUSH_BIT;
    }
}

void mark_push(cpd_problem* P)
{
    P->push_on = false;
    // off by default: the fp64 atomics cost more than the gathers they replace
    // (C5: primal step 0.75 -> 2.45 ms for dual step 1.20 -> 1.11 ms,
    // profiles/r01_kernel_iterations.md v22); CPD_PUSH=1 enables
    const char* pe = getenv("CPD_PUSH");
    if (!(pe && pe[0] == '1')) return;
    if (P->split >= 0 || !P->AT.sell.on || !P->A.plan.warp || P->m >= PUSH_BIT) return;
    const int64_t N = P->AT.sell.padded;
    k_mark_push<<<(int)std::min<int64_t>((N + 255) / 256, 65536), 256>>>(N, P->AT.sell.col.p, P->A.p.p);
    CPD_CUDA(cudaGetLastError());
    CPD_CUDA(cudaDeviceSynchronize());
    // short-row nonzeros (their K2 reads move to K1's push)
    std::vector<int32_t> hp((size_t)P->m + 1);
    CPD_CUDA(cudaMemcpy(hp.data(), P->A.p.p, sizeof(int32_t) * hp.size(), cudaMemcpyDeviceToHost));
    int64_t sn = 0;
    for (int32_t i = 0; i < P->m; ++i)
        if (hp[i + 1] - hp[i] <= WLONG) sn += hp[i + 1] - hp[i];
    P->push_nnz = sn;
    P->push_on = true;
}

// SELL-32 of rows [r0, r0 + rows) of M's CSR into S (S.on = false when padding > max_ratio).
static void build_sell_rows(const Matrix& M, Sell& S, int32_t r0, int32_t rows, int64_t nnz, double max_ratio,
                            int32_t c0 = 0, int32_t c1 = 0, bool rev = false)
{
    S.rev = rev;
    S.c0 = c0;
    S.c1 = c1;
    S.on = false;
    S.r0 = r0;
    S.rows = rows;
    const int32_t ns = (int32_t)(((int64_t)rows + 31) / 32);
    if (nnz == 0 || rows == 0) return;
    DBuf<int64_t> len((size_t)ns + 1);
    CPD_CUDA(cudaMemset(len.p, 0, sizeof(int64_t) * ((size_t)ns + 1)));
    const int g = (int)std::min<int64_t>(((int64_t)ns + 255) / 256, 4096);
    k_sell_len<<<g, 256>>>(rows, ns, M.p.p, len.p, r0, c1 > c0 ? M.j.p : nullptr, c0, c1);
    CPD_CUDA(cudaGetLastError());
    S.sp.alloc((size_t)ns + 1);
    size_t tb = 0;
    CPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, S.sp.p, ns + 1));
    DBuf<unsigned char> tmp(tb);
    CPD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.p, S.sp.p, ns + 1));
    int64_t padded = 0;
    CPD_CUDA(cudaMemcpy(&padded, S.sp.p + ns, sizeof(int64_t), cudaMemcpyDeviceToHost));
    S.padded = padded;
    if ((double)padded > max_ratio * (double)nnz) {
        S.sp.free();
        return;
    }
    S.col.alloc((size_t)std::max<int64_t>(padded, 1));
    S.val.alloc((size_t)std::max<int64_t>(padded, 1));
    const int g2 = (int)std::min<int64_t>(((int64_t)ns * 32 + 255) / 256, 65536);
    k_sell_fill<<<g2, 256>>>(rows, ns, M.p.p, M.j.p, M.x.p, S.sp.p, S.col.p, S.val.p, r0, c0, c1, rev);
    CPD_CUDA(cudaGetLastError());
    CPD_CUDA(cudaDeviceSynchronize());
    S.nslice = ns;
    S.on = true;
}

// rev: each lane's entries in descending column order (A^T of a renumbered problem: the
// hot rows of A, its lowest columns, become each lane's last entries — hot-row fusion)
void build_sell(Matrix& M, int64_t nnz, double max_ratio, bool rev)
{
    build_sell_rows(M, M.sell, 0, M.rows, nnz, max_ratio, 0, 0, rev);
}

// Short rows of a warp-plan layout whose rows are ordered by decreasing length (hot-row
// renumbering): rows [r_s, rows) with <= WLONG nonzeros form a suffix, and their dual
// step runs as a SELL-32 pass (lane = row, no segmented scan, no row search) instead of
// the warp plan's rows items.  CPD_SSELL=0 keeps the rows items.
void build_short_sell(Matrix& M, const std::vector<int32_t>& rp)
{
    M.sell_short.on = false;
    M.sell_half[0].on = M.sell_half[1].on = false;
    const char* e = getenv("CPD_SSELL");
    if ((e && e[0] == '0') || !M.plan.warp) return;
    const int32_t rows = M.rows;
    int32_t rs = rows;
    while (rs > 0 && (int64_t)rp[rs] - rp[rs - 1] <= WLONG) --rs;
    for (int32_t r = 0; r < rs; ++r)   // suffix property: every earlier row is long
        if ((int64_t)rp[r + 1] - rp[r] <= WLONG) return;
    if (rs >= rows) return;
    const int64_t nz = (int64_t)rp[rows] - rp[rs];
    // two column halves (each half of the gathered vector L2-resident) when the vector
    // is larger than ~64 MB; CPD_SSELL=1 forces one pass, =2 two
    const bool halves = (e && e[0] == '2') || (!(e && e[0] == '1') && (int64_t)M.cols * 8 > (64ll << 20));
    if (halves) {
        const int32_t h = (M.cols + 1) / 2;
        build_sell_rows(M, M.sell_half[0], rs, rows - rs, nz, 2.0, 0, h);
        build_sell_rows(M, M.sell_half[1], rs, rows - rs, nz, 2.0, h, M.cols);
        if (M.sell_half[0].on && M.sell_half[1].on) return;   // running sums: Ctx::sshortA
        M.sell_half[0].on = M.sell_half[1].on = false;
    }
    build_sell_rows(M, M.sell_short, rs, rows - rs, nz, 1.25);
}

// ------------------------------------------------------------ hot-row renumbering
__global__ void k_remap(int64_t N, int32_t* j, const int32_t* pinv)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < N; q += (int64_t)gridDim.x * blockDim.x)
        j[q] = pinv[j[q]];
}
__global__ void k_gather_d(int64_t N, double* dst, const double* src, const int32_t* idx)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

thread_local bool g_no_renumber = false;

// Rows of A ordered by decreasing length (stable) when the HOT_ROWS longest rows
// hold >= 30% of the nonzeros (C5's Zipf rows): the most-gathered entries of y then
// form a prefix that k_sell keeps in shared memory.  Every y-side
// array is stored in this internal order; the ABI maps y / b / senses / r.
__global__ void k_perm_lens(int32_t rows, const int32_t* perm, const int32_t* p, int32_t* len, int32_t* pinv)
{
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < rows; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = perm[k];
        len[k] = p[r + 1] - p[r];
        pinv[r] = (int32_t)k;
    }
}

// Hot-row renumbering wanted? (the HOT_ROWS longest rows hold >= 30% of the nonzeros;
// single GPU; CPD_HOTROWS=0 disables).  maxlen: the longest row.
static bool hot_rows_wanted(const cpd_problem* P, const std::vector<int32_t>& hp, int32_t* maxlen_out)
{
    const int32_t m = P->m;
    const char* e = getenv("CPD_HOTROWS");
    if ((e && e[0] == '0') || g_no_renumber || m <= HOT_ROWS || P->nnz == 0) return false;
    int32_t maxlen = 0;
    std::vector<int32_t> lens(m);
    for (int32_t i = 0; i < m; ++i) {
        lens[i] = hp[i + 1] - hp[i];
        maxlen = std::max(maxlen, lens[i]);
    }
    std::nth_element(lens.begin(), lens.begin() + HOT_ROWS, lens.end(), std::greater<int32_t>());
    int64_t top = 0;
    for (int32_t k = 0; k < HOT_ROWS; ++k) top += lens[k];
    if (maxlen_out) *maxlen_out = maxlen;
    return 10 * top >= 3 * P->nnz;
}

// Column renumbering: with the rows ranked by decreasing length, each
// column j gets the key "rank of its longest non-heavy row" and the columns are stably
// sorted by it, so the columns of every long (not heavy) row cluster in x and that row's
// gathers in the dual step share 32-byte sectors (C5 simulation: -35% L2 sectors for the
// long rows).  Internal column k = user column cperm[k]; the ABI maps every n-vector.
// Runs before the row renumbering (which then tie-breaks on the new column halves);
// single GPU, with the hot-row renumbering; CPD_COLSORT=0 disables.
static void transpose(int32_t rows, int32_t cols, int64_t nnz, const int32_t* p, const int32_t* j,
                      const double* x, int32_t* tp, int32_t* tj, double* tx, int sms);
// new row k = old row perm[k] for a layout of short rows: a warp per row, lane-strided
// copy (coalesced; the rows of CSR(A^T) are short)
__global__ void k_permute_rows_warp(int32_t rows, const int32_t* perm, const int32_t* op, const int32_t* oj,
                                    const double* ox, const int32_t* np, int32_t* nj, double* nx)
{
    const int lane = threadIdx.x & 31;
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < rows;
         k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t src = op[perm[k]], len = op[perm[k] + 1] - src, dst = np[k];
        for (int32_t q = lane; q < len; q += 32) {
            nj[dst + q] = oj[src + q];
            nx[dst + q] = ox[src + q];
        }
    }
}

// short rows' entry count in the first half of the NEW column order (tie-break of the
// row renumbering, so a SELL slice of short rows is even in both column halves)
__global__ void k_h0_count(int32_t n, const int32_t* tp, const int32_t* tj, const int32_t* cpinv, const int32_t* ap,
                           int32_t half, int32_t* h0)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t nj = cpinv ? cpinv[j] : (int32_t)j;
        if (nj >= half) continue;
        for (int32_t q = tp[j]; q < tp[j + 1]; ++q) {
            const int32_t i = tj[q];
            if (ap[i + 1] - ap[i] <= WLONG) atomicAdd(&h0[i], 1);
        }
    }
}
__global__ void k_len_keys_h0(int32_t rows, const int32_t* p, const int32_t* h0, int32_t maxlen, uint64_t* key,
                              int32_t* val)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t len = p[r + 1] - p[r];
        const uint64_t sec = len <= WLONG ? (uint64_t)(WLONG - h0[r]) : 0;
        key[r] = ((uint64_t)(maxlen - len) << 8) | sec;
        val[r] = (int32_t)r;
    }
}

__global__ void k_rank_rows(int32_t rows, const int32_t* perm, int32_t* rank)
{
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < rows; k += (int64_t)gridDim.x * blockDim.x)
        rank[perm[k]] = (int32_t)k;
}
__global__ void k_col_keys(int32_t n, const int32_t* tp, const int32_t* tj, const int32_t* rank, const int32_t* ap,
                           int64_t hmin, int32_t none, int32_t* key, int32_t* val)
{
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        int32_t best = none;
        for (int32_t q = tp[j]; q < tp[j + 1]; ++q) {
            const int32_t i = tj[q];
            if ((int64_t)ap[i + 1] - ap[i] < hmin) best = min(best, rank[i]);
        }
        key[j] = best;
        val[j] = (int32_t)j;
    }
}
// Combined renumbering from CSR(A^T), one transpose:
//  rows of A by decreasing length (hot-row renumbering; short rows tie-broken by their
//  entry count in the first half of the NEW column order), and, unless CPD_COLSORT=0,
//  columns by the length rank of their longest non-heavy row (column renumbering).
//  CSR(A^T) gets its rows permuted (columns) and its entries remapped (rows); CSR(A) is
//  then the stable transpose of it, so every row of A has ascending (new) columns.
static void renumber(cpd_problem* P, std::vector<int32_t>& hp)
{
    int32_t maxlen = 0;
    if (!hot_rows_wanted(P, hp, &maxlen)) return;
    const char* e = getenv("CPD_COLSORT");
    const bool cols_on = !(e && e[0] == '0');
    const int32_t m = P->m, n = P->n;
    const int64_t nnz = P->nnz;
    const int sms = P->num_sms;
    auto grid = [&](int64_t N) { return (int)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, (int64_t)sms * 16)); };
    int end_bit = 9;
    while ((1LL << (end_bit - 8)) <= (long long)maxlen) ++end_bit;
    auto sort_rows = [&](const DBuf<uint64_t>& k, DBuf<int32_t>& val, DBuf<int32_t>& perm) {
        DBuf<uint64_t> k2(m);
        size_t tb = 0;
        CPD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k.p, k2.p, val.p, perm.p, m, 0, end_bit));
        DBuf<unsigned char> tmp(tb);
        CPD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k.p, k2.p, val.p, perm.p, m, 0, end_bit));
    };
    DBuf<uint64_t> key(m);
    DBuf<int32_t> val(m), h0(m), rperm(m), rpinv(m);
    CPD_CUDA(cudaMemset(h0.p, 0, sizeof(int32_t) * m));
    DBuf<int32_t> cperm, cpinv;
    if (cols_on) {
        // rank of every row by length (ties: index), the column keys, their stable sort
        DBuf<int32_t> rank(m), rp0(m);
        k_len_keys_h0<<<grid(m), 256>>>(m, P->A.p.p, h0.p, maxlen, key.p, val.p);   // h0 = 0: length only
        sort_rows(key, val, rp0);
        k_rank_rows<<<grid(m), 256>>>(m, rp0.p, rank.p);
        DBuf<int32_t> ckey(n), ckey2(n), cval(n);
        cperm.alloc(n);
        cpinv.alloc(n);
        k_col_keys<<<grid(n), 256>>>(n, P->AT.p.p, P->AT.j.p, rank.p, P->A.p.p, heavy_min(), m, ckey.p, cval.p);
        int cb = 1;
        while ((1LL << cb) <= (long long)m) ++cb;
        size_t tb = 0;
        CPD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ckey.p, ckey2.p, cval.p, cperm.p, n, 0, cb));
        DBuf<unsigned char> tmp(tb);
        CPD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, ckey.p, ckey2.p, cval.p, cperm.p, n, 0, cb));
        k_rank_rows<<<grid(n), 256>>>(n, cperm.p, cpinv.p);   // cpinv[old column] = new column
    }
    // rows: length, then first-half count in the new column order
    k_h0_count<<<grid(n), 256>>>(n, P->AT.p.p, P->AT.j.p, cols_on ? cpinv.p : nullptr, P->A.p.p,
                                 (int32_t)((n + 1) / 2), h0.p);
    k_len_keys_h0<<<grid(m), 256>>>(m, P->A.p.p, h0.p, maxlen, key.p, val.p);
    sort_rows(key, val, rperm);
    k_rank_rows<<<grid(m), 256>>>(m, rperm.p, rpinv.p);   // rpinv[old row] = new row
    // CSR(A^T): rows in the new column order, entries renamed to the new rows
    if (cols_on) {
        DBuf<int32_t> nlen((size_t)n + 1), ntp((size_t)n + 1), tmpinv(n);
        k_perm_lens<<<grid(n), 256>>>(n, cperm.p, P->AT.p.p, nlen.p, tmpinv.p);
        CPD_CUDA(cudaMemset(nlen.p + n, 0, sizeof(int32_t)));
        size_t sb = 0;
        CPD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sb, nlen.p, ntp.p, n + 1));
        DBuf<unsigned char> stmp(sb);
        CPD_CUDA(cub::DeviceScan::ExclusiveSum(stmp.p, sb, nlen.p, ntp.p, n + 1));
        DBuf<int32_t> nj(std::max<int64_t>(nnz, 1));
        DBuf<double> nx(std::max<int64_t>(nnz, 1));
        k_permute_rows_warp<<<(int)std::min<int64_t>(((int64_t)n * 32 + 255) / 256, (int64_t)sms * 64), 256>>>(
            n, cperm.p, P->AT.p.p, P->AT.j.p, P->AT.x.p, ntp.p, nj.p, nx.p);
        CPD_CUDA(cudaGetLastError());
        P->AT.p = std::move(ntp);
        P->AT.j = std::move(nj);
        P->AT.x = std::move(nx);
    }
    k_remap<<<grid(nnz), 256>>>(nnz, P->AT.j.p, rpinv.p);
    {   // each row of A^T in ascending new row order (A^T's SELL reverses it: hot-row fusion)
        DBuf<int32_t> sj(std::max<int64_t>(nnz, 1));
        DBuf<double> sx(std::max<int64_t>(nnz, 1));
        size_t tb = 0;
        CPD_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tb, P->AT.j.p, sj.p, P->AT.x.p, sx.p, nnz, n,
                                                     P->AT.p.p, P->AT.p.p + 1));
        DBuf<unsigned char> tmp(std::max<size_t>(tb, 1));
        CPD_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp.p, tb, P->AT.j.p, sj.p, P->AT.x.p, sx.p, nnz, n,
                                                     P->AT.p.p, P->AT.p.p + 1));
        P->AT.j = std::move(sj);
        P->AT.x = std::move(sx);
    }
    // CSR(A) = the stable transpose: new rows, ascending new columns
    transpose(n, m, nnz, P->AT.p.p, P->AT.j.p, P->AT.x.p, P->A.p.p, P->A.j.p, P->A.x.p, sms);
    // vectors in the new orders
    DBuf<double> t(std::max(std::max(n, m), 1));
    k_gather_d<<<grid(m), 256>>>(m, t.p, P->b.p, rperm.p);
    CPD_CUDA(cudaMemcpy(P->b.p, t.p, sizeof(double) * m, cudaMemcpyDeviceToDevice));
    if (cols_on) {
        auto gather = [&](DBuf<double>& v) {
            k_gather_d<<<grid(n), 256>>>(n, t.p, v.p, cperm.p);
            CPD_CUDA(cudaMemcpy(v.p, t.p, sizeof(double) * n, cudaMemcpyDeviceToDevice));
        };
        gather(P->c);
        if (!P->uniform_bounds) {
            gather(P->lb);
            gather(P->ub);
        }
    }
    CPD_CUDA(cudaGetLastError());
    P->h_rperm.resize(m);
    CPD_CUDA(cudaMemcpy(P->h_rperm.data(), rperm.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
    CPD_CUDA(cudaMemcpy(hp.data(), P->A.p.p, sizeof(int32_t) * ((size_t)m + 1), cudaMemcpyDeviceToHost));
    P->rperm = std::move(rperm);
    if (cols_on) P->cperm = std::move(cperm);
    P->hot = HOT_ROWS;
}

// ------------------------------------------------------------ validation
// err[class] = smallest offending index (atomicMin), INT64_MAX if none.
enum { ERR_ROWPTR = 0, ERR_COL = 1, ERR_ORDER = 2, ERR_VAL = 3, ERR_B = 4, ERR_C = 5, ERR_BND = 6,
       ERR_MISMATCH = 7, NERR = 8 };

__device__ __forceinline__ void note(unsigned long long* err, int cls, long long idx)
{
    atomicMin(&err[cls], (unsigned long long)idx);
}

__global__ void k_check_rowptr(int32_t rows, const int32_t* p, int64_t nnz, unsigned long long* err)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = p[r];
        bool bad = (r == 0 && v != 0) || (r == rows && (int64_t)v != nnz) || v < 0 || (int64_t)v > nnz;
        if (r > 0 && p[r - 1] > v) bad = true;
        if (bad) note(err, ERR_ROWPTR, r);
    }
}

// Per nonzero: column range, strictly increasing columns within a row, finite nonzero value.
__global__ void k_check_entries(int32_t rows, int32_t cols, int64_t nnz, const int32_t* p,
                                const int32_t* j, const double* x, unsigned long long* err)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x) {
        // row of q: last r with p[r] <= q
        int32_t lo = 0, hi = rows;   // p[lo] <= q < p[hi]
        while (hi - lo > 1) {
            const int32_t mid = lo + (hi - lo) / 2;
            if (p[mid] <= q) lo = mid; else hi = mid;
        }
        const int32_t col = j[q];
        if (col < 0 || col >= cols) note(err, ERR_COL, q);
        if (q > p[lo] && j[q - 1] >= col) note(err, ERR_ORDER, q);
        const double v = x[q];
        if (!isfinite(v)) note(err, ERR_VAL, q);
        if (v == 0.0) note(err, ERR_VAL, q);
    }
}

__global__ void k_check_finite(int64_t N, const double* v, unsigned long long* err, int cls)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(v[i])) note(err, cls, i);
}

// lb <= ub, no NaN, lb != +inf, ub != -inf; uniform-ness flags in flags[0] (lb), flags[1] (ub).
__global__ void k_check_bounds(int64_t n, const double* lb, const double* ub, unsigned long long* err,
                               int* flags)
{
    const double l0 = lb[0], u0 = ub[0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double l = lb[i], u = ub[i];
        if (isnan(l) || isnan(u) || l > u || l == INFINITY || u == -INFINITY) note(err, ERR_BND, i);
        if (!(l == l0)) flags[0] = 1;
        if (!(u == u0)) flags[1] = 1;
    }
}

__global__ void k_fill(int64_t N, double* v, double val)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = val;
}

__global__ void k_iota(int64_t N, int32_t* v)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}

// Row pointers of the transpose from its SORTED keys: tp[c] = #keys < c.  Position q
// (0..nnz, nnz = sentinel) where the key steps from a to b starts rows a+1..b, so each
// tp entry is written exactly once (no atomics: a histogram with atomics serialised on
// the Zipf head's counters, 27 ms per transpose on C5).
__global__ void k_row_starts(int64_t nnz, const int32_t* keys, int32_t cols, int32_t* tp)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= nnz;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = q == 0 ? -1 : keys[q - 1];
        const int32_t b = q == nnz ? cols : keys[q];
        for (int32_t c = a + 1; c <= b; ++c) tp[c] = (int32_t)q;
    }
}

// tj[q] = source row of the permuted nonzero; tx[q] = its value.
__global__ void k_gather_transpose(int32_t rows, int64_t nnz, const int32_t* p, const double* x,
                                   const int32_t* perm, int32_t* tj, double* tx)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t src = perm[q];
        int32_t lo = 0, hi = rows;
        while (hi - lo > 1) {
            const int32_t mid = lo + (hi - lo) / 2;
            if (p[mid] <= src) lo = mid; else hi = mid;
        }
        tj[q] = lo;
        tx[q] = x[src];
    }
}

__device__ __forceinline__ long long bits_of(int32_t v) { return v; }
__device__ __forceinline__ long long bits_of(double v) { return __double_as_longlong(v); }

template <class T>
__global__ void k_compare(int64_t N, const T* a, const T* b, unsigned long long* err)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        if (bits_of(a[i]) != bits_of(b[i])) note(err, ERR_MISMATCH, i);
}

static int grid_of(int64_t N, int sms)
{
    const int64_t g = (N + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * 16));
}

// Stable transpose of CSR (rows x cols) into CSR (cols x rows): radix sort of the
// column keys (stable => source-row order kept inside each new row).
static void transpose(int32_t rows, int32_t cols, int64_t nnz, const int32_t* p, const int32_t* j,
                      const double* x, int32_t* tp, int32_t* tj, double* tx, int sms)
{
    DBuf<int32_t> keys_out(std::max<int64_t>(nnz, 1)), idx(std::max<int64_t>(nnz, 1)),
        perm(std::max<int64_t>(nnz, 1));
    if (nnz > 0) {
        k_iota<<<grid_of(nnz, sms), 256>>>(nnz, idx.p);
        int end_bit = 1;
        while ((1LL << end_bit) < (long long)cols) ++end_bit;
        size_t tmp_bytes = 0;
        CPD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, j, keys_out.p, idx.p, perm.p,
                                                 (int)nnz, 0, end_bit));
        DBuf<unsigned char> tmp(tmp_bytes);
        CPD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, j, keys_out.p, idx.p, perm.p,
                                                 (int)nnz, 0, end_bit));
        k_gather_transpose<<<grid_of(nnz, sms), 256>>>(rows, nnz, p, x, perm.p, tj, tx);
    }
    k_row_starts<<<grid_of(nnz + 1, sms), 256>>>(nnz, keys_out.p, cols, tp);
    CPD_CUDA(cudaGetLastError());
    CPD_CUDA(cudaDeviceSynchronize());
}

template <class T>
static void upload(DBuf<T>& dst, const T* src, size_t count, int mem)
{
    dst.alloc(std::max<size_t>(count, 1));
    if (count)
        CPD_CUDA(cudaMemcpy(dst.p, src, sizeof(T) * count,
                            mem == CPD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
}

static void check_errors(const DBuf<unsigned long long>& err, bool transposed_given)
{
    unsigned long long h[NERR];
    CPD_CUDA(cudaMemcpy(h, err.p, sizeof(h), cudaMemcpyDeviceToHost));
    const unsigned long long NONE = ~0ULL;
    auto msg = [&](int cls) { return std::to_string((long long)h[cls]); };
    if (h[ERR_ROWPTR] != NONE) throw Error(CPD_E_CSR, "bad rowptr at index " + msg(ERR_ROWPTR));
    if (h[ERR_COL] != NONE) throw Error(CPD_E_CSR, "column index out of range at nonzero " + msg(ERR_COL));
    if (h[ERR_ORDER] != NONE)
        throw Error(CPD_E_CSR, "columns not strictly increasing (unsorted or duplicate) at nonzero " +
                                   msg(ERR_ORDER));
    if (h[ERR_VAL] != NONE) throw Error(CPD_E_CSR, "explicit zero or non-finite value at nonzero " + msg(ERR_VAL));
    if (h[ERR_B] != NONE) throw Error(CPD_E_NONFINITE, "non-finite b at row " + msg(ERR_B));
    if (h[ERR_C] != NONE) throw Error(CPD_E_NONFINITE, "non-finite c at column " + msg(ERR_C));
    if (h[ERR_BND] != NONE) throw Error(CPD_E_BOUNDS, "invalid bounds (lb > ub, NaN, lb=+inf or ub=-inf) at column " + msg(ERR_BND));
    if (transposed_given && h[ERR_MISMATCH] != NONE)
        throw Error(CPD_E_CSR, "CSR(A) and CSR(A^T) describe different matrices (first mismatch at " +
                                   msg(ERR_MISMATCH) + ")");
}

static void validate_csr(int32_t rows, int32_t cols, int64_t nnz, const Matrix& M,
                         DBuf<unsigned long long>& err, int sms)
{
    k_check_rowptr<<<grid_of((int64_t)rows + 1, sms), 256>>>(rows, M.p.p, nnz, err.p);
    CPD_CUDA(cudaGetLastError());
    check_errors(err, false);   // entries check needs a monotone rowptr
    if (nnz > 0)
        k_check_entries<<<grid_of(nnz, sms), 256>>>(rows, cols, nnz, M.p.p, M.j.p, M.x.p, err.p);
    CPD_CUDA(cudaGetLastError());
    check_errors(err, false);
}

}  // namespace cpd

namespace cpd {
// ------------------------------------------------------------ diagonal preconditioning
// per row of a CSR layout: max |a| (mode 0) or sum |a| (mode 1), then sqrt (1 if 0);
// a CTA per row (strided per thread, block tree: fixed order), so long rows do not
// serialise on one warp
__global__ void k_row_absred(int32_t rows, const int32_t* p, const double* x, int mode, double* out)
{
    __shared__ double sw[8];
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        double v = 0.0;
        for (int64_t q = p[r] + threadIdx.x; q < p[r + 1]; q += blockDim.x) {
            const double a = fabs(x[q]);
            v = mode ? v + a : (a > v ? a : v);
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double t = __shfl_xor_sync(0xffffffffu, v, o);
            v = mode ? v + t : (t > v ? t : v);
        }
        __syncthreads();
        if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = mode ? t + sw[w] : (sw[w] > t ? sw[w] : t);
            out[r] = t > 0.0 ? sqrt(t) : 1.0;
        }
    }
}

// x_q <- x_q / (rho_i kappa_j) for entry q of row `r`, column `c` of a layout:
// A (swap 0): rho = rs[r], kappa = cs[c];  A^T (swap 1): rho = cs[c], kappa = rs[r]
// (entry-parallel; the row of entry q by binary search)
__global__ void k_apply_scale(int32_t rows, int64_t nnz, const int32_t* p, const int32_t* j, double* x,
                              const double* rs, const double* cs, int swap)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
        int32_t lo = 0, hi = rows;
        while (hi - lo > 1) {
            const int32_t mid = lo + (hi - lo) / 2;
            if (p[mid] <= q) lo = mid; else hi = mid;
        }
        const double den = swap ? cs[j[q]] * rs[lo] : rs[lo] * cs[j[q]];
        x[q] = x[q] / den;
    }
}

// op 0: v /= d; op 1: v *= d; op 2: out = 1 / v
__global__ void k_vec_op(int64_t N, double* v, const double* d, int op, double* out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        if (op == 0) v[i] = v[i] / d[i];
        else if (op == 1) v[i] = d[i] * v[i];
        else out[i] = 1.0 / v[i];
    }
}

// Ruiz (ruiz_iters passes of row / column max) then one Pock-Chambolle pass (row /
// column sums, alpha = 1), exactly the oracle's orc_scale order of operations.
void scale_problem(cpd_problem* P, int32_t ruiz_iters, int32_t pc)
{
    const int32_t m = P->m, n = P->n;
    const int sms = P->num_sms;
    auto gr = [&](int64_t rows) { return (int)std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)sms * 64)); };
    P->sr.alloc(m);
    P->ss.alloc(n);
    P->ir.alloc(m);
    P->is.alloc(n);
    DBuf<double> rho(m), kap(n);
    k_fill<<<grid_of(m, sms), 256>>>(m, P->sr.p, 1.0);
    k_fill<<<grid_of(n, sms), 256>>>(n, P->ss.p, 1.0);
    for (int pass = 0; pass < ruiz_iters + (pc ? 1 : 0); ++pass) {
        const int mode = pass >= ruiz_iters ? 1 : 0;
        k_row_absred<<<gr(m), 256>>>(m, P->A.p.p, P->A.x.p, mode, rho.p);
        k_row_absred<<<gr(n), 256>>>(n, P->AT.p.p, P->AT.x.p, mode, kap.p);
        k_apply_scale<<<grid_of(P->nnz, sms), 256>>>(m, P->nnz, P->A.p.p, P->A.j.p, P->A.x.p, rho.p, kap.p, 0);
        k_apply_scale<<<grid_of(P->nnz, sms), 256>>>(n, P->nnz, P->AT.p.p, P->AT.j.p, P->AT.x.p, kap.p, rho.p, 1);
        k_vec_op<<<grid_of(m, sms), 256>>>(m, P->sr.p, rho.p, 0, nullptr);
        k_vec_op<<<grid_of(n, sms), 256>>>(n, P->ss.p, kap.p, 0, nullptr);
        CPD_CUDA(cudaGetLastError());
    }
    // original bounds kept; the LP vectors become the scaled ones
    P->lb0.alloc(n);
    P->ub0.alloc(n);
    CPD_CUDA(cudaMemcpy(P->lb0.p, P->lb.p, sizeof(double) * n, cudaMemcpyDeviceToDevice));
    CPD_CUDA(cudaMemcpy(P->ub0.p, P->ub.p, sizeof(double) * n, cudaMemcpyDeviceToDevice));
    P->uniform0 = P->uniform_bounds;
    P->l00 = P->l0;
    P->u00 = P->u0;
    k_vec_op<<<grid_of(m, sms), 256>>>(m, P->b.p, P->sr.p, 1, nullptr);
    k_vec_op<<<grid_of(n, sms), 256>>>(n, P->c.p, P->ss.p, 1, nullptr);
    k_vec_op<<<grid_of(n, sms), 256>>>(n, P->lb.p, P->ss.p, 0, nullptr);
    k_vec_op<<<grid_of(n, sms), 256>>>(n, P->ub.p, P->ss.p, 0, nullptr);
    k_vec_op<<<grid_of(m, sms), 256>>>(m, P->sr.p, nullptr, 2, P->ir.p);
    k_vec_op<<<grid_of(n, sms), 256>>>(n, P->ss.p, nullptr, 2, P->is.p);
    CPD_CUDA(cudaGetLastError());
    P->uniform_bounds = false;
    // derived copies of the values
    if (P->AT.sell.on) build_sell(P->AT, P->nnz, 1.25, P->AT.sell.rev);
    if (P->A.sell.on) build_sell(P->A, P->nnz, 1.25);
    if (P->A.sell_short.on) {   // the scaled values of the short-row suffix
        const int32_t r0 = P->A.sell_short.r0, nr = P->A.sell_short.rows;
        int32_t q[2];
        CPD_CUDA(cudaMemcpy(&q[0], P->A.p.p + r0, sizeof(int32_t), cudaMemcpyDeviceToHost));
        CPD_CUDA(cudaMemcpy(&q[1], P->A.p.p + r0 + nr, sizeof(int32_t), cudaMemcpyDeviceToHost));
        build_sell_rows(P->A, P->A.sell_short, r0, nr, (int64_t)q[1] - q[0], 1e30);
    }
    for (int hh = 0; hh < 2; ++hh)
        if (P->A.sell_half[hh].on) {
            Sell& S = P->A.sell_half[hh];
            build_sell_rows(P->A, S, S.r0, S.rows, (int64_t)1 << 62, 1e30, S.c0, S.c1);
        }
    if (P->push_on) mark_push(P);
    for (Matrix* M : {&P->A, &P->AT})
        if (M->plan.short_on) {
            const int g = (int)std::min<int64_t>(((int64_t)M->rows * 32 + 255) / 256, 65536);   // a warp per row
            k_short_fill<<<g, 256>>>(M->rows, M->plan.short_nslab, WLONG, M->p.p, M->j.p, M->x.p,
                                     M->plan.short_ptr.p, M->plan.short_col.p, M->plan.short_val.p,
                                     M->plan.short_width);
        }
    CPD_CUDA(cudaGetLastError());
    CPD_CUDA(cudaDeviceSynchronize());
    P->scaled = true;
}
}  // namespace cpd

using namespace cpd;

// Implementation of cpd_problem_create (called from the ABI layer).
// CPD_TIMING=1: per-phase wall time of problem creation on stderr (device synchronised)
struct PhaseTimer {
    bool on;
    std::chrono::steady_clock::time_point t;
    PhaseTimer() : on(getenv("CPD_TIMING") && getenv("CPD_TIMING")[0] == '1'), t(std::chrono::steady_clock::now()) {}
    void mark(const char* what)
    {
        if (!on) return;
        cudaDeviceSynchronize();
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[cpd create] %-22s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

cpd_problem* cpd_problem_create_impl(int32_t m, int32_t n, int64_t nnz, const int32_t* Ap,
                                     const int32_t* Aj, const double* Ax, const int32_t* ATp,
                                     const int32_t* ATj, const double* ATx, const double* b,
                                     const double* c, const double* lb, const double* ub,
                                     int32_t mem, int32_t device)
{
    PhaseTimer tm;
    if (m < 1 || n < 1 || nnz < 0 || nnz >= (1LL << 31))
        throw Error(CPD_E_DIM, "need m >= 1, n >= 1, 0 <= nnz < 2^31");
    if (mem != CPD_HOST && mem != CPD_DEVICE) throw Error(CPD_E_ARG, "mem must be CPD_HOST or CPD_DEVICE");
    const bool haveA = Ap && (Aj || nnz == 0) && (Ax || nnz == 0);
    const bool haveAT = ATp && (ATj || nnz == 0) && (ATx || nnz == 0);
    if (!haveA && !haveAT) throw Error(CPD_E_ARG, "need CSR(A) or CSR(A^T)");
    if ((Ap || Aj || Ax) && !haveA) throw Error(CPD_E_ARG, "CSR(A) given partially");
    if ((ATp || ATj || ATx) && !haveAT) throw Error(CPD_E_ARG, "CSR(A^T) given partially");
    if (!b || !c) throw Error(CPD_E_ARG, "b and c are required");
    int ndev = 0;
    CPD_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw Error(CPD_E_ARG, "bad device ordinal");
    CPD_CUDA(cudaSetDevice(device));

    auto* P = new cpd_problem();
    try {
        P->device = device;
        P->m = m;
        P->n = n;
        P->nnz = nnz;
        // single-GPU layout (cpd_problem_create_dist overrides these)
        P->m_glob = m;
        P->n_glob = n;
        P->own_len[0] = m;
        P->own_len[1] = n;
        P->rank_gofs[0] = {0};
        P->rank_gofs[1] = {0};
        P->rank_len[0] = {m};
        P->rank_len[1] = {n};
        CPD_CUDA(cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, device));
        const int sms = P->num_sms;
        DBuf<unsigned long long> err(NERR);
        CPD_CUDA(cudaMemset(err.p, 0xff, sizeof(unsigned long long) * NERR));
        P->A.rows = m; P->A.cols = n;
        P->AT.rows = n; P->AT.cols = m;
        Matrix* given = haveA ? &P->A : &P->AT;
        if (haveA) {
            upload(P->A.p, Ap, (size_t)m + 1, mem);
            upload(P->A.j, Aj, (size_t)nnz, mem);
            upload(P->A.x, Ax, (size_t)nnz, mem);
            validate_csr(m, n, nnz, P->A, err, sms);
        } else {
            upload(P->AT.p, ATp, (size_t)n + 1, mem);
            upload(P->AT.j, ATj, (size_t)nnz, mem);
            upload(P->AT.x, ATx, (size_t)nnz, mem);
            validate_csr(n, m, nnz, P->AT, err, sms);
        }
        tm.mark("upload+validate");
        Matrix* other = haveA ? &P->AT : &P->A;
        other->p.alloc((size_t)other->rows + 1);
        other->j.alloc(std::max<int64_t>(nnz, 1));
        other->x.alloc(std::max<int64_t>(nnz, 1));
        transpose(given->rows, given->cols, nnz, given->p.p, given->j.p, given->x.p, other->p.p,
                  other->j.p, other->x.p, sms);
        tm.mark("transpose");
        if (haveA && haveAT) {
            // compare the caller's CSR(A^T) with the device transpose of CSR(A), bit for bit
            Matrix T;
            upload(T.p, ATp, (size_t)n + 1, mem);
            upload(T.j, ATj, (size_t)nnz, mem);
            upload(T.x, ATx, (size_t)nnz, mem);
            k_compare<int32_t><<<grid_of((int64_t)n + 1, sms), 256>>>((int64_t)n + 1, T.p.p, P->AT.p.p, err.p);
            if (nnz) {
                k_compare<int32_t><<<grid_of(nnz, sms), 256>>>(nnz, T.j.p, P->AT.j.p, err.p);
                k_compare<double><<<grid_of(nnz, sms), 256>>>(nnz, T.x.p, P->AT.x.p, err.p);
            }
            CPD_CUDA(cudaGetLastError());
            check_errors(err, true);
        }
        upload(P->b, b, (size_t)m, mem);
        upload(P->c, c, (size_t)n, mem);
        k_check_finite<<<grid_of(m, sms), 256>>>(m, P->b.p, err.p, ERR_B);
        k_check_finite<<<grid_of(n, sms), 256>>>(n, P->c.p, err.p, ERR_C);
        P->lb.alloc(n);
        P->ub.alloc(n);
        if (lb) CPD_CUDA(cudaMemcpy(P->lb.p, lb, sizeof(double) * n,
                                    mem == CPD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
        else k_fill<<<grid_of(n, sms), 256>>>(n, P->lb.p, 0.0);
        if (ub) CPD_CUDA(cudaMemcpy(P->ub.p, ub, sizeof(double) * n,
                                    mem == CPD_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
        else k_fill<<<grid_of(n, sms), 256>>>(n, P->ub.p, INFINITY);
        DBuf<int> flags(2);
        CPD_CUDA(cudaMemset(flags.p, 0, sizeof(int) * 2));
        k_check_bounds<<<grid_of(n, sms), 256>>>(n, P->lb.p, P->ub.p, err.p, flags.p);
        CPD_CUDA(cudaGetLastError());
        check_errors(err, false);
        int hf[2];
        CPD_CUDA(cudaMemcpy(hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost));
        P->uniform_bounds = (hf[0] == 0 && hf[1] == 0);
        if (P->uniform_bounds) {
            CPD_CUDA(cudaMemcpy(&P->l0, P->lb.p, sizeof(double), cudaMemcpyDeviceToHost));
            CPD_CUDA(cudaMemcpy(&P->u0, P->ub.p, sizeof(double), cudaMemcpyDeviceToHost));
        }
        tm.mark("vectors+bounds");
        // SpMV plans (host pass over the row pointers)
        std::vector<int32_t> hp((size_t)m + 1);
        CPD_CUDA(cudaMemcpy(hp.data(), P->A.p.p, sizeof(int32_t) * hp.size(), cudaMemcpyDeviceToHost));
        tm.mark("rowptr D2H");
        renumber(P, hp);
        tm.mark("renumber rows + columns");
        // A: warp-item plan for k_csrw unless CPD_WARP=0 (then the TMA plan of k_spmv)
        // default: warp plan when rows longer than WLONG carry >= 25% of the nonzeros
        // (C3, C5: measured faster); short-row matrices keep the TMA plan (C2, C4)
        const char* we = getenv("CPD_WARP");
        int64_t long_nnz = 0;
        for (int32_t r = 0; r < m; ++r) {
            const int64_t len = (int64_t)hp[r + 1] - hp[r];
            if (len > WLONG) long_nnz += len;
        }
        bool warpA = 4 * long_nnz >= nnz && nnz > 0;
        if (we) warpA = we[0] != '0';
        // hot-row fusion of the top rows into the primal step (renumbered problems;
        // env CPD_HOTD = rows, 0 disables; default CPD_HOTD_DEFAULT)
        const char* hde = getenv("CPD_HOTD");
        const int32_t hotd_req = P->hot > 0 ? (hde ? atoi(hde) : CPD_HOTD_DEFAULT) : 0;
        build_plan(m, n, hp, P->A.p.p, P->A.j.p, P->A.x.p, P->A.plan, warpA, hotd_req);
        build_short_sell(P->A, hp);
        tm.mark("plan A");
        // SELL-32 where the rows are short and even (padding <= 25%); CPD_SELL=0 disables
        const char* se = getenv("CPD_SELL");
        const bool sell_ok = !(se && se[0] == '0');
        // (A^T only: for A the dual epilogue's four staged vectors favour the TMA plan
        // kernel, measured on C4 — profiles/r01_kernel_iterations.md)
        if (sell_ok && nnz <= (int64_t)n * 64) build_sell(P->AT, nnz, 1.25, P->hot > 0);
        tm.mark("sell");
        // every A^T pass runs on SELL when it is on: its TMA plan is only needed otherwise
        if (!P->AT.sell.on) {
            std::vector<int32_t> htp((size_t)n + 1);   // (only here: 4n B of host memory to zero-fill)
            CPD_CUDA(cudaMemcpy(htp.data(), P->AT.p.p, sizeof(int32_t) * htp.size(), cudaMemcpyDeviceToHost));
            build_plan(n, m, htp, P->AT.p.p, P->AT.j.p, P->AT.x.p, P->AT.plan);
        } else {
            P->AT.plan.seg.assign(2, 0);
        }
        tm.mark("plan AT");
        mark_push(P);
        CPD_CUDA(cudaDeviceSynchronize());
    } catch (...) {
        delete P;
        throw;
    }
    return P;
}
