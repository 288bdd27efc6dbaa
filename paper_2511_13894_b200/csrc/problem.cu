// problem.cu — cpd_problem: device copies, device-side validation, device
// transpose (stable radix sort by column), uniform-bound detection, SpMV plans.
// The problem statement is P:64-92 (A m x n, b, c, bounds handled implicitly).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

namespace cpd {

// ------------------------------------------------------------------ plans
// Stream entries: consecutive rows with <= CAP nonzeros and <= RMAX rows; rows
// longer than CAP become ceil(len/CAP) long-row chunks.  Threads per row in a
// stream entry: smallest power of two with ~<= 4 nonzeros per thread (<= 32).
void build_plan(int32_t rows, const std::vector<int32_t>& rp, Plan& plan)
{
    std::vector<PlanEntry> ent;
    std::vector<int64_t> loff;
    int64_t chunks = 0, nstream = 0, nlongent = 0;
    int32_t r0 = 0;
    int64_t cur = 0;
    auto flush = [&](int32_t r1) {
        if (r1 > r0) {
            const int nr = r1 - r0;
            const double avg = (double)cur / nr;
            int lg = 0;
            while (lg < 5 && (double)(1 << lg) * 4.0 < avg) ++lg;
            ent.push_back(PlanEntry{r0, r1, lg, -1});
            ++nstream;
        }
    };
    for (int32_t r = 0; r < rows; ++r) {
        const int64_t len = (int64_t)rp[r + 1] - rp[r];
        if (len > CAP) {
            flush(r);
            const int32_t nch = (int32_t)((len + CAP - 1) / CAP);
            const int32_t lid = (int32_t)loff.size();
            loff.push_back(chunks);
            chunks += nch;
            for (int32_t c = 0; c < nch; ++c) ent.push_back(PlanEntry{r, c, -1, lid});
            nlongent += nch;
            r0 = r + 1;
            cur = 0;
            continue;
        }
        if (cur + len > CAP || (r - r0) >= RMAX) {
            flush(r);
            r0 = r;
            cur = 0;
        }
        cur += len;
    }
    flush(rows);
    if (ent.size() > (size_t)INT32_MAX) throw Error(CPD_E_DIM, "plan too large");
    plan.nent = (int32_t)ent.size();
    plan.nlong = (int32_t)loff.size();
    plan.chunks = chunks;
    plan.stream_entries = nstream;
    plan.long_entries = nlongent;
    plan.ent.alloc(std::max<size_t>(ent.size(), 1));
    CPD_CUDA(cudaMemcpy(plan.ent.p, ent.data(), sizeof(PlanEntry) * ent.size(), cudaMemcpyHostToDevice));
    plan.long_off.alloc(std::max<size_t>(loff.size(), 1));
    if (!loff.empty())
        CPD_CUDA(cudaMemcpy(plan.long_off.p, loff.data(), sizeof(int64_t) * loff.size(),
                            cudaMemcpyHostToDevice));
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

__global__ void k_count(int64_t nnz, const int32_t* j, int32_t* cnt)
{
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
         q += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[j[q]], 1);
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
        perm(std::max<int64_t>(nnz, 1)), cnt((size_t)cols + 1);
    CPD_CUDA(cudaMemset(cnt.p, 0, sizeof(int32_t) * ((size_t)cols + 1)));
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
        k_count<<<grid_of(nnz, sms), 256>>>(nnz, j, cnt.p + 1);
        k_gather_transpose<<<grid_of(nnz, sms), 256>>>(rows, nnz, p, x, perm.p, tj, tx);
    }
    size_t scan_bytes = 0;
    CPD_CUDA(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, cnt.p, tp, cols + 1));
    DBuf<unsigned char> stmp(scan_bytes);
    CPD_CUDA(cub::DeviceScan::InclusiveSum(stmp.p, scan_bytes, cnt.p, tp, cols + 1));
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

using namespace cpd;

// Implementation of cpd_problem_create (called from the ABI layer).
cpd_problem* cpd_problem_create_impl(int32_t m, int32_t n, int64_t nnz, const int32_t* Ap,
                                     const int32_t* Aj, const double* Ax, const int32_t* ATp,
                                     const int32_t* ATj, const double* ATx, const double* b,
                                     const double* c, const double* lb, const double* ub,
                                     int32_t mem, int32_t device)
{
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
        Matrix* other = haveA ? &P->AT : &P->A;
        other->p.alloc((size_t)other->rows + 1);
        other->j.alloc(std::max<int64_t>(nnz, 1));
        other->x.alloc(std::max<int64_t>(nnz, 1));
        transpose(given->rows, given->cols, nnz, given->p.p, given->j.p, given->x.p, other->p.p,
                  other->j.p, other->x.p, sms);
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
        // SpMV plans (host pass over the row pointers)
        std::vector<int32_t> hp((size_t)m + 1), htp((size_t)n + 1);
        CPD_CUDA(cudaMemcpy(hp.data(), P->A.p.p, sizeof(int32_t) * hp.size(), cudaMemcpyDeviceToHost));
        CPD_CUDA(cudaMemcpy(htp.data(), P->AT.p.p, sizeof(int32_t) * htp.size(), cudaMemcpyDeviceToHost));
        build_plan(m, hp, P->A.plan);
        build_plan(n, htp, P->AT.plan);
        CPD_CUDA(cudaDeviceSynchronize());
    } catch (...) {
        delete P;
        throw;
    }
    return P;
}
