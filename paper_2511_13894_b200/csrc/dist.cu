// dist.cu — multi-GPU plumbing: partition of the LP
// over ranks, extraction of this rank's block, the NCCL communicator and the
// collectives the passes use.  One process per GPU; the 128-byte NCCL id is
// broadcast by the caller (torch.distributed), so the library needs no launcher.
//
// Scheme ("shard the long vector, exchange the short one"):
//   partition 0 = row-block (north_star): rank p keeps rows R_p of A (nnz-balanced),
//       y/b/Ax sharded with them; A^T y is partial on every rank -> reduce-scatter
//       into equal slices of the n-side, primal step on the slice, all-gather x+.
//   partition 1 = col-block: rank p keeps columns C_p (nnz-balanced), x/c/bounds
//       sharded with them; A x+ is partial -> reduce-scatter into equal slices of
//       the m-side, dual step on the slice, all-gather y+.
// Scalars (norms, dots, counts) are allreduced before every device decision.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

#ifdef CPD_HAVE_NCCL
#include <nccl.h>
#include <nccl_device.h>
#endif
#include <cstdlib>

cpd_problem* cpd_problem_create_impl(int32_t m, int32_t n, int64_t nnz, const int32_t* Ap,
                                     const int32_t* Aj, const double* Ax, const int32_t* ATp,
                                     const int32_t* ATj, const double* ATx, const double* b,
                                     const double* c, const double* lb, const double* ub,
                                     int32_t mem, int32_t device);

namespace cpd {

#ifdef CPD_HAVE_NCCL
#define CPD_NCCL(call)                                                                        \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) throw ::cpd::Error(CPD_E_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)
static ncclComm_t comm_of(const cpd_problem* P) { return (ncclComm_t)P->comm; }
#endif

void dist_destroy(cpd_problem* P)
{
#ifdef CPD_HAVE_NCCL
    if (P->comm) ncclCommDestroy((ncclComm_t)P->comm);
#endif
    P->comm = nullptr;
}

#ifdef CPD_HAVE_NCCL
// base of every rank's receive window (NCCL symmetric memory, LSA over NVLink)
__global__ void k_peer_bases(ncclWindow_t w, int world, double** out)
{
    for (int q = threadIdx.x; q < world; q += blockDim.x) out[q] = (double*)ncclGetPeerPointer(w, 0, q);
}
#endif

void Ctx::p2p_setup()
{
    const char* e = getenv("CPD_P2P");
    if (P->split < 0 || !(e && e[0] == '1')) return;
#ifdef CPD_HAVE_NCCL
    const size_t bytes = ((size_t)P->world * 2 * P->L * sizeof(double) + 4095) & ~(size_t)4095;
    void* buf = nullptr;
    CPD_NCCL(ncclMemAlloc(&buf, bytes));
    winbuf = (double*)buf;
    CPD_CUDA(cudaMemset(winbuf, 0, bytes));
    ncclWindow_t w;
    CPD_NCCL(ncclCommWindowRegister(comm_of(P), buf, bytes, &w, NCCL_WIN_COLL_SYMMETRIC));
    win = w;
    peer.alloc(P->world);
    k_peer_bases<<<1, 32, 0, st>>>(w, P->world, peer.p);
    CPD_CUDA(cudaGetLastError());
    CPD_CUDA(cudaStreamSynchronize(st));
    p2p = true;
#endif
}

void Ctx::p2p_teardown()
{
#ifdef CPD_HAVE_NCCL
    if (win) ncclCommWindowDeregister(comm_of(P), (ncclWindow_t)win);
    if (winbuf) ncclMemFree(winbuf);
#endif
    win = nullptr;
    winbuf = nullptr;
    p2p = false;
}

void Ctx::allreduce_sum(double* buf, int64_t count)
{
    if (P->split < 0) return;
#ifdef CPD_HAVE_NCCL
    CPD_NCCL(ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, comm_of(P), st));
#else
    throw Error(CPD_E_NCCL, "built without NCCL");
#endif
}

void Ctx::allreduce_max_host(double* v)
{
    if (P->split < 0) return;
#ifdef CPD_HAVE_NCCL
    DBuf<double> d(1);
    CPD_CUDA(cudaMemcpyAsync(d.p, v, sizeof(double), cudaMemcpyHostToDevice, st));
    CPD_NCCL(ncclAllReduce(d.p, d.p, 1, ncclDouble, ncclMax, comm_of(P), st));
    CPD_CUDA(cudaMemcpyAsync(v, d.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    CPD_CUDA(cudaStreamSynchronize(st));
#endif
}

void Ctx::reduce_scatter(const double* send, double* rv, int64_t count)
{
#ifdef CPD_HAVE_NCCL
    CPD_NCCL(ncclReduceScatter(send, rv, (size_t)count, ncclDouble, ncclSum, comm_of(P), st));
#else
    throw Error(CPD_E_NCCL, "built without NCCL");
#endif
}

void Ctx::all_gather_inplace(double* buf, int64_t count)
{
#ifdef CPD_HAVE_NCCL
    CPD_NCCL(ncclAllGather(buf + (int64_t)P->rank * count, buf, (size_t)count, ncclDouble, comm_of(P), st));
#else
    throw Error(CPD_E_NCCL, "built without NCCL");
#endif
}

void Ctx::all_gather(const double* send, double* rv, int64_t count)
{
#ifdef CPD_HAVE_NCCL
    CPD_NCCL(ncclAllGather(send, rv, (size_t)count, ncclDouble, comm_of(P), st));
#else
    throw Error(CPD_E_NCCL, "built without NCCL");
#endif
}

// Contiguous blocks of rows with weights w_r = len_r + 1 (nonzeros plus the
// row's vector work), balanced: bounds[q] = first row whose prefix weight reaches
// q W / world; every block non-empty.
static std::vector<int64_t> balanced_blocks(const std::vector<int64_t>& len, int world)
{
    const int64_t R = (int64_t)len.size();
    std::vector<int64_t> pre(R + 1, 0);
    for (int64_t r = 0; r < R; ++r) pre[r + 1] = pre[r] + len[r] + 1;
    const double W = (double)pre[R];
    std::vector<int64_t> bnd(world + 1, 0);
    bnd[world] = R;
    for (int q = 1; q < world; ++q) {
        const double target = W * q / world;
        int64_t r = std::lower_bound(pre.begin(), pre.end(), (int64_t)std::ceil(target)) - pre.begin();
        r = std::max<int64_t>(r, bnd[q - 1] + 1);
        r = std::min<int64_t>(r, R - (world - q));
        bnd[q] = r;
    }
    return bnd;
}

// Slice / block layout of one rank, shared by cpd_problem_create_dist
// and the host-only cpd_dist_layout: `bnd` = the partition's block bounds.  Side 0 =
// m-side (rows of A), side 1 = n-side (rows of A^T).  The split side (the one whose
// local rows are ALL rows: n-side for row-block, m-side for col-block) is cut into
// `world` equal slices of L = ceil(rows / world) (the last ones shorter, possibly
// empty); the other side is owned by blocks.  poff = offset of the owned part inside
// the rank's local arrays (the local problem holds every row of the split side).
struct DistLayout {
    int split;
    int64_t L;
    std::vector<int64_t> gofs[2], len[2];   // per rank
};
static DistLayout dist_layout(int32_t m, int32_t n, int world, int partition, const std::vector<int64_t>& bnd)
{
    DistLayout d;
    d.split = partition == 0 ? 1 : 0;
    const int64_t rows_split = d.split == 1 ? n : m;
    d.L = (rows_split + world - 1) / world;
    for (int s = 0; s < 2; ++s) {
        d.gofs[s].assign(world, 0);
        d.len[s].assign(world, 0);
        for (int q = 0; q < world; ++q) {
            if (s == d.split) {
                const int64_t o = std::min<int64_t>((int64_t)q * d.L, rows_split);
                d.gofs[s][q] = o;
                d.len[s][q] = std::min<int64_t>(d.L, rows_split - o);
            } else {
                d.gofs[s][q] = bnd[q];
                d.len[s][q] = bnd[q + 1] - bnd[q];
            }
        }
    }
    return d;
}

}  // namespace cpd

using namespace cpd;

extern "C" {

/* see include/cpd.h */
int cpd_dist_layout(int32_t m, int32_t n, const int32_t* AT_rowptr, const int32_t* AT_col, int32_t world,
                    int32_t partition, int32_t rank, int64_t out[12])
{
    if (!out || world < 1 || rank < 0 || rank >= world) return CPD_E_ARG;
    if (partition < 0) partition = (n >= m) ? 1 : 0;
    std::vector<int64_t> bnd(world + 1);
    const int rc = cpd_partition(m, n, AT_rowptr, AT_col, world, partition, bnd.data());
    if (rc != CPD_OK) return rc;
    const DistLayout d = dist_layout(m, n, world, partition, bnd);
    out[0] = partition;
    out[1] = d.split;
    out[2] = d.L;
    out[3] = bnd[rank];
    out[4] = bnd[rank + 1];
    for (int s = 0; s < 2; ++s) {
        out[5 + s] = d.len[s][rank];
        out[7 + s] = d.gofs[s][rank];
        out[9 + s] = (s == d.split) ? d.gofs[s][rank] : 0;
    }
    out[11] = partition == 1 ? (bnd[rank + 1] - bnd[rank]) : n;   // local rows of A^T
    return CPD_OK;
}

/* see include/cpd.h */
int cpd_partition(int32_t m, int32_t n, const int32_t* AT_rowptr, const int32_t* AT_col, int32_t world,
                  int32_t partition, int64_t* bounds)
{
    try {
        if (!AT_rowptr || !bounds || world < 1 || m < 1 || n < 1 || (partition != 0 && partition != 1))
            return CPD_E_ARG;
        if (world > std::min(m, n)) return CPD_E_ARG;
        std::vector<int64_t> len;
        if (partition == 1) {   // column blocks: column j = row j of A^T
            len.resize(n);
            for (int32_t j = 0; j < n; ++j) len[j] = (int64_t)AT_rowptr[j + 1] - AT_rowptr[j];
        } else {                // row blocks: row counts of A
            if (!AT_col && AT_rowptr[n] > 0) return CPD_E_ARG;
            len.assign(m, 0);
            const int64_t nnz = AT_rowptr[n];
            for (int64_t q = 0; q < nnz; ++q) {
                const int32_t i = AT_col[q];
                if (i < 0 || i >= m) return CPD_E_CSR;
                len[i] += 1;
            }
        }
        const std::vector<int64_t> b = balanced_blocks(len, world);
        std::copy(b.begin(), b.end(), bounds);
    } catch (...) {
        return CPD_E_ARG;
    }
    return CPD_OK;
}

int cpd_nccl_get_unique_id(char id[128])
{
#ifdef CPD_HAVE_NCCL
    if (!id) return CPD_E_ARG;
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return CPD_E_NCCL;
    static_assert(sizeof(u) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(id, &u, 128);
    return CPD_OK;
#else
    (void)id;
    return CPD_E_NCCL;
#endif
}

}  // extern "C"

// Called from the ABI layer in solver.cu (error text via its cpd_last_error).
cpd_problem* cpd_problem_create_dist_impl(int32_t rank, int32_t world, const char id[128], int32_t partition,
                                          int32_t m, int32_t n, int64_t nnz, const int32_t* ATp,
                                          const int32_t* ATj, const double* ATx, const double* b,
                                          const double* c, const double* lb, const double* ub, int32_t device)
{
    if (world < 1 || rank < 0 || rank >= world) throw Error(CPD_E_ARG, "need 0 <= rank < world");
    if (m < 1 || n < 1 || nnz < 0 || nnz >= (1LL << 31)) throw Error(CPD_E_DIM, "need m >= 1, n >= 1, 0 <= nnz < 2^31");
    if (world > std::min(m, n)) throw Error(CPD_E_DIM, "world size exceeds min(m, n)");
    if (!ATp || (nnz > 0 && (!ATj || !ATx)) || !b || !c || !id) throw Error(CPD_E_ARG, "NULL argument");
    if ((int64_t)ATp[n] != nnz || ATp[0] != 0) throw Error(CPD_E_CSR, "AT_rowptr does not span [0, nnz]");
    if (partition < 0) partition = (n >= m) ? 1 : 0;   // shard the long side
    if (partition > 1) throw Error(CPD_E_ARG, "partition must be -1, 0 (row-block) or 1 (col-block)");
    std::vector<int64_t> bnd(world + 1);
    int rc = cpd_partition(m, n, ATp, ATj, world, partition, bnd.data());
    if (rc != CPD_OK) throw Error(rc, "partition failed (bad CSR(A^T))");
    const int split = partition == 0 ? 1 : 0;
    const int64_t rows_split = split == 1 ? n : m;
    const int64_t L = (rows_split + world - 1) / world;
    const int64_t b0 = bnd[rank], b1 = bnd[rank + 1];

    cpd_problem* P = nullptr;
    struct NoRenumber {   // the local block keeps the user's row order (gofs mapping)
        NoRenumber() { cpd::g_no_renumber = true; }
        ~NoRenumber() { cpd::g_no_renumber = false; }
    } nr_guard;
    if (partition == 1) {
        // columns [b0, b1): rows b0..b1 of CSR(A^T), global row indices of A
        std::vector<int32_t> p((size_t)(b1 - b0) + 1);
        for (int64_t j = b0; j <= b1; ++j) p[j - b0] = ATp[j] - ATp[b0];
        const int64_t nz = p.back();
        P = cpd_problem_create_impl(m, (int32_t)(b1 - b0), nz, nullptr, nullptr, nullptr, p.data(),
                                    nz ? ATj + ATp[b0] : nullptr, nz ? ATx + ATp[b0] : nullptr, b, c + b0,
                                    lb ? lb + b0 : nullptr, ub ? ub + b0 : nullptr, CPD_HOST, device);
    } else {
        // rows [b0, b1) of A: keep those entries of every column, local row index
        std::vector<int32_t> p((size_t)n + 1, 0), j;
        std::vector<double> x;
        for (int32_t col = 0; col < n; ++col) {
            for (int64_t q = ATp[col]; q < ATp[col + 1]; ++q) {
                const int32_t i = ATj[q];
                if (i >= b0 && i < b1) {
                    j.push_back((int32_t)(i - b0));
                    x.push_back(ATx[q]);
                }
            }
            p[col + 1] = (int32_t)j.size();
        }
        const int64_t nz = (int64_t)j.size();
        P = cpd_problem_create_impl((int32_t)(b1 - b0), n, nz, nullptr, nullptr, nullptr, p.data(),
                                    nz ? j.data() : nullptr, nz ? x.data() : nullptr, b + b0, c, lb, ub, CPD_HOST,
                                    device);
    }
    try {
        P->world = world;
        P->rank = rank;
        P->split = split;
        P->push_on = false;   // the short-row push is a single-GPU path
        P->m_glob = m;
        P->n_glob = n;
        P->L = L;
        const DistLayout d = dist_layout(m, n, world, partition, bnd);
        for (int s = 0; s < 2; ++s) {
            P->rank_gofs[s] = d.gofs[s];
            P->rank_len[s] = d.len[s];
            P->own_len[s] = (int32_t)P->rank_len[s][rank];
            P->gofs[s] = P->rank_gofs[s][rank];
            P->poff[s] = (s == split) ? P->gofs[s] : 0;   // the local problem holds all rows of the split side
        }
#ifdef CPD_HAVE_NCCL
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        ncclComm_t comm;
        CPD_CUDA(cudaSetDevice(device));
        CPD_NCCL(ncclCommInitRank(&comm, world, u, rank));
        P->comm = comm;
#else
        throw Error(CPD_E_NCCL, "built without NCCL");
#endif
    } catch (...) {
        delete P;
        throw;
    }
    return P;
}

cpd_problem::~cpd_problem() { cpd::dist_destroy(this); }
