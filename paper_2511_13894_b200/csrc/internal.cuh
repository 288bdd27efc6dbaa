// internal.cuh — host-side structures of libcpd (problem, solver, execution context).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cpd.h"
#include "kernels.cuh"

namespace cpd {

// Error carried across the internal layers; converted to a cpd_error code at the ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CPD_CUDA(call)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            throw ::cpd::Error(e_ == cudaErrorMemoryAllocation ? CPD_E_NOMEM : CPD_E_CUDA,     \
                               std::string(#call) + ": " + cudaGetErrorString(e_));            \
    } while (0)

// Device-memory cache behind DBuf (devmem.cu): exact-size reuse after a device
// synchronisation, so repeated problem creations do not re-map multi-GB buffers.
cudaError_t dev_alloc(void** p, size_t bytes);
void dev_free(void* p, size_t bytes);
void dev_trim();
size_t dev_cached_bytes();

// Device buffer with RAII.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    // +64 bytes of padding: TMA bulk copies read 16-byte-aligned supersets of ranges.
    void alloc(size_t count)
    {
        free();
        n = count;
        if (count) CPD_CUDA(dev_alloc(reinterpret_cast<void**>(&p), sizeof(T) * count + 64));
    }
    void free()
    {
        if (p) dev_free(p, sizeof(T) * n + 64);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { free(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept
    {
        if (this != &o) {
            free();
            p = o.p; n = o.n; o.p = nullptr; o.n = 0;
        }
        return *this;
    }
};

// nnz-balanced SpMV plan of one CSR layout (immutable, shared by solvers).
struct Plan {
    DBuf<PlanEntry> ent;
    DBuf<int32_t> long_row, long_ptr, long_ents;
    int32_t nent = 0, nlong = 0;
    int32_t warp = 0;     // 1: warp-item plan for k_csrw (<= 32 rows / <= WCAP nnz per item)
    int32_t nfin_heavy = 0;   // long rows finished by a CTA each (long_ents = finish order)
    std::vector<int32_t> seg;   // item ranges launched separately: rows items, then one per column slab
    int32_t nheavy = 0, nhb = 0;          // heavy rows (k_dense) and column blocks of HB
    DBuf<PlanEntry> dense_ent;            // {slot, block, q0, q1} grouped by block
    DBuf<uint16_t> dense_col16;           // [nnz] column offset in the HB block of the heavy rows' entries
    DBuf<int32_t> dense_ptr;              // [nhb + 1] item range of each block
    int32_t dense_maxitems = 0;           // most items in one block (k_dense smem)
    // hot-row fusion: rows 0..hotd-1 formed by the primal step; the fused dual step's
    // dense items without them
    int32_t hotd = 0;
    int64_t hot_nnz = 0;                  // entries of rows 0..hotd-1 (the fused dual step skips them)
    DBuf<PlanEntry> dense_ent_f;
    DBuf<int32_t> dense_ptr_f;
    int32_t dense_maxitems_f = 0;
    // short rows by column slab (k_csrw slab mode): [nslab][rows + 1] pointers, entries slab-major
    int32_t short_on = 0;
    int32_t short_nslab = 1;
    int32_t short_ilv = 0;      // short slabs == piece slabs: interleave the passes
    int64_t short_width = 0;
    int64_t short_nnz = 0;
    DBuf<int32_t> short_ptr, short_col;
    DBuf<PlanEntry> short_ent;   // [nslab][seg[1]] rows items with p0/p1 in the slab-major copy
    DBuf<double> short_val;
    int64_t rows_entries = 0, single_entries = 0, long_pieces = 0;
    int32_t nslab = 1;
};
// rows x cols CSR with device column array d_col; long rows are cut into CAP pieces
// at column-slab boundaries and their pieces ordered slab-major.
void build_plan(int32_t rows, int32_t cols, const std::vector<int32_t>& rowptr, const int32_t* d_p,
                const int32_t* d_col, const double* d_val, Plan& plan, bool warp = false, int32_t hotd_req = 0);

// SELL-32 copy of a CSR layout whose rows are short and of similar length
// (DESIGN.md §6): slices of 32 consecutive rows, each padded to its longest row,
// stored column-major inside the slice so lane = row reads coalesced.
struct Sell {
    DBuf<int64_t> sp;      // [nslice + 1] slice starts (padded entries)
    DBuf<int32_t> col;     // -1 = padding
    DBuf<double> val;
    int32_t nslice = 0;
    int64_t padded = 0;
    int32_t r0 = 0, rows = 0;   // the rows [r0, r0 + rows) of the layout it holds
    int32_t c0 = 0, c1 = 0;     // c1 > c0: only their entries in columns [c0, c1)
    bool rev = false;           // each lane's entries in descending column order
    bool on = false;
};

struct Matrix {
    DBuf<int32_t> p, j;
    DBuf<double> x;
    int32_t rows = 0, cols = 0;
    Plan plan;
    Sell sell;
    Sell sell_short;   // warp plan: SELL-32 of the short-row suffix (replaces the rows items)
    Sell sell_half[2]; // or the same rows split by column half (two passes, running sums in the Ctx)
    DevCsr dev() const { return DevCsr{p.p, j.p, x.p, rows}; }
    DevSell dsell() const { return DevSell{sell.sp.p, sell.col.p, sell.val.p, rows, sell.nslice}; }
    DevSell dsell_short() const
    {
        DevSell d{sell_short.sp.p, sell_short.col.p, sell_short.val.p, sell_short.rows, sell_short.nslice};
        d.r0 = sell_short.r0;
        return d;
    }
    // half pass h: h = 0 stores its sums in buf, h = 1 starts from them
    DevSell dsell_half(int h, double* buf) const
    {
        const Sell& S = sell_half[h];
        DevSell d{S.sp.p, S.col.p, S.val.p, S.rows, S.nslice};
        d.r0 = S.r0;
        if (h == 0) d.part = buf; else d.init = buf;
        return d;
    }
};
// SELL-32 of the short-row suffix of a warp-plan layout (rows sorted by length).
void build_short_sell(Matrix& M, const std::vector<int32_t>& rp);
// Build M.sell when the padded size is at most `max_ratio` x nnz (else M.sell.on = false).
void build_sell(Matrix& M, int64_t nnz, double max_ratio, bool rev = false);

}  // namespace cpd

struct cpd_problem {
    int device = 0;
    int32_t m = 0, n = 0;
    int64_t nnz = 0;
    cpd::Matrix A, AT;
    cpd::DBuf<double> b, c, lb, ub;
    bool uniform_bounds = false;
    double l0 = 0.0, u0 = 0.0;
    int num_sms = 148;
    // solvers created on this problem and not yet destroyed: their captured graphs
    // hold device pointers of the problem, so scale / set_senses refuse while > 0
    mutable std::atomic<int> live_solvers{0};
    // ---- distribution.  Side 0 = m-side (rows of A: y, b, Ax),
    // side 1 = n-side (rows of A^T: x, c, bounds).  The local matrices are this
    // rank's block: row-block (split = 1) keeps rows R_p of A, so A has m_p rows and
    // A^T all n rows; col-block (split = 0) keeps columns C_p, so A^T has n_p rows
    // and A all m rows.  The side whose local rows are ALL rows is the split side:
    // its products are partial, reduce-scattered into equal slices of length L, and
    // its state vectors hold only the owned slice.  world == 1: split = -1.
    int world = 1, rank = 0, split = -1;
    int32_t m_glob = 0, n_glob = 0;
    int32_t own_len[2] = {0, 0};     // owned length of each side's state vectors
    int64_t poff[2] = {0, 0};        // offset of the owned part in this problem's b / c, lb, ub
    int64_t gofs[2] = {0, 0};        // global index of owned element 0
    int64_t L = 0;                   // slice length of the split side
    std::vector<int64_t> rank_gofs[2], rank_len[2];   // every rank's owned part (global)
    void* comm = nullptr;            // ncclComm_t (split >= 0)
    // ---- hot-row renumbering: internal row k of A = user row rperm[k];
    // the first `hot` internal rows are the longest (their y entries staged in smem)
    cpd::DBuf<int32_t> rperm;
    std::vector<int32_t> h_rperm;
    int32_t hot = 0;
    // ---- column renumbering: internal column k = user column cperm[k]
    // (empty: the user's order); every n-vector crossing the ABI is mapped
    cpd::DBuf<int32_t> cperm;
    // ---- short-row push: SELL(A^T) entries of short rows flagged
    bool push_on = false;
    int64_t push_nnz = 0;
    // ---- row senses (cpd_problem_set_senses; NEXT-2): local rows of A, null = all '='
    cpd::DBuf<int8_t> sense;
    bool has_sense = false;
    const int8_t* sense_own() const { return has_sense ? sense.p + poff[0] : nullptr; }
    // ---- diagonal preconditioning (cpd_problem_scale; R-3): the device LP is
    // the scaled one (A^ = diag(r) A diag(s), b^ = r b, c^ = s c, l^ = l/s, u^ = u/s);
    // sr = r, ss = s, ir = 1/r, is = 1/s; lb0/ub0 the original bounds.  Unscaled: nulls.
    bool scaled = false;
    cpd::DBuf<double> sr, ss, ir, is, lb0, ub0;
    bool uniform0 = false;
    double l00 = 0.0, u00 = 0.0;
    const double* w_m() const { return scaled ? ir.p : nullptr; }
    const double* w_n() const { return scaled ? is.p : nullptr; }
    const double* s_n() const { return scaled ? ss.p : nullptr; }
    // original bounds of the owned n-side part
    cpd::Bounds bounds_orig() const
    {
        if (!scaled) return bounds_own();
        if (uniform0) return cpd::Bounds{nullptr, nullptr, l00, u00};
        return cpd::Bounds{lb0.p, ub0.p, 0.0, 0.0};
    }
    cpd::Bounds bounds() const
    {
        if (uniform_bounds) return cpd::Bounds{nullptr, nullptr, l0, u0};
        return cpd::Bounds{lb.p, ub.p, 0.0, 0.0};
    }
    // bounds of the owned n-side part
    cpd::Bounds bounds_own() const
    {
        if (uniform_bounds) return cpd::Bounds{nullptr, nullptr, l0, u0};
        return cpd::Bounds{lb.p + poff[1], ub.p + poff[1], 0.0, 0.0};
    }
    const double* b_own() const { return b.p + poff[0]; }
    const double* c_own() const { return c.p + poff[1]; }
    ~cpd_problem();
};

namespace cpd {

// Per-stream execution context: control block, reduction scratch, long-row
// scratch for both layouts.
bool fuse_ok(const cpd_problem* P);   // hot-row fusion applies (solver.cu)

struct Ctx {
    const cpd_problem* P = nullptr;
    cudaStream_t st = nullptr;
    // the dual step's heavy-row dense blocks run on `side`, concurrently with the other
    // sub-kernels (DRAM-bound next to L2-bound), forked / joined with events on `st`
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool conc = false;   // CPD_CONC=1: measured neutral to -13% next to the 16-bit k_dense
    double dense_frac = 0.5;
    DBuf<Ctl> ctl_main, ctl_aux;      // run control block / scratch block for one-off evaluations
    Ctl* h_main = nullptr;           // pinned mirrors
    Ctl* h_aux = nullptr;
    Ctl* ctl = nullptr;              // active block (main unless an AuxScope is open)
    Ctl* h_ctl = nullptr;
    DBuf<double> bpart;
    DBuf<unsigned> ctr;
    DBuf<double> lpartA, lpartAT;     // long-row piece partials of each layout
    DBuf<double> shortA, shortAT;     // running row sums of the short-row slab passes
    DBuf<double> sshortA;             // running row sums of the short-row SELL half passes
    double* push_acc = nullptr;       // set around the primal/dual pair of a batch (short-row push)
    DBuf<double> hotpart;             // hot-row fusion: per-warp partials [hotd][hot_stride]
    int32_t hot_stride = 0;
    bool fuse = false;                // set around the primal/dual pair of a batch (hot-row fusion)
    DBuf<double> red;                 // this rank's totals of the last reduction (distributed)
    DBuf<double> part, recv;          // reduce-scatter send [world][2][L] / receive [2][L] buffers
    // fused split product (CPD_P2P=1): symmetric receive window [world][2][L] and the
    // device table of every rank's window base
    bool p2p = false;
    void* win = nullptr;              // ncclWindow_t
    double* winbuf = nullptr;         // ncclMemAlloc'ed
    DBuf<double*> peer;
    void p2p_setup();
    void p2p_teardown();
    int grid_elem = 0;
    int64_t launches = 0;            // kernels of this library launched on `st` (graph nodes included)
    explicit Ctx(const cpd_problem* p);
    ~Ctx();
    DevPlan planA() const;
    DevPlan planA_fused() const;
    DevPlan planAT() const;
    void pull_ctl();                                   // D2H of the control block + sync
    void set_i64(int64_t* dev_field, int64_t v);
    void set_i32(int32_t* dev_field, int32_t v);
    void push_ctl(const Ctl& h);                      // H2D of a whole control block
    void sync();
    template <class F>
    int grid_for(F kernel);
    // collectives on the problem's communicator, on `st` (no-ops when split < 0)
    void allreduce_sum(double* buf, int64_t count);
    void allreduce_max_host(double* v);                // host scalar, synchronous
    void reduce_scatter(const double* send, double* recv, int64_t count);
    void all_gather_inplace(double* buf, int64_t count);   // buf[world * count], own chunk at rank * count
    void all_gather(const double* send, double* recv, int64_t count);
};

// Launch helpers (templates instantiated in solver.cu).
// Switches a Ctx to its auxiliary control block for the scope's lifetime, so
// one-off evaluations never disturb the state of a run in progress.
struct AuxScope {
    Ctx& cx;
    explicit AuxScope(Ctx& c) : cx(c) { cx.ctl = cx.ctl_aux.p; cx.h_ctl = cx.h_aux; }
    ~AuxScope() { cx.ctl = cx.ctl_main.p; cx.h_ctl = cx.h_main; }
};

template <int NV, class Epi>
void launch_spmv(Ctx& cx, const Matrix& M, const DevPlan& dp, VecSel v0, VecSel v1, const Epi& epi,
                 Gate g, double* red = nullptr);
template <class Op>
void launch_elem(Ctx& cx, int64_t N, const Op& op, Gate g, double* red = nullptr);

extern thread_local bool g_no_renumber;   // set by cpd_problem_create_dist around the local create

// diagonal preconditioning of a problem (problem.cu)
void scale_problem(cpd_problem* P, int32_t ruiz_iters, int32_t pc);
// flag the short-row entries of SELL(A^T) for the push (problem.cu)
void mark_push(cpd_problem* P);

// distributed problem plumbing (dist.cu)
void dist_destroy(cpd_problem* P);

}  // namespace cpd
