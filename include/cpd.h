/*
 * cpd.h — C ABI of the B200-native restarted-PDHG + corner-push hot path
 * (arXiv 2511.13894, "Corner push PDHG").  Library: paper_2511_13894_b200/libcpd.so
 *
 * The problem:   min c^T x  s.t.  A x = b,  lb <= x <= ub
 * with its dual            max b^T y (+ bound terms)  s.t.  A^T y + z = c,
 * bounds handled implicitly by projection.  Residuals r_P = b - Ax,
 * r_D = c - A^T y - z; termination by the three relative tests of
 * P:119-131; the iteration is R-PDHG;
 * the steering phase is Algorithm 1 with the early stop of
 * P:391-395; the corner statistics are those of P:200-210 and P:438-452.
 *
 * Conventions
 *  - Every function returns int: CPD_OK (0) or a negative cpd_error.  No C++
 *    exception crosses the ABI.  cpd_last_error() gives a thread-local message
 *    for the last failing call on that thread.
 *  - Solve OUTCOMES (converged / iteration limit / ...) are cpd_status values in
 *    cpd_result.status, not errors.
 *  - Arrays passed in are BORROWED for the duration of the call and copied; the
 *    library never keeps a caller pointer.  Output arrays are caller-allocated.
 *  - `mem` arguments say where caller arrays live: CPD_HOST (any host memory;
 *    page-locked memory copies faster) or CPD_DEVICE (device pointers on the
 *    problem's device).
 *  - Indices are int32 (nnz < 2^31), values fp64 (IEEE binary64); all device
 *    arithmetic is fp64.
 *  - Handles are not thread-safe; distinct handles may be used from distinct
 *    threads.  Each handle lives on one CUDA device and owns one stream.
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    needs one fails with CPD_E_CUDA.
 */
#ifndef CPD_H
#define CPD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define CPD_VERSION 1

enum cpd_error {
    CPD_OK = 0,
    CPD_E_ARG = -1,        /* NULL handle/pointer, bad enum, bad parameter value */
    CPD_E_DIM = -2,        /* m < 1, n < 1, nnz < 0 or nnz >= 2^31 */
    CPD_E_BOUNDS = -3,     /* lb_j > ub_j, NaN bound, lb_j = +inf or ub_j = -inf (j in message) */
    CPD_E_CSR = -4,        /* bad rowptr, column out of range, unsorted/duplicate column in a
                              row, explicit zero, or CSR(A) and CSR(A^T) disagree */
    CPD_E_NONFINITE = -5,  /* NaN/Inf in A, b or c (only bounds may be infinite) */
    CPD_E_CUDA = -6,       /* CUDA runtime error (message has the CUDA error string) */
    CPD_E_NCCL = -7,       /* NCCL error */
    CPD_E_STATE = -8,      /* call not valid in the handle's state (e.g. scale while a solver is alive) */
    CPD_E_NOMEM = -9       /* device allocation failed */
};

enum cpd_status {
    CPD_RUNNING = -1,
    CPD_CONVERGED = 0,
    CPD_ITER_LIMIT = 1,
    CPD_TIME_LIMIT = 2,
    CPD_NUMERICAL_FAILURE = 3  /* non-finite iterate; `iterations` = first offending iteration */
};

enum cpd_mem { CPD_HOST = 0, CPD_DEVICE = 1 };

const char *cpd_last_error(void);
int cpd_version(void);

typedef struct cpd_problem cpd_problem;   /* owns device copies of A (both layouts), b, c, lb, ub */
typedef struct cpd_solver cpd_solver;     /* owns iterate, workspace, stream, CUDA graphs */

/* Create a problem on `device`.
 *  CSR(A):   A_rowptr[m+1], A_col[nnz], A_val[nnz]     (row i of A)
 *  CSR(A^T): AT_rowptr[n+1], AT_col[nnz], AT_val[nnz]  (row j of A^T = column j of A)
 *  Either layout may be omitted (all three pointers NULL); the library then builds
 *  it on the device by a stable transpose.  If both are given they are checked to
 *  be the same matrix, bit for bit.  Within each row column indices must be
 *  strictly increasing (this is how duplicates are excluded) and values nonzero.
 *  b[m], c[n] finite.  lb[n], ub[n]: NULL => lb = 0, ub = +inf; entries may be
 *  -inf / +inf respectively; lb_j <= ub_j.
 *  Validation runs on the device; on failure *out is untouched and the message
 *  names the first offending index.  The library may store the rows of A in
 *  another order internally (hot-row renumbering); every vector in or
 *  out of the ABI is in the caller's order. */
int cpd_problem_create(int32_t m, int32_t n, int64_t nnz,
                       const int32_t *A_rowptr, const int32_t *A_col, const double *A_val,
                       const int32_t *AT_rowptr, const int32_t *AT_col, const double *AT_val,
                       const double *b, const double *c, const double *lb, const double *ub,
                       int32_t mem, int32_t device, cpd_problem **out);
int cpd_problem_destroy(cpd_problem *p);
/* m, n, nnz, number of long (split) rows in each layout's SpMV plan. */
int cpd_problem_info(const cpd_problem *p, int64_t info[8]);
/* Which SpMV engine paths the problem's plans use, for tests and
 * diagnostics: out[16] = {A warp plan (k_csrw) 1/0, A heavy rows (k_dense), A dense
 * column blocks, A column slabs of the long pieces, A short-row slab passes
 * (0 = off), A long rows, A long pieces, A rows items, A^T SELL-32 1/0, hot rows
 * (renumbered), A TMA plan entries (k_spmv), columns renumbered 1/0, fused hot rows
 * (hot-row fusion: the primal step forms their dual-step products; 0 = off), 0, 0, 0}.
 * Renumbering is internal: every vector in or out of the ABI is in the caller's order. */
int cpd_problem_plan_info(const cpd_problem *p, int64_t out[16]);

/* Solver parameters (every constant of the R-PDHG reading, §8(c)). */
typedef struct {
    double eps_rel;        /* 1e-4: relative tolerance of P:124-126 */
    double eps_abs;        /* 1e-6: classification tolerance */
    int64_t max_iters;     /* iteration limit (status CPD_ITER_LIMIT) */
    double time_limit_s;   /* <= 0: none; checked between launch batches */
    int32_t check_every;   /* K = 64: restart-check cadence, 1..1024 */
    double step_scale;     /* 0.9: eta = step_scale / sigma_hat */
    double step_size;      /* > 0: eta given explicitly (parity runs); else power iteration */
    int32_t power_iters;   /* 128: K_pow */
    uint64_t seed;         /* 7: power-iteration start vector U(seed, j) - 0.5 */
    double primal_weight;  /* > 0: omega0 given; else ||c||/||b|| (1 if either < 1e-10) */
    int32_t restart;       /* 0 none, 1 adaptive restart to average/current */
    double beta_suff, beta_nec, beta_art, theta;   /* 0.2, 0.8, 0.36, 0.5 */
    int32_t use_graph;     /* 1: CUDA-graph batches of K iterations (default); 0: eager launches */
    int32_t profile;       /* 1: CUDA events around every hot kernel (cpd_get_kernel_times) */
    /* NEXT-1 (the cuPDLP+ lineage of the paper's PDHG; readings H-1..H-4) */
    int32_t method;        /* 0: R-PDHG (restart to average / current); 1: reflected restarted
                              Halpern PDHG: z+ = l((1+reflection) T(z) - reflection z) + (1-l) z_anchor,
                              l = (t+1)/(t+2), restarts on the fixed-point residual ||z - T(z)||_M,
                              termination and the returned point are those of T(z) (single GPU only) */
    double reflection;     /* 1.0 */
    int32_t pid;           /* 1: PID primal weight at restarts on e = log(dy/dx) - log omega */
    double kp, ki, kd;     /* 0.99, 0.01, 0: PID gains (log omega += kp e + ki sum e + kd (e - e_prev)) */
} cpd_params;
void cpd_params_default(cpd_params *p);

typedef struct {
    int32_t status;            /* cpd_status */
    int32_t returned_average;  /* 1: the returned point is the running average (S-4) */
    int64_t iterations, restarts;
    double pobj, dobj, gap, rp_norm, rd_norm, score, step_size, primal_weight, wall_s;
} cpd_result;

typedef struct {
    int64_t off_bound;          /* #{j: x_j - lb_j > eps_abs and ub_j - x_j > eps_abs} (Fig. 1) */
    int64_t off_bound_strict;   /* same with tolerance 0 */
    int64_t off_bound_model;    /* same w.r.t. the corner model's bounds (lb^, ub^) */
    int64_t zero_rc;            /* d = #{|z_j| <= eps_abs} */
    int64_t candidates;         /* #{off-bound and |z_j| < eps_abs} */
    int64_t fix_lb, fix_ub;     /* Algorithm 1 bound-map counts */
    int64_t est_primal_pushes;  /* max(p - m, 0) */
    int64_t est_dual_pushes;    /* max(m - d, 0) */
    int32_t is_candidate;       /* candidates >= max(2m, floor) */
    int64_t rows_eq;            /* inequality rows the corner model made '=' */
} cpd_stats;

typedef struct {
    double eps_abs;            /* 1e-6: Algorithm 1 threshold */
    double obj_scale;          /* 1.0: obj = obj_scale * Uniform[0,1)^n */
    uint64_t seed;             /* objective seed: obj_j = obj_scale * U(seed, j) */
    const double *obj;         /* NULL: generate on device; else caller objective [n] in `obj_mem` */
    int32_t obj_mem;           /* cpd_mem of `obj` */
    int64_t min_iters;         /* 100 */
    int64_t max_iters;
    double time_limit_s;
    int32_t traj_every;        /* record (k, off_bound, ||r_P||) every K iterations if > 0 */
    int64_t candidate_floor;   /* 100000 */
} cpd_corner_params;
void cpd_corner_params_default(cpd_corner_params *p);

int cpd_solver_create(const cpd_problem *p, const cpd_params *prm, cpd_solver **out);
int cpd_solver_destroy(cpd_solver *s);

/* Phase 1: R-PDHG from the solver's current iterate (zeros after
 * create or cpd_set_iterate(NULL, NULL)) to eps_rel or a limit.  Afterwards the
 * current iterate is the returned point (x, y). */
int cpd_solve(cpd_solver *s, cpd_result *out);

/* Steering phase = Algorithm 1 after a cpd_solve:
 *   z = c - A^T y;  lb^_j = x_j if z_j < -eps_abs;  ub^_j = x_j if z_j > eps_abs;
 *   obj = obj_scale * U[0,1)^n;  R-PDHG on (A, b, obj, lb^, ub^) from (x, 0) with
 *   a fresh primal weight, until k >= min_iters and ||b - A x_k||_2 <= eps_rel (1 + ||b||_2)
 *   (P:391-395).  Returns x^ as the current x; y and z stay phase 1's.
 *   before/after (either may be NULL): statistics of x and x^ with phase-1 z. */
int cpd_corner_push(cpd_solver *s, const cpd_corner_params *cp, cpd_result *out,
                    cpd_stats *before, cpd_stats *after);

/* Exactly k more R-PDHG iterations on the original model with termination tests
 * off (restarts as configured) — lockstep parity with the oracle.  The first call
 * after create / cpd_set_iterate / cpd_solve starts a new run from the current
 * iterate (including the power iteration when step_size <= 0). */
/* NEXT-4 dual corner push ("similar techniques ... to reduce the number of dual superbasic
 * variables"; readings D-1..D-4).  From the solver's current (x, y)
 * (normally the phase-1 solution): the dual corner model frees every column strictly off
 * its bounds by > eps_abs (its dual row becomes z_j = 0), keeps [l, inf) for columns at a
 * lower bound and (-inf, u] at an upper bound (so its dual feasible set is M's dual optimal
 * face for x); PDHG (the solver's method) runs on it from (x, y), fresh primal weight,
 * phase-1 step size, until k >= min_iters and every column's dual violation is <= eps_abs
 * (or max_iters / time_limit).  The solver then holds (x, yhat): x is unchanged.  before /
 * after (nullable): cpd_stats of (x, z) and (x, zhat); zero_rc (d) and est_dual_pushes
 * (m - d) are the quantities the push lowers.  Uses eps_abs, min_iters, max_iters,
 * time_limit_s, candidate_floor of `params` (NULL = defaults).  CPD_E_STATE for scaled or
 * distributed problems. */
int cpd_dual_corner_push(cpd_solver *s, const cpd_corner_params *params, cpd_result *out, cpd_stats *before,
                         cpd_stats *after);
/* On-the-fly choice of the push phases from phase-1 statistics (host only; reading D-4):
 * primal = candidate criterion; dual = est_dual_pushes > 0 and
 * min(m, off_bound) > zero_rc (the dual push can only bring the off-bound columns' reduced
 * costs to 0). */
int cpd_corner_decide(const cpd_stats *st, int32_t m, int32_t *primal, int32_t *dual);
int cpd_step(cpd_solver *s, int64_t k);

/* Current iterate: x[n], y[m], z[n] (z = c - A^T y for phase-1 y); any may be NULL. */
int cpd_get_iterate(const cpd_solver *s, double *x, double *y, double *z, int32_t mem);
/* Set the starting iterate (warm start).  NULL => zeros.  Ends any run. */
int cpd_set_iterate(cpd_solver *s, const double *x, const double *y, int32_t mem);
/* Statistics of the current x against (lb, ub), the corner model (if any) and
 * z = c - A^T y_phase1. */
int cpd_get_stats(const cpd_solver *s, int64_t candidate_floor, cpd_stats *out);
/* Trajectory of the last corner push: (k, off_bound, ||r_P||_2), up to cap entries. */
int cpd_get_trajectory(const cpd_solver *s, int64_t *k, int64_t *off_bound, double *rp,
                       int64_t cap, int64_t *len);

/* Stand-alone device entry points (parity of each step in isolation). */
/* sigma_hat ~ ||A||_2 by `iters` power iterations from U(seed, j) - 0.5. */
int cpd_power_sigma(const cpd_problem *p, int32_t iters, uint64_t seed, double *sigma);
/* KKT terms of (x, y) on the ORIGINAL model (reading S-6):
 * out = {||r_P||, ||r_D||, pobj, dobj, r_P ratio, r_D ratio, gap ratio, score}. */
int cpd_problem_score(const cpd_problem *p, const double *x, const double *y, int32_t mem,
                      double out[8]);
/* Corner statistics of x with z (NULL: no z-based counts) and optional model
 * bounds lhat/uhat (NULL: off_bound_model = 0); all arrays in `mem`. */
int cpd_compute_stats(const cpd_problem *p, const double *x, const double *z,
                      const double *lhat, const double *uhat, double eps_abs,
                      int64_t candidate_floor, int32_t mem, cpd_stats *out);

/* Per-kernel device time accumulated while profile=1 (CUDA events on the
 * solver's stream, active launches only).  names/ms/launches are parallel arrays
 * of length *len (<= cap); names point to static strings.  Reset with reset=1. */
int cpd_get_kernel_times(cpd_solver *s, const char **names, double *ms, int64_t *launches,
                         int32_t cap, int32_t *len, int32_t reset);
/* Launch accounting of a solver: out = {kernels of this library launched on the
 * solver's stream so far (every node of a graph launch counted), CUDA-graph
 * launches, kernels per phase-1 batch graph, kernels per corner batch graph}. */
int cpd_solver_counters(const cpd_solver *s, int64_t out[4]);
/* Algorithmic bytes one launch of kernel `name` moves (DESIGN.md byte model). */
int cpd_kernel_bytes(const cpd_solver *s, const char *name, double *bytes);

/* Device-memory cache (not a paper operation: the library's allocator).
 * Buffers a destroyed problem or solver freed are kept per device in exact-size bins
 * and reused after a device synchronisation (at most CPD_MEMCACHE_MB of idle memory,
 * default a quarter of the device; env CPD_MEMCACHE=0 bypasses it).  cached_bytes
 * reports the idle bytes held for `device`; release frees them (cudaFree) — call it
 * before handing the memory to another allocator in the same process.  Errors:
 * CPD_E_ARG for a bad device ordinal or a NULL out pointer. */
int cpd_memcache_info(int32_t device, int64_t *cached_bytes);
int cpd_memcache_release(int32_t device);

/* ------------------------------------------------------------------ inequality rows
 * Row senses ("handled implicitly"):
 * sense[m] (GLOBAL rows, int8) 0 '=' (A_i x = b_i), 1 '<=' (A_i x <= b_i), 2 '>='.
 * The dual step is projected onto y_i >= 0 ('>='), y_i <= 0 ('<='); the primal
 * residual counts violations only; the corner model turns an inequality row whose
 * slack has a non-trivial reduced cost (|y*_i| > eps_abs) into an equality
 * (cpd_stats.rows_eq counts them).  Call before creating solvers: CPD_E_STATE
 * while a solver created on `p` is alive (its captured graphs hold the problem's
 * device pointers).  CPD_E_ARG on a value outside {0, 1, 2}. */
int cpd_problem_set_senses(cpd_problem *p, const int8_t *sense, int32_t mem);

/* ------------------------------------------------------------------ preconditioning
 * Diagonal scaling of the problem (the cuPDLP+ lineage the
 * paper's PDHG follows; reading R-3): `ruiz_iters` Ruiz passes
 * (rho_i = sqrt(max_j |a_ij|), kappa_j = sqrt(max_i |a_ij|)) then, if pock_chambolle,
 * one Pock-Chambolle alpha = 1 pass (square roots of row / column sums of |a_ij|);
 * each pass a_ij /= rho_i kappa_j.  The device LP becomes A^ = diag(r) A diag(s),
 * b^ = r b, c^ = s c, l^ = l / s, u^ = u / s; solvers iterate on it (step size, primal
 * weight and restart distances in the scaled space) while termination, restart
 * scores, the steering stop and all statistics are those of the ORIGINAL LP
 * (P:119-131), and every iterate in or out of the ABI is original-space.
 * Call once, before creating solvers; single-GPU problems only (CPD_E_ARG otherwise,
 * CPD_E_STATE if already scaled or while a solver created on `p` is alive). */
int cpd_problem_scale(cpd_problem *p, int32_t ruiz_iters, int32_t pock_chambolle);
/* The scale vectors r[m], s[n] (host); CPD_E_STATE if the problem is not scaled. */
int cpd_problem_get_scaling(const cpd_problem *p, double *r, double *s);

/* ------------------------------------------------------------------ multi-GPU
 * One process per GPU.  The LP is split into
 * contiguous blocks balanced by nonzeros (+1 per row for the vector work):
 *   partition 0 = row-block (BJ north_star): rank p keeps rows R_p of A; y, b, Ax
 *     are sharded with them; A^T y is partial on every rank and is reduce-scattered
 *     into equal slices of length L = ceil(n / world) of the n-side, where the
 *     primal step runs; x+ is all-gathered for the local A x+.
 *   partition 1 = col-block: rank p keeps columns C_p; x, c, bounds are sharded;
 *     A x+ is partial, reduce-scattered into slices of the m-side where the dual
 *     step runs; y+ is all-gathered for the local A^T y.
 *   partition -1 = col-block if n >= m else row-block ("shard the long vector").
 * Every scalar the device decisions use is allreduced first, so all ranks take
 * the same decisions.  All calls on a distributed problem or its solvers are
 * COLLECTIVE: every rank makes them in the same order.  cpd_get_iterate /
 * cpd_set_iterate / cpd_problem_score / cpd_compute_stats take and return GLOBAL
 * vectors; cpd_problem_info reports global m, n and LOCAL nnz. */

/* Host-only (no device needed): bounds[world + 1] of the contiguous blocks of
 * columns (partition 1) or rows (partition 0) this library assigns to each rank,
 * from the GLOBAL CSR(A^T).  CPD_E_ARG if world > min(m, n). */
int cpd_partition(int32_t m, int32_t n, const int32_t *AT_rowptr, const int32_t *AT_col, int32_t world,
                  int32_t partition, int64_t *bounds);
/* Host-only (no device needed): the layout cpd_problem_create_dist gives rank `rank`
 * (partition -1 = auto, as there).  out[12] = {partition, split side (0 m-side: y, b,
 * Ax sliced; 1 n-side: x, c, bounds sliced), L = slice length ceil(rows of the split
 * side / world), block [begin, end) of the sharded side (columns for partition 1,
 * rows for 0), owned length of side 0, of side 1, global index of the owned part's
 * element 0 on side 0, on side 1, offset of the owned part in the rank's local
 * side-0 arrays, side-1 arrays, local rows of A^T}.  Errors as cpd_partition. */
int cpd_dist_layout(int32_t m, int32_t n, const int32_t *AT_rowptr, const int32_t *AT_col, int32_t world,
                    int32_t partition, int32_t rank, int64_t out[12]);
/* 128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it). */
int cpd_nccl_get_unique_id(char id[128]);
/* Create this rank's block of the GLOBAL LP (CSR(A^T) + b, c, lb, ub, all in host
 * memory, borrowed for the call) on `device`, and the NCCL communicator of
 * `world` ranks from `id`.  Validation as cpd_problem_create, on the block. */
int cpd_problem_create_dist(int32_t rank, int32_t world, const char id[128], int32_t partition,
                            int32_t m, int32_t n, int64_t nnz,
                            const int32_t *AT_rowptr, const int32_t *AT_col, const double *AT_val,
                            const double *b, const double *c, const double *lb, const double *ub,
                            int32_t device, cpd_problem **out);
/* info = {world, rank, partition (-1 single GPU), L, owned m-side length, owned
 * n-side length, global index of the first owned m-side / n-side element, local
 * rows of A, local rows of A^T}. */
int cpd_problem_dist_info(const cpd_problem *p, int64_t info[10]);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* CPD_H */
