/*
 * ORACLE — plain, slow, single-threaded fp64 CPU implementation of the hot path
 * of "Corner push PDHG" (arXiv 2511.13894).  TEST INFRASTRUCTURE ONLY: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load or call it.  It shares no code with the CUDA path
 * (paper_2511_13894_b200/csrc) and neither includes the other.
 *
 * Compiled: gcc -O2 -fno-fast-math -ffp-contract=off -shared -fPIC (no SIMD
 * intrinsics, no OpenMP, no BLAS).  Every formula below is written as the paper
 * (or the SURVEY.md §8(c) reading of it, listed in DESIGN.md "Readings") states
 * it, with no blocking, fusion or algebraic rewriting:
 *
 *   P:64-87    primal/dual pair  min c^T x, Ax=b, x>=0 | max b^T y, A^T y + z = c, z>=0
 *   P:89-92    general bounds handled implicitly -> projection onto [l,u] (S-6, S-14)
 *   P:109-117  r_P = b - A x,  r_D = c - A^T y - z
 *   P:119-131  relative termination tests (2-norms), converged <=> all three hold
 *   P:21-27, P:412-414 + SURVEY §8(c) R-PDHG   the iteration (S-1..S-5, S-16)
 *   P:268-293  Algorithm 1 (corner model M^: bound map, Uniform[0,1]^n objective,
 *              warm start (x, 0)), P:318-329 + P:391-395 early termination
 *   P:200-210, P:330-381, P:438-452   off-bound / zero-reduced-cost counts,
 *              push estimates, candidate criterion
 *
 * Pins (tests/test_oracle_*.py, `-m "not gpu"`): 2x2 hand-stepped iterate
 * (tests/golden/pdhg_2x2.json), 1x1 closed form, dense recomputation of
 * residuals, certificate fixed point, SVD / closed-form operator norms, brute
 * force vertex enumeration + HiGHS optima, SplitMix64 published outputs,
 * Algorithm-1 bound-map and count examples.  Iteration COUNTS to eps have no
 * closed form: "parity unpinned" beyond this file.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ types */
typedef struct {
    int32_t m, n;
    const int32_t *Ap, *Aj; const double *Ax;     /* CSR(A)   (m rows) */
    const int32_t *ATp, *ATj; const double *ATx;  /* CSR(A^T) (n rows) */
    const double *b;                              /* m */
    const int8_t *sense;   /* m or NULL (all '='): 0 '=' , 1 '<=' (Ax <= b), 2 '>=' (Ax >= b)
                              (inequality rows handled implicitly) */
} orc_lp;

typedef struct {
    double eps_rel, eps_abs;
    int64_t max_iters;
    double time_limit_s;
    int32_t check_every;     /* K: restart-check cadence on t (PDLP lineage) */
    double step_scale;       /* eta = step_scale / sigma_hat */
    double step_size;        /* > 0: eta given explicitly */
    int32_t power_iters;     /* K_pow */
    uint64_t seed;           /* power-iteration start vector seed */
    double primal_weight;    /* > 0: omega0 given explicitly */
    int32_t restart;         /* 0 none, 1 adaptive restart to average/current */
    double beta_suff, beta_nec, beta_art, theta;
    /* NEXT-1 (cuPDLP+ lineage; reading H-1..H-4) */
    int32_t method;          /* 0 R-PDHG (averages), 1 reflected restarted Halpern PDHG */
    double reflection;       /* rho of z+ = lambda((1+rho) T(z) - rho z) + (1-lambda) z_anchor */
    int32_t pid;             /* 1: PID primal weight at restarts (else theta smoothing) */
    double kp, ki, kd;       /* PID gains on e = log(dy/dx) - log omega */
} orc_params;

typedef struct {
    int32_t status;          /* 0 converged, 1 iter limit, 2 time limit, 3 numerical failure, -1 running */
    int32_t returned_average;
    int64_t iterations, restarts;
    double pobj, dobj, gap, rp_norm, rd_norm, score, step_size, primal_weight, wall_s;
} orc_result;

typedef struct {
    double rp, rd, pobj, dobj, r_p, r_d, r_g, score;
} orc_score_t;

typedef struct {
    int64_t off_bound, off_bound_strict, off_bound_model, zero_rc, candidates,
            fix_lb, fix_ub, est_primal_pushes, est_dual_pushes;
    int32_t is_candidate;
} orc_stats_t;

enum { MODE_FULL = 0, MODE_PRIMAL_ONLY = 1, MODE_NONE = 2, MODE_DUAL_ONLY = 3 };

/* ---------------------------------------------------------- basic helpers */

/* Counter-based U[0,1): SplitMix64 finalizer of seed + (j+1)*golden (SURVEY §8(c)
 * "U(seed, j)"); the (j+1)-th output of a SplitMix64 stream seeded with `seed`. */
uint64_t orc_splitmix(uint64_t seed, int64_t j)
{
    uint64_t s = seed + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ULL;
    s = (s ^ (s >> 30)) * 0xBF58476D1CE4E5B9ULL;
    s = (s ^ (s >> 27)) * 0x94D049BB133111EBULL;
    s ^= s >> 31;
    return s;
}

double orc_u01(uint64_t seed, int64_t j)
{
    return (double)(orc_splitmix(seed, j) >> 11) * (1.0 / 9007199254740992.0);
}

/* CSR transpose by counting sort (the oracle's own loader). */
void orc_transpose(int32_t nrows, int32_t ncols, const int32_t *p, const int32_t *j,
                   const double *x, int32_t *tp, int32_t *tj, double *tx)
{
    int64_t *next = (int64_t *)calloc((size_t)ncols + 1, sizeof(int64_t));
    for (int32_t r = 0; r < nrows; ++r)
        for (int64_t k = p[r]; k < p[r + 1]; ++k) next[j[k] + 1]++;
    for (int32_t c = 0; c < ncols; ++c) next[c + 1] += next[c];
    for (int32_t c = 0; c <= ncols; ++c) tp[c] = (int32_t)next[c];
    for (int32_t r = 0; r < nrows; ++r)
        for (int64_t k = p[r]; k < p[r + 1]; ++k) {
            int64_t d = next[j[k]]++;
            tj[d] = r;
            tx[d] = x[k];
        }
    free(next);
}

/* out = M v for CSR M with `rows` rows: out_r = sum_k M_rk v_k (in storage order). */
void orc_spmv(int32_t rows, const int32_t *p, const int32_t *j, const double *x,
              const double *v, double *out)
{
    for (int32_t r = 0; r < rows; ++r) {
        double s = 0.0;
        for (int64_t k = p[r]; k < p[r + 1]; ++k) s += x[k] * v[j[k]];
        out[r] = s;
    }
}

double orc_norm2(int64_t n, const double *v)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

static double dot(int64_t n, const double *a, const double *b)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------- residuals, score */

/* Row i of r_P = b - A x counts its violation only:
 * '=' r;  '<=' (Ax <= b, feasible when r >= 0) min(r, 0);  '>=' max(r, 0). */
static double row_violation(const orc_lp *lp, int32_t i, double r)
{
    int s = lp->sense ? lp->sense[i] : 0;
    if (s == 1) return r < 0.0 ? r : 0.0;
    if (s == 2) return r > 0.0 ? r : 0.0;
    return r;
}

/* Dual sign constraint of row i for L = c^T x + y^T (b - A x): '>=' rows y >= 0,
 * '<=' rows y <= 0, '=' free (projection of the dual step). */
static double dual_proj(const orc_lp *lp, int32_t i, double v)
{
    int s = lp->sense ? lp->sense[i] : 0;
    if (s == 1) return v < 0.0 ? v : 0.0;
    if (s == 2) return v > 0.0 ? v : 0.0;
    return v;
}

/* KKT score of (x, y) for objective c and bounds [l, u] (S-3, S-6):
 *   z = c - A^T y;  r_P = b - A x
 *   r_D_j = z_j - [l_j > -inf] max(z_j,0) + [u_j < inf] max(-z_j,0)  (violation part)
 *   pobj = c^T x;  dobj = b^T y + sum_{l_j>-inf} l_j max(z_j,0) - sum_{u_j<inf} u_j max(-z_j,0)
 *   score = max(||r_P||/(1+||b||), ||r_D||/(1+||c||), |pobj-dobj|/(1+|pobj|+|dobj|)) */
void orc_score(const orc_lp *lp, const double *c, const double *l, const double *u,
               double nb, double nc, const double *x, const double *y, orc_score_t *out)
{
    int32_t m = lp->m, n = lp->n;
    double *ax = (double *)malloc(sizeof(double) * (m ? m : 1));
    double *aty = (double *)malloc(sizeof(double) * (n ? n : 1));
    orc_spmv(m, lp->Ap, lp->Aj, lp->Ax, x, ax);
    orc_spmv(n, lp->ATp, lp->ATj, lp->ATx, y, aty);
    double rp2 = 0.0;
    for (int32_t i = 0; i < m; ++i) {
        double r = row_violation(lp, i, lp->b[i] - ax[i]);
        rp2 += r * r;
    }
    double rd2 = 0.0, pobj = 0.0, bound_terms = 0.0;
    for (int32_t j = 0; j < n; ++j) {
        double z = c[j] - aty[j];
        double zp = z > 0.0 ? z : 0.0;
        double zm = -z > 0.0 ? -z : 0.0;
        double rd = z;
        if (l[j] > -INFINITY) { rd -= zp; bound_terms += l[j] * zp; }
        if (u[j] < INFINITY)  { rd += zm; bound_terms -= u[j] * zm; }
        rd2 += rd * rd;
        pobj += c[j] * x[j];
    }
    double dobj = dot(m, lp->b, y) + bound_terms;
    out->rp = sqrt(rp2);
    out->rd = sqrt(rd2);
    out->pobj = pobj;
    out->dobj = dobj;
    out->r_p = out->rp / (1.0 + nb);
    out->r_d = out->rd / (1.0 + nc);
    out->r_g = fabs(pobj - dobj) / (1.0 + fabs(pobj) + fabs(dobj));
    double s = out->r_p;
    if (out->r_d > s) s = out->r_d;
    if (out->r_g > s) s = out->r_g;
    out->score = s;
    free(ax);
    free(aty);
}

/* Operator-norm estimate (S-2): v0_j = U(seed,j) - 0.5, normalised; K power
 * iterations v <- A^T A v / ||A^T A v||; sigma_hat = sqrt(||A^T A v||) at the last. */
double orc_power_sigma(const orc_lp *lp, int32_t iters, uint64_t seed)
{
    int32_t m = lp->m, n = lp->n;
    double *v = (double *)malloc(sizeof(double) * (n ? n : 1));
    double *w = (double *)malloc(sizeof(double) * (m ? m : 1));
    double *u = (double *)malloc(sizeof(double) * (n ? n : 1));
    for (int32_t j = 0; j < n; ++j) v[j] = orc_u01(seed, j) - 0.5;
    double nv = orc_norm2(n, v);
    for (int32_t j = 0; j < n; ++j) v[j] = v[j] / nv;
    double nu = 0.0;
    for (int32_t it = 0; it < iters; ++it) {
        orc_spmv(m, lp->Ap, lp->Aj, lp->Ax, v, w);
        orc_spmv(n, lp->ATp, lp->ATj, lp->ATx, w, u);
        nu = orc_norm2(n, u);
        if (!(nu > 0.0)) break;
        for (int32_t j = 0; j < n; ++j) v[j] = u[j] / nu;
    }
    free(v); free(w); free(u);
    return sqrt(nu);
}

/* ------------------------------------------------ diagonal preconditioning */

/* Ruiz + Pock-Chambolle scaling of A (the cuPDLP+ lineage the
 * paper's PDHG follows; reading R-3).  On CSR(A) (m rows)
 * in place, r (m) and s (n) start at 1:
 *   Ruiz, `ruiz_iters` passes:  rho_i = sqrt(max_j |a_ij|), kappa_j = sqrt(max_i |a_ij|)
 *   then, if pc, one Pock-Chambolle (alpha = 1) pass:
 *                               rho_i = sqrt(sum_j |a_ij|),  kappa_j = sqrt(sum_i |a_ij|)
 *   each pass (a zero row/column gets 1):  a_ij <- a_ij / (rho_i kappa_j),
 *                                          r_i <- r_i / rho_i,  s_j <- s_j / kappa_j
 * so that the scaled matrix is diag(r) A diag(s). */
void orc_scale(int32_t m, int32_t n, const int32_t *Ap, const int32_t *Aj, double *Ax,
               int32_t ruiz_iters, int32_t pc, double *r, double *s)
{
    double *rho = (double *)malloc(sizeof(double) * (m ? m : 1));
    double *kap = (double *)malloc(sizeof(double) * (n ? n : 1));
    for (int32_t i = 0; i < m; ++i) r[i] = 1.0;
    for (int32_t j = 0; j < n; ++j) s[j] = 1.0;
    for (int32_t pass = 0; pass < ruiz_iters + (pc ? 1 : 0); ++pass) {
        int sum = pass >= ruiz_iters;   /* the Pock-Chambolle pass */
        for (int32_t i = 0; i < m; ++i) rho[i] = 0.0;
        for (int32_t j = 0; j < n; ++j) kap[j] = 0.0;
        for (int32_t i = 0; i < m; ++i)
            for (int64_t k = Ap[i]; k < Ap[i + 1]; ++k) {
                double a = fabs(Ax[k]);
                int32_t j = Aj[k];
                if (sum) { rho[i] += a; kap[j] += a; }
                else {
                    if (a > rho[i]) rho[i] = a;
                    if (a > kap[j]) kap[j] = a;
                }
            }
        for (int32_t i = 0; i < m; ++i) rho[i] = rho[i] > 0.0 ? sqrt(rho[i]) : 1.0;
        for (int32_t j = 0; j < n; ++j) kap[j] = kap[j] > 0.0 ? sqrt(kap[j]) : 1.0;
        for (int32_t i = 0; i < m; ++i)
            for (int64_t k = Ap[i]; k < Ap[i + 1]; ++k) Ax[k] = Ax[k] / (rho[i] * kap[Aj[k]]);
        for (int32_t i = 0; i < m; ++i) r[i] = r[i] / rho[i];
        for (int32_t j = 0; j < n; ++j) s[j] = s[j] / kap[j];
    }
    free(rho);
    free(kap);
}

/* ------------------------------------------------------------------ R-PDHG */
typedef struct {
    const orc_lp *lp;
    orc_params prm;
    const double *c, *l, *u;   /* objective and bounds in use (M or M^) */
    int mode;                  /* MODE_* */
    double target;             /* primal-only: ||b - Ax|| <= target */
    int64_t min_iters;
    double nb, nc, eta, omega;
    double *x, *y, *xavg, *yavg, *xr, *yr, *xn, *yn, *aty, *xbar, *axbar;
    int64_t k, t, restarts;
    double S_r, S_prev;
    /* Halpern (method 1): anchor, last PDHG output T(z) = (xh, yh), fixed-point
     * residuals r0 (at the anchor) / r_prev (last check), PID state */
    double *xa, *ya, *xh, *yh, *dxv;
    double r0, r_prev, r_last, pid_int, pid_eprev;
    int status, returned_average;
    double t0;
    /* scaled run (orc_set_original): score and primal residual on the ORIGINAL LP at
     * the unscaled point x = s x^, y = r y^ (P:119-131 are criteria of the LP as given) */
    const orc_lp *orig;
    const double *oc, *ol, *ou, *sr, *sc;
    double onb, onc;
    double *ux, *uy;
} orc_state;

void orc_destroy(orc_state *s)
{
    if (!s) return;
    free(s->x); free(s->y); free(s->xavg); free(s->yavg); free(s->xr); free(s->yr);
    free(s->xn); free(s->yn); free(s->aty); free(s->xbar); free(s->axbar);
    free(s->ux); free(s->uy);
    free(s->xa); free(s->ya); free(s->xh); free(s->yh); free(s->dxv);
    free(s);
}

static double score_of(orc_state *s, const double *x, const double *y, orc_score_t *o)
{
    if (s->orig) {
        for (int32_t j = 0; j < s->lp->n; ++j) s->ux[j] = s->sc[j] * x[j];
        for (int32_t i = 0; i < s->lp->m; ++i) s->uy[i] = s->sr[i] * y[i];
        orc_score(s->orig, s->oc, s->ol, s->ou, s->onb, s->onc, s->ux, s->uy, o);
        return o->score;
    }
    orc_score(s->lp, s->c, s->l, s->u, s->nb, s->nc, x, y, o);
    return o->score;
}

static double proj(double v, double lo, double hi)
{
    double r = v > lo ? v : lo;   /* max(v, lo) */
    return r < hi ? r : hi;       /* min(., hi) */
}

/* Create a run of R-PDHG on (A, b, c, [l,u]) (SURVEY §8(c) "Setup").
 * eta_in > 0 overrides prm->step_size / power iteration; omega_in > 0 overrides
 * prm->primal_weight.  x_init/y_init NULL => 0. */
orc_state *orc_create(const orc_lp *lp, const orc_params *prm, const double *c,
                      const double *l, const double *u, const double *x_init,
                      const double *y_init, int mode, double target, int64_t min_iters,
                      double eta_in)
{
    int32_t m = lp->m, n = lp->n;
    orc_state *s = (orc_state *)calloc(1, sizeof(orc_state));
    size_t N = (size_t)(n ? n : 1), M = (size_t)(m ? m : 1);
    s->lp = lp; s->prm = *prm; s->c = c; s->l = l; s->u = u;
    s->mode = mode; s->target = target; s->min_iters = min_iters;
    s->x = (double *)calloc(N, 8); s->xavg = (double *)calloc(N, 8);
    s->xr = (double *)calloc(N, 8); s->xn = (double *)calloc(N, 8);
    s->aty = (double *)calloc(N, 8); s->xbar = (double *)calloc(N, 8);
    s->y = (double *)calloc(M, 8); s->yavg = (double *)calloc(M, 8);
    s->yr = (double *)calloc(M, 8); s->yn = (double *)calloc(M, 8);
    s->axbar = (double *)calloc(M, 8);
    s->xa = (double *)calloc(N, 8); s->xh = (double *)calloc(N, 8); s->dxv = (double *)calloc(N, 8);
    s->ya = (double *)calloc(M, 8); s->yh = (double *)calloc(M, 8);
    s->t0 = now_s();
    s->nb = orc_norm2(m, lp->b);
    s->nc = orc_norm2(n, c);
    if (eta_in > 0.0) s->eta = eta_in;
    else if (prm->step_size > 0.0) s->eta = prm->step_size;
    else s->eta = prm->step_scale / orc_power_sigma(lp, prm->power_iters, prm->seed);
    if (prm->primal_weight > 0.0) s->omega = prm->primal_weight;
    else s->omega = (s->nc > 1e-10 && s->nb > 1e-10) ? s->nc / s->nb : 1.0;
    for (int32_t j = 0; j < n; ++j) s->x[j] = proj(x_init ? x_init[j] : 0.0, l[j], u[j]);
    for (int32_t i = 0; i < m; ++i) s->y[i] = y_init ? y_init[i] : 0.0;
    memcpy(s->xr, s->x, N * 8);
    memcpy(s->yr, s->y, M * 8);
    memcpy(s->xa, s->x, N * 8);   /* Halpern anchor z^0 = starting point */
    memcpy(s->ya, s->y, M * 8);
    memcpy(s->xh, s->x, N * 8);
    memcpy(s->yh, s->y, M * 8);
    s->r0 = INFINITY; s->r_prev = INFINITY; s->r_last = INFINITY;
    s->pid_int = 0.0; s->pid_eprev = 0.0;
    orc_score_t o;
    s->S_r = score_of(s, s->x, s->y, &o);
    s->S_prev = INFINITY;
    s->k = 0; s->t = 0; s->restarts = 0;
    s->status = -1; s->returned_average = 0;
    if (mode == MODE_FULL && s->S_r <= prm->eps_rel) s->status = 0;
    return s;
}

double orc_get_eta(const orc_state *s) { return s->eta; }
double orc_get_omega(const orc_state *s) { return s->omega; }
int64_t orc_get_k(const orc_state *s) { return s->k; }

/* Restart bookkeeping of a run (read-only test access for the restart pins,
 * tests/golden/restart_2x2.json): reference score S_r, previous candidate score
 * S_prev, iterations since the last restart t, and the restart count (Halpern: the
 * fixed-point residuals r0 at the anchor and r_prev at the last check in S_r / S_prev). */
void orc_get_restart_state(const orc_state *s, double *S_r, double *S_prev, int64_t *t,
                           int64_t *restarts)
{
    *S_r = s->prm.method == 1 ? s->r0 : s->S_r;
    *S_prev = s->prm.method == 1 ? s->r_prev : s->S_prev;
    *t = s->t;
    *restarts = s->restarts;
}

/* Mark a run as the scaled image of `orig` (objective oc, bounds ol/ou in original
 * space, x = sc x^, y = sr y^): termination, restart scores and the primal-only
 * residual are then evaluated on the original LP; everything else (steps, primal
 * weight, restart distances) stays in the scaled space.  Re-scores the start. */
void orc_set_original(orc_state *s, const orc_lp *orig, const double *oc, const double *ol,
                      const double *ou, const double *sr, const double *sc)
{
    s->orig = orig; s->oc = oc; s->ol = ol; s->ou = ou; s->sr = sr; s->sc = sc;
    s->onb = orc_norm2(orig->m, orig->b);
    s->onc = orc_norm2(orig->n, oc);
    s->ux = (double *)calloc((size_t)(s->lp->n ? s->lp->n : 1), 8);
    s->uy = (double *)calloc((size_t)(s->lp->m ? s->lp->m : 1), 8);
    orc_score_t o;
    s->S_r = score_of(s, s->x, s->y, &o);
    s->status = -1;
    if (s->mode == MODE_FULL && s->S_r <= s->prm.eps_rel) s->status = 0;
}

static double primal_res(orc_state *s, const double *x)
{
    const orc_lp *lp = s->lp;
    if (s->orig) {   /* ||b - A x|| of the original LP at x = s x^ */
        for (int32_t j = 0; j < lp->n; ++j) s->ux[j] = s->sc[j] * x[j];
        lp = s->orig;
        x = s->ux;
    }
    orc_spmv(lp->m, lp->Ap, lp->Aj, lp->Ax, x, s->axbar);
    double r2 = 0.0;
    for (int32_t i = 0; i < lp->m; ++i) {
        double r = row_violation(lp, i, lp->b[i] - s->axbar[i]);
        r2 += r * r;
    }
    return sqrt(r2);
}

/* Number of columns whose dual violation r_D_j (S-6, w.r.t. the run's bounds) exceeds
 * eps_abs in absolute value: the dual corner push stops when it is 0 (reading D-3). */
static int64_t dual_viol_count(orc_state *s, const double *y)
{
    const orc_lp *lp = s->lp;
    orc_spmv(lp->n, lp->ATp, lp->ATj, lp->ATx, y, s->aty);
    int64_t cnt = 0;
    for (int32_t j = 0; j < lp->n; ++j) {
        double z = s->c[j] - s->aty[j];
        double zp = z > 0.0 ? z : 0.0, zm = -z > 0.0 ? -z : 0.0, rd = z;
        if (s->l[j] > -INFINITY) rd -= zp;
        if (s->u[j] < INFINITY) rd += zm;
        cnt += fabs(rd) > s->prm.eps_abs;
    }
    return cnt;
}

/* Primal-weight update at a restart from the anchor movement (dx, dy): theta
 * smoothing (S-1, PDLP lineage) or, with pid, a PID controller on the log-ratio error
 * e = log(dy/dx) - log omega (reading H-3):
 *   log omega <- log omega + kp e + ki sum(e) + kd (e - e_prev). */
static void weight_update(orc_state *s, double dx, double dy)
{
    const orc_params *P = &s->prm;
    if (!(dx > 1e-10 && dy > 1e-10)) return;
    if (P->pid) {
        double e = log(dy / dx) - log(s->omega);
        s->pid_int += e;
        double lw = log(s->omega) + P->kp * e + P->ki * s->pid_int + P->kd * (e - s->pid_eprev);
        s->pid_eprev = e;
        s->omega = exp(lw);
    } else {
        s->omega = exp(P->theta * log(dy / dx) + (1.0 - P->theta) * log(s->omega));
    }
}

/* Reflected restarted Halpern PDHG (NEXT-1; readings H-1..H-4), step by step:
 *   (xh, yh) = T(x, y)   (the PDHG map of R-PDHG: projected primal step, extrapolated dual step)
 *   r^2 = ||xh-x||^2/tau + ||yh-y||^2/sigma + 2 <yh-y, A(xh-x)>   (fixed-point residual, M-norm)
 *   lambda = (t+1)/(t+2);  z <- lambda((1+rho) zh - rho z) + (1-lambda) z_anchor;  t++, k++
 *   r0 <- r when t was 0 (the residual at the anchor)
 *   primal-only: stop at k >= min_iters with ||b - A xh|| <= target, returning zh
 *   every K (t mod K = 0): score(zh) <= eps (mode full) -> return zh; restart test on r:
 *     r <= b_suff r0, or (r <= b_nec r0 and r > r_prev), or t >= b_art k  ->
 *     weight update from the anchor movement, z = z_anchor = zh, t = 0
 *   k = max_iters -> return zh (ITER_LIMIT).  The returned point is always zh (in the box). */
static int orc_run_halpern(orc_state *s, int64_t steps)
{
    const orc_lp *lp = s->lp;
    int32_t m = lp->m, n = lp->n;
    const orc_params *P = &s->prm;
    const double rho = P->reflection;
    for (int64_t it = 0; it < steps && s->status < 0; ++it) {
        double tau = s->eta / s->omega;
        double sigma = s->eta * s->omega;
        /* (xh, yh) = T(z) */
        orc_spmv(n, lp->ATp, lp->ATj, lp->ATx, s->y, s->aty);
        for (int32_t j = 0; j < n; ++j)
            s->xh[j] = proj(s->x[j] - tau * (s->c[j] - s->aty[j]), s->l[j], s->u[j]);
        for (int32_t j = 0; j < n; ++j) s->xbar[j] = 2.0 * s->xh[j] - s->x[j];
        orc_spmv(m, lp->Ap, lp->Aj, lp->Ax, s->xbar, s->axbar);
        for (int32_t i = 0; i < m; ++i)
            s->yh[i] = dual_proj(lp, i, s->y[i] + sigma * (lp->b[i] - s->axbar[i]));
        int bad = 0;
        for (int32_t j = 0; j < n; ++j) bad |= !isfinite(s->xh[j]);
        for (int32_t i = 0; i < m; ++i) bad |= !isfinite(s->yh[i]);
        if (bad) { s->status = 3; s->k += 1; break; }
        /* fixed-point residual of z in the M-norm */
        double dx2 = 0.0, dy2 = 0.0, cross = 0.0;
        for (int32_t j = 0; j < n; ++j) { s->dxv[j] = s->xh[j] - s->x[j]; dx2 += s->dxv[j] * s->dxv[j]; }
        orc_spmv(m, lp->Ap, lp->Aj, lp->Ax, s->dxv, s->axbar);   /* A (xh - x) */
        for (int32_t i = 0; i < m; ++i) {
            double d = s->yh[i] - s->y[i];
            dy2 += d * d;
            cross += d * s->axbar[i];
        }
        double r2 = dx2 / tau + dy2 / sigma + 2.0 * cross;
        double r = sqrt(r2 > 0.0 ? r2 : 0.0);
        if (s->t == 0) s->r0 = r;
        s->r_last = r;
        /* Halpern step with reflection */
        double lam = (double)(s->t + 1) / (double)(s->t + 2);
        for (int32_t j = 0; j < n; ++j)
            s->x[j] = lam * ((1.0 + rho) * s->xh[j] - rho * s->x[j]) + (1.0 - lam) * s->xa[j];
        for (int32_t i = 0; i < m; ++i)
            s->y[i] = lam * ((1.0 + rho) * s->yh[i] - rho * s->y[i]) + (1.0 - lam) * s->ya[i];
        s->t += 1;
        s->k += 1;
        orc_score_t o;
        if (s->mode == MODE_PRIMAL_ONLY) {
            if (s->k >= s->min_iters && primal_res(s, s->xh) <= s->target) { s->status = 0; break; }
        }
        if (s->t % P->check_every == 0) {
            double S = score_of(s, s->xh, s->yh, &o);
            if (s->mode == MODE_FULL && S <= P->eps_rel) { s->status = 0; break; }
            if (s->mode == MODE_DUAL_ONLY && s->k >= s->min_iters && dual_viol_count(s, s->yh) == 0) {
                s->status = 0; break;
            }
            if (P->restart) {
                if (r <= P->beta_suff * s->r0 || (r <= P->beta_nec * s->r0 && r > s->r_prev) ||
                    (double)s->t >= P->beta_art * (double)s->k) {
                    double ddx = 0.0, ddy = 0.0;
                    for (int32_t j = 0; j < n; ++j) { double d = s->xh[j] - s->xa[j]; ddx += d * d; }
                    for (int32_t i = 0; i < m; ++i) { double d = s->yh[i] - s->ya[i]; ddy += d * d; }
                    weight_update(s, sqrt(ddx), sqrt(ddy));
                    memcpy(s->x, s->xh, sizeof(double) * n);
                    memcpy(s->y, s->yh, sizeof(double) * m);
                    memcpy(s->xa, s->xh, sizeof(double) * n);
                    memcpy(s->ya, s->yh, sizeof(double) * m);
                    s->t = 0;
                    s->r_prev = INFINITY;
                    s->restarts += 1;
                } else {
                    s->r_prev = r;
                }
            }
        }
        if (s->mode != MODE_NONE) {
            if (s->k == P->max_iters) { s->status = 1; break; }
            if (P->time_limit_s > 0.0 && now_s() - s->t0 > P->time_limit_s) { s->status = 2; break; }
        }
    }
    return s->status;
}

/* Run up to `steps` more iterations (SURVEY §8(c) "loop"); returns status
 * (-1 = still running after `steps`). */
int orc_run(orc_state *s, int64_t steps)
{
    const orc_lp *lp = s->lp;
    int32_t m = lp->m, n = lp->n;
    const orc_params *P = &s->prm;
    if (P->method == 1) return orc_run_halpern(s, steps);
    for (int64_t it = 0; it < steps && s->status < 0; ++it) {
        double tau = s->eta / s->omega;
        double sigma = s->eta * s->omega;
        /* x+ = proj(x - tau (c - A^T y)) */
        orc_spmv(n, lp->ATp, lp->ATj, lp->ATx, s->y, s->aty);
        for (int32_t j = 0; j < n; ++j)
            s->xn[j] = proj(s->x[j] - tau * (s->c[j] - s->aty[j]), s->l[j], s->u[j]);
        /* y+ = y + sigma (b - A (2 x+ - x)) */
        for (int32_t j = 0; j < n; ++j) s->xbar[j] = 2.0 * s->xn[j] - s->x[j];
        orc_spmv(m, lp->Ap, lp->Aj, lp->Ax, s->xbar, s->axbar);
        for (int32_t i = 0; i < m; ++i)
            s->yn[i] = dual_proj(lp, i, s->y[i] + sigma * (lp->b[i] - s->axbar[i]));
        int bad = 0;
        for (int32_t j = 0; j < n; ++j) bad |= !isfinite(s->xn[j]);
        for (int32_t i = 0; i < m; ++i) bad |= !isfinite(s->yn[i]);
        if (bad) { s->status = 3; s->k += 1; break; }
        s->t += 1;
        for (int32_t j = 0; j < n; ++j) s->xavg[j] += (s->xn[j] - s->xavg[j]) / (double)s->t;
        for (int32_t i = 0; i < m; ++i) s->yavg[i] += (s->yn[i] - s->yavg[i]) / (double)s->t;
        memcpy(s->x, s->xn, sizeof(double) * n);
        memcpy(s->y, s->yn, sizeof(double) * m);
        s->k += 1;
        orc_score_t o;
        if (s->mode == MODE_FULL) {
            if (score_of(s, s->x, s->y, &o) <= P->eps_rel) { s->status = 0; break; }
        } else if (s->mode == MODE_PRIMAL_ONLY) {
            if (s->k >= s->min_iters && primal_res(s, s->x) <= s->target) { s->status = 0; break; }
        } else if (s->mode == MODE_DUAL_ONLY) {   /* dual corner push stop (NEXT-4, reading D-3) */
            if (s->k >= s->min_iters && dual_viol_count(s, s->y) == 0) { s->status = 0; break; }
        }
        if (P->restart && s->t % P->check_every == 0) {
            double S_a = score_of(s, s->xavg, s->yavg, &o);
            double S_c = score_of(s, s->x, s->y, &o);
            if (s->mode == MODE_FULL && S_a <= P->eps_rel) {
                s->status = 0; s->returned_average = 1; break;
            }
            int use_avg = S_a < S_c;                       /* tie -> current (S-14) */
            const double *xc = use_avg ? s->xavg : s->x;
            const double *yc = use_avg ? s->yavg : s->y;
            double S = use_avg ? S_a : S_c;
            if (S <= P->beta_suff * s->S_r ||
                (S <= P->beta_nec * s->S_r && S > s->S_prev) ||
                (double)s->t >= P->beta_art * (double)s->k) {
                double dx2 = 0.0, dy2 = 0.0;
                for (int32_t j = 0; j < n; ++j) { double d = xc[j] - s->xr[j]; dx2 += d * d; }
                for (int32_t i = 0; i < m; ++i) { double d = yc[i] - s->yr[i]; dy2 += d * d; }
                weight_update(s, sqrt(dx2), sqrt(dy2));
                if (use_avg) {
                    memcpy(s->x, s->xavg, sizeof(double) * n);
                    memcpy(s->y, s->yavg, sizeof(double) * m);
                }
                memcpy(s->xr, s->x, sizeof(double) * n);
                memcpy(s->yr, s->y, sizeof(double) * m);
                s->S_r = S;
                s->S_prev = INFINITY;
                s->t = 0;
                memset(s->xavg, 0, sizeof(double) * n);
                memset(s->yavg, 0, sizeof(double) * m);
                s->restarts += 1;
            } else {
                s->S_prev = S;
            }
        }
        if (s->mode != MODE_NONE) {
            if (s->k == P->max_iters) { s->status = 1; break; }
            if (P->time_limit_s > 0.0 && now_s() - s->t0 > P->time_limit_s) { s->status = 2; break; }
        }
    }
    return s->status;
}

/* The iterate a finished run returns (current, or the average when the average
 * satisfied the tolerance at a check). */
void orc_get(const orc_state *s, double *x, double *y)
{
    const double *xs = s->returned_average ? s->xavg : s->x;
    const double *ys = s->returned_average ? s->yavg : s->y;
    if (s->prm.method == 1 && s->k > 0) { xs = s->xh; ys = s->yh; }   /* Halpern: T(z), the in-box point */
    if (x) memcpy(x, xs, sizeof(double) * s->lp->n);
    if (y) memcpy(y, ys, sizeof(double) * s->lp->m);
}

/* The internal iterate z = (x, y) (R-PDHG: the current iterate; Halpern: the Halpern
 * sequence, which may leave the box) — test access for the Halpern pins. */
void orc_get_z(const orc_state *s, double *x, double *y)
{
    if (x) memcpy(x, s->x, sizeof(double) * s->lp->n);
    if (y) memcpy(y, s->y, sizeof(double) * s->lp->m);
}

void orc_result_of(orc_state *s, orc_result *r)
{
    double *x = (double *)malloc(sizeof(double) * (s->lp->n ? s->lp->n : 1));
    double *y = (double *)malloc(sizeof(double) * (s->lp->m ? s->lp->m : 1));
    orc_get(s, x, y);
    orc_score_t o;
    score_of(s, x, y, &o);
    r->status = s->status;
    r->returned_average = s->returned_average;
    r->iterations = s->k;
    r->restarts = s->restarts;
    r->pobj = o.pobj; r->dobj = o.dobj; r->gap = fabs(o.pobj - o.dobj);
    r->rp_norm = o.rp; r->rd_norm = o.rd; r->score = o.score;
    r->step_size = s->eta; r->primal_weight = s->omega;
    r->wall_s = now_s() - s->t0;
    free(x); free(y);
}

/* ----------------------------------------------------- Algorithm 1 */

/* z = c - A^T y ("reduced costs"). */
void orc_reduced_costs(const orc_lp *lp, const double *c, const double *y, double *z)
{
    orc_spmv(lp->n, lp->ATp, lp->ATj, lp->ATx, y, z);
    for (int32_t j = 0; j < lp->n; ++j) z[j] = c[j] - z[j];
}

/* Corner model M^ (Algorithm 1 line 2):
 *   lb^_j = x_j if z_j < -eps_abs else lb_j;  ub^_j = x_j if z_j > eps_abs else ub_j;
 *   obj_j = obj_scale * U(seed, j)  (Uniform[0,1]^n; obj_scale P:771-779, S-12).
 * chat may be NULL (caller supplies the objective). */
void orc_corner_model(int32_t n, const double *x, const double *z, const double *l,
                      const double *u, double eps_abs, double obj_scale, uint64_t seed,
                      double *lhat, double *uhat, double *chat, int64_t *fix_lb, int64_t *fix_ub)
{
    int64_t fl = 0, fu = 0;
    for (int32_t j = 0; j < n; ++j) {
        if (z[j] < -eps_abs) { lhat[j] = x[j]; fl++; } else lhat[j] = l[j];
        if (z[j] > eps_abs)  { uhat[j] = x[j]; fu++; } else uhat[j] = u[j];
        if (chat) chat[j] = obj_scale * orc_u01(seed, j);
    }
    *fix_lb = fl;
    *fix_ub = fu;
}

/* Dual corner model (NEXT-4: "similar techniques ... to reduce the number of dual
 * superbasic variables"; readings D-1..D-4).  From the phase-1
 * point x, each column is classified against the original bounds with tolerance eps:
 *   off   (x - l > eps and u - x > eps): lhat = -inf, uhat = +inf   -> its dual row
 *         becomes the equality z_j = 0 (complementary slackness with x);
 *   lower (x - l <= eps, l finite):       lhat = l,    uhat = +inf   -> z_j >= 0;
 *   upper (otherwise, at a finite u):     lhat = -inf, uhat = u      -> z_j <= 0;
 * so the model's dual feasible set is M's dual optimal face for x (D-1); A, b, c are
 * unchanged (D-2).  Returns the three class counts in cnt[3]. */
void orc_dual_corner_model(int32_t n, const double *x, const double *l, const double *u, double eps_abs,
                           double *lhat, double *uhat, int64_t *cnt)
{
    cnt[0] = cnt[1] = cnt[2] = 0;
    for (int32_t j = 0; j < n; ++j) {
        if (x[j] - l[j] > eps_abs && u[j] - x[j] > eps_abs) {
            lhat[j] = -INFINITY; uhat[j] = INFINITY; cnt[0]++;
        } else if (x[j] - l[j] <= eps_abs && l[j] > -INFINITY) {
            lhat[j] = l[j]; uhat[j] = INFINITY; cnt[1]++;
        } else {
            lhat[j] = -INFINITY; uhat[j] = u[j]; cnt[2]++;
        }
    }
}

/* Corner model row senses: an inequality row whose slack has a
 * non-trivial reduced cost (|y_i| > eps_abs) becomes an equality ("fixing the slack
 * upper bound to zero"); returns the number of rows changed. */
int64_t orc_corner_senses(int32_t m, const int8_t *sense, const double *y, double eps_abs, int8_t *shat)
{
    int64_t k = 0;
    for (int32_t i = 0; i < m; ++i) {
        int s = sense ? sense[i] : 0;
        if (s != 0 && fabs(y[i]) > eps_abs) { shat[i] = 0; k++; }
        else shat[i] = (int8_t)s;
    }
    return k;
}

/* Off-bound test (Fig. 1 axis P:336; S-10): strictly inside by > tol
 * on both sides; an infinite bound never counts as "at bound". */
static int off_bound(double x, double lo, double hi, double tol)
{
    return (x - lo > tol) && (hi - x > tol);
}

/* Corner statistics a10 (S-9):
 *   p = #off-bound (tol eps_abs, bounds [l,u]); p_strict (tol 0); p^ w.r.t. [l^,u^];
 *   d = #{|z_j| <= eps_abs};  cand = #{off_j and |z_j| < eps_abs};
 *   est_primal = max(p - m, 0); est_dual = max(m - d, 0);
 *   candidate <=> cand >= max(2m, floor). z and lhat/uhat may be NULL. */
void orc_stats(int32_t m, int32_t n, const double *x, const double *z, const double *l,
               const double *u, const double *lhat, const double *uhat, double eps_abs,
               int64_t floor_, orc_stats_t *st)
{
    memset(st, 0, sizeof(*st));
    for (int32_t j = 0; j < n; ++j) {
        int off = off_bound(x[j], l[j], u[j], eps_abs);
        st->off_bound += off;
        st->off_bound_strict += off_bound(x[j], l[j], u[j], 0.0);
        if (lhat && uhat) st->off_bound_model += off_bound(x[j], lhat[j], uhat[j], eps_abs);
        if (z) {
            st->zero_rc += fabs(z[j]) <= eps_abs;
            st->candidates += off && fabs(z[j]) < eps_abs;
        }
    }
    st->est_primal_pushes = st->off_bound > m ? st->off_bound - m : 0;
    st->est_dual_pushes = z ? (m > st->zero_rc ? m - st->zero_rc : 0) : 0;
    int64_t thr = 2 * (int64_t)m > floor_ ? 2 * (int64_t)m : floor_;
    st->is_candidate = z ? st->candidates >= thr : 0;
}
