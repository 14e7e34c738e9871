/*
 * oracle.h -- plain fp64 CPU oracle for the batched alternating-minimisation
 * (AM) iteration of arXiv 2109.13030 (Rastgar et al., "GPU Accelerated Batch
 * Multi-Convex Trajectory Optimization for a Rectangular Holonomic Mobile
 * Robot").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2109_13030_b200/) never links, imports or calls it,
 * and this code shares nothing with it.
 *
 * Citations "P:n" are lines of /root/reference/PAPER.md (LaTeX source);
 * equation numbers follow the source order.  The readings
 * of ambiguous passages are the G-numbers of SURVEY.md §8c, listed again in
 * DESIGN.md.
 *
 * Layout conventions (all arrays row-major, fp64, caller-owned):
 *   basis      P, Pd, Pdd           [q][nv]          (Eq. 8)
 *   xi1        (c_x, c_c, c_y, c_s)  [4 nv]
 *   xi2        c_psi                 [nv]
 *   F          [rows][4 nv], rows = 2 * R, R = 2q + m n q + q   (Eq. 10-11)
 *              per channel: velocity q | acceleration q | collision
 *              (for j < n: for i < m: q rows) | copy-consistency q;
 *              x channel first (columns c_x, c_c), then y (columns c_y, c_s)
 *   g          [rows] same order                    (Eq. 10-11)
 *   bnd        [3][6]: x, y, psi  x  (p0, v0, a0, pT, vT, aT)
 *   obs_xy     [n][2][q]             obstacle centre trajectories
 *   obs_ab     [n][2]                effective semi-axes (a_j, b_j)
 *   init       [B][3][nv]            (c_x, c_y, c_psi) initial Bernstein coeffs
 *   coeffs     [B][5][nv]            (c_x, c_c, c_y, c_s, c_psi)
 *   lambda     [B][5][nv]            (lambda (4 nv), lambda_psi (nv))
 */
#ifndef BMC_ORACLE_H
#define BMC_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int q;                   /* time samples on [0, T], t_k = k T / (q - 1)     */
  double T;                /* horizon [s]                                      */
  int degree;              /* Bernstein degree, nv = degree + 1                */
  int m;                   /* footprint circles                                */
  const double* r;         /* [m] circle offsets along the heading     */
  double v_max, a_max;     /* Eq. 1c bounds                                    */
  double rho, rho_psi;     /* Eq. 12 / Eq. 19 / Eq. 23 weights (G5)            */
  double w_copy;           /* smoothness weight on the c, s blocks (G10)       */
  unsigned boundary_mask;  /* bit0 x(0) bit1 x'(0) bit2 x''(0) bit3 x(T) ... (G11) */
  int alpha_rule;          /* 0: alpha = atan2(yt, xt) (Eq. 21a); 1: atan2(a yt, b xt) (G8) */
  int lampsi_printed_sign; /* 0: gradient-consistent Eq. 23b (G4); 1: as printed */
  double res_tol;          /* feasibility threshold tau on r1 (G17)            */
  /* fp32 rounding model (parity harness only):
   * 0 = the oracle proper (fp64 throughout).  1 = the same iteration with every
   * quantity that the product path holds in fp32 rounded to fp32 at the point
   * where it is formed (round to nearest); with noise_seed != 0 those roundings
   * are stochastic (up or down with probability given by the distance to the
   * two fp32 neighbours, keyed by seed, instance, iteration, site, sample), so
   * an ensemble of seeds measures how far fp32 rounding alone moves the result. */
  int fp32_model;
  unsigned long long noise_seed;
} or_params;

typedef struct or_ctx or_ctx;

/* error codes */
#define OR_OK 0
#define OR_EINVAL 1
#define OR_ESINGULAR 2
#define OR_ENOMEM 3

/* Bernstein basis and its time derivatives at t_k = k T/(q-1) (Eq. 8). */
int or_basis(int q, double T, int degree, double* P, double* Pd, double* Pdd);

/* Problem construction for n obstacles: F, Q-bar, the two KKT inverses. */
or_ctx* or_create(const or_params* p, int n_obs, int* err);
void or_destroy(or_ctx* c);
int or_nv(const or_ctx* c);
int or_nb(const or_ctx* c);
int or_rows(const or_ctx* c);
const double* or_F(const or_ctx* c);        /* [rows][4nv]            */
const double* or_Qbar(const or_ctx* c);     /* [4nv][4nv]             */
const double* or_A(const or_ctx* c);        /* [nb][nv] boundary rows */
const double* or_kkt1(const or_ctx* c);     /* [4nv+2nb]^2 matrix     */
const double* or_kkt1_inv(const or_ctx* c);
const double* or_kktpsi(const or_ctx* c);   /* [nv+nb]^2              */
const double* or_kktpsi_inv(const or_ctx* c);
const double* or_basis_P(const or_ctx* c);  /* [q][nv] */
const double* or_basis_Pd(const or_ctx* c);
const double* or_basis_Pdd(const or_ctx* c);

/* Whole batch solve: K AM iterations per instance (OpenMP over instances).
 * res_trace [B][K] may be NULL; lambda_in may be NULL (cold start).
 * best[0] = global index (index_base + l) of the best instance,
 * best[1] = its packed key (bit 62 infeasible | fp32 bits of value << 30 | index). */
int or_solve(or_ctx* c, int B, int K, long long index_base, const double* bnd,
             const double* obs_xy, const double* obs_ab, const double* init,
             const double* lambda_in, double* coeffs, double* lambda_out,
             double* residual, double* cost, double* res_trace, long long* best,
             int nthreads);

/* Single instance with full per-iteration traces (k = 0 is the initialisation).
 * xi1_tr [K+1][4nv], xi2_tr [K+1][nv], lam_tr [K+1][5nv], g_tr [K+1][rows],
 * theta_tr [K+1][q], r1_tr [K+1], rpsi_tr [K+1]; any pointer may be NULL. */
int or_trace_instance(or_ctx* c, int K, const double* bnd, const double* obs_xy,
                      const double* obs_ab, const double* init, const double* lambda_in,
                      double* xi1_tr, double* xi2_tr, double* lam_tr, double* g_tr,
                      double* theta_tr, double* r1_tr, double* rpsi_tr);

/* Sub-step closed forms (Eq. 21-22), exposed for the grid pins. */
void or_project_obstacle(double xt, double yt, double a, double b, int rule,
                         double* alpha, double* d);
void or_project_bound(double vx, double vy, double bound, double* alpha, double* d);

/* Pieces of the iteration on explicit F and g (Eq. 12, 17, 23a). */
double or_penalty(const or_ctx* c, const double* xi1, const double* g); /* 0.5||F xi1 - g||^2 */
void or_lambda_step(const or_ctx* c, const double* lam, const double* xi1,
                    const double* g, double* lam_out);
int or_xi1_step(const or_ctx* c, const double* lam, const double* g,
                const double* bnd, double* xi1_out);
int or_xi2_step(const or_ctx* c, const double* lampsi, const double* theta,
                const double* bnd, double* xi2_out);

/* STOMP-style initial samples (sampler.c, reading G28).
 * Philox4x32-10 block; the STOMP covariance factor (L [nf][nf] lower, nf = degree - 5);
 * the 12 normals of instance g (10 used); init [B][3][nv] = line + noise. */
#include <stdint.h>
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
int or_stomp_factor(int degree, double* L, int* nfree);
void or_stomp_normals(uint64_t seed, uint64_t stream, long long g, double z[12]);
int or_sample_init(int degree, long long B, long long index_base, uint64_t seed, uint64_t stream,
                   const double* bnd, double sigma_x, double sigma_y, int line_first, double* init);

#ifdef __cplusplus
}
#endif
#endif
