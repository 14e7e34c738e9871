/*
 * bmc.h -- C-ABI of the B200-native batch multi-convex trajectory optimiser
 * (the batched alternating-minimisation iteration of arXiv 2109.13030,
 * Rastgar et al., "GPU Accelerated Batch Multi-Convex Trajectory
 * Optimization for a Rectangular Holonomic Mobile Robot").
 *
 * Citations "P:n" are lines of the paper's LaTeX source; equation
 * numbers follow its source order.  Readings "Gk" of ambiguous passages are
 * listed in DESIGN.md ("Readings of the paper").
 *
 * What a solve computes, per batch instance l ("l trajectory
 * optimizations in parallel"; all instances share the boundary conditions
 * and the obstacles; they differ in their initial samples):
 *
 *   xi1 = (c_x, c_c, c_y, c_s), xi2 = c_psi: Bernstein coefficients of x, the
 *   copy c ~ cos psi, y, the copy s ~ sin psi, and psi (Eq. 8-9).
 *   Initialisation (G15): xi2 := c_psi^0, xi3/xi4 := closed forms on
 *   the initial trajectory (c_c = c_s = 0), lambda := lambda_in or 0.
 *   Then `iters` AM iterations, each:
 *     1. xi1 <- KKT solve of Eq. 13/17 (one-shot form Eq. 4)
 *     2. theta = atan2(P c_s, P c_c); xi2 <- KKT solve of Eq. 19
 *     3. alpha_ij, alpha_v, alpha_a closed forms, Eq. 21a-c
 *     4. d_ij >= 1, d_v, d_a in [0,1] closed forms, Eq. 22a-c + clip
 *     5. lambda <- lambda - rho F^T (F xi1 - g)             Eq. 23a (G3)
 *        lambda_psi <- lambda_psi - rho_psi P^T (P xi2 - theta)  Eq. 23b (G4)
 *   Outputs: coefficients, multipliers, residuals r1 = ||F xi1 - g||_2 and
 *   r_psi = ||theta - P xi2||_2 (Eq. 12), cost
 *   J = sum_t (xdd^2 + ydd^2 + psidd^2) (Eq. 1a) and the batch argmin
 *   ("best cost trajectory"; rule G17).
 *
 * Threading / streams: every function is re-entrant across contexts.  Calls
 * of bmc_solve on ONE context must be ordered on one stream (they share the
 * context's argmin workspace); bmc_solve_host has a workspace of its own and
 * may overlap them, also from another thread (the context's host-side state is
 * locked; host solves on one context run one at a time).  A constant blob
 * uploaded on one stream is waited for (event) by solves on another until the
 * upload is known complete.  CUDA graphs: once a context has solved a given
 * obstacle count (constants uploaded and complete, shared-memory opt-in set),
 * bmc_solve issues only the kernel launch on the stream and can be captured
 * (tests/test_gpu_context.py).
 * bmc_last_error() is thread-local.
 *
 * Determinism: an instance's outputs depend on its own inputs, the context and
 * the team size (warps per instance, bmc_problem.team) -- never on B, on its
 * position in the batch, on index_base or on the other instances.  With a
 * fixed team a sharded solve reproduces the unsharded one bit for bit.
 */
#ifndef BMC_H
#define BMC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes (int32) ------------------------------------------------ */
#define BMC_OK 0
#define BMC_EINVAL 1      /* invalid argument; bmc_last_error() names it          */
#define BMC_ESINGULAR 2   /* boundary rows rank-deficient or KKT singular */
#define BMC_ECUDA 3       /* CUDA runtime error (message from cudaGetErrorString) */
#define BMC_ENOMEM 4      /* host or device allocation failed                      */

/* Opaque context, owned by the library: host fp64 constants, the per-n_obs
 * device constant blobs (Q_bar depends on n through F^T F) and the
 * argmin workspace. */
typedef struct bmc_ctx bmc_ctx;

/* Stream handle: a cudaStream_t / CUstream (NULL = legacy default stream). */
typedef struct CUstream_st* bmc_stream_t;

/* Problem constants shared by every solve on the context (bmc_setup). */
typedef struct {
  int32_t q;               /* time samples on [0, T], t_k = k T/(q-1); 3 <= q <= 128      */
  double T;                /* horizon [s] > 0 ("around 30s")                        */
  int32_t degree;          /* Bernstein degree, must be 10 (n_v = 11; G12)               */
  int32_t m;               /* footprint circles, 1 <= m <= 8                      */
  const double* r;         /* [m] circle offsets along the heading axis [m]; copied      */
  double v_max, a_max;     /* Eq. 1c bounds, > 0                                         */
  double rho, rho_psi;     /* Eq. 12 / Eq. 19 penalty weights, > 0 (G5, G14)             */
  double w_copy;           /* smoothness weight of the c, s blocks in Q, >= 0 (G10)      */
  uint32_t boundary_mask;  /* bits x(0), x'(0), x''(0), x(T), x'(T), x''(T); default 0x3F */
  int32_t alpha_rule;      /* 0: alpha = atan2(yt, xt) (Eq. 21a); 1: atan2(a yt, b xt) (G8) */
  double res_tol;          /* feasibility threshold tau on r1 for the argmin (G17)       */
  int32_t device;          /* CUDA device ordinal                                        */
} bmc_params;

/* One batch (or one shard of a batch) to solve. */
typedef struct {
  int64_t B;               /* instances in this call, >= 1                                */
  int64_t index_base;      /* global index of instance 0 (sharded solves); B+base < 2^30 */
  int32_t n_obs;           /* obstacles n, 0 <= n <= 160                                  */
  int32_t iters;           /* AM iterations K >= 0 (K = 0 evaluates the initialisation)  */
  double bnd[3][6];        /* x, y, psi  x  (p0, v0, a0, pT, vT, aT); selected by the mask */
  const float* obs_xy;     /* [n][2][q] obstacle centre trajectories x_j(t_k), y_j(t_k)  */
  const float* obs_ab;     /* [n][2] effective (inflated) semi-axes a_j, b_j > 0 (G13)   */
  const float* init;       /* [B][3][11] initial Bernstein coefficients c_x, c_y, c_psi  */
  const float* lambda_in;  /* [B][5][11] warm-start multipliers (lambda, lambda_psi) or NULL */
  int32_t team;            /* warps per instance: 1, 2 or 4; 0 = chosen from B (bmc_team_for).
                              The fp64 partial sums of an instance are combined in warp
                              order, so its output bits depend on the team size: pass the
                              team of the whole batch when solving shards of it. */
} bmc_problem;

/* Outputs.  Layouts are row-major fp32 (int64 for best). */
typedef struct {
  float* coeffs;           /* [B][5][11] c_x, c_c, c_y, c_s, c_psi (Bernstein)            */
  float* lambda_out;       /* [B][5][11] final lambda (4 blocks) and lambda_psi, or NULL */
  float* residual;         /* [B][2] r1 = ||F xi1 - g||_2, r_psi = ||theta - P xi2||_2   */
  float* cost;             /* [B] J = sum_t (xdd^2 + ydd^2 + psidd^2)                     */
  float* res_trace;        /* [B][iters] r1 after every iteration, or NULL               */
  int64_t* best;           /* [2] {global best index, packed key}:
                              key = infeasible << 62 | fp32bits(v) << 30 | index,
                              infeasible = !(r1 <= tau) or non-finite; v = J if feasible
                              else r1; the minimum key wins (ties -> lowest index) */
} bmc_result;

/* Build the context: Bernstein basis, boundary rows, per-channel KKT
 * inverses in fp64 (Eq. 3-4 "constant" inverse).  The device is
 * params->device.  Returns BMC_EINVAL (bad parameter, message says which),
 * BMC_ESINGULAR (the KKT is singular even with an obstacle), BMC_ECUDA or
 * BMC_ENOMEM; *out is NULL on error.  The KKT depends on n_obs through F^T F:
 * bmc_solve returns BMC_ESINGULAR for an n_obs that makes it singular (n_obs = 0
 * with no position row in boundary_mask). */
int32_t bmc_setup(const bmc_params* params, bmc_ctx** out);

/* Device solve, asynchronous on `stream`.  Every pointer in `prob` and `res`
 * is a caller-owned DEVICE pointer on params.device (contiguous, 16-byte
 * aligned); the library reads/writes them only during the stream-ordered
 * execution of this call and never frees or retains them.  The first solve
 * with a new n_obs builds that n's constants on the host and uploads them
 * asynchronously on `stream`; the context keeps the constants of at most 8
 * obstacle counts (evicting the least recently used synchronises the device).
 * Errors: BMC_EINVAL (B < 1, n or K out of range, NULL required pointer,
 * misaligned pointer), BMC_ESINGULAR (the KKT of this n_obs is singular),
 * BMC_ECUDA (launch failure), BMC_ENOMEM. */
int32_t bmc_solve(bmc_ctx* ctx, const bmc_problem* prob, const bmc_result* res,
                  bmc_stream_t stream);

/* End-to-end solve with HOST pointers; synchronous.  Same layouts and errors
 * as bmc_solve.  The obstacle arrays (read by every CTA) and res_trace are
 * staged through context-owned device buffers (cudaMemcpyAsync on the
 * context's stream).  Every other array that lies in page-locked host memory
 * (cudaHostAlloc / cudaHostRegister, e.g. torch pin_memory) is accessed in
 * place by the kernel: init and lambda_in are read once per instance and the
 * outputs written once, over PCIe inside this call (no separate copy);
 * pageable arrays are staged like the obstacles. */
int32_t bmc_solve_host(bmc_ctx* ctx, const bmc_problem* prob_host, const bmc_result* res_host);

/* ---- multi-GPU best-of-batch exchange ----------------------
 * A batch sharded over ranks (bmc_problem.index_base = first global index of
 * the shard) has one global argmin: the minimum packed key over all ranks.
 * Record layout (BMC_RECORD_WORDS int64 per rank, device memory):
 *   word 0 = packed key, words 1.. = as fp32: the 55 coefficients of that
 *   instance (c_x, c_c, c_y, c_s, c_psi), then its residuals r1, r_psi and its
 *   cost J (floats 55..57; zero when `residual` / `cost` are NULL), zero padded.
 * bmc_pack_best writes this rank's record from the `best`, `coeffs` and
 * (optionally) `residual` and `cost` of a finished bmc_solve (stream-ordered
 * after it) -- on one GPU this is also the device-side gather of the best
 * instance's outputs into one 256-byte block; the caller all-gathers the
 * records (e.g. NCCL all_gather over NVLink); bmc_select_best picks the
 * minimum key and writes best_out[2] = {global index, key} and
 * coeffs_out[55] (the coefficients; the whole record is in `records`).  Both are one-warp kernels on `stream`.  A rank with an
 * empty shard contributes best = {0, -1} (key ~0: never the minimum unless
 * every rank is empty); bmc_pack_best then reads no coefficients.  Errors:
 * BMC_EINVAL (NULL pointer, nranks < 1), BMC_ECUDA (launch failure); both
 * set bmc_last_error(). */
#define BMC_RECORD_WORDS 32
int32_t bmc_pack_best(const int64_t* best, const float* coeffs, const float* residual, const float* cost,
                      int64_t index_base, int64_t* record, bmc_stream_t stream);
int32_t bmc_select_best(const int64_t* records, int32_t nranks, int64_t* best_out, float* coeffs_out,
                        bmc_stream_t stream);

/* ---- STOMP-style initial samples on the device ---------
 * "Our batch optimizer was always initialized with a Gaussian
 * distribution proposed in [STOMP] centered around a straight-line
 * trajectory."  Reading G28: init[l] = the constant-velocity
 * segment from (bnd[0][0], bnd[1][0]) to (bnd[0][3], bnd[1][3]) as degree-10
 * Bernstein control points (c_k = p0 + (pT - p0) k / 10), plus on the control
 * points 3..7 (which enter no position, velocity or acceleration at either end)
 * the STOMP smoothness noise s L z, L L^T = R^-1 / max diag(R^-1), R = D^T D
 * with D the second difference of the control polygon restricted to those
 * points; s = sigma_x for x, sigma_y for y; c_psi = 0.  z: 10 standard
 * normals of global instance g = index_base + l from Philox4x32-10 (key =
 * seed, counters (g, stream + j), j = 0..2) through Box-Muller in fp64 -- the
 * same counter-based stream as the test oracle, so a sample depends only on
 * (seed, stream, g), never on the batch split.  line_first: global instance 0
 * is the unperturbed segment.  Output: device init [B][3][11] fp32
 * (bmc_problem.init layout), caller-owned.  One kernel on `stream`.
 * Errors: BMC_EINVAL (B < 0, init NULL with B > 0, non-finite bnd or sigma,
 * degree != 10), BMC_ECUDA (launch failure). */
typedef struct {
  int64_t B, index_base;
  uint64_t seed, stream;
  double bnd[3][6];        /* x, y, psi x (p0, v0, a0, pT, vT, aT); p0 and pT of x, y are used */
  double sigma_x, sigma_y; /* [m] */
  int32_t line_first;
} bmc_sample_params;
int32_t bmc_sample_init(bmc_ctx* ctx, const bmc_sample_params* sp, float* init, bmc_stream_t stream);

/* The team size (warps per instance) bmc_solve picks for a batch of B
 * instances with team = 0 on this context's device: 1, 2 or 4; 0 if B < 1. */
int32_t bmc_team_for(const bmc_ctx* ctx, int64_t B);

/* Kernel launches issued by the last bmc_solve / bmc_solve_host on ctx. */
int32_t bmc_last_launch_count(const bmc_ctx* ctx);

/* Release everything owned by the context (NULL is a no-op). */
void bmc_destroy(bmc_ctx* ctx);

/* Message of the last error on the calling thread ("" if none). */
const char* bmc_last_error(void);

/* ABI version (major * 100 + minor). */
int32_t bmc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BMC_H */
