/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle of the batched
 * AM iteration of arXiv 2109.13030 (see oracle.h for layouts).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs, never by the product path.
 * Shares no code, header, table or constant generator with the CUDA path.
 *
 * Structure on purpose differs from the GPU path: F and g are materialised
 * explicitly (Eq. 10-11), F^T F and F^T g are dense products,
 * the KKT systems of Eq. 3/4 are inverted once by Gauss-Jordan
 * and applied to [-q_bar; b] per instance, and every closed form uses libm
 * atan2 / cos / sin literally (Eq. 21-22).
 *
 * Readings of ambiguous passages:
 *   G1  KKT right-hand side is (-q_bar, b)              (Eq. 3)
 *   G2  q_bar = -lambda - rho F^T g                      (Eq. 17)
 *   G3  lambda <- lambda - rho F^T (F xi1 - g)           (Eq. 23a)
 *   G4  lambda_psi <- lambda_psi - rho_psi P^T (P xi2 - theta)  (Eq. 23b, P:575;
 *       printed sign selectable with lampsi_printed_sign)
 *   G5  rho_psi in the heading QP as well                (Eq. 19)
 *   G6  d_v, d_a clipped to [0,1]; d_ij >= 1
 *   G7  g carries v_max and a_max                        (Eq. 6)
 *   G8  alpha_ij = atan2(yt, xt) (rule 0) or atan2(a yt, b xt) (rule 1)
 *   G9  alpha, d use cos/sin psi; F rows use the copies c, s
 *   G10 copy blocks carry smoothness weight w_copy (default 0)
 *   G11 boundary rows {x, x', x''} at t=0 and t=T selected by a mask
 *   G15 xi3, xi4 initialised by the closed forms on the initial trajectory;
 *       the initial copies c_c = c_s = 0
 *   G17 best = argmin J among r1 <= tau, else argmin r1, ties -> lowest index
 *   G18 atan2(0, 0) := 0
 */
#include "oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

struct or_ctx {
  or_params p;
  double* r;   /* copy of the offsets */
  int n, nv, q, m, nb, R, rows, cols;
  int bsel[6];
  double *P, *Pd, *Pdd; /* [q][nv] */
  double *P32, *Pd32, *Pdd32; /* fp32 model only: the basis rounded to fp32 */
  double* A;            /* [nb][nv] */
  double* F;            /* [rows][cols] */
  double* Qbar;         /* [cols][cols] */
  double *K1, *K1inv;   /* (cols + 2 nb)^2 */
  double *Kp, *Kpinv;   /* (nv + nb)^2 */
};

/* ------------------------------------------------------------------ basis */

static double binom(int n, int k) {
  if (k < 0 || k > n) return 0.0;
  double v = 1.0;
  for (int i = 1; i <= k; ++i) v = v * (double)(n - k + i) / (double)i;
  return v;
}

/* Bernstein polynomial B_{k,n}(tau) = C(n,k) tau^k (1-tau)^(n-k). */
static double bern(int n, int k, double tau) {
  if (k < 0 || k > n) return 0.0;
  return binom(n, k) * pow(tau, k) * pow(1.0 - tau, n - k);
}

/* Eq. 8: x = P c, xdot = Pd c, xddot = Pdd c; the basis kind,
 * degree and sampling are the reading G12 (Bernstein, t_k = kT/(q-1)). */
int or_basis(int q, double T, int degree, double* P, double* Pd, double* Pdd) {
  if (degree < 2 || q < degree + 1 || !(T > 0.0)) return OR_EINVAL;
  const int n = degree, nv = degree + 1;
  for (int i = 0; i < q; ++i) {
    const double tau = (double)i / (double)(q - 1);
    for (int k = 0; k < nv; ++k) {
      P[i * nv + k] = bern(n, k, tau);
      Pd[i * nv + k] = (double)n / T * (bern(n - 1, k - 1, tau) - bern(n - 1, k, tau));
      Pdd[i * nv + k] = (double)n * (double)(n - 1) / (T * T) *
                        (bern(n - 2, k - 2, tau) - 2.0 * bern(n - 2, k - 1, tau) +
                         bern(n - 2, k, tau));
    }
  }
  return OR_OK;
}

/* ------------------------------------------------------- dense linear alg */

/* Gauss-Jordan inverse with partial pivoting.  Returns OR_ESINGULAR when a
 * pivot is below 1e-13 of the largest entry. */
static int gj_inverse(const double* M, int N, double* Minv) {
  double* a = (double*)malloc(sizeof(double) * (size_t)N * (size_t)(2 * N));
  if (!a) return OR_ENOMEM;
  double amax = 0.0;
  for (int i = 0; i < N; ++i) {
    for (int j = 0; j < N; ++j) {
      a[i * 2 * N + j] = M[i * N + j];
      if (fabs(M[i * N + j]) > amax) amax = fabs(M[i * N + j]);
    }
    for (int j = 0; j < N; ++j) a[i * 2 * N + N + j] = (i == j) ? 1.0 : 0.0;
  }
  for (int col = 0; col < N; ++col) {
    int piv = col;
    for (int i = col + 1; i < N; ++i)
      if (fabs(a[i * 2 * N + col]) > fabs(a[piv * 2 * N + col])) piv = i;
    if (!(fabs(a[piv * 2 * N + col]) > 1e-13 * amax)) {
      free(a);
      return OR_ESINGULAR;
    }
    if (piv != col)
      for (int j = 0; j < 2 * N; ++j) {
        double t = a[col * 2 * N + j];
        a[col * 2 * N + j] = a[piv * 2 * N + j];
        a[piv * 2 * N + j] = t;
      }
    const double d = a[col * 2 * N + col];
    for (int j = 0; j < 2 * N; ++j) a[col * 2 * N + j] /= d;
    for (int i = 0; i < N; ++i) {
      if (i == col) continue;
      const double f = a[i * 2 * N + col];
      if (f == 0.0) continue;
      for (int j = 0; j < 2 * N; ++j) a[i * 2 * N + j] -= f * a[col * 2 * N + j];
    }
  }
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) Minv[i * N + j] = a[i * 2 * N + N + j];
  free(a);
  return OR_OK;
}

/* ----------------------------------------------------------------- create */

int or_nv(const or_ctx* c) { return c->nv; }
int or_nb(const or_ctx* c) { return c->nb; }
int or_rows(const or_ctx* c) { return c->rows; }
const double* or_F(const or_ctx* c) { return c->F; }
const double* or_Qbar(const or_ctx* c) { return c->Qbar; }
const double* or_A(const or_ctx* c) { return c->A; }
const double* or_kkt1(const or_ctx* c) { return c->K1; }
const double* or_kkt1_inv(const or_ctx* c) { return c->K1inv; }
const double* or_kktpsi(const or_ctx* c) { return c->Kp; }
const double* or_kktpsi_inv(const or_ctx* c) { return c->Kpinv; }
const double* or_basis_P(const or_ctx* c) { return c->P; }
const double* or_basis_Pd(const or_ctx* c) { return c->Pd; }
const double* or_basis_Pdd(const or_ctx* c) { return c->Pdd; }

void or_destroy(or_ctx* c) {
  if (!c) return;
  free(c->r);
  free(c->P);
  free(c->Pd);
  free(c->Pdd);
  free(c->P32);
  free(c->Pd32);
  free(c->Pdd32);
  free(c->A);
  free(c->F);
  free(c->Qbar);
  free(c->K1);
  free(c->K1inv);
  free(c->Kp);
  free(c->Kpinv);
  free(c);
}

/* row index of the collision row (obstacle j, circle i, time t) inside a
 * channel block: velocity q | acceleration q | collision m n q | copy q */
static int row_coll(const or_ctx* c, int j, int i, int t) {
  return 2 * c->q + (j * c->m + i) * c->q + t;
}
static int row_copy(const or_ctx* c, int t) { return 2 * c->q + c->m * c->n * c->q + t; }

or_ctx* or_create(const or_params* p, int n_obs, int* err) {
  int e = OR_OK;
  or_ctx* c = NULL;
  if (!p || p->degree < 2 || p->q < p->degree + 1 || !(p->T > 0.0) || p->m < 1 || !p->r ||
      n_obs < 0 || !(p->rho > 0.0) || !(p->rho_psi > 0.0) || !(p->v_max > 0.0) ||
      !(p->a_max > 0.0) || p->w_copy < 0.0 || (p->boundary_mask & ~0x3Fu) ||
      (p->fp32_model && p->degree + 1 > 32)) {
    e = OR_EINVAL;
    goto fail;
  }
  c = (or_ctx*)calloc(1, sizeof(or_ctx));
  if (!c) {
    e = OR_ENOMEM;
    goto fail;
  }
  c->p = *p;
  c->n = n_obs;
  c->q = p->q;
  c->m = p->m;
  c->nv = p->degree + 1;
  c->r = (double*)malloc(sizeof(double) * (size_t)p->m);
  memcpy(c->r, p->r, sizeof(double) * (size_t)p->m);
  c->p.r = c->r;
  const int q = c->q, nv = c->nv, m = c->m, n = c->n;
  c->R = 2 * q + m * n * q + q;
  c->rows = 2 * c->R;
  c->cols = 4 * nv;
  c->P = (double*)malloc(sizeof(double) * (size_t)q * nv);
  c->Pd = (double*)malloc(sizeof(double) * (size_t)q * nv);
  c->Pdd = (double*)malloc(sizeof(double) * (size_t)q * nv);
  or_basis(q, p->T, p->degree, c->P, c->Pd, c->Pdd);
  if (p->fp32_model) { /* fp32 model: the evaluation basis is held in fp32 */
    c->P32 = (double*)malloc(sizeof(double) * (size_t)q * nv);
    c->Pd32 = (double*)malloc(sizeof(double) * (size_t)q * nv);
    c->Pdd32 = (double*)malloc(sizeof(double) * (size_t)q * nv);
    for (int i = 0; i < q * nv; ++i) {
      c->P32[i] = (double)(float)c->P[i];
      c->Pd32[i] = (double)(float)c->Pd[i];
      c->Pdd32[i] = (double)(float)c->Pdd[i];
    }
  }

  /* boundary rows A: "first and last rows of P and its derivatives" (G11) */
  c->nb = 0;
  for (int bit = 0; bit < 6; ++bit)
    if (p->boundary_mask & (1u << bit)) c->bsel[c->nb++] = bit;
  c->A = (double*)calloc((size_t)(c->nb > 0 ? c->nb : 1) * nv, sizeof(double));
  for (int r = 0; r < c->nb; ++r) {
    const int bit = c->bsel[r];
    const double* src = (bit % 3 == 0) ? c->P : (bit % 3 == 1) ? c->Pd : c->Pdd;
    const int t = (bit < 3) ? 0 : q - 1;
    for (int k = 0; k < nv; ++k) c->A[r * nv + k] = src[t * nv + k];
  }

  /* F (Eq. 10-11): per channel [A_v 0; A_a 0; A_ob; [0 P]] on (pos, copy) */
  const int rows = c->rows, cols = c->cols, R = c->R;
  c->F = (double*)calloc((size_t)rows * cols, sizeof(double));
  if (!c->F) {
    e = OR_ENOMEM;
    goto fail;
  }
  for (int ch = 0; ch < 2; ++ch) {
    const int r0 = ch * R, c0 = ch * 2 * nv; /* pos block c0.., copy block c0+nv.. */
    for (int t = 0; t < q; ++t)
      for (int k = 0; k < nv; ++k) {
        c->F[(size_t)(r0 + t) * cols + c0 + k] = c->Pd[t * nv + k];      /* A_v */
        c->F[(size_t)(r0 + q + t) * cols + c0 + k] = c->Pdd[t * nv + k]; /* A_a */
        c->F[(size_t)(r0 + row_copy(c, t)) * cols + c0 + nv + k] = c->P[t * nv + k];
      }
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i)
        for (int t = 0; t < q; ++t)
          for (int k = 0; k < nv; ++k) {
            const size_t row = (size_t)(r0 + row_coll(c, j, i, t));
            c->F[row * cols + c0 + k] = c->P[t * nv + k];                 /* P     */
            c->F[row * cols + c0 + nv + k] = c->r[i] * c->P[t * nv + k];  /* r_i P */
          }
  }

  /* Q = blkdiag(Pdd^T Pdd, w_copy Pdd^T Pdd, Pdd^T Pdd, w_copy Pdd^T Pdd) (G10);
   * Q_bar = Q + rho F^T F (Eq. 17) by a dense product. */
  c->Qbar = (double*)calloc((size_t)cols * cols, sizeof(double));
  for (int blk = 0; blk < 4; ++blk) {
    const double w = (blk % 2 == 0) ? 1.0 : p->w_copy;
    for (int a = 0; a < nv; ++a)
      for (int b = 0; b < nv; ++b) {
        double s = 0.0;
        for (int t = 0; t < q; ++t) s += c->Pdd[t * nv + a] * c->Pdd[t * nv + b];
        c->Qbar[(blk * nv + a) * cols + blk * nv + b] += w * s;
      }
  }
  for (int row = 0; row < rows; ++row) {
    const double* f = c->F + (size_t)row * cols;
    for (int a = 0; a < cols; ++a) {
      if (f[a] == 0.0) continue;
      for (int b = 0; b < cols; ++b) c->Qbar[a * cols + b] += p->rho * f[a] * f[b];
    }
  }

  /* KKT of Eq. 3 for xi1: [[Q_bar, A_full^T], [A_full, 0]], A_full acts on c_x, c_y */
  const int N1 = cols + 2 * c->nb;
  c->K1 = (double*)calloc((size_t)N1 * N1, sizeof(double));
  c->K1inv = (double*)calloc((size_t)N1 * N1, sizeof(double));
  for (int a = 0; a < cols; ++a)
    for (int b = 0; b < cols; ++b) c->K1[a * N1 + b] = c->Qbar[a * cols + b];
  for (int ch = 0; ch < 2; ++ch)
    for (int r = 0; r < c->nb; ++r)
      for (int k = 0; k < nv; ++k) {
        const int row = cols + ch * c->nb + r, col = ch * 2 * nv + k;
        c->K1[row * N1 + col] = c->A[r * nv + k];
        c->K1[col * N1 + row] = c->A[r * nv + k];
      }
  e = gj_inverse(c->K1, N1, c->K1inv);
  if (e != OR_OK) goto fail;

  /* KKT of Eq. 19 for xi2: [[Pdd^T Pdd + rho_psi P^T P, A^T], [A, 0]] */
  const int Np = nv + c->nb;
  c->Kp = (double*)calloc((size_t)Np * Np, sizeof(double));
  c->Kpinv = (double*)calloc((size_t)Np * Np, sizeof(double));
  for (int a = 0; a < nv; ++a)
    for (int b = 0; b < nv; ++b) {
      double s = 0.0;
      for (int t = 0; t < q; ++t)
        s += c->Pdd[t * nv + a] * c->Pdd[t * nv + b] + p->rho_psi * c->P[t * nv + a] * c->P[t * nv + b];
      c->Kp[a * Np + b] = s;
    }
  for (int r = 0; r < c->nb; ++r)
    for (int k = 0; k < nv; ++k) {
      c->Kp[(nv + r) * Np + k] = c->A[r * nv + k];
      c->Kp[k * Np + nv + r] = c->A[r * nv + k];
    }
  e = gj_inverse(c->Kp, Np, c->Kpinv);
  if (e != OR_OK) goto fail;
  if (err) *err = OR_OK;
  return c;
fail:
  or_destroy(c);
  if (err) *err = e;
  return NULL;
}

/* ------------------------------------------------------------ sub-steps */

/* Eq. 21a + Eq. 22a + clip: alpha_ij then d_ij >= 1. */
void or_project_obstacle(double xt, double yt, double a, double b, int rule, double* alpha,
                         double* d) {
  double al;
  if (xt == 0.0 && yt == 0.0)
    al = 0.0; /* G18 */
  else
    al = (rule == 0) ? atan2(yt, xt) : atan2(a * yt, b * xt);
  const double ca = cos(al), sa = sin(al);
  const double dstar = (a * xt * ca + b * yt * sa) / (a * a * ca * ca + b * b * sa * sa);
  *alpha = al;
  *d = dstar > 1.0 ? dstar : 1.0;
}

/* Eq. 21b/c + Eq. 22b/c with the bound included (G7), clipped to [0,1] (G6). */
void or_project_bound(double vx, double vy, double bound, double* alpha, double* d) {
  const double al = (vx == 0.0 && vy == 0.0) ? 0.0 : atan2(vy, vx);
  const double dstar = (vx * cos(al) + vy * sin(al)) / bound;
  *alpha = al;
  *d = dstar < 0.0 ? 0.0 : (dstar > 1.0 ? 1.0 : dstar);
}

static void mat_T_vec(const or_ctx* c, const double* v, double* out) { /* out = F^T v */
  for (int a = 0; a < c->cols; ++a) out[a] = 0.0;
  for (int row = 0; row < c->rows; ++row) {
    const double* f = c->F + (size_t)row * c->cols;
    const double vr = v[row];
    for (int a = 0; a < c->cols; ++a) out[a] += f[a] * vr;
  }
}

static void resid_vec(const or_ctx* c, const double* xi1, const double* g, double* res) {
  for (int row = 0; row < c->rows; ++row) { /* res = F xi1 - g */
    const double* f = c->F + (size_t)row * c->cols;
    double s = 0.0;
    for (int a = 0; a < c->cols; ++a) s += f[a] * xi1[a];
    res[row] = s - g[row];
  }
}

double or_penalty(const or_ctx* c, const double* xi1, const double* g) {
  double* res = (double*)malloc(sizeof(double) * (size_t)c->rows);
  resid_vec(c, xi1, g, res);
  double s = 0.0;
  for (int row = 0; row < c->rows; ++row) s += res[row] * res[row];
  free(res);
  return 0.5 * s;
}

/* Eq. 23a with F^T (G3). */
void or_lambda_step(const or_ctx* c, const double* lam, const double* xi1, const double* g,
                    double* lam_out) {
  double* res = (double*)malloc(sizeof(double) * (size_t)c->rows);
  double* ft = (double*)malloc(sizeof(double) * (size_t)c->cols);
  resid_vec(c, xi1, g, res);
  mat_T_vec(c, res, ft);
  for (int a = 0; a < c->cols; ++a) lam_out[a] = lam[a] - c->p.rho * ft[a];
  free(res);
  free(ft);
}

static void boundary_b(const or_ctx* c, const double* bnd, int ch, double* b) {
  for (int r = 0; r < c->nb; ++r) b[r] = bnd[ch * 6 + c->bsel[r]];
}

/* Eq. 17 + Eq. 4: xi1 = first 4nv entries of KKT1^{-1} [lambda + rho F^T g; b_x; b_y]. */
int or_xi1_step(const or_ctx* c, const double* lam, const double* g, const double* bnd,
                double* xi1_out) {
  const int cols = c->cols, N1 = cols + 2 * c->nb;
  double* rhs = (double*)malloc(sizeof(double) * (size_t)N1);
  double* ft = (double*)malloc(sizeof(double) * (size_t)cols);
  mat_T_vec(c, g, ft);
  for (int a = 0; a < cols; ++a) rhs[a] = lam[a] + c->p.rho * ft[a];
  boundary_b(c, bnd, 0, rhs + cols);
  boundary_b(c, bnd, 1, rhs + cols + c->nb);
  for (int a = 0; a < cols; ++a) {
    double s = 0.0;
    for (int b = 0; b < N1; ++b) s += c->K1inv[a * N1 + b] * rhs[b];
    xi1_out[a] = s;
  }
  free(rhs);
  free(ft);
  return OR_OK;
}

/* Eq. 19 + Eq. 4: xi2 = first nv entries of KKTpsi^{-1} [lambda_psi + rho_psi P^T theta; b_psi]. */
int or_xi2_step(const or_ctx* c, const double* lampsi, const double* theta, const double* bnd,
                double* xi2_out) {
  const int nv = c->nv, q = c->q, Np = nv + c->nb;
  double* rhs = (double*)malloc(sizeof(double) * (size_t)Np);
  for (int k = 0; k < nv; ++k) {
    double s = 0.0;
    for (int t = 0; t < q; ++t) s += c->P[t * nv + k] * theta[t];
    rhs[k] = lampsi[k] + c->p.rho_psi * s;
  }
  boundary_b(c, bnd, 2, rhs + nv);
  for (int a = 0; a < nv; ++a) {
    double s = 0.0;
    for (int b = 0; b < Np; ++b) s += c->Kpinv[a * Np + b] * rhs[b];
    xi2_out[a] = s;
  }
  free(rhs);
  return OR_OK;
}

/* ------------------------------------------------------------- iteration */

typedef struct {
  double *x, *xd, *xdd, *y, *yd, *ydd, *psi, *cc, *ss, *theta;
} traj_t;

static void eval_vec(const double* B, int q, int nv, const double* coef, double* out) {
  for (int t = 0; t < q; ++t) {
    double s = 0.0;
    for (int k = 0; k < nv; ++k) s += B[t * nv + k] * coef[k];
    out[t] = s;
  }
}

/* Positions and derivatives from xi1, heading from xi2 (Eq. 8); copies c, s. */
static void eval_traj(const or_ctx* c, const double* xi1, const double* xi2, traj_t* tr) {
  const int q = c->q, nv = c->nv;
  eval_vec(c->P, q, nv, xi1 + 0 * nv, tr->x);
  eval_vec(c->Pd, q, nv, xi1 + 0 * nv, tr->xd);
  eval_vec(c->Pdd, q, nv, xi1 + 0 * nv, tr->xdd);
  eval_vec(c->P, q, nv, xi1 + 1 * nv, tr->cc);
  eval_vec(c->P, q, nv, xi1 + 2 * nv, tr->y);
  eval_vec(c->Pd, q, nv, xi1 + 2 * nv, tr->yd);
  eval_vec(c->Pdd, q, nv, xi1 + 2 * nv, tr->ydd);
  eval_vec(c->P, q, nv, xi1 + 3 * nv, tr->ss);
  eval_vec(c->P, q, nv, xi2, tr->psi);
}

/* xi3 (Eq. 21) and xi4 (Eq. 22) from the current trajectory, then g (Eq. 10-11). */
static void build_g(const or_ctx* c, const traj_t* tr, const double* obs_xy, const double* obs_ab,
                    double* g) {
  const int q = c->q, m = c->m, n = c->n, R = c->R;
  double al, d;
  for (int t = 0; t < q; ++t) {
    or_project_bound(tr->xd[t], tr->yd[t], c->p.v_max, &al, &d); /* alpha_v, d_v */
    g[t] = d * c->p.v_max * cos(al);
    g[R + t] = d * c->p.v_max * sin(al);
    or_project_bound(tr->xdd[t], tr->ydd[t], c->p.a_max, &al, &d); /* alpha_a, d_a */
    g[q + t] = d * c->p.a_max * cos(al);
    g[R + q + t] = d * c->p.a_max * sin(al);
    g[row_copy(c, t)] = cos(tr->psi[t]);
    g[R + row_copy(c, t)] = sin(tr->psi[t]);
  }
  for (int j = 0; j < n; ++j) {
    const double* ox = obs_xy + (size_t)j * 2 * q;
    const double* oy = ox + q;
    const double a = obs_ab[2 * j], b = obs_ab[2 * j + 1];
    for (int i = 0; i < m; ++i)
      for (int t = 0; t < q; ++t) {
        const double xt = tr->x[t] + c->r[i] * cos(tr->psi[t]) - ox[t]; /* G9 */
        const double yt = tr->y[t] + c->r[i] * sin(tr->psi[t]) - oy[t];
        or_project_obstacle(xt, yt, a, b, c->p.alpha_rule, &al, &d);
        g[row_coll(c, j, i, t)] = ox[t] + a * d * cos(al);      /* b_ob1 */
        g[R + row_coll(c, j, i, t)] = oy[t] + b * d * sin(al);  /* b_ob2 */
      }
  }
}

static void heading_target(const or_ctx* c, const traj_t* tr) {
  for (int t = 0; t < c->q; ++t) /* theta = atan2(s, c) (Eq. 19), G18 */
    tr->theta[t] = (tr->ss[t] == 0.0 && tr->cc[t] == 0.0) ? 0.0 : atan2(tr->ss[t], tr->cc[t]);
}

/* ------------------------------------------------ fp32 rounding model
 * (or_params.fp32_model; parity harness only).
 * The same iteration as above, with each quantity that the product path holds
 * in fp32 rounded where it is formed; everything else (the KKT steps, P^T theta,
 * F^T of the residual rows, lambda, J) stays fp64 as it is there.  Sites:
 *   evaluation: coefficients (positions relative to the boundary line, the
 *     frame the product path keeps positions in), the fp32 basis, and every
 *     evaluated sample x, y, xdot, ydot, xddot, yddot, psi, c, s (x, y, psi,
 *     c, s: every partial sum of the k-ordered FMA chain, eval32);
 *   cos psi, sin psi, theta = atan2(s, c);
 *   obstacle positions relative to the boundary line (once, to nearest);
 *   circle centres, (x~, y~), and every projection offset delta = g - v;
 *   the copy residuals e = c - cos psi.
 * The residual rows then read (F xi1 - g) = r_i e - delta (collision),
 * -delta (velocity, acceleration), e (copy), i.e. g is rebuilt around the
 * fp64 rows of F xi1 from the rounded offsets. */
typedef struct {
  const or_ctx* c;
  unsigned long long seed; /* 0: round to nearest */
  long long inst;
  int it;
  double xr0, xrd, yr0, yrd; /* boundary line: x_ref(tau) = xr0 + xrd tau, tau = t/(q-1) */
} r32_t;

static unsigned long long mix64(unsigned long long z) { /* splitmix64 finaliser */
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* v rounded to fp32: to nearest, or stochastically (probability of rounding
 * up = distance to the lower neighbour / spacing) when the model is seeded. */
static double r32(const r32_t* z, int site, long long idx, double v) {
  const float f = (float)v;
  if (!z->seed || !isfinite(v) || !isfinite(f) || (double)f == v) return (double)f;
  float lo = f, hi = f;
  if ((double)f < v)
    hi = nextafterf(f, INFINITY);
  else
    lo = nextafterf(f, -INFINITY);
  const double p = (v - (double)lo) / ((double)hi - (double)lo);
  unsigned long long h = mix64(z->seed);
  h = mix64(h ^ (unsigned long long)z->inst);
  h = mix64(h ^ ((unsigned long long)(z->it + 2) << 40) ^ ((unsigned long long)site << 32) ^
            (unsigned long long)idx);
  const double u = (double)(h >> 11) * 0x1.0p-53;
  return u < p ? (double)hi : (double)lo;
}

/* sum_k B[t][k] coef_k as the product path forms it (the coefficients rounded
 * first): a chain of fused multiply-adds in k order, every partial sum held in
 * fp32 and so rounded where it is formed (the product of two fp32 values is exact
 * in fp64, so r32(s + B coef) is one fp32 FMA) */
static double eval32(const r32_t* z, int site, const double* B, int t, const double* coef) {
  const int nv = z->c->nv;
  double s = 0.0;
  for (int k = 0; k < nv; ++k) s = r32(z, site, (long long)t * 16 + k, s + B[t * nv + k] * coef[k]);
  return s;
}

/* theta from the fp32 copies (model counterpart of heading_target) */
static void heading_target32(const r32_t* z, const double* xi1, traj_t* tr) {
  const or_ctx* c = z->c;
  const int q = c->q, nv = c->nv;
  double cc[32], ss[32];
  for (int k = 0; k < nv; ++k) {
    cc[k] = r32(z, 1, k, xi1[1 * nv + k]);
    ss[k] = r32(z, 2, k, xi1[3 * nv + k]);
  }
  for (int t = 0; t < q; ++t) {
    const double c32 = eval32(z, 3, c->P32, t, cc), s32 = eval32(z, 4, c->P32, t, ss);
    tr->theta[t] = (s32 == 0.0 && c32 == 0.0) ? 0.0 : r32(z, 5, t, atan2(s32, c32));
  }
}

/* g of Eq. 10-11 in the model (counterpart of build_g); tr holds the fp64 samples */
static void build_g32(const r32_t* z, const double* xi1, const double* xi2, const traj_t* tr,
                      const double* obs_xy, const double* obs_ab, double* g) {
  const or_ctx* c = z->c;
  const int q = c->q, m = c->m, n = c->n, R = c->R, nv = c->nv;
  double cx[32], cy[32], cc[32], ss[32], cp[32];
  for (int k = 0; k < nv; ++k) { /* Bernstein control points of the line: xr0 + xrd k / degree */
    cx[k] = r32(z, 10, k, xi1[0 * nv + k] - (z->xr0 + z->xrd * (double)k / (double)(nv - 1)));
    cy[k] = r32(z, 11, k, xi1[2 * nv + k] - (z->yr0 + z->yrd * (double)k / (double)(nv - 1)));
    cc[k] = r32(z, 12, k, xi1[1 * nv + k]);
    ss[k] = r32(z, 13, k, xi1[3 * nv + k]);
    cp[k] = r32(z, 14, k, xi2[k]);
  }
  for (int t = 0; t < q; ++t) {
    const double tau = (double)t / (double)(q - 1);
    const double xr = z->xr0 + z->xrd * tau, yr = z->yr0 + z->yrd * tau;
    const double x32 = eval32(z, 20, c->P32, t, cx), y32 = eval32(z, 21, c->P32, t, cy);
    const double xd = r32(z, 22, t, tr->xd[t]), yd = r32(z, 23, t, tr->yd[t]);
    const double xdd = r32(z, 24, t, tr->xdd[t]), ydd = r32(z, 25, t, tr->ydd[t]);
    const double psi = eval32(z, 26, c->P32, t, cp);
    const double c32 = eval32(z, 27, c->P32, t, cc), s32 = eval32(z, 28, c->P32, t, ss);
    const double cps = r32(z, 29, t, cos(psi)), sps = r32(z, 30, t, sin(psi));
    const double ec = r32(z, 31, t, c32 - cps), es = r32(z, 32, t, s32 - sps);
    double al, d;
    or_project_bound(xd, yd, c->p.v_max, &al, &d); /* offsets delta = g - v */
    g[t] = tr->xd[t] + r32(z, 33, t, d * c->p.v_max * cos(al) - xd);
    g[R + t] = tr->yd[t] + r32(z, 34, t, d * c->p.v_max * sin(al) - yd);
    or_project_bound(xdd, ydd, c->p.a_max, &al, &d);
    g[q + t] = tr->xdd[t] + r32(z, 35, t, d * c->p.a_max * cos(al) - xdd);
    g[R + q + t] = tr->ydd[t] + r32(z, 36, t, d * c->p.a_max * sin(al) - ydd);
    g[row_copy(c, t)] = tr->cc[t] - ec;
    g[R + row_copy(c, t)] = tr->ss[t] - es;
    for (int j = 0; j < n; ++j) {
      const double a = obs_ab[2 * j], b = obs_ab[2 * j + 1];
      const double ox = (double)(float)(obs_xy[(size_t)j * 2 * q + t] - xr);  /* once, to nearest */
      const double oy = (double)(float)(obs_xy[(size_t)j * 2 * q + q + t] - yr);
      for (int i = 0; i < m; ++i) {
        const long long id = ((long long)j * m + i) * q + t;
        const double X = r32(z, 40, id, x32 + c->r[i] * cps), Y = r32(z, 41, id, y32 + c->r[i] * sps);
        const double xt = r32(z, 42, id, X - ox), yt = r32(z, 43, id, Y - oy);
        or_project_obstacle(xt, yt, a, b, c->p.alpha_rule, &al, &d);
        const double dx = r32(z, 44, id, a * d * cos(al) - xt), dy = r32(z, 45, id, b * d * sin(al) - yt);
        /* residual row (x + r_i c) - g = r_i e - delta */
        g[row_coll(c, j, i, t)] = tr->x[t] + c->r[i] * tr->cc[t] - c->r[i] * ec + dx;
        g[R + row_coll(c, j, i, t)] = tr->y[t] + c->r[i] * tr->ss[t] - c->r[i] * es + dy;
      }
    }
  }
}

static long long pack_key(double r1, double J, double tau, long long gidx) {
  int infeasible = !(r1 <= tau);
  const double v = infeasible ? r1 : J;
  uint32_t bits;
  const float f = (float)v;
  if (!isfinite(v) || !isfinite(f)) {
    infeasible = 1;
    bits = 0x7F800000u;
  } else {
    const float fz = (f > 0.0f) ? f : 0.0f;
    memcpy(&bits, &fz, sizeof(bits));
  }
  return ((long long)infeasible << 62) | ((long long)bits << 30) | (gidx & ((1LL << 30) - 1));
}

typedef struct {
  double *coeffs, *lam_out, *res, *cost, *res_trace;
  double *xi1_tr, *xi2_tr, *lam_tr, *g_tr, *theta_tr, *r1_tr, *rpsi_tr;
} inst_out;

static int run_instance(const or_ctx* c, int K, long long gidx, const double* bnd,
                        const double* obs_xy, const double* obs_ab, const double* init,
                        const double* lam_in, inst_out* o) {
  const int q = c->q, nv = c->nv, cols = c->cols, rows = c->rows;
  const double rho = c->p.rho, rho_psi = c->p.rho_psi;
  double* buf = (double*)calloc((size_t)(3 * cols + 4 * nv + 2 * rows + 10 * q), sizeof(double));
  if (!buf) return OR_ENOMEM;
  double* xi1 = buf;
  double* lam = xi1 + cols;
  double* ft = lam + cols;
  double* xi2 = ft + cols;
  double* lampsi = xi2 + nv;
  double* ptheta = lampsi + nv;
  double* g = ptheta + 2 * nv;
  double* res = g + rows;
  traj_t tr;
  double* tb = res + rows;
  tr.x = tb;
  tr.xd = tb + q;
  tr.xdd = tb + 2 * q;
  tr.y = tb + 3 * q;
  tr.yd = tb + 4 * q;
  tr.ydd = tb + 5 * q;
  tr.psi = tb + 6 * q;
  tr.cc = tb + 7 * q;
  tr.ss = tb + 8 * q;
  tr.theta = tb + 9 * q;

  /* step 1: initialise xi2, xi3, xi4 (G15); copies start at zero */
  for (int k = 0; k < nv; ++k) {
    xi1[0 * nv + k] = init[0 * nv + k];
    xi1[1 * nv + k] = 0.0;
    xi1[2 * nv + k] = init[1 * nv + k];
    xi1[3 * nv + k] = 0.0;
    xi2[k] = init[2 * nv + k];
  }
  for (int a = 0; a < cols; ++a) lam[a] = lam_in ? lam_in[a] : 0.0;
  for (int k = 0; k < nv; ++k) lampsi[k] = lam_in ? lam_in[cols + k] : 0.0;
  /* fp32 rounding model (off for the oracle proper): positions are held
   * relative to the boundary line p(0) -> p(T), else p(0), else p(T), else 0 */
  r32_t z;
  memset(&z, 0, sizeof(z));
  z.c = c;
  z.seed = c->p.noise_seed;
  z.inst = gidx;
  z.it = -1;
  {
    const unsigned mk = c->p.boundary_mask;
    const int h0 = (mk & 1u) != 0, hT = (mk & 8u) != 0;
    z.xr0 = h0 ? bnd[0] : (hT ? bnd[3] : 0.0);
    z.yr0 = h0 ? bnd[6] : (hT ? bnd[9] : 0.0);
    z.xrd = (h0 && hT) ? bnd[3] - bnd[0] : 0.0;
    z.yrd = (h0 && hT) ? bnd[9] - bnd[6] : 0.0;
  }
  const int model = c->p.fp32_model != 0;
  eval_traj(c, xi1, xi2, &tr);
  if (model) {
    heading_target32(&z, xi1, &tr);
    build_g32(&z, xi1, xi2, &tr, obs_xy, obs_ab, g);
  } else {
    heading_target(c, &tr);
    build_g(c, &tr, obs_xy, obs_ab, g);
  }

#define RECORD(kk)                                                                  \
  do {                                                                              \
    if (o->xi1_tr) memcpy(o->xi1_tr + (size_t)(kk)*cols, xi1, sizeof(double) * cols); \
    if (o->xi2_tr) memcpy(o->xi2_tr + (size_t)(kk)*nv, xi2, sizeof(double) * nv);     \
    if (o->lam_tr) {                                                                \
      memcpy(o->lam_tr + (size_t)(kk) * 5 * nv, lam, sizeof(double) * cols);        \
      memcpy(o->lam_tr + (size_t)(kk) * 5 * nv + cols, lampsi, sizeof(double) * nv); \
    }                                                                               \
    if (o->g_tr) memcpy(o->g_tr + (size_t)(kk)*rows, g, sizeof(double) * rows);       \
    if (o->theta_tr) memcpy(o->theta_tr + (size_t)(kk)*q, tr.theta, sizeof(double) * q); \
  } while (0)

  double r1 = 0.0, rpsi = 0.0;
#define RESIDUALS()                                                         \
  do {                                                                      \
    resid_vec(c, xi1, g, res);                                              \
    double s_ = 0.0;                                                        \
    for (int row = 0; row < rows; ++row) s_ += res[row] * res[row];         \
    r1 = sqrt(s_);                                                          \
    double sp_ = 0.0;                                                       \
    for (int t = 0; t < q; ++t) sp_ += (tr.theta[t] - tr.psi[t]) * (tr.theta[t] - tr.psi[t]); \
    rpsi = sqrt(sp_);                                                       \
  } while (0)

  RESIDUALS();
  RECORD(0);
  if (o->r1_tr) o->r1_tr[0] = r1;
  if (o->rpsi_tr) o->rpsi_tr[0] = rpsi;

  for (int it = 0; it < K; ++it) {
    z.it = it;
    /* step 2: xi1 (Eq. 13, 17, 4) */
    or_xi1_step(c, lam, g, bnd, xi1);
    /* step 3: xi2 with the convex surrogate (Eq. 18-19) */
    eval_vec(c->P, q, nv, xi1 + 1 * nv, tr.cc);
    eval_vec(c->P, q, nv, xi1 + 3 * nv, tr.ss);
    if (model)
      heading_target32(&z, xi1, &tr);
    else
      heading_target(c, &tr);
    or_xi2_step(c, lampsi, tr.theta, bnd, xi2);
    /* steps 4-5: xi3, xi4 closed forms (Eq. 20-22) on the new trajectory */
    eval_traj(c, xi1, xi2, &tr);
    if (model)
      build_g32(&z, xi1, xi2, &tr, obs_xy, obs_ab, g);
    else
      build_g(c, &tr, obs_xy, obs_ab, g);
    /* step 6: multipliers (Eq. 23a-b, G3, G4) */
    resid_vec(c, xi1, g, res);
    mat_T_vec(c, res, ft);
    for (int a = 0; a < cols; ++a) lam[a] -= rho * ft[a];
    for (int k = 0; k < nv; ++k) {
      double s = 0.0;
      for (int t = 0; t < q; ++t) s += c->P[t * nv + k] * (tr.psi[t] - tr.theta[t]);
      ptheta[k] = s; /* P^T (P xi2 - theta) */
    }
    for (int k = 0; k < nv; ++k)
      lampsi[k] += (c->p.lampsi_printed_sign ? rho_psi : -rho_psi) * ptheta[k];
    RESIDUALS();
    RECORD(it + 1);
    if (o->r1_tr) o->r1_tr[it + 1] = r1;
    if (o->rpsi_tr) o->rpsi_tr[it + 1] = rpsi;
    if (o->res_trace) o->res_trace[it] = r1;
  }

  /* outputs: cost J = sum_t (xdd^2 + ydd^2 + psidd^2) (Eq. 1a, G17) */
  double J = 0.0;
  for (int t = 0; t < q; ++t) {
    double psidd = 0.0;
    for (int k = 0; k < nv; ++k) psidd += c->Pdd[t * nv + k] * xi2[k];
    J += tr.xdd[t] * tr.xdd[t] + tr.ydd[t] * tr.ydd[t] + psidd * psidd;
  }
  if (o->coeffs) {
    memcpy(o->coeffs, xi1, sizeof(double) * cols);
    memcpy(o->coeffs + cols, xi2, sizeof(double) * nv);
  }
  if (o->lam_out) {
    memcpy(o->lam_out, lam, sizeof(double) * cols);
    memcpy(o->lam_out + cols, lampsi, sizeof(double) * nv);
  }
  if (o->res) {
    o->res[0] = r1;
    o->res[1] = rpsi;
  }
  if (o->cost) o->cost[0] = J;
#undef RECORD
#undef RESIDUALS
  free(buf);
  return OR_OK;
}

int or_trace_instance(or_ctx* c, int K, const double* bnd, const double* obs_xy,
                      const double* obs_ab, const double* init, const double* lambda_in,
                      double* xi1_tr, double* xi2_tr, double* lam_tr, double* g_tr,
                      double* theta_tr, double* r1_tr, double* rpsi_tr) {
  if (!c || K < 0 || !bnd || (c->n > 0 && (!obs_xy || !obs_ab)) || !init) return OR_EINVAL;
  inst_out o;
  memset(&o, 0, sizeof(o));
  o.xi1_tr = xi1_tr;
  o.xi2_tr = xi2_tr;
  o.lam_tr = lam_tr;
  o.g_tr = g_tr;
  o.theta_tr = theta_tr;
  o.r1_tr = r1_tr;
  o.rpsi_tr = rpsi_tr;
  return run_instance(c, K, 0, bnd, obs_xy, obs_ab, init, lambda_in, &o);
}

int or_solve(or_ctx* c, int B, int K, long long index_base, const double* bnd,
             const double* obs_xy, const double* obs_ab, const double* init,
             const double* lambda_in, double* coeffs, double* lambda_out, double* residual,
             double* cost, double* res_trace, long long* best, int nthreads) {
  if (!c || B < 1 || K < 0 || !bnd || (c->n > 0 && (!obs_xy || !obs_ab)) || !init || !coeffs ||
      !residual || !cost)
    return OR_EINVAL;
  const int nv = c->nv;
  int err = OR_OK;
#ifdef _OPENMP
  if (nthreads < 1) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
  for (int l = 0; l < B; ++l) {
    inst_out o;
    memset(&o, 0, sizeof(o));
    o.coeffs = coeffs + (size_t)l * 5 * nv;
    o.lam_out = lambda_out ? lambda_out + (size_t)l * 5 * nv : NULL;
    o.res = residual + 2 * (size_t)l;
    o.cost = cost + l;
    o.res_trace = res_trace ? res_trace + (size_t)l * K : NULL;
    const int e = run_instance(c, K, index_base + l, bnd, obs_xy, obs_ab, init + (size_t)l * 3 * nv,
                               lambda_in ? lambda_in + (size_t)l * 5 * nv : NULL, &o);
    if (e != OR_OK) {
#ifdef _OPENMP
#pragma omp critical
#endif
      err = e;
    }
  }
  (void)nthreads;
  if (err != OR_OK) return err;
  if (best) {
    long long kmin = 0;
    for (int l = 0; l < B; ++l) {
      const long long key = pack_key(residual[2 * l], cost[l], c->p.res_tol, index_base + l);
      if (l == 0 || key < kmin) kmin = key;
    }
    best[0] = kmin & ((1LL << 30) - 1);
    best[1] = kmin;
  }
  return OR_OK;
}
