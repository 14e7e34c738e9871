// setup.cpp -- host fp64 precompute of the per-(params, n) constants
// (product path).  Everything here runs once per context / obstacle count;
// the per-iteration work is in bmc_kernel.cu.
//
//  * Bernstein basis and derivatives at t_k = k T/(q-1) (Eq. 8),
//    evaluated with the de Casteljau recurrence.
//  * Boundary rows A = first/last rows of P, Pdot, Pddot (G11).
//  * F^T F in closed form per channel (Eq. 10-11): with the rows
//    velocity [Pd 0], acceleration [Pdd 0], collision [P r_i P] (m n blocks)
//    and copy [0 P]:
//        F^T F = [[Pd'Pd + Pdd'Pdd + n m P'P,  n R1 P'P      ],
//                 [n R1 P'P,                    (n R2 + 1) P'P]]
//    with R1 = sum r_i, R2 = sum r_i^2.  x and y channels are identical and
//    decoupled, so one 22x22 block serves both.
//  * Q_bar = Q + rho F^T F (Eq. 17), Q = blkdiag(Pdd'Pdd, w_copy Pdd'Pdd)
//    (G10); KKT = [[Q_bar, [A 0]^T], [[A 0], 0]] (Eq. 3);
//    its inverse by LU with partial pivoting (the "constant" of Eq. 4).
//  * Heading KKT of Eq. 19: [[Pdd'Pdd + rho_psi P'P, A^T], [A, 0]].
//  * M = rho K11 F^T F, so that the kernel's xi1 step
//        xi1' = K11 (lambda + rho F^T g) + K12 b
//             = M xi1 + K11 (lambda - rho h) + K12 b,   h = F^T (F xi1 - g)
//    never forms F^T g from large absolute positions.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "bmc_internal.h"

namespace bmc {

namespace {

// de Casteljau: all Bernstein polynomials of degree n at tau, out[0..n].
void bernstein_all(int n, double tau, double* out) {
  out[0] = 1.0;
  for (int d = 1; d <= n; ++d) {
    out[d] = tau * out[d - 1];
    for (int k = d - 1; k >= 1; --k) out[k] = (1.0 - tau) * out[k] + tau * out[k - 1];
    out[0] = (1.0 - tau) * out[0];
  }
}

// In-place LU with partial pivoting, then inverse column by column.
bool lu_inverse(std::vector<double> a, int N, std::vector<double>& inv) {
  std::vector<int> piv(N);
  double amax = 0.0;
  for (double v : a) amax = std::fmax(amax, std::fabs(v));
  for (int k = 0; k < N; ++k) {
    int p = k;
    for (int i = k + 1; i < N; ++i)
      if (std::fabs(a[i * N + k]) > std::fabs(a[p * N + k])) p = i;
    piv[k] = p;
    if (!(std::fabs(a[p * N + k]) > 1e-13 * amax)) return false;
    if (p != k)
      for (int j = 0; j < N; ++j) std::swap(a[k * N + j], a[p * N + j]);
    for (int i = k + 1; i < N; ++i) {
      a[i * N + k] /= a[k * N + k];
      const double l = a[i * N + k];
      for (int j = k + 1; j < N; ++j) a[i * N + j] -= l * a[k * N + j];
    }
  }
  inv.assign((size_t)N * N, 0.0);
  std::vector<double> x(N);
  for (int c = 0; c < N; ++c) {
    for (int i = 0; i < N; ++i) x[i] = (i == c) ? 1.0 : 0.0;
    for (int k = 0; k < N; ++k) std::swap(x[k], x[piv[k]]);
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < i; ++j) x[i] -= a[i * N + j] * x[j];
    for (int i = N - 1; i >= 0; --i) {
      for (int j = i + 1; j < N; ++j) x[i] -= a[i * N + j] * x[j];
      x[i] /= a[i * N + i];
    }
    for (int i = 0; i < N; ++i) inv[i * N + c] = x[i];
  }
  return true;
}

}  // namespace

// STOMP smoothness prior on the control points 3..7 of a degree-10 curve:
// R = D^T D (D: second difference of the control polygon), Sigma = R^-1
// normalised to unit maximum variance, L its Cholesky factor (G28).
int stomp_factor(double L[5][5]) {
  constexpr int nf = 5, f0 = 3;
  std::vector<double> R(nf * nf), Rinv;
  for (int a = 0; a < nf; ++a)
    for (int b = 0; b < nf; ++b) {
      double s = 0.0;
      for (int i = 0; i < NV - 2; ++i) {   // rows of D: (1, -2, 1) at columns i .. i+2
        auto d = [&](int k) { return k == i ? 1.0 : k == i + 1 ? -2.0 : k == i + 2 ? 1.0 : 0.0; };
        s += d(f0 + a) * d(f0 + b);
      }
      R[a * nf + b] = s;
    }
  if (!lu_inverse(R, nf, Rinv)) return 2;
  double dmax = 0.0;
  for (int a = 0; a < nf; ++a) dmax = std::fmax(dmax, Rinv[a * nf + a]);
  for (int a = 0; a < nf; ++a)
    for (int b = 0; b < nf; ++b) L[a][b] = 0.0;
  for (int i = 0; i < nf; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = Rinv[i * nf + j] / dmax;
      for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
      if (i == j) {
        if (!(s > 0.0)) return 2;
        L[i][i] = std::sqrt(s);
      } else {
        L[i][j] = s / L[j][j];
      }
    }
  return 0;
}

int build_consts(const SetupParams& p, int n, HostConsts* out, std::string* err) {
  const int q = p.q, QP = Q_MAX, deg = NV - 1;  // fixed sample stride (compile-time in the kernel)
  out->q = q;
  out->QP = QP;
  out->n = n;
  out->m = p.m;
  std::vector<double> P(q * NV), Pd(q * NV), Pdd(q * NV);
  double b0[NV], b1[NV], b2[NV];
  const double c1 = deg / p.T, c2 = deg * (deg - 1) / (p.T * p.T);
  for (int t = 0; t < q; ++t) {
    const double tau = (double)t / (double)(q - 1);
    bernstein_all(deg, tau, b0);
    bernstein_all(deg - 1, tau, b1);
    bernstein_all(deg - 2, tau, b2);
    for (int k = 0; k < NV; ++k) {
      P[t * NV + k] = b0[k];
      const double lo1 = (k >= 1) ? b1[k - 1] : 0.0, hi1 = (k <= deg - 1) ? b1[k] : 0.0;
      Pd[t * NV + k] = c1 * (lo1 - hi1);
      const double u0 = (k >= 2) ? b2[k - 2] : 0.0, u1 = (k >= 1 && k - 1 <= deg - 2) ? b2[k - 1] : 0.0,
                   u2 = (k <= deg - 2) ? b2[k] : 0.0;
      Pdd[t * NV + k] = c2 * (u0 - 2.0 * u1 + u2);
    }
  }
  // boundary rows
  int nb = 0;
  double A[NB_MAX][NV];
  for (int bit = 0; bit < 6; ++bit) {
    if (!(p.mask & (1u << bit))) continue;
    const std::vector<double>& src = (bit % 3 == 0) ? P : (bit % 3 == 1) ? Pd : Pdd;
    const int t = (bit < 3) ? 0 : q - 1;
    for (int k = 0; k < NV; ++k) A[nb][k] = src[t * NV + k];
    ++nb;
  }
  out->nb = nb;
  // Gram matrices
  double GPP[NV][NV], GDD[NV][NV], GAA[NV][NV];
  for (int a = 0; a < NV; ++a)
    for (int b = 0; b < NV; ++b) {
      double s0 = 0, s1 = 0, s2 = 0;
      for (int t = 0; t < q; ++t) {
        s0 += P[t * NV + a] * P[t * NV + b];
        s1 += Pd[t * NV + a] * Pd[t * NV + b];
        s2 += Pdd[t * NV + a] * Pdd[t * NV + b];
      }
      GPP[a][b] = s0;
      GDD[a][b] = s1;
      GAA[a][b] = s2;
    }
  double R1 = 0, R2 = 0;
  for (int i = 0; i < p.m; ++i) {
    R1 += p.r[i];
    R2 += p.r[i] * p.r[i];
  }
  // F^T F (22x22) and Q_bar
  double FtF[NV2][NV2], Qb[NV2][NV2];
  for (int a = 0; a < NV; ++a)
    for (int b = 0; b < NV; ++b) {
      FtF[a][b] = GDD[a][b] + GAA[a][b] + (double)n * p.m * GPP[a][b];
      FtF[a][NV + b] = FtF[NV + a][b] = (double)n * R1 * GPP[a][b];
      FtF[NV + a][NV + b] = ((double)n * R2 + 1.0) * GPP[a][b];
    }
  for (int a = 0; a < NV2; ++a)
    for (int b = 0; b < NV2; ++b) Qb[a][b] = p.rho * FtF[a][b];
  for (int a = 0; a < NV; ++a)
    for (int b = 0; b < NV; ++b) {
      Qb[a][b] += GAA[a][b];
      Qb[NV + a][NV + b] += p.w_copy * GAA[a][b];
    }
  // xi1 KKT per channel
  const int N1 = NV2 + nb;
  std::vector<double> K(N1 * N1, 0.0), Ki;
  for (int a = 0; a < NV2; ++a)
    for (int b = 0; b < NV2; ++b) K[a * N1 + b] = Qb[a][b];
  for (int rr = 0; rr < nb; ++rr)
    for (int k = 0; k < NV; ++k) K[(NV2 + rr) * N1 + k] = K[k * N1 + NV2 + rr] = A[rr][k];
  if (!lu_inverse(K, N1, Ki)) {
    *err = "singular xi1 KKT matrix (rank-deficient boundary rows or Q_bar not positive definite on null(A))";
    return 2;
  }
  // heading KKT
  const int Np = NV + nb;
  std::vector<double> Kp(Np * Np, 0.0), Kpi;
  for (int a = 0; a < NV; ++a)
    for (int b = 0; b < NV; ++b) Kp[a * Np + b] = GAA[a][b] + p.rho_psi * GPP[a][b];
  for (int rr = 0; rr < nb; ++rr)
    for (int k = 0; k < NV; ++k) Kp[(NV + rr) * Np + k] = Kp[k * Np + NV + rr] = A[rr][k];
  if (!lu_inverse(Kp, Np, Kpi)) {
    *err = "singular heading KKT matrix (rank-deficient boundary rows)";
    return 2;
  }
  // blob (transposed storage)
  double* f = out->blob_f64;
  std::memset(f, 0, sizeof(out->blob_f64));
  // With sum r_i = 0 the coupling block n R1 P'P of F^T F vanishes, the xi1 KKT
  // separates into the c_x block (with the boundary rows) and the c_c block, and M,
  // K11 are block diagonal: the off-diagonal blocks are stored as exact zeros and the
  // kernel skips them.
  out->blockdiag = (R1 == 0.0) ? 1 : 0;
  for (int k = 0; k < NV2; ++k)
    for (int j = 0; j < NV2; ++j) {
      double mkj = 0.0;  // (rho K11 F^T F)[k][j]
      for (int l = 0; l < NV2; ++l) mkj += Ki[k * N1 + l] * FtF[l][j];
      const bool off = out->blockdiag && ((k < NV) != (j < NV));
      f[BlobLayout::Mt + j * NV2 + k] = off ? 0.0 : p.rho * mkj;
      f[BlobLayout::K11t + j * NV2 + k] = off ? 0.0 : Ki[k * N1 + j];
      if (out->blockdiag && !off) {   // row-major copy of the own block
        const int jj = j - (k < NV ? 0 : NV);
        f[BlobLayout::Mb + k * BlobLayout::BD_ROW + jj] = p.rho * mkj;
        f[BlobLayout::Kb + k * BlobLayout::BD_ROW + jj] = Ki[k * N1 + j];
      }
    }
  for (int rr = 0; rr < nb; ++rr)
    for (int k = 0; k < NV2; ++k) f[BlobLayout::K12t + rr * NV2 + k] = Ki[k * N1 + NV2 + rr];
  for (int k = 0; k < NV; ++k) {
    for (int j = 0; j < NV; ++j) {
      f[BlobLayout::Kp11t + j * NV + k] = Kpi[k * Np + j];
      f[BlobLayout::Gppt + j * NV + k] = p.rho_psi * GPP[k][j];
      f[BlobLayout::Gdd + j * NV + k] = GAA[k][j];
    }
    for (int rr = 0; rr < nb; ++rr) f[BlobLayout::Kp12t + rr * NV + k] = Kpi[k * Np + NV + rr];
  }
  delete[] out->pt;
  delete[] out->pt64;
  const int S64 = BlobLayout::p64_stride(QP);
  constexpr int PR = BlobLayout::PT_ROW;
  out->pt = new float[PR * QP];
  out->pt64 = new double[NV * S64];
  std::memset(out->pt, 0, sizeof(float) * PR * QP);
  std::memset(out->pt64, 0, sizeof(double) * NV * S64);
  for (int k = 0; k < NV; ++k)
    for (int t = 0; t < q; ++t) {
      out->pt[t * PR + k] = (float)P[t * NV + k];
      out->pt64[k * S64 + t] = P[t * NV + k];
    }
  // The kernel evaluates Pdot c as P (Dm c) and Pdot^T u as Dm^T (P^T u) with the
  // tridiagonal Dm of bmc_kernel.cuh (dm_apply); check the identity Pdot = P Dm,
  // Pddot = P Dm^2 on this grid (it is exact up to rounding).
  {
    double dev = 0.0, scale = 0.0;
    for (int t = 0; t < q; ++t)
      for (int k = 0; k < NV; ++k) {
        double d1 = 0.0, d2 = 0.0;
        for (int j = std::max(0, k - 2); j <= std::min(deg, k + 2); ++j) {
          // (Dm)[j][k] and (Dm^2)[j][k]
          auto dm = [&](int r, int c) -> double {
            if (c == r - 1) return -r / p.T;
            if (c == r) return (2.0 * r - deg) / p.T;
            if (c == r + 1) return (deg - r) / p.T;
            return 0.0;
          };
          double dm2 = 0.0;
          for (int i = std::max(0, j - 1); i <= std::min(deg, j + 1); ++i) dm2 += dm(j, i) * dm(i, k);
          d1 += P[t * NV + j] * dm(j, k);
          d2 += P[t * NV + j] * dm2;
        }
        dev = std::fmax(dev, std::fmax(std::fabs(d1 - Pd[t * NV + k]) * p.T,
                                       std::fabs(d2 - Pdd[t * NV + k]) * p.T * p.T));
        scale = std::fmax(scale, std::fmax(std::fabs(Pd[t * NV + k]) * p.T, std::fabs(Pdd[t * NV + k]) * p.T * p.T));
      }
    if (!(dev <= 1e-12 * scale)) {
      if (err) *err = "internal: Bernstein derivative identity check failed";
      return 2;
    }
  }
  return 0;
}

}  // namespace bmc
