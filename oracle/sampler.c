/*
 * sampler.c -- fp64 oracle of the STOMP-style initial samples.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Shares no code with the CUDA
 * sampler; both implement the same counter-based generator (Philox4x32-10,
 * Salmon et al., SC'11) so that the random numbers are identical by
 * construction.
 *
 * "Our batch optimizer was always initialized with a Gaussian
 * distribution proposed in [STOMP] centered around a straight-line
 * trajectory."  Reading G28: the line is the constant-velocity
 * segment between bnd p0 and pT (control points c_k = p0 + (pT - p0) k / deg),
 * the Gaussian is STOMP's smoothness prior N(0, s^2 R^-1), R = D^T D with D
 * the second difference of the control polygon, restricted to the control
 * points 3..deg-3 (those enter no position, velocity or acceleration at either
 * end), normalised to unit maximum variance; c_psi = 0.
 *
 * Normals for instance g (global index): Philox4x32-10 with key
 * (seed_lo, seed_hi) and counters (g_lo, g_hi, stream_lo + j, stream_hi),
 * j = 0, 1, 2 -> 12 uint32 x_0..x_11; pairs (x_2p, x_2p+1) through
 * Box-Muller: u1 = (x_2p + 0.5) 2^-32, u2 = (x_2p+1 + 0.5) 2^-32,
 * n_2p = sqrt(-2 ln u1) cos(2 pi u2), n_2p+1 = sqrt(-2 ln u1) sin(2 pi u2);
 * z_x = n_0..n_4, z_y = n_5..n_9.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "oracle.h"

/* Philox4x32 round constants (Salmon et al., SC'11, Table 2 / Random123). */
#define PH_M0 0xD2511F53u
#define PH_M1 0xCD9E8D57u
#define PH_W0 0x9E3779B9u
#define PH_W1 0xBB67AE85u

void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += PH_W0; k1 += PH_W1; }   /* key schedule: bump before rounds 1..9 */
    const uint64_t p0 = (uint64_t)PH_M0 * c0, p1 = (uint64_t)PH_M1 * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* STOMP covariance factor: L lower with L L^T = Sigma (5 x 5 for degree 10). */
int or_stomp_factor(int degree, double* L, int* nfree) {
  const int nv = degree + 1, f0 = 3, nf = nv - 6;
  if (nf < 1 || nf > 16) return OR_EINVAL;
  double R[16 * 16], S[16 * 16];
  /* R = D^T D restricted to the free points; D rows i: (1, -2, 1) at i, i+1, i+2 */
  for (int a = 0; a < nf; ++a)
    for (int b = 0; b < nf; ++b) {
      double s = 0.0;
      for (int i = 0; i < nv - 2; ++i) {
        const int ka = f0 + a, kb = f0 + b;
        const double da = (ka == i) ? 1.0 : (ka == i + 1) ? -2.0 : (ka == i + 2) ? 1.0 : 0.0;
        const double db = (kb == i) ? 1.0 : (kb == i + 1) ? -2.0 : (kb == i + 2) ? 1.0 : 0.0;
        s += da * db;
      }
      R[a * nf + b] = s;
    }
  /* S = R^-1 by Gauss-Jordan with partial pivoting */
  double A[16 * 32];
  for (int a = 0; a < nf; ++a)
    for (int b = 0; b < 2 * nf; ++b) A[a * 2 * nf + b] = (b < nf) ? R[a * nf + b] : (b - nf == a ? 1.0 : 0.0);
  for (int c = 0; c < nf; ++c) {
    int p = c;
    for (int r = c + 1; r < nf; ++r)
      if (fabs(A[r * 2 * nf + c]) > fabs(A[p * 2 * nf + c])) p = r;
    if (fabs(A[p * 2 * nf + c]) < 1e-14) return OR_ESINGULAR;
    for (int b = 0; b < 2 * nf; ++b) { double t = A[c * 2 * nf + b]; A[c * 2 * nf + b] = A[p * 2 * nf + b]; A[p * 2 * nf + b] = t; }
    const double piv = A[c * 2 * nf + c];
    for (int b = 0; b < 2 * nf; ++b) A[c * 2 * nf + b] /= piv;
    for (int r = 0; r < nf; ++r)
      if (r != c) {
        const double f = A[r * 2 * nf + c];
        for (int b = 0; b < 2 * nf; ++b) A[r * 2 * nf + b] -= f * A[c * 2 * nf + b];
      }
  }
  double smax = 0.0;
  for (int a = 0; a < nf; ++a)
    for (int b = 0; b < nf; ++b) S[a * nf + b] = A[a * 2 * nf + nf + b];
  for (int a = 0; a < nf; ++a) smax = fmax(smax, S[a * nf + a]);
  for (int a = 0; a < nf * nf; ++a) S[a] /= smax;
  /* Cholesky S = L L^T */
  memset(L, 0, sizeof(double) * nf * nf);
  for (int i = 0; i < nf; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = S[i * nf + j];
      for (int k = 0; k < j; ++k) s -= L[i * nf + k] * L[j * nf + k];
      if (i == j) {
        if (!(s > 0.0)) return OR_ESINGULAR;
        L[i * nf + i] = sqrt(s);
      } else {
        L[i * nf + j] = s / L[j * nf + j];
      }
    }
  *nfree = nf;
  return OR_OK;
}

/* The 10 standard normals of instance g (layout above). */
void or_stomp_normals(uint64_t seed, uint64_t stream, long long g, double z[12]) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[12];
  for (int j = 0; j < 3; ++j) {
    const uint32_t ctr[4] = {(uint32_t)(uint64_t)g, (uint32_t)((uint64_t)g >> 32), (uint32_t)stream + (uint32_t)j,
                             (uint32_t)(stream >> 32)};
    or_philox4x32_10(ctr, key, x + 4 * j);
  }
  const double two32 = 4294967296.0, two_pi = 6.283185307179586476925286766559;
  for (int p = 0; p < 6; ++p) {
    const double u1 = ((double)x[2 * p] + 0.5) / two32, u2 = ((double)x[2 * p + 1] + 0.5) / two32;
    const double r = sqrt(-2.0 * log(u1));
    z[2 * p] = r * cos(two_pi * u2);
    z[2 * p + 1] = r * sin(two_pi * u2);
  }
}

int or_sample_init(int degree, long long B, long long index_base, uint64_t seed, uint64_t stream,
                   const double* bnd, double sigma_x, double sigma_y, int line_first, double* init) {
  const int nv = degree + 1;
  double L[256];
  int nf = 0;
  const int rc = or_stomp_factor(degree, L, &nf);
  if (rc != OR_OK) return rc;
  if (nf > 5) return OR_EINVAL;   /* 10 normals per instance: degree <= 10 */
  for (long long l = 0; l < B; ++l) {
    const long long g = index_base + l;
    double* o = init + l * 3 * nv;
    for (int k = 0; k < nv; ++k) {   /* the straight segment p0 -> pT */
      o[0 * nv + k] = bnd[0 * 6 + 0] + (bnd[0 * 6 + 3] - bnd[0 * 6 + 0]) * k / degree;
      o[1 * nv + k] = bnd[1 * 6 + 0] + (bnd[1 * 6 + 3] - bnd[1 * 6 + 0]) * k / degree;
      o[2 * nv + k] = 0.0;
    }
    if (line_first && g == 0) continue;
    double z[12];
    or_stomp_normals(seed, stream, g, z);
    for (int a = 0; a < nf; ++a) {   /* eps = s L z on the control points 3 .. deg-3 */
      double ex = 0.0, ey = 0.0;
      for (int b = 0; b <= a; ++b) {
        ex += L[a * nf + b] * z[b];
        ey += L[a * nf + b] * z[5 + b];
      }
      o[0 * nv + 3 + a] += sigma_x * ex;
      o[1 * nv + 3 + a] += sigma_y * ey;
    }
  }
  return OR_OK;
}
