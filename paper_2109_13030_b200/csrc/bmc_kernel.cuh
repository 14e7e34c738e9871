// bmc_kernel.cuh -- fused batched AM iteration of arXiv 2109.13030 on sm_100a.
//
// A team of T warps (1..4) owns one batch instance l for all K iterations
// (instances are independent, "each instance in the batch is
// independent"); a CTA of ipc teams shares one shared-memory copy of the
// batch-invariant data: the basis P and the KKT inverses (bulk-copied by TMA,
// cp.async.bulk + mbarrier) and the obstacle trajectories.
//
// Time samples are processed in rounds of 32 lanes (t = 32 u + lane); warp w
// of a team takes rounds u = T-1-w, 2T-1-w, ...  Samples t >= q of the last
// round have a zero basis row and far-away obstacle slots and drop out.
// Teams of 2 are formed across the SMSP pairs (warps (0, 2) and (1, 3) of
// every group of 4), which balances the four schedulers at 7 teams per CTA.
//
// Per iteration (paper step order):
//   A  xi1 step (Eq. 13/17 via Eq. 4):  xi1' = M xi1 + K11 (lambda - rho h) + K12 b
//      in fp64 (lane k < 22 owns row k; one channel per warp for T >= 2);
//   B  c, s = P c_c, P c_s; theta = atan2(s, c); P^T theta (warp transpose-reduce);
//   C  xi2 step (Eq. 19) and lambda_psi (Eq. 23b, G4) in fp64 (lanes k < 11);
//   D  x, xdot, xddot, y, ..., psi at the lane's t (deviation from the boundary
//      line, fp32); velocity / acceleration projections (Eq. 21b-c, 22b-c:
//      projection onto the v_max / a_max disk); collision projections over all
//      (j, i) (Eq. 21a, 22a) reduced in registers to D = sum_ij delta_ij and
//      E = sum_i r_i sum_j delta_ij, delta_ij = (a d cos alpha, b d sin alpha)
//      - (x~, y~); then the contraction h = F^T (F xi1 - g) in closed form
//      (Eq. 10-11):
//        h_pos  = P^T (n R1 e - D) - Pd^T dv - Pdd^T da,
//        h_copy = P^T ((n R2 + 1) e - E),      e = c - cos(psi)  (G9)
//      with Pd = P Dm, Pdd = P Dm^2 (Dm: Bernstein derivative, tridiagonal),
//      so D2 is one FP64 tensor-core product G = P^T [U0..U7];
//   E  lambda <- lambda - rho h (Eq. 23a with F^T, G3).
// The residual r1 = ||F xi1 - g|| is accumulated in the last iteration (or
// every iteration in trace mode) from the same per-row quantities.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include <atomic>
#include <stdint.h>
#include <stdio.h>

#include "bmc_internal.h"

namespace bmc {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int QP = Q_MAX;   // sample stride of every per-sample smem array
constexpr int JB = 4;       // obstacles per collision block (coll_circ)

constexpr int T_MAX = QP / 32;   // warps per instance ("team"): at most one per round
constexpr int QP64 = QP + 4;     // row stride of the fp64 basis (BlobLayout::p64_stride)
constexpr int QPU = QP + 4;      // row stride of WarpSmem::U
constexpr int HP_SLOTS = 8 * 12; // per-warp partial contractions (D2), doubles

// Per-instance state shared by the TT warps of its team (per-warp arrays sized
// by the compile-time team size: shared memory bounds the instances per SM for
// large batches).  The x and y channels of xi1 are decoupled in the xi1 step and
// the lambda step (Eq. 10: F and the KKT are block diagonal over channels), so a
// team gives each channel to one warp; the small heading step runs redundantly
// in every warp.
// slot of coefficient k (0..21) in WarpSmem::xi1 / rhs
__host__ __device__ constexpr int xpad(int k) { return k + (k >= NV ? 1 : 0); }

template <int TT>
struct alignas(16) WarpSmemT {
  // [ch][xpad(k)] current xi1 (fp64), written by the channel's owner; the copy
  // block starts at 12 (16-byte aligned pairs for the block-diagonal step)
  double xi1[2][24];
  double rhs[2][24];      // [ch][xpad(k)] lambda - rho h
  double xi2w[TT][12];    // per-warp copies of xi2 (the heading step is redundant)
  double rhspw[TT][12];
  // fp32 coefficients interleaved per Bernstein index k: c_x - c_ref_x,
  // c_y - c_ref_y, Dm c_x, Dm c_y, Dm^2 c_x, Dm^2 c_y (Dm: the derivative
  // operator on coefficients, Pdot = P Dm); the copies
  // (c_c, c_s) per k, two indices per 16-byte load
  alignas(16) float cpos[NV + 1][4];   // (c_x - c_ref_x, c_y - c_ref_y, Dm c_x, Dm c_y)
  alignas(16) float cdd[NV + 1][2];    // (Dm^2 c_x, Dm^2 c_y), two indices per 16-byte load
  alignas(16) float ccs[NV + 1][2];
  float cf4[TT][12];      // per-warp fp32 c_psi
  float2 cs[QP];                // copies (c, s) per sample
  float th[QP];                 // theta per sample
  double part_th[TT][16];       // per-warp P^T theta partials, summed in warp order
  float part_res[TT][4];
  alignas(16) float U[8][QP + 4];   // per-sample vectors of F^T (F xi1 - g) (phase D1 -> D2);
                                // stride QP + 4: MMA B-fragment columns on distinct banks.
                                // TT = 1: also the D2 partial slots once the round loop is done
  float2 pxy[QP];               // x, y and psi at the previous evaluation (culling clock)
  float ppsi[QP];
  float clk[T_MAX];             // per-round movement clocks (culling)
  float pad_[T_MAX];
  double thsum[TT >= 2 ? QP : 2];   // FM: sum over the iterations of theta per sample (lambda_psi output)
};
static_assert(sizeof(WarpSmemT<1>) % 16 == 0 && sizeof(WarpSmemT<2>) % 16 == 0 && sizeof(WarpSmemT<4>) % 16 == 0,
              "WarpSmem must keep 16-byte alignment");
static_assert(HP_SLOTS * sizeof(double) <= sizeof(float) * 8 * (QP + 4), "D2 partials fit in U (TT = 1)");
__host__ __device__ inline size_t ws_bytes(int T) {
  return T == 1 ? sizeof(WarpSmemT<1>) : T == 2 ? sizeof(WarpSmemT<2>) : sizeof(WarpSmemT<4>);
}

// Team barrier: named barrier per team (id 1 + team) over its 32 T threads.
__device__ __forceinline__ void team_sync(int team, int T) {
  if (T == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(32 * T) : "memory");
  }
}

// u_x[22], u_y[22], u_psi[11] (+pad), then the per-lane weights of Dm and
// Dm^T (DM_LO, DM_DI, DM_HI, DMT_LO, DMT_HI; [5][32], see dm_apply)
constexpr int U_DOUBLES = 56 + 5 * 32 + 16;
constexpr int DM_TAB = 56;
constexpr int CG_TAB = 56 + 5 * 32;   // FM: sum over the pinned j of (rho_psi P^T P)[k][j] u_psi[j], lanes k < 11

// Development aid (make PROFILE=1): per-warp cycle counts of each phase.
#ifdef BMC_PROFILE
constexpr int PROF_SLOTS = 16;
struct PhaseClock {
  long long acc[PROF_SLOTS] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = 0;
  long long s0 = 0;   // sub-phase timer (does not move t0)
};
#define BMC_TICK(pc, i)                  \
  do {                                   \
    const long long t1_ = clock64();     \
    (pc).acc[i] += t1_ - (pc).t0;        \
    (pc).t0 = t1_;                       \
  } while (0)
// sub-phase split of D1 (slots 12..15) on its own timer
#define BMC_SUB(pc, i)                   \
  do {                                   \
    const long long t1_ = clock64();     \
    if ((i) >= 0) (pc).acc[i] += t1_ - (pc).s0; \
    (pc).s0 = t1_;                       \
  } while (0)
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BMC_STAMP(i) \
  do {                                                                       \
    if (threadIdx.x == 0 && a.prof_t) a.prof_t[(long long)blockIdx.x * 8 + (i)] = gtimer(); \
  } while (0)
#else
#define BMC_STAMP(i) ((void)0)
struct PhaseClock {};
#define BMC_TICK(pc, i) ((void)0)
#define BMC_SUB(pc, i) ((void)0)
#endif

// obstacles are padded to a multiple of JB with far-away, zero-radius dummies
__host__ __device__ inline int pad_obstacles(int n) { return (n + JB - 1) / JB * JB; }

// clearance / active-list stride: padded obstacles + the far dummy, JB-aligned
__host__ __device__ inline int clr_stride(int n) { return pad_obstacles(n) + JB; }

// Layout after the constant blob: obstacles [npad + 1][QP] (row npad: the far
// dummy), abi [npad + 1], ell [npad + 1], u = K12 b, WarpSmem[ipc], clearance stamps
// [ipc][4][nclr], active lists [ipc * T][nclr], D2 partials [ipc * T][HP_SLOTS],
// the mbarrier of the blob copy.
__host__ __device__ inline size_t smem_bytes(int n, int ipc, int T) {
  const int np = pad_obstacles(n) + 1;
  return BlobLayout::bytes(QP) + (size_t)np * QP * sizeof(float2) + 2 * (size_t)np * sizeof(float4) +
         U_DOUBLES * sizeof(double) + (size_t)ipc * ws_bytes(T) +
         (size_t)ipc * (T_MAX + T) * clr_stride(n) * sizeof(float) +
         (T > 1 ? (size_t)ipc * T * HP_SLOTS * sizeof(double) : 0) +
         16;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {   // release, CTA scope
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
// MUFU.RSQ without the denormal fix-up sequence (x = 0 -> +inf).
// fp32 -> fp64 without the -ftz denormal flush (a flush would cost an extra FMUL)
__device__ __forceinline__ double f2d(float x) {
  double d;
  asm("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(x));
  return d;
}
// fp64 -> fp32, round to nearest, without the -ftz flush of fp32 denormals (ptxas
// emulates that flush with a compare and a multiply after every conversion); the
// converted quantities never lie in the fp32 denormal range except 0
__device__ __forceinline__ float d2f(double x) {
  float f;
  asm("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(x));
  return f;
}
__device__ __forceinline__ float sqrt_approx(float x) {   // MUFU.SQRT, ~1 ulp
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32 pairs (FFMA2 / FADD2 / FMUL2, sm_100): one instruction for two
// lanes' worth of fp32 work, each half rounded exactly like the scalar op, so
// pairing changes no result bit.
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {   // one FADD2 with a negated operand
  float2 d;
  asm("sub.rn.ftz.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// FP64 tensor-core MMA D = A B + D, m8n8k4 (A row-major 8x4, B col-major 4x8):
// a = A[lane / 4][lane % 4], b = B[lane % 4][lane / 4],
// d[i] = D[lane / 4][2 (lane % 4) + i].
// Operands must not come from lane-dependent selects: the compiler may split the
// mma.sync into predicated copies, which deadlocks the warp (tests/test_sass.py).
__device__ __forceinline__ void mma_f64_884(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// atan2 for theta (Eq. 19): octant reduction and atan(a) = a + a^3 Q(a^2) on
// [0, 1], Q of degree 8 from a weighted least-squares fit of the relative
// error (2.6e-9 in exact arithmetic, so the fp32 result carries rounding only:
// |error| < 7e-8 rad, unbiased -- a systematic fit error would add up
// coherently in P^T theta).  pi/2 and pi enter as hi + lo pairs.
// atan2(0, 0) = 0 (G18); signed zeros and the x < 0 half-plane follow atan2f.
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float atan2_fast(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float a = mn * rcp_approx(mx);
  const float s = a * a;
  float p = -1.793621520e-03f;
  p = fmaf(p, s, 1.091460537e-02f);
  p = fmaf(p, s, -3.117784606e-02f);
  p = fmaf(p, s, 5.795759474e-02f);
  p = fmaf(p, s, -8.403450456e-02f);
  p = fmaf(p, s, 1.095218584e-01f);
  p = fmaf(p, s, -1.426424170e-01f);
  p = fmaf(p, s, 1.999854829e-01f);
  p = fmaf(p, s, -3.333329909e-01f);
  float r = fmaf(a * s, p, a);
  r = (ay > ax) ? (1.57079637f - r) + -4.37113883e-08f : r;
  r = (x < 0.f) ? (3.14159274f - r) + -8.74227766e-08f : r;
  r = copysignf(r, y);
  return (mx == 0.f) ? 0.f : r;
}

// sin and cos of the heading (G9) without the Payne-Hanek path of sincosf:
// j = rint(x 2/pi), Cody-Waite reduction r = x - j pi/2 with a three-part pi/2
// (P1 has 8 significant bits, so j P1 is exact for |j| < 2^16), and the
// classic single-precision minimax polynomials on [-pi/4, pi/4] (Cephes sinf /
// cosf); |error| < 1e-7 for |x| < 1e3 rad, unbiased (tests/test_kernel_math.py).
// Headings beyond 1e5 rad only occur in diverged instances.
__device__ __forceinline__ void sincos_fast(float x, float* sp, float* cp) {
  const float j = rintf(x * 0.636619772367581343f);
  float r = fmaf(j, -1.5703125f, x);
  r = fmaf(j, -4.83751296997070312e-4f, r);
  r = fmaf(j, -7.54978995489188216e-8f, r);
  const float r2 = r * r;
  float ps = fmaf(r2, -1.9515295891e-4f, 8.3321608736e-3f);
  ps = fmaf(r2, ps, -1.6666654611e-1f);
  const float sn = fmaf(r * r2, ps, r);
  float pc = fmaf(r2, 2.443315711e-5f, -1.388731625e-3f);
  pc = fmaf(r2, pc, 4.166664568e-2f);
  const float cs = fmaf(r2 * r2, pc, fmaf(-0.5f, r2, 1.f));
  const int q = (int)j;
  const float s1 = (q & 1) ? cs : sn, c1 = (q & 1) ? sn : cs;
  *sp = (q & 2) ? -s1 : s1;
  *cp = ((q + 1) & 2) ? -c1 : c1;
}

// ------------------------------------------------------------ warp reductions
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// One butterfly stage of the transpose-reduce: CNT values -> CNT/2 values.
template <int CNT, typename V>
__device__ __forceinline__ void tr_stage(V* v, int off, bool upper) {
#pragma unroll
  for (int i = 0; i < CNT / 2; ++i) {
    const V send = upper ? v[i] : v[i + CNT / 2];
    const V keep = upper ? v[i + CNT / 2] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, off);
  }
}
// 32 values per lane -> lane l holds the warp total of value l.
template <typename V>
__device__ __forceinline__ V transpose_reduce32(V* v, int lane) {
  tr_stage<32>(v, 16, lane & 16);
  tr_stage<16>(v, 8, lane & 8);
  tr_stage<8>(v, 4, lane & 4);
  tr_stage<4>(v, 2, lane & 2);
  tr_stage<2>(v, 1, lane & 1);
  return v[0];
}
// 16 values per lane -> lane l holds the warp total of value l >> 1.
template <typename V>
__device__ __forceinline__ V transpose_reduce16(V* v, int lane) {
  tr_stage<16>(v, 16, lane & 16);
  tr_stage<8>(v, 8, lane & 8);
  tr_stage<4>(v, 4, lane & 4);
  tr_stage<2>(v, 2, lane & 2);
  return v[0] + __shfl_xor_sync(FULL, v[0], 1);
}

// N (power of two <= 32) values per lane -> after log2 N transpose stages each
// lane holds a partial of value lane >> (5 - log2 N); plain butterflies over
// the remaining lane bits finish the warp total.
template <int CNT, int OFF, typename V>
__device__ __forceinline__ void tr_stages(V* v, int lane) {
  if constexpr (CNT > 1) {
    tr_stage<CNT>(v, OFF, lane & OFF);
    tr_stages<CNT / 2, OFF / 2>(v, lane);
  }
}
template <int N, typename V>
__device__ __forceinline__ V tr_reduce(V* v, int lane) {
  tr_stages<N, 16>(v, lane);
  constexpr int first_plain = 16 / N;   // offset after the transpose stages
#pragma unroll
  for (int o = first_plain; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(FULL, v[0], o);
  return v[0];
}

// Bernstein derivative on coefficients (degree n = 10, t in [0, T]):
// Pdot = P Dm exactly, Dm tridiagonal with Dm[k][k-1] = -k / T,
// Dm[k][k] = (2k - n) / T, Dm[k][k+1] = (n - k) / T (derivative of B_{k,n}
// written in the degree-n basis by degree elevation).  Lane k < 11 holds
// entry k; the per-lane weights (zero outside the band and for k >= 11) come
// from the table staged in shared memory.
__device__ __forceinline__ double band_apply(double c, const double* tab, int lo_row, int hi_row, int k) {
  const double lo = __shfl_up_sync(FULL, c, 1), hi = __shfl_down_sync(FULL, c, 1);
  return fma(tab[lo_row * 32 + k], lo, fma(tab[hi_row * 32 + k], hi, tab[1 * 32 + k] * c));
}
// (Dm c)_k = (-k c_{k-1} + (2k - n) c_k + (n - k) c_{k+1}) / T
__device__ __forceinline__ double dm_apply(double c, const double* tab, int k) { return band_apply(c, tab, 0, 2, k); }
// (Dm^T g)_k = ((n - k + 1) g_{k-1} + (2k - n) g_k - (k + 1) g_{k+1}) / T
__device__ __forceinline__ double dmT_apply(double g, const double* tab, int k) { return band_apply(g, tab, 3, 4, k); }
// the table: rows DM_LO, DM_DI, DM_HI, DMT_LO, DMT_HI over lanes 0..31
__device__ __forceinline__ void dm_table(double* tab, int k, double T) {
  const int n = NV - 1;
  const bool in = k < NV;
  tab[0 * 32 + k] = (in && k >= 1) ? -k / T : 0.0;
  tab[1 * 32 + k] = in ? (2.0 * k - n) / T : 0.0;
  tab[2 * 32 + k] = (in && k < n) ? (n - k) / T : 0.0;
  tab[3 * 32 + k] = (in && k >= 1) ? (n - k + 1) / T : 0.0;
  tab[4 * 32 + k] = (in && k < n) ? -(k + 1) / T : 0.0;
}

__device__ __forceinline__ void load12(const float* src, float (&c)[NV]) {
  const float4 a = reinterpret_cast<const float4*>(src)[0];
  const float4 b = reinterpret_cast<const float4*>(src)[1];
  const float4 d = reinterpret_cast<const float4*>(src)[2];
  c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w;
  c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
  c[8] = d.x; c[9] = d.y; c[10] = d.z;
}

// the fp32 basis row of sample t (BlobLayout: [QP][12], three 16-byte loads)
__device__ __forceinline__ void load_basis_row(const float* Pt, int t, float (&p)[NV]) {
  load12(Pt + t * BlobLayout::PT_ROW, p);
}

// Per-kernel constants of the projection phase (registers / constant bank).
struct Proj {
  const float* Pt;       // smem basis [QP][12] (fp32, per-sample rows)
  const double* Pt64;    // the same basis in fp64 (contractions)
  const float2* obs;     // smem obstacles [n][QP], relative to the boundary line
  const float4* abi;     // smem (a, b, a b, kind) per obstacle
  const float4* ell;     // smem (1/a, 1/b, max(a, b), 0) per obstacle (culled ellipses, NEXT-4)
  int q, n, rounds;
  bool all_circ;         // every obstacle a circle (a = b): culled closed form
  bool all_cull;         // every obstacle a circle or a scaled-rule ellipse (G8): culled, ELL form
  float nR1, nR2p1, v_max, a_max;
  float rabs;            // max_i |r_i| (culling clock)
  float* clr;            // smem clearance stamps of the instance, [4 rounds][nclr]
  int* list;             // smem active list of the warp, [nclr]
  int npad, nclr;        // padded obstacle count (index npad = far dummy), stride
  double* hp;            // smem D2 partials of the team's warps, [T][HP_SLOTS]
  const double* dmtab;   // smem weights of Dm, Dm^T (dm_table)
  bool no_cull;          // testing aid: test every obstacle (KernelArgs::no_cull)
};

// --------------------------------------------------- collision projections
// For every obstacle j and circle i at sample t:
// x~ = X_i - x_j, y~ = Y_i - y_j (X_i = x + r_i cos psi, G9) and the
// closed-form offset delta = (a d cos alpha, b d sin alpha) - (x~, y~) of
// Eq. 21a / 22a:
//   kind 0 (a == b, either rule):  delta = (x~, y~) max(a / |(x~,y~)| - 1, 0)
//   kind 1 (literal atan2(y~,x~)): delta = (x~ (a f - 1), y~ (b f - 1)),
//                                  f = max(1/rho, (a x~^2 + b y~^2)/(a^2 x~^2 + b^2 y~^2))
//   kind 2 (scaled, G8):           delta = (x~, y~) max(ab / sqrt(b^2 x~^2 + a^2 y~^2) - 1, 0)
// The residual terms (r_i e - delta)^2 are accumulated as
// base + delta (delta - 2 r_i e), with base = sum_i (r_i e)^2 per obstacle.
//
// Circular obstacles (coll_circ): delta = 0 unless |(x~, y~)| < a, and the
// closed form max(a / |(x~, y~)| - 1, 0) is exactly zero outside, so every
// obstacle of the round's active list (see `build_active`) runs it at all M
// circle centres: no inside test, no warp vote, no data-dependent branch (an
// earlier variant tested the segment of circle centres first and ran the
// closed form only where some lane was inside; this one has fewer dependent
// steps per obstacle and the same result bits).  The pass records, per
// visited obstacle, the round's clearance min over samples and circles of
// |centre - o_j| - a_j, stamped with the movement clock A.
// NB obstacles of the active list (one basic block: their loads and MUFU
// latencies overlap), then the warp reductions of their stamps.  Returns true
// in some lane if a circle centre sits exactly on an obstacle centre (G18).
// ELL (NEXT-4, scenes with scaled-rule ellipses, G8): the closed form of the
// scaled rule, delta = (x~, y~) max(1 / |(x~ / a, y~ / b)| - 1, 0), exactly zero
// outside the ellipse, with the stamp taken against the bounding circle of
// radius max(a, b) (ell[j] = (1/a, 1/b, max(a, b), 0); circles: a = b).
template <int M, int NB, bool ELL>
__device__ __forceinline__ bool coll_block(const bool RES, const float2* __restrict__ ob,
                                           const float4* __restrict__ abi, const float4* __restrict__ ell,
                                           const int* __restrict__ list, int jb,
                                           float* __restrict__ clr, float A, int lane, const float2 (&XY)[M],
                                           const float (&rec)[M], const float (&res_s)[M], float2 (&D)[M],
                                           float& rc) {
  float r2m[NB];
#pragma unroll
  for (int jj = 0; jj < NB; ++jj) {
    const int j = list[jb + jj];
    const float2 o = ob[j * QP];
    const float a = abi[j].x;
    float2 inv = make_float2(0.f, 0.f);
    if (ELL) inv = *reinterpret_cast<const float2*>(&ell[j]);
    float r2min = INFINITY;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const float2 tt = sub2(XY[i], o);   // (x~, y~)
      const float r2 = fmaf(tt.y, tt.y, tt.x * tt.x);
      float sc;
      if (ELL) {
        const float2 u = mul2(tt, inv);   // (x~ / a, y~ / b)
        sc = fmaxf(rsqrt_ftz(fmaf(u.y, u.y, u.x * u.x)) - 1.f, 0.f);
      } else {
        sc = fmaxf(fmaf(a, rsqrt_ftz(r2), -1.f), 0.f);
      }
      const float2 dd = mul2(bc2(sc), tt);
      D[i] = add2(D[i], dd);
      if (RES) rc = fmaf(dd.x, dd.x - 2.f * rec[i], fmaf(dd.y, dd.y - 2.f * res_s[i], rc));
      r2min = fminf(r2min, r2);
    }
    r2m[jj] = r2min;
  }
  unsigned qm = 1u;
#pragma unroll
  for (int jj = 0; jj < NB; ++jj) {
    // round minimum (non-negative floats order as their bit patterns)
    const unsigned mn = __reduce_min_sync(FULL, __float_as_uint(r2m[jj]));
    qm = (lane == jj) ? mn : qm;
  }
  {   // lanes < NB stamp their obstacle (predicated store, no divergent block)
    const int j = list[jb + min(lane, NB - 1)];
    const float v = sqrt_approx(__uint_as_float(qm)) - (ELL ? ell[j].z : abi[j].x) * 1.00001f + A;
    if (lane < NB) clr[j] = v;
  }
  return qm == 0u;
}

// The active list in blocks of JB obstacles, then a block of 2 and one of 1
// for the remainder: most rounds have one or two active obstacles, and padding
// them to a block of 4 with far dummies cost 1-3 % (C3, C4).
template <int M, bool ELL>
__device__ __forceinline__ unsigned coll_circ(const bool RES, const float2* __restrict__ ob,
                                              const float4* __restrict__ abi, const float4* __restrict__ ell,
                                              const int* __restrict__ list, int na,
                                              float* __restrict__ clr, float A, int lane, const float2 (&XY)[M],
                                              const float (&rec)[M], const float (&res_s)[M], float2 (&D)[M],
                                              float& rc) {
  bool zero = false;
  int jb = 0;
#pragma unroll 1
  for (; jb + JB <= na; jb += JB)
    zero |= coll_block<M, JB, ELL>(RES, ob, abi, ell, list, jb, clr, A, lane, XY, rec, res_s, D, rc);
  if (jb + 2 <= na) {
    zero |= coll_block<M, 2, ELL>(RES, ob, abi, ell, list, jb, clr, A, lane, XY, rec, res_s, D, rc);
    jb += 2;
  }
  if (jb < na) zero |= coll_block<M, 1, ELL>(RES, ob, abi, ell, list, jb, clr, A, lane, XY, rec, res_s, D, rc);
  return __any_sync(FULL, zero) ? 1u : 0u;
}

// Any obstacle kinds, one obstacle at a time.  GUARD handles x~ = y~ = 0
// exactly (G18: alpha = 0, d = 1 -> delta = (a, 0)).
template <int M>
__device__ __forceinline__ void coll_general(const bool RES, const bool GUARD, const float2* __restrict__ ob,
                                             const float4* __restrict__ abi,
                                             int n, int g, int S, const float2 (&XY)[M],
                                             const float (&rec)[M], const float (&res_s)[M], float2 (&D)[M],
                                             float& rc) {
#pragma unroll 1
  for (int j = g; j < n; j += S) {
    const float2 o = ob[j * QP];
    const float4 ab = abi[j];
    const float a = ab.x, b = ab.y;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const float xt = XY[i].x - o.x, yt = XY[i].y - o.y;
      const float x2 = xt * xt, y2 = yt * yt;
      float dx, dy;
      if (ab.w == 1.f) {
        // f = N / D >= 1 / rho (d* >= 1): a f - 1 = b (a - b) y~^2 / D and
        // b f - 1 = a (b - a) x~^2 / D exactly, formed without the cancellation of
        // a f - 1 (a far obstacle leaves a f ~ 1, and fp32 would keep only the
        // rounding error of a f); otherwise f = 1 / rho (inside, d = 1)
        const float N = fmaf(b, y2, a * x2), D = fmaf(b * b, y2, a * a * x2);
        const float ri = rsqrt_ftz(x2 + y2), rD = rcp_approx(D);   // ~1 ulp, no cancellation after it
        const bool out = N * rD >= ri;
        const float amb = a - b;   // exact (Sterbenz) for b <= a <= 2 b and vice versa
        const float kx = b * amb, ky = -a * amb;   // per obstacle
        const float fx = out ? kx * y2 * rD : fmaf(a, ri, -1.f);
        const float fy = out ? ky * x2 * rD : fmaf(b, ri, -1.f);
        dx = xt * fx;
        dy = yt * fy;
      } else {
        const float R2 = (ab.w == 0.f) ? x2 + y2 : fmaf(a * a, y2, b * b * x2);
        const float num = (ab.w == 0.f) ? a : ab.z;
        const float sc = fmaxf(fmaf(num, rsqrt_ftz(R2), -1.f), 0.f);
        dx = sc * xt;
        dy = sc * yt;
      }
      if (GUARD && x2 + y2 == 0.f) { dx = a; dy = 0.f; }
      D[i].x += dx;
      D[i].y += dy;
      if (RES) rc = fmaf(dx, dx - 2.f * rec[i], fmaf(dy, dy - 2.f * res_s[i], rc));
    }
  }
}

// ------------------------------------------------------ temporal culling
// Every iteration moves the circle centres of sample t by at most
//   |(dx, dy)| + max_i |r_i| |dpsi|        (|d cos psi| <= |d psi|)
// where (dx, dy, dpsi) is the change of the evaluated x, y, psi since the
// previous evaluation.  A per-(instance, round) clock A sums the warp maximum of
// this bound over the iterations.  An obstacle whose stamped clearance
// (coll_circ) still exceeds the movement since its stamp plus CULL_MARGIN
// cannot have any circle inside it in this round, so its contribution is
// exactly zero and it is skipped: the result is bitwise that of testing it.
// The margin covers the fp32 rounding of the evaluated samples (< 1e-4 m for
// deviations up to 1 km).
constexpr float CULL_MARGIN = 2e-3f;

// Active list of one round: obstacles whose clearance no longer covers the
// movement since it was stamped.  Returns its length.
__device__ __forceinline__ int build_active(const float* __restrict__ clr, int* __restrict__ list, int npad,
                                            float lim, int lane) {
  int na = 0;
  if (npad <= 32) {   // the common case: one ballot
    const bool act = (lane < npad) && !(clr[lane] > lim);   // NaN clock or stamp: active
    const unsigned bal = __ballot_sync(FULL, act);
    if (act) list[__popc(bal & ((1u << lane) - 1u))] = lane;
    na = __popc(bal);
  } else {   // two words per step: both loads and ballots in flight
    const unsigned below = (1u << lane) - 1u;
#pragma unroll 1
    for (int j0 = 0; j0 < npad; j0 += 64) {
      const int ja = j0 + lane, jb = ja + 32;
      const bool aa = (ja < npad) && !(clr[ja] > lim);
      const bool ab = (jb < npad) && !(clr[jb] > lim);
      const unsigned ba = __ballot_sync(FULL, aa), bb = __ballot_sync(FULL, ab);
      const int nA = __popc(ba);
      if (aa) list[na + __popc(ba & below)] = ja;
      if (ab) list[na + nA + __popc(bb & below)] = jb;
      na += nA + __popc(bb);
    }
  }
  __syncwarp();
  return na;
}

// ---------------------------------------------------------------- phase B
// c, s at every sample, theta = atan2(s, c) (Eq. 19; G18) into the
// warp's smem arrays, and the warp total of P^T theta into ws->pth[0..10].
// FM (all six boundary rows, P:269 / G11): the rows pin c_psi[0..2] and c_psi[8..10]
// (position, velocity and acceleration at both ends involve only those
// coefficients), so the heading step's KKT inverse Kp11 = Z (Z^T H Z)^-1 Z^T with
// Z = [e3 .. e7] vanishes outside rows / columns 3..7: xi2 needs only the entries
// 3..7 of P^T theta.  The other six enter only lambda_psi's boundary components,
// which feed nothing until the output: their theta terms are summed per sample
// over the iterations (thsum) and contracted once at the end.
template <bool FM, class WarpSmem>
__device__ __forceinline__ void phase_theta(const float* __restrict__ Pt, const double* __restrict__ Pt64,
                                            WarpSmem* ws, int lane, int q, int w, int T, bool sum_theta) {
  float2 ccs[NV + 1];   // (c_c, c_s) per Bernstein index
#pragma unroll
  for (int k = 0; k < NV + 1; k += 2) {
    const float4 v = reinterpret_cast<const float4*>(&ws->ccs[0][0])[k >> 1];
    ccs[k] = make_float2(v.x, v.y);
    ccs[k + 1] = make_float2(v.z, v.w);
  }
  constexpr int NA = FM ? 5 : 16;
  double acc[NA];   // P^T theta in fp64 (exact products, no cancellation loss)
#pragma unroll
  for (int k = 0; k < NA; ++k) acc[k] = 0.0;
  const int nr = (q + 31) >> 5;
#pragma unroll 2
  for (int uu = 0; uu < QP / 32; ++uu) {   // two rounds in flight: independent atan2 chains
    const int u = (T - 1 - w) + uu * T;      // this warp's rounds (the leader gets the last, lightest)
    if (u >= nr) break;
    const int t = 32 * u + lane;
    float p[NV];
    load_basis_row(Pt, t, p);
    float2 cs = make_float2(0.f, 0.f);   // (c, s) = (P c_c, P c_s)
#pragma unroll
    for (int k = 0; k < NV; ++k) cs = fma2(bc2(p[k]), ccs[k], cs);
    const float tht = atan2_fast(cs.y, cs.x);   // atan2(0, 0) = 0 (G18)
    ws->cs[t] = cs;
    ws->th[t] = tht;
    const double thd = f2d(tht);
    if constexpr (FM) {
#pragma unroll
      for (int j = 0; j < 5; ++j) acc[j] = fma(Pt64[(3 + j) * QP64 + t], thd, acc[j]);
      if (sum_theta) ws->thsum[t] += thd;
    } else {
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = fma(Pt64[k * QP64 + t], thd, acc[k]);
    }
  }
  if constexpr (FM) {
    // entries 3..6 as 4 transpose-reduce slots, entry 7 as a butterfly sum: the
    // lane bits pair in the same order as below, so the entries are bitwise the same
    const double v4 = tr_reduce<4>(acc, lane);       // entry 3 + (lane >> 3)
    const double v1 = warp_sum(acc[4]);              // entry 7
    if (!(lane & 7)) ws->part_th[w][3 + (lane >> 3)] = v4;
    if (lane == 0) ws->part_th[w][7] = v1;
  } else {
    // 11 entries as 8 + 4 transpose-reduce slots
    const double v8 = tr_reduce<8>(acc, lane);        // entry lane >> 2
    const double v4 = tr_reduce<4>(acc + 8, lane);    // entry 8 + (lane >> 3)
    if (!(lane & 3)) ws->part_th[w][lane >> 2] = v8;
    if (!(lane & 7) && 8 + (lane >> 3) < NV) ws->part_th[w][8 + (lane >> 3)] = v4;
  }
}

// FM, end of the solve: the boundary components k in {0, 1, 2, 8, 9, 10} of
// rho_psi sum_it P^T theta_it (from thsum), summed over the team into part_th[w][k].
template <class WarpSmem>
__device__ __forceinline__ void theta_sum_boundary(const double* __restrict__ Pt64, WarpSmem* ws, int lane, int q,
                                                   int w, int T) {
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const int nr = (q + 31) >> 5;
#pragma unroll 1
  for (int u = T - 1 - w; u < nr; u += T) {
    const int t = 32 * u + lane;
    const double ts = ws->thsum[t];
#pragma unroll
    for (int i = 0; i < 6; ++i) acc[i] = fma(Pt64[(i < 3 ? i : i + 5) * QP64 + t], ts, acc[i]);
  }
  const double v8 = tr_reduce<8>(acc, lane);   // slot lane >> 2: k = slot (< 3) or slot + 5
  const int slot = lane >> 2;
  if (!(lane & 3) && slot < 6) ws->part_th[w][slot < 3 ? slot : slot + 5] = v8;
}

// ---------------------------------------------------------------- phase D
// D1 (per round): trajectory at the lane's sample, velocity / acceleration and
// collision projections, and the per-sample vectors of h = F^T (F xi1 - g)
//   U0 = n R1 e_c - D_x, U1 = (n R2 + 1) e_c - E_x, U2, U3 likewise for y,
//   U4 = -dv_x, U5 = -da_x, U6 = -dv_y, U7 = -da_y
// written to shared memory; D2: contraction with P, Pdot, Pddot (FP64 MMA).
template <int M, bool RES, bool ELLK, class WarpSmem>
__device__ __forceinline__ void phase_project(const Proj& pa, const float (&r)[M], WarpSmem* ws,
                                              int lane, int w, int T, int team, double (&hreg)[2],
                                              float& clkreg, PhaseClock& pc) {
  const int q = pa.q, n = pa.n;
  const float* __restrict__ Pt = pa.Pt;
  float res = 0.f, rps = 0.f;
  // D2: partial G = P^T U over this warp's own samples on the FP64 tensor
  // cores (q x 11 basis, U = [U0 .. U7]: 11 x 8 outputs, all of them used):
  // two m8n8k4 row tiles (basis rows 0..15, rows >= 11 clamped and
  // discarded), k = 4 samples per step, issued right after each round's U so
  // the MMAs overlap the next round's projections.  The Pdot / Pddot terms
  // follow from G through Pdot^T u = Dm^T (P^T u) (see dm_apply), after the
  // team sum.  fp64 products and sums: h -> 0 at a fixed point of the
  // multipliers, so the sum over samples cancels and fp32 accumulation would
  // dominate the error.  Each warp contracts the
  // samples it projected itself, so no team barrier separates D1 from D2.
  const double* __restrict__ P64 = pa.Pt64;
  const int aoff0 = (lane >> 2) * QP64 + (lane & 3), aoff1 = min(8 + (lane >> 2), NV - 1) * QP64 + (lane & 3);
  const float* __restrict__ ucol = &ws->U[lane >> 2][lane & 3];   // B fragment: U[k = lane % 4][n = lane / 4]
  // two accumulator sets (even / odd MMA steps): dependent chains of 4, not 8
  double g0[2] = {0.0, 0.0}, g1[2] = {0.0, 0.0}, e0[2] = {0.0, 0.0}, e1[2] = {0.0, 0.0};
  auto contract_round = [&](int u) {
    const int t0 = 32 * u;
    const float* __restrict__ up = ucol + t0;
    const double* __restrict__ a0 = P64 + aoff0 + t0;
    const double* __restrict__ a1 = P64 + aoff1 + t0;
    if (t0 + 32 <= q) {   // full round: 8 steps, immediate offsets
#pragma unroll
      for (int st = 0; st < 8; ++st) {
        const double b = f2d(up[4 * st]);
        if (st & 1) {
          mma_f64_884(e0, a0[4 * st], b);
          mma_f64_884(e1, a1[4 * st], b);
        } else {
          mma_f64_884(g0, a0[4 * st], b);
          mma_f64_884(g1, a1[4 * st], b);
        }
      }
    } else {
      const int ns = (q - t0 + 3) >> 2;
#pragma unroll 1
      for (int st = 0; st < ns; ++st) {
        const double b = f2d(up[4 * st]);
        mma_f64_884(g0, a0[4 * st], b);
        mma_f64_884(g1, a1[4 * st], b);
      }
    }
  };
#pragma unroll 1
  for (int u = T - 1 - w; u < pa.rounds; u += T) {   // this warp's rounds (leader: the lightest)
    // samples t >= q of the last round have a zero basis row and far-away
    // obstacle slots: they project to nothing and are excluded from the sums
    const int t = 32 * u + lane;
    const bool valid = t < q;
    BMC_SUB(pc, -1);
    // x = P c, xdot = Pdot c = P (Dm c), xddot = P (Dm^2 c): one basis row per k
    // (x, y), (xdot, ydot), (xddot, yddot) as fp32 pairs (FFMA2), psi scalar
    float2 xy = make_float2(0.f, 0.f), xyd = xy, xydd = xy;
    float psi = 0.f;
    {
      float cp[NV], pr[NV];
      load12(ws->cf4[w], cp);
      load_basis_row(Pt, t, pr);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const float p = pr[k];
        const float4 c0 = *reinterpret_cast<const float4*>(&ws->cpos[k][0]);
        float4 c1;   // Dm^2 c of indices k, k + 1
        if (!(k & 1)) c1 = reinterpret_cast<const float4*>(&ws->cdd[0][0])[k >> 1];
        xy = fma2(bc2(p), make_float2(c0.x, c0.y), xy);
        xyd = fma2(bc2(p), make_float2(c0.z, c0.w), xyd);
        xydd = fma2(bc2(p), (k & 1) ? make_float2(c1.z, c1.w) : make_float2(c1.x, c1.y), xydd);
        psi = fmaf(p, cp[k], psi);
      }
    }
    const float x = xy.x, y = xy.y;
    // velocity / acceleration: g = projection onto the bound disk (G6, G7)
    // negated offsets -(g - v) = v max(1 - v_max / |v|, 0) (bitwise the negation of the
    // offset v min(v_max / |v| - 1, 0))
    const float nsv = fmaxf(fmaf(-pa.v_max, rsqrt_ftz(fmaf(xyd.y, xyd.y, xyd.x * xyd.x)), 1.f), -0.f);
    const float nsa = fmaxf(fmaf(-pa.a_max, rsqrt_ftz(fmaf(xydd.y, xydd.y, xydd.x * xydd.x)), 1.f), -0.f);
    const float2 dv = mul2(xyd, bc2(nsv)), da = mul2(xydd, bc2(nsa));
    const float dvx = dv.x, dvy = dv.y, dax = da.x, day = da.y;   // negated offsets
    if (RES && valid) res += dvx * dvx + dvy * dvy + dax * dax + day * day;
    float2 hd;   // heading (cos psi, sin psi)
    sincos_fast(psi, &hd.y, &hd.x);
    const float2 ecs = sub2(ws->cs[t], hd);   // (c - cos psi, s - sin psi)
    const float ec = ecs.x, es = ecs.y;
    float2 XY[M], D[M];
    float rec[M], res_s[M];
    float base = 0.f;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      XY[i] = fma2(bc2(r[i]), hd, xy);   // circle centre (x + r_i cos psi, y + r_i sin psi)
      D[i] = make_float2(0.f, 0.f);
      rec[i] = 0.f;
      res_s[i] = 0.f;
    }
    if (RES) {   // residual-only terms
#pragma unroll
      for (int i = 0; i < M; ++i) {
        rec[i] = r[i] * ec;
        res_s[i] = r[i] * es;
        base = fmaf(rec[i], rec[i], fmaf(res_s[i], res_s[i], base));
      }
    }
    float rc = 0.f;
    const float2* ob = pa.obs + t;
    BMC_SUB(pc, 12);   // evaluation, velocity / acceleration, heading
    // circular obstacles and scaled-rule ellipses: culled closed forms
    // (coll_circ); literal-rule ellipses: the plain loop.  x~ = y~ = 0 exactly
    // (G18, rare: detected by the stamp reductions when culled, by a non-finite
    // sum in the plain loop) reruns the round with the guarded plain loop; one
    // call site keeps the hot loop small in the instruction cache.
    bool general = ELLK ? !pa.all_cull : !pa.all_circ;
    bool rerun = false;   // warp-uniform: x~ = y~ = 0 exactly somewhere -> guarded pass (G18)
    if (!general) {
      float* clr = pa.clr + u * pa.nclr;
      const float clk0 = __shfl_sync(FULL, clkreg, u);
      // movement bound of this evaluation (see "temporal culling") -> the round's clock
      const float2 dxy = sub2(xy, ws->pxy[t]);
      const float ppsi0 = ws->ppsi[t];
      ws->pxy[t] = xy;
      ws->ppsi[t] = psi;
      const float2 sq = mul2(dxy, dxy);
      // |.| of a NaN keeps a NaN bit pattern, which is above +inf: the clock becomes NaN
      const float mv = fmaf(pa.rabs, fabsf(psi - ppsi0), sqrt_approx(sq.x + sq.y) * 1.000001f);
      const float A = clk0 + __uint_as_float(__reduce_max_sync(FULL, __float_as_uint(fabsf(mv))));
      if (lane == u) clkreg = A;
      const int na = build_active(clr, pa.list, pa.npad, pa.no_cull ? INFINITY : A + CULL_MARGIN, lane);
#ifdef BMC_PROFILE
      pc.acc[9] += na;
#endif
      BMC_SUB(pc, 13);   // culling clock and active list
      // the exact zero shows up in the stamp reductions (a round minimum r2 of 0)
      if (!ELLK || pa.all_circ)
        rerun = coll_circ<M, false>(RES, ob, pa.abi, pa.ell, pa.list, na, clr, A, lane, XY, rec, res_s, D, rc) != 0u;
      else
        rerun = coll_circ<M, ELLK>(RES, ob, pa.abi, pa.ell, pa.list, na, clr, A, lane, XY, rec, res_s, D, rc) != 0u;
    }
    else {   // the plain loop (ellipses the culled pass cannot take): a non-finite sum flags the exact zero
      coll_general<M>(RES, false, ob, pa.abi, n, 0, 1, XY, rec, res_s, D, rc);
      float chk = rc;
#pragma unroll
      for (int i = 0; i < M; ++i) chk += D[i].x + D[i].y;
      rerun = __any_sync(FULL, !isfinite(chk));
    }
    if (rerun) {   // rare: redo the round with the guarded plain loop (G18)
#pragma unroll
      for (int i = 0; i < M; ++i) D[i] = make_float2(0.f, 0.f);
      rc = 0.f;
      coll_general<M>(RES, true, ob, pa.abi, n, 0, 1, XY, rec, res_s, D, rc);
    }
    BMC_SUB(pc, 14);   // collision projections
    float2 nDs = make_float2(0.f, 0.f), nE = nDs;   // -sum_i delta_i, -sum_i r_i delta_i
#pragma unroll
    for (int i = 0; i < M; ++i) {
      nDs = sub2(nDs, D[i]);
      nE = fma2(bc2(-r[i]), D[i], nE);
    }
    {
      const float2 u02 = fma2(bc2(pa.nR1), ecs, nDs);
      const float2 u13 = fma2(bc2(pa.nR2p1), ecs, nE);
      ws->U[0][t] = u02.x;
      ws->U[1][t] = u13.x;
      ws->U[2][t] = u02.y;
      ws->U[3][t] = u13.y;
      ws->U[4][t] = dvx;   // -(g_v - v): the velocity / acceleration offsets are stored negated
      ws->U[5][t] = dax;
      ws->U[6][t] = dvy;
      ws->U[7][t] = day;
    }
    if (valid) {
      if (RES) res += fmaf((float)n, base, rc) + ec * ec + es * es;
      const float dth = ws->th[t] - psi;
      rps = fmaf(dth, dth, rps);
    }
    __syncwarp();   // the round's U is complete
    contract_round(u);
    BMC_SUB(pc, 15);   // U and the round's MMAs
  }
  __syncwarp();
  BMC_TICK(pc, 10);
  // C fragment: G[row g8 (+ 8)][column 2 c4 + i] -> partial slots [column][row]
  {
    const int g8 = lane >> 2, c4 = lane & 3;
    double* hp = pa.hp + w * HP_SLOTS;
    hp[(2 * c4) * 12 + g8] = g0[0] + e0[0];
    hp[(2 * c4 + 1) * 12 + g8] = g0[1] + e0[1];
    if (8 + g8 < NV) {
      hp[(2 * c4) * 12 + 8 + g8] = g1[0] + e1[0];
      hp[(2 * c4 + 1) * 12 + 8 + g8] = g1[1] + e1[1];
    }
  }
  if (RES) {   // residual partials must be visible to the team before the barrier
    res = warp_sum(res);
    rps = warp_sum(rps);
    if (lane == 0) {
      ws->part_res[w][0] = res;
      ws->part_res[w][1] = rps;
    }
  }
  BMC_TICK(pc, 5);
  team_sync(team, T);   // every warp's partials are in place
  BMC_TICK(pc, 6);
  // channel owners (T = 1: the warp owns both; T >= 2: warps 0 and 1) sum the
  // team's partials in warp order and assemble
  //   h_pos  = P^T U0 + Dm^T (P^T U4) + Dm^T Dm^T (P^T U5)   (x; y: U2, U6, U7)
  //   h_copy = P^T U1                                          (x; y: U3)
  // channels owned (compile-time for teams of 1 and 2: no branch)
  const int nch = (T == 1) ? 2 : (T == 2 ? 1 : (w < 2 ? 1 : 0));
  const int k = lane;
#pragma unroll
  for (int ci = 0; ci < 2; ++ci) {   // unrolled: hreg stays in registers
    if (ci >= nch) break;
    const int ch = (T == 1) ? ci : w;
    // lanes k < 11: (P^T U)[k] of U0/U2 (gp), U4/U6 (gv), U5/U7 (ga);
    // lanes 11..21: gp = (P^T U1/U3)[k - 11].  Branch-free: other lanes read
    // clamped slots and meet zero weights in dmT_apply.
    const int kk = (k < NV) ? k : min(k - NV, NV - 1);
    const int colp = (k < NV) ? 2 * ch : 2 * ch + 1;
    double gp = 0.0, gv = 0.0, ga = 0.0;
#pragma unroll
    for (int ww = 0; ww < T_MAX; ++ww) {
      if (ww < T) {
        const double* hp = pa.hp + ww * HP_SLOTS;
        gp += hp[colp * 12 + kk];
        gv += hp[(4 + 2 * ch) * 12 + kk];
        ga += hp[(5 + 2 * ch) * 12 + kk];
      }
    }
    // Dm^T gv + Dm^T Dm^T ga = Dm^T (gv + Dm^T ga)
    const double z = dmT_apply(ga, pa.dmtab, k) + gv;
    const double d = dmT_apply(z, pa.dmtab, k);
    hreg[ci] = (k < NV) ? gp + d : gp;   // lane k holds h[k] (k < 22) of its channel
  }
}

// ---------------------------------------------------------------- kernel
#ifdef BMC_MAXNREG   // experiments: register cap below the 128 of 16 warps per SM
#define BMC_KERNEL_BOUNDS __maxnreg__(BMC_MAXNREG)
#else
#define BMC_KERNEL_BOUNDS __launch_bounds__(512)
#endif
// ELLK: scaled-rule ellipses (alpha_rule 1) take the culled pass (coll_circ<M, true>);
// with the literal rule (alpha_rule 0) ellipses have no zero offset outside (G8), so
// that kernel keeps only the circle form and sends ellipse scenes to the plain loop.
// BD: M and K11 block diagonal (symmetric footprint, sum r_i = 0: every configured
// one); a compile-time branch, so the common kernel carries only its mat-vec.
template <int M, int TT, bool ELLK, bool BD, bool FM>
__global__ void BMC_KERNEL_BOUNDS bmc_am_kernel(const __grid_constant__ KernelArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, wpc = blockDim.x >> 5;
  const int n = a.n, q = a.q, K = a.iters;
  const double* sf = reinterpret_cast<const double*>(smem);
  const float* Pt = reinterpret_cast<const float*>(smem + BlobLayout::bytes_f64);
  const double* Pt64 = reinterpret_cast<const double*>(smem + BlobLayout::bytes_f64 + BlobLayout::bytes_f32(QP));
  float2* obs = reinterpret_cast<float2*>(smem + BlobLayout::bytes(QP));
  const int npad = pad_obstacles(n), nclr = clr_stride(n);
  float4* abi = reinterpret_cast<float4*>(obs + (size_t)(npad + 1) * QP);
  float4* ell = abi + npad + 1;
  double* ub = reinterpret_cast<double*>(ell + npad + 1);
  using WarpSmem = WarpSmemT<TT>;
  WarpSmem* wsbase = reinterpret_cast<WarpSmem*>(ub + U_DOUBLES);
  constexpr int T = TT;                              // warps per instance (compile time: folds the
  const int ipc = wpc / T;                           // team bookkeeping), instances per CTA
  // instance slot in the CTA and rank in its team.  Warp i runs on SMSP i % 4.
  // Teams of 2 straddle the scheduler pairs: in every group of 4 warps, warps
  // (0, 2) and (1, 3) form the teams, so rank 0 (rounds 1, 3: one round plus
  // the tail at q = 100) sits on SMSP 0 or 1 and rank 1 (rounds 0, 2) on SMSP 2
  // or 3; a trailing pair (wpc % 4 == 2) forms one team on SMSPs 0 and 1.  With
  // 7 teams (C3) SMSPs 0 and 1 hold 4 warps and 2 and 3 hold 3: the light ranks
  // go where the schedulers are busiest (C3 0.623 -> 0.592 ms).
  int team_, w_;
  if (T == 2) {
    const int g = warp >> 2, rr = warp & 3;
    if (4 * g + 3 < wpc) {
      team_ = 2 * g + (rr & 1);
      w_ = rr >> 1;
    } else {
      team_ = 2 * g;
      w_ = rr;
    }
  } else {
    team_ = warp / T;
    w_ = warp - team_ * T;
  }
  const int team = team_, w = w_;
  float* clr_base = reinterpret_cast<float*>(wsbase + ipc);
  int* list_base = reinterpret_cast<int*>(clr_base + (size_t)ipc * T_MAX * nclr);
  double* hp_base = reinterpret_cast<double*>(list_base + (size_t)wpc * nclr);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(hp_base + (TT > 1 ? (size_t)wpc * HP_SLOTS : 0));

  BMC_STAMP(0);   // CTA start
  // --- stage the batch-invariant data -------------------------------------
  if (tid == 0) mbar_init(mbar, 1);
  __syncthreads();
  const unsigned blob_bytes = (unsigned)BlobLayout::bytes(QP);
  if (tid == 0) {
    mbar_arrive_expect_tx(mbar, blob_bytes);
    constexpr unsigned CHUNK = 16384;
    for (unsigned off = 0; off < blob_bytes; off += CHUNK) {
      const unsigned nbytes = (blob_bytes - off < CHUNK) ? (blob_bytes - off) : CHUNK;
      bulk_g2s(smem + off, a.blob + off, nbytes, mbar);
    }
  }
  // obstacles relative to the boundary line (x_ref(t), y_ref(t)), computed in
  // fp64 and rounded once; padding samples far away
  const double inv_q1 = 1.0 / (double)(q - 1);
  for (int idx = tid; idx < (npad + 1) * QP; idx += blockDim.x) {
    const int j = idx / QP, t = idx - j * QP;
    float2 v = make_float2(1.0e4f, 1.0e4f);
    if (t < q && j < n) {
      const double tau = (double)t * inv_q1;
      v = make_float2(d2f((double)__ldg(a.obs_xy + (size_t)(2 * j) * q + t) - fma(a.ref_dx, tau, a.ref_x0)),
                      d2f((double)__ldg(a.obs_xy + (size_t)(2 * j + 1) * q + t) - fma(a.ref_dy, tau, a.ref_y0)));
    }
    obs[idx] = v;
  }
  int circ = 1, cull = 1;
  for (int j = n + tid; j <= npad; j += blockDim.x) {   // far dummies: zero offset under either form
    abi[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    ell[j] = make_float4(1.f, 1.f, 0.f, 0.f);
  }
  for (int i = tid; i < ipc * T_MAX * nclr; i += blockDim.x) clr_base[i] = -1.0e30f;   // never tested
  for (int j = tid; j < n; j += blockDim.x) {
    const float aa = __ldg(a.obs_ab + 2 * j), bb = __ldg(a.obs_ab + 2 * j + 1);
    const float kind = (aa == bb) ? 0.f : (a.alpha_rule == 0 ? 1.f : 2.f);
    // z: a b (numerator of the scaled rule, coll_general)
    abi[j] = make_float4(aa, bb, aa * bb, kind);
    ell[j] = make_float4(1.f / aa, 1.f / bb, fmaxf(aa, bb), 0.f);
    circ &= (aa == bb);
    cull &= (kind != 1.f);   // the literal rule has no zero offset outside the ellipse (G8)
  }
  for (int i = tid; i < ipc * (NV + 1) * 4; i += blockDim.x)
    (&wsbase[i / ((NV + 1) * 4)].cpos[0][0])[i % ((NV + 1) * 4)] = 0.f;
  for (int i = tid; i < ipc * (NV + 1) * 2; i += blockDim.x)
    (&wsbase[i / ((NV + 1) * 2)].cdd[0][0])[i % ((NV + 1) * 2)] = 0.f;
  for (int i = tid; i < ipc * (NV + 1) * 2; i += blockDim.x)
    (&wsbase[i / ((NV + 1) * 2)].ccs[0][0])[i % ((NV + 1) * 2)] = 0.f;
  for (int i = tid; i < ipc * TT * 12; i += blockDim.x)
    (&wsbase[i / (TT * 12)].cf4[0][0])[i % (TT * 12)] = 0.f;
  for (int i = tid; i < ipc * 8 * QPU; i += blockDim.x) (&wsbase[i / (8 * QPU)].U[0][0])[i % (8 * QPU)] = 0.f;
  for (int i = tid; i < ipc * (3 * QP + 2 * T_MAX); i += blockDim.x)
    (&wsbase[i / (3 * QP + 2 * T_MAX)].pxy[0].x)[i % (3 * QP + 2 * T_MAX)] = 0.f;
  if (FM)
    for (int i = tid; i < ipc * QP; i += blockDim.x) wsbase[i / QP].thsum[i % QP] = 0.0;
  BMC_STAMP(4);   // staging loops issued (thread 0)
  const bool all_circ = __syncthreads_and(circ);
  const bool all_cull = __syncthreads_and(cull);
  BMC_STAMP(5);   // staging done
  mbar_wait(mbar, 0);
  BMC_STAMP(6);   // blob landed
  __syncthreads();
  if (tid < 32) dm_table(ub + DM_TAB, tid, a.T);
  if (tid < NV2) {   // u = K12 b per channel (boundary part of Eq. 4)
    double sx = 0.0, sy = 0.0;
    for (int rr = 0; rr < a.nb; ++rr) {
      sx = fma(sf[BlobLayout::K12t + rr * NV2 + tid], a.b[0][rr], sx);
      sy = fma(sf[BlobLayout::K12t + rr * NV2 + tid], a.b[1][rr], sy);
    }
    ub[tid] = sx;
    ub[NV2 + tid] = sy;
    if (tid < NV) {
      double s = 0.0;
      for (int rr = 0; rr < a.nb; ++rr) s = fma(sf[BlobLayout::Kp12t + rr * NV + tid], a.b[2][rr], s);
      ub[2 * NV2 + tid] = s;
    }
  }
  __syncthreads();
  if (FM && tid < NV) {   // the pinned coefficients' part of (rho_psi P^T P) xi2 (xi2[j] = u_psi[j] there)
    double s = 0.0;
    for (int j = 0; j < NV; ++j)
      if (j < 3 || j > 7) s = fma(sf[BlobLayout::Gppt + j * NV + tid], ub[2 * NV2 + j], s);
    ub[CG_TAB + tid] = s;
  }
  __syncthreads();
  BMC_STAMP(1);   // prologue done

  Proj pa;
  pa.Pt = Pt;
  pa.Pt64 = Pt64;
  pa.obs = obs;
  pa.abi = abi;
  pa.q = q;
  pa.n = n;
  pa.rounds = (q + 31) / 32;
  pa.all_circ = all_circ;
  pa.all_cull = all_cull;
  pa.ell = ell;
  pa.nR1 = a.nR1;
  pa.nR2p1 = a.nR2p1;
  pa.v_max = a.v_max;
  pa.a_max = a.a_max;
  pa.rabs = 0.f;
  for (int i = 0; i < M; ++i) pa.rabs = fmaxf(pa.rabs, fabsf(a.r[i]));
  pa.npad = npad;
  pa.nclr = nclr;
  pa.clr = clr_base + (size_t)team * T_MAX * nclr;
  pa.list = list_base + (size_t)warp * nclr;
  pa.hp = (TT > 1) ? hp_base + (size_t)team * T * HP_SLOTS : reinterpret_cast<double*>(&wsbase[team].U[0][0]);
  pa.dmtab = ub + DM_TAB;
  pa.no_cull = a.no_cull != 0;
  float r[M];
#pragma unroll
  for (int i = 0; i < M; ++i) r[i] = a.r[i];

  WarpSmem* ws = wsbase + team;
  // Every warp runs the iteration (a warp past the end of the batch redoes the
  // last instance and writes nothing): no branch around the shuffles, so the
  // compiler emits no divergence fallback paths for them.
  const long long l_raw = (long long)blockIdx.x * ipc + team;
  const bool active = l_raw < a.B;
  const long long l = active ? l_raw : a.B - 1;
  {
    const int k = lane;
    const double rho = a.rho, rho_psi = a.rho_psi;
    const double* dmtab = ub + DM_TAB;
    // channels owned by this warp (phases A, D2, E): both for T = 1, channel w for w < 2
    const int nown = (T == 1) ? 2 : (T == 2 ? 1 : (w < 2 ? 1 : 0));   // compile-time for T <= 2
    const int chb = (T == 1) ? 0 : w;
    double xi[2] = {0.0, 0.0}, lam[2] = {0.0, 0.0}, cref[2] = {0.0, 0.0};
    double hreg[2] = {0.0, 0.0};   // h = F^T (F xi1 - g) of the owned channels, lane k: entry k (phase D2)
    float clkreg = 0.f;            // culling clock of round `lane` (lanes < rounds)
    const float* ini = a.init + l * 3 * NV;
    const float* li = a.lambda_in ? a.lambda_in + l * 5 * NV : nullptr;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (c >= nown) break;
      const int ch = chb + c;
      // Bernstein control points of the boundary line (linear precision: c_k = x0 + dx k / 10)
      const double r0 = ch ? a.ref_y0 : a.ref_x0, rd = ch ? a.ref_dy : a.ref_dx;
      cref[c] = (k < NV) ? fma(rd, (double)k / (NV - 1), r0) : 0.0;
      if (k < NV) xi[c] = ini[ch * NV + k];   // step 1: copies start at 0 (G15)
      if (li && k < NV2) lam[c] = li[ch * NV2 + k];
    }
    double xi2r = (k < NV) ? (double)ini[2 * NV + k] : 0.0;
    double lamp = (li && k < NV) ? (double)li[2 * NV2 + k] : 0.0;
    // lambda_psi step of Eq. 23b, deferred from phase C to the next phase A (where it
    // overlaps the xi1 mat-vec): lamp <- lamp - (rho_psi P^T P xi2 - rho_psi P^T theta)
    double pth_prev = 0.0;
    bool lp_pending = false;
    auto lampsi_step = [&]() {
      const int k1 = min(k, NV - 1);
      double g4[4] = {0.0, 0.0, 0.0, 0.0};
      if (FM) {   // xi2 moves only in its coefficients 3..7
        g4[0] = ub[CG_TAB + k1];
#pragma unroll
        for (int j = 3; j < 8; ++j) g4[j & 3] = fma(sf[BlobLayout::Gppt + j * NV + k1], ws->xi2w[w][j], g4[j & 3]);
      } else {
#pragma unroll
        for (int j = 0; j < NV; ++j) g4[j & 3] = fma(sf[BlobLayout::Gppt + j * NV + k1], ws->xi2w[w][j], g4[j & 3]);
      }
      const double v = lamp - (((g4[0] + g4[1]) + (g4[2] + g4[3])) - rho_psi * pth_prev);
      lamp = (k < NV) ? v : 0.0;
    };
    if (k < NV) { ws->cf4[w][k] = d2f(xi2r); ws->xi2w[w][k] = xi2r; }

    float r1sq = 0.f, rpsq = 0.f;
    const bool trace = a.res_trace != nullptr;
    // it = -1 is the initialisation of xi3, xi4 / g on the initial trajectory
    // (G15); every phase has a single call site so each is inlined once.
    // Team protocol per iteration: A (channel owners) | B (all, own rounds) |
    // C (all, redundant) + D1 (all, own rounds) | D2 + E (channel owners).
    PhaseClock pc;
#ifdef BMC_PROFILE
    pc.t0 = clock64();
#endif
#pragma unroll 1
    for (int it = -1; it < K; ++it) {
      // ---- A: xi1 step, Eq. 13/17 via Eq. 4 (fp64), for the owned channels --------
      // (both channels for T = 1: their mat-vecs are independent and interleave)
      double vnew[2] = {0.0, 0.0};
      if (it >= 0) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c >= nown) break;
          if (k < NV2) ws->rhs[chb + c][xpad(k)] = lam[c] - rho * hreg[c];
        }
        __syncwarp();
        if (nown > 0 && lp_pending) lampsi_step();
        // every lane runs row min(k, 21) (no divergent branch); lanes >= 22 keep 0
        const int kc = min(k, NV2 - 1);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c >= nown) break;
          const int ch = chb + c;
          // 8 independent fp64 chains (depth <= 6): the step is latency-bound.  With a
          // symmetric footprint M and K11 are block diagonal (setup.cpp): row k only
          // meets the columns of its own block (c_x rows 0..10, c_c rows 11..21).
          double acc[8] = {ub[ch * NV2 + kc], 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
          if (BD) {   // row kc of its block and the block's vector entries, two per 16-byte load
            const int j0 = (kc < NV) ? 0 : xpad(NV);
            const double2* mrow = reinterpret_cast<const double2*>(sf + BlobLayout::Mb + kc * BlobLayout::BD_ROW);
            const double2* krow = reinterpret_cast<const double2*>(sf + BlobLayout::Kb + kc * BlobLayout::BD_ROW);
            const double2* xv = reinterpret_cast<const double2*>(&ws->xi1[ch][j0]);
            const double2* rv = reinterpret_cast<const double2*>(&ws->rhs[ch][j0]);
#pragma unroll
            for (int jj = 0; jj < NV; jj += 2) {
              const double2 m2 = mrow[jj >> 1], k2 = krow[jj >> 1], x2 = xv[jj >> 1], r2 = rv[jj >> 1];
              acc[jj & 3] = fma(m2.x, x2.x, acc[jj & 3]);
              acc[4 + (jj & 3)] = fma(k2.x, r2.x, acc[4 + (jj & 3)]);
              if (jj + 1 < NV) {
                acc[(jj + 1) & 3] = fma(m2.y, x2.y, acc[(jj + 1) & 3]);
                acc[4 + ((jj + 1) & 3)] = fma(k2.y, r2.y, acc[4 + ((jj + 1) & 3)]);
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < NV2; ++j) {
              acc[j & 3] = fma(sf[BlobLayout::Mt + j * NV2 + kc], ws->xi1[ch][xpad(j)], acc[j & 3]);
              acc[4 + (j & 3)] = fma(sf[BlobLayout::K11t + j * NV2 + kc], ws->rhs[ch][xpad(j)], acc[4 + (j & 3)]);
            }
          }
          const double v = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
          vnew[c] = (k < NV2) ? v : 0.0;
        }
        __syncwarp();   // every lane has read xi1 and rhs
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c >= nown) break;
        const int ch = chb + c;
        if (it >= 0) xi[c] = vnew[c];
        {
          // position (deviation from the boundary line), Dm c and Dm^2 c in fp64
          // (Dm tridiagonal: (Dm c)_k = (-k c_{k-1} + (2k - n) c_k + (n - k) c_{k+1}) / T,
          // n = 10; lanes >= 11 hold the copy block and meet zero weights)
          const double d1 = dm_apply(xi[c], dmtab, k);
          const double d2 = dm_apply(d1, dmtab, k);
          // predicated stores (no divergent block): lanes k < 11 the position block,
          // lanes 11..21 the copy block
          const int kp = min(k, NV - 1), kq = min(max(k - NV, 0), NV - 1);
          const float xf = d2f(xi[c] - cref[c]), d1f = d2f(d1), d2ff = d2f(d2), cf = d2f(xi[c]);
          if (k < NV) {
            ws->cpos[kp][ch] = xf;
            ws->cpos[kp][2 + ch] = d1f;
            ws->cdd[kp][ch] = d2ff;
          }
          if (k >= NV && k < NV2) ws->ccs[kq][ch] = cf;
        }
        if (k < NV2) ws->xi1[ch][xpad(k)] = xi[c];
      }
      if (nown == 0 && lp_pending) lampsi_step();   // warps without a channel (T = 4)
      lp_pending = false;
      BMC_TICK(pc, 0);
      team_sync(team, T);
      BMC_TICK(pc, 1);
      // ---- B: heading target --------------------------------------------------
      phase_theta<FM>(Pt, Pt64, ws, lane, q, w, T, it >= 0);
      BMC_TICK(pc, 2);
      team_sync(team, T);
      BMC_TICK(pc, 3);
      // ---- C: xi2 step + lambda_psi (Eq. 19, 23b), every warp, same order ------
      // lanes run row min(k, 10) without divergent branches; lanes >= 11 keep 0
      const int k1 = min(k, NV - 1);
      double pth = 0.0;
#pragma unroll
      for (int ww = 0; ww < T_MAX; ++ww)
        if (ww < T) pth += ws->part_th[ww][k1];
      if (FM && (k1 < 3 || k1 > 7)) pth = 0.0;   // not formed per iteration (see phase_theta)
      if (it >= 0) {
        if (k < NV) ws->rhspw[w][k] = lamp + rho_psi * pth;
        __syncwarp();
        {
          double s4[4] = {ub[2 * NV2 + k1], 0.0, 0.0, 0.0};
          if (FM) {   // Kp11 vanishes outside rows / columns 3..7
#pragma unroll
            for (int j = 3; j < 8; ++j) s4[j & 3] = fma(sf[BlobLayout::Kp11t + j * NV + k1], ws->rhspw[w][j], s4[j & 3]);
          } else {
#pragma unroll
            for (int j = 0; j < NV; ++j) s4[j & 3] = fma(sf[BlobLayout::Kp11t + j * NV + k1], ws->rhspw[w][j], s4[j & 3]);
          }
          const double v = (s4[0] + s4[1]) + (s4[2] + s4[3]);
          xi2r = (k < NV) ? v : 0.0;
          if (k < NV) {
            ws->xi2w[w][k] = xi2r;
            ws->cf4[w][k] = d2f(xi2r);
          }
        }
        pth_prev = pth;        // the lambda_psi step runs in the next phase A
        lp_pending = true;
      }
      __syncwarp();
      BMC_TICK(pc, 4);
      // ---- D: projections (own rounds) + contraction (owned channels) ---------
      const bool want_res = trace ? (it >= 0) : (it == K - 1);
      // residual terms only where they are reported: a compile-time flag keeps the
      // hot (RES = false) copy free of the per-round re-evaluation of a runtime flag
      if (want_res)
        phase_project<M, true, ELLK>(pa, r, ws, lane, w, T, team, hreg, clkreg, pc);
      else
        phase_project<M, false, ELLK>(pa, r, ws, lane, w, T, team, hreg, clkreg, pc);
      __syncwarp();
      BMC_TICK(pc, 7);
      if (want_res) {   // every warp's D1 is done (barrier inside phase_project)
        r1sq = 0.f;
        rpsq = 0.f;
        for (int ww = 0; ww < T; ++ww) {
          r1sq += ws->part_res[ww][0];
          rpsq += ws->part_res[ww][1];
        }
      }
      if (it >= 0) {
        // ---- E: multipliers (Eq. 23a with F^T, G3) -------------------------------
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c >= nown) break;
          if (k < NV2) lam[c] -= rho * hreg[c];
        }
        if (trace && w == 0 && lane == 0 && active) a.res_trace[l * K + it] = sqrtf(fmaxf(r1sq, 0.f));
      }
      BMC_TICK(pc, 8);
    }
#ifdef BMC_PROFILE
    if (lane == 0 && a.prof)
      for (int i = 0; i < PROF_SLOTS; ++i)   // logical order (team, rank): the host analysis groups by it
        a.prof[((long long)blockIdx.x * wpc + team * T + w) * PROF_SLOTS + i] = pc.acc[i];
#endif
    __syncwarp();
    BMC_STAMP(7);   // thread 0's team left the iteration loop
    if (lp_pending) lampsi_step();   // the last iteration's lambda_psi step
    if constexpr (FM) {   // the boundary components' theta terms, contracted once
      theta_sum_boundary(Pt64, ws, lane, q, w, T);
      team_sync(team, T);
      if (k < 3 || (k > 7 && k < NV)) {
        double s = 0.0;
#pragma unroll
        for (int ww = 0; ww < T_MAX; ++ww)
          if (ww < T) s += ws->part_th[ww][k];
        lamp += rho_psi * s;
      }
    }
    // ---- outputs ----------------------------------------------------------------
    if (active) {
      float* co = a.coeffs + l * 5 * NV;
      float* lo = a.lambda_out ? a.lambda_out + l * 5 * NV : nullptr;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c >= nown) break;
        const int ch = chb + c;
        if (k < NV2) {
          co[ch * NV2 + k] = (float)xi[c];
          if (lo) lo[ch * NV2 + k] = (float)lam[c];
        }
      }
      if (w == 0) {
        if (k < NV) {
          co[2 * NV2 + k] = (float)xi2r;
          if (lo) lo[2 * NV2 + k] = (float)lamp;
        }
        double jpart = 0.0;
        if (k < NV) {   // J = sum_ch c^T (Pdd^T Pdd) c, fp64 (Eq. 1a, G17)
          double gx = 0.0, gy = 0.0, gp = 0.0;
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            const double gg = sf[BlobLayout::Gdd + j * NV + k];
            gx = fma(gg, ws->xi1[0][j], gx);
            gy = fma(gg, ws->xi1[1][j], gy);
            gp = fma(gg, ws->xi2w[0][j], gp);
          }
          jpart = gx * ws->xi1[0][k] + gy * ws->xi1[1][k] + gp * xi2r;
        }
        const double J = warp_sum(jpart);
        if (lane == 0) {
          const float r1 = sqrtf(fmaxf(r1sq, 0.f)), rp = sqrtf(rpsq);
          a.residual[2 * l] = r1;
          a.residual[2 * l + 1] = rp;
          a.cost[l] = (float)J;
          // packed argmin key (G17): infeasible << 62 | fp32 bits(value) << 30 | index
          unsigned long long infeasible = !((double)r1 <= a.res_tol);
          const double v = infeasible ? (double)r1 : J;
          const float vf = __double2float_rn(v);
          unsigned bits;
          if (!isfinite(v) || !isfinite(vf) || !isfinite(J) || !isfinite(r1)) {
            infeasible = 1;
            bits = 0x7F800000u;
          } else {
            bits = __float_as_uint(vf > 0.f ? vf : 0.f);
          }
          const unsigned long long gidx = (unsigned long long)(a.index_base + l) & ((1ull << 30) - 1);
          const unsigned long long key = (infeasible << 62) | ((unsigned long long)bits << 30) | gidx;
          atomicMin(a.ws_key, key);
          __threadfence();
        }
      }
    }
  }
  // ---- grid-wide argmin: the last CTA publishes and resets the workspace ----
  __syncthreads();
  BMC_STAMP(2);   // every team done (outputs written)
  if (tid == 0) {
    __threadfence();
    const unsigned ticket = atomicAdd(a.ws_count, 1u);
    if (ticket == gridDim.x - 1) {
      __threadfence();
      const unsigned long long key = atomicExch(a.ws_key, ~0ull);
      a.best[0] = (long long)(key & ((1ull << 30) - 1));
      a.best[1] = (long long)key;
      atomicExch(a.ws_count, 0u);
    }
  }
  BMC_STAMP(3);   // CTA exit
}

}  // namespace

size_t kernel_smem_bytes(int QPx, int n, int ipc, int team);

// Launch of one (M, team size) kernel variant.
template <int M, int TT, bool ELLK, bool BD, bool FM>
cudaError_t launch_am_mt(const KernelArgs& a, int ipc, cudaStream_t s) {
  // the shared-memory opt-in is per device: one bit per device ordinal (set on
  // the current device, which bmc_solve made params.device); racing threads
  // both set the attribute, which is idempotent
  static std::atomic<unsigned long long> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const unsigned long long bit = 1ull << (dev & 63);
  if (dev >= 64 || !(attr_done.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(bmc_am_kernel<M, TT, ELLK, BD, FM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    attr_done.fetch_or(bit, std::memory_order_release);
#ifdef BMC_PROFILE
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, bmc_am_kernel<M, TT, ELLK, BD, FM>) == cudaSuccess)
      fprintf(stderr, "[bmc prof] kernel<%d,%d>: %d regs, max %d threads/block, %zu B local\n", M, TT, fa.numRegs,
              fa.maxThreadsPerBlock, fa.localSizeBytes);
#endif
  }
  const size_t smem = smem_bytes(a.n, ipc, TT);
  const unsigned grid = (unsigned)((a.B + ipc - 1) / ipc);
  bmc_am_kernel<M, TT, ELLK, BD, FM><<<grid, 32 * TT * ipc, smem, s>>>(a);
  return cudaGetLastError();
}

template <int M, int TT, bool FM>
cudaError_t launch_am_f(const KernelArgs& a, int ipc, cudaStream_t s) {
  if (a.blockdiag)
    return a.alpha_rule ? launch_am_mt<M, TT, true, true, FM>(a, ipc, s) : launch_am_mt<M, TT, false, true, FM>(a, ipc, s);
  return a.alpha_rule ? launch_am_mt<M, TT, true, false, FM>(a, ipc, s) : launch_am_mt<M, TT, false, false, FM>(a, ipc, s);
}

// FM (the full boundary set) for teams of 2 and 4: the per-sample theta sums need
// shared memory that the one-warp-per-instance launches (large batches) do not have
template <int M, int TT>
cudaError_t launch_am_t(const KernelArgs& a, int ipc, cudaStream_t s) {
  if (TT >= 2 && a.nb == NB_MAX) return launch_am_f<M, TT, TT >= 2>(a, ipc, s);
  return launch_am_f<M, TT, false>(a, ipc, s);
}

// One translation unit per circle count M (bmc_kernel_m<M>.cu) instantiates
// this; bmc_launch.cu dispatches on m.  Team sizes 1, 2, 4.
template <int M>
cudaError_t launch_am_m(const KernelArgs& a, int ipc, cudaStream_t s) {
  switch (a.team) {
    case 1: return launch_am_t<M, 1>(a, ipc, s);
    case 2: return launch_am_t<M, 2>(a, ipc, s);
    case 4: return launch_am_t<M, 4>(a, ipc, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bmc
