// bmc_internal.h -- shared between the host setup (setup.cpp), the C-ABI
// (bmc_api.cpp) and the fused kernel (bmc_kernel.cu).  Product path only.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

#ifdef __CUDACC__
#define BMC_HD __host__ __device__
#else
#define BMC_HD
#endif

namespace bmc {

constexpr int NV = 11;        // Bernstein degree 10 (n_v = 11, G12)
constexpr int NV2 = 2 * NV;   // per-channel xi1 block (pos, copy)
constexpr int NB_MAX = 6;     // boundary rows per channel (G11)
constexpr int M_MAX = 8;      // footprint circles
constexpr int Q_MAX = 128;    // time samples (4 rounds of 32 lanes)
constexpr int N_MAX = 160;    // obstacles staged in shared memory

// Device constant blob, one per obstacle count n (Q_bar = Q + rho F^T F
// depends on n through F^T F).  fp64 part first, then fp32 basis.
// All matrices are stored TRANSPOSED ("[j][k]": element (row k, col j) at
// j*ld + k) so lane k of a warp reads row k of a mat-vec at consecutive
// addresses.
struct BlobLayout {
  // fp64 section (offsets in doubles)
  static constexpr int Mt = 0;                 // [22][22] (rho K11 F^T F)^T
  static constexpr int K11t = Mt + NV2 * NV2;  // [22][22] K11^T
  static constexpr int K12t = K11t + NV2 * NV2;   // [6][22]  K12^T (rows >= nb zero)
  static constexpr int Kp11t = K12t + NB_MAX * NV2;  // [11][11]
  static constexpr int Kp12t = Kp11t + NV * NV;      // [6][11]
  static constexpr int Gppt = Kp12t + NB_MAX * NV;   // [11][11] rho_psi P^T P
  static constexpr int Gdd = Gppt + NV * NV;         // [11][11] Pdd^T Pdd (cost)
  // block-diagonal M and K11 (sum r_i = 0), row-major: row k holds the 11 entries
  // of its own block (columns j0 .. j0 + 10, j0 = 0 or 11) and 3 zeros; the
  // 112-byte stride keeps each quarter-warp of a 16-byte load on distinct banks
  static constexpr int BD_ROW = 14;
  static constexpr int Mb = (Gdd + NV * NV + 1) & ~1;     // [22][BD_ROW]
  static constexpr int Kb = Mb + NV2 * BD_ROW;            // [22][BD_ROW]
  static constexpr int n_doubles_raw = Kb + NV2 * BD_ROW;
  static constexpr int n_doubles = (n_doubles_raw + 1) & ~1;   // 16-byte multiple
  static constexpr size_t bytes_f64 = sizeof(double) * n_doubles;
  // fp32 section: Pt[QP][PT_ROW] = the basis row of sample t (11 values + a zero
  // pad: three 16-byte loads per sample), zero for t >= q (Pdot = P Dm and
  // Pddot = P Dm^2 are applied on the coefficient side, bmc_kernel.cuh dm_apply)
  static constexpr int PT_ROW = 12;
  BMC_HD static size_t bytes_f32(int QP) { return sizeof(float) * PT_ROW * (size_t)QP; }
  // fp64 copy of the same basis for the F^T (F xi - g) and P^T theta contractions,
  // row stride QP + 4 doubles: the 8 rows of an FP64 MMA A-fragment then fall
  // on distinct shared-memory banks
  BMC_HD static int p64_stride(int QP) { return QP + 4; }
  BMC_HD static size_t bytes_p64(int QP) { return sizeof(double) * NV * (size_t)p64_stride(QP); }
  BMC_HD static size_t bytes(int QP) { return bytes_f64 + bytes_f32(QP) + bytes_p64(QP); }
};

// Kernel arguments (passed by value).
struct KernelArgs {
  const unsigned char* blob;   // device constant blob for this n
  const float* obs_xy;         // [n][2][q]
  const float* obs_ab;         // [n][2]
  const float* init;           // [B][3][11]
  const float* lambda_in;      // [B][5][11] or null
  float* coeffs;               // [B][5][11]
  float* lambda_out;           // [B][5][11] or null
  float* residual;             // [B][2]
  float* cost;                 // [B]
  float* res_trace;            // [B][K] or null
  long long* best;             // [2]
  unsigned long long* ws_key;  // argmin workspace (reset by the last CTA)
  unsigned int* ws_count;
  long long B, index_base;
  int q, QP, NT, n, m, nb, iters, alpha_rule;
  int team;                    // warps per instance (1..4); CTA = team * ipc warps
  float r[M_MAX];
  float nR1, nR2p1;            // n sum r_i, n sum r_i^2 + 1 (F^T F closed form)
  float v_max, a_max;
  double rho, rho_psi, res_tol, T;
  double b[3][NB_MAX];         // selected boundary values: x, y, psi
  // boundary line x_ref(t) = ref_x0 + ref_dx t/T (same for y): positions are
  // evaluated in fp32 as deviations from it
  double ref_x0, ref_dx, ref_y0, ref_dy;
  long long* prof;             // [warps][12] phase cycles (PROFILE builds only) or null
  long long* prof_t;           // [grid][4] globaltimer stamps per CTA (PROFILE builds only) or null
  int no_cull;                 // testing aid (BMC_NOCULL): every obstacle tested every round
  int blockdiag;               // M, K11 block diagonal (symmetric footprint, sum r_i = 0)
};

struct SetupParams {
  int q;
  double T;
  int m;
  const double* r;
  double rho, rho_psi, w_copy;
  unsigned mask;
};

// STOMP sampler (bmc_sample.cu; contract in include/bmc.h bmc_sample_init)
struct SampleArgs {
  float* init;                 // [B][3][11]
  long long B, index_base;
  unsigned long long seed, stream;
  double x0, xT, y0, yT;       // segment end points
  double sigma_x, sigma_y;
  double L[5][5];              // STOMP factor (lower), setup.cpp stomp_factor
  int line_first;
};
cudaError_t launch_stomp(const SampleArgs& a, cudaStream_t s);
// L L^T = R^-1 / max diag (R = D^T D on the control points 3..7 of degree 10)
int stomp_factor(double L[5][5]);

// host-side constants for one (params, n)
struct HostConsts {
  int q, QP, nb, n, m;
  int blockdiag = 0;       // sum r_i = 0: M and K11 are block diagonal (c_x | c_c blocks)
  double blob_f64[BlobLayout::n_doubles];
  float* pt = nullptr;     // [11][QP]
  double* pt64 = nullptr;  // [11][p64_stride(QP)]
  ~HostConsts() { delete[] pt; delete[] pt64; }
};

// bmc_api.cpp: set the calling thread's bmc_last_error() message; returns code.
int32_t set_last_error(int32_t code, const std::string& msg);

// setup.cpp: fp64 constants for obstacle count n; 0 or 2 (singular) with *err.
int build_consts(const SetupParams& p, int n, HostConsts* out, std::string* err);

}  // namespace bmc
