// bmc_api.cpp -- the C-ABI of include/bmc.h: argument validation, the
// context (host constants, per-n device blobs, argmin workspace), device and
// host-buffer solves.  No compute happens here beyond the one-off fp64 setup
// (setup.cpp); every step of the iteration runs in bmc_kernel.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/bmc.h"
#include "bmc_internal.h"

namespace bmc {
cudaError_t launch_am(const KernelArgs& a, int wpc, cudaStream_t s);
size_t kernel_smem_bytes(int QP, int n, int ipc, int team);
}  // namespace bmc

using namespace bmc;

namespace {

thread_local std::string g_err;

int32_t fail(int32_t code, const std::string& msg) {
  g_err = msg;
  return code;
}
int32_t cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? BMC_ENOMEM : BMC_ECUDA;
}

struct DeviceGuard {  // restore the caller's current device
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

struct Blob {
  unsigned char* d = nullptr;   // device constants of one obstacle count
  unsigned char* h = nullptr;   // page-locked host copy (source of the asynchronous upload)
  int nb = 0;
  int blockdiag = 0;
  unsigned long long used = 0;  // LRU tick
  cudaEvent_t ready = nullptr;  // recorded after the upload: solves on other streams wait for it
  cudaStream_t upload_stream = nullptr;
  bool uploaded = false;        // the upload is known complete: no wait needed (and none issued,
                                // so steady-state solves can be captured into a CUDA graph)
};

void free_blob(Blob& b) {
  cudaFree(b.d);
  if (b.h) cudaFreeHost(b.h);
  if (b.ready) cudaEventDestroy(b.ready);
}

constexpr size_t BLOB_CACHE_MAX = 8;   // obstacle counts kept per context

struct HostBuf {  // context-owned device buffers for bmc_solve_host
  void* p = nullptr;
  size_t cap = 0;
};

}  // namespace

int32_t bmc::set_last_error(int32_t code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct bmc_ctx {
  bmc_params p{};
  std::vector<double> r;
  int q = 0, QP = 0, NT = 0;
  std::map<int, Blob> blobs;   // by n_obs, at most BLOB_CACHE_MAX (least recently used evicted)
  unsigned long long tick = 0;
  unsigned long long* ws_key = nullptr;   // argmin workspace of bmc_solve
  unsigned int* ws_count = nullptr;
  unsigned long long* ws_key_h = nullptr; // ... and of bmc_solve_host (its own stream)
  unsigned int* ws_count_h = nullptr;
  cudaStream_t hstream = nullptr;
  HostBuf hb[10];
  std::atomic<int32_t> last_launches{0};
  // host-side state shared by the entry points (blob cache, LRU tick): solves from
  // several threads on one context serialise their launch sequences on `mu`;
  // bmc_solve_host additionally holds `hmu` for its staging buffers and stream
  std::mutex mu, hmu;
};

extern "C" {

int32_t bmc_version(void) { return 102; }

const char* bmc_last_error(void) { return g_err.c_str(); }

int32_t bmc_last_launch_count(const bmc_ctx* ctx) { return ctx ? ctx->last_launches.load() : 0; }

int32_t bmc_sample_init(bmc_ctx* ctx, const bmc_sample_params* sp, float* init, bmc_stream_t stream) {
  if (!ctx) return fail(BMC_EINVAL, "ctx is NULL");
  if (!sp) return fail(BMC_EINVAL, "sample params is NULL");
  if (sp->B < 0) return fail(BMC_EINVAL, "B < 0");
  if (sp->B > 0 && !init) return fail(BMC_EINVAL, "init is NULL");
  if (ctx->p.degree != 10) return fail(BMC_EINVAL, "degree must be 10");
  if (!std::isfinite(sp->sigma_x) || !std::isfinite(sp->sigma_y)) return fail(BMC_EINVAL, "non-finite sigma");
  for (int ch = 0; ch < 2; ++ch)
    if (!std::isfinite(sp->bnd[ch][0]) || !std::isfinite(sp->bnd[ch][3])) return fail(BMC_EINVAL, "non-finite bnd");
  SampleArgs a;
  std::memset(&a, 0, sizeof(a));
  a.init = init;
  a.B = sp->B;
  a.index_base = sp->index_base;
  a.seed = sp->seed;
  a.stream = sp->stream;
  a.x0 = sp->bnd[0][0];
  a.xT = sp->bnd[0][3];
  a.y0 = sp->bnd[1][0];
  a.yT = sp->bnd[1][3];
  a.sigma_x = sp->sigma_x;
  a.sigma_y = sp->sigma_y;
  a.line_first = sp->line_first != 0;
  if (stomp_factor(a.L) != 0) return fail(BMC_ESINGULAR, "STOMP covariance factor");
  DeviceGuard g(ctx->p.device);
  cudaError_t e = launch_stomp(a, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "stomp_kernel launch");
  g_err.clear();
  return BMC_OK;
}

static int32_t validate_params(const bmc_params* p) {
  if (!p) return fail(BMC_EINVAL, "params is NULL");
  if (p->degree != 10) return fail(BMC_EINVAL, "degree must be 10 (n_v = 11)");
  if (p->q < p->degree + 1) return fail(BMC_EINVAL, "q < degree + 1");
  if (p->q > Q_MAX) return fail(BMC_EINVAL, "q > 128");
  if (!(p->T > 0.0) || !std::isfinite(p->T)) return fail(BMC_EINVAL, "T must be > 0");
  if (p->m < 1 || p->m > M_MAX) return fail(BMC_EINVAL, "m must be in [1, 8]");
  if (!p->r) return fail(BMC_EINVAL, "r is NULL");
  for (int i = 0; i < p->m; ++i)
    if (!std::isfinite(p->r[i])) return fail(BMC_EINVAL, "r has a non-finite entry");
  if (!(p->v_max > 0.0) || !(p->a_max > 0.0)) return fail(BMC_EINVAL, "v_max and a_max must be > 0");
  if (!(p->rho > 0.0) || !(p->rho_psi > 0.0)) return fail(BMC_EINVAL, "rho and rho_psi must be > 0");
  if (!(p->w_copy >= 0.0)) return fail(BMC_EINVAL, "w_copy must be >= 0");
  if (p->boundary_mask & ~0x3Fu) return fail(BMC_EINVAL, "boundary_mask has bits above 0x3F");
  if (p->alpha_rule != 0 && p->alpha_rule != 1) return fail(BMC_EINVAL, "alpha_rule must be 0 or 1");
  if (std::isnan(p->res_tol)) return fail(BMC_EINVAL, "res_tol is NaN");
  return BMC_OK;
}

static SetupParams setup_params(const bmc_ctx* c) {
  SetupParams s;
  s.q = c->p.q;
  s.T = c->p.T;
  s.m = c->p.m;
  s.r = c->r.data();
  s.rho = c->p.rho;
  s.rho_psi = c->p.rho_psi;
  s.w_copy = c->p.w_copy;
  s.mask = c->p.boundary_mask;
  return s;
}

int32_t bmc_setup(const bmc_params* params, bmc_ctx** out) {
  if (!out) return fail(BMC_EINVAL, "out is NULL");
  *out = nullptr;
  int32_t rc = validate_params(params);
  if (rc != BMC_OK) return rc;
  // the boundary rows and the KKT with one obstacle are checked now; the KKT of
  // a given n is checked when that n is first solved (with no obstacle and no
  // position row among the boundary rows it is singular: a constant shift of x
  // changes nothing the cost or the constraints see)
  bmc_ctx* c = new (std::nothrow) bmc_ctx();
  if (!c) return fail(BMC_ENOMEM, "host allocation failed");
  c->p = *params;
  c->r.assign(params->r, params->r + params->m);
  c->p.r = c->r.data();
  c->q = params->q;
  c->QP = Q_MAX;   // fixed sample stride of the shared-memory layout
  c->NT = c->QP / 32;
  {
    HostConsts hc;
    std::string err;
    if (build_consts(setup_params(c), 1, &hc, &err) != 0) {
      delete c;
      return fail(BMC_ESINGULAR, err);
    }
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  if (params->device < 0 || params->device >= ndev) {
    delete c;
    return fail(BMC_EINVAL, "device ordinal out of range");
  }
  DeviceGuard g(params->device);
  void* ws = nullptr;
  e = cudaMalloc(&ws, 32);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMalloc(workspace)");
  }
  char* wb = reinterpret_cast<char*>(ws);
  c->ws_key = reinterpret_cast<unsigned long long*>(wb);
  c->ws_count = reinterpret_cast<unsigned int*>(wb + 8);
  c->ws_key_h = reinterpret_cast<unsigned long long*>(wb + 16);
  c->ws_count_h = reinterpret_cast<unsigned int*>(wb + 24);
  if ((e = cudaMemset(c->ws_key, 0xFF, 8)) != cudaSuccess || (e = cudaMemset(c->ws_count, 0, 8)) != cudaSuccess ||
      (e = cudaMemset(c->ws_key_h, 0xFF, 8)) != cudaSuccess || (e = cudaMemset(c->ws_count_h, 0, 8)) != cudaSuccess) {
    bmc_destroy(c);
    return cuda_fail(e, "cudaMemset(workspace)");
  }
  *out = c;
  g_err.clear();
  return BMC_OK;
}

void bmc_destroy(bmc_ctx* c) {
  if (!c) return;
  DeviceGuard g(c->p.device);
  for (auto& kv : c->blobs) free_blob(kv.second);
  if (c->ws_key) cudaFree(c->ws_key);
  for (auto& b : c->hb) cudaFree(b.p);
  if (c->hstream) cudaStreamDestroy(c->hstream);
  delete c;
}

// Constants for obstacle count n: built on the host (fp64, setup.cpp) the first
// time n is seen and uploaded asynchronously on the solve's stream from a
// page-locked copy the context keeps.  At most BLOB_CACHE_MAX counts are kept;
// evicting the least recently used one synchronises the device first (a solve
// on another stream may still read it), which only happens when more than
// BLOB_CACHE_MAX distinct counts are in use.
static int32_t get_blob(bmc_ctx* c, int n, cudaStream_t stream, Blob** out) {
  auto it = c->blobs.find(n);
  if (it != c->blobs.end()) {
    it->second.used = ++c->tick;
    *out = &it->second;
    return BMC_OK;
  }
  HostConsts hc;
  std::string err;
  if (build_consts(setup_params(c), n, &hc, &err) != 0) return fail(BMC_ESINGULAR, err);
  cudaError_t e;
  if (c->blobs.size() >= BLOB_CACHE_MAX) {
    auto lru = c->blobs.begin();
    for (auto jt = c->blobs.begin(); jt != c->blobs.end(); ++jt)
      if (jt->second.used < lru->second.used) lru = jt;
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize(blob eviction)");
    free_blob(lru->second);
    c->blobs.erase(lru);
  }
  Blob b;
  b.nb = hc.nb;
  b.blockdiag = hc.blockdiag;
  b.used = ++c->tick;
  const size_t bytes = BlobLayout::bytes(hc.QP);
  if ((e = cudaHostAlloc(reinterpret_cast<void**>(&b.h), bytes, cudaHostAllocDefault)) != cudaSuccess)
    return cuda_fail(e, "cudaHostAlloc(blob)");
  std::memcpy(b.h, hc.blob_f64, BlobLayout::bytes_f64);
  std::memcpy(b.h + BlobLayout::bytes_f64, hc.pt, BlobLayout::bytes_f32(hc.QP));
  std::memcpy(b.h + BlobLayout::bytes_f64 + BlobLayout::bytes_f32(hc.QP), hc.pt64, BlobLayout::bytes_p64(hc.QP));
  if ((e = cudaMalloc(&b.d, bytes)) != cudaSuccess) {
    cudaFreeHost(b.h);
    return cuda_fail(e, "cudaMalloc(blob)");
  }
  if ((e = cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming)) != cudaSuccess) {
    b.ready = nullptr;
    free_blob(b);
    return cuda_fail(e, "cudaEventCreate(blob)");
  }
  if ((e = cudaMemcpyAsync(b.d, b.h, bytes, cudaMemcpyHostToDevice, stream)) != cudaSuccess ||
      (e = cudaEventRecord(b.ready, stream)) != cudaSuccess) {
    free_blob(b);
    return cuda_fail(e, "cudaMemcpyAsync(blob)");
  }
  b.upload_stream = stream;
  c->blobs[n] = b;
  *out = &c->blobs[n];
  return BMC_OK;
}

static bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

static int32_t validate_problem(const bmc_ctx* c, const bmc_problem* pr, const bmc_result* rs) {
  if (!c) return fail(BMC_EINVAL, "ctx is NULL");
  if (!pr || !rs) return fail(BMC_EINVAL, "problem or result is NULL");
  if (pr->B < 1) return fail(BMC_EINVAL, "B must be >= 1");
  if (pr->index_base < 0 || pr->B + pr->index_base > (1ll << 30))
    return fail(BMC_EINVAL, "index_base + B must be in [1, 2^30]");
  if (pr->n_obs < 0 || pr->n_obs > N_MAX) return fail(BMC_EINVAL, "n_obs must be in [0, 160]");
  if (pr->iters < 0) return fail(BMC_EINVAL, "iters must be >= 0");
  if (pr->team != 0 && pr->team != 1 && pr->team != 2 && pr->team != 4)
    return fail(BMC_EINVAL, "team must be 0, 1, 2 or 4");
  if (pr->n_obs > 0 && (!pr->obs_xy || !pr->obs_ab)) return fail(BMC_EINVAL, "obs_xy / obs_ab is NULL");
  if (!pr->init) return fail(BMC_EINVAL, "init is NULL");
  if (!rs->coeffs || !rs->residual || !rs->cost || !rs->best)
    return fail(BMC_EINVAL, "coeffs, residual, cost and best are required");
  const void* f32[] = {pr->obs_xy, pr->obs_ab, pr->init, pr->lambda_in, rs->coeffs,
                       rs->lambda_out, rs->residual, rs->cost, rs->res_trace};
  for (const void* p : f32)
    if (p && !aligned(p, 4)) return fail(BMC_EINVAL, "misaligned fp32 pointer");
  if (!aligned(rs->best, 8)) return fail(BMC_EINVAL, "misaligned best pointer");
  for (int ch = 0; ch < 3; ++ch)
    for (int j = 0; j < 6; ++j)
      if (!std::isfinite(pr->bnd[ch][j])) return fail(BMC_EINVAL, "bnd has a non-finite entry");
  return BMC_OK;
}

// Launch shape: `team` warps per instance, `ipc` instances per CTA.
// Occupancy model: <= 16 warps per SM (<= 128 registers per thread); the
// batch is spread so that every SM holds ceil(B / 148) instances, and small
// batches spend the spare warps on teams (one 32-sample round each).
// team_req != 0 fixes the team; BMC_TEAM / BMC_IPC / BMC_WMAX / BMC_WCTA
// override the automatic choice (experiments).
static void launch_shape(const bmc_ctx* c, int64_t B, int32_t team_req, int* ipc_out, int* team_out) {
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->p.device);
  const int rounds = (c->q + 31) / 32;
  int wmax = 16;   // resident warps per SM at the kernel's register budget
  if (const char* s = std::getenv("BMC_WMAX")) wmax = std::max(1, std::min(32, std::atoi(s)));
  // batches beyond one wave of wmax instances per SM: as many CTA waves as
  // needed at wmax, then the fewest instances per CTA that still fit in them
  // (B = 4096: 2 waves of 14 instead of 1.73 waves of 16 -- every wave costs
  // the same time, and fewer warps per SM run each wave faster)
  const int64_t waves = std::max<int64_t>(1, (B + (int64_t)dev_sms * wmax - 1) / ((int64_t)dev_sms * wmax));
  int ipc = (int)std::min<int64_t>(wmax, (B + dev_sms * waves - 1) / (dev_sms * waves));
  int team = std::max(1, std::min(rounds, wmax / std::max(1, ipc)));
  if (team_req == 0) {
    if (const char* s = std::getenv("BMC_TEAM")) team = std::atoi(s);
    if (const char* s = std::getenv("BMC_IPC")) ipc = std::atoi(s);
    if (team < 1 || team > 4) team = 1;
    if (team == 3) team = (ipc * 4 <= wmax) ? 4 : 2;   // kernels exist for teams of 1, 2, 4
  } else {
    team = team_req;
  }
  int wcta = 16;   // warps per CTA (__launch_bounds__(512)); BMC_WCTA: register-capped experiment builds
  if (const char* s = std::getenv("BMC_WCTA")) wcta = std::max(1, std::min(32, std::atoi(s)));
  if (ipc < 1 || ipc * team > wcta) ipc = std::max(1, wcta / team);
  *ipc_out = ipc;
  *team_out = team;
}

int32_t bmc_team_for(const bmc_ctx* c, int64_t B) {
  if (!c || B < 1) return 0;
  DeviceGuard g(c->p.device);
  int ipc = 1, team = 1;
  launch_shape(c, B, 0, &ipc, &team);
  return team;
}

static int32_t solve_impl(bmc_ctx* c, const bmc_problem* pr, const bmc_result* rs, cudaStream_t s,
                          unsigned long long* ws_key, unsigned int* ws_count) {
  std::lock_guard<std::mutex> lock(c->mu);
  Blob* blob = nullptr;
  int32_t rc = get_blob(c, pr->n_obs, s, &blob);
  if (rc != BMC_OK) return rc;
  // the upload may have been issued on another stream (bmc_solve vs bmc_solve_host)
  if (!blob->uploaded) {
    if (blob->upload_stream != s) {
      cudaError_t ew = cudaStreamWaitEvent(s, blob->ready, 0);
      if (ew != cudaSuccess) return cuda_fail(ew, "cudaStreamWaitEvent(blob)");
    }
    if (cudaEventQuery(blob->ready) == cudaSuccess)
      blob->uploaded = true;
    else
      cudaGetLastError();   // cudaErrorNotReady is a status, not an error
  }
  int ipc = 1, team = 1;
  launch_shape(c, pr->B, pr->team, &ipc, &team);
  while (ipc > 1 && kernel_smem_bytes(c->QP, pr->n_obs, ipc, team) > 227 * 1024) --ipc;
  if (kernel_smem_bytes(c->QP, pr->n_obs, ipc, team) > 227 * 1024)
    return fail(BMC_EINVAL, "n_obs * q too large for shared memory");
  const int wpc = ipc;   // launch_am takes instances per CTA
  KernelArgs a;
  std::memset(&a, 0, sizeof(a));
  a.blob = blob->d;
  a.obs_xy = pr->obs_xy;
  a.obs_ab = pr->obs_ab;
  a.init = pr->init;
  a.lambda_in = pr->lambda_in;
  a.coeffs = rs->coeffs;
  a.lambda_out = rs->lambda_out;
  a.residual = rs->residual;
  a.cost = rs->cost;
  a.res_trace = (pr->iters > 0) ? rs->res_trace : nullptr;
  a.best = reinterpret_cast<long long*>(rs->best);
  a.ws_key = ws_key;
  a.ws_count = ws_count;
  a.B = pr->B;
  a.index_base = pr->index_base;
  a.q = c->q;
  a.QP = c->QP;
  a.NT = c->NT;
  a.n = pr->n_obs;
  a.m = c->p.m;
  a.nb = blob->nb;
  a.iters = pr->iters;
  a.team = team;
  a.alpha_rule = c->p.alpha_rule;
  double R1 = 0.0, R2 = 0.0;
  for (int i = 0; i < c->p.m; ++i) {
    a.r[i] = (float)c->r[i];
    R1 += c->r[i];
    R2 += c->r[i] * c->r[i];
  }
  a.nR1 = (float)(pr->n_obs * R1);
  a.nR2p1 = (float)(pr->n_obs * R2 + 1.0);
  a.v_max = (float)c->p.v_max;
  a.a_max = (float)c->p.a_max;
  a.rho = c->p.rho;
  a.rho_psi = c->p.rho_psi;
  a.res_tol = c->p.res_tol;
  int r = 0;
  for (int bit = 0; bit < 6; ++bit) {
    if (!(c->p.boundary_mask & (1u << bit))) continue;
    for (int ch = 0; ch < 3; ++ch) a.b[ch][r] = pr->bnd[ch][bit];
    ++r;
  }
  a.T = c->p.T;
  // reference line for the fp32 deviation frame: start -> goal position when
  // both are constrained, else the start (or the origin)
  const bool has0 = c->p.boundary_mask & 1u, hasT = c->p.boundary_mask & 8u;
  a.ref_x0 = has0 ? pr->bnd[0][0] : (hasT ? pr->bnd[0][3] : 0.0);
  a.ref_y0 = has0 ? pr->bnd[1][0] : (hasT ? pr->bnd[1][3] : 0.0);
  a.ref_dx = (has0 && hasT) ? pr->bnd[0][3] - pr->bnd[0][0] : 0.0;
  a.ref_dy = (has0 && hasT) ? pr->bnd[1][3] - pr->bnd[1][0] : 0.0;
  // development aid: BMC_PROF=1 with a PROFILE=1 build prints per-phase cycles
  const bool prof = std::getenv("BMC_PROF") != nullptr;
  // testing aid: BMC_NOCULL=1 disables the exact culling (results must be bitwise equal)
  if (const char* e = std::getenv("BMC_NOCULL")) a.no_cull = std::atoi(e) != 0;
  a.blockdiag = blob->blockdiag;
  const long long nwarps = ((pr->B + ipc - 1) / ipc) * (long long)ipc * team;
  if (prof && cudaMalloc(&a.prof, sizeof(long long) * 16 * nwarps) == cudaSuccess)
    cudaMemsetAsync(a.prof, 0, sizeof(long long) * 16 * nwarps, s);
  const long long ngrid = (pr->B + ipc - 1) / ipc;
  if (prof && cudaMalloc(&a.prof_t, sizeof(long long) * 8 * ngrid) == cudaSuccess)
    cudaMemsetAsync(a.prof_t, 0, sizeof(long long) * 8 * ngrid, s);
  cudaError_t e = launch_am(a, wpc, s);
  c->last_launches = 1;
  if (e != cudaSuccess) return cuda_fail(e, "bmc_am_kernel launch");
  if (prof && a.prof) {
    std::vector<long long> hp(16 * nwarps);
    cudaStreamSynchronize(s);
    cudaMemcpy(hp.data(), a.prof, sizeof(long long) * hp.size(), cudaMemcpyDeviceToHost);
    cudaFree(a.prof);
    if (a.prof_t) {   // per-CTA wall clock (globaltimer, ns): start spread, prologue, loop, epilogue
      std::vector<long long> ht(8 * ngrid);
      cudaMemcpy(ht.data(), a.prof_t, sizeof(long long) * ht.size(), cudaMemcpyDeviceToHost);
      cudaFree(a.prof_t);
      long long t0 = ht[0], t3 = ht[3], s_last = ht[0];
      double seg[6] = {0, 0, 0, 0, 0, 0};   // start->issued, issued->staged, staged->blob, blob->prologue, loop, epilogue
      for (long long b = 0; b < ngrid; ++b) {
        const long long* h = &ht[8 * b];
        t0 = std::min(t0, h[0]);
        s_last = std::max(s_last, h[0]);
        t3 = std::max(t3, h[3]);
        seg[0] += h[4] - h[0];
        seg[1] += h[5] - h[4];
        seg[2] += h[6] - h[5];
        seg[3] += h[1] - h[6];
        seg[4] += h[7] - h[1];
        seg[5] += h[3] - h[7];
      }
      std::fprintf(stderr, "[bmc prof] CTA wall (us, means): start spread %.2f | staging issued %.2f, staged %.2f, "
                   "blob wait %.2f, setup %.2f | loop (team 0) %.2f | outputs + argmin %.2f | first start -> last exit %.2f\n",
                   (s_last - t0) * 1e-3, seg[0] / ngrid * 1e-3, seg[1] / ngrid * 1e-3, seg[2] / ngrid * 1e-3,
                   seg[3] / ngrid * 1e-3, seg[4] / ngrid * 1e-3, seg[5] / ngrid * 1e-3, (t3 - t0) * 1e-3);
    }
    const char* names[16] = {"A", "bar1", "B", "bar2", "C", "D2mma", "bar3", "D2+", "E", "tested", "D1", "needed",
                             "D1eval", "D1cull", "D1coll", "D1U+mma"};
    for (int role = 0; role < team; ++role) {
      double tot[16] = {0};
      long long cnt = 0;
      for (long long wv = role; wv < nwarps; wv += team, ++cnt)
        for (int i = 0; i < 16; ++i) tot[i] += (double)hp[wv * 16 + i];
      std::fprintf(stderr, "[bmc prof] team=%d ipc=%d warp-role %d cycles/iter:", team, ipc, role);
      for (int i = 0; i < 16; ++i) std::fprintf(stderr, " %s=%.1f", names[i], tot[i] / cnt / (pr->iters + 1));
      std::fprintf(stderr, "\n");
    }
    // per team slot of the CTA (warp ids rise with the slot): loop cycles per iteration
    std::fprintf(stderr, "[bmc prof] loop cycles/iter by team slot:");
    for (int slot = 0; slot < ipc; ++slot) {
      double tot = 0.0;
      long long cnt = 0;
      for (long long wv = (long long)slot * team; wv < nwarps; wv += (long long)ipc * team, ++cnt)
        for (int i = 0; i <= 10; ++i)
          if (i != 9) tot += (double)hp[wv * 16 + i];
      std::fprintf(stderr, " %.0f", tot / cnt / (pr->iters + 1));
    }
    std::fprintf(stderr, "\n");
    // spread over teams (instances): loop cycles of a team = max over its warps
    std::vector<double> tt;
    for (long long t0 = 0; t0 + team <= nwarps; t0 += team) {
      double mx = 0.0;
      for (int wv = 0; wv < team; ++wv) {
        double tot = 0.0;
        for (int i = 0; i <= 10; ++i)
          if (i != 9) tot += (double)hp[(t0 + wv) * 16 + i];
        mx = std::max(mx, tot);
      }
      tt.push_back(mx / (pr->iters + 1));
    }
    if (const char* fn = std::getenv("BMC_PROF_DUMP")) {   // per team (= instance): loop cycles/iter, tested,
      if (FILE* f = std::fopen(fn, "w")) {                 // then per rank: D1 cycles/iter and tested
        for (size_t i = 0; i < tt.size(); ++i) {
          long long tested = 0;
          for (int wv = 0; wv < team; ++wv) tested += hp[(i * team + wv) * 16 + 9];
          std::fprintf(f, "%zu %.1f %lld", i, tt[i], tested);
          for (int wv = 0; wv < team; ++wv)
            std::fprintf(f, " %.1f %lld", (double)hp[(i * team + wv) * 16 + 10] / (pr->iters + 1),
                         hp[(i * team + wv) * 16 + 9]);
          std::fprintf(f, "\n");
        }
        std::fclose(f);
      }
    }
    std::sort(tt.begin(), tt.end());
    double mean = 0.0;
    for (double v : tt) mean += v;
    mean /= std::max<size_t>(1, tt.size());
    std::fprintf(stderr, "[bmc prof] team loop cycles/iter: mean %.0f p10 %.0f p50 %.0f p90 %.0f p99 %.0f max %.0f\n", mean,
                 tt[tt.size() / 10], tt[tt.size() / 2], tt[tt.size() * 9 / 10], tt[tt.size() * 99 / 100], tt.back());
  }
  return BMC_OK;
}

int32_t bmc_solve(bmc_ctx* c, const bmc_problem* pr, const bmc_result* rs, bmc_stream_t stream) {
  int32_t rc = validate_problem(c, pr, rs);
  if (rc != BMC_OK) return rc;
  DeviceGuard g(c->p.device);
  c->last_launches = 0;
  rc = solve_impl(c, pr, rs, reinterpret_cast<cudaStream_t>(stream), c->ws_key, c->ws_count);
  if (rc == BMC_OK) g_err.clear();
  return rc;
}

static int32_t ensure(bmc_ctx* c, int slot, size_t bytes, void** out) {
  HostBuf& b = c->hb[slot];
  if (b.cap < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    cudaError_t e = cudaMalloc(&b.p, bytes < 256 ? 256 : bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(host-solve buffer)");
    b.cap = bytes < 256 ? 256 : bytes;
  }
  *out = b.p;
  return BMC_OK;
}

int32_t bmc_solve_host(bmc_ctx* c, const bmc_problem* ph, const bmc_result* rh) {
  int32_t rc = validate_problem(c, ph, rh);
  if (rc != BMC_OK) return rc;
  std::lock_guard<std::mutex> hlock(c->hmu);
  DeviceGuard g(c->p.device);
  c->last_launches = 0;
  cudaError_t e;
  if (!c->hstream && (e = cudaStreamCreateWithFlags(&c->hstream, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_fail(e, "cudaStreamCreate");
  const size_t B = (size_t)ph->B, n = (size_t)ph->n_obs, q = (size_t)c->q, K = (size_t)ph->iters;
  const size_t sz[10] = {n * 2 * q * 4, n * 2 * 4, B * 33 * 4, B * 55 * 4, B * 55 * 4,
                         B * 55 * 4, B * 2 * 4, B * 4, B * (K ? K : 1) * 4, 16};
  void* d[10];
  for (int i = 0; i < 10; ++i)
    if ((rc = ensure(c, i, sz[i], &d[i])) != BMC_OK) return rc;
  // page-locked host arrays are used in place (zero-copy; the kernel reads init /
  // lambda_in once per instance and writes each output once); the rest is staged
  auto mapped = [](const void* hp) -> void* {
    if (!hp) return nullptr;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, hp) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return (at.type == cudaMemoryTypeHost) ? at.devicePointer : nullptr;
  };
  void* m_init = mapped(ph->init);
  void* m_lam = mapped(ph->lambda_in);
  void* m_co = mapped(rh->coeffs);
  void* m_lo = mapped(rh->lambda_out);
  void* m_res = mapped(rh->residual);
  void* m_cost = mapped(rh->cost);
  void* m_best = mapped(rh->best);
  bmc_problem pd = *ph;
  bmc_result rd;
  pd.obs_xy = n ? (const float*)d[0] : nullptr;
  pd.obs_ab = n ? (const float*)d[1] : nullptr;
  pd.init = m_init ? (const float*)m_init : (const float*)d[2];
  pd.lambda_in = ph->lambda_in ? (m_lam ? (const float*)m_lam : (const float*)d[3]) : nullptr;
  rd.coeffs = m_co ? (float*)m_co : (float*)d[4];
  rd.lambda_out = rh->lambda_out ? (m_lo ? (float*)m_lo : (float*)d[5]) : nullptr;
  rd.residual = m_res ? (float*)m_res : (float*)d[6];
  rd.cost = m_cost ? (float*)m_cost : (float*)d[7];
  rd.res_trace = rh->res_trace ? (float*)d[8] : nullptr;
  rd.best = m_best ? (int64_t*)m_best : (int64_t*)d[9];
  cudaStream_t s = c->hstream;
#define H2D(dst, src, bytes) \
  if ((bytes) && (e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) return cuda_fail(e, "H2D")
#define D2H(dst, src, bytes) \
  if ((bytes) && (e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return cuda_fail(e, "D2H")
  if (n) {
    H2D(d[0], ph->obs_xy, sz[0]);
    H2D(d[1], ph->obs_ab, sz[1]);
  }
  if (!m_init) H2D(d[2], ph->init, sz[2]);
  if (ph->lambda_in && !m_lam) H2D(d[3], ph->lambda_in, sz[3]);
  rc = solve_impl(c, &pd, &rd, s, c->ws_key_h, c->ws_count_h);
  if (rc != BMC_OK) return rc;
  if (!m_co) D2H(rh->coeffs, d[4], sz[4]);
  if (rh->lambda_out && !m_lo) D2H(rh->lambda_out, d[5], sz[5]);
  if (!m_res) D2H(rh->residual, d[6], sz[6]);
  if (!m_cost) D2H(rh->cost, d[7], sz[7]);
  const size_t trace_bytes = rh->res_trace ? B * K * 4 : 0;
  D2H(rh->res_trace, d[8], trace_bytes);
  if (!m_best) D2H(rh->best, d[9], 16);
#undef H2D
#undef D2H
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  g_err.clear();
  return BMC_OK;
}

}  // extern "C"
