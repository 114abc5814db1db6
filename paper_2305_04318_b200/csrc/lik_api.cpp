// C ABI of liblik.so (include/lik.h): validation, workspace, wave scheduling,
// kernel launches and stage timing.  Host code only; every arithmetic step of
// the likelihood runs in the CUDA kernels (matern_build.cu, chol_fused.cu).
#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/lik.h"
#include "lik_internal.cuh"

using lik::PointConst;
using lik::SlotGeom;

struct lik_ctx {
  int device = 0;
  unsigned flags = 0;
  int nsm = 0;
  cudaStream_t own_stream = nullptr;
  std::string err;
  // device workspace (grown on demand)
  double* ws = nullptr;
  size_t ws_bytes = 0;
  PointConst* pc = nullptr;
  size_t pc_cap = 0;
  double* bt = nullptr;
  size_t bt_bytes = 0;
  double* S = nullptr;
  double* table = nullptr;
  size_t table_bytes = 0;
  cudaTextureObject_t table_tex = 0;  // over `table` (the build's texture-path coefficient loads)
  const double* table_tex_ptr = nullptr;
  size_t table_tex_bytes = 0;
  double* coords_p = nullptr;  // sites in Morton order (device)
  size_t coords_p_bytes = 0;
  int* perm = nullptr;         // Morton order (device)
  double* prof_scratch = nullptr;  // profile coefficients (lik_profiles_device)
  size_t prof_scratch_bytes = 0;
  size_t perm_bytes = 0;
  std::vector<int> hperm;
  // host-API staging buffers
  char* io = nullptr;
  size_t io_bytes = 0;
  char* chunk_buf = nullptr;  // per-chunk outputs when M + p > 64
  size_t chunk_bytes = 0;
  int wave_points = 0;
  bool force_fused = std::getenv("LIK_NO_SMALL") != nullptr;  // A/B: keep chol_fused for small n
  // free-memory query of the last call (cudaMemGetInfo costs 0.1-5 ms of host time):
  // a call with the same K and slot size reuses it, so it gets the same wave size
  // and the workspace it already holds
  size_t avail_cache = 0, avail_slot = 0;
  int avail_K = -1;
  // timing
  double stage_ms[LIK_NSTAGES] = {0, 0, 0, 0};
  long long stage_n[LIK_NSTAGES] = {0, 0, 0, 0};
  std::vector<cudaEvent_t> ev;
  // Calls may be enqueued on different streams but share the workspace above: each
  // call's work waits for the previous call's (done_ev, recorded on its stream at
  // its end), so a later call never overwrites buffers an earlier one still reads.
  cudaEvent_t done_ev = nullptr;
  bool done_recorded = false;
};

// A validated, device-resident dataset (lik_dataset_create): the per-call prep
// products, made once, so repeated evaluations need no host work.
struct lik_dataset {
  int device = 0, n = 0, p = 0, M = 0;
  double* coords_p = nullptr;  // sites in Morton order
  double* bt = nullptr;        // Bᵀ rows (r × npad)
  double* S = nullptr;         // Σ log y, d²min, d²max
  double* lambdas = nullptr;   // M
};

namespace {

int fail(lik_ctx* c, int code, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
int fail(lik_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CUDA_TRY(ctx, call)                                                                 \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? LIK_ENOMEM : LIK_ECUDA, "%s: %s", \
                  #call, cudaGetErrorString(e_));                                           \
  } while (0)

template <class T>
int ensure(lik_ctx* c, T** p, size_t* cap, size_t bytes) {
  if (*cap >= bytes && *p) return LIK_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc((void**)p, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(c, LIK_ENOMEM, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
  }
  *cap = bytes;
  return LIK_OK;
}

// Call-level validation on host copies of the (small) dataset.
int validate(lik_ctx* c, int n, int p, const double* coords, const double* y, const double* X,
             int K, int M, const double* lambdas) {
  if (p < 1) return fail(c, LIK_EINVAL, "p = %d < 1", p);
  if (n < p + 2) return fail(c, LIK_EINVAL, "n = %d < p + 2 = %d", n, p + 2);
  if (K < 1) return fail(c, LIK_EINVAL, "K = %d < 1", K);
  if (M < 1) return fail(c, LIK_EINVAL, "M = %d < 1", M);
  if (p > 63) return fail(c, LIK_EINVAL, "p = %d > 63", p);
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(coords[2 * i]) || !std::isfinite(coords[2 * i + 1]))
      return fail(c, LIK_EINVAL, "coords[%d] is not finite", i);
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(y[i])) return fail(c, LIK_EINVAL, "y[%d] is not finite", i);
  for (long i = 0; i < (long)n * p; ++i)
    if (!std::isfinite(X[i])) return fail(c, LIK_EINVAL, "X[%ld][%ld] is not finite", i / p, i % p);
  for (int m = 0; m < M; ++m)
    if (!std::isfinite(lambdas[m])) return fail(c, LIK_EINVAL, "lambdas[%d] is not finite", m);
  for (int i = 0; i < n; ++i)
    if (!(y[i] > 0.0)) return fail(c, LIK_EDOMAIN, "y[%d] = %g <= 0 (Box-Cox needs log y)", i, y[i]);
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) {
    return coords[2 * a] < coords[2 * b] ||
           (coords[2 * a] == coords[2 * b] && coords[2 * a + 1] < coords[2 * b + 1]);
  });
  for (int t = 1; t < n; ++t) {
    const int a = idx[t - 1], b = idx[t];
    if (coords[2 * a] == coords[2 * b] && coords[2 * a + 1] == coords[2 * b + 1])
      return fail(c, LIK_EDOMAIN, "sites %d and %d coincide", std::min(a, b), std::max(a, b));
  }
  // full column rank of X (modified Gram-Schmidt, relative threshold)
  std::vector<double> Q((size_t)n * p);
  std::copy(X, X + (size_t)n * p, Q.begin());
  for (int a = 0; a < p; ++a) {
    double n0 = 0.0;
    for (int i = 0; i < n; ++i) n0 += X[(size_t)i * p + a] * X[(size_t)i * p + a];
    for (int b = 0; b < a; ++b) {
      double d = 0.0;
      for (int i = 0; i < n; ++i) d += Q[(size_t)i * p + a] * Q[(size_t)i * p + b];
      for (int i = 0; i < n; ++i) Q[(size_t)i * p + a] -= d * Q[(size_t)i * p + b];
    }
    double nr = 0.0;
    for (int i = 0; i < n; ++i) nr += Q[(size_t)i * p + a] * Q[(size_t)i * p + a];
    if (n0 == 0.0 || !(nr > 1e-20 * n0))
      return fail(c, LIK_ERANK, "X is not of full column rank (column %d)", a);
    nr = std::sqrt(nr);
    for (int i = 0; i < n; ++i) Q[(size_t)i * p + a] /= nr;
  }
  return LIK_OK;
}

// Site order for the Matérn build: Morton (Z-curve) order of the coordinates, so
// that consecutive sites are spatial neighbours (locality of the per-warp
// Chebyshev octaves).  A symmetric permutation of the sites (with y and X rows)
// leaves V's determinant, the quadratic forms and hence every output unchanged.
void morton_order(int n, const double* coords, std::vector<int>& perm) {
  double xmin = coords[0], xmax = coords[0], ymin = coords[1], ymax = coords[1];
  for (int i = 1; i < n; ++i) {
    xmin = std::min(xmin, coords[2 * i]);
    xmax = std::max(xmax, coords[2 * i]);
    ymin = std::min(ymin, coords[2 * i + 1]);
    ymax = std::max(ymax, coords[2 * i + 1]);
  }
  const double span = std::max(std::max(xmax - xmin, ymax - ymin), 1e-300);
  auto spread = [](uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffULL;
    v = (v | v << 16) & 0x1f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
  };
  std::vector<std::pair<uint64_t, int>> key(n);
  for (int i = 0; i < n; ++i) {
    const uint64_t qx = (uint64_t)((coords[2 * i] - xmin) / span * 2097151.0);
    const uint64_t qy = (uint64_t)((coords[2 * i + 1] - ymin) / span * 2097151.0);
    key[i] = {spread(qx) | (spread(qy) << 1), i};
  }
  std::sort(key.begin(), key.end());
  perm.resize(n);
  for (int i = 0; i < n; ++i) perm[i] = key[i].second;
}

// LIK_HOST_TRACE=1: per-section wall times of the host side of a call (stderr).
struct HostTrace {
  bool on = std::getenv("LIK_HOST_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto u = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[lik host] %-22s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(u - t).count());
    t = u;
  }
};

// The texture object over the table buffer (re-created when the buffer changes).
int table_texture(lik_ctx* c) {
  if (c->table_tex && c->table_tex_ptr == c->table && c->table_tex_bytes == c->table_bytes) return LIK_OK;
  if (c->table_tex) cudaDestroyTextureObject(c->table_tex);
  c->table_tex = 0;
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = c->table;
  rd.res.linear.desc = cudaCreateChannelDesc<int4>();
  rd.res.linear.sizeInBytes = c->table_bytes / 16 * 16;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  CUDA_TRY(c, cudaCreateTextureObject(&c->table_tex, &rd, &td, nullptr));
  c->table_tex_ptr = c->table;
  c->table_tex_bytes = c->table_bytes;
  return LIK_OK;
}

// Order this call's work on `st` after the previous call's (any stream).
cudaError_t after_previous(lik_ctx* c, cudaStream_t st) {
  return c->done_recorded ? cudaStreamWaitEvent(st, c->done_ev, 0) : cudaSuccess;
}
cudaError_t mark_done(lik_ctx* c, cudaStream_t st) {
  const cudaError_t e = cudaEventRecord(c->done_ev, st);
  c->done_recorded = e == cudaSuccess;
  return e;
}

// NVTX range (header-only nvtx3; a no-op unless a tool such as nsys / ncu --nvtx
// injects itself).  Host ranges around the enqueue of each stage: under a tool the
// per-stage kernels are attributed to lik.prep / lik.setup / lik.build / lik.chol.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

cudaEvent_t ev_get(lik_ctx* c, size_t i) {
  while (c->ev.size() <= i) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev.push_back(e);
  }
  return c->ev[i];
}

// The hot path on device buffers (inputs already validated).
struct Extras {
  double *detReml = nullptr, *ssqYX = nullptr, *ssqBetahat = nullptr, *ssqResidual = nullptr,
         *loglik_reml = nullptr, *sigma2hat_reml = nullptr;
};

// The per-call prep products (sites in Morton order, Bᵀ rows, Σ log y and the
// distance range), when a prepared dataset (lik_dataset) supplies them.
struct Prepared {
  const double* coords_p;
  const double* bt;
  const double* S;
};

int run_device(lik_ctx* c, int n, int p, const double* coords, const double* y, const double* X,
               int K, const double* params, int M, const double* lambdas, double* loglik,
               double* betahat, double* sigma2hat, double* logdetV, int* status, cudaStream_t st,
               const double* hcoords, const Extras& ex = Extras(), const Prepared* pre = nullptr) {
  HostTrace tr;
  Nvtx nv_call("lik.eval");
  CUDA_TRY(c, after_previous(c, st));
  const SlotGeom g = lik::make_geom(n, M + p);
  // small augmented matrices take chol_small (build + factor in one kernel, the matrix in
  // shared memory): no workspace slot; a wave is bounded only by the table buffer
  const bool small = !c->force_fused && lik::small_path_fits(n, M + p, p);
  const size_t slot_bytes = small ? (size_t)lik::TABLE_D * sizeof(double) : g.slot_d * sizeof(double);
  // Wave size W (points per table/build/chol launch).  All CTAs of a chol launch
  // start together and the launch ends with its slowest point, so fewer, larger
  // launches lose less to that tail (the CTA scheduler backfills within a launch):
  // by default the fewest waves of at most 16 × (resident CTAs per GPU) points that
  // fit in half the free HBM, each a whole number of CTA rounds except the last.
  // lik_set_wave_points overrides (85 % cap).  The build grid carries the wave in
  // gridDim.y, so W ≤ 65,535.
  auto wave_size = [&](size_t avail) -> int {
    const size_t cap = std::min<size_t>((size_t)(0.85 * (double)avail) / slot_bytes, 65535);
    if (cap < 1) return 0;
    if (c->wave_points > 0) return (int)std::min<size_t>((size_t)std::min(c->wave_points, K), cap);
    // waves are whole multiples of the resident CTAs (res), so only the last
    // launch ends on a partly filled round
    const int res = c->nsm * lik::chol_ctas_per_sm();
    const size_t half = std::max<size_t>(1, (size_t)(0.5 * (double)avail) / slot_bytes);
    int wmax = (int)std::min<size_t>(std::min<size_t>((size_t)16 * res, half), 65535);
    if (wmax >= res) wmax -= wmax % res;
    const int nw = (K + wmax - 1) / wmax;
    int w = (K + nw - 1) / nw;
    if (w > res) w = std::min({wmax, (w + res - 1) / res * res, K});
    return w;
  };
  auto query_avail = [&]() {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t avail = fr + c->ws_bytes;
    c->avail_cache = avail;
    c->avail_slot = slot_bytes;
    c->avail_K = K;
    return avail;
  };
  const bool cached = c->avail_K == K && c->avail_slot == slot_bytes;
  int W = wave_size(cached ? c->avail_cache : query_avail());
  tr.mark("memgetinfo");
  int rc;
  // the free-memory figure may be stale (another allocation since it was cached, or
  // another process): on failure query again and retry with a smaller wave
  for (int attempt = 0;; ++attempt) {
    if (W < 1) {
      c->avail_K = -1;
      return fail(c, LIK_ENOMEM, "one workspace slot (%zu bytes) exceeds free HBM", slot_bytes);
    }
    if (small) {
      W = std::min(K, 65535);
      break;
    }
    if ((rc = ensure(c, &c->ws, &c->ws_bytes, (size_t)W * slot_bytes)) == LIK_OK) break;
    cudaGetLastError();  // clear the allocation error
    if (attempt >= 8) {
      c->avail_K = -1;
      return rc;
    }
    W = std::min(wave_size(query_avail()), W / 2);
  }
  c->err.clear();
  size_t pcb = c->pc_cap * sizeof(PointConst);
  if ((rc = ensure(c, &c->pc, &pcb, (size_t)K * sizeof(PointConst)))) return rc;
  c->pc_cap = pcb / sizeof(PointConst);
  if ((rc = ensure(c, &c->table, &c->table_bytes, (size_t)W * lik::TABLE_D * sizeof(double))))
    return rc;
  if ((rc = table_texture(c))) return rc;
  const bool timing = c->flags & LIK_FLAG_TIMING;
  const int nwaves = (K + W - 1) / W;
  size_t ei = 0;
  const double *coords_p, *bt, *S;
  if (pre) {  // prepared dataset: no host work, no prep launches
    coords_p = pre->coords_p;
    bt = pre->bt;
    S = pre->S;
    if (timing) CUDA_TRY(c, cudaEventRecord(ev_get(c, ei++), st));
  } else {
    if ((rc = ensure(c, &c->bt, &c->bt_bytes, (size_t)g.r * g.nt * lik::TB * sizeof(double) + 64)))
      return rc;
    if (!c->S) CUDA_TRY(c, cudaMalloc(&c->S, 4 * sizeof(double)));  // Σ log y, d²min, d²max
    if ((rc = ensure(c, &c->coords_p, &c->coords_p_bytes, (size_t)n * 2 * sizeof(double)))) return rc;
    tr.mark("ensure");
    const int* dperm = nullptr;
    if (!(c->flags & LIK_FLAG_NATURAL_ORDER)) {
      morton_order(n, hcoords, c->hperm);
      if ((rc = ensure(c, &c->perm, &c->perm_bytes, (size_t)n * sizeof(int)))) return rc;
      CUDA_TRY(c, cudaMemcpyAsync(c->perm, c->hperm.data(), (size_t)n * sizeof(int),
                                  cudaMemcpyHostToDevice, st));
      dperm = c->perm;
    }
    tr.mark("morton+h2d");
    if (timing) CUDA_TRY(c, cudaEventRecord(ev_get(c, ei++), st));
    Nvtx nv("lik.prep");
    CUDA_TRY(c, lik::launch_prep(coords, y, X, lambdas, dperm, n, p, M, g.nt * lik::TB, c->coords_p,
                                 c->bt, c->S, st));
    CUDA_TRY(c, lik::launch_dist_range(c->coords_p, n, c->S + 1, st));
    coords_p = c->coords_p;
    bt = c->bt;
    S = c->S;
  }
  if (timing) CUDA_TRY(c, cudaEventRecord(ev_get(c, ei++), st));
  {
    Nvtx nv("lik.setup");
    CUDA_TRY(c, lik::launch_setup(params, K, c->pc, st));
  }
  if (timing) CUDA_TRY(c, cudaEventRecord(ev_get(c, ei++), st));
  for (int w = 0; w < nwaves; ++w) {
    const int k0 = w * W, kw = std::min(W, K - k0);
    {
      Nvtx nvb("lik.build");
      CUDA_TRY(c, lik::launch_table(lik::cheb_sub_for(g.n), c->pc, k0, kw, c->table, S + 1, st));
      if (!small)
        CUDA_TRY(c, lik::launch_build(lik::cheb_sub_for(g.n), coords_p, g, c->pc, k0, kw, c->table,
                                      c->table_tex, bt, c->ws, st));
    }
    if (timing) CUDA_TRY(c, cudaEventRecord(ev_get(c, ei++), st));
    lik::CholArgs a;
    a.ws = c->ws;
    a.g = g;
    a.M = M;
    a.p = p;
    a.pc = c->pc;
    a.k0 = k0;
    a.lambdas = lambdas;
    a.S = S;
    a.loglik = loglik;
    a.betahat = betahat;
    a.sigma2hat = sigma2hat;
    a.logdetV = logdetV;
    a.status = status;
    a.detReml = ex.detReml;
    a.ssqYX = ex.ssqYX;
    a.ssqBetahat = ex.ssqBetahat;
    a.ssqResidual = ex.ssqResidual;
    a.loglik_reml = ex.loglik_reml;
    a.sigma2hat_reml = ex.sigma2hat_reml;
    Nvtx nvc("lik.chol");
    if (small)
      CUDA_TRY(c, lik::launch_chol_small(a, coords_p, bt, g.nt * lik::TB, c->table, c->table_tex, kw, st));
    else
      CUDA_TRY(c, lik::launch_chol(a, kw, st));
    if (timing) CUDA_TRY(c, cudaEventRecord(ev_get(c, ei++), st));
  }
  tr.mark("launches");
  CUDA_TRY(c, mark_done(c, st));
  if (timing) {
    CUDA_TRY(c, cudaEventSynchronize(c->ev[ei - 1]));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    c->stage_ms[LIK_STAGE_PREP] += ms;
    c->stage_n[LIK_STAGE_PREP] += pre ? 0 : 3;  // prep, dist_init, dist_range
    cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]);
    c->stage_ms[LIK_STAGE_SETUP] += ms;
    c->stage_n[LIK_STAGE_SETUP] += 1;
    for (int w = 0; w < nwaves; ++w) {
      cudaEventElapsedTime(&ms, c->ev[2 + 2 * w], c->ev[3 + 2 * w]);
      c->stage_ms[LIK_STAGE_BUILD] += ms;
      cudaEventElapsedTime(&ms, c->ev[3 + 2 * w], c->ev[4 + 2 * w]);
      c->stage_ms[LIK_STAGE_CHOL] += ms;
    }
    c->stage_n[LIK_STAGE_BUILD] += (small ? 1 : 2) * nwaves;  // table (+ build)
    c->stage_n[LIK_STAGE_CHOL] += nwaves;
  }
  return LIK_OK;
}

// M + p > 64 (more λ than one augmented tile row holds): the λ are evaluated in chunks
// of 64 − p, each a full pass (the factorisation is repeated per chunk — the kernels
// keep r = M + p ≤ 64), into temporaries whose columns are copied into place; log|V| is
// the same for every chunk; a point's status is the first failure, or NEG_RESID if any
// chunk has a failed λ column.
__global__ void merge_status_kernel(int K, const int* __restrict__ chunk, int* __restrict__ status) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int a = status[k], b = chunk[k];
  if (a == LIK_PT_OK && b == LIK_PT_NEG_RESID) status[k] = LIK_PT_NEG_RESID;
}

int run_lambda_chunks(lik_ctx* c, int n, int p, const double* coords, const double* y, const double* X,
                      int K, const double* params, int M, const double* lambdas, double* loglik,
                      double* betahat, double* sigma2hat, double* logdetV, int* status,
                      cudaStream_t st, const double* hcoords) {
  const int Mc = 64 - p;
  const size_t chunk_d = (size_t)K * Mc * (2 + p) + K;
  int rc;
  if ((rc = ensure(c, &c->chunk_buf, &c->chunk_bytes, chunk_d * 8 + (size_t)K * 4 + 64))) return rc;
  double* cll = reinterpret_cast<double*>(c->chunk_buf);
  double* cbh = cll + (size_t)K * Mc;
  double* cs2 = cbh + (size_t)K * Mc * p;
  double* cld = cs2 + (size_t)K * Mc;
  int* cst = reinterpret_cast<int*>(cld + K);
  for (int m0 = 0; m0 < M; m0 += Mc) {
    const int mc = std::min(Mc, M - m0);
    const bool first = m0 == 0;
    if ((rc = run_device(c, n, p, coords, y, X, K, params, mc, lambdas + m0, cll, cbh, cs2,
                         first ? logdetV : cld, first ? status : cst, st, hcoords)))
      return rc;
    CUDA_TRY(c, cudaMemcpy2DAsync(loglik + m0, (size_t)M * 8, cll, (size_t)mc * 8, (size_t)mc * 8, K,
                                  cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(c, cudaMemcpy2DAsync(sigma2hat + m0, (size_t)M * 8, cs2, (size_t)mc * 8, (size_t)mc * 8, K,
                                  cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(c, cudaMemcpy2DAsync(betahat + (size_t)m0 * p, (size_t)M * p * 8, cbh, (size_t)mc * p * 8,
                                  (size_t)mc * p * 8, K, cudaMemcpyDeviceToDevice, st));
    if (!first) {
      merge_status_kernel<<<(K + 255) / 256, 256, 0, st>>>(K, cst, status);
      CUDA_TRY(c, cudaGetLastError());
    }
    CUDA_TRY(c, mark_done(c, st));  // the chunk buffer is reused by the next chunk on st
  }
  return LIK_OK;
}

bool any_null(std::initializer_list<const void*> ps) {
  for (const void* q : ps)
    if (!q) return true;
  return false;
}

}  // namespace

extern "C" {

int lik_create(lik_ctx** out, int cuda_device, unsigned flags) {
  if (!out) return LIK_EINVAL;
  *out = nullptr;
  if (flags & ~(LIK_FLAG_TIMING | LIK_FLAG_NATURAL_ORDER)) return LIK_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev)
    return LIK_ECUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess) return LIK_ECUDA;
  if (prop.major != 10 || prop.minor != 0) return LIK_ECUDA;  // built for sm_100a only
  if (cudaSetDevice(cuda_device) != cudaSuccess) return LIK_ECUDA;
  lik_ctx* c = new lik_ctx;
  c->device = cuda_device;
  c->flags = flags;
  c->nsm = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming) != cudaSuccess) {
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
    return LIK_ECUDA;
  }
  // the table kernel's DCT matrices (device globals of this device; idempotent)
  if (lik::launch_cheb_init(c->own_stream) != cudaSuccess || cudaStreamSynchronize(c->own_stream) != cudaSuccess) {
    cudaEventDestroy(c->done_ev);
    cudaStreamDestroy(c->own_stream);
    delete c;
    return LIK_ECUDA;
  }
  *out = c;
  return LIK_OK;
}

void lik_destroy(lik_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->own_stream) cudaStreamSynchronize(c->own_stream);
  cudaFree(c->ws);
  cudaFree(c->pc);
  cudaFree(c->bt);
  cudaFree(c->S);
  cudaFree(c->table);
  cudaFree(c->coords_p);
  cudaFree(c->perm);
  cudaFree(c->prof_scratch);
  cudaFree(c->io);
  cudaFree(c->chunk_buf);
  for (auto e : c->ev) cudaEventDestroy(e);
  if (c->done_ev) cudaEventDestroy(c->done_ev);
  if (c->table_tex) cudaDestroyTextureObject(c->table_tex);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
}

const char* lik_last_error(const lik_ctx* c) { return c ? c->err.c_str() : "null context"; }

int lik_eval_batch_device(lik_ctx* c, int n, int p, const double* coords, const double* y,
                          const double* X, int K, const double* params, int M,
                          const double* lambdas, double* loglik, double* betahat,
                          double* sigma2hat, double* logdetV, int* status, void* cuda_stream) {
  return lik_eval_batch_device_ex(c, n, p, coords, y, X, K, params, M, lambdas, loglik, betahat,
                                  sigma2hat, logdetV, status, nullptr, nullptr, nullptr, nullptr,
                                  nullptr, nullptr, cuda_stream);
}

int lik_eval_batch_device_ex(lik_ctx* c, int n, int p, const double* coords, const double* y,
                             const double* X, int K, const double* params, int M,
                             const double* lambdas, double* loglik, double* betahat,
                             double* sigma2hat, double* logdetV, int* status, double* detReml,
                             double* ssqYX, double* ssqBetahat, double* ssqResidual,
                             double* loglik_reml, double* sigma2hat_reml, void* cuda_stream) {
  if (!c) return LIK_EINVAL;
  c->err.clear();
  if (any_null({coords, y, X, params, lambdas, loglik, betahat, sigma2hat, logdetV, status}))
    return fail(c, LIK_EINVAL, "NULL pointer argument");
  if (n < 1 || p < 1 || M < 1 || K < 1 || n < p + 2 || p > 63)
    return validate(c, n, p, nullptr, nullptr, nullptr, K, M, nullptr);
  if (M + p > 64 && (detReml || ssqYX || ssqBetahat || ssqResidual || loglik_reml || sigma2hat_reml))
    return fail(c, LIK_ENOTIMPL, "the Table-1 / REML outputs need M + p <= 64 (M + p = %d)", M + p);
  HostTrace tr;
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  std::vector<double> h((size_t)n * (3 + p) + M);
  double* hc = h.data();
  double* hy = hc + 2 * (size_t)n;
  double* hX = hy + n;
  double* hl = hX + (size_t)n * p;
  CUDA_TRY(c, cudaMemcpyAsync(hc, coords, 2 * (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaMemcpyAsync(hy, y, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaMemcpyAsync(hX, X, (size_t)n * p * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaMemcpyAsync(hl, lambdas, (size_t)M * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  tr.mark("d2h+sync");
  int rc = validate(c, n, p, hc, hy, hX, K, M, hl);
  if (rc) return rc;
  tr.mark("validate");
  Extras ex;
  ex.detReml = detReml;
  ex.ssqYX = ssqYX;
  ex.ssqBetahat = ssqBetahat;
  ex.ssqResidual = ssqResidual;
  ex.loglik_reml = loglik_reml;
  ex.sigma2hat_reml = sigma2hat_reml;
  if (M + p > 64)
    return run_lambda_chunks(c, n, p, coords, y, X, K, params, M, lambdas, loglik, betahat,
                             sigma2hat, logdetV, status, st, hc);
  return run_device(c, n, p, coords, y, X, K, params, M, lambdas, loglik, betahat, sigma2hat,
                    logdetV, status, st, hc, ex);
}

int lik_eval_batch(lik_ctx* c, int n, int p, const double* coords, const double* y,
                   const double* X, int K, const double* params, int M, const double* lambdas,
                   double* loglik, double* betahat, double* sigma2hat, double* logdetV,
                   int* status) {
  if (!c) return LIK_EINVAL;
  c->err.clear();
  if (any_null({coords, y, X, params, lambdas, loglik, betahat, sigma2hat, logdetV, status}))
    return fail(c, LIK_EINVAL, "NULL pointer argument");
  if (n < 1 || p < 1 || M < 1 || K < 1 || n < p + 2 || p > 63)
    return validate(c, n, p, nullptr, nullptr, nullptr, K, M, nullptr);
  int rc = validate(c, n, p, coords, y, X, K, M, lambdas);
  if (rc) return rc;
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = c->own_stream;
  const size_t in_d = (size_t)n * (3 + p) + (size_t)K * 5 + M;
  const size_t out_d = (size_t)K * M * (2 + p) + K;
  const size_t bytes = (in_d + out_d) * 8 + (size_t)K * 4 + 256;
  if ((rc = ensure(c, &c->io, &c->io_bytes, bytes))) return rc;
  double* d = reinterpret_cast<double*>(c->io);
  double* dc = d;
  double* dy = dc + 2 * (size_t)n;
  double* dX = dy + n;
  double* dp = dX + (size_t)n * p;
  double* dl = dp + (size_t)K * 5;
  double* dll = dl + M;
  double* dbh = dll + (size_t)K * M;
  double* ds2 = dbh + (size_t)K * M * p;
  double* dld = ds2 + (size_t)K * M;
  int* dst = reinterpret_cast<int*>(dld + K);
  CUDA_TRY(c, cudaMemcpyAsync(dc, coords, 2 * (size_t)n * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(dy, y, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(dX, X, (size_t)n * p * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(dp, params, (size_t)K * 5 * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(dl, lambdas, (size_t)M * 8, cudaMemcpyHostToDevice, st));
  rc = M + p > 64 ? run_lambda_chunks(c, n, p, dc, dy, dX, K, dp, M, dl, dll, dbh, ds2, dld, dst, st, coords)
                  : run_device(c, n, p, dc, dy, dX, K, dp, M, dl, dll, dbh, ds2, dld, dst, st, coords);
  if (rc) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(loglik, dll, (size_t)K * M * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaMemcpyAsync(betahat, dbh, (size_t)K * M * p * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaMemcpyAsync(sigma2hat, ds2, (size_t)K * M * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaMemcpyAsync(logdetV, dld, (size_t)K * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaMemcpyAsync(status, dst, (size_t)K * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  return LIK_OK;
}

int lik_profiles_device(lik_ctx* c, int n, int p, int K, int M, const double* y,
                        const double* ssqYX, const double* logdetV, const int* status,
                        const double* lambdas, int G, const double* beta_grid, double* prof_beta,
                        int Sg, const double* sigma_grid, double* prof_sigma, double* prof_lambda,
                        void* cuda_stream) {
  if (!c) return LIK_EINVAL;
  c->err.clear();
  if (any_null({y, ssqYX, logdetV, status, lambdas, prof_lambda}) ||
      (G > 0 && (!beta_grid || !prof_beta)) || (Sg > 0 && (!sigma_grid || !prof_sigma)))
    return fail(c, LIK_EINVAL, "NULL pointer argument");
  if ((long long)K * M > (1LL << 30) || (long long)K * (p + 1) > (1LL << 30))
    return fail(c, LIK_EINVAL, "K*M=%lld exceeds 2^30", (long long)K * M);
  if (p < 1 || p > 32 || n < p + 2 || K < 1 || M < 1 || G < 0 || Sg < 0)
    return fail(c, LIK_EINVAL, "bad sizes n=%d p=%d K=%d M=%d G=%d Sg=%d (1 <= p <= 32)", n, p, K, M,
                G, Sg);
  CUDA_TRY(c, cudaSetDevice(c->device));
  const size_t need = lik::profile_scratch(p, K, M, G, Sg) * sizeof(double);
  int rc;
  if ((rc = ensure(c, &c->prof_scratch, &c->prof_scratch_bytes, need))) return rc;
  const cudaStream_t st = (cudaStream_t)cuda_stream;
  CUDA_TRY(c, after_previous(c, st));
  CUDA_TRY(c, lik::launch_profiles(n, p, K, M, y, ssqYX, logdetV, status, lambdas, G, beta_grid,
                                   prof_beta, Sg, sigma_grid, prof_sigma, prof_lambda,
                                   c->prof_scratch, st));
  CUDA_TRY(c, mark_done(c, st));
  return LIK_OK;
}

int lik_get_stage_times(lik_ctx* c, double* ms, long long* launches) {
  if (!c || !(c->flags & LIK_FLAG_TIMING) || !ms || !launches) return LIK_EINVAL;
  for (int s = 0; s < LIK_NSTAGES; ++s) {
    ms[s] = c->stage_ms[s];
    launches[s] = c->stage_n[s];
  }
  return LIK_OK;
}

int lik_reset_stage_times(lik_ctx* c) {
  if (!c) return LIK_EINVAL;
  for (int s = 0; s < LIK_NSTAGES; ++s) {
    c->stage_ms[s] = 0.0;
    c->stage_n[s] = 0;
  }
  return LIK_OK;
}

int lik_dataset_create(lik_ctx* c, lik_dataset** out, int n, int p, const double* coords,
                       const double* y, const double* X, int M, const double* lambdas) {
  if (!c) return LIK_EINVAL;
  c->err.clear();
  if (!out) return fail(c, LIK_EINVAL, "NULL pointer argument");
  *out = nullptr;
  if (any_null({coords, y, X, lambdas})) return fail(c, LIK_EINVAL, "NULL pointer argument");
  int rc = validate(c, n, p, coords, y, X, 1, M, lambdas);
  if (rc) return rc;
  if (M + p > 64) return fail(c, LIK_ENOTIMPL, "a prepared dataset needs M + p <= 64 (M + p = %d)", M + p);
  CUDA_TRY(c, cudaSetDevice(c->device));
  const SlotGeom g = lik::make_geom(n, M + p);
  const int npad = g.nt * lik::TB;
  lik_dataset* ds = new lik_dataset;
  ds->device = c->device;
  ds->n = n;
  ds->p = p;
  ds->M = M;
  double *dc = nullptr, *dy = nullptr, *dX = nullptr;
  int* dperm = nullptr;
  auto cleanup = [&]() {
    cudaFree(dc);
    cudaFree(dy);
    cudaFree(dX);
    cudaFree(dperm);
  };
  cudaError_t e = cudaSuccess;
  if ((e = cudaMalloc(&ds->coords_p, (size_t)n * 2 * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&ds->bt, (size_t)g.r * npad * sizeof(double) + 64)) != cudaSuccess ||
      (e = cudaMalloc(&ds->S, 4 * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&ds->lambdas, (size_t)M * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&dc, (size_t)n * 2 * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&dy, (size_t)n * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&dX, (size_t)n * p * sizeof(double))) != cudaSuccess) {
    cleanup();
    lik_dataset_destroy(ds);
    return fail(c, LIK_ENOMEM, "dataset allocation: %s", cudaGetErrorString(e));
  }
  const cudaStream_t st = c->own_stream;
  const int* pperm = nullptr;
  std::vector<int> hperm;
  if (!(c->flags & LIK_FLAG_NATURAL_ORDER)) {
    morton_order(n, coords, hperm);
    if ((e = cudaMalloc(&dperm, (size_t)n * sizeof(int))) == cudaSuccess)
      e = cudaMemcpyAsync(dperm, hperm.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice, st);
    pperm = dperm;
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(dc, coords, (size_t)n * 2 * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dy, y, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dX, X, (size_t)n * p * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ds->lambdas, lambdas, (size_t)M * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = lik::launch_prep(dc, dy, dX, ds->lambdas, pperm, n, p, M, npad, ds->coords_p, ds->bt, ds->S, st);
  if (e == cudaSuccess) e = lik::launch_dist_range(ds->coords_p, n, ds->S + 1, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cleanup();
  if (e != cudaSuccess) {
    lik_dataset_destroy(ds);
    return fail(c, LIK_ECUDA, "dataset preparation: %s", cudaGetErrorString(e));
  }
  *out = ds;
  return LIK_OK;
}

int lik_dataset_eval_device(lik_ctx* c, const lik_dataset* ds, int K, const double* params,
                            double* loglik, double* betahat, double* sigma2hat, double* logdetV,
                            int* status, void* cuda_stream) {
  if (!c) return LIK_EINVAL;
  c->err.clear();
  if (!ds || any_null({params, loglik, betahat, sigma2hat, logdetV, status}))
    return fail(c, LIK_EINVAL, "NULL pointer argument");
  if (K < 1) return fail(c, LIK_EINVAL, "K = %d < 1", K);
  if (ds->device != c->device)
    return fail(c, LIK_EINVAL, "dataset lives on device %d, context on %d", ds->device, c->device);
  CUDA_TRY(c, cudaSetDevice(c->device));
  const Prepared pre{ds->coords_p, ds->bt, ds->S};
  return run_device(c, ds->n, ds->p, nullptr, nullptr, nullptr, K, params, ds->M, ds->lambdas,
                    loglik, betahat, sigma2hat, logdetV, status, (cudaStream_t)cuda_stream, nullptr,
                    Extras(), &pre);
}

void lik_dataset_destroy(lik_dataset* ds) {
  if (!ds) return;
  cudaFree(ds->coords_p);
  cudaFree(ds->bt);
  cudaFree(ds->S);
  cudaFree(ds->lambdas);
  delete ds;
}

int lik_set_wave_points(lik_ctx* c, int pts) {
  if (!c || pts < 0) return LIK_EINVAL;
  c->wave_points = pts;
  return LIK_OK;
}

int lik_debug_build_V(lik_ctx* c, int n, const double* coords, int K, const double* params,
                      double* V) {
  if (!c) return LIK_EINVAL;
  c->err.clear();
  if (any_null({coords, params, V})) return fail(c, LIK_EINVAL, "NULL pointer argument");
  if (n < 1 || K < 1 || K > 65535)
    return fail(c, LIK_EINVAL, "n = %d, K = %d (1 <= K <= 65535 per debug call)", n, K);
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t st = c->own_stream;
  std::vector<double> hc(2 * (size_t)n);
  CUDA_TRY(c, cudaMemcpy(hc.data(), coords, 2 * (size_t)n * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(hc[2 * i]) || !std::isfinite(hc[2 * i + 1]))
      return fail(c, LIK_EINVAL, "coords[%d] is not finite", i);
  const SlotGeom g = lik::make_geom(n, 0);
  int rc;
  if ((rc = ensure(c, &c->ws, &c->ws_bytes, (size_t)K * g.slot_d * sizeof(double)))) return rc;
  size_t pcb = c->pc_cap * sizeof(PointConst);
  if ((rc = ensure(c, &c->pc, &pcb, (size_t)K * sizeof(PointConst)))) return rc;
  c->pc_cap = pcb / sizeof(PointConst);
  if ((rc = ensure(c, &c->table, &c->table_bytes, (size_t)K * lik::TABLE_D * sizeof(double))))
    return rc;
  if ((rc = table_texture(c))) return rc;
  if (!c->S) CUDA_TRY(c, cudaMalloc(&c->S, 4 * sizeof(double)));
  CUDA_TRY(c, after_previous(c, st));
  CUDA_TRY(c, lik::launch_dist_range(coords, n, c->S + 1, st));
  CUDA_TRY(c, lik::launch_setup(params, K, c->pc, st));
  CUDA_TRY(c, lik::launch_table(lik::cheb_sub_for(g.n), c->pc, 0, K, c->table, c->S + 1, st));
  CUDA_TRY(c, lik::launch_build(lik::cheb_sub_for(g.n), coords, g, c->pc, 0, K, c->table, c->table_tex,
                                nullptr, c->ws, st));
  CUDA_TRY(c, lik::launch_unpack_V(g, c->pc, K, c->ws, V, st));
  CUDA_TRY(c, mark_done(c, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  return LIK_OK;
}

}  // extern "C"
