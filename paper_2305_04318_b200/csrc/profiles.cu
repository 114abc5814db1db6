// Profile log-likelihoods over the K×M grid of evaluated points (SURVEY §8(f)
// NEXT-2; paper §3.4-3.6), from the Table-1 summaries that
// lik_eval_batch_device_ex exports (ssqYX, log|V|, status).
//
//  β_a profile: with β_a fixed at b, β_{−a} and σ² profiled out, the
//    paper writes q(b) = Q0(b) − (g0 − b g1)ᵀ H₋ₐ⁻¹ (g0 − b g1)   (P:347-351,
//    H₋ₐ = (XᵀV⁻¹X) without row/column a).  That is the minimum over β₋ₐ of the
//    quadratic Q(β) = y'ᵀV⁻¹y' − 2βᵀXᵀV⁻¹y' + βᵀXᵀV⁻¹Xβ at β_a = b, which by the
//    block inverse of H = XᵀV⁻¹X equals
//      q(b) = q̂ + (b − β̂_a)² / (H⁻¹)_aa,   q̂ = Q(β̂),  β̂ = H⁻¹XᵀV⁻¹y',
//    so one factorisation of H per point serves every a (the oracle keeps the
//    paper's per-a deletion; R27).  The form is a sum of non-negative
//    terms (no cancellation).  ℓ(b) = −½[n log(q/n) + log|V| + n log 2π + n] + (λ−1)S,
//    ℓ_p(β_a = b) = max over (k, m)                                (Eq. profilebetai)
//  σ profile: ℓ(σ) = −½[q/σ² + n log σ² + log|V| + n log 2π] + (λ−1)S
//    with q = ssqResidual, maximised over (k, m)                   (Eq. profileSigma)
//  λ profile: max over k of ℓ_p(ω_k, λ_m).
//
// factor_kernel: one thread per k — Cholesky L of H, hinv[a][k] = 1/(H⁻¹)_aa.
// solve_kernel: one thread per (k, m) — q̂ = y'ᵀV⁻¹y' − ‖L⁻¹g‖², β̂ = L⁻ᵀL⁻¹g,
//   stored as qfull[k·M + m], bh[a][k·M + m] (coalesced for the β scan).
// max kernels: blocks per (grid value, slice of the (k, m) range), then a fixed-order
// max over the slices (exact).
#include <algorithm>
#include <cfloat>
#include "lik_internal.cuh"

namespace lik {
namespace {

constexpr int PMAX = 32;

// Cholesky of the m×m SPD matrix in `a` (row-major, stride ld), in place; 0 = ok.
__device__ int chol_small(double* a, int m, int ld) {
  for (int c = 0; c < m; ++c) {
    double d = a[c * ld + c];
    for (int k = 0; k < c; ++k) d -= a[c * ld + k] * a[c * ld + k];
    if (!(d > 0.0)) return 1;
    const double l = sqrt(d);
    a[c * ld + c] = l;
    for (int i = c + 1; i < m; ++i) {
      double s = a[i * ld + c];
      for (int k = 0; k < c; ++k) s -= a[i * ld + k] * a[c * ld + k];
      a[i * ld + c] = s / l;
    }
  }
  return 0;
}

// one thread per point k: L = chol(XᵀV⁻¹X) (p×p, row-major, NaN-filled if the point
// failed or H is not SPD), hinv[a·K + k] = 1/(H⁻¹)_aa with (H⁻¹)_aa = ‖L⁻¹e_a‖²
__global__ void factor_kernel(int p, int K, int M, const double* __restrict__ ssqYX,
                              const int* __restrict__ status, double* __restrict__ Lbuf,
                              double* __restrict__ hinv) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int r = M + p;
  const double* C = ssqYX + (size_t)k * r * r;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  double H[PMAX * PMAX], x[PMAX];
  for (int i = 0; i < p; ++i)
    for (int j = 0; j <= i; ++j) H[i * p + j] = C[(size_t)(M + i) * r + (M + j)];
  // failed points are skipped; a NEG_RESID point only in its failed λ columns (R12,
  // solve_kernel marks them NaN, which every max below ignores)
  const bool ok = (status[k] == 0 || status[k] == 3) && chol_small(H, p, p) == 0;
  double* L = Lbuf + (size_t)k * p * p;
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) L[i * p + j] = ok && j <= i ? H[i * p + j] : (ok ? 0.0 : nan);
  for (int a = 0; a < p; ++a) {
    double s2 = 0.0;
    if (ok) {
      // x = L⁻¹ e_a: zero above row a
      for (int i = a; i < p; ++i) {
        double t = i == a ? 1.0 : 0.0;
        for (int j = a; j < i; ++j) t -= H[i * p + j] * x[j];
        x[i] = t / H[i * p + i];
        s2 += x[i] * x[i];
      }
    }
    hinv[(size_t)a * K + k] = ok ? 1.0 / s2 : nan;
  }
}

// one thread per (k, m): g = XᵀV⁻¹y'_m, w = L⁻¹g, q̂ = y'ᵀV⁻¹y' − ‖w‖² (Step 8),
// β̂ = L⁻ᵀw
__global__ void solve_kernel(int p, int K, int M, const double* __restrict__ ssqYX,
                             const double* __restrict__ Lbuf, double* __restrict__ qfull,
                             double* __restrict__ bh) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K * M) return;
  const int k = e / M, m = e - k * M, r = M + p;
  const size_t KM = (size_t)K * M;
  const double* C = ssqYX + (size_t)k * r * r;
  const double* L = Lbuf + (size_t)k * p * p;
  double w[PMAX];
  double s2 = 0.0;
  for (int i = 0; i < p; ++i) {
    double t = C[(size_t)(M + i) * r + m];
    for (int j = 0; j < i; ++j) t -= L[i * p + j] * w[j];
    w[i] = t / L[i * p + i];
    s2 += w[i] * w[i];
  }
  // Step 8; NaN propagates from a failed point's L; a column whose Step 8 is not
  // resolved (q ≤ 1e-10·y'ᵀV⁻¹y', R12) is NaN too
  const double yy = C[(size_t)m * r + m], qv = yy - s2;
  qfull[e] = qv > 1e-10 * yy ? qv : __longlong_as_double(0x7ff8000000000000LL);
  for (int i = p - 1; i >= 0; --i) {
    double t = w[i];
    for (int j = i + 1; j < p; ++j) t -= L[j * p + i] * w[j];
    w[i] = t / L[i * p + i];
    bh[(size_t)i * KM + e] = w[i];
  }
}

__device__ double block_max(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// S = Σ log y (fixed-order reduction, one block)
__global__ void sumlog_kernel(const double* __restrict__ y, int n, double* __restrict__ S) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) s += log(y[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *S = red[0];
}

// The maxima over the K×M grid are split into NSL slices of (k, m) per output value
// (grid dimension z), each block writing its slice's maximum; finalize_kernel takes
// the max over the slices in a fixed order.  fmax is exact, so the result does not
// depend on the split.
// (K·M ≤ 2³⁰ is checked by the API, so 32-bit indices suffice)
__device__ __forceinline__ void slice_range(int total, int nsl, int sl, int& lo, int& hi) {
  const int per = (total + nsl - 1) / nsl;
  lo = min(total, per * sl);
  hi = min(total, lo + per);
}

// grid = (G, p, NSL): slice sl of ℓ_p(β_a = beta_grid[a·G + g]) → part[(a·G + g)·NSL + sl]
__global__ void __launch_bounds__(256) beta_max_kernel(int n, int p, int K, int M, int G, int nsl,
                                                       const double* __restrict__ qfull,
                                                       const double* __restrict__ bh,
                                                       const double* __restrict__ hinv,
                                                       const double* __restrict__ logdetV,
                                                       const int* __restrict__ status,
                                                       const double* __restrict__ lambdas,
                                                       const double* __restrict__ S,
                                                       const double* __restrict__ beta_grid,
                                                       double* __restrict__ part) {
  __shared__ double red[256];
  const int g = blockIdx.x, a = blockIdx.y, sl = blockIdx.z;
  const double b = beta_grid[(size_t)a * G + g];
  // ℓ = −½(n log(q/n) + log|V| + n log 2π + n) + (λ−1)S, with log(q/n) = log q − log n
  const double nd = (double)n, c0 = nd * (1.8378770664093454836 + 1.0 - log(nd)), Sv = *S;
  const double* bha = bh + (size_t)a * K * M;
  const double* hia = hinv + (size_t)a * K;
  int lo, hi;
  slice_range(K * M, nsl, sl, lo, hi);
  double best = -INFINITY;
  for (int e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    const int k = e / M, m = e - k * M;
    if (status[k] != 0 && status[k] != 3) continue;  // NEG_RESID columns: qfull = NaN
    const double d = b - bha[e];
    const double q = fma(d * d, hia[k], qfull[e]);
    const double l = -0.5 * (nd * log(q) + logdetV[k] + c0) + (lambdas[m] - 1.0) * Sv;
    best = fmax(best, l);
  }
  best = block_max(best, red);
  if (threadIdx.x == 0) part[((size_t)a * G + g) * nsl + sl] = best;
}

// grid = (Sg + M, NSL): blocks t < Sg give slices of ℓ_p(σ_t); blocks Sg + m of ℓ_p(λ_m)
__global__ void __launch_bounds__(256) sigma_lambda_kernel(int n, int K, int M, int Sg, int nsl,
                                                           const double* __restrict__ qfull,
                                                           const double* __restrict__ logdetV,
                                                           const int* __restrict__ status,
                                                           const double* __restrict__ lambdas,
                                                           const double* __restrict__ S,
                                                           const double* __restrict__ sigma_grid,
                                                           double* __restrict__ part) {
  __shared__ double red[256];
  const int t = blockIdx.x, sl = blockIdx.y;
  const double nd = (double)n, ln2pi = 1.8378770664093454836, Sv = *S;
  double best = -INFINITY;
  int lo, hi;
  if (t < Sg) {
    const double s2 = sigma_grid[t] * sigma_grid[t], is2 = 1.0 / s2;
    const double c1 = nd * (log(s2) + ln2pi);
    slice_range(K * M, nsl, sl, lo, hi);
    for (int e = lo + threadIdx.x; e < hi; e += blockDim.x) {
      const int k = e / M, m = e - k * M;
      if (status[k] != 0 && status[k] != 3) continue;
      const double l = -0.5 * (qfull[e] * is2 + c1 + logdetV[k]) + (lambdas[m] - 1.0) * Sv;
      best = fmax(best, l);
    }
  } else {
    const int m = t - Sg;
    const double c0 = nd * (ln2pi + 1.0 - log(nd)), lt = (lambdas[m] - 1.0) * Sv;
    slice_range(K, nsl, sl, lo, hi);
    for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
      if (status[k] != 0 && status[k] != 3) continue;
      const double q = qfull[(size_t)k * M + m];
      const double l = -0.5 * (nd * log(q) + logdetV[k] + c0) + lt;
      best = fmax(best, l);
    }
  }
  best = block_max(best, red);
  if (threadIdx.x == 0) part[(size_t)t * nsl + sl] = best;
}

// out[i] = max over the nsl slices of part[i·nsl + ·] (fixed order)
__global__ void finalize_kernel(const double* __restrict__ part, int count, int nsl,
                                double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double best = -INFINITY;
  for (int sl = 0; sl < nsl; ++sl) best = fmax(best, part[(size_t)i * nsl + sl]);
  out[i] = best;
}

}  // namespace

int profile_slices(long long K, int M) {
  const long long per_thread = 64;  // (k, m) pairs per thread and slice
  return (int)std::max<long long>(1, std::min<long long>(64, (K * M + 256 * per_thread - 1) / (256 * per_thread)));
}

size_t profile_partials(int p, int G, int Sg, int M, int nsl) {
  return ((size_t)p * G + Sg + M) * nsl;
}

size_t profile_scratch(int p, int K, int M, int G, int Sg) {
  const size_t KM = (size_t)K * M;
  return (size_t)K * p * p + (size_t)p * K + KM + (size_t)p * KM + 2 +
         profile_partials(p, G, Sg, M, profile_slices(K, M));
}

cudaError_t launch_profiles(int n, int p, int K, int M, const double* y, const double* ssqYX,
                            const double* logdetV, const int* status, const double* lambdas,
                            int G, const double* beta_grid, double* prof_beta, int Sg,
                            const double* sigma_grid, double* prof_sigma, double* prof_lambda,
                            double* scratch, cudaStream_t st) {
  const int nsl = profile_slices(K, M);
  const size_t KM = (size_t)K * M;
  double* Lbuf = scratch;
  double* hinv = Lbuf + (size_t)K * p * p;
  double* qfull = hinv + (size_t)p * K;
  double* bh = qfull + KM;
  double* S = bh + (size_t)p * KM;
  double* part = S + 2;
  sumlog_kernel<<<1, 256, 0, st>>>(y, n, S);
  factor_kernel<<<(K + 127) / 128, 128, 0, st>>>(p, K, M, ssqYX, status, Lbuf, hinv);
  solve_kernel<<<(int)((KM + 127) / 128), 128, 0, st>>>(p, K, M, ssqYX, Lbuf, qfull, bh);
  double* pb = part;                          // p·G values
  double* ps = part + (size_t)p * G * nsl;    // Sg + M values
  if (G > 0) {
    beta_max_kernel<<<dim3(G, p, nsl), 256, 0, st>>>(n, p, K, M, G, nsl, qfull, bh, hinv, logdetV,
                                                      status, lambdas, S, beta_grid, pb);
    finalize_kernel<<<(p * G + 127) / 128, 128, 0, st>>>(pb, p * G, nsl, prof_beta);
  }
  sigma_lambda_kernel<<<dim3(Sg + M, nsl), 256, 0, st>>>(n, K, M, Sg, nsl, qfull, logdetV, status,
                                                         lambdas, S, sigma_grid, ps);
  if (Sg > 0) finalize_kernel<<<(Sg + 127) / 128, 128, 0, st>>>(ps, Sg, nsl, prof_sigma);
  finalize_kernel<<<(M + 127) / 128, 128, 0, st>>>(ps + (size_t)Sg * nsl, M, nsl, prof_lambda);
  return cudaGetLastError();
}

}  // namespace lik
