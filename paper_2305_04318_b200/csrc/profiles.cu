// Profile log-likelihoods over the K×M grid of evaluated points (SURVEY §8(f)
// NEXT-2; paper §3.4-3.6), from the Table-1 summaries that
// lik_eval_batch_device_ex exports (ssqYX, log|V|, status).
//
//  β_a profile: with β_a fixed at b, β_{−a} and σ² profiled out,
//    q(b) = Q0(b) − (g0 − b g1)ᵀ H⁻¹ (g0 − b g1)
//         = A0 − 2b A1 + b² A2,
//    A0 = y'ᵀV⁻¹y' − g0ᵀH⁻¹g0,  A1 = (XᵀV⁻¹y')_a − g1ᵀH⁻¹g0,
//    A2 = (XᵀV⁻¹X)_aa − g1ᵀH⁻¹g1,  H = (XᵀV⁻¹X)_[−a,−a], g0 = (XᵀV⁻¹y')_[−a],
//    g1 = (XᵀV⁻¹X)_[−a,a];  ℓ(b) = −½[n log(q/n) + log|V| + n log 2π + n] + (λ−1)S,
//    ℓ_p(β_a = b) = max over (k, m)                                (Eq. profilebetai)
//  σ profile: ℓ(σ) = −½[q/σ² + n log σ² + log|V| + n log 2π] + (λ−1)S
//    with q = ssqResidual, maximised over (k, m)                   (Eq. profileSigma)
//  λ profile: max over k of ℓ_p(ω_k, λ_m).
//
// coef_kernel: one thread per (k, a), a ≤ p (a = p: the full β̂ residual q).
// max kernels: one block per grid value, a fixed-order max reduction (exact).
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

// w = L⁻¹ v (forward substitution), returns ‖w‖² = vᵀ(LLᵀ)⁻¹v
__device__ double quad_small(const double* L, int m, int ld, const double* v, double* w) {
  double s2 = 0.0;
  for (int i = 0; i < m; ++i) {
    double s = v[i];
    for (int k = 0; k < i; ++k) s -= L[i * ld + k] * w[k];
    w[i] = s / L[i * ld + i];
    s2 += w[i] * w[i];
  }
  return s2;
}

__global__ void coef_kernel(int p, int K, int M, const double* __restrict__ ssqYX,
                            const int* __restrict__ status, double* __restrict__ coefs,
                            double* __restrict__ qfull) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= K * (p + 1)) return;
  const int k = idx / (p + 1), a = idx % (p + 1);
  const int r = M + p;
  const double* C = ssqYX + (size_t)k * r * r;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  double H[PMAX * PMAX], g0[PMAX], g1[PMAX], w[PMAX], w1[PMAX];
  // H = XᵀV⁻¹X without row/column a (a = p: the full matrix)
  int ii = 0;
  for (int i = 0; i < p; ++i) {
    if (i == a) continue;
    int jj = 0;
    for (int j = 0; j < p; ++j) {
      if (j == a) continue;
      H[ii * PMAX + jj] = C[(size_t)(M + i) * r + (M + j)];
      ++jj;
    }
    ++ii;
  }
  const int pm = ii;
  const bool ok = status[k] == 0 && (pm == 0 || chol_small(H, pm, PMAX) == 0);
  double t11 = 0.0;
  if (ok && a < p) {
    ii = 0;
    for (int i = 0; i < p; ++i)
      if (i != a) g1[ii++] = C[(size_t)(M + i) * r + (M + a)];
    t11 = pm ? quad_small(H, pm, PMAX, g1, w1) : 0.0;
  }
  for (int m = 0; m < M; ++m) {
    ii = 0;
    for (int i = 0; i < p; ++i)
      if (i != a) g0[ii++] = C[(size_t)(M + i) * r + m];
    const double yy = C[(size_t)m * r + m];
    if (a == p) {
      qfull[(size_t)k * M + m] = ok ? yy - (pm ? quad_small(H, pm, PMAX, g0, w) : 0.0) : nan;
    } else {
      double* o = coefs + (((size_t)k * p + a) * M + m) * 3;
      if (!ok) {
        o[0] = o[1] = o[2] = nan;
        continue;
      }
      const double t00 = pm ? quad_small(H, pm, PMAX, g0, w) : 0.0;
      double t01 = 0.0;
      for (int i = 0; i < pm; ++i) t01 += w[i] * w1[i];  // g0ᵀH⁻¹g1 = (L⁻¹g0)·(L⁻¹g1)
      o[0] = yy - t00;
      o[1] = C[(size_t)(M + a) * r + m] - t01;
      o[2] = C[(size_t)(M + a) * r + (M + a)] - t11;
    }
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

// grid = (G, p): ℓ_p(β_a = beta_grid[a·G + g])
__global__ void __launch_bounds__(256) beta_max_kernel(int n, int p, int K, int M, int G,
                                                       const double* __restrict__ coefs,
                                                       const double* __restrict__ logdetV,
                                                       const int* __restrict__ status,
                                                       const double* __restrict__ lambdas,
                                                       const double* __restrict__ S,
                                                       const double* __restrict__ beta_grid,
                                                       double* __restrict__ out) {
  __shared__ double red[256];
  const int g = blockIdx.x, a = blockIdx.y;
  const double b = beta_grid[(size_t)a * G + g];
  const double nd = (double)n, c0 = nd * 1.8378770664093454836 + nd, Sv = *S;
  double best = -INFINITY;
  for (int e = threadIdx.x; e < K * M; e += blockDim.x) {
    const int k = e / M, m = e % M;
    if (status[k] != 0) continue;
    const double* o = coefs + (((size_t)k * p + a) * M + m) * 3;
    const double q = o[0] - 2.0 * b * o[1] + b * b * o[2];
    const double l = -0.5 * (nd * log(q / nd) + logdetV[k] + c0) + (lambdas[m] - 1.0) * Sv;
    best = fmax(best, l);
  }
  best = block_max(best, red);
  if (threadIdx.x == 0) out[(size_t)a * G + g] = best;
}

// grid = Sg + M: blocks t < Sg give ℓ_p(σ_t); blocks Sg + m give ℓ_p(λ_m)
__global__ void __launch_bounds__(256) sigma_lambda_kernel(int n, int K, int M, int Sg,
                                                           const double* __restrict__ qfull,
                                                           const double* __restrict__ logdetV,
                                                           const int* __restrict__ status,
                                                           const double* __restrict__ lambdas,
                                                           const double* __restrict__ S,
                                                           const double* __restrict__ sigma_grid,
                                                           double* __restrict__ out_sigma,
                                                           double* __restrict__ out_lambda) {
  __shared__ double red[256];
  const int t = blockIdx.x;
  const double nd = (double)n, ln2pi = 1.8378770664093454836, Sv = *S;
  double best = -INFINITY;
  if (t < Sg) {
    const double s2 = sigma_grid[t] * sigma_grid[t];
    for (int e = threadIdx.x; e < K * M; e += blockDim.x) {
      const int k = e / M, m = e % M;
      if (status[k] != 0) continue;
      const double l = -0.5 * (qfull[e] / s2 + nd * log(s2) + logdetV[k] + nd * ln2pi) +
                       (lambdas[m] - 1.0) * Sv;
      best = fmax(best, l);
    }
    best = block_max(best, red);
    if (threadIdx.x == 0) out_sigma[t] = best;
  } else {
    const int m = t - Sg;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      if (status[k] != 0) continue;
      const double q = qfull[(size_t)k * M + m];
      const double l = -0.5 * (nd * log(q / nd) + logdetV[k] + nd * ln2pi + nd) + (lambdas[m] - 1.0) * Sv;
      best = fmax(best, l);
    }
    best = block_max(best, red);
    if (threadIdx.x == 0) out_lambda[m] = best;
  }
}

}  // namespace

cudaError_t launch_profiles(int n, int p, int K, int M, const double* y, const double* ssqYX,
                            const double* logdetV, const int* status, const double* lambdas,
                            int G, const double* beta_grid, double* prof_beta, int Sg,
                            const double* sigma_grid, double* prof_sigma, double* prof_lambda,
                            double* coefs, double* qfull, double* S, cudaStream_t st) {
  sumlog_kernel<<<1, 256, 0, st>>>(y, n, S);
  const int nth = K * (p + 1);
  coef_kernel<<<(nth + 127) / 128, 128, 0, st>>>(p, K, M, ssqYX, status, coefs, qfull);
  if (G > 0) beta_max_kernel<<<dim3(G, p), 256, 0, st>>>(n, p, K, M, G, coefs, logdetV, status,
                                                          lambdas, S, beta_grid, prof_beta);
  sigma_lambda_kernel<<<Sg + M, 256, 0, st>>>(n, K, M, Sg, qfull, logdetV, status, lambdas, S,
                                               sigma_grid, prof_sigma, prof_lambda);
  return cudaGetLastError();
}

}  // namespace lik
