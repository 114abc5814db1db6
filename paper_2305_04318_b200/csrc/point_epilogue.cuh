// Per-point failure outputs and the per-point epilogue (Steps 5-8 of §3.3,
// P:320-323, Eq. 4, Eq. profile, REML Eq. remlpro), shared
// by the factorisation kernels (chol_fused.cu, chol_small.cu).  Product path only.
#pragma once
#include <cfloat>
#include "../../include/lik.h"
#include "lik_internal.cuh"

namespace lik {

// status[k] = code; ℓ_p = −∞, every other output of the point NaN.
__device__ inline void point_failure(const CholArgs& A, int k, int code, int tid, int nthr) {
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  for (int e = tid; e < A.M; e += nthr) {
    A.loglik[(size_t)k * A.M + e] = -INFINITY;
    A.sigma2hat[(size_t)k * A.M + e] = nan;
    if (A.ssqBetahat) A.ssqBetahat[(size_t)k * A.M + e] = nan;
    if (A.ssqResidual) A.ssqResidual[(size_t)k * A.M + e] = nan;
    if (A.loglik_reml) A.loglik_reml[(size_t)k * A.M + e] = -INFINITY;
    if (A.sigma2hat_reml) A.sigma2hat_reml[(size_t)k * A.M + e] = nan;
  }
  if (A.ssqYX) {
    const int r = A.M + A.p;
    for (int e = tid; e < r * r; e += nthr) A.ssqYX[(size_t)k * r * r + e] = nan;
  }
  if (A.detReml && tid == 0) A.detReml[k] = nan;
  for (int e = tid; e < A.M * A.p; e += nthr) A.betahat[(size_t)k * A.M * A.p + e] = nan;
  if (tid == 0) {
    A.logdetV[k] = nan;
    A.status[k] = code;
  }
}

// Steps 5-8 from the cross products ssqYX = BᵀV⁻¹B (Cm: r×r, row-major, stride ldc,
// full), log|V| = logdet (valid in thread lead_tid): XᵀV⁻¹X = QQᵀ (Step 5; Q's
// diagonal is stored as 1/Q_cc; pivot ≤
// p·ε·max diag ⇒ XVX_NOT_PD), c = Q⁻¹XᵀV⁻¹y' (Step 6), ssqBetahat = cᵀc (Step 7),
// q = y'ᵀV⁻¹y' − ssqBetahat (Step 8; R12), β̂ = Q⁻ᵀc, σ̂² = q/n, ℓ_p, and the optional
// Table-1 / REML outputs.  Q: p×p scratch (stride ldq); scratch: NULL or 2·p·min(M, nthr)
// doubles; flag: ≥ 3 ints with flag[2] = 0
// on entry; scal: ≥ 3 doubles.  Called by all nthr threads of the CTA (it contains
// barriers).
__device__ inline void point_epilogue(const CholArgs& A, int k, const double* Cm, int ldc, double* Q,
                                      int ldq, double logdet, int* flag, double* scal, int tid,
                                      int nthr, int lead_tid, double* scratch = nullptr) {
  const int M = A.M, p = A.p, r = M + p, n_sites = A.g.n;
  if (A.ssqYX)
    for (int e = tid; e < r * r; e += nthr) A.ssqYX[(size_t)k * r * r + e] = Cm[(e / r) * ldc + e % r];
  if (tid == lead_tid) {
    double xmax = 0.0;
    for (int a = 0; a < p; ++a) xmax = fmax(xmax, Cm[(M + a) * ldc + (M + a)]);
    const double tolp = p * DBL_EPSILON * xmax;
    int bad = 0;
    for (int c = 0; c < p && !bad; ++c) {
      double d = Cm[(M + c) * ldc + (M + c)];
      for (int kk = 0; kk < c; ++kk) d -= Q[c * ldq + kk] * Q[c * ldq + kk];
      if (!(d > tolp)) {
        bad = 1;
        break;
      }
      // the diagonal holds 1/Q_cc (every later use multiplies by it: no division on the
      // per-λ chains)
      const double rl = rsqrt(d);
      Q[c * ldq + c] = rl;
      for (int i = c + 1; i < p; ++i) {
        double s = Cm[(M + i) * ldc + (M + c)];
        for (int kk = 0; kk < c; ++kk) s -= Q[i * ldq + kk] * Q[c * ldq + kk];
        Q[i * ldq + c] = s * rl;
      }
    }
    flag[1] = bad;
    scal[1] = logdet;  // log|V| = Σ log pivots (Step 2)
    double ldx = 0.0;  // log|XᵀV⁻¹X| = 2 Σ log Q_cc (Step 5, Table 1 detReml)
    if (!bad)
      for (int c = 0; c < p; ++c) ldx -= 2.0 * log(Q[c * ldq + c]);
    scal[2] = ldx;
  }
  __syncthreads();
  if (flag[1]) {
    point_failure(A, k, LIK_PT_XVX_NOT_PD, tid, nthr);
    return;
  }
  const double S = *A.S;
  const double n = (double)n_sites;
  const double ldV = scal[1], ldx = scal[2];
  const double ln2pi = 1.8378770664093454836;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  for (int m = tid; m < M; m += nthr) {
    // c and β̂ of this λ: in `scratch` (shared memory, 2p doubles per thread) when given —
    // local memory misses the small L1 left beside a large shared-memory carve-out
    double cvl[64], btl[64];
    double* cv = scratch ? scratch + 2 * p * tid : cvl;
    double* bt = scratch ? cv + p : btl;
    double sb = 0.0;
    for (int a = 0; a < p; ++a) {  // Step 6: c = Q⁻¹ XᵀV⁻¹y'
      double s = Cm[(M + a) * ldc + m];
      for (int b = 0; b < a; ++b) s -= Q[a * ldq + b] * cv[b];
      cv[a] = s * Q[a * ldq + a];
      sb += cv[a] * cv[a];  // Step 7: ssqBetahat = cᵀc
    }
    const double yy = Cm[m * ldc + m];
    const double q = yy - sb;  // Step 8: ssqResidual
    // R12: the subtraction resolves q only when q > 1e-10·yy; otherwise the λ
    // column fails (ℓ_p = −∞, σ̂²/β̂ NaN, status NEG_RESID) — no OK column can
    // report q ≤ 0 (log σ̂² = −∞ would make ℓ_p = +∞)
    const bool neg = !(q > 1e-10 * yy);
    for (int a = p - 1; a >= 0; --a) {  // β̂ = Q⁻ᵀ c (Eq. betahat)
      double s = cv[a];
      for (int b = a + 1; b < p; ++b) s -= Q[b * ldq + a] * bt[b];
      bt[a] = s * Q[a * ldq + a];
    }
    const size_t km = (size_t)k * M + m;
    if (A.ssqBetahat) A.ssqBetahat[km] = sb;
    if (A.ssqResidual) A.ssqResidual[km] = yy - sb;
    if (neg) {
      A.loglik[km] = -INFINITY;
      A.sigma2hat[km] = nan;
      for (int a = 0; a < p; ++a) A.betahat[km * p + a] = nan;
      if (A.loglik_reml) A.loglik_reml[km] = -INFINITY;
      if (A.sigma2hat_reml) A.sigma2hat_reml[km] = nan;
      atomicExch(&flag[2], 1);
    } else {
      const double s2 = q / n;  // Eq. 4
      const double jac = (A.lambdas[m] - 1.0) * S;
      // Eq. (profile): −2ℓ_p = n log σ̂² + log|V| − 2(λ−1)Σ log y + n log 2π + n
      A.loglik[km] = -0.5 * (n * log(s2) + ldV + n * ln2pi + n) + jac;
      A.sigma2hat[km] = s2;
      for (int a = 0; a < p; ++a) A.betahat[km * p + a] = bt[a];
      if (A.loglik_reml || A.sigma2hat_reml) {
        // Eq. remlpro with σ̂²_reml = q/(n−p) (Eq. sigmahat_reml_y)
        const double np_ = n - p, s2r = q / np_;
        if (A.sigma2hat_reml) A.sigma2hat_reml[km] = s2r;
        if (A.loglik_reml)
          A.loglik_reml[km] = -0.5 * (np_ * log(s2r) + ldV + ldx + n * ln2pi + np_) + jac;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (A.detReml) A.detReml[k] = ldx;
    A.logdetV[k] = ldV;
    A.status[k] = flag[2] ? LIK_PT_NEG_RESID : LIK_PT_OK;
  }
}

}  // namespace lik
