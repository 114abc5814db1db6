// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct FP64 CPU implementation of what the hot
// path of arXiv 2305.04318 computes: the Gaussian LGM profile log-likelihood
// for K correlation-parameter points omega_k, each with M Box-Cox lambdas.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.  The product path
// (paper_2305_04318_b200/) never links, imports or calls it, and this file
// shares no code, headers, tables or helpers with it.
//
// Citations: "P:<line>" = /root/reference/PAPER.md line (section / equation
// named beside it).  Readings of the paper where it is silent or garbled are
// numbered R<k> and listed in DESIGN.md §3.
//
// Every function below is pinned by a "-m 'not gpu'" test in
// tests/test_oracle_pins.py against something other than itself (worked
// examples, closed forms, mpmath brute force, invariants).  Parity unpinned:
// nothing on the hot path (the paper's real-data tables are out of scope).
// ============================================================================
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cfloat>
#include <stdexcept>
#include <thread>
#include <vector>
#include <algorithm>

namespace {

const double kPi = 3.14159265358979323846264338327950288;

// Status codes (same meaning as the ABI's, declared independently here).
enum { PT_OK = 0, PT_V_NOT_PD = 1, PT_XVX_NOT_PD = 2, PT_NEG_RESID = 3, PT_BAD_PARAM = 4 };
enum { OK = 0, EINVAL_ = -1, EDOMAIN_ = -2, ERANK_ = -3 };

// ---------------------------------------------------------------------------
// Box-Cox transform, P:59-66 (§2): b(y;λ) = (y^λ − 1)/λ for λ ≠ 0, log y at λ = 0.
// R14: the λ = 0 branch is taken for |λ| < 1e-10; (y^λ − 1) is evaluated as
// expm1(λ log y), which is the same number without cancellation.
// ---------------------------------------------------------------------------
double boxcox(double y, double lambda) {
  if (std::fabs(lambda) < 1e-10) return std::log(y);
  return std::expm1(lambda * std::log(y)) / lambda;
}

// ---------------------------------------------------------------------------
// Anisotropic distance d(x), P:104-120 (Eq. matern, second line), literally:
//   d = || diag(1/φX, 1/φY) · [[cos φA, −sin φA],[sin φA, cos φA]] · (x1, x2) ||
// R3: φY = φX / φR.
// ---------------------------------------------------------------------------
double aniso_distance(double x1, double x2, double phiX, double phiR, double phiA) {
  const double phiY = phiX / phiR;
  const double c = std::cos(phiA), s = std::sin(phiA);
  const double u = c * x1 - s * x2;     // first row of the rotation
  const double v = s * x1 + c * x2;     // second row of the rotation
  const double a = u / phiX, b = v / phiY;
  return std::sqrt(a * a + b * b);
}

// ---------------------------------------------------------------------------
// log K_nu(z) by the integral representation (DLMF 10.32.9)
//     K_nu(z) = ∫_0^∞ exp(−z cosh t) cosh(nu t) dt,
// evaluated with the trapezoid rule in log space (the integrand is even and
// entire in t, so the rule converges geometrically).  Used only where the
// library routine overflows or underflows (R9).
// ---------------------------------------------------------------------------
double log_bessel_k_integral(double nu, double z) {
  // log of the integrand: −z cosh t + log cosh(nu t)
  auto f = [nu, z](double t) {
    const double a = nu * t;
    return -z * std::cosh(t) + a + std::log1p(std::exp(-2.0 * a)) - std::log(2.0);
  };
  // peak near z sinh t = nu tanh(nu t); start from t* = asinh(nu / z)
  double tstar = std::asinh(nu / z);
  // width of the peak ~ 1/sqrt(z cosh t* + small)
  double curv = z * std::cosh(tstar);
  double sigma = 1.0 / std::sqrt(curv + 1.0);
  double h = std::min(0.02, sigma / 24.0);
  // locate the maximum by ternary search (f is unimodal on t >= 0: f'(0) = 0 and
  // f' = −z sinh t + nu tanh(nu t) changes sign at most once)
  double lo = 0.0, hi = tstar + 20.0 * sigma + 1.0;
  for (int it = 0; it < 200; ++it) {
    const double m1 = lo + (hi - lo) / 3.0, m2 = hi - (hi - lo) / 3.0;
    if (f(m1) < f(m2)) lo = m1; else hi = m2;
  }
  const double fmax = std::max(f(0.0), f(0.5 * (lo + hi)));
  // trapezoid over [0, T]; the integrand is even so the t = 0 node has weight 1/2
  double sum = 0.5 * std::exp(f(0.0) - fmax);
  double t = h;
  for (long k = 1; k < 50000000; ++k, t = k * h) {
    double g = f(t) - fmax;
    sum += std::exp(g);
    if (t > tstar && g < -60.0) break;
  }
  return fmax + std::log(h * sum);
}

// log K_nu(z): the library routine (libstdc++ std::cyl_bessel_k) where it is
// finite and normal, otherwise the integral above (R9).
double log_bessel_k(double nu, double z) {
  double k = 0.0;
  bool ok = true;
  try {
    k = std::cyl_bessel_k(nu, z);
  } catch (...) {
    ok = false;
  }
  if (ok && std::isfinite(k) && k > 1e-290) return std::log(k);
  return log_bessel_k_integral(nu, z);
}

// ---------------------------------------------------------------------------
// Matérn correlation, P:100-103 and P:122-123 (§2.1):
//   ρ(d; κ) = 2^{1−κ}/Γ(κ) · (√(8κ) d)^κ · K_κ(√(8κ) d)
// R1: the prefactor is printed as 2^{κ−1}/Γ(κ); that gives ρ(0+) ≠ 1,
//     so the normalised 2^{1−κ}/Γ(κ) is used.
// R7: for κ ≥ 1e3 the Gaussian limit exp(−2d²) stated at P:123 is used.
// R8: ρ is evaluated in log space; ρ := 0 where log ρ < −745 (exp underflows).
// ---------------------------------------------------------------------------
double matern_rho(double d, double kappa) {
  if (d == 0.0) return 1.0;
  if (kappa >= 1e3) return std::exp(-2.0 * d * d);
  const double z = std::sqrt(8.0 * kappa) * d;
  const double logrho = (1.0 - kappa) * std::log(2.0) - std::lgamma(kappa) +
                        kappa * std::log(z) + log_bessel_k(kappa, z);
  return std::exp(logrho);
}

bool params_valid(const double* w) {
  for (int i = 0; i < 5; ++i)
    if (!std::isfinite(w[i])) return false;
  return w[0] > 0.0 && w[1] > 0.0 && w[2] >= 0.0 && w[3] > 0.0;
}

// ---------------------------------------------------------------------------
// V = R + ν² I, P:86 (Eq. 1 block) and P:311 (§3.3 Step 1):
//   R_ij = ρ(s_i − s_j; ω), ν² on the diagonal.  Row-major n×n, full.
// ---------------------------------------------------------------------------
void build_V(int n, const double* coords, const double* w, double* V) {
  const double phiX = w[0], kappa = w[1], nugget = w[2], phiR = w[3], phiA = w[4];
  for (int i = 0; i < n; ++i) {
    V[(size_t)i * n + i] = 1.0 + nugget;
    for (int j = 0; j < i; ++j) {
      const double hx = coords[2 * i] - coords[2 * j];
      const double hy = coords[2 * i + 1] - coords[2 * j + 1];
      const double rho = matern_rho(aniso_distance(hx, hy, phiX, phiR, phiA), kappa);
      V[(size_t)i * n + j] = rho;
      V[(size_t)j * n + i] = rho;
    }
  }
}

// ---------------------------------------------------------------------------
// Unblocked LDLᵀ, P:312 (§3.3 Step 2): V = L D Lᵀ, L unit lower triangular.
// L is written into the strict lower triangle of A (row-major n×n); D into D.
// R11: a pivot D_j ≤ n·ε·max_i V_ii means "not positive definite".
// Returns 0 on success, 1 if not PD.
// ---------------------------------------------------------------------------
int ldl(int n, double* A, double* D) {
  double vmax = 0.0;
  for (int i = 0; i < n; ++i) vmax = std::max(vmax, A[(size_t)i * n + i]);
  const double tol = n * DBL_EPSILON * vmax;
  for (int j = 0; j < n; ++j) {
    double* Lj = A + (size_t)j * n;
    double dj = Lj[j];
    for (int k = 0; k < j; ++k) dj -= Lj[k] * Lj[k] * D[k];
    if (!(dj > tol)) return 1;
    D[j] = dj;
    for (int i = j + 1; i < n; ++i) {
      double* Li = A + (size_t)i * n;
      double s = Li[j];
      for (int k = 0; k < j; ++k) s -= Li[k] * Lj[k] * D[k];
      Li[j] = s / dj;
    }
  }
  return 0;
}

// Forward substitution with unit lower L (strict lower part of A):
// solves L Z = B for Z (n×r, row-major), P:313 (§3.3 Step 3).
void forward_unit(int n, const double* A, int r, const double* B, double* Z) {
  for (int i = 0; i < n; ++i) {
    for (int t = 0; t < r; ++t) {
      double s = B[(size_t)i * r + t];
      for (int k = 0; k < i; ++k) s -= A[(size_t)i * n + k] * Z[(size_t)k * r + t];
      Z[(size_t)i * r + t] = s;
    }
  }
}

struct PointResult {
  int status;
  double logdetV;               // Table 1 detVar
  double detReml;               // Table 1 detReml = log|XᵀV⁻¹X|
  std::vector<double> ssqYX;    // Table 1 ssqYX, r×r, r = M + p, columns [y'_1..y'_M | X]
  std::vector<double> ssqBetahat, ssqResidual, qdirect;  // M each
  std::vector<double> loglik, sigma2, beta;               // M, M, M×p
  std::vector<double> loglik_reml, sigma2_reml;           // M, M (Appendix, REML)
};

// ---------------------------------------------------------------------------
// One parameter point through the paper's Steps 1-8 (§3.3) and the
// profile likelihood (Eq. profile).
//   S = Σ log y_i; B = [y'_1 .. y'_M | X] (n × r).
// ---------------------------------------------------------------------------
PointResult eval_point(int n, int p, const double* coords, const double* X, int M,
                       const double* lambdas, const double* Bmat, double S, const double* w) {
  PointResult R;
  const int r = M + p;
  R.status = PT_OK;
  R.logdetV = NAN;
  R.detReml = NAN;
  R.ssqYX.assign((size_t)r * r, NAN);
  R.ssqBetahat.assign(M, NAN);
  R.ssqResidual.assign(M, NAN);
  R.qdirect.assign(M, NAN);
  R.loglik.assign(M, -INFINITY);
  R.sigma2.assign(M, NAN);
  R.beta.assign((size_t)M * p, NAN);
  R.loglik_reml.assign(M, -INFINITY);
  R.sigma2_reml.assign(M, NAN);
  if (!params_valid(w)) { R.status = PT_BAD_PARAM; return R; }

  // Step 1: Matérn variance matrix V
  std::vector<double> A((size_t)n * n);
  build_V(n, coords, w, A.data());
  // Step 2: V = L D Lᵀ, log|V| = Σ log D
  std::vector<double> D(n);
  if (ldl(n, A.data(), D.data())) { R.status = PT_V_NOT_PD; return R; }
  double logdet = 0.0;
  for (int j = 0; j < n; ++j) logdet += std::log(D[j]);
  R.logdetV = logdet;
  // Step 3: Z = L⁻¹ (y', X)
  std::vector<double> Z((size_t)n * r);
  forward_unit(n, A.data(), r, Bmat, Z.data());
  // Step 4: ssqYX = (y', X)ᵀ V⁻¹ (y', X) = Zᵀ D⁻¹ Z (Table 1)
  for (int a = 0; a < r; ++a)
    for (int b = 0; b < r; ++b) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += Z[(size_t)i * r + a] * Z[(size_t)i * r + b] / D[i];
      R.ssqYX[(size_t)a * r + b] = s;
    }
  // Step 5: XᵀV⁻¹X = Q P Qᵀ; its block sits at rows/cols M..M+p-1
  std::vector<double> XX((size_t)p * p), Pd(p);
  for (int a = 0; a < p; ++a)
    for (int b = 0; b < p; ++b) XX[(size_t)a * p + b] = R.ssqYX[(size_t)(M + a) * r + (M + b)];
  if (ldl(p, XX.data(), Pd.data())) {  // failed point: every output NaN / −∞ (ABI convention)
    R.status = PT_XVX_NOT_PD;
    R.logdetV = NAN;
    R.ssqYX.assign((size_t)r * r, NAN);
    return R;
  }
  double detReml = 0.0;
  for (int a = 0; a < p; ++a) detReml += std::log(Pd[a]);
  R.detReml = detReml;

  for (int m = 0; m < M; ++m) {
    // Step 6: c = Q⁻¹ XᵀV⁻¹y'_m
    std::vector<double> Xy(p), c(p), beta(p);
    for (int a = 0; a < p; ++a) Xy[a] = R.ssqYX[(size_t)(M + a) * r + m];
    forward_unit(p, XX.data(), 1, Xy.data(), c.data());
    // Step 7: ssqBetahat = cᵀ P⁻¹ c
    double sb = 0.0;
    for (int a = 0; a < p; ++a) sb += c[a] * c[a] / Pd[a];
    R.ssqBetahat[m] = sb;
    // Step 8: ssqResidual = y'ᵀV⁻¹y' − ssqBetahat
    R.ssqResidual[m] = R.ssqYX[(size_t)m * r + m] - sb;
    // R12: Step 8's subtraction resolves q only when q > 1e-10·y'ᵀV⁻¹y'; otherwise
    // (y'_m numerically in span(X), or negative by rounding) the λ column fails:
    // status NEG_RESID, ℓ_p = −∞, σ̂²/β̂ NaN for that column (the others stand).
    if (!(R.ssqResidual[m] > 1e-10 * R.ssqYX[(size_t)m * r + m])) {
      R.status = PT_NEG_RESID;
      continue;
    }
    // β̂ = (XᵀV⁻¹X)⁻¹ XᵀV⁻¹y' (Eq. betahat) = Q⁻ᵀ P⁻¹ c (back substitution)
    for (int a = p - 1; a >= 0; --a) {
      double s = c[a] / Pd[a];
      for (int b = a + 1; b < p; ++b) s -= XX[(size_t)b * p + a] * beta[b];
      beta[a] = s;
    }
    // Eq. 4 literally: q = (y' − Xβ̂)ᵀ V⁻¹ (y' − Xβ̂), through the factors
    std::vector<double> res(n), zr(n);
    for (int i = 0; i < n; ++i) {
      double s = Bmat[(size_t)i * r + m];
      for (int a = 0; a < p; ++a) s -= X[(size_t)i * p + a] * beta[a];
      res[i] = s;
    }
    forward_unit(n, A.data(), 1, res.data(), zr.data());
    double q = 0.0;
    for (int i = 0; i < n; ++i) q += zr[i] * zr[i] / D[i];
    R.qdirect[m] = q;
    const double sigma2 = q / n;  // Eq. 4
    // Eq. profile:
    // −2ℓ_p = n log(q/n) + log|V| − 2(λ−1)Σ log y + n log 2π + n
    const double m2l = n * std::log(sigma2) + logdet - 2.0 * (lambdas[m] - 1.0) * S +
                       n * std::log(2.0 * kPi) + n;
    R.loglik[m] = -0.5 * m2l;
    R.sigma2[m] = sigma2;
    // REML (Appendix): σ̂²_reml = q/(n−p) (Eq. sigmahat_reml_y) and Eq. remlpro
    // (P:902-905): −2ℓ*_p = (n−p) log(q/(n−p)) + log|V| + log|XᵀV⁻¹X|
    //                      − 2(λ−1)Σ log y + n log 2π + n − p
    const double s2r = q / (n - p);
    const double m2lr = (n - p) * std::log(s2r) + logdet + detReml -
                        2.0 * (lambdas[m] - 1.0) * S + n * std::log(2.0 * kPi) + (n - p);
    R.loglik_reml[m] = -0.5 * m2lr;
    R.sigma2_reml[m] = s2r;
    for (int a = 0; a < p; ++a) R.beta[(size_t)m * p + a] = beta[a];
  }
  return R;
}

// Call-level validation (R6, SPEC-style data contract): returns OK or <0.
int validate(int n, int p, const double* coords, const double* y, const double* X, int K,
             const double* params, int M, const double* lambdas) {
  if (!coords || !y || !X || !params || !lambdas) return EINVAL_;
  if (p < 1 || n < p + 2 || K < 1 || M < 1) return EINVAL_;
  for (int i = 0; i < 2 * n; ++i) if (!std::isfinite(coords[i])) return EINVAL_;
  for (int i = 0; i < n; ++i) if (!std::isfinite(y[i])) return EINVAL_;
  for (int i = 0; i < n * p; ++i) if (!std::isfinite(X[i])) return EINVAL_;
  for (int m = 0; m < M; ++m) if (!std::isfinite(lambdas[m])) return EINVAL_;
  for (int i = 0; i < n; ++i) if (!(y[i] > 0.0)) return EDOMAIN_;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j)
      if (coords[2 * i] == coords[2 * j] && coords[2 * i + 1] == coords[2 * j + 1]) return EDOMAIN_;
  // full column rank of X: modified Gram-Schmidt with a relative threshold
  std::vector<double> Q((size_t)n * p);
  for (int i = 0; i < n * p; ++i) Q[i] = X[i];
  for (int a = 0; a < p; ++a) {
    double norm0 = 0.0;
    for (int i = 0; i < n; ++i) norm0 += X[(size_t)i * p + a] * X[(size_t)i * p + a];
    for (int b = 0; b < a; ++b) {
      double dot = 0.0;
      for (int i = 0; i < n; ++i) dot += Q[(size_t)i * p + a] * Q[(size_t)i * p + b];
      for (int i = 0; i < n; ++i) Q[(size_t)i * p + a] -= dot * Q[(size_t)i * p + b];
    }
    double nrm = 0.0;
    for (int i = 0; i < n; ++i) nrm += Q[(size_t)i * p + a] * Q[(size_t)i * p + a];
    if (!(nrm > 1e-20 * norm0) || norm0 == 0.0) return ERANK_;
    nrm = std::sqrt(nrm);
    for (int i = 0; i < n; ++i) Q[(size_t)i * p + a] /= nrm;
  }
  return OK;
}

}  // namespace

// ============================================================================
// Exported C entry points (ctypes).  All arrays row-major FP64, caller-owned.
// ============================================================================
extern "C" {

double oracle_boxcox(double y, double lambda) { return boxcox(y, lambda); }
double oracle_aniso_distance(double x1, double x2, double phiX, double phiR, double phiA) {
  return aniso_distance(x1, x2, phiX, phiR, phiA);
}
double oracle_log_bessel_k(double nu, double z) { return log_bessel_k(nu, z); }
double oracle_log_bessel_k_integral(double nu, double z) { return log_bessel_k_integral(nu, z); }
double oracle_matern_rho(double d, double kappa) { return matern_rho(d, kappa); }

// V (n×n, full, row-major) for one parameter point params5 = {φX, κ, ν², φR, φA}.
void oracle_build_V(int n, const double* coords, const double* params5, double* V) {
  build_V(n, coords, params5, V);
}

// LDLᵀ of a caller matrix (overwritten: strict lower = L).  Returns 0 / 1 (not PD).
int oracle_ldl(int n, double* A, double* D) { return ldl(n, A, D); }

int oracle_validate(int n, int p, const double* coords, const double* y, const double* X, int K,
                    const double* params, int M, const double* lambdas) {
  return validate(n, p, coords, y, X, K, params, M, lambdas);
}

// Full batched evaluation with the ABI's output layout:
//   loglik K×M, betahat K×M×p, sigma2hat K×M, logdetV K, status K.
// Optional (may be NULL): ssqYX K×r×r, detReml K, ssqResidual K×M (Step 8 form),
// qdirect K×M (Eq. 4 form), ssqBetahat K×M, loglik_reml K×M (Eq. remlpro),
// sigma2_reml K×M.  nthreads ≥ 1 std::threads over points.
int oracle_eval(int n, int p, const double* coords, const double* y, const double* X, int K,
                const double* params, int M, const double* lambdas, double* loglik,
                double* betahat, double* sigma2hat, double* logdetV, int* status,
                double* ssqYX, double* detReml, double* ssqResidual, double* qdirect,
                double* ssqBetahat, double* loglik_reml, double* sigma2_reml, int nthreads) {
  int rc = validate(n, p, coords, y, X, K, params, M, lambdas);
  if (rc != OK) return rc;
  if (!loglik || !betahat || !sigma2hat || !logdetV || !status) return EINVAL_;
  const int r = M + p;
  // S = Σ log y_i (Jacobian); B = [b(y; λ_1) .. b(y; λ_M) | X]
  double S = 0.0;
  for (int i = 0; i < n; ++i) S += std::log(y[i]);
  std::vector<double> B((size_t)n * r);
  for (int i = 0; i < n; ++i) {
    for (int m = 0; m < M; ++m) B[(size_t)i * r + m] = boxcox(y[i], lambdas[m]);
    for (int a = 0; a < p; ++a) B[(size_t)i * r + M + a] = X[(size_t)i * p + a];
  }
  if (nthreads < 1) nthreads = 1;
  auto work = [&](int tid) {
    for (int k = tid; k < K; k += nthreads) {
      PointResult R = eval_point(n, p, coords, X, M, lambdas, B.data(), S, params + 5 * (size_t)k);
      status[k] = R.status;
      logdetV[k] = R.logdetV;
      for (int m = 0; m < M; ++m) {
        loglik[(size_t)k * M + m] = R.loglik[m];
        sigma2hat[(size_t)k * M + m] = R.sigma2[m];
        for (int a = 0; a < p; ++a) betahat[((size_t)k * M + m) * p + a] = R.beta[(size_t)m * p + a];
        if (ssqResidual) ssqResidual[(size_t)k * M + m] = R.ssqResidual[m];
        if (qdirect) qdirect[(size_t)k * M + m] = R.qdirect[m];
        if (ssqBetahat) ssqBetahat[(size_t)k * M + m] = R.ssqBetahat[m];
        if (loglik_reml) loglik_reml[(size_t)k * M + m] = R.loglik_reml[m];
        if (sigma2_reml) sigma2_reml[(size_t)k * M + m] = R.sigma2_reml[m];
      }
      if (ssqYX) for (int t = 0; t < r * r; ++t) ssqYX[(size_t)k * r * r + t] = R.ssqYX[t];
      if (detReml) detReml[k] = R.detReml;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return OK;
}

// ---------------------------------------------------------------------------
// Profile log-likelihoods over the K×M grid (§3.4-3.6), from the Table-1
// summaries (the caller passes the oracle's own ssqYX, logdetV, status).
//  β_a profile (Eq. profilebetai): for β_a = b,
//    Q0 = y'ᵀV⁻¹y' − 2b (XᵀV⁻¹y')_a + b² (XᵀV⁻¹X)_aa
//    T  = (g0 − b g1)ᵀ H⁻¹ (g0 − b g1),  H = (XᵀV⁻¹X)_[−a,−a],
//         g0 = (XᵀV⁻¹y')_[−a], g1 = (XᵀV⁻¹X)_[−a,a]
//    q(b) = Q0 − T;  ℓ = −½[n log(q/n) + log|V| + n log 2π + n] + (λ−1)S,
//    out_beta[a·G + g] = max over (k, m) of ℓ at b = beta_grid[a·G + g].
//  σ profile (Eq. profileSigma): with q = ssqResidual (β̂ profiled),
//    ℓ(σ) = −½[q/σ² + n log σ² + log|V| + n log 2π] + (λ−1)S, max over (k, m).
//  λ profile: out_lambda[m] = max over k of ℓ_p(ω_k, λ_m).
// ---------------------------------------------------------------------------
void oracle_profiles(int n, int p, int K, int M, const double* ssqYX, const double* logdetV,
                     const int* status, const double* lambdas, const double* y, int G,
                     const double* beta_grid, double* out_beta, int Sg,
                     const double* sigma_grid, double* out_sigma, double* out_lambda) {
  const int r = M + p;
  double S = 0.0;
  for (int i = 0; i < n; ++i) S += std::log(y[i]);
  const double ln2pi = std::log(2.0 * kPi);
  for (int e = 0; e < p * G; ++e) out_beta[e] = -INFINITY;
  for (int e = 0; e < Sg; ++e) out_sigma[e] = -INFINITY;
  for (int m = 0; m < M; ++m) out_lambda[m] = -INFINITY;
  for (int k = 0; k < K; ++k) {
    // failed points are skipped; a NEG_RESID point only in its failed λ columns (R12)
    if (status[k] != PT_OK && status[k] != PT_NEG_RESID) continue;
    const double* C = ssqYX + (size_t)k * r * r;
    auto c = [&](int i, int j) { return C[(size_t)i * r + j]; };
    // full XᵀV⁻¹X factor for β̂ (σ and λ profiles)
    std::vector<double> XX((size_t)p * p), Dx(p);
    for (int a = 0; a < p; ++a)
      for (int b = 0; b < p; ++b) XX[(size_t)a * p + b] = c(M + a, M + b);
    if (ldl(p, XX.data(), Dx.data())) continue;
    for (int m = 0; m < M; ++m) {
      const double jac = (lambdas[m] - 1.0) * S;
      // q = y'ᵀV⁻¹y' − (XᵀV⁻¹y')ᵀ(XᵀV⁻¹X)⁻¹(XᵀV⁻¹y')  (Step 8)
      std::vector<double> xy(p), u(p);
      for (int a = 0; a < p; ++a) xy[a] = c(M + a, m);
      forward_unit(p, XX.data(), 1, xy.data(), u.data());
      double sb = 0.0;
      for (int a = 0; a < p; ++a) sb += u[a] * u[a] / Dx[a];
      const double q = c(m, m) - sb;
      if (!(q > 1e-10 * c(m, m))) continue;  // R12: the column failed
      const double lp = -0.5 * (n * std::log(q / n) + logdetV[k] + n * ln2pi + n) + jac;
      out_lambda[m] = std::max(out_lambda[m], lp);
      for (int t = 0; t < Sg; ++t) {
        const double s2 = sigma_grid[t] * sigma_grid[t];
        const double l = -0.5 * (q / s2 + n * std::log(s2) + logdetV[k] + n * ln2pi) + jac;
        out_sigma[t] = std::max(out_sigma[t], l);
      }
      for (int a = 0; a < p; ++a) {
        // H = (XᵀV⁻¹X) without row/column a, g0, g1
        const int pm = p - 1;
        std::vector<double> H((size_t)pm * pm + 1), Dh(pm + 1), g0(pm + 1), g1(pm + 1);
        std::vector<double> w0(pm + 1), w1(pm + 1);
        int ii = 0;
        for (int i = 0; i < p; ++i) {
          if (i == a) continue;
          int jj = 0;
          for (int j = 0; j < p; ++j) {
            if (j == a) continue;
            H[(size_t)ii * pm + jj] = c(M + i, M + j);
            ++jj;
          }
          g0[ii] = c(M + i, m);
          g1[ii] = c(M + i, M + a);
          ++ii;
        }
        bool okH = true;
        if (pm > 0) {
          okH = ldl(pm, H.data(), Dh.data()) == 0;
          forward_unit(pm, H.data(), 1, g0.data(), w0.data());
          forward_unit(pm, H.data(), 1, g1.data(), w1.data());
        }
        if (!okH) continue;
        double t00 = 0.0, t01 = 0.0, t11 = 0.0;  // g0ᵀH⁻¹g0, g0ᵀH⁻¹g1, g1ᵀH⁻¹g1
        for (int i = 0; i < pm; ++i) {
          t00 += w0[i] * w0[i] / Dh[i];
          t01 += w0[i] * w1[i] / Dh[i];
          t11 += w1[i] * w1[i] / Dh[i];
        }
        for (int gg = 0; gg < G; ++gg) {
          const double b = beta_grid[(size_t)a * G + gg];
          const double Q0 = c(m, m) - 2.0 * b * c(M + a, m) + b * b * c(M + a, M + a);
          const double T = t00 - 2.0 * b * t01 + b * b * t11;
          const double qb = Q0 - T;
          const double l = -0.5 * (n * std::log(qb / n) + logdetV[k] + n * ln2pi + n) + jac;
          double& o = out_beta[(size_t)a * G + gg];
          o = std::max(o, l);
        }
      }
    }
  }
}

}  // extern "C"
