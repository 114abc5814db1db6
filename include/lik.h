/* ==========================================================================
 * lik.h — C ABI of the B200 (sm_100a) batched profile-likelihood library
 * (liblik.so, built from paper_2305_04318_b200/csrc/).
 *
 * What it computes (arXiv 2305.04318, PAPER.md "P:<line>"):
 *   For every correlation-parameter point ω_k = (φX, κ, ν², φR, φA) and every
 *   Box-Cox λ_m, the Gaussian linear geostatistical model profile
 *   log-likelihood ℓ_p(ω_k, λ_m; y) of Eq. (profile), P:145-148:
 *
 *     −2ℓ_p = n log(q/n) + log|V| − 2(λ−1) Σ log y_i + n log(2π) + n,
 *     q     = (y' − Xβ̂)ᵀ V⁻¹ (y' − Xβ̂)              (Eq. 4,  P:141)
 *     β̂     = (XᵀV⁻¹X)⁻¹ XᵀV⁻¹ y'                     (Eq. betahat)
 *     σ̂²    = q / n                                   (Eq. 4,  P:141)
 *     y'    = b(y; λ) = (y^λ − 1)/λ, log y at λ = 0   (§2)
 *     V     = R + ν² I, R_ij = ρ(s_i − s_j)           (Eq. 1 block)
 *     ρ(x)  = 2^{1−κ}/Γ(κ) (√(8κ) d)^κ K_κ(√(8κ) d)   (Eq. matern, P:100-103;
 *             prefactor read as 2^{1−κ}, R1)
 *     d(x)  = ‖diag(1/φX, 1/φY) Rot(φA) x‖, φY = φX/φR (R3)
 *
 *   following the paper's Steps 1-8 (§3.3): Matérn matrix, Cholesky
 *   of V with log|V|, triangular solve against [y'_1..y'_M | X], the cross
 *   products (Table 1), the p×p Cholesky of XᵀV⁻¹X, β̂, ssqBetahat
 *   and ssqResidual.  All M λ share one factorisation per point.
 *
 * Conventions (all entry points):
 *   - FP64 everywhere; matrices row-major; all buffers caller-owned (the
 *     library never frees or retains caller memory beyond the call).
 *   - coords: n×2 (x_i, y_i); y: n, all > 0; X: n×p (full column rank);
 *     params: K×5 {φX, κ, ν², φR, φA [radians]}; lambdas: M.
 *   - outputs: loglik K×M (ℓ_p, not −2ℓ_p), betahat K×M×p, sigma2hat K×M,
 *     logdetV K, status K (LIK_PT_*).
 *   - limits: 1 ≤ p ≤ 63, n ≥ p + 2, K ≥ 1, M ≥ 1.  With M + p > 64 the λ are
 *     evaluated in chunks of 64 − p (the factorisation is repeated per chunk; the
 *     kernels take r = M + p ≤ 64); the Table-1 / REML outputs of
 *     lik_eval_batch_device_ex and prepared datasets need M + p ≤ 64 (LIK_ENOTIMPL).
 *   - Call-level errors return < 0, write no outputs, and set the message
 *     returned by lik_last_error (naming the offending index).
 *   - Point-level failures never fail the call: status[k] != 0,
 *     loglik[k,·] = −inf, betahat/sigma2hat = NaN, logdetV[k] = NaN
 *     (for LIK_PT_NEG_RESID only the failing λ columns are −inf / NaN).
 *   - Results are bitwise deterministic for given inputs, independent of K,
 *     the wave size, the stream and the number of GPUs.
 *   - One lik_ctx per host thread; a ctx is bound to one CUDA device.
 *   - The device work of successive calls on one ctx runs in call order even when
 *     they are enqueued on different streams (each call's work waits on an event
 *     the previous call recorded at its end), because they share the ctx's
 *     workspace.  Caller buffers follow the usual stream rules.
 * ========================================================================== */
#ifndef LIK_H_
#define LIK_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lik_ctx lik_ctx; /* opaque */

/* Call-level return codes. */
enum {
  LIK_OK = 0,
  LIK_EINVAL = -1,   /* NULL pointer, bad sizes (n < p+2, p < 1, p > 63, K < 1, M < 1),
                        non-finite coords / y / X / lambdas */
  LIK_EDOMAIN = -2,  /* some y_i <= 0 (Box-Cox needs log y) or two coincident sites */
  LIK_ERANK = -3,    /* X not of full column rank */
  LIK_ENOMEM = -4,   /* device workspace allocation failed */
  LIK_ECUDA = -5,    /* a CUDA runtime error (message has the CUDA error string) */
  LIK_ENOTIMPL = -6  /* entry point or option not implemented (summaries / datasets with M + p > 64) */
};

/* Per-point status codes (status[k]). */
enum {
  LIK_PT_OK = 0,
  LIK_PT_V_NOT_PD = 1,    /* a Cholesky pivot of V <= n·eps·max V_ii (R11) */
  LIK_PT_XVX_NOT_PD = 2,  /* a pivot of XᵀV⁻¹X <= p·eps·max diag (Step 5) */
  LIK_PT_NEG_RESID = 3,   /* for some λ_m, Step 8's ssqResidual = y'ᵀV⁻¹y' − ssqBetahat is not
                             > 1e-10·y'ᵀV⁻¹y' (R12): y'_m numerically in
                             span(X), or negative by rounding.  Only those λ columns fail. */
  LIK_PT_BAD_PARAM = 4    /* φX <= 0, κ <= 0, ν² < 0, φR <= 0 or a non-finite parameter */
};

/* lik_create flags */
#define LIK_FLAG_TIMING 1u /* record CUDA events around every kernel launch (lik_get_stage_times) */
#define LIK_FLAG_NATURAL_ORDER 2u /* keep the caller's site order (default: Morton order for the
                                     Matérn build; results agree to rounding, invariance of ℓ_p
                                     under a symmetric permutation of the sites) */

/* Stages reported by lik_get_stage_times. */
enum {
  LIK_STAGE_PREP = 0,   /* Box-Cox columns, Σ log y (a1) */
  LIK_STAGE_SETUP = 1,  /* per-point constants (a2 prologue) */
  LIK_STAGE_BUILD = 2,  /* matern_build: ln ρ Chebyshev table + V tiles + [y'|X]ᵀ rows (a2) */
  LIK_STAGE_CHOL = 3,   /* chol_fused: Cholesky, solve, cross products, epilogue (a3-a7) */
  LIK_NSTAGES = 4
};

/* Create a context on CUDA device `cuda_device` (ordinal in the process's
 * visible set).  *out receives the context.  Returns LIK_OK, LIK_EINVAL
 * (out == NULL, unknown flag) or LIK_ECUDA (no such device / not sm_100). */
int lik_create(lik_ctx** out, int cuda_device, unsigned flags);

/* Release the context and its device workspace.  NULL is a no-op. */
void lik_destroy(lik_ctx* ctx);

/* Message describing the last non-OK return on this context ("" if none).
 * The pointer stays valid until the next call on ctx. */
const char* lik_last_error(const lik_ctx* ctx);

/* Batched evaluation, HOST pointers (the north_star's lik_eval_batch).
 * Copies the inputs to the device, runs the whole path on the context's own
 * stream, copies the outputs back and synchronises before returning. */
int lik_eval_batch(lik_ctx* ctx, int n, int p, const double* coords, const double* y,
                   const double* X, int K, const double* params, int M, const double* lambdas,
                   double* loglik, double* betahat, double* sigma2hat, double* logdetV,
                   int* status);

/* Same arguments, all DEVICE pointers (on ctx's device), enqueued on
 * `cuda_stream` (a cudaStream_t; NULL = the legacy default stream).  The
 * dataset (coords, y, X: ≤ n·(3+p) doubles) is read back to the host for the
 * call-level validation, so the call synchronises once on entry; the hot path
 * is then enqueued and the call returns without waiting for it (unless
 * LIK_FLAG_TIMING is set, in which case it waits to read the events). */
int lik_eval_batch_device(lik_ctx* ctx, int n, int p, const double* coords, const double* y,
                          const double* X, int K, const double* params, int M,
                          const double* lambdas, double* loglik, double* betahat,
                          double* sigma2hat, double* logdetV, int* status, void* cuda_stream);

/* lik_eval_batch_device plus the Table-1 summaries and the REML profile
 * likelihood (Table 1, Appendix).
 * Extra outputs (device pointers; each may be NULL to skip it):
 *   detReml     K      log|XᵀV⁻¹X| (Table 1 detReml; Step 5)
 *   ssqYX       K×r×r  [y'_1..y'_M | X]ᵀ V⁻¹ [y'_1..y'_M | X], r = M + p (Table 1
 *                      ssqYX: y'ᵀV⁻¹y' upper-left diagonal, XᵀV⁻¹X lower-right,
 *                      XᵀV⁻¹y' lower-left; Step 4)
 *   ssqBetahat  K×M    (Xβ̂)ᵀV⁻¹(Xβ̂) (Step 7)
 *   ssqResidual K×M    ssqYX_yy − ssqBetahat (Step 8; unclamped)
 *   loglik_reml K×M    ℓ*_p of Eq. remlpro:
 *                      −2ℓ*_p = (n−p) log(q/(n−p)) + log|V| + log|XᵀV⁻¹X|
 *                               − 2(λ−1)Σ log y + n log 2π + n − p
 *   sigma2hat_reml K×M q/(n−p) (Eq. sigmahat_reml_y)
 * Failed points get NaN summaries and −inf REML likelihoods (same status). */
int lik_eval_batch_device_ex(lik_ctx* ctx, int n, int p, const double* coords, const double* y,
                             const double* X, int K, const double* params, int M,
                             const double* lambdas, double* loglik, double* betahat,
                             double* sigma2hat, double* logdetV, int* status, double* detReml,
                             double* ssqYX, double* ssqBetahat, double* ssqResidual,
                             double* loglik_reml, double* sigma2hat_reml, void* cuda_stream);

/* Profile log-likelihoods over the K×M grid of evaluated points (SURVEY §8(f)
 * NEXT-2; §3.4-3.6), from the summaries of lik_eval_batch_device_ex.
 * All pointers are device pointers; the call is enqueued on `cuda_stream`.
 *   y          n      the response (Jacobian term Σ log y)
 *   ssqYX      K×r×r  Table-1 cross products, r = M + p;  logdetV K;  status K
 *              (points with status other than OK / NEG_RESID are skipped; a
 *              NEG_RESID point only in its failed λ columns, R12);  lambdas M
 *   beta_grid  p×G    values b of each coefficient β_a;  prof_beta p×G:
 *              ℓ_p(β_a = b) = max over (k, m) of ℓ with β_{−a}, σ² profiled out
 *              (Eq. profilebetai)
 *   sigma_grid Sg     values of σ;  prof_sigma Sg: max over (k, m) of ℓ(σ, β̂)
 *              (Eq. profileSigma)
 *   prof_lambda M     max over k of ℓ_p(ω_k, λ_m)
 * Limits: 1 ≤ p ≤ 32, G ≥ 0, Sg ≥ 0, K·M ≤ 2³⁰, K·(p+1) ≤ 2³⁰.  Returns LIK_OK, LIK_EINVAL, LIK_ENOMEM, LIK_ECUDA. */
int lik_profiles_device(lik_ctx* ctx, int n, int p, int K, int M, const double* y,
                        const double* ssqYX, const double* logdetV, const int* status,
                        const double* lambdas, int G, const double* beta_grid, double* prof_beta,
                        int Sg, const double* sigma_grid, double* prof_sigma, double* prof_lambda,
                        void* cuda_stream);

/* Accumulated per-stage device time (ms, from CUDA events on the launching
 * stream) and launch counts since the last reset; arrays of LIK_NSTAGES.
 * Requires LIK_FLAG_TIMING (else LIK_EINVAL). */
int lik_get_stage_times(lik_ctx* ctx, double* ms, long long* launches);
int lik_reset_stage_times(lik_ctx* ctx);

/* Prepared datasets: validate and upload (coords, y, X, lambdas) once — host
 * pointers, the same layouts, validation and error codes as lik_eval_batch —
 * then evaluate any number of parameter batches on it with
 * lik_dataset_eval_device: device pointers for params and the outputs (layouts as
 * in lik_eval_batch), enqueued on `cuda_stream` with no host synchronisation and
 * no host copy of the data (lik_eval_batch_device validates on the host on every
 * call).  Results are bitwise identical to lik_eval_batch_device on the same
 * inputs.  A dataset belongs to the device of the context that created it; it must
 * outlive the evaluations enqueued on it (destroy only after they completed).
 * (The paper's workflow: one dataset, many representative-point batches.) */
typedef struct lik_dataset lik_dataset;
int lik_dataset_create(lik_ctx* ctx, lik_dataset** out, int n, int p, const double* coords,
                       const double* y, const double* X, int M, const double* lambdas);
int lik_dataset_eval_device(lik_ctx* ctx, const lik_dataset* ds, int K, const double* params,
                            double* loglik, double* betahat, double* sigma2hat, double* logdetV,
                            int* status, void* cuda_stream);
void lik_dataset_destroy(lik_dataset* ds);

/* Points per wave, i.e. per build/factor launch (0 = automatic: the fewest
 * waves of at most 16 × (2 × #SMs) points within half the free HBM, each a
 * multiple of 2 × #SMs except the last;
 * an explicit value is capped at 85 % of free HBM and at 65,535; if the
 * allocation fails, the wave is re-sized from a fresh free-memory query).  The workspace holds one
 * slot per wave point (C4: 17.9 MB).  Small matrices (8⌈n/8⌉ + 8⌈(M+p)/8⌉ ≤ 216 rows, the
 * whole-octave table layout: n < 256) take the shared-memory path instead — one CTA per
 * point builds and factors its matrix on chip, no workspace, waves of up to 65,535
 * points.  Results do not depend on the wave size (determinism tests). */
int lik_set_wave_points(lik_ctx* ctx, int points_per_wave);

/* Debug / parity entry: the dense V = R + ν²I (n×n full, row-major) for each
 * of K ≤ 65,535 points, written by the same matern_build kernel the hot path uses.
 * Device pointers; synchronous.  Same validation as lik_eval_batch_device
 * for n, coords and params (bad points give an all-NaN matrix). */
int lik_debug_build_V(lik_ctx* ctx, int n, const double* coords, int K, const double* params,
                      double* V);

#ifdef __cplusplus
}
#endif
#endif /* LIK_H_ */
