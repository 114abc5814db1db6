// Device FP64 Matérn correlation ρ, evaluated without Bessel functions.
//
// ρ(d; κ) = 2^{1−κ}/Γ(κ) · z^κ K_κ(z),  z = √(8κ) d          (Eq. matern; R1)
//
// With the integral representation (DLMF 10.32.10)
//   K_κ(z) = ½ (z/2)^κ ∫_0^∞ exp(−t − z²/(4t)) t^{−κ−1} dt
// and the substitution t = z²/(4w), the prefactor cancels exactly and
//   ρ = (1/Γ(κ)) ∫_0^∞ w^{κ−1} e^{−w} e^{−s/(4w)} dw,   s = z² = 8κ d²,
// i.e. ρ = E[exp(−s/(4W))] for W ~ Gamma(κ, 1) — the Matérn correlation as a scale
// mixture of Gaussians.  Nothing cancels between large terms (ρ ∈ (0, 1], ρ(0) = 1),
// nothing overflows for large κ at small z and nothing underflows at large z (the sum is
// carried in log space), and one formula covers every κ < 1e3 (R7: the Gaussian limit
// exp(−2d²) above).  The build never forms z: only s = 8κ d² (no square root).
//
// Quadrature.  With w = κ e^x,
//   ln ρ = C(κ) + ln ∫_{−∞}^{∞} e^{G(x; s)} dx,
//   G(x; s) = κ (x − (e^x − 1)) − (s/(4κ)) e^{−x},
//   C(κ)    = κ ln κ − κ − ln Γ(κ)
//           = ½ ln κ − ½ ln 2π − Σ_j B_2j / (2j(2j−1) κ^{2j−1})   (Stirling, used for κ ≥ 10,
//             so the O(κ ln κ) terms cancel analytically, not in floating point).
// G is strictly concave (G'' = −κe^x − (s/4κ)e^{−x}) and entire, with double-exponential
// tails, so the trapezoid rule on the whole line converges geometrically in 1/h: its
// relative error is the Fourier transform of e^G at 2π/h — |Γ(κ + 2πi/h)/Γ(κ)| at s = 0,
// ≈ exp(−2π²σ²/h²) around a Gaussian-like peak — which stays below 1e-17 for
//   h ≤ min(0.165, 0.45 σ),  σ² = −1/G''(x*) = 1/(κ r),  r = √(1 + s/κ²)
// (checked against mpmath for κ ∈ [0.01, 999]; tools/quad_step_check.py: 1.9e-17 at 0.45 σ.
// 0.6 σ would save 1.4 % on the small-n shapes but reaches 1.0e-15 near κ r ≈ 13, where
// 0.6 σ meets the cap and the Gaussian estimate fails).
//  The peak: G'(x*) = 0 ⇔ e^{x*} = (1 + r)/2.
// Nodes are summed outwards from the peak until G falls 40 below G(x*) (e^{−40} = 4e-18).
// Measured against mpmath besselk (50 digits) over κ ∈ [0.01, 999], z ∈ [1e-8, 700]:
// |Δ ln ρ| ≤ 2.1e-15 · max(1, |ln ρ|) (R8).
#pragma once
#include "lik_internal.cuh"

namespace lik {

#ifndef LIK_QUAD_ALPHA
#define LIK_QUAD_ALPHA 0.45
#endif
constexpr double kHalfLn2Pi = 0.91893853320467274178;  // ½ ln 2π
constexpr double kQuadHmax = 0.165;                    // trapezoid step cap (s → 0, small κ)
constexpr double kQuadAlpha = LIK_QUAD_ALPHA;          // step / σ
constexpr double kQuadCut = 40.0;                      // nodes kept while G ≥ G(x*) − 40
constexpr int kQuadMaxNodes = 1 << 16;                 // per side (only tiny κ at tiny s approach it)

// C(κ) = κ ln κ − κ − ln Γ(κ)  (once per point).
__device__ inline double matern_lnC(double k) {
  if (k >= 10.0) {
    // ln Γ(κ) = (κ − ½) ln κ − κ + ½ ln 2π + Σ_{j=1..8} B_2j / (2j(2j−1) κ^{2j−1}); the first
    // omitted term is < 2e-18 at κ = 10
    const double c[8] = {1.0 / 12.0, -1.0 / 360.0, 1.0 / 1260.0, -1.0 / 1680.0,
                         1.0 / 1188.0, -691.0 / 360360.0, 1.0 / 156.0, -3617.0 / 122400.0};
    const double k2 = 1.0 / (k * k);
    double t = c[7];
#pragma unroll
    for (int j = 6; j >= 0; --j) t = fma(t, k2, c[j]);
    return 0.5 * log(k) - kHalfLn2Pi - t / k;
  }
  return k * log(k) - k - lgamma(k);
}

// Peak x* of G(·; s) and the trapezoid step for that s.
__device__ __forceinline__ void quad_peak_step(double k, double s, double& xs, double& h) {
  const double q = s / (k * k);
  const double r = sqrt(1.0 + q);
  xs = log1p(q / (2.0 * (1.0 + r)));  // ln((1 + r)/2), r − 1 = q/(1 + r) without cancellation
  h = fmin(kQuadHmax, kQuadAlpha * rsqrt(k * r));
}

// e^x and e^x − 1 for a quadrature node: expm1 near 0 (where e^x − 1 cancels); e^x
// itself elsewhere — never 1 + expm1(x), which loses all digits of e^x for x ≲ −30
// (the left tails of small κ reach x ≈ −40 at the smallest s).
__device__ __forceinline__ void quad_exp(double x, double& ex, double& em) {
  ex = exp(x);
  em = fabs(x) < 0.5 ? expm1(x) : ex - 1.0;
}

// G(x; s) with a = s/(4κ).
__device__ __forceinline__ double quad_G(double k, double a, double x) {
  double ex, em;
  quad_exp(x, ex, em);
  return k * (x - em) - a / ex;
}

// Exact ln ρ at s = z² > 0 (Bessel mode).  Used for the table's interval edges and for
// the elements outside the point's table (rare); the table nodes use the octave-shared
// grid of table_kernel, the same rule.
static __device__ __noinline__ double log_rho_exact(const PointConst& P, double s) {
  const double k = P.kappa, a = s * P.inv4k;
  double xs, h;
  quad_peak_step(k, s, xs, h);
  const double gs = quad_G(k, a, xs);
  double sum = 1.0;  // the node at the peak
  for (int i = 1; i < kQuadMaxNodes; ++i) {
    const double g = quad_G(k, a, xs + i * h) - gs;
    if (g < -kQuadCut) break;
    sum += exp(g);
  }
  for (int i = 1; i < kQuadMaxNodes; ++i) {
    const double g = quad_G(k, a, xs - i * h) - gs;
    if (g < -kQuadCut) break;
    sum += exp(g);
  }
  return P.lnC + gs + log(h * sum);
}

// Scaled anisotropic distance d(h)², P:104-120 (R3: φY = φX/φR).
__device__ __forceinline__ double aniso_d2(const PointConst& P, double hx, double hy) {
  const double u = P.cX * hx - P.sX * hy;
  const double v = P.sY * hx + P.cY * hy;
  return u * u + v * v;
}

// ρ for a site pair at offset (hx, hy) by direct (exact) evaluation.
__device__ __forceinline__ double matern_rho_exact(const PointConst& P, double hx, double hy) {
  const double d2 = aniso_d2(P, hx, hy);
  if (d2 == 0.0) return 1.0;
  if (P.mode == MODE_GAUSS) return exp(-2.0 * d2);
  const double lr = log_rho_exact(P, P.eightk * d2);
  return lr < -760.0 ? 0.0 : exp(lr);
}

// 2^(j/16), j = 0..15, correctly rounded (mpmath).  16 entries = 128 bytes: one
// entry per bank pair, so a half-warp's data-dependent lookups never conflict (a
// 32-entry table doubled the exp's shared-memory wavefronts).
static __constant__ double kExp2Tab[16] = {
    1.0, 1.0442737824274138, 1.0905077326652577, 1.1387886347566916,
    1.189207115002721, 1.241857812073484, 1.2968395546510096, 1.3542555469368927,
    1.4142135623730951, 1.4768261459394993, 1.5422108254079407, 1.6104903319492543,
    1.681792830507429, 1.7562521603732995, 1.8340080864093424, 1.9152065613971474};

// 2^y for y ≤ ~0 (the table path's ρ = 2^{log2 ρ}): k = rint(16y), r = y − k/16 (exact,
// |r| ≤ 1/32), 2^r − 1 = Σ_{j=1..7} (r ln 2)^j / j! (truncation < 2e-18), 2^y =
// 2^(k>>4) · T[k & 15] · (1 + q) with T[j] = 2^(j/16) (etab, shared memory), the power
// of two added to the exponent field.  Results below 2^−1021 (ρ < 4.5e-308, R8) are
// flushed to 0 — so is the −2000 of the table's underflow octave.  ≤ 1 ulp.
__device__ __forceinline__ double exp2_neg(double y, const double* etab) {
  const double shift = 6755399441055744.0;  // 1.5·2^52: round-to-nearest integer in the low bits
  const double kds = fma(y, 16.0, shift);
  const double kd = kds - shift;
  const int k = __double2loint(kds);
  const double r = fma(kd, -0.0625, y);
  double q = fma(r, 1.5252733804059840e-05, 1.5403530393381608e-04);  // (ln2)^7/7!, (ln2)^6/6!
  q = fma(q, r, 1.3333558146428443e-03);
  q = fma(q, r, 9.6181291076284772e-03);
  q = fma(q, r, 5.5504108664821580e-02);
  q = fma(q, r, 2.4022650695910071e-01);
  q = fma(q, r, 6.9314718055994531e-01);
  q *= r;
  const double tj = etab[k & 15];
  const double v = fma(tj, q, tj);  // ∈ [0.97, 1.97]
  const int m = k >> 4;
  const double out = __hiloint2double(__double2hiint(v) + (m << 20), __double2loint(v));
  return m >= -1021 ? out : 0.0;
}

// Table evaluation of NE elements, interleaved (independent Horner chains for ILP).
// s = z² from the point's scaled rotation (no square root); the octave o of s is
// clamped to [olo, oz] (oz: the underflow octave, or ohi); elements whose octave lies
// outside [olo, ohs] (ohs = ohi, or "none" when the table reaches the underflow octave)
// need the exact path and set bit `bit + e` of `slow`; their returned value is
// meaningless.  CHECK = false skips the flags (five integer operations per element): for
// the pairs of distinct real sites of a point whose s range lies inside its table
// (PointConst::range_ok), which the table covers by construction.
template <int NE, int SUB, bool CHECK = true>
__device__ __forceinline__ void matern_rho_tableN(const PointConst& P, const double* coef,
                                                  const double* etab, int olo, int oz, unsigned span,
                                                  const double (&hx)[NE], const double (&hy)[NE],
                                                  double (&v)[NE], unsigned& slow, int bit) {
  constexpr int CHEB_N = Cheb<SUB>::N, CHEB_STRIDE = Cheb<SUB>::STRIDE, LG = Cheb<SUB>::LOG2SUB;
  double t[NE], h[NE];
  const double2* cp[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double u = fma(P.qX, hx[e], -P.qS * hy[e]);
    const double w = fma(P.qT, hx[e], P.qY * hy[e]);
    const double sv = fma(u, u, w * w);  // s = z² = 8κ d²
    const int hi = __double2hiint(sv);
    if (CHECK) {
      const int o = (hi >> 20) - (1023 + CHEB_ELO);
      slow |= (unsigned)((unsigned)(o - olo) > span) << (bit + e);
    }
    // interval = SUB·octave + the top log2(SUB) mantissa bits: one shift of the high word;
    // clamped to [SUB·olo, SUB·oz + SUB − 1] (above: the underflow octave's constant)
    const int iv = min(max((hi >> (20 - LG)) - SUB * (1023 + CHEB_ELO), SUB * olo), SUB * oz + SUB - 1);
    // t ∈ [−1, 1) from the mantissa alone: the mantissa without its top LG bits (the
    // interval) under the exponent field 1023 + LG + 1 is 2^{LG+1} + (the position in the
    // interval) ∈ [2^{LG+1}, 2^{LG+1} + 2); minus the centre 2^{LG+1} + 1 — exact, one LOP3
    // and one DADD
    t[e] = __hiloint2double((hi & (0x000fffff >> LG)) | ((1023 + LG + 1) << 20), __double2loint(sv)) -
           (double)((1 << (LG + 1)) + 1);
    cp[e] = reinterpret_cast<const double2*>(coef + iv * CHEB_STRIDE);
  }
#ifdef LIK_BUILD_PREFETCH
  // Horner with the next coefficient pair of every chain loaded one step ahead
  double2 un[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) un[e] = cp[e][CHEB_N / 2 - 1];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double2 u = un[e];
    un[e] = cp[e][CHEB_N / 2 - 2];
    h[e] = fma(u.y, t[e], u.x);
  }
#pragma unroll
  for (int mm = CHEB_N / 2 - 2; mm >= 0; --mm) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const double2 u = un[e];
      if (mm > 0) un[e] = cp[e][mm - 1];
      h[e] = fma(fma(h[e], t[e], u.y), t[e], u.x);
    }
  }
#else
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double2 u = cp[e][CHEB_N / 2 - 1];
    h[e] = fma(u.y, t[e], u.x);
  }
#pragma unroll
  for (int mm = CHEB_N / 2 - 2; mm >= 0; --mm) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const double2 u = cp[e][mm];
      h[e] = fma(fma(h[e], t[e], u.y), t[e], u.x);
    }
  }
#endif
#pragma unroll
  for (int e = 0; e < NE; ++e) v[e] = exp2_neg(h[e], etab);
}

#if LIK_BUILD_TEXMASK
// The build's coefficient loads split between two pipes: the pairs mm with bit mm of
// LIK_BUILD_TEXMASK set come through the texture path (tex1Dfetch<int4> on the table in
// global memory, L1-resident), the others from shared memory.  With every pair from
// shared memory the build was bound by the shared-memory data pipe (88 % of its
// wavefronts, ~2.2 distinct intervals per quarter-warp: each LDS.128 took 4 wavefronts);
// all through the texture path: 325 ms per C4 step; two of the eight pairs (mm 2 and 5):
// 165 ms (from 194), DESIGN.md §5.
template <int NE, int SUB, bool CHECK = true>
__device__ __forceinline__ void matern_rho_tableN_tex(const PointConst& P, cudaTextureObject_t tex,
                                                      long long tbase, const double* coef,
                                                      const double* etab, int olo,
                                                      int oz, unsigned span, const double (&hx)[NE],
                                                      const double (&hy)[NE], double (&v)[NE],
                                                      unsigned& slow, int bit) {
  constexpr int CHEB_N = Cheb<SUB>::N, CHEB_STRIDE = Cheb<SUB>::STRIDE, LG = Cheb<SUB>::LOG2SUB;
  double t[NE], h[NE];
  long long cp[NE];
  int ci[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double u = fma(P.qX, hx[e], -P.qS * hy[e]);
    const double w = fma(P.qT, hx[e], P.qY * hy[e]);
    const double sv = fma(u, u, w * w);
    const int hi = __double2hiint(sv);
    if (CHECK) {
      const int o = (hi >> 20) - (1023 + CHEB_ELO);
      slow |= (unsigned)((unsigned)(o - olo) > span) << (bit + e);
    }
    const int iv = min(max((hi >> (20 - LG)) - SUB * (1023 + CHEB_ELO), SUB * olo), SUB * oz + SUB - 1);
    t[e] = __hiloint2double((hi & (0x000fffff >> LG)) | ((1023 + LG + 1) << 20), __double2loint(sv)) -
           (double)((1 << (LG + 1)) + 1);
    cp[e] = tbase + (long long)iv * (CHEB_STRIDE / 2);
    ci[e] = iv * CHEB_STRIDE;
  }
  auto fetch = [&](int e, int mm) {
    if ((LIK_BUILD_TEXMASK >> mm) & 1) {
      const int4 q = tex1Dfetch<int4>(tex, (int)(cp[e] + mm));
      return make_double2(__hiloint2double(q.y, q.x), __hiloint2double(q.w, q.z));
    }
    return reinterpret_cast<const double2*>(coef + ci[e])[mm];
  };
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const double2 u = fetch(e, CHEB_N / 2 - 1);
    h[e] = fma(u.y, t[e], u.x);
  }
#pragma unroll
  for (int mm = CHEB_N / 2 - 2; mm >= 0; --mm) {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const double2 u = fetch(e, mm);
      h[e] = fma(fma(h[e], t[e], u.y), t[e], u.x);
    }
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) v[e] = exp2_neg(h[e], etab);
}
#endif

}  // namespace lik
