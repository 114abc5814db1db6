// chol_small — the whole hot path of one parameter point in one CTA, for small
// augmented matrices (n_pad + r_pad ≤ SMALL_NMAX rows; the paper's own runs have
// n = 100 and 829 sites, C1/C2 n = 100/200): Matérn build (Step 1), Cholesky
// with log|V| (Step 2), the solve against [y'|X] (Step 3), the cross
// products (Step 4) and the epilogue (Steps 5-8, Eq. profile), with the
// augmented matrix A = [[V, B], [Bᵀ, 0]] held entirely in shared memory — no
// workspace in HBM, one launch per wave.
//
// Storage: the lower triangle of S = −A in 8×8 tiles (tile (I, J), J ≤ I, at
// I(I+1)/2 + J; 64 doubles, row-major with the XOR swizzle toff(), so the DMMA
// fragment loads are bank-conflict free).  Keeping −A makes every update a plain
// D = L·Lᵀ + C on the FP64 tensor cores (mma.sync.m8n8k4.f64 → DMMA.8x8x4), and the
// Schur block left after eliminating the V columns is +BᵀV⁻¹B = ssqYX.  V is padded
// to n_pad = 8⌈n/8⌉ with identity rows (log|V| and L⁻¹B unchanged); the r rows of Bᵀ
// start at n_pad.
//
// Right-looking elimination, one 8-column tile column k per step, with lookahead: a
// panel group of four warps brings column k+1 up to date with column k, factors its
// diagonal tile in registers (one rsqrt per pivot — the 8 pivots are the only serial
// chain) and solves the column below it (L_i,k+1 = A_i,k+1 L_k+1,k+1⁻ᵀ = S (−W)ᵀ),
// while the other warps apply column k to the columns ≥ k+2 (S_ij += L_ik L_jkᵀ, row
// segments, four independent tiles at a time).  One CTA barrier per step: the pivot
// chain and the solve of step k+1 run beside the trailing update of step k.
#include <cfloat>
#include <algorithm>
#include <cstdint>
#include "../../include/lik.h"
#include "lik_internal.cuh"
#include "matern_rho.cuh"
#include "point_epilogue.cuh"

#ifdef LIK_PHASE_TIMERS
__device__ unsigned long long g_lik_small_phase[36];
// (the clock read carries a memory clobber so it stays on its side of the barriers; a
// BAR.SYNC still blocks the warp only at a later instruction, so a barrier's wait can show
// up in the phase after it)
__device__ __forceinline__ long long sph_clock() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) : : "memory");
  return t;
}
#define SPH_INIT() long long sph_t = sph_clock(); long long sph_acc[12] = {0}
#define SPH(i) do { const long long t_ = sph_clock(); sph_acc[i] += t_ - sph_t; sph_t = t_; } while (0)
#define SPH_FLUSH(w, slot) do { if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) == (w)) for (int i_ = 0; i_ < 12; ++i_) atomicAdd(&g_lik_small_phase[12 * (slot) + i_], (unsigned long long)sph_acc[i_]); } while (0)
#else
#define SPH_INIT() do {} while (0)
#define SPH(i) do {} while (0)
#define SPH_FLUSH(w, slot) do {} while (0)
#endif

#ifndef LIK_SMALL_PIV2
#define LIK_SMALL_PIV2 1  // two pivots per step in the 8×8 factorisation (0: one; Swiss −0.7 %, C2 −0.5 %)
#endif
#ifndef LIK_SMALL_REGCHAIN
#define LIK_SMALL_REGCHAIN 1  // dependent 8×8 products chained through the registers
#endif
#ifndef LIK_SMALL_UCH
#define LIK_SMALL_UCH 2  // trailing-update tiles per chunk (C2 −6 %, Swiss −4 % against 4: the update competes less with the panel chain)
#endif

namespace lik {
namespace {

__device__ __forceinline__ void dmma8(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Element (a, b) of an 8×8 tile: row-major, column bit 2 flipped by row bit 1.  A/B
// fragment loads (lane → row lane/4, column 4kk + lane%4) and C fragment loads (lane →
// row lane/4, columns 2(lane%4) + {0, 1}, one 16-byte load) hit distinct banks.
__device__ __forceinline__ int toff(int a, int b) { return a * 8 + (b ^ ((a & 2) << 1)); }
__device__ __forceinline__ int tri8(int I, int J) { return I * (I + 1) / 2 + J; }

struct SmallLayout {
  int T, Tv;        // tile rows (n_pad + r_pad)/8, V tile columns n_pad/8
  int npad;         // 8⌈n/8⌉
  int off_tab, off_sites, off_w, off_dlog, off_misc;  // doubles
};

// A/B fragment (k-step kk) of tile X
__device__ __forceinline__ double frag_ab(const double* X, int lane, int kk) {
  return X[toff(lane >> 2, 4 * kk + (lane & 3))];
}

// The lead warp: factor the 8×8 diagonal tile (stored as −A) and write −W = −L⁻¹ into
// Wn and the pivots into piv; a pivot ≤ tol sets *bad.  Every lane holds the whole lower
// triangle (broadcast loads) and factors it redundantly: no shuffles, so the only serial
// chain is rsqrt → scale → update of the next pivot (≈ 90 cycles per pivot; the
// one-row-per-lane version with shuffles took ≈ 2,200 cycles per tile).  Lane l carries
// column l of W = L⁻¹ along in axpy form (x ← e_l; after pivot m: x_m /= L_mm, x_i −=
// L_im x_m), which consumes column m of L right after it is formed, so the registers of
// the factored columns are free again.
__device__ __forceinline__ void factor8(const double* Skk, double* Wn, double* piv, double tol,
                                        int* bad) {
  const int lane = threadIdx.x & 31, l = lane & 7;
  double a[36];  // a[i(i+1)/2 + j] = A_ij, j ≤ i
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) a[i * (i + 1) / 2 + j] = -Skk[toff(i, j)];
  int fail = 0;
  double mypiv = 1.0;
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (i == l) ? 1.0 : 0.0;
#if LIK_SMALL_PIV2
  // two pivots per step: for the 2×2 block [[d0, e], [e, f]] both reciprocal square roots
  // (1/L_cc = rsqrt(d0), 1/L_c1c1 = √d0 · rsqrt(d0 f − e²)) issue together, so the
  // chain carries 4 rsqrt latencies per tile instead of 8
#define A_(i, j) a[(i) * ((i) + 1) / 2 + (j)]
#pragma unroll
  for (int c = 0; c < 8; c += 2) {
    const int c1 = c + 1;
    const double d0 = A_(c, c), e = A_(c1, c), f = A_(c1, c1);
    const double det = fma(d0, f, -e * e);
    const double r0 = rsqrt(d0), rd = rsqrt(det);
    const double d1 = det * (r0 * r0);  // the second pivot, det / d0
    fail |= !(d0 > tol) || !(d1 > tol);
    if (l == c) mypiv = d0;
    if (l == c1) mypiv = d1;
    const double l10 = e * r0;           // L_c1c
    const double r1 = rd * (d0 * r0);    // 1 / L_c1c1
#pragma unroll
    for (int i = c1 + 1; i < 8; ++i) {
      A_(i, c) *= r0;                                  // L_ic
      A_(i, c1) = (A_(i, c1) - A_(i, c) * l10) * r1;  // L_ic1
    }
#pragma unroll
    for (int i = c1 + 1; i < 8; ++i)
#pragma unroll
      for (int j = c1 + 1; j <= i; ++j) A_(i, j) -= A_(i, c) * A_(j, c) + A_(i, c1) * A_(j, c1);
    // W column l: forward substitution in axpy form
    x[c] *= r0;
    x[c1] = (x[c1] - l10 * x[c]) * r1;
#pragma unroll
    for (int i = c1 + 1; i < 8; ++i) x[i] -= A_(i, c) * x[c] + A_(i, c1) * x[c1];
  }
#undef A_
#else
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double d = a[c * (c + 1) / 2 + c];
    fail |= !(d > tol);
    const double r = rsqrt(d);
    if (l == c) mypiv = d;
#pragma unroll
    for (int i = c + 1; i < 8; ++i) a[i * (i + 1) / 2 + c] *= r;  // column c of L (below the diagonal)
#pragma unroll
    for (int i = c + 1; i < 8; ++i)
#pragma unroll
      for (int j = c + 1; j <= i; ++j) a[i * (i + 1) / 2 + j] -= a[i * (i + 1) / 2 + c] * a[j * (j + 1) / 2 + c];
    // W column l: x_c = x_c / L_cc, then x_i −= L_ic x_c
    x[c] *= r;
#pragma unroll
    for (int i = c + 1; i < 8; ++i) x[i] -= a[i * (i + 1) / 2 + c] * x[c];
  }
#endif
  if (lane < 8) {
#pragma unroll
    for (int m = 0; m < 8; ++m) Wn[toff(m, l)] = -x[m];
    piv[l] = mypiv;
  }
  if (lane == 0 && fail) *bad = 1;
}

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    chol_small_kernel(CholArgs A, SmallLayout Lt, const double* __restrict__ coords,
                      const double* __restrict__ Bt, int ldb, const double* __restrict__ table,
                      cudaTextureObject_t table_tex) {
  constexpr int NW = NT / 32, LEAD = NW - 1;
  constexpr int CHEB_STRIDE = Cheb<1>::STRIDE;
  extern __shared__ __align__(16) double sm[];
  double* S = sm;
  double* coef = sm + Lt.off_tab;
  double2* sxy = reinterpret_cast<double2*>(sm + Lt.off_sites);
  double* Wn = sm + Lt.off_w;  // −W of the column being solved (8×8 tile)
  double* dlog = sm + Lt.off_dlog;
  double* scal = sm + Lt.off_misc;
  double* etab = scal + 8;
  int* flag = reinterpret_cast<int*>(etab + 16);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = A.k0 + blockIdx.x;
  SPH_INIT();
  const PointConst P = A.pc[k];
  const int n = A.g.n, r = A.g.r, T = Lt.T, Tv = Lt.Tv;
  if (P.mode == MODE_BAD) {
    point_failure(A, k, LIK_PT_BAD_PARAM, tid, NT);
    return;
  }
  // ---- load the point's table, the sites, exp2 table
  const int ezo = P.e_zero - CHEB_ELO;
  const int olo = P.olo, oz = max(olo, min(P.ohi, ezo));
  const unsigned span = ezo <= P.ohi ? 0x7fffffffu : (unsigned)(P.ohi - olo);
  if (P.mode == MODE_BESSEL) {
    const double2* src = reinterpret_cast<const double2*>(table + (size_t)blockIdx.x * Cheb<1>::TABLE_D);
    double2* dst = reinterpret_cast<double2*>(coef);
    for (int e = olo * CHEB_STRIDE / 2 + tid; e < (oz + 1) * CHEB_STRIDE / 2; e += NT) dst[e] = src[e];
  }
  for (int i = tid; i < n; i += NT) sxy[i] = reinterpret_cast<const double2*>(coords)[i];
  if (tid < 16) etab[tid] = kExp2Tab[tid];
  if (tid < 4) flag[tid] = 0;
  __syncthreads();

  SPH(0);
  // ---- Step 1: S = −A (lower tile triangle).  Each warp fills two tiles per pass (four
  // independent table evaluations per lane: the chains of coefficient loads and FMAs
  // overlap)
  const int ntile = T * (T + 1) / 2;
  const int ea = lane >> 3, eb = lane & 7;  // this lane's elements (ea, eb) and (ea + 4, eb) of a tile
  for (int t0 = warp; t0 < ntile; t0 += 2 * NW) {
    int I[2], J[2];
    bool on[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int t = min(t0 + q * NW, ntile - 1);
      on[q] = t0 + q * NW < ntile;
      int ii = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
      while (tri8(ii + 1, 0) <= t) ++ii;
      while (tri8(ii, 0) > t) --ii;
      I[q] = ii;
      J[q] = t - tri8(ii, 0);
    }
    double hx[4], hy[4], rho[4] = {0.5, 0.5, 0.5, 0.5};
    unsigned slow = 0u;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = 8 * J[q] + eb;
      const double2 sj = j < n ? sxy[j] : make_double2(0.0, 0.0);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = 8 * I[q] + ea + 4 * e;
        const double2 si = i < n ? sxy[i] : make_double2(0.0, 0.0);
        hx[2 * q + e] = si.x - sj.x;
        hy[2 * q + e] = si.y - sj.y;
      }
    }
    const bool vtile = I[0] < Tv || I[1] < Tv;
#ifdef LIK_SMALL_NO_RHO  // timing experiment only: results are wrong
    if (false) {
#else
    if (vtile) {
#endif
      if (P.mode == MODE_BESSEL) {
#if LIK_BUILD_TEXMASK
        // some coefficient pairs through the texture path (see matern_rho.cuh)
        matern_rho_tableN_tex<4, 1>(P, table_tex, (long long)blockIdx.x * (Cheb<1>::TABLE_D / 2), coef, etab,
                                    olo, oz, span, hx, hy, rho, slow, 0);
#else
        matern_rho_tableN<4, 1>(P, coef, etab, olo, oz, span, hx, hy, rho, slow, 0);
#endif
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) rho[e] = exp(-2.0 * aniso_d2(P, hx[e], hy[e]));
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!on[q]) continue;
      double* X = S + (t0 + q * NW) * 64;
      const int j = 8 * J[q] + eb;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = 8 * I[q] + ea + 4 * e, x = 2 * q + e;
        double v;
        if (I[q] < Tv) {
          if (i >= n || j >= n)
            v = (i == j) ? -1.0 : 0.0;
          else if (j > i)
            v = 0.0;
          else if (i == j)
            v = -(1.0 + P.nugget);
          else
            v = ((slow >> x) & 1u) ? -matern_rho_exact(P, hx[x], hy[x]) : -rho[x];
        } else {
          const int tr = 8 * (I[q] - Tv) + ea + 4 * e;
          v = (J[q] < Tv && tr < r && j < n) ? -Bt[(size_t)tr * ldb + j] : 0.0;
        }
        X[toff(ea + 4 * e, eb)] = v;
      }
    }
  }
  __syncthreads();
  SPH(1);
#ifdef LIK_SMALL_EXIT_AFTER_BUILD  // timing experiment only: results are wrong
  if (tid < 1000000) return;
#endif
  // ---- Steps 2-4: right-looking elimination of the Tv V tile columns, two tile columns
  // (a 16-column panel) per step: every trailing tile then takes 4 DMMAs per load and
  // store of its accumulator (shared-memory traffic per DMMA −33 % against one column
  // per step; with one column the updates saturated the shared-memory bandwidth and the
  // lead's loads queued behind them).
  // Roles by SM sub-partition (warp w issues on SMSP w mod 4): the lead (warp NW−1,
  // SMSP 3) runs the pivot chain, whose dependent FP64 operations would otherwise queue
  // behind other warps' DMMAs on the sub-partition's FP64 pipe (a DMMA-issuing
  // neighbour on the same SMSP starves it completely, tools/phase0/chain_bench.cu); so no
  // other warp of SMSP 3 issues DMMAs during the elimination.  G = the lead and warps
  // NW−4..NW−2 (SMSPs 0-2): at step p they bring the next panel up to date with panel p,
  // the lead factors its 16×16 diagonal block (two 8×8 tiles in registers, the solve and
  // update between them by DMMA), and after a named barrier the other three solve the
  // panel's rows below.  U = the warps below NW−4 on SMSPs 0-2: they apply panel p to
  // the columns beyond the next panel.  One CTA barrier per step.
  const double tol = n * DBL_EPSILON * (1.0 + P.nugget);
  const int co = toff(lane >> 2, 2 * (lane & 3));
  constexpr int NG = 4, NU = (NW - NG) / 4 * 3;
  const bool in_g = warp >= NW - NG;
  const int g = warp - (NW - NG);  // 0..3 in G; g = 3 is the lead
  const bool in_u = !in_g && (warp & 3) != 3;
  const int uw = (warp >> 2) * 3 + (warp & 3);  // U index 0..NU−1
  double* Wa = Wn;
  double* Wb = Wn + 64;
  auto tile = [&](int i, int j) { return S + tri8(i, j) * 64; };
  // X ← X (−W)ᵀ in place (the solve L_ij = A_ij L_jj⁻ᵀ with S = −A and Wn = −L_jj⁻¹)
  auto solve_tile = [&](double* X, const double* W) {
    const double x0 = frag_ab(X, lane, 0), x1 = frag_ab(X, lane, 1);
    const double w0 = frag_ab(W, lane, 0), w1 = frag_ab(W, lane, 1);
    double c[2] = {0.0, 0.0};
    dmma8(c, x0, w0);
    dmma8(c, x1, w1);
    __syncwarp();
    *reinterpret_cast<double2*>(X + co) = make_double2(c[0], c[1]);
    __syncwarp();
  };
  // C += L_a Lbᵀ (one 8×8 product, two DMMAs)
  auto upd_tile = [&](double* C, const double* La, const double* Lb) {
    const double a0 = frag_ab(La, lane, 0), a1 = frag_ab(La, lane, 1);
    const double b0 = frag_ab(Lb, lane, 0), b1 = frag_ab(Lb, lane, 1);
    const double2 cv = *reinterpret_cast<const double2*>(C + co);
    double c[2] = {cv.x, cv.y};
    dmma8(c, a0, b0);
    dmma8(c, a1, b1);
    *reinterpret_cast<double2*>(C + co) = make_double2(c[0], c[1]);
    __syncwarp();
  };
  auto g_bar = []() { asm volatile("bar.sync 1, %0;" ::"n"(NG * 32) : "memory"); };
  // G, part 2 for the panel starting at column a (a < Tv): the lead factors the
  // diagonal block; after the named barrier the other G warps solve rows ≥ a + 2
  auto g_factor_solve = [&](int a) {
    const int b = a + 1;  // b < T always (the B rows follow the V rows)
    // (a single-column panel, b ≥ Tv: column b is a Schur column and gets column a's
    // contribution from the step loop with the rest of the panel's update)
#if LIK_SMALL_REGCHAIN
    // Products whose left operand was just computed take it from the registers: with the
    // k order of an 8×8 product permuted so that k-step e covers the columns 2t + e (t =
    // lane mod 4), an operand in the accumulator layout (lane: row lane/4, columns 2t and
    // 2t + 1) is its own A fragment — and, for X·Xᵀ, its own B fragment; a B operand in
    // shared memory is read in the same order (bperm).  No store → load round trip
    // between the dependent products of a row.
    auto bperm = [&](const double* Y, int e) { return Y[toff(lane >> 2, 2 * (lane & 3) + e)]; };
    if (g == NG - 1) {
      factor8(tile(a, a), Wa, dlog + 8 * a, tol, &flag[0]);
      __syncwarp();
      double* Tba = tile(b, a);
      double l[2] = {0.0, 0.0};  // L_ba = S_ba (−W_aa)ᵀ
      {
        const double x0 = frag_ab(Tba, lane, 0), x1 = frag_ab(Tba, lane, 1);
        const double w0 = frag_ab(Wa, lane, 0), w1 = frag_ab(Wa, lane, 1);
        dmma8(l, x0, w0);
        dmma8(l, x1, w1);
      }
      __syncwarp();
      *reinterpret_cast<double2*>(Tba + co) = make_double2(l[0], l[1]);
      if (b < Tv) {
        double* Tbb = tile(b, b);  // S_bb += L_ba L_baᵀ, both operands from the registers
        const double2 cv = *reinterpret_cast<const double2*>(Tbb + co);
        double c[2] = {cv.x, cv.y};
        dmma8(c, l[0], l[0]);
        dmma8(c, l[1], l[1]);
        *reinterpret_cast<double2*>(Tbb + co) = make_double2(c[0], c[1]);
        __syncwarp();
        factor8(Tbb, Wb, dlog + 8 * b, tol, &flag[0]);
      } else {
        __syncwarp();
      }
    }
    SPH(8);
    g_bar();
    SPH(9);
    if (g < NG - 1) {
      const double* Tba = tile(b, a);
      double lb0 = 0.0, lb1 = 0.0, wb0 = 0.0, wb1 = 0.0;
      if (b < Tv) {
        lb0 = bperm(Tba, 0);
        lb1 = bperm(Tba, 1);
        wb0 = bperm(Wb, 0);
        wb1 = bperm(Wb, 1);
      }
      const double wa0 = frag_ab(Wa, lane, 0), wa1 = frag_ab(Wa, lane, 1);
      for (int i = a + 2 + g; i < T; i += NG - 1) {
        double* Tia = tile(i, a);
        double* Tib = tile(i, b);
        const double x0 = frag_ab(Tia, lane, 0), x1 = frag_ab(Tia, lane, 1);
        double2 cv = make_double2(0.0, 0.0);
        if (b < Tv) cv = *reinterpret_cast<const double2*>(Tib + co);
        double l[2] = {0.0, 0.0};  // L_ia = S_ia (−W_aa)ᵀ
        dmma8(l, x0, wa0);
        dmma8(l, x1, wa1);
        __syncwarp();
        *reinterpret_cast<double2*>(Tia + co) = make_double2(l[0], l[1]);
        if (b < Tv) {
          double c[2] = {cv.x, cv.y};  // S_ib += L_ia L_baᵀ
          dmma8(c, l[0], lb0);
          dmma8(c, l[1], lb1);
          double o[2] = {0.0, 0.0};    // L_ib = S_ib (−W_bb)ᵀ
          dmma8(o, c[0], wb0);
          dmma8(o, c[1], wb1);
          *reinterpret_cast<double2*>(Tib + co) = make_double2(o[0], o[1]);
        }
        __syncwarp();
      }
    }
#else
    if (g == NG - 1) {
      factor8(tile(a, a), Wa, dlog + 8 * a, tol, &flag[0]);
      __syncwarp();
      solve_tile(tile(b, a), Wa);
      if (b < Tv) {
        upd_tile(tile(b, b), tile(b, a), tile(b, a));
        factor8(tile(b, b), Wb, dlog + 8 * b, tol, &flag[0]);
      }
    }
    SPH(8);
    g_bar();
    SPH(9);
    if (g < NG - 1) {
      for (int i = a + 2 + g; i < T; i += NG - 1) {
        solve_tile(tile(i, a), Wa);
        if (b < Tv) {
          upd_tile(tile(i, b), tile(i, a), tile(b, a));
          solve_tile(tile(i, b), Wb);
        }
      }
    }
#endif
  };
  if (in_g) g_factor_solve(0);  // panel 0
  __syncthreads();
  SPH(2);
  for (int c0 = 0; c0 < Tv; c0 += 2) {
    const int c1 = c0 + 1;
    const bool two = c1 < Tv;        // panel columns c0 (and c1)
    const int a = c0 + (two ? 2 : 1);  // the next panel's first column
    if (in_g) {
      // (1) columns a, a+1 (those < T) += panel (c0, c1), rows ≥ column; the lead takes
      // the diagonal block, the other G warps the rows ≥ a + 2
      if (a < T) {
        const int b = a + 1;  // < T when a < Tv; may be ≥ T only for a Schur column a
        const int npc = two ? 2 : 1;
        // fragments of the panel's rows a and b (the B operands of every update below)
        double fa[2][2], fb[2][2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int c = q == 0 ? c0 : c1;
          if (q < npc) {
            fa[q][0] = frag_ab(tile(a, c), lane, 0);
            fa[q][1] = frag_ab(tile(a, c), lane, 1);
            if (b < T) {
              fb[q][0] = frag_ab(tile(b, c), lane, 0);
              fb[q][1] = frag_ab(tile(b, c), lane, 1);
            }
          }
        }
        if (g == NG - 1) {
          // the diagonal block (a, a), (b, a), (b, b): three independent accumulators
          double acc[3][2];
          const int nt3 = b < T ? 3 : 1;
          double* C3[3] = {tile(a, a), b < T ? tile(b, a) : nullptr, b < T ? tile(b, b) : nullptr};
#pragma unroll
          for (int t = 0; t < 3; ++t)
            if (t < nt3) {
              const double2 cv = *reinterpret_cast<const double2*>(C3[t] + co);
              acc[t][0] = cv.x;
              acc[t][1] = cv.y;
            }
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
              if (q < npc) {
                dmma8(acc[0], fa[q][kk], fa[q][kk]);
                if (nt3 == 3) {
                  dmma8(acc[1], fb[q][kk], fa[q][kk]);
                  dmma8(acc[2], fb[q][kk], fb[q][kk]);
                }
              }
#pragma unroll
          for (int t = 0; t < 3; ++t)
            if (t < nt3) *reinterpret_cast<double2*>(C3[t] + co) = make_double2(acc[t][0], acc[t][1]);
        } else {
          // rows i ≥ a + 2: tiles (i, a) and (i, b), two independent accumulators
          for (int i = a + 2 + g; i < T; i += NG - 1) {
            double acc[2][2];
            double* Ca = tile(i, a);
            double* Cb = tile(i, b);
            double2 cv = *reinterpret_cast<const double2*>(Ca + co);
            acc[0][0] = cv.x;
            acc[0][1] = cv.y;
            cv = *reinterpret_cast<const double2*>(Cb + co);
            acc[1][0] = cv.x;
            acc[1][1] = cv.y;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              if (q < npc) {
                const double* Li = tile(i, q == 0 ? c0 : c1);
                const double l0 = frag_ab(Li, lane, 0), l1 = frag_ab(Li, lane, 1);
                dmma8(acc[0], l0, fa[q][0]);
                dmma8(acc[1], l0, fb[q][0]);
                dmma8(acc[0], l1, fa[q][1]);
                dmma8(acc[1], l1, fb[q][1]);
              }
            }
            *reinterpret_cast<double2*>(Ca + co) = make_double2(acc[0][0], acc[0][1]);
            *reinterpret_cast<double2*>(Cb + co) = make_double2(acc[1][0], acc[1][1]);
          }
        }
        // (2)-(3) factor and solve the next panel
        if (a < Tv) {
          __syncwarp();
          SPH(3);
          g_factor_solve(a);
          SPH(4);
        }
      }
    } else if (in_u) {
      // U: S_ij += L_i,c0 L_j,c0ᵀ (+ L_i,c1 L_j,c1ᵀ) for the tiles j_lo ≤ j ≤ i, j_lo = a + 2,
      // taken row by row as one flat sequence split into NU equal contiguous ranges (balanced
      // to ±1 tile); UCH tiles of a row at a time (independent accumulators between a
      // tile's DMMAs, the row's L fragments reused)
      constexpr int UCH = LIK_SMALL_UCH;
      const int j_lo = a + 2;
      const int mrows = T - j_lo;
      if (mrows > 0) {
        const int ntu = mrows * (mrows + 1) / 2;
        int tau = (int)((long long)ntu * uw / NU);
        const int tau_end = (int)((long long)ntu * (uw + 1) / NU);
        // flat index → (i, j): row i = j_lo + ri holds ri + 1 tiles, starting at ri(ri+1)/2
        int ri = (int)((sqrtf(8.0f * tau + 1.0f) - 1.0f) * 0.5f);
        while ((ri + 1) * (ri + 2) / 2 <= tau) ++ri;
        while (ri * (ri + 1) / 2 > tau) --ri;
        int j = j_lo + (tau - ri * (ri + 1) / 2);
        while (tau < tau_end) {
          const int i = j_lo + ri;
          const int cnt = min(min(UCH, i - j + 1), tau_end - tau);
          const double* L0 = tile(i, c0);
          const double a00 = frag_ab(L0, lane, 0), a01 = frag_ab(L0, lane, 1);
          double a10 = 0.0, a11 = 0.0;
          if (two) {
            const double* L1 = tile(i, c1);
            a10 = frag_ab(L1, lane, 0);
            a11 = frag_ab(L1, lane, 1);
          }
          double bq[UCH][2], cq[UCH][2];
#pragma unroll
          for (int q = 0; q < UCH; ++q) {
            if (q < cnt) {
              const double* B0 = tile(j + q, c0);
              bq[q][0] = frag_ab(B0, lane, 0);
              bq[q][1] = frag_ab(B0, lane, 1);
              const double2 cv = *reinterpret_cast<const double2*>(tile(i, j + q) + co);
              cq[q][0] = cv.x;
              cq[q][1] = cv.y;
            }
          }
#pragma unroll
          for (int q = 0; q < UCH; ++q)
            if (q < cnt) dmma8(cq[q], a00, bq[q][0]);
#pragma unroll
          for (int q = 0; q < UCH; ++q)
            if (q < cnt) dmma8(cq[q], a01, bq[q][1]);
          if (two) {
            // (the second column's fragments loaded after the first column's DMMAs: loading
            // them up front costs registers, and the spills cost more than the latency)
#pragma unroll
            for (int q = 0; q < UCH; ++q) {
              if (q < cnt) {
                const double* B1 = tile(j + q, c1);
                bq[q][0] = frag_ab(B1, lane, 0);
                bq[q][1] = frag_ab(B1, lane, 1);
              }
            }
#pragma unroll
            for (int q = 0; q < UCH; ++q)
              if (q < cnt) dmma8(cq[q], a10, bq[q][0]);
#pragma unroll
            for (int q = 0; q < UCH; ++q)
              if (q < cnt) dmma8(cq[q], a11, bq[q][1]);
          }
#pragma unroll
          for (int q = 0; q < UCH; ++q)
            if (q < cnt) *reinterpret_cast<double2*>(tile(i, j + q) + co) = make_double2(cq[q][0], cq[q][1]);
          tau += cnt;
          j += cnt;
          if (j > i) {
            ++ri;
            j = j_lo;
          }
        }
      }
    }
    SPH(5);
    __syncthreads();
    SPH(6);
  }

  if (flag[0]) {
    point_failure(A, k, LIK_PT_V_NOT_PD, tid, NT);
    return;
  }
  // log|V| = Σ log pivots (Step 2): per lane the log of the product of its ≤ 7 pivots
  // (each in [n·ε·(1 + ν²), 1 + ν²]: no overflow or underflow; one log on the chain instead
  // of seven), then a fixed butterfly (deterministic)
  double logdet = 0.0;
  if (warp == LEAD) {
    double pr = 1.0;
    for (int i = lane; i < n; i += 32) pr *= dlog[i];
    double s = log(pr);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    logdet = s;
  }
  // ssqYX = BᵀV⁻¹B: the Schur block (rows / columns ≥ n_pad) of S, mirrored; Cm and Q
  // take the table / sites memory (no longer read)
  double* Cm = coef;
  double* Q = Cm + r * r;
  for (int e = tid; e < r * r; e += NT) {
    const int a = e / r, b = e % r, hi = max(a, b), lo = min(a, b);
    Cm[e] = S[tri8(Tv + hi / 8, Tv + lo / 8) * 64 + toff(hi & 7, lo & 7)];
  }
  __syncthreads();
  point_epilogue(A, k, Cm, r, Q, A.p, logdet, flag, scal, tid, NT, LEAD * 32, Q + A.p * A.p);
  SPH(7);
  SPH_FLUSH(LEAD, 0);
  SPH_FLUSH(0, 1);
  SPH_FLUSH(NW - 4, 2);
}

}  // namespace

#ifdef LIK_PHASE_TIMERS
extern "C" int lik_debug_small_phase_cycles(unsigned long long* out36, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out36, g_lik_small_phase, sizeof(unsigned long long) * 36);
  if (reset) {
    unsigned long long z[36] = {0};
    cudaMemcpyToSymbol(g_lik_small_phase, z, sizeof z);
  }
  return 0;
}
#endif

constexpr int SMALL_NMAX = 216;  // rows of the augmented matrix (n_pad + r_pad) the small path takes

static SmallLayout small_layout(int n, int r, int p) {
  SmallLayout L;
  L.npad = (n + 7) & ~7;
  const int rpad = (r + 7) & ~7;
  L.T = (L.npad + rpad) / 8;
  L.Tv = L.npad / 8;
  int off = L.T * (L.T + 1) / 2 * 64;
  L.off_tab = off;
  off += Cheb<1>::TABLE_D + 2 * n;  // table, then the sites
  L.off_sites = L.off_tab + Cheb<1>::TABLE_D;
  // Cm (r×r), Q (p×p) and the c / β̂ rows of the epilogue alias the table and the sites
  off = std::max(off, L.off_tab + r * r + p * p + 2 * r * p);  // + the epilogue's c, β̂ rows
  off = (off + 1) & ~1;
  L.off_w = off;
  off += 128;
  L.off_dlog = off;
  off += L.npad;
  L.off_misc = off;  // scal (8), etab (16), flags (4 ints)
  return L;
}

static size_t small_smem_bytes(const SmallLayout& L) { return (size_t)(L.off_misc + 8 + 16 + 2) * sizeof(double); }

bool small_path_fits(int n, int r, int p) {
  const SmallLayout L = small_layout(n, r, p);
  return cheb_sub_for(n) == 1 && 8 * L.T <= SMALL_NMAX && small_smem_bytes(L) <= 227 * 1024;
}

cudaError_t launch_chol_small(const CholArgs& a, const double* coords, const double* Bt, int ldb,
                              const double* table, cudaTextureObject_t table_tex, int kw, cudaStream_t st) {
  const SmallLayout L = small_layout(a.g.n, a.g.r, a.p);
  const size_t smem = small_smem_bytes(L);
  cudaError_t e;
#ifndef LIK_SMALL_NT1
#define LIK_SMALL_NT1 512  // threads of a CTA when one fits per SM
#endif
#ifndef LIK_SMALL_NT2
#define LIK_SMALL_NT2 256  // threads of each CTA when two fit per SM
#endif
  constexpr int NT1 = LIK_SMALL_NT1, NT2 = LIK_SMALL_NT2;
  static_assert(NT1 >= 256 && NT2 >= 256, "the panel group takes four warps, the update group needs more");
  if (smem <= 113 * 1024) {  // two CTAs per SM: one's pivot chain beside the other's updates
    e = cudaFuncSetAttribute(chol_small_kernel<NT2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    chol_small_kernel<NT2, 2><<<kw, NT2, smem, st>>>(a, L, coords, Bt, ldb, table, table_tex);
  } else {
    e = cudaFuncSetAttribute(chol_small_kernel<NT1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    chol_small_kernel<NT1, 1><<<kw, NT1, smem, st>>>(a, L, coords, Bt, ldb, table, table_tex);
  }
  return cudaGetLastError();
}

}  // namespace lik
