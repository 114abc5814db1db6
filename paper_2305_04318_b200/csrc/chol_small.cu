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
// Right-looking elimination, one 8-column tile column k per step, with lookahead:
//   phase A (all warps):  L_ik = A_ik L_kk⁻ᵀ = S_ik (−W_k)ᵀ for the tiles below the
//                         diagonal (W_k = L_kk⁻¹ from the previous phase);
//   phase B: the lead warp updates tile (k+1, k+1), factors it in registers (one
//            rsqrt per pivot, the 8 pivots the only serial chain) and inverts it
//            (−W_{k+1}); the other warps update every other trailing tile,
//            S_ij += L_ik L_jkᵀ, in row blocks of up to 4 tiles (L_ik reused).
// Two CTA barriers per step.  The pivot chain of step k+1 runs beside the trailing
// update of step k.
#include <cfloat>
#include <algorithm>
#include <cstdint>
#include "../../include/lik.h"
#include "lik_internal.cuh"
#include "matern_rho.cuh"
#include "point_epilogue.cuh"

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

// The lead warp: factor the 8×8 diagonal tile (stored as −A), one row per lane
// (lanes 8-31 mirror lanes 0-7), and write −W = −L⁻¹ into Wn and the pivots into piv.
// A pivot ≤ tol sets *bad.
__device__ __forceinline__ void factor8(const double* Skk, double* Wn, double* piv, double tol,
                                        int* bad) {
  const int lane = threadIdx.x & 31, l = lane & 7;
  double a[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) a[m] = (m <= l) ? -Skk[toff(l, m)] : 0.0;
  int fail = 0;
  double my_piv = 1.0, my_rinv = 1.0;
  double piv_next = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double pv = piv_next;
    fail |= !(pv > tol);
    const double rinv = rsqrt(pv);
    if (l == c) {
      a[c] = pv * rinv;
      my_piv = pv;
      my_rinv = rinv;
    } else if (l > c) {
      a[c] *= rinv;
    }
    if (c + 1 < 8) {  // the next pivot from lane c+1's own update, broadcast once
      const double pn = a[c + 1] - a[c] * a[c];
      piv_next = __shfl_sync(0xffffffffu, pn, c + 1);
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      if (m > c) {
        const double lm = __shfl_sync(0xffffffffu, a[c], m);
        if (l >= m) a[m] -= a[c] * lm;
      }
    }
  }
  // column l of W = L⁻¹ by forward substitution (x = e_l)
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (i == l) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] *= __shfl_sync(0xffffffffu, my_rinv, i);
#pragma unroll
    for (int m = 0; m < 8; ++m)
      if (m > i) x[m] -= __shfl_sync(0xffffffffu, a[i], m) * x[i];
  }
  if (lane < 8) {
#pragma unroll
    for (int m = 0; m < 8; ++m) Wn[toff(m, l)] = -x[m];
    piv[l] = my_piv;
  }
  if (lane == 0 && fail) *bad = 1;
}

// S_ij += L_ik L_jkᵀ for j = j0 .. j1 (one warp; L_ik's fragments reused)
__device__ __forceinline__ void update_row(double* S, int i, int k, int j0, int j1, int lane) {
  const double* Lik = S + tri8(i, k) * 64;
  const double a0 = frag_ab(Lik, lane, 0), a1 = frag_ab(Lik, lane, 1);
  const int co = toff(lane >> 2, 2 * (lane & 3));
  for (int j = j0; j <= j1; ++j) {
    const double* Ljk = S + tri8(j, k) * 64;
    double* C = S + tri8(i, j) * 64;
    double2 cv = *reinterpret_cast<const double2*>(C + co);
    double c[2] = {cv.x, cv.y};
    dmma8(c, a0, frag_ab(Ljk, lane, 0));
    dmma8(c, a1, frag_ab(Ljk, lane, 1));
    *reinterpret_cast<double2*>(C + co) = make_double2(c[0], c[1]);
  }
}

template <int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 1)
    chol_small_kernel(CholArgs A, SmallLayout Lt, const double* __restrict__ coords,
                      const double* __restrict__ Bt, int ldb, const double* __restrict__ table) {
  constexpr int NW = NT / 32, LEAD = NW - 1;
  constexpr int CHEB_STRIDE = Cheb<1>::STRIDE;
  extern __shared__ __align__(16) double sm[];
  double* S = sm;
  double* coef = sm + Lt.off_tab;
  double2* sxy = reinterpret_cast<double2*>(sm + Lt.off_sites);
  double* Wn = sm + Lt.off_w;  // two 8×8 tiles (−W, double-buffered by step parity)
  double* dlog = sm + Lt.off_dlog;
  double* scal = sm + Lt.off_misc;
  double* etab = scal + 8;
  int* flag = reinterpret_cast<int*>(etab + 16);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = A.k0 + blockIdx.x;
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

  // ---- Step 1: S = −A (lower tile triangle)
  const int ntile = T * (T + 1) / 2;
  const int ea = lane >> 3, eb = lane & 7;  // this lane's elements (ea, eb) and (ea + 4, eb)
  for (int t = warp; t < ntile; t += NW) {
    int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (tri8(I + 1, 0) <= t) ++I;
    while (tri8(I, 0) > t) --I;
    const int J = t - tri8(I, 0);
    double* X = S + t * 64;
    double v[2] = {0.0, 0.0};
    if (I < Tv) {
      const int j = 8 * J + eb;
      double hx[2], hy[2];
      const double2 sj = j < n ? sxy[j] : make_double2(0.0, 0.0);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = 8 * I + ea + 4 * e;
        const double2 si = i < n ? sxy[i] : make_double2(0.0, 0.0);
        hx[e] = si.x - sj.x;
        hy[e] = si.y - sj.y;
      }
      double rho[2];
      unsigned slow = 0u;
      if (P.mode == MODE_BESSEL) {
        matern_rho_tableN<2, 1>(P, coef, etab, olo, oz, span, hx, hy, rho, slow, 0);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) rho[e] = exp(-2.0 * aniso_d2(P, hx[e], hy[e]));
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = 8 * I + ea + 4 * e;
        if (i >= n || j >= n)
          v[e] = (i == j) ? -1.0 : 0.0;
        else if (j > i)
          v[e] = 0.0;
        else if (i == j)
          v[e] = -(1.0 + P.nugget);
        else
          v[e] = ((slow >> e) & 1u) ? -matern_rho_exact(P, hx[e], hy[e]) : -rho[e];
      }
    } else if (J < Tv) {
      const int j = 8 * J + eb;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tr = 8 * (I - Tv) + ea + 4 * e;
        v[e] = (tr < r && j < n) ? -Bt[(size_t)tr * ldb + j] : 0.0;
      }
    }
    X[toff(ea, eb)] = v[0];
    X[toff(ea + 4, eb)] = v[1];
  }
  __syncthreads();

  // ---- Steps 2-4: right-looking elimination of the Tv V tile columns
  const double tol = n * DBL_EPSILON * (1.0 + P.nugget);
  if (warp == LEAD) factor8(S, Wn, dlog, tol, &flag[0]);
  __syncthreads();
  const int co = toff(lane >> 2, 2 * (lane & 3));
  for (int kc = 0; kc < Tv; ++kc) {
    // phase A: L_ik = S_ik (−W_k)ᵀ, i > kc
    const double* W = Wn + (kc & 1) * 64;
    const double w0 = frag_ab(W, lane, 0), w1 = frag_ab(W, lane, 1);
    for (int i = kc + 1 + warp; i < T; i += NW) {
      double* X = S + tri8(i, kc) * 64;
      double c[2] = {0.0, 0.0};
      dmma8(c, frag_ab(X, lane, 0), w0);
      dmma8(c, frag_ab(X, lane, 1), w1);
      __syncwarp();
      *reinterpret_cast<double2*>(X + co) = make_double2(c[0], c[1]);
    }
    __syncthreads();
    // phase B: trailing update S_ij += L_i,kc L_j,kcᵀ, kc < j ≤ i
    if (kc + 1 < T) {
      if (warp == LEAD) {
        update_row(S, kc + 1, kc, kc + 1, kc + 1, lane);
        if (kc + 1 < Tv) {
          __syncwarp();
          factor8(S + tri8(kc + 1, kc + 1) * 64, Wn + ((kc + 1) & 1) * 64, dlog + 8 * (kc + 1), tol,
                  &flag[0]);
        }
      } else {
        // rows i ≥ kc+2, columns kc+1..i in blocks of 4; unit u → warp u mod (NW−1)
        int u = 0;
        for (int i = kc + 2; i < T; ++i) {
          for (int j0 = kc + 1; j0 <= i; j0 += 4, ++u) {
            if (u % (NW - 1) != warp) continue;
            update_row(S, i, kc, j0, min(j0 + 3, i), lane);
          }
        }
      }
    }
    __syncthreads();
  }

  if (flag[0]) {
    point_failure(A, k, LIK_PT_V_NOT_PD, tid, NT);
    return;
  }
  // log|V| = Σ log pivots (Step 2): per-lane partial sums in a fixed order, then a fixed
  // butterfly (deterministic)
  double logdet = 0.0;
  if (warp == LEAD) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += log(dlog[i]);
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
  point_epilogue(A, k, Cm, r, Q, A.p, logdet, flag, scal, tid, NT, LEAD * 32);
}

}  // namespace

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
  // Cm (r×r) and Q (p×p) of the epilogue alias the table and the sites
  off = std::max(off, L.off_tab + r * r + p * p);
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
                              const double* table, int kw, cudaStream_t st) {
  const SmallLayout L = small_layout(a.g.n, a.g.r, a.p);
  const size_t smem = small_smem_bytes(L);
  cudaError_t e;
  if (smem <= 113 * 1024) {  // two CTAs per SM: one's pivot chain beside the other's updates
    e = cudaFuncSetAttribute(chol_small_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    chol_small_kernel<256><<<kw, 256, smem, st>>>(a, L, coords, Bt, ldb, table);
  } else {
    e = cudaFuncSetAttribute(chol_small_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    chol_small_kernel<512><<<kw, 512, smem, st>>>(a, L, coords, Bt, ldb, table);
  }
  return cudaGetLastError();
}

}  // namespace lik
