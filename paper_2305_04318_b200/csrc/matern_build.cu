// Dataset prep (Box-Cox columns, Σ log y), per-point constants, and the
// Matérn tile build of the augmented matrix [[V, B], [Bᵀ, 0]].
//   prep_kernel   — a1: y'_m = b(y; λ_m) (R14), Bᵀ rows, S = Σ log y
//   setup_kernel  — per-point constants of ω_k (R1, R3, R7)
//   build_kernel  — a2 "matern_build": V = R + ν²I tiles (P:86, P:311 Step 1)
#include <algorithm>
#include <cfloat>
#include "matern_rho.cuh"
#include "lik_internal.cuh"

namespace lik {

// ---------------------------------------------------------------------------
// prep: grid = r + 2 blocks.  Block t < r writes row t of Bᵀ (r × npad,
// zero-padded); block r computes S = Σ log y_i with a fixed-order reduction;
// block r + 1 gathers the (possibly reordered) site coordinates.  Sites are
// taken in the order perm (Morton order chosen by the host for locality of the
// Matérn build); the likelihood is invariant under a symmetric permutation of
// the sites (with y and X rows).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) prep_kernel(const double* __restrict__ coords,
                                                   const double* __restrict__ y,
                                                   const double* __restrict__ X,
                                                   const double* __restrict__ lambdas,
                                                   const int* __restrict__ perm, int n, int p, int M,
                                                   int npad, double* __restrict__ coords_p,
                                                   double* __restrict__ Bt, double* __restrict__ S) {
  const int t = blockIdx.x;
  const int r = M + p;
  if (t < r) {
    for (int i = threadIdx.x; i < npad; i += blockDim.x) {
      double v = 0.0;
      if (i < n) {
        const int src = perm ? perm[i] : i;
        if (t < M) {
          const double lam = lambdas[t];
          const double ly = log(y[src]);
          v = (fabs(lam) < 1e-10) ? ly : expm1(lam * ly) / lam;
        } else {
          v = X[(size_t)src * p + (t - M)];
        }
      }
      Bt[(size_t)t * npad + i] = v;
    }
  } else if (t == r) {
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
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int src = perm ? perm[i] : i;
      coords_p[2 * i] = coords[2 * src];
      coords_p[2 * i + 1] = coords[2 * src + 1];
    }
  }
}

cudaError_t launch_prep(const double* coords, const double* y, const double* X,
                        const double* lambdas, const int* perm, int n, int p, int M, int npad,
                        double* coords_p, double* Bt, double* S, cudaStream_t st) {
  prep_kernel<<<M + p + 2, 256, 0, st>>>(coords, y, X, lambdas, perm, n, p, M, npad, coords_p, Bt, S);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// setup: one thread per parameter point.
// ---------------------------------------------------------------------------
__global__ void setup_kernel(const double* __restrict__ params, int K, PointConst* __restrict__ pc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const double phiX = params[5 * (size_t)k + 0], kappa = params[5 * (size_t)k + 1];
  const double nug = params[5 * (size_t)k + 2], phiR = params[5 * (size_t)k + 3];
  const double phiA = params[5 * (size_t)k + 4];
  PointConst P;
  bool ok = isfinite(phiX) && isfinite(kappa) && isfinite(nug) && isfinite(phiR) &&
            isfinite(phiA) && phiX > 0.0 && kappa > 0.0 && nug >= 0.0 && phiR > 0.0;
  P.mode = ok ? (kappa >= 1e3 ? MODE_GAUSS : MODE_BESSEL) : MODE_BAD;
  double c = 1.0, s = 0.0;
  if (ok) sincos(phiA, &s, &c);
  const double phiY = phiX / phiR;  // R3
  P.cX = c / phiX;
  P.sX = s / phiX;
  P.sY = s / phiY;
  P.cY = c / phiY;
  const double r8k = sqrt(8.0 * kappa);
  P.qX = r8k * P.cX;
  P.qS = r8k * P.sX;
  P.qT = r8k * P.sY;
  P.qY = r8k * P.cY;
  P.kappa = kappa;
  P.eightk = 8.0 * kappa;
  P.inv4k = 0.25 / kappa;
  P.nugget = nug;
  P.e_zero = 1 << 20;  // set by table_kernel
  P.olo = 0;
  P.ohi = CHEB_NOCT - 1;
  P.range_ok = 0;
  P.lnC = ok && P.mode == MODE_BESSEL ? matern_lnC(kappa) : 0.0;
  pc[k] = P;
}

cudaError_t launch_setup(const double* params, int K, PointConst* pc, cudaStream_t st) {
  setup_kernel<<<(K + 127) / 128, 128, 0, st>>>(params, K, pc);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// dist_range: min / max squared Euclidean distance over all site pairs.  Blocks
// reduce their share of the pairs and combine with 64-bit integer atomics on the
// IEEE bit patterns (for non-negative doubles they order like the values), so the
// result is exact and independent of the order.
// ---------------------------------------------------------------------------
__global__ void dist_init_kernel(double* __restrict__ dstat) {
  dstat[0] = INFINITY;
  dstat[1] = 0.0;
}

__global__ void __launch_bounds__(256) dist_range_kernel(const double* __restrict__ coords, int n,
                                                         double* __restrict__ dstat) {
  __shared__ double lo[256], hi[256];
  double mn = INFINITY, mx = 0.0;
  const long long np = (long long)n * (n - 1) / 2;
  for (long long e = (long long)blockIdx.x * 256 + threadIdx.x; e < np; e += (long long)gridDim.x * 256) {
    // pair e → (i, j), i > j, e = i(i−1)/2 + j
    int i = (int)((sqrt(8.0 * (double)e + 1.0) + 1.0) * 0.5);
    while ((long long)i * (i - 1) / 2 > e) --i;
    while ((long long)(i + 1) * i / 2 <= e) ++i;
    const int j = (int)(e - (long long)i * (i - 1) / 2);
    const double dx = coords[2 * i] - coords[2 * j], dy = coords[2 * i + 1] - coords[2 * j + 1];
    const double d2 = dx * dx + dy * dy;
    mn = fmin(mn, d2);
    mx = fmax(mx, d2);
  }
  lo[threadIdx.x] = mn;
  hi[threadIdx.x] = mx;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      lo[threadIdx.x] = fmin(lo[threadIdx.x], lo[threadIdx.x + w]);
      hi[threadIdx.x] = fmax(hi[threadIdx.x], hi[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicMin(reinterpret_cast<long long*>(&dstat[0]), __double_as_longlong(lo[0]));
    atomicMax(reinterpret_cast<long long*>(&dstat[1]), __double_as_longlong(hi[0]));
  }
}

cudaError_t launch_dist_range(const double* coords, int n, double* dstat, cudaStream_t st) {
  dist_init_kernel<<<1, 1, 0, st>>>(dstat);
  const long long np = (long long)n * (n - 1) / 2;
  // ~4 pairs per thread (a latency chain each: the pair index needs a square root)
  const int blocks = (int)std::max<long long>(1, std::min<long long>(1184, (np + 256 * 4 - 1) / (256 * 4)));
  dist_range_kernel<<<blocks, 256, 0, st>>>(coords, n, dstat);
  return cudaGetLastError();
}

// Monomial coefficients of the Chebyshev polynomials: kTco.v[j·N + k] = coefficient
// of t^k in T_j (T_0 = 1, T_1 = t, T_j = 2t T_{j−1} − T_{j−2}); integers, exact in FP64.
template <int N>
struct TcoTable {
  double v[N * N];
};
template <int N>
constexpr TcoTable<N> make_tco() {
  TcoTable<N> t{};
  t.v[0] = 1.0;
  t.v[N + 1] = 1.0;
  for (int jj = 2; jj < N; ++jj)
    for (int kk = 0; kk < N; ++kk)
      t.v[jj * N + kk] = (kk > 0 ? 2.0 * t.v[(jj - 1) * N + kk - 1] : 0.0) - t.v[(jj - 2) * N + kk];
  return t;
}
// The DCT-II matrices cos(π j (i + ½) / N) of the table layouts, written once per process
// by cheb_init_kernel (lik_create) instead of N² cospi per point in every table block.
template <int N>
struct CosTable {
  double v[N * N];
};
__device__ CosTable<Cheb<1>::N> g_cosm1;
__device__ CosTable<Cheb<CHEB_SUB_LARGE>::N> g_cosmL;
template <int N>
__device__ void fill_cos(CosTable<N>& t) {
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) t.v[e] = cospi((e / N) * ((e % N) + 0.5) / N);
}
__global__ void cheb_init_kernel() {
  fill_cos(g_cosm1);
  fill_cos(g_cosmL);
}
cudaError_t launch_cheb_init(cudaStream_t st) {
  cheb_init_kernel<<<1, 256, 0, st>>>();
  return cudaGetLastError();
}
__device__ const TcoTable<Cheb<1>::N> kTco1 = make_tco<Cheb<1>::N>();
__device__ const TcoTable<Cheb<CHEB_SUB_LARGE>::N> kTcoL = make_tco<Cheb<CHEB_SUB_LARGE>::N>();

// ---------------------------------------------------------------------------
// table: one block per point of the wave.  ln ρ is evaluated exactly (the
// Gamma-mixture quadrature of matern_rho.cuh) at the interval edges and at CHEB_N
// Chebyshev nodes of every interval (CHEB_SUB per binary octave of s = z²) below
// the underflow octave e_zero, detrended by the line through the edge values (so
// the DCT works on a small function) and turned into Chebyshev coefficients
// (DCT-II), then monomial ones with the line added back.  ln ρ(√s) is analytic on
// each interval (its only finite singularity is the branch point s = 0: 3
// half-widths from the centre of a whole octave, 5 from that of [1, 1.5)·2^e), so
// degree 19 resp. 15 reaches the FP64 rounding floor (~1e-16·max(1, |ln ρ|)),
// DESIGN.md §5.
//
// The nodes of a unit of octaves (three for SUB = 1, one for SUB = 2) share a quadrature
// grid: one warp per unit, one lane per node or interval edge (SUB = 1: 3 × (20 + 1) + 1
// = 64 = two passes of 32 lanes).  The grid step is the one of the unit's largest s (the
// finest: the peak's curvature κr grows with s), and the grid spans the union of the
// nodes' windows — from where G(·; s_min) falls 40 below its peak on the left (the
// smallest s has the longest left tail) to where G(·; s_max) does on the right.  Per grid node the warp computes
// A = κ(x − (e^x − 1)) and B = e^{−x}/(4κ) once (into shared memory), so each lane's
// G(x; s) = A − s·B costs one FMA and its term one exp.
// ---------------------------------------------------------------------------
#ifndef LIK_TABLE_NT
#define LIK_TABLE_NT 256  // threads per point (the octaves are spread over its warps)
#endif
constexpr int TABLE_NT = LIK_TABLE_NT;
#ifndef LIK_TABLE_UOCT
#define LIK_TABLE_UOCT 3  // octaves per shared quadrature grid in the whole-octave layout
#endif

template <int SUB>
__global__ void __launch_bounds__(TABLE_NT) table_kernel(PointConst* __restrict__ pc, int k0,
                                                    double* __restrict__ table,
                                                    const double* __restrict__ dstat) {
  constexpr int CHEB_SUB = SUB, CHEB_N = Cheb<SUB>::N, CHEB_STRIDE = Cheb<SUB>::STRIDE;
  constexpr int CHEB_NINT = Cheb<SUB>::NINT, TABLE_D = Cheb<SUB>::TABLE_D;
  const int k = k0 + blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const PointConst P = pc[k];
  if (P.mode != MODE_BESSEL) return;
  extern __shared__ double tsm[];  // dynamic: f and cheb (CHEB_NINT·CHEB_N doubles each)
  double* f = tsm;
  double* cheb = tsm + CHEB_NINT * CHEB_N;  // also the warps' quadrature scratch
  __shared__ double edge[CHEB_NINT + 1];
  __shared__ int ez, next_oct;
  __shared__ double etab[16];
  constexpr double kLog2e = 1.4426950408889634074;
  __shared__ double tco[CHEB_N * CHEB_N];   // tco[j][k] = coefficient of t^k in T_j
  __shared__ double cosm[CHEB_N * CHEB_N];  // cosm[j][i] = cos(π j (i + ½) / N), the DCT-II matrix
  if (tid < 16) etab[tid] = kExp2Tab[tid];
  if (tid == 0) next_oct = 0;
  for (int e = tid; e < CHEB_N * CHEB_N; e += TABLE_NT) {
    if constexpr (SUB == 1) {
      tco[e] = kTco1.v[e];
      cosm[e] = g_cosm1.v[e];
    } else {
      tco[e] = kTcoL.v[e];
      cosm[e] = g_cosmL.v[e];
    }
  }
  // This point's s = 8κ·|Q h|² lies in [8κ·d²min/φ²max, 8κ·d²max/φ²min] (the singular
  // values of the anisotropy map Q are 1/φX, 1/φY): only those octaves are built (for
  // SUB > 1 widened by one on each side); the build sends anything outside [olo, ohi]
  // to the exact evaluation.
  const double q_lo = fmin(P.cX * P.cX + P.sX * P.sX, P.sY * P.sY + P.cY * P.cY);
  const double q_hi = fmax(P.cX * P.cX + P.sX * P.sX, P.sY * P.sY + P.cY * P.cY);
  const double s_lo = P.eightk * dstat[0] * q_lo, s_hi = P.eightk * dstat[1] * q_hi;
  // (± one octave of margin where the build skips the range flags for points inside it,
  // range_ok; the whole-octave layout feeds the small path, which always flags, so it
  // builds just the octaves of [s_lo, s_hi] — 12 % fewer for the Swiss shape)
  constexpr int MARGIN = SUB == 1 ? 0 : 1;
  const int olo = s_lo > 0.0 ? max(0, min(CHEB_NOCT - 1, ilogb(s_lo) - CHEB_ELO - MARGIN)) : 0;
  const int ohi = s_hi > 0.0 ? max(olo, min(CHEB_NOCT - 1, ilogb(s_hi) - CHEB_ELO + MARGIN)) : olo;
  __syncthreads();  // etab, next_oct
  // ln ρ at the nodes (f, not yet detrended) and at the interval edges s = 2^(ELO + iv/SUB)
  // · (1 + (iv mod SUB)/SUB) (edge), all from the octave's shared quadrature grid
  {
    const double kap = P.kappa, i4k = P.inv4k;
    constexpr int QCAP = (CHEB_NINT * CHEB_N / (TABLE_NT / 32) / 2) / 32 * 32;  // grid chunk (scratch in cheb[])
    static_assert(QCAP >= 64, "grid scratch");
    double* qa = cheb + warp * 2 * QCAP;
    double* qb = qa + QCAP;
    constexpr int NODES = CHEB_SUB * CHEB_N;
    // a unit of UOCT consecutive octaves shares one quadrature grid: its slots are, per
    // octave, the NODES Chebyshev nodes and the SUB lower interval edges, then the top
    // edge of the unit's last octave (kept only at ohi, else it is the next unit's first
    // edge).  SUB = 1: 3 × 21 + 1 = 64 slots = two passes with every lane busy (one octave
    // per warp left 10 of 32 lanes idle), and the window search, the grid and the per-octave
    // setup once per three octaves; the grid of a unit is ~10 % longer than an octave's.
    constexpr int UOCT = CHEB_SUB == 1 ? LIK_TABLE_UOCT : 1;
    constexpr int PER = NODES + CHEB_SUB;
    constexpr int NSLOT = UOCT * PER + 1;
    constexpr int NPASS = (NSLOT + 31) / 32;
    // units handed out dynamically (their grids differ a lot in length); each unit's values
    // do not depend on which warp computes them (units start at olo + UOCT·u)
    for (;;) {
      int o0 = 0;
      if (lane == 0) o0 = olo + atomicAdd(&next_oct, UOCT);
      o0 = __shfl_sync(0xffffffffu, o0, 0);
      if (o0 > ohi) break;
      const int nu = min(UOCT, ohi - o0 + 1);  // octaves in this unit
      const int e = CHEB_ELO + o0;
      const double s0 = ldexp(1.0, e), s1 = ldexp(1.0, e + nu);
      double x0, x1, h0, h;
      quad_peak_step(kap, s0, x0, h0);
      quad_peak_step(kap, s1, x1, h);  // the finest step of the unit
      const double a0 = s0 * i4k, a1 = s1 * i4k;
      const double g0 = quad_G(kap, a0, x0), g1 = quad_G(kap, a1, x1);
      // left extent from the peak of s0, right extent from the peak of s1
      int L = 0, R = 0;
      for (int base = 0; base < kQuadMaxNodes; base += 32) {
        const unsigned bad = __ballot_sync(0xffffffffu, quad_G(kap, a0, x0 - (base + lane + 1) * h) - g0 < -kQuadCut);
        L = base + (bad ? __ffs(bad) - 1 : 32);
        if (bad) break;
      }
      for (int base = 0; base < kQuadMaxNodes; base += 32) {
        const unsigned bad = __ballot_sync(0xffffffffu, quad_G(kap, a1, x1 + (base + lane + 1) * h) - g1 < -kQuadCut);
        R = base + (bad ? __ffs(bad) - 1 : 32);
        if (bad) break;
      }
      const double xl = x0 - L * h;
      const int nq = L + (int)ceil((x1 - x0) / h) + R + 1;
      for (int pass = 0; pass < NPASS; ++pass) {
        // this lane's s: a Chebyshev node or a lower interval edge of octave o = o0 + oo
        // (oo < nu), or the unit's top edge (slot nu·PER: the lower edge of octave o0 + nu,
        // kept only when the unit ends at ohi)
        const int slot = pass * 32 + lane;
        const int oo = slot / PER, w = slot % PER;
        const int o = o0 + oo;
        const bool in_oct = oo < nu;
        const bool is_node = in_oct && w < NODES;
        const int eix = in_oct ? w - NODES : 0;
        const bool active = in_oct || (slot == nu * PER && o0 + nu - 1 == ohi);
        double sn;
        if (is_node) {
          const int part = w / CHEB_N, i = w % CHEB_N;
          sn = ldexp(1.0 + (double)part / CHEB_SUB + (0.5 / CHEB_SUB) * (1.0 + cosm[CHEB_N + i]), CHEB_ELO + o);
        } else {
          sn = ldexp(1.0 + (double)max(eix, 0) / CHEB_SUB, CHEB_ELO + o);
        }
        double xs, hs;
        quad_peak_step(kap, sn, xs, hs);
        const double gs = quad_G(kap, sn * i4k, xs), gs2 = kLog2e * gs;
        double sum = 0.0;
        for (int c0 = 0; c0 < nq; c0 += QCAP) {
          // the grid chunk (a grid that fits the scratch is generated once per unit, in the
          // first pass; a longer one chunk by chunk in every pass)
          if (pass == 0 || nq > QCAP) {
            __syncwarp();
            for (int j = lane; j < QCAP && c0 + j < nq; j += 32) {
              const double x = xl + (c0 + j) * h;
              double ex, em;
              quad_exp(x, ex, em);
              qa[j] = kLog2e * (kap * (x - em));  // base 2: the terms are 2^(G·log2 e)
              qb[j] = kLog2e * (i4k / ex);
            }
          }
          __syncwarp();
          const int cn = min(QCAP, nq - c0);
          if (active) {
            // four partial sums (independent exp chains), combined in a fixed order; the
            // table-driven 2^y (≤ 1 ulp; terms below 2^−1021 are 0, far below the e^−40 cut)
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
            int j = 0;
            for (; j + 4 <= cn; j += 4) {
#pragma unroll
              for (int u = 0; u < 4; ++u) s4[u] += exp2_neg(fma(-sn, qb[j + u], qa[j + u]) - gs2, etab);
            }
            for (; j < cn; ++j) s4[0] += exp2_neg(fma(-sn, qb[j], qa[j]) - gs2, etab);
            sum += (s4[0] + s4[1]) + (s4[2] + s4[3]);
          }
        }
        __syncwarp();
        const double lr = P.lnC + gs + log(h * sum);
        if (active) {
          if (is_node) {
            const int part = w / CHEB_N, i = w % CHEB_N;
            f[(o * CHEB_SUB + part) * CHEB_N + i] = lr;
          } else {
            edge[o * CHEB_SUB + eix] = lr;  // (the top edge: octave o0 + nu, eix 0)
          }
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    int e0 = CHEB_ELO + CHEB_NOCT + 64;  // sentinel: never underflows inside the table range
    for (int o = olo; o <= ohi + 1; ++o)
      if (edge[o * CHEB_SUB] < -750.0) {
        e0 = CHEB_ELO + o;
        break;
      }
    ez = e0;
    pc[k].e_zero = e0;
    pc[k].olo = olo;
    pc[k].ohi = ohi;
    // a full octave of margin on both sides (neither end clipped at the table's limits)
    pc[k].range_ok = s_lo >= ldexp(1.0, CHEB_ELO + olo + 1) && s_hi < ldexp(1.0, CHEB_ELO + ohi);
  }
  __syncthreads();
  // detrend: g = ln ρ − L_iv(x), L_iv the line through the interval's edge values
  for (int idx = olo * CHEB_SUB * CHEB_N + tid; idx < (ohi + 1) * CHEB_SUB * CHEB_N; idx += TABLE_NT) {
    const int iv = idx / CHEB_N, i = idx % CHEB_N;
    const double xc = cosm[CHEB_N + i];  // cos(π (i + ½) / N)
    f[idx] -= 0.5 * (edge[iv] + edge[iv + 1]) + 0.5 * (edge[iv + 1] - edge[iv]) * xc;
  }
  __syncthreads();
  // Chebyshev coefficients of g (DCT-II), then monomial coefficients in t (T_j has
  // integer coefficients, exact in FP64) so the build evaluates a plain Horner scheme.
  for (int idx = olo * CHEB_SUB * CHEB_N + tid; idx < (ohi + 1) * CHEB_SUB * CHEB_N; idx += TABLE_NT) {
    const int iv = idx / CHEB_N, jj = idx % CHEB_N;
    double cc = 0.0;
    if (CHEB_ELO + iv / CHEB_SUB < ez) {
      for (int ii = 0; ii < CHEB_N; ++ii) cc += f[iv * CHEB_N + ii] * cosm[jj * CHEB_N + ii];
      cc *= (jj == 0 ? 1.0 : 2.0) / CHEB_N;
    }
    cheb[idx] = cc;
  }
  __syncthreads();
  // monomial coefficients of log2 ρ = log2(e)·(line + Σ c_j T_j(t)); the octave e_zero
  // (if built) holds the constant −2000, which the build's 2^y flushes to 0
  double* T = table + (size_t)blockIdx.x * TABLE_D;
  for (int idx = olo * CHEB_SUB * CHEB_STRIDE + tid; idx < (ohi + 1) * CHEB_SUB * CHEB_STRIDE; idx += TABLE_NT) {
    const int iv = idx / CHEB_STRIDE, kk = idx % CHEB_STRIDE;
    double a = 0.0;
    if (CHEB_ELO + iv / CHEB_SUB < ez) {
      for (int jj = CHEB_N - 1; jj >= kk; --jj) a += cheb[iv * CHEB_N + jj] * tco[jj * CHEB_N + kk];
      if (kk == 0) a += 0.5 * (edge[iv] + edge[iv + 1]);  // the line's value at t = 0
      if (kk == 1) a += 0.5 * (edge[iv + 1] - edge[iv]);  // the line's slope in t
      a *= kLog2e;
    } else if (kk == 0) {
      a = -2000.0;
    }
    T[idx] = a;
  }
}

cudaError_t launch_table(int sub, PointConst* pc, int k0, int kw, double* table, const double* dstat,
                         cudaStream_t st) {
  auto go = [&](auto kern, int nint_n) -> cudaError_t {
    const int smem = 2 * nint_n * (int)sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<kw, TABLE_NT, smem, st>>>(pc, k0, table, dstat);
    return cudaGetLastError();
  };
  if (sub == CHEB_SUB_LARGE) return go(table_kernel<CHEB_SUB_LARGE>, Cheb<CHEB_SUB_LARGE>::NINT * Cheb<CHEB_SUB_LARGE>::N);
  return go(table_kernel<1>, Cheb<1>::NINT * Cheb<1>::N);
}

// ---------------------------------------------------------------------------
// build: grid = (ntri + nt tiles, kw points), 256 threads, 16 elements each.
// Tile (i, j), i ≥ j, of V = R + ν²I (lower tile triangle; the strict upper
// triangle of a diagonal tile is not referenced by the factorisation and is
// written as 0).  Padded rows/columns (index ≥ n) hold the identity, which
// leaves log|V| and L⁻¹B unchanged.  Augmented tile j holds Bᵀ[:, 64j:64j+64].
// ---------------------------------------------------------------------------
#ifndef LIK_BUILD_TILES
#define LIK_BUILD_TILES 8
#endif
constexpr int BUILD_TILES = LIK_BUILD_TILES;  // tiles of one point per block (amortises the table load)
#ifndef LIK_BUILD_NE
#define LIK_BUILD_NE 4  // 4: 35.4 ms, 2: 36.1 ms per 2,960 C4 points
#endif
constexpr int BUILD_NE = LIK_BUILD_NE;  // elements per thread evaluated interleaved (2 or 4)

#ifndef LIK_BUILD_VEC
#define LIK_BUILD_VEC 0  // 1: two columns per thread, 16-byte stores
#endif
#ifndef LIK_BUILD_MINB
#define LIK_BUILD_MINB 4  // 64 registers, 4 blocks (32 warps) per SM: 36.8 vs 40.6 ms per 2,960 C4 points
#endif
template <int SUB>
__global__ void __launch_bounds__(256, LIK_BUILD_MINB) build_kernel(const double* __restrict__ coords, SlotGeom g,
                                                    const PointConst* __restrict__ pc, int k0,
                                                    const double* __restrict__ table,
                                                    const double* __restrict__ Bt,
                                                    double* __restrict__ ws, cudaTextureObject_t tex) {
  constexpr int CHEB_STRIDE = Cheb<SUB>::STRIDE, TABLE_D = Cheb<SUB>::TABLE_D;
  const int slot = blockIdx.y;
  const PointConst P = pc[k0 + slot];
  if (P.mode == MODE_BAD) return;
  const int npad = g.nt * TB;
  __shared__ __align__(16) double2 sxy[2][TB];  // (x, y) of the tile's row and column sites
  extern __shared__ __align__(16) double coef[];  // the point's table (TABLE_D doubles, dynamic)
  __shared__ double etab[16];
  if (threadIdx.x < 16) etab[threadIdx.x] = kExp2Tab[threadIdx.x];
  // octaves [olo, oz] of the table; oz = the underflow octave (constant −2000) if built
  const int ezo = P.e_zero - CHEB_ELO;
  const int olo = P.olo, oz = max(olo, min(P.ohi, ezo));
  const unsigned span = ezo <= P.ohi ? 0x7fffffffu : (unsigned)(P.ohi - olo);
  if (P.mode == MODE_BESSEL) {
    const double2* src = reinterpret_cast<const double2*>(table + (size_t)slot * TABLE_D);
    double2* dst = reinterpret_cast<double2*>(coef);
    for (int e = olo * SUB * CHEB_STRIDE / 2 + threadIdx.x; e < (oz + 1) * SUB * CHEB_STRIDE / 2; e += 256)
      dst[e] = src[e];
  }
#if LIK_BUILD_VEC
  // thread -> columns c, c + 1 (c even), rows r0 + 8q (q < 8): a warp covers the 64
  // columns of one row, and each element pair (c, c + 1) of a row leaves as one 16-byte
  // store (the swizzle XORs multiples of 4 into the column: pairs stay adjacent)
  const int c = 2 * (threadIdx.x & 31), r0 = threadIdx.x >> 5;
  constexpr int RSTEP = 8, NQ = 8;
#else
  // thread -> column c, rows r0 + 4q (q < 16): a warp covers 32 consecutive
  // columns of one row; with Morton-ordered sites their s values mostly share an
  // interval, so the coefficient loads are shared-memory broadcasts.
  const int c = threadIdx.x & 63, r0 = threadIdx.x >> 6;
  constexpr int RSTEP = 4, NQ = 16;
#endif
  for (int tt = 0; tt < BUILD_TILES; ++tt) {
    const int tile = blockIdx.x * BUILD_TILES + tt;
    if (tile >= g.ntri + g.nt) break;
    double* T = ws + (size_t)slot * g.slot_d + (size_t)tile * TILE_D;
    if (tile >= g.ntri) {
      const int j = tile - g.ntri;
      for (int e = threadIdx.x; e < TILE_D; e += 256) {
        const int r = e >> 6, cc = e & 63;
        T[sw_off(r, cc)] = (r < g.r) ? Bt[(size_t)r * npad + j * TB + cc] : 0.0;
      }
      continue;
    }
    // tile (i, j) from the packed index
    int i = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
    while (tri_index(i + 1, 0) <= tile) ++i;
    while (tri_index(i, 0) > tile) --i;
    const int j = tile - tri_index(i, 0);
    __syncthreads();  // previous tile's coordinates are no longer read
    if (threadIdx.x < 2 * TB) {
      const int side = threadIdx.x >> 6, l = threadIdx.x & 63;
      const int gi = (side ? j : i) * TB + l;
      sxy[side][l] = gi < g.n ? reinterpret_cast<const double2*>(coords)[gi] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const bool regular = (i > j) && ((i + 1) * TB <= g.n);
    // the thread's rows r0 + RSTEP·q share the swizzle of r0 (rows differ by multiples of 4)
    double* Tc = T + sw_off(r0, c);
    unsigned slow = 0u;  // bit = element index of the thread (row-major over its rows × columns)
#if LIK_BUILD_VEC
    const double2 cj0 = sxy[1][c], cj1 = sxy[1][c + 1];
#else
    const double2 cj = sxy[1][c];
#endif
    if (P.mode == MODE_BESSEL) {
#pragma unroll 2
      for (int q = 0; q < NQ; q += BUILD_NE / (LIK_BUILD_VEC ? 2 : 1)) {
        double hx[BUILD_NE], hy[BUILD_NE], v[BUILD_NE];
#pragma unroll
        for (int e = 0; e < BUILD_NE; ++e) {
#if LIK_BUILD_VEC
          const double2 ri = sxy[0][r0 + RSTEP * (q + (e >> 1))];
          const double2 cj = (e & 1) ? cj1 : cj0;
#else
          const double2 ri = sxy[0][r0 + RSTEP * (q + e)];
#endif
          hx[e] = ri.x - cj.x;
          hy[e] = ri.y - cj.y;
        }
        const int bit = LIK_BUILD_VEC ? 2 * q : q;
#if LIK_BUILD_TEXMASK
        const long long tb = (long long)slot * (TABLE_D / 2);
        if (regular && P.range_ok)
          matern_rho_tableN_tex<BUILD_NE, SUB, false>(P, tex, tb, coef, etab, olo, oz, span, hx, hy, v, slow, bit);
        else
          matern_rho_tableN_tex<BUILD_NE, SUB, true>(P, tex, tb, coef, etab, olo, oz, span, hx, hy, v, slow, bit);
#else
        if (regular && P.range_ok)
          matern_rho_tableN<BUILD_NE, SUB, false>(P, coef, etab, olo, oz, span, hx, hy, v, slow, bit);
        else
          matern_rho_tableN<BUILD_NE, SUB, true>(P, coef, etab, olo, oz, span, hx, hy, v, slow, bit);
#endif
#if LIK_BUILD_VEC
#pragma unroll
        for (int e = 0; e < BUILD_NE; e += 2)
          *reinterpret_cast<double2*>(Tc + (q + e / 2) * RSTEP * KC) = make_double2(v[e], v[e + 1]);
#else
#pragma unroll
        for (int e = 0; e < BUILD_NE; ++e) Tc[(q + e) * RSTEP * KC] = v[e];
#endif
      }
    } else {
#pragma unroll 4
      for (int q = 0; q < NQ; ++q) {
        const double2 ri = sxy[0][r0 + RSTEP * q];
#if LIK_BUILD_VEC
        *reinterpret_cast<double2*>(Tc + q * RSTEP * KC) =
            make_double2(exp(-2.0 * aniso_d2(P, ri.x - cj0.x, ri.y - cj0.y)),
                         exp(-2.0 * aniso_d2(P, ri.x - cj1.x, ri.y - cj1.y)));
#else
        Tc[q * RSTEP * KC] = exp(-2.0 * aniso_d2(P, ri.x - cj.x, ri.y - cj.y));
#endif
      }
    }
    if (!regular || slow) {
      // fix-up pass (rewrites): padding, diagonal, unused upper triangle, outside the table
#pragma unroll 1
      for (int idx = 0; idx < 16; ++idx) {
        const int r = r0 + RSTEP * (LIK_BUILD_VEC ? idx >> 1 : idx);
        const int cc = c + (LIK_BUILD_VEC ? idx & 1 : 0);
        const int gi = i * TB + r, gj = j * TB + cc;
        double v;
        if (gi >= g.n || gj >= g.n) {
          v = (gi == gj) ? 1.0 : 0.0;
        } else if (gi == gj) {
          v = 1.0 + P.nugget;
        } else if (i == j && cc > r) {
          v = 0.0;
        } else if ((slow >> idx) & 1u) {
          const double2 ri = sxy[0][r];
          const double2 cjj = sxy[1][cc];
          v = matern_rho_exact(P, ri.x - cjj.x, ri.y - cjj.y);
        } else {
          continue;
        }
        T[sw_off(r, cc)] = v;
      }
    }
  }
}

cudaError_t launch_build(int sub, const double* coords, const SlotGeom& g, const PointConst* pc, int k0,
                         int kw, const double* table, cudaTextureObject_t table_tex, const double* Bt,
                         double* ws, cudaStream_t st) {
  const cudaTextureObject_t tex = table_tex;
  dim3 grid((g.ntri + g.nt + BUILD_TILES - 1) / BUILD_TILES, kw);
  auto go = [&](auto kern, int table_d) -> cudaError_t {
    const int smem = table_d * (int)sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 256, smem, st>>>(coords, g, pc, k0, table, Bt, ws, tex);
    return cudaGetLastError();
  };
  if (sub == CHEB_SUB_LARGE) return go(build_kernel<CHEB_SUB_LARGE>, Cheb<CHEB_SUB_LARGE>::TABLE_D);
  return go(build_kernel<1>, Cheb<1>::TABLE_D);
}

// ---------------------------------------------------------------------------
// unpack (debug / parity only): tiles of V -> dense n×n row-major, mirrored.
// ---------------------------------------------------------------------------
__global__ void unpack_V_kernel(SlotGeom g, const PointConst* __restrict__ pc,
                                const double* __restrict__ ws, double* __restrict__ V) {
  const int k = blockIdx.y;
  const size_t nn = (size_t)g.n * g.n;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn;
       e += (size_t)gridDim.x * blockDim.x) {
    int a = (int)(e / g.n), b = (int)(e % g.n);
    double v;
    if (pc[k].mode == MODE_BAD) {
      v = __longlong_as_double(0x7ff8000000000000LL);
    } else {
      if (b > a) { int t = a; a = b; b = t; }
      const int i = a / TB, j = b / TB;
      v = ws[(size_t)k * g.slot_d + (size_t)tri_index(i, j) * TILE_D + sw_off(a % TB, b % TB)];
    }
    V[(size_t)k * nn + e] = v;
  }
}

cudaError_t launch_unpack_V(const SlotGeom& g, const PointConst* pc, int kw, const double* ws,
                            double* V, cudaStream_t st) {
  dim3 grid(256, kw);
  unpack_V_kernel<<<grid, 256, 0, st>>>(g, pc, ws, V);
  return cudaGetLastError();
}

}  // namespace lik
