// Internal declarations shared by the liblik.so translation units (product
// path only; nothing here is shared with the CPU oracle).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace lik {

// ---------------------------------------------------------------------------
// Tile layout of the per-point workspace ("slot") in HBM.
//
// The augmented matrix  A = [[V, B], [Bᵀ, 0]]  with B = [y'_1..y'_M | X]
// (n × r) is stored as 64×64 FP64 tiles: the lower tile-triangle of V
// (tile (i,j), i ≥ j, index i(i+1)/2 + j) followed by one row of nt
// "augmented" tiles holding Bᵀ (rows t < r, column block j).  Factoring A by
// the left-looking Cholesky leaves L (n×n) in the V tiles and Zᵀ = (L⁻¹B)ᵀ in
// the augmented row, and −BᵀV⁻¹B as the Schur complement of the last block
// (§3.3 Steps 2-4).
//
// Inside a tile the 64 columns are split into four 64×16 "chunks" (8 KB,
// contiguous), each row-major with an XOR swizzle of the column index so that
// the DMMA fragment loads from shared memory are bank-conflict free after a
// 1-D bulk copy (cp.async.bulk) of the chunk.  Because the tiles of one tile
// row are contiguous, the row panel L[i, 0:j] is one contiguous run of
// 4j chunks.
// ---------------------------------------------------------------------------
constexpr int TB = 64;              // tile edge
#ifndef LIK_KC
#define LIK_KC 16
#endif
constexpr int KC = LIK_KC;          // chunk width (k-extent of one pipeline stage): 8 or 16
constexpr int CHUNKS = TB / KC;     // chunks per tile
constexpr int TILE_D = TB * TB;     // doubles per tile
constexpr int CHUNK_D = TB * KC;    // doubles per chunk
static_assert(KC == 8 || KC == 16, "chunk width");

// XOR swizzle of the column within a chunk row: the 16 lanes of a half-warp read
// rows r0..r0+3 × columns 4q..4q+3 of a DMMA fragment; the swizzle spreads them over
// 16 distinct 8-byte bank slots (KC = 16: rows differ by 16 doubles; KC = 8: by 8).
__host__ __device__ __forceinline__ int swz(int row) {
  return KC == 16 ? ((row & 3) << 2) : (((row >> 1) & 1) << 2);
}
__host__ __device__ __forceinline__ int sw_off(int row, int col) {
  return (col / KC) * CHUNK_D + row * KC + ((col % KC) ^ swz(row));
}
__host__ __device__ __forceinline__ int tri_index(int i, int j) { return i * (i + 1) / 2 + j; }

struct SlotGeom {
  int n;       // sites
  int nt;      // tiles per dimension = ceil(n / 64)
  int vlast;   // valid rows of the last tile (1..64)
  int ntri;    // nt(nt+1)/2
  int r;       // M + p (augmented rows)
  int Ra;      // r rounded up to a multiple of 8 (rows copied / computed)
  size_t slot_d;  // doubles per slot = (ntri + nt) * TILE_D
  // Merged tail: when the last V tile is ragged and its padding can hold the r
  // augmented rows (off + Ra ≤ 64, off = vlast rounded up to 16), the B rows are
  // treated as rows off.. of the last tile row (a virtual tile assembled from two
  // bulk copies), so no separate augmented tile row is processed and the last
  // diagonal tile's partial factorisation leaves −BᵀV⁻¹B as its Schur block.
  int merged;
  int off;
};

inline SlotGeom make_geom(int n, int r) {
  SlotGeom g;
  g.n = n;
  g.nt = (n + TB - 1) / TB;
  g.vlast = n - (g.nt - 1) * TB;
  g.ntri = g.nt * (g.nt + 1) / 2;
  g.r = r;
  g.Ra = (r + 7) & ~7;
  g.slot_d = (size_t)(g.ntri + g.nt) * TILE_D;
  g.off = (g.vlast + 15) & ~15;
  g.merged = (r > 0 && g.vlast < TB && g.off + g.Ra <= TB) ? 1 : 0;
  return g;
}

// Per-point constants (one per parameter point), written by setup_kernel.
enum { MODE_BESSEL = 0, MODE_GAUSS = 1, MODE_BAD = 2 };
struct PointConst {
  double cX, sX, sY, cY;   // u/φX = cX hx − sX hy,  v/φY = sY hx + cY hy
  double qX, qS, qT, qY;   // the same rows scaled by √(8κ): s = z² = (qX hx − qS hy)² + (qT hx + qY hy)²
  double kappa;            // κ
  double eightk;           // 8κ (s = z² = 8κ d², exact)
  double inv4k;            // 1/(4κ)  (the Gamma-mixture quadrature, matern_rho.cuh)
  double lnC;              // κ ln κ − κ − ln Γ(κ)
  double nugget;           // ν²
  int mode;                // MODE_*
  int e_zero;              // ρ ≡ 0 (ln ρ < −750) for s = z² ≥ 2^e_zero (set by table_kernel)
  int olo, ohi;            // table octaves built for this point (its range of s ± 1 octave)
  int range_ok;            // the point's whole s range lies inside [2^(ELO+olo), 2^(ELO+ohi+1))
                           // (not clipped at the table's ends): pairs of distinct sites need
                           // no range check
};

// Per-point Chebyshev table of log2 ρ on binary octaves of s = z² = 8κ·d² ∈ [2^e,
// 2^{e+1}), e = CHEB_ELO .. CHEB_ELO + CHEB_NOCT − 1 (the build needs no square
// root).  Each interval (CHEB_SUB per octave) stores CHEB_N doubles (16-byte aligned
// pairs, then 2 pad doubles): the monomial coefficients, in t ∈ [−1, 1) (an exact power-of-two map of s),
// of the degree CHEB_N − 1 Chebyshev interpolant of log2 ρ(√s) (base 2, so the build's
// exp is a plain 2^y).  Below 2^CHEB_ELO the exact evaluation is used; at and above
// 2^e_zero ρ = 0: the interval of the octave e_zero holds the constant −2000 (2^−2000
// flushes to 0), and the build clamps every larger s to it.
// Two table layouts, chosen per call from n (cheb_sub_for): SUB = 1 whole octaves
// with degree 19; SUB = CHEB_SUB_LARGE = 4 splits every octave into quarters
// ([1, 1.25), …, [1.75, 2) × 2^e; interval = SUB·octave + the top two mantissa bits of
// s) with degree 11 — the worst quarter sees the branch point at s = 0 from 9
// half-widths (Bernstein ρ = 17.9 vs 5.8), so the truncation stays ≤ 2e-17·max(1,
// |ln ρ|).  Quarters cost the table kernel 2.4× the exact evaluations per point and save
// the build 8 DFMA and 4 LDS.128 per element against whole octaves (C4 build −9 %
// against halves with degree 15), so they pay from a few hundred sites on.
constexpr int CHEB_ELO = -52;
constexpr int CHEB_NOCT = 80;
template <int SUB>
struct Cheb {
  static_assert(SUB == 1 || SUB == 2 || SUB == 4 || SUB == 8, "intervals per octave");
  static constexpr int LOG2SUB = SUB == 1 ? 0 : SUB == 2 ? 1 : SUB == 4 ? 2 : 3;
  // coefficients per interval: the truncation of the worst interval [1, 1 + 1/SUB)·2^e
  // stays ≤ 2e-17·max(1, |ln ρ|) (mpmath, κ ∈ [0.2, 200]), far below the rounding floor
  static constexpr int N = SUB == 1 ? 20 : SUB == 2 ? 16 : SUB == 4 ? 12 : 10;
  // + 2 pad doubles: consecutive intervals start 16 bytes (4 banks) apart, so lanes of a
  // warp reading the same pair of different intervals hit different banks (a stride of
  // a multiple of 128 bytes serialises them: build 1.6× slower, measured)
  static constexpr int STRIDE = N + 2;
  static constexpr int NINT = CHEB_NOCT * SUB;  // intervals
  static constexpr int TABLE_D = STRIDE * NINT;
};
// the layout for n ≥ LIK_CHEB_SUB_MIN_N (the whole-octave layout below)
#ifndef LIK_CHEB_SUB_LARGE
#define LIK_CHEB_SUB_LARGE 4
#endif
constexpr int CHEB_SUB_LARGE = LIK_CHEB_SUB_LARGE;
constexpr int TABLE_D = Cheb<1>::TABLE_D > Cheb<CHEB_SUB_LARGE>::TABLE_D ? Cheb<1>::TABLE_D
                                                                         : Cheb<CHEB_SUB_LARGE>::TABLE_D;
#ifndef LIK_CHEB_SUB_MIN_N
#define LIK_CHEB_SUB_MIN_N 256
#endif
inline int cheb_sub_for(int n) { return n >= LIK_CHEB_SUB_MIN_N ? CHEB_SUB_LARGE : 1; }

// Launch wrappers (defined in the .cu files).  All enqueue on `st`.
// prep: Box-Cox rows of Bᵀ, S = Σ log y, and the site gather coords_p[i] = coords[perm[i]]
// (perm == nullptr: identity).
cudaError_t launch_prep(const double* coords, const double* y, const double* X,
                        const double* lambdas, const int* perm, int n, int p, int M, int npad,
                        double* coords_p, double* Bt, double* S, cudaStream_t st);
cudaError_t launch_setup(const double* params, int K, PointConst* pc, cudaStream_t st);
// once per process (lik_create): the DCT matrices of the table kernel
cudaError_t launch_cheb_init(cudaStream_t st);
// dist_range: dstat[0] = min, dstat[1] = max squared Euclidean distance over the
// site pairs (bounds each point's range of s = z² for the table).
cudaError_t launch_dist_range(const double* coords, int n, double* dstat, cudaStream_t st);
cudaError_t launch_table(int sub, PointConst* pc, int k0, int kw, double* table, const double* dstat,
                         cudaStream_t st);
#ifndef LIK_BUILD_TEXMASK
#define LIK_BUILD_TEXMASK 0x24  // coefficient pairs fetched through the texture path (0: none)
#endif
// table_tex: a texture object (int4 elements) over `table` for the build's texture-path
// coefficient loads (make_table_tex)
cudaError_t launch_build(int sub, const double* coords, const SlotGeom& g, const PointConst* pc, int k0,
                         int kw, const double* table, cudaTextureObject_t table_tex, const double* Bt,
                         double* ws, cudaStream_t st);
cudaError_t launch_unpack_V(const SlotGeom& g, const PointConst* pc, int kw, const double* ws,
                            double* V, cudaStream_t st);

struct CholArgs {
  double* ws;
  SlotGeom g;
  int M, p;
  const PointConst* pc;
  int k0;                  // first point of the wave
  const double* lambdas;   // M
  const double* S;         // Σ log y (device scalar)
  double* loglik;          // K×M
  double* betahat;         // K×M×p
  double* sigma2hat;       // K×M
  double* logdetV;         // K
  int* status;             // K
  // optional Table-1 / REML outputs (NULL = skip)
  double* detReml;         // K
  double* ssqYX;           // K×r×r
  double* ssqBetahat;      // K×M
  double* ssqResidual;     // K×M
  double* loglik_reml;     // K×M
  double* sigma2hat_reml;  // K×M
};
cudaError_t launch_chol(const CholArgs& a, int kw, cudaStream_t st);
// chol_small.cu: the whole path for small augmented matrices in one kernel (no
// workspace); small_path_fits says whether (n, r = M + p) takes it.
bool small_path_fits(int n, int r, int p);
cudaError_t launch_chol_small(const CholArgs& a, const double* coords, const double* Bt, int ldb,
                              const double* table, cudaTextureObject_t table_tex, int kw, cudaStream_t st);
size_t chol_smem_bytes();
int profile_slices(long long K, int M);                       // slices of the (k, m) range
size_t profile_partials(int p, int G, int Sg, int M, int nsl);  // doubles of partial maxima
size_t profile_scratch(int p, int K, int M, int G, int Sg);     // doubles of scratch
cudaError_t launch_profiles(int n, int p, int K, int M, const double* y, const double* ssqYX,
                            const double* logdetV, const int* status, const double* lambdas,
                            int G, const double* beta_grid, double* prof_beta, int Sg,
                            const double* sigma_grid, double* prof_sigma, double* prof_lambda,
                            double* scratch, cudaStream_t st);
int chol_ctas_per_sm();

}  // namespace lik
