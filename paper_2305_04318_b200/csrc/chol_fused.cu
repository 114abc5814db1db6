// chol_fused — one CTA per parameter point: the paper's Steps 2-8 (§3.3,
// P:312-323) on the augmented matrix  A = [[V, B], [Bᵀ, 0]],  B = [y'|X].
//
// Left-looking (Crout) blocked Cholesky over 64×64 tiles:
//   for tile column j:   for row blocks (two tile rows at a time, i ≥ j, then the
//   augmented row):
//     C  = A_ij − Σ_{k<j} L_ik L_jkᵀ            (FP64 DMMA.8x8x4 tensor cores)
//     i = j:  C = L_jj L_jjᵀ in shared memory: 8-column panels, the 8×8 diagonal
//             blocks factored and inverted in registers by the lead warp, panel
//             products / trailing updates / the block-recursive L_jj⁻¹ on DMMA,
//             with lookahead; log|V| += Σ log pivots
//     i > j:  L_ij = C L_jj⁻ᵀ                   (DMMA, from the warp's registers)
// The augmented row ends up holding Zᵀ = (L⁻¹B)ᵀ (Step 3), and its final
// diagonal block  Σ_k Z_k Z_kᵀ = BᵀV⁻¹B  is the cross-product matrix ssqYX of
// Table 1 (Step 4).  When the B rows fit in the padding of the last
// diagonal tile ("merged tail"), they ride in that tile instead, and its partial
// factorisation leaves −BᵀV⁻¹B as the Schur block.  The epilogue does Steps 5-8
// and Eq. (profile).
//
// Operand staging: tiles are stored as contiguous 64×16 swizzled chunks
// (lik_internal.cuh), so each pipeline stage is three 1-D bulk copies
// (cp.async.bulk, the TMA engine) completing on an mbarrier; a 3-stage ring.
// The L_j panel (B operand, reused by every row block of column j) is loaded
// with an L2 evict_last policy, the streamed A panels with evict_first.
// 256 threads = 8 warps; warp w owns 16 full rows (all 64 columns) of tile row
// w/4 of the 128×64 row block: 2×8 DMMA 8×8 accumulators, so the triangular
// solve runs from its own registers and row blocks need no CTA barrier.  Two
// CTAs per SM (≤ 128 registers, ~105 KB shared memory each), so the serial
// phases of one point (diagonal factorisation, inverse) overlap the DMMA phases
// of the other.
//
// Ordering rules of the stage protocol (each one was needed):
// a warp releases a stage (empty mbarrier arrive) only after a CTA fence, so its
// shared-memory loads of the stage have completed before the producer's next bulk
// copy overwrites it; generic stores into ring memory (the staging tile) and into
// L tiles later read by bulk copies are followed by fence.proxy.async before the
// barrier that precedes those copies; mbarrier phases are waited by parity, which
// is safe because no warp can run more than one phase ahead of a stage.
#include <cfloat>
#include <cstdint>
#include <cstdio>
#include "../../include/lik.h"
#include "lik_internal.cuh"
#include "point_epilogue.cuh"

#ifdef LIK_PHASE_TIMERS
__device__ unsigned long long g_lik_phase[16];
#define PH_INIT() long long ph_t = clock64(); long long ph_acc[16] = {0}
#define PH(i) do { const long long t_ = clock64(); ph_acc[i] += t_ - ph_t; ph_t = t_; } while (0)
#define PH_FLUSH() do { if (threadIdx.x == 224) for (int i_ = 0; i_ < 16; ++i_) atomicAdd(&g_lik_phase[i_], (unsigned long long)ph_acc[i_]); } while (0)
#else
#define PH_INIT() do {} while (0)
#define PH(i) do {} while (0)
#define PH_FLUSH() do {} while (0)
#endif

#ifdef LIK_CTA_TRACE
// debug: per-CTA start / end (%globaltimer, ns) and SM id of the last launch
__device__ unsigned long long g_lik_cta_trace[1 << 16][3];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#endif
namespace lik {
namespace {

constexpr int NT = 256;
// Serial critical-path work (pivot chain, k-loop prologue copies, log-det) runs on the
// highest warp id: the SM's warp arbiter issues highest-wid first, so warp 0 would
// starve behind the co-resident CTA's DMMA warps.
constexpr int LEAD_WARP = NT / 32 - 1;
constexpr int LEAD_TID = LEAD_WARP * 32;
#ifndef LIK_NSTAGE
#define LIK_NSTAGE (KC == 8 ? 6 : 3)
#endif
constexpr int NSTAGE = LIK_NSTAGE;  // stage ring depth (3 fits two CTAs per SM)
constexpr int STAGE_D = 3 * CHUNK_D;             // A rows of tile a, A rows of tile b, B rows
constexpr int OFF_SCRATCH = 2 * TILE_D;          // 32×32 scratch after the staging tiles
constexpr int OFF_LINV = NSTAGE * STAGE_D;
constexpr int OFF_DLOG = OFF_LINV + TILE_D;
constexpr int OFF_MISC = OFF_DLOG + 64;          // 8 doubles of scalars
constexpr int OFF_MBAR = OFF_MISC + 8;           // NSTAGE full + NSTAGE empty uint64
constexpr int SMEM_D = OFF_MBAR + 2 * NSTAGE + 4;  // + int flags[4]
static_assert(OFF_SCRATCH + 32 * 32 <= OFF_LINV, "staging + scratch must fit in the stage ring");

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async;\n" ::: "memory");
}

// Warp tile: 16 rows × 64 columns (full rows of the 128×64 row block), as MI = 2
// row groups × NI = 8 column groups of 8×8 DMMA accumulators.  Owning full rows
// lets the triangular solve L = C·L_jj⁻ᵀ run from the warp's own registers.
constexpr int MI = 2, NI = 8;
typedef double Acc[MI][NI][2];

// One chunk (KC/4 k-steps of 4) of  acc += A_rows · B_rowsᵀ  for this warp.
// MFULL: both 8-row groups of the warp are live (the common case), so the DMMA
// sequence is branch- and predicate-free.  NL: column groups computed (NI, or fewer
// for a diagonal tile, whose columns beyond the warp's rows are never read).
#ifndef LIK_KPAIR
#define LIK_KPAIR 1
#endif
template <bool MFULL, int NL = NI>
__device__ __forceinline__ void mma_chunk(Acc& acc, const double* __restrict__ Ab, int rbase,
                                          int mlim, const double* __restrict__ Bb, int lane) {
  const int lr = lane >> 2, lc = lane & 3, sw = swz(lr);
#if LIK_KPAIR
  // Two k-steps per 16-byte load: within each group of 8 columns, the first step
  // takes the even columns and the second the odd ones (each column once, the same
  // assignment for A and B), so lane lc needs the adjacent pair (2lc, 2lc+1) — one
  // LDS.128.  The swizzle XORs multiples of 4, so the pair stays adjacent and
  // aligned; rows with (r & 3) < 2 and ≥ 2 fall in opposite bank halves (4
  // wavefronts per 512 bytes: conflict-free).  B fragments in two halves of NL/2
  // keep the live registers close to the one-step form.
  static_assert(KC % 8 == 0, "k pairs");
#pragma unroll
  for (int kp = 0; kp < KC / 8; ++kp) {
    const int kcol = ((kp * 8 + 2 * lc) ^ sw);
    double2 a[MI];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
      a[mi] = *reinterpret_cast<const double2*>(Ab + (rbase + mi * 8 + lr) * KC + kcol);
    constexpr int NH = NL >= 4 ? NL / 2 : NL;
#pragma unroll
    for (int h = 0; h < NL / NH; ++h) {
      double2 b[NH];
#pragma unroll
      for (int q = 0; q < NH; ++q)
        b[q] = *reinterpret_cast<const double2*>(Bb + ((h * NH + q) * 8 + lr) * KC + kcol);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
        if (MFULL || mi < mlim) {
#pragma unroll
          for (int q = 0; q < NH; ++q) dmma(acc[mi][h * NH + q], a[mi].x, b[q].x);
        }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
        if (MFULL || mi < mlim) {
#pragma unroll
          for (int q = 0; q < NH; ++q) dmma(acc[mi][h * NH + q], a[mi].y, b[q].y);
        }
    }
  }
#else
#pragma unroll
  for (int kk = 0; kk < KC / 4; ++kk) {
    const int kcol = ((kk * 4) ^ sw) + lc;
    double a[MI], b[NL];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) a[mi] = Ab[(rbase + mi * 8 + lr) * KC + kcol];
#pragma unroll
    for (int ni = 0; ni < NL; ++ni) b[ni] = Bb[(ni * 8 + lr) * KC + kcol];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
      if (MFULL || mi < mlim) {
#pragma unroll
        for (int ni = 0; ni < NL; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
      }
  }
#endif
}

// nlim < NI only for the warps of a diagonal tile with all rows live: warp rows
// [rbase, rbase + 16) need the column groups < rbase/8 + 2 (the strict upper
// triangle beyond them is never read: the factorisation and the Schur block read
// the lower triangle only).
__device__ __forceinline__ void mma_chunk_any(Acc& acc, const double* Ab, int rbase, int mlim,
                                              int nlim, const double* Bb, int lane) {
  if (mlim == MI) {
    if (nlim == NI)
      mma_chunk<true>(acc, Ab, rbase, MI, Bb, lane);
    else if (nlim == 2)
      mma_chunk<true, 2>(acc, Ab, rbase, MI, Bb, lane);
    else if (nlim == 4)
      mma_chunk<true, 4>(acc, Ab, rbase, MI, Bb, lane);
    else
      mma_chunk<true, 6>(acc, Ab, rbase, MI, Bb, lane);
  } else if (mlim > 0) {
    mma_chunk<false>(acc, Ab, rbase, mlim, Bb, lane);
  }
}

// acc ← acc · Xᵀ in place, X = L⁻¹ (64×64 lower triangular, swizzled shared memory):
// (C Xᵀ)[r][c] = Σ_{k ≤ c} C[r][k] X[c][k].  The output column group nt needs C's
// columns ≤ 8nt+7 only, so the groups are produced from the last to the first and
// each overwrites its own C group once computed.  The A fragment C[r][4s + lane%4]
// is taken from the accumulator layout (C[r][8t + 2q + e] in lane (r, q), element e)
// with two shuffles within the lane quad; k-steps above the triangle are skipped.
#ifndef LIK_TRSM_PERM
#define LIK_TRSM_PERM 1
#endif
__device__ __forceinline__ void trsm_reg(Acc& acc, const double* __restrict__ X, int lane) {
#if LIK_TRSM_PERM
  // The k (column-of-C) order of the product is free, so k-step (g, e) takes the columns
  // 8g + 2t + e (t = lane mod 4): exactly the element e of column group g that the lane
  // already holds in the accumulator layout — the A fragments come straight from the
  // registers, no shuffles; B = L_jj⁻ᵀ is read in the same permuted order.
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int nt = NI - 1; nt >= 0; --nt) {
    double o[MI][2];
#pragma unroll
    for (int m = 0; m < MI; ++m) o[m][0] = o[m][1] = 0.0;
#pragma unroll
    for (int g = 0; g <= nt; ++g) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double b = X[sw_off(8 * nt + lr, 8 * g + 2 * lc + e)];
#pragma unroll
        for (int m = 0; m < MI; ++m) dmma(o[m], acc[m][g][e], b);
      }
    }
#pragma unroll
    for (int m = 0; m < MI; ++m) {
      acc[m][nt][0] = o[m][0];
      acc[m][nt][1] = o[m][1];
    }
  }
#else
  const int lr = lane >> 2, lc = lane & 3, quad = lane & ~3, hi = lc >> 1;
  const bool odd = lc & 1;
#pragma unroll
  for (int nt = NI - 1; nt >= 0; --nt) {
    double o[MI][2];
#pragma unroll
    for (int m = 0; m < MI; ++m) o[m][0] = o[m][1] = 0.0;
#pragma unroll
    for (int s = 0; s <= 2 * nt + 1; ++s) {
      const int src = quad | (2 * (s & 1) + hi);
      double a[MI];
#pragma unroll
      for (int m = 0; m < MI; ++m) {
        const double v0 = __shfl_sync(0xffffffffu, acc[m][s >> 1][0], src);
        const double v1 = __shfl_sync(0xffffffffu, acc[m][s >> 1][1], src);
        a[m] = odd ? v1 : v0;
      }
      const double b = X[sw_off(8 * nt + lr, 4 * s + lc)];
#pragma unroll
      for (int m = 0; m < MI; ++m) dmma(o[m], a[m], b);
    }
#pragma unroll
    for (int m = 0; m < MI; ++m) {
      acc[m][nt][0] = o[m][0];
      acc[m][nt][1] = o[m][1];
    }
  }
#endif
}

// acc = acc − T  (T = the A_ij tile in global memory), i.e. −C.
__device__ __forceinline__ void frag_sub_from(Acc& acc, const double* __restrict__ T, int rbase,
                                              int mlim, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
    if (mi < mlim) {
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const double2 v =
            *reinterpret_cast<const double2*>(T + sw_off(rbase + mi * 8 + lr, ni * 8 + 2 * lc));
        acc[mi][ni][0] -= v.x;
        acc[mi][ni][1] -= v.y;
      }
    }
}

// acc −= T (T split: rows < off from T1, rows ≥ off from T2 at row − off)
__device__ __forceinline__ void frag_sub_from2(Acc& acc, const double* __restrict__ T1,
                                               const double* __restrict__ T2, int off, int rbase,
                                               int mlim, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
    if (mi < mlim) {
      const int row = rbase + mi * 8 + lr;
      const double* T = row < off ? T1 : T2;
      const int rr = row < off ? row : row - off;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const double2 v = *reinterpret_cast<const double2*>(T + sw_off(rr, ni * 8 + 2 * lc));
        acc[mi][ni][0] -= v.x;
        acc[mi][ni][1] -= v.y;
      }
    }
}

template <bool NEG>
__device__ __forceinline__ void frag_store2(const Acc& acc, double* __restrict__ T1,
                                            double* __restrict__ T2, int off, int rbase, int mlim,
                                            int lane) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
    if (mi < mlim) {
      const int row = rbase + mi * 8 + lr;
      double* T = row < off ? T1 : T2;
      const int rr = row < off ? row : row - off;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
        *reinterpret_cast<double2*>(T + sw_off(rr, ni * 8 + 2 * lc)) =
            NEG ? make_double2(-acc[mi][ni][0], -acc[mi][ni][1])
                : make_double2(acc[mi][ni][0], acc[mi][ni][1]);
    }
}

template <bool NEG>
__device__ __forceinline__ void frag_store(const Acc& acc, double* __restrict__ T, int rbase,
                                           int mlim, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
    if (mi < mlim) {
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
        *reinterpret_cast<double2*>(T + sw_off(rbase + mi * 8 + lr, ni * 8 + 2 * lc)) =
            NEG ? make_double2(-acc[mi][ni][0], -acc[mi][ni][1])
                : make_double2(acc[mi][ni][0], acc[mi][ni][1]);
    }
}

__device__ __forceinline__ void frag_zero(Acc& acc) {
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
}

struct Pipe {
  double* stages;
  uint64_t* mbar;     // "full" barriers: complete when a stage's bulk copies landed
  uint64_t* empty;    // "empty" barriers: complete when all 8 warps finished reading a stage
  uint32_t seq;       // chunks consumed so far (same value in every thread)
  uint64_t pol_stream, pol_keep;
};

// A k-loop operand: rows [0, r1) of row panel p1 and, for a merged tail tile,
// rows [0, r2) of row panel p2 placed at buffer row r1 (r1 a multiple of 16, so the
// chunk swizzle, which depends on row & 3, is preserved).
struct Src {
  const double* p1;
  int r1;
  const double* p2;
  int r2;
};

#ifdef LIK_BOUNDS_CHECK
// Debug builds: every bulk-copy source range and tile pointer must lie inside the
// point's workspace slot [lo, hi) (compute-sanitizer is unavailable on the pool).
#define LIK_CHECK_RANGE(ptr, ndoubles, lo, hi)                                              \
  do {                                                                                      \
    if ((const double*)(ptr) < (lo) || (const double*)(ptr) + (ndoubles) > (hi)) {          \
      printf("lik bounds: block %d ptr %p + %ld outside [%p, %p)\n", blockIdx.x, (const void*)(ptr), \
             (long)(ndoubles), (const void*)(lo), (const void*)(hi));                       \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define LIK_CHECK_RANGE(ptr, ndoubles, lo, hi) do {} while (0)
#endif

// acc += Σ_q A_q B_qᵀ over nq chunks streamed from global memory:
//   A rows of tile a: gA0 + q·CHUNK_D (cA0 rows copied), tile b: gA1 (cA1 rows),
//   B rows: gB (cB rows).
// There is no CTA-wide barrier, per chunk or between k-loops: each warp waits only
// for its data (full mbarrier) and releases the stage with a non-blocking arrive on
// its empty mbarrier; every copy into a stage first waits for the release of the
// stage's previous round (the ring runs on across k-loops: pp.seq counts chunks).
// At the start of chunk q one warp (rotating) refills the stage of chunk q−1 with
// chunk q−1+NSTAGE; the first NSTAGE chunks are issued by the lead thread.
// MODE: the chunk product, fixed for the whole k-loop — 0 all rows and column
// groups, 2/4/6 a diagonal tile's first column groups, 1 a partly filled row block,
// 9 no rows (the warp still takes part in the stage protocol); −1 decides per chunk.
template <int MODE>
__device__ __forceinline__ void kloop_m(Acc& acc, Pipe& pp, Src A0, Src A1, Src B, int nq,
                                        bool mine_b, int rbase, int mlim, int nlim, int lane,
                                        const double* slot_lo, const double* slot_hi) {
  const int tid = threadIdx.x;
  const uint32_t seq = pp.seq;
  auto copy = [&](double* dst, const Src& sr, int q, uint32_t bar, uint64_t pol) {
    if (sr.r1) LIK_CHECK_RANGE(sr.p1 + (size_t)q * CHUNK_D, sr.r1 * KC, slot_lo, slot_hi);
    if (sr.r2) LIK_CHECK_RANGE(sr.p2 + (size_t)q * CHUNK_D, sr.r2 * KC, slot_lo, slot_hi);
#ifdef LIK_EXP_SAMESRC
    q = 0;  // timing experiment only: every copy re-reads chunk 0 (L2-resident stream)
#endif
    if (sr.r1) bulk_g2s(saddr(dst), sr.p1 + (size_t)q * CHUNK_D, sr.r1 * KC * 8, bar, pol);
    if (sr.r2)
      bulk_g2s(saddr(dst + sr.r1 * KC), sr.p2 + (size_t)q * CHUNK_D, sr.r2 * KC * 8, bar, pol);
  };
  auto issue = [&](int q) {
    const uint32_t s = (seq + q) % NSTAGE;
    double* st = pp.stages + s * STAGE_D;
    const uint32_t bar = saddr(&pp.mbar[s]);
    mbar_expect_tx(bar, (uint32_t)(A0.r1 + A0.r2 + A1.r1 + A1.r2 + B.r1 + B.r2) * KC * 8);
    copy(st, A0, q, bar, pp.pol_stream);
    copy(st + CHUNK_D, A1, q, bar, pp.pol_stream);
    copy(st + 2 * CHUNK_D, B, q, bar, pp.pol_keep);
  };
  // The stage of chunk q−1 is refilled at the start of chunk q by warp (seq + q) mod 8:
  // the duty (wait for the release by all warps, arm, copy) rotates, so no warp is
  // always the last to start a chunk (measured: −3.4 % k-loop time with one CTA per
  // SM, +0.7 % throughput with two).  The same rule on both paths below, since the
  // warps of one row block may take different paths.
  auto producer = [&](int q) { return (tid >> 5) == (int)((seq + q) & 7) && (tid & 31) == 0; };
  if (tid == LEAD_TID)
    for (int q = 0; q < NSTAGE && q < nq; ++q) {
      const uint32_t u = seq + q;
      if (u >= NSTAGE) mbar_wait(saddr(&pp.empty[u % NSTAGE]), (u / NSTAGE - 1) & 1);
      issue(q);
    }
  // (A software-pipelined variant of this loop — next k-step's fragments loaded
  // before the current DMMAs, double-buffered — gave no speed-up with two CTAs per
  // SM and, with the full-row warp tiles, produced run-to-run differences at
  // ~0.1 % of the points; removed.  tests/test_gpu_parity.py checks bitwise
  // repeatability over several CTA rounds.)
  for (int q = 0; q < nq; ++q) {
    if (producer(q) && q >= 1 && q - 1 + NSTAGE < nq) {
      const uint32_t u = seq + q - 1;
      mbar_wait(saddr(&pp.empty[u % NSTAGE]), (u / NSTAGE) & 1);
      issue(q - 1 + NSTAGE);
    }
    const uint32_t s = (seq + q) % NSTAGE;
#ifdef LIK_PHASE_TIMERS
    const long long tw0 = clock64();
#endif
    mbar_wait(saddr(&pp.mbar[s]), ((seq + q) / NSTAGE) & 1);
#ifdef LIK_PHASE_TIMERS
    if (tid == 224) atomicAdd(&g_lik_phase[q == 0 ? 9 : 15], (unsigned long long)(clock64() - tw0));
#endif
    const double* st = pp.stages + s * STAGE_D;
    const double* Ab = st + (mine_b ? CHUNK_D : 0);
    if constexpr (MODE == -1) mma_chunk_any(acc, Ab, rbase, mlim, nlim, st + 2 * CHUNK_D, lane);
    else if constexpr (MODE == 0) mma_chunk<true>(acc, Ab, rbase, MI, st + 2 * CHUNK_D, lane);
    else if constexpr (MODE == 2 || MODE == 4 || MODE == 6)
      mma_chunk<true, MODE>(acc, Ab, rbase, MI, st + 2 * CHUNK_D, lane);
    else if constexpr (MODE == 1) mma_chunk<false>(acc, Ab, rbase, mlim, st + 2 * CHUNK_D, lane);
    __syncwarp();
    // The release must not overtake this warp's shared-memory loads of the stage:
    // the DMMAs consuming them may be scheduled after the arrive, and
    // mbarrier.arrive.release alone was measured not to hold back loads still in
    // flight — the producer's next bulk copy then overwrote a stage being read
    // (run-to-run differences at ~0.5 % of the points with the full-tile loop
    // specialised; this was also the v13 race).  The CTA fence waits for them.
    if (lane == 0) {
      __threadfence_block();
      mbar_arrive(saddr(&pp.empty[s]));
    }
  }
  pp.seq = seq + nq;
}

// Which chunk products get a k-loop of their own (no per-chunk dispatch): bit 0 full
// tiles (the default: +0.8 % at C4), bit 1 partial row blocks, bit 2 diagonal tiles,
// bit 3 rowless warps; the rest dispatch per chunk (mma_chunk_any).
#ifndef LIK_KLOOP_TMPL_MASK
#define LIK_KLOOP_TMPL_MASK 1
#endif
__device__ __forceinline__ void kloop(Acc& acc, Pipe& pp, Src A0, Src A1, Src B, int nq,
                                      bool mine_b, int rbase, int mlim, int nlim, int lane,
                                      const double* slot_lo, const double* slot_hi) {
#define KL(M) kloop_m<M>(acc, pp, A0, A1, B, nq, mine_b, rbase, mlim, nlim, lane, slot_lo, slot_hi)
  constexpr int TM = LIK_KLOOP_TMPL_MASK;
  if (mlim == MI && nlim == NI && (TM & 1)) KL(0);
  else if (mlim == MI && nlim == 2 && (TM & 4)) KL(2);
  else if (mlim == MI && nlim == 4 && (TM & 4)) KL(4);
  else if (mlim == MI && nlim == 6 && (TM & 4)) KL(6);
  else if (mlim > 0 && mlim < MI && (TM & 2)) KL(1);
  else if (mlim == 0 && (TM & 8)) KL(9);
  else KL(-1);
#undef KL
}

// 32×32 scratch (T): two swizzled 32×16 halves, the chunk layout's bank pattern.
__device__ __forceinline__ int t_off(int r, int c) {
  return (c >> 4) * 512 + r * 16 + ((c & 15) ^ ((r & 3) << 2));
}

#ifndef LIK_PW
#define LIK_PW 8
#endif
constexpr int PW = LIK_PW;  // panel width of the diagonal-tile factorisation (8 or 16)
static_assert(PW == 8 || PW == 16, "panel width");

// Step (a) of a panel at c0 (the lead warp): factor the PW×PW diagonal block D_p in
// registers — lane l holds row l; one rsqrt per pivot gives L_cc and 1/L_cc, and
// the update of the trailing columns uses the pivot column fetched by shuffles —
// then invert it (lane l computes column l of D_p⁻¹, right-looking, so the
// dependent chain is two ops per step).  Only the pivot chain is serial; it uses no
// divisions (the FP64 pipe is shared with the co-resident CTA's DMMAs, so every
// dependent FP64 op on it is slow).  Pivots ≥ vloc are skipped (their rows and
// columns of D_p⁻¹ are 0).  dlog[c0 + c] = pivot_c (pivots_to_log takes the logs); a pivot ≤ tol sets flag[0].
__device__ __forceinline__ void factor_block(double* S, double* X, int c0, int vloc, double tol,
                                             double* dlog, int* flag) {
  const int lane = threadIdx.x & 31, l = lane & (PW - 1);
  double a[PW];
#pragma unroll
  for (int k = 0; k < PW; ++k) a[k] = (k <= l) ? S[sw_off(c0 + l, c0 + k)] : 0.0;
  int bad = 0;
  double my_piv = 1.0, my_rinv = 1.0;
  double piv_next = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll
  for (int c = 0; c < PW; ++c) {
    if (c < vloc) {
      const double piv = piv_next;
      bad |= !(piv > tol);
      const double rinv = rsqrt(piv);
      if (l == c) {
        a[c] = piv * rinv;
        my_piv = piv;
        my_rinv = rinv;
      } else if (l > c) {
        a[c] *= rinv;
      }
      // the next pivot from lane c+1's own registers (the same FMA as its update
      // below), broadcast once: the serial chain waits for one shuffle per pivot
      if (c + 1 < PW) {
        const double pn = a[c + 1] - a[c] * a[c];
        piv_next = __shfl_sync(0xffffffffu, pn, c + 1);
      }
#pragma unroll
      for (int k = 0; k < PW; ++k) {  // constant trip count: a[] stays in registers
        if (k > c) {
          const double lk = __shfl_sync(0xffffffffu, a[c], k);
          if (l >= k) a[k] -= a[c] * lk;
        }
      }
    }
  }
  if (lane < PW && l < vloc) dlog[c0 + l] = my_piv;  // log taken later, off the lead warp (pivots_to_log)
  double x[PW];
#pragma unroll
  for (int i = 0; i < PW; ++i) x[i] = (i == l && l < vloc) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < PW; ++i) {
    if (i < vloc) {
      x[i] *= __shfl_sync(0xffffffffu, my_rinv, i);
#pragma unroll
      for (int k = 0; k < PW; ++k)
        if (k > i) x[k] -= __shfl_sync(0xffffffffu, a[i], k) * x[i];
    }
  }
  if (lane < PW) {
#pragma unroll
    for (int k = 0; k < PW; ++k) {
      if (k <= l) S[sw_off(c0 + l, c0 + k)] = a[k];
      X[sw_off(c0 + k, c0 + l)] = (k < vloc && l < vloc) ? x[k] : 0.0;  // column l of D_p⁻¹
    }
  }
  if (lane == 0 && bad) flag[0] = 1;
}

// Steps (b) and (c) of the panel at c0 of the tile S (swizzled), with D_p⁻¹ in X, on
// the FP64 tensor cores:
//   (b) L[i, panel] = S[i, panel] · D_p⁻ᵀ   for rows i ∈ [c0+PW, 64): warp w owns rows
//       c0+PW+8w..+7 (all column tiles), so the in-place store needs no barrier;
//   (c) S[i, k] −= L[i, panel] · L[k, panel]ᵀ  for the 8×8 tiles on/below the diagonal
//       of [c0+PW, 64)², one warp per tile.
// DMMA fragments (m8n8k4): a = A[r + lane/4][k + lane%4], b = B[k + lane%4][n + lane/4],
// c = C[r + lane/4][n + 2(lane%4) + {0,1}].
// One 8-row tile (rows b0 + 8·rtile, b0 = c0 + PW) of step (b), in place.
__device__ __forceinline__ void panel_tile(double* S, const double* X, int c0, int rtile) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  const int r = c0 + PW + 8 * rtile;
  double c[PW / 8][2];
#pragma unroll
  for (int nt = 0; nt < PW / 8; ++nt) c[nt][0] = c[nt][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < PW / 4; ++ks) {
    const double a = S[sw_off(r + lr, c0 + 4 * ks + lc)];
#pragma unroll
    for (int nt = 0; nt < PW / 8; ++nt) {
      if (4 * ks > 8 * nt + 7) continue;  // D_p⁻¹ is lower triangular
      dmma(c[nt], a, X[sw_off(c0 + 8 * nt + lr, c0 + 4 * ks + lc)]);
    }
  }
#pragma unroll
  for (int nt = 0; nt < PW / 8; ++nt)
    *reinterpret_cast<double2*>(S + sw_off(r + lr, c0 + 8 * nt + 2 * lc)) = make_double2(c[nt][0], c[nt][1]);
}

__device__ __forceinline__ void panel_product(double* S, const double* X, int c0) {  // (b)
  const int warp = threadIdx.x >> 5, rt = (TB - c0 - PW) >> 3;
  if (warp < rt) panel_tile(S, X, c0, warp);
}

// Named barrier 1 (barrier 0 is __syncthreads): the lead warp arrives after its
// shared-memory stores, the other warps wait there (all NT threads counted).
__device__ __forceinline__ void named_arrive1() { asm volatile("bar.arrive 1, %0;\n" ::"n"(NT) : "memory"); }
__device__ __forceinline__ void named_sync1() { asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory"); }

// (c) for tile t of the lower triangle of [c0+PW, 64)² in 8×8 tiles (t = 0: the
// next diagonal block).
__device__ __forceinline__ void trailing_tile(double* S, int c0, int t) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3, b0 = c0 + PW;
  int ti = 0;
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  const int ri = b0 + 8 * ti, rk = b0 + 8 * (t - ti * (ti + 1) / 2);
  double c[2] = {0.0, 0.0};
#pragma unroll
  for (int ks = 0; ks < PW / 4; ++ks)
    dmma(c, S[sw_off(ri + lr, c0 + 4 * ks + lc)], S[sw_off(rk + lr, c0 + 4 * ks + lc)]);
  double2* q = reinterpret_cast<double2*>(S + sw_off(ri + lr, rk + 2 * lc));
  const double2 o = *q;
  *q = make_double2(o.x - c[0], o.y - c[1]);
}

__device__ void panel_update(double* S, const double* X, int c0) {  // (b) then (c), all warps
  panel_product(S, X, c0);
  __syncthreads();
  const int rt = (TB - c0 - PW) >> 3;
  for (int t = threadIdx.x >> 5; t < rt * (rt + 1) / 2; t += NT / 32) trailing_tile(S, c0, t);
  __syncthreads();
}

// dlog[c] = log(pivot_c) for c < v, by threads 0..v−1 (the lead warp, whose serial
// chain gates every panel, stores the raw pivots); visible after the caller's next
// __syncthreads.
__device__ __forceinline__ void pivots_to_log(double* dlog, int v) {
  if ((int)threadIdx.x < v) dlog[threadIdx.x] = log(dlog[threadIdx.x]);
}

// Blocked Cholesky + inverse of a 64×64 tile in shared memory (lower part used)
// whose rows/columns ≥ v are the identity padding of V.  64/PW panels:
//   (a) the lead warp factors the PW×PW diagonal block D_p and inverts it into X
//       (the diagonal blocks of L⁻¹) — factor_block,
//   (b)+(c) panel product and trailing update on the tensor cores — panel_update.
// Then L⁻¹ is assembled from the D_p⁻¹ by block recursion (PW → … → 64) on the
// tensor cores:  X_ba = −X_bb (L_ba X_aa)  for the off-diagonal blocks.
// dlog[c] = log(pivot_c).  Returns nonzero (uniformly) if a pivot is ≤ tol (R11).
// T is a 32×32 scratch.
#ifdef LIK_PHASE_TIMERS
#define SUB(i) do { if (threadIdx.x == 224) { const long long t_ = clock64(); atomicAdd(&g_lik_phase[i], (unsigned long long)(t_ - sub_t)); sub_t = t_; } } while (0)
#else
#define SUB(i) do {} while (0)
#endif
__device__ int potrf_inv64(double* S, int v, double tol, double* dlog, int* flag, double* X,
                           double* T) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef LIK_PHASE_TIMERS
  long long sub_t = clock64();
#endif
  if (v < TB) {  // identity padding (those rows of the staging tile were not computed)
    for (int e = tid; e < TILE_D; e += NT) {
      const int rr = e >> 6, kk = e & 63;
      if (rr >= v && kk <= rr) S[sw_off(rr, kk)] = (rr == kk) ? 1.0 : 0.0;
    }
    __syncthreads();
  }
  // Lookahead: after the panel product of panel p, the lead warp updates the next
  // diagonal block (the first ND trailing tiles) and factors it at once, while the
  // other warps update the rest of the trailing matrix (disjoint tiles).
  if (warp == LEAD_WARP) factor_block(S, X, 0, PW, tol, dlog, flag);
  SUB(10);
  __syncthreads();
  SUB(11);
#ifndef LIK_EXP_SAMESRC
  if (flag[0]) return 1;
#endif
  for (int c0 = 0; c0 + PW < TB; c0 += PW) {
    const int rt = (TB - c0 - PW) >> 3, ntile = rt * (rt + 1) / 2;
    constexpr int NR = PW / 8;                        // row tiles of the next diagonal block
    constexpr int ND = (PW / 8) * (PW / 8 + 1) / 2;  // trailing tiles of the next diagonal block
#ifndef LIK_POTRF_TWO_BARRIERS
    // One CTA barrier per panel: the lead warp computes the panel product of the next
    // diagonal block's rows itself (their inputs were final at the previous barrier),
    // signals the other warps through named barrier 1, updates and factors that
    // block; the other warps compute the remaining rows, wait for the lead's rows at
    // barrier 1 (only the trailing tiles below the next block read them) and update
    // the rest of the trailing matrix.
    if (warp == LEAD_WARP) {
      for (int q = 0; q < NR; ++q) panel_tile(S, X, c0, q);
      __syncwarp();
      __threadfence_block();  // the stores complete before the non-blocking arrive (cf. kloop)
      named_arrive1();
      for (int t = 0; t < ND; ++t) trailing_tile(S, c0, t);
      __syncwarp();
      factor_block(S, X, c0 + PW, PW, tol, dlog, flag);
    } else {
      for (int q = NR + warp; q < rt; q += NT / 32 - 1) panel_tile(S, X, c0, q);
      named_sync1();
      for (int t = ND + warp; t < ntile; t += NT / 32 - 1) trailing_tile(S, c0, t);
    }
#else
    panel_product(S, X, c0);
    __syncthreads();
    if (warp == LEAD_WARP) {
      for (int t = 0; t < ND; ++t) trailing_tile(S, c0, t);
      __syncwarp();
      factor_block(S, X, c0 + PW, PW, tol, dlog, flag);
    } else {
      for (int t = ND + warp; t < ntile; t += NT / 32 - 1) trailing_tile(S, c0, t);
    }
#endif
    __syncthreads();
    SUB(13);
#ifndef LIK_EXP_SAMESRC
    if (flag[0]) return 1;
#endif
  }
  // strictly-upper parts of X (above the PW-blocks on its diagonal) are zero
  for (int e = tid; e < TILE_D; e += NT) {
    const int i = e >> 6, c = e & 63;
    if (c / PW > i / PW) X[sw_off(i, c)] = 0.0;
  }
  pivots_to_log(dlog, v);
  __syncthreads();
  if (PW == 8) {  // level 8 → 16: X_{(2g+1),(2g)} = −X_{(2g+1),(2g+1)} (L_{(2g+1),(2g)} X_{(2g),(2g)})
    const int lr = lane >> 2, lc = lane & 3, o = 16 * warp;
    if (warp < 4) {
      double c[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
        dmma(c, S[sw_off(o + 8 + lr, o + 4 * ks + lc)], X[sw_off(o + 4 * ks + lc, o + lr)]);
      T[t_off(8 * warp + lr, 2 * lc)] = c[0];
      T[t_off(8 * warp + lr, 2 * lc + 1)] = c[1];
    }
    __syncthreads();
    if (warp < 4) {
      double c[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
        dmma(c, X[sw_off(o + 8 + lr, o + 8 + 4 * ks + lc)], T[t_off(8 * warp + 4 * ks + lc, lr)]);
      *reinterpret_cast<double2*>(X + sw_off(o + 8 + lr, o + 2 * lc)) = make_double2(-c[0], -c[1]);
    }
    __syncthreads();
  }
  // L⁻¹ off-diagonal blocks by block recursion on the tensor cores, one 8×8 tile per
  // warp: level 16 → 32 (blocks (1,0) of each 32-block), then 32 → 64.
  {
    const int lr = lane >> 2, lc = lane & 3;
    const int h = warp >> 2, i0 = ((warp >> 1) & 1) * 8, n0 = (warp & 1) * 8, o = 32 * h;
    double c[2] = {0.0, 0.0};
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {  // T_h = L_{(2h+1),(2h)} X_{(2h),(2h)}  (X lower: k ≥ n)
      if (4 * ks + 3 < n0) continue;
      dmma(c, S[sw_off(o + 16 + i0 + lr, o + 4 * ks + lc)], X[sw_off(o + 4 * ks + lc, o + n0 + lr)]);
    }
    T[t_off(16 * h + i0 + lr, n0 + 2 * lc)] = c[0];
    T[t_off(16 * h + i0 + lr, n0 + 2 * lc + 1)] = c[1];
    __syncthreads();
    c[0] = c[1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {  // X_{(2h+1),(2h)} = −X_{(2h+1),(2h+1)} T_h  (k ≤ i)
      if (4 * ks > i0 + 7) continue;
      dmma(c, X[sw_off(o + 16 + i0 + lr, o + 16 + 4 * ks + lc)], T[t_off(16 * h + 4 * ks + lc, n0 + lr)]);
    }
    *reinterpret_cast<double2*>(X + sw_off(o + 16 + i0 + lr, o + n0 + 2 * lc)) = make_double2(-c[0], -c[1]);
    __syncthreads();
    double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int u = 0; u < 2; ++u) {  // level 32 → 64: T = L21 X11  (two tiles per warp)
      const int tile = warp + 8 * u, r0 = (tile >> 2) * 8, m0 = (tile & 3) * 8;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        if (4 * ks + 3 < m0) continue;
        dmma(d[u], S[sw_off(32 + r0 + lr, 4 * ks + lc)], X[sw_off(4 * ks + lc, m0 + lr)]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int tile = warp + 8 * u, r0 = (tile >> 2) * 8, m0 = (tile & 3) * 8;
      T[t_off(r0 + lr, m0 + 2 * lc)] = d[u][0];
      T[t_off(r0 + lr, m0 + 2 * lc + 1)] = d[u][1];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {  // X21 = −X22 T  (k ≤ i)
      const int tile = warp + 8 * u, r0 = (tile >> 2) * 8, m0 = (tile & 3) * 8;
      double e[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        if (4 * ks > r0 + 7) continue;
        dmma(e, X[sw_off(32 + r0 + lr, 32 + 4 * ks + lc)], T[t_off(4 * ks + lc, m0 + lr)]);
      }
      *reinterpret_cast<double2*>(X + sw_off(32 + r0 + lr, m0 + 2 * lc)) = make_double2(-e[0], -e[1]);
    }
  }
  SUB(14);
  return 0;
}

// Partial Cholesky of the merged last diagonal tile: pivots are the first v
// (= vlast) columns; the augmented rows start at row `off` (a multiple of 16 ≥ v).
// Panels of 16 as in potrf_inv64 (factor + invert the pivot block in registers,
// panel product, trailing update), stopping after the last pivot panel: the
// block rows/cols ≥ off then hold C_BB − Z Zᵀ = −BᵀV⁻¹B (the Schur complement).
__device__ int potrf_tail(double* S, int v, double tol, double* dlog, int* flag, double* X) {
  const int warp = threadIdx.x >> 5;
  for (int c0 = 0; c0 < v; c0 += PW) {
    if (warp == LEAD_WARP) factor_block(S, X, c0, min(PW, v - c0), tol, dlog, flag);
    __syncthreads();
    if (flag[0]) return 1;
    if (c0 + PW < TB) panel_update(S, X, c0);
  }
  pivots_to_log(dlog, v);
  __syncthreads();
  return 0;
}

__device__ void write_point_failure(const CholArgs& A, int k, int code) {
  point_failure(A, k, code, threadIdx.x, NT);
}

#ifndef LIK_MIN_BLOCKS
#define LIK_MIN_BLOCKS 2
#endif
#ifdef LIK_CHOL_MAXREG  // experiment: a register cap below the 2-CTA/SM one
#define LIK_CHOL_BOUNDS __maxnreg__(LIK_CHOL_MAXREG)
#else
#define LIK_CHOL_BOUNDS __launch_bounds__(NT, LIK_MIN_BLOCKS)
#endif
__global__ void LIK_CHOL_BOUNDS chol_fused_kernel(CholArgs A) {
  extern __shared__ __align__(1024) double sm[];
#ifdef LIK_CTA_TRACE
  const unsigned long long t_start = gtimer();
#endif
  double* staging = sm;  // aliases the stage ring (used only between k-loops)
  double* Linv = sm + OFF_LINV;
  double* dlog = sm + OFF_DLOG;
  double* scal = sm + OFF_MISC;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + OFF_MBAR);
  uint64_t* mbar_empty = mbar + NSTAGE;
  int* flag = reinterpret_cast<int*>(sm + OFF_MBAR + 2 * NSTAGE);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int sel = w >> 2;           // the warp's tile row in a row block: 0 → ia, 1 → ib
  const int rbase = 16 * (w & 3);   // its 16 rows of that tile (all 64 columns)
  const bool mine_b = sel == 1;
  const int k = A.k0 + blockIdx.x;
  const SlotGeom g = A.g;
  const int nt = g.nt, r = g.r;
  double* ws = A.ws + (size_t)blockIdx.x * g.slot_d;
  const int mode = A.pc[k].mode;
  const double nugget = A.pc[k].nugget;

  if (mode == MODE_BAD) {
    write_point_failure(A, k, LIK_PT_BAD_PARAM);
    return;
  }
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) mbar_init(saddr(&mbar[s]), 1);
    for (int s = 0; s < NSTAGE; ++s) mbar_init(saddr(&mbar_empty[s]), NT / 32);
    flag[0] = flag[1] = flag[2] = 0;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  Pipe pp{sm, mbar, mbar_empty, 0u, policy_evict_first(), policy_evict_last()};
  const double tol = g.n * DBL_EPSILON * (1.0 + nugget);
  double logdet = 0.0;  // meaningful in thread 0
  const bool MG = g.merged;  // merged tail (see SlotGeom): tile row nt−1 also carries the B rows
  auto is_m = [&](int ti) { return MG && ti == nt - 1; };
  auto valid_rows = [&](int ti) {
    return ti == nt ? g.Ra : (is_m(ti) ? g.off + g.Ra : (ti == nt - 1 ? g.vlast : TB));
  };
  auto copy_rows = [&](int ti) { return ti == nt ? g.Ra : TB; };
  auto tile_ptr = [&](int ti, int tj) -> double* {
    double* t = ws + (size_t)(ti == nt ? g.ntri + tj : tri_index(ti, tj)) * TILE_D;
    LIK_CHECK_RANGE(t, TILE_D, ws, ws + g.slot_d);
    return t;
  };
  auto src = [&](int ti) -> Src {  // k-loop operand: the row panel of tile row ti
    if (ti < 0) return Src{nullptr, 0, nullptr, 0};
    if (is_m(ti)) return Src{tile_ptr(ti, 0), g.off, tile_ptr(nt, 0), g.Ra};
    return Src{tile_ptr(ti, 0), copy_rows(ti), nullptr, 0};
  };

  Acc acc;
  PH_INIT();
  // Row blocks run without CTA barriers (each warp solves its own rows from its
  // registers); the barriers are at a column's first row block (the diagonal tile is
  // staged in the ring's shared memory and factored by all warps) and at its end
  // (the proxy fence before the column's L tiles are read through TMA, and L_jj⁻¹
  // is rewritten by the next column).
  for (int j = 0; j < nt; ++j) {
    const int nrow = MG ? nt - j : nt - j + 1;  // tile rows j..nt-1 (and the augmented row)
    for (int rb = 0; rb < nrow; rb += 2) {
      const int ia = j + rb;
      const int ib = (rb + 1 < nrow) ? j + rb + 1 : -1;
#ifndef LIK_NO_PREFETCH
      if (tid == LEAD_TID && j > 0) {
        // the A_ij tiles are applied after the k-loop; start pulling them into L2 now
        prefetch_l2(tile_ptr(ia, j), (uint32_t)copy_rows(ia) * TB * 8);
        if (ib >= 0) prefetch_l2(tile_ptr(ib, j), (uint32_t)copy_rows(ib) * TB * 8);
      }
#endif
      const int ti = sel ? ib : ia;  // −1: this warp has no tile in a single-row block
      const int vmine = ti >= 0 ? valid_rows(ti) : 0;
      const int mlim = max(0, min(MI, (vmine - rbase + 7) >> 3));
#ifndef LIK_NO_DIAG_SKIP
      const int nlim = (rb == 0 && sel == 0) ? min(NI, (rbase >> 3) + 2) : NI;  // diagonal tile
#else
      const int nlim = NI;
#endif
      // acc = Σ_k L_ik L_jkᵀ − A_ij = −C
      frag_zero(acc);
      PH(0);
      if (j > 0)
        kloop(acc, pp, src(ia), src(ib), src(j), CHUNKS * j, mine_b, rbase, mlim, nlim, lane, ws,
              ws + g.slot_d);
      PH(1);
      if (ti >= 0) {
        if (is_m(ti))
          frag_sub_from2(acc, tile_ptr(ti, j), tile_ptr(nt, j), g.off, rbase, mlim, lane);
        else
          frag_sub_from(acc, tile_ptr(ti, j), rbase, mlim, lane);
      }
      if (rb == 0) {
        __syncthreads();  // every warp is past the k-loop: the ring's memory is free
        PH(2);
        if (sel == 0) frag_store<true>(acc, staging, rbase, mlim, lane);  // C_jj
        __syncthreads();
        PH(3);
        if (is_m(j)) {
          // merged last diagonal tile: partial factorisation; its Schur block is −BᵀV⁻¹B
          if (potrf_tail(staging, g.vlast, tol, dlog, flag, Linv)) {
            write_point_failure(A, k, LIK_PT_V_NOT_PD);
            return;
          }
          if (tid == LEAD_TID) {
            double s = 0.0;
            for (int c = 0; c < g.vlast; ++c) s += dlog[c];
            logdet += s;
          }
        } else {
          // diagonal tile: factor, log-determinant, inverse for this column's solves
          if (potrf_inv64(staging, valid_rows(j), tol, dlog, flag, Linv, sm + OFF_SCRATCH)) {
            write_point_failure(A, k, LIK_PT_V_NOT_PD);
            return;
          }
          if (tid == LEAD_TID) {
            double s = 0.0;
            for (int c = 0; c < valid_rows(j); ++c) s += dlog[c];
            logdet += s;
          }
          PH(4);
          // The staging tile and scratch alias the stage ring, and the next row
          // block's first chunks are written there by bulk copies (async proxy):
          // order this column's generic stores to them before those copies (a CTA
          // barrier alone does not order the two proxies).
          fence_proxy_async();
          __syncthreads();  // L_jj⁻¹ complete; the ring's memory is free again
          PH(5);
        }
      }
      // L_ij = C L_jj⁻ᵀ from the warp's registers (acc = −C gives −L_ij)
      if (ti >= 0 && !(rb == 0 && sel == 0) && mlim > 0) {
        trsm_reg(acc, Linv, lane);
        if (is_m(ti))
          frag_store2<true>(acc, tile_ptr(ti, j), tile_ptr(nt, j), g.off, rbase, mlim, lane);
        else
          frag_store<true>(acc, tile_ptr(ti, j), rbase, mlim, lane);
      }
      PH(6);
      // L tiles written in column j are read through TMA only from column j+1 on
      // (and by the final block), so one proxy fence per column suffices.
      if (rb + 2 >= nrow) {
        fence_proxy_async();
        __syncthreads();
      }
#ifdef LIK_DEBUG_RB_BARRIER
      else {
        __syncthreads();
      }
#endif
      PH(7);
    }
  }

  // ssqYX = BᵀV⁻¹B (Table 1, Step 4)
  if (!MG) {
    // separate augmented row: acc = Σ_k Z_k Z_kᵀ over its final block (warps 0-3)
    const int mlim = mine_b ? 0 : max(0, min(MI, (g.Ra - rbase + 7) >> 3));
    frag_zero(acc);
    kloop(acc, pp, src(nt), Src{nullptr, 0, nullptr, 0}, src(nt), CHUNKS * nt, false, rbase, mlim,
          NI, lane, ws, ws + g.slot_d);
    __syncthreads();
    frag_store<false>(acc, staging, rbase, mlim, lane);
    __syncthreads();
  }
  // Steps 5-8 and Eq. (profile)
  double* Cm = Linv;             // r×r, plain row-major with stride 64
  double* Q = staging + TILE_D;  // p×p Cholesky factor of XᵀV⁻¹X (stride 64)
  for (int e = tid; e < r * r; e += NT) {
    const int a = e / r, b = e % r;
    // merged: the Schur block (lower triangle) of the last diagonal tile is −BᵀV⁻¹B
    Cm[a * 64 + b] = MG ? -staging[sw_off(g.off + max(a, b), g.off + min(a, b))] : staging[sw_off(a, b)];
  }
  __syncthreads();
  point_epilogue(A, k, Cm, 64, Q, 64, logdet, flag, scal, tid, NT, LEAD_TID);
  PH(8);
  PH_FLUSH();
#ifdef LIK_CTA_TRACE
  if (tid == 0 && blockIdx.x < (1 << 16)) {
    g_lik_cta_trace[blockIdx.x][0] = t_start;
    g_lik_cta_trace[blockIdx.x][1] = gtimer();
    g_lik_cta_trace[blockIdx.x][2] = smid();
  }
#endif
}

}  // namespace

size_t chol_smem_bytes() { return (size_t)SMEM_D * sizeof(double); }

#ifdef LIK_CTA_TRACE
extern "C" int lik_debug_cta_trace(unsigned long long* out, int n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_lik_cta_trace, sizeof(unsigned long long) * 3 * (size_t)n);
  return 0;
}
#endif
#ifdef LIK_PHASE_TIMERS
extern "C" int lik_debug_phase_cycles(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, g_lik_phase, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_lik_phase, z, sizeof z);
  }
  return 0;
}
#endif
int chol_ctas_per_sm() { return 2; }

cudaError_t launch_chol(const CholArgs& a, int kw, cudaStream_t st) {
  const size_t smem = chol_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(chol_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  chol_fused_kernel<<<kw, NT, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace lik
