// Microbenchmark: the chol_fused k-loop's synchronisation protocol (modes 1-2 without TMA).
// The inner loop is the production one (8 swizzled LDS.64 + 16 DMMA.8x8x4 per
// k-step, 4 k-steps per 64x16 chunk, fragments of step t+1 loaded before step t's
// DMMAs); the stage ring lives in shared memory and is never rewritten.
//   mode 0: no synchronisation (inner loop only)
//   mode 1: per chunk, every warp waits on the stage's "full" mbarrier and
//           releases it on an "empty" mbarrier (8 warp arrivals); the lead warp
//           (warp 7) waits for empty(q-1) and then "refills" stage q-1+NSTAGE by
//           arriving on its full barrier (count 1) — the production protocol with
//           the copy latency set to zero.
//   mode 2: mode 1 with the lead role rotated over the warps (warp q % 8).
//   mode 3: mode 1 with real refills: the lead warp arms the full barrier with
//           expect_tx and issues three 8 KB cp.async.bulk copies (L2-resident
//           source) per chunk, as chol_fused does.
//   mode 4: mode 3 split into k-loop calls of CALL_Q chunks (chol_fused averages
//           42 per row block at C4), each with its own prologue (three copies,
//           wait for the first) and a __syncthreads after it.
// Usage: dmma_sync [ctas_per_sm]   prints one JSON line per mode.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int KC = 16, NSTAGE = 3, CHUNK_D = 64 * KC, STAGE_D = 3 * CHUNK_D, CALL_Q = 42;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  }
}

template <int MODE, bool T16 = false>
__global__ void __launch_bounds__(256, 2) k(double* out, int nq, const double* src) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NSTAGE * STAGE_D);
  uint64_t* empty = full + NSTAGE;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, wr = w >> 1, wc = w & 1;
  for (int e = tid; e < NSTAGE * STAGE_D; e += 256) sm[e] = 1e-3 * (e % 7);
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) { mbar_init(saddr(&full[s]), 1); mbar_init(saddr(&empty[s]), 8); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // T16: warp tile 16 rows x 64 columns (full rows); else 32 x 32
  constexpr int MI = T16 ? 2 : 4, NI = T16 ? 8 : 4;
  const int rbase = T16 ? 16 * (w & 3) : (wr & 1) * 32, cbase = T16 ? 0 : wc * 32;
  const int lr = lane >> 2, lc = lane & 3, sw = (lr & 3) << 2;
  const int aoff = (T16 ? w >= 4 : wr >= 2) ? CHUNK_D : 0;
  double acc[MI][NI][2] = {};
  double fa[2][MI], fb[2][NI];
  auto load = [&](double (&a)[MI], double (&b)[NI], const double* st, int kk) {
    const int kcol = ((kk * 4) ^ sw) + lc;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) a[mi] = st[aoff + (rbase + mi * 8 + lr) * KC + kcol];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) b[ni] = st[2 * CHUNK_D + (cbase + ni * 8 + lr) * KC + kcol];
  };
  auto lead = [&](int q) { return MODE == 2 ? (q % 8) : 7; };
  // prologue: the "copies" of the first NSTAGE chunks land immediately
  auto refill = [&](int s) {
    if (MODE >= 3) {
      const uint32_t bar = saddr(&full[s]);
      mbar_expect_tx(bar, 3 * CHUNK_D * 8);
      const double* g = src + (size_t)(blockIdx.x % 64) * STAGE_D;
      for (int c = 0; c < 3; ++c) bulk_g2s(saddr(sm + s * STAGE_D + c * CHUNK_D), g + c * CHUNK_D, CHUNK_D * 8, bar);
    } else {
      mbar_arrive(saddr(&full[s]));
    }
  };
  const int calls = MODE == 4 ? (nq + CALL_Q - 1) / CALL_Q : 1;
  uint32_t seq = 0;  // chunks consumed so far (ring position and barrier phases)
  for (int call = 0; call < calls; ++call) {
    const int nc = MODE == 4 ? min(CALL_Q, nq - call * CALL_Q) : nq;
    auto slot = [&](int q) { return (seq + q) % NSTAGE; };
    auto par = [&](int q) { return ((seq + q) / NSTAGE) & 1; };
    if (MODE && tid == 0)
      for (int q = 0; q < NSTAGE && q < nc; ++q) refill(slot(q));
    if (MODE) mbar_wait(saddr(&full[slot(0)]), par(0));
    load(fa[0], fb[0], sm + slot(0) * STAGE_D, 0);
    for (int q = 0; q < nc; ++q) {
      if (MODE && w == lead(q) && lane == 0 && q >= 1 && q - 1 + NSTAGE < nc) {
        mbar_wait(saddr(&empty[slot(q - 1)]), par(q - 1));
        refill(slot(q - 1 + NSTAGE));
      }
      __syncwarp();
      const double* st = sm + slot(q) * STAGE_D;
#pragma unroll
      for (int kk = 0; kk < KC / 4; ++kk) {
        const int cur = kk & 1;
        if (kk + 1 < KC / 4) load(fa[cur ^ 1], fb[cur ^ 1], st, kk + 1);
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], fa[cur][mi], fb[cur][ni]);
      }
      if (MODE) {
        __syncwarp();
        if (lane == 0) mbar_arrive(saddr(&empty[slot(q)]));
      }
      if (q + 1 < nc) {
        if (MODE) mbar_wait(saddr(&full[slot(q + 1)]), par(q + 1));
        load(fa[0], fb[0], sm + slot(q + 1) * STAGE_D, 0);
      }
    }
    seq += nc;
    if (MODE == 4) __syncthreads();
  }
  double s = 0;
  for (int mi = 0; mi < MI; ++mi)
    for (int ni = 0; ni < NI; ++ni) s += acc[mi][ni][0] + acc[mi][ni][1];
  if (s == 1234.5) out[0] = s;
  // every issued copy is for a chunk < nq, which all warps waited on: none is in flight here
}

template <int MODE, bool T16 = false>
void run(int bpsm, double* o) {
  const size_t smem = NSTAGE * STAGE_D * 8 + 64;
  cudaFuncSetAttribute(k<MODE, T16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = 148 * bpsm, nq = 20000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  static double* src = nullptr;
  if (!src) {
    cudaMalloc(&src, (size_t)64 * STAGE_D * 8);
    cudaMemset(src, 0, (size_t)64 * STAGE_D * 8);
  }
  k<MODE, T16><<<grid, 256, smem>>>(o, 100, src);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  k<MODE, T16><<<grid, 256, smem>>>(o, nq, src);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = (double)grid * 8 * nq * 4 * 16 * 512.0;
  printf("{\"kind\":\"dmma_sync\",\"mode\":%d,\"tile\":\"%s\",\"ctas_per_sm\":%d,\"tflops\":%.2f,\"err\":\"%s\"}\n", MODE,
         T16 ? "16x64" : "32x32", bpsm, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  double* o;
  cudaMalloc(&o, 8);
  for (int bpsm = 1; bpsm <= 2; ++bpsm) {
    run<0>(bpsm, o);
    run<1>(bpsm, o);
    run<2>(bpsm, o);
    run<3>(bpsm, o);
    run<4>(bpsm, o);
    run<0, true>(bpsm, o);
    run<4, true>(bpsm, o);
  }
  return 0;
}
