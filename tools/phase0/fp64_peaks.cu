// Phase-0 microbenchmark: FP64 pipe peaks on sm_100a (DMMA.8x8x4 vs DFMA),
// plus a check of the m8n8k4.f64 fragment layout used by the Cholesky kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c][0] = threadIdx.x * 1e-9; acc[c][1] = c * 1e-9; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c][0], acc[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// half the warps DMMA, half DFMA (same FMA count per warp-iteration scaled)
__global__ void k_mixed(double* out, int iters, double a, double b) {
  int w = threadIdx.x >> 5;
  double s = 0;
  if (w & 1) {
    double acc[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) { acc[c][0] = 0; acc[c][1] = 0; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c) dmma(acc[c][0], acc[c][1], a, b);
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
  } else {
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = c;
    // 8 DMMA = 2048 FMA per warp = 64 per lane -> 8 iters of 8 DFMA
    for (int it = 0; it < iters * 8; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], a, b);
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c];
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void k_layout(const double* A, const double* B, double* C) {
  // A 8x4 row-major, B 4x8 row-major (k x n), C 8x8 row-major
  int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];
  double b = B[(l & 3) * 8 + (l >> 2)];
  double c0 = 0, c1 = 0;
  dmma(c0, c1, a, b);
  C[(l >> 2) * 8 + 2 * (l & 3) + 0] = c0;
  C[(l >> 2) * 8 + 2 * (l & 3) + 1] = c1;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"smem_per_block_optin\":%zu,\"l2\":%d,\"clock_khz\":%d}\n",
         prop.name, prop.multiProcessorCount, prop.sharedMemPerBlockOptin, prop.l2CacheSize, clk_khz);
  // layout check
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = (i * 7 % 11) - 5; hB[i] = (i * 5 % 13) - 6; }
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) {
    double s = 0; for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c]; ref[r * 8 + c] = s; }
  double *dA, *dB, *dC, *dout;
  CK(cudaMalloc(&dA, 256)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dC, 512)); CK(cudaMalloc(&dout, 64));
  CK(cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice));
  k_layout<<<1, 32>>>(dA, dB, dC); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost));
  int bad = 0; for (int i = 0; i < 64; ++i) bad += (hC[i] != ref[i]);
  printf("{\"dmma_layout_mismatches\":%d}\n", bad);

  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = prop.multiProcessorCount;
  const int iters = 20000;
  for (int bpsm = 1; bpsm <= 4; bpsm *= 2) {
    for (int threads = 128; threads <= 512; threads *= 2) {
      int grid = sms * bpsm;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_dmma<8><<<grid, threads>>>(dout, iters, 1.0000001, 0.999999);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fma = (double)grid * (threads / 32) * iters * 8 * 256.0;
        if (rep) printf("{\"kind\":\"dmma\",\"bpsm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", bpsm, threads, ms, 2 * fma / ms / 1e9);
      }
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_dfma<8><<<grid, threads>>>(dout, iters, 1.0000001, 0.999999);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fma = (double)grid * threads * iters * 8.0;
        if (rep) printf("{\"kind\":\"dfma\",\"bpsm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", bpsm, threads, ms, 2 * fma / ms / 1e9);
      }
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_mixed<<<grid, threads>>>(dout, iters / 2, 1.0000001, 0.999999);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fma = (double)grid * (threads / 32) * (iters / 2) * 8 * 256.0;
        if (rep) printf("{\"kind\":\"mixed\",\"bpsm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", bpsm, threads, ms, 2 * fma / ms / 1e9);
      }
    }
  }
  // long sustained DMMA run (~4 s) for clocks under FP64 load
  {
    int grid = sms * 2, threads = 256;
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) k_dmma<8><<<grid, threads>>>(dout, iters * 5, 1.0000001, 0.999999);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = 20.0 * grid * (threads / 32) * iters * 5 * 8 * 256.0;
    printf("{\"kind\":\"dmma_sustained\",\"ms\":%.3f,\"tflops\":%.2f}\n", ms, 2 * fma / ms / 1e9);
  }
  return 0;
}
