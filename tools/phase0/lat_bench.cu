// Dependent-chain latencies (one warp, cycles per op): DFMA, DMUL, double rsqrt(),
// FP32 rsqrt, SHFL (double), DMMA.8x8x4 (accumulator chain), LDS.64.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma8(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__global__ void lat(long long* out, double* sink, double seed) {
  __shared__ double sh[64];
  const int lane = threadIdx.x;
  sh[lane] = lane; sh[lane + 32] = lane + 32;
  __syncwarp();
  const int N = 1024;
  double x = seed + lane * 1e-3, y = 1.0;
  long long t0, t1;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = fma(x, 0.9999999, 1e-7); t1 = clock64(); out[0] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = x * 1.0000001; t1 = clock64(); out[1] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = rsqrt(x) + 0.5; t1 = clock64(); out[2] = t1 - t0;
  float f = (float)x;
  t0 = clock64(); for (int i = 0; i < N; ++i) f = rsqrtf(f) + 0.5f; t1 = clock64(); out[3] = t1 - t0;
  x += f;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31); t1 = clock64(); out[4] = t1 - t0;
  double c[2] = {x, y};
  t0 = clock64(); for (int i = 0; i < N; ++i) dmma8(c, 1.0000001, 0.5); t1 = clock64(); out[5] = t1 - t0;
  int idx = lane;
  t0 = clock64(); for (int i = 0; i < N; ++i) idx = (int)sh[idx & 63]; t1 = clock64(); out[6] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = x + 1e-9; t1 = clock64(); out[7] = t1 - t0;
  sink[lane] = x + c[0] + c[1] + idx;
}
int main() {
  long long* o; double* s; cudaMalloc(&o, 8 * 8); cudaMalloc(&s, 32 * 8);
  lat<<<1, 32>>>(o, s, 1.5); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, s, 1.5); cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, o, 64, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "dmul", "rsqrt_f64", "rsqrtf_f32", "shfl_f64", "dmma_8x8x4", "lds", "dadd"};
  for (int i = 0; i < 8; ++i) printf("{\"op\":\"%s\",\"cycles\":%.1f}\n", nm[i], h[i] / 1024.0);
  return 0;
}
