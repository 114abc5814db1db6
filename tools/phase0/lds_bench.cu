// Shared-memory load throughput by width and address pattern (cycles per warp-load, one
// SM fully occupied): broadcast (all lanes one address), 4 distinct addresses (8 lanes
// each), fully distinct.  Decides how the Matérn build should fetch its per-interval
// coefficients.
#include <cstdio>
#include <cuda_runtime.h>
template <int W, int PAT>
__global__ void __launch_bounds__(1024) k(long long* out, double* sink, int iters) {
  __shared__ __align__(16) double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += 1024) sm[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int base = PAT == 0 ? 0 : (PAT == 1 ? (lane >> 3) * 18 : lane * 18);  // stride 18 doubles = 144 B
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int o = base + ((it * 2) & 1023);
    if (W == 16) {
      const double2 v = *reinterpret_cast<const double2*>(sm + (o & ~1));
      acc += v.x + v.y;
    } else if (W == 8) {
      acc += sm[o];
    } else {
      acc += (double)reinterpret_cast<const float*>(sm)[o];
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * 1024 + threadIdx.x] = acc;
}
template <int W, int PAT>
void run(const char* name, long long* d, double* s) {
  const int iters = 4096;
  k<W, PAT><<<148, 1024>>>(d, s, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double m = 0; for (int i = 0; i < 148; ++i) m += h[i]; m /= 148;
  // 32 warps per SM each issue `iters` loads
  printf("{\"width\":%d,\"pattern\":\"%s\",\"cycles_per_warp_load_per_SM\":%.3f}\n", W, name, m / (iters * 32.0));
}
int main() {
  long long* d; double* s;
  cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 148 * 1024 * 8);
  run<16, 0>("broadcast", d, s); run<16, 1>("4 addresses", d, s); run<16, 2>("32 distinct", d, s);
  run<8, 0>("broadcast", d, s); run<8, 1>("4 addresses", d, s); run<8, 2>("32 distinct", d, s);
  run<4, 0>("broadcast", d, s); run<4, 1>("4 addresses", d, s); run<4, 2>("32 distinct", d, s);
  return 0;
}
