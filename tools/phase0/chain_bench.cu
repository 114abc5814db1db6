// Microbenchmark: latency of the 8x8 pivot chain (factor + inverse, one warp) alone and
// next to other warps of the SM issuing (mode 1) DMMAs from registers, (mode 2) shared
// memory LDS.128/STS.128, (mode 3) DFMAs — on the chain warp's own SM sub-partition or
// not (neighbours on SMSP 3 or only on SMSPs 0-2).  Prints cycles per factor.
#include <cstdio>
#include <cuda_runtime.h>
// v2 = 2: the lead times a chain of 64 dependent DMMAs (cycles per 64) instead

__device__ __forceinline__ void dmma8(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ int toff(int a, int b) { return a * 8 + (b ^ ((a & 2) << 1)); }

__device__ __forceinline__ void factor8(double* Skk, double* Wn, double* piv, double tol, int* bad) {
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
    if (l == c) { a[c] = pv * rinv; my_piv = pv; my_rinv = rinv; }
    else if (l > c) a[c] *= rinv;
    if (c + 1 < 8) { const double pn = a[c + 1] - a[c] * a[c]; piv_next = __shfl_sync(0xffffffffu, pn, c + 1); }
#pragma unroll
    for (int m = 0; m < 8; ++m)
      if (m > c) { const double lm = __shfl_sync(0xffffffffu, a[c], m); if (l >= m) a[m] -= a[c] * lm; }
  }
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (i == l) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] *= __shfl_sync(0xffffffffu, my_rinv, i);
#pragma unroll
    for (int m = 0; m < 8; ++m) if (m > i) x[m] -= __shfl_sync(0xffffffffu, a[i], m) * x[i];
  }
  if (lane < 8) {
#pragma unroll
    for (int m = 0; m < 8; ++m) Wn[toff(m, l)] = -x[m];
    piv[l] = my_piv;
  }
  if (lane == 0 && fail) *bad = 1;
}


// v2: every lane holds the whole lower triangle (36 doubles) and factors it redundantly:
// no shuffles; the only serial chain is rsqrt -> scale -> update of the next pivot.
__device__ __forceinline__ void factor8v2(const double* Skk, double* Wn, double* piv, double tol, int* bad) {
  const int lane = threadIdx.x & 31, l = lane & 7;
  double a[36];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) a[i * (i + 1) / 2 + j] = -Skk[toff(i, j)];
  int fail = 0;
  double rv[8], mypiv = 1.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double d = a[c * (c + 1) / 2 + c];
    fail |= !(d > tol);
    const double r = rsqrt(d);
    rv[c] = r;
    if (l == c) mypiv = d;
    a[c * (c + 1) / 2 + c] = d * r;
#pragma unroll
    for (int i = c + 1; i < 8; ++i) a[i * (i + 1) / 2 + c] *= r;
#pragma unroll
    for (int i = c + 1; i < 8; ++i)
#pragma unroll
      for (int j = c + 1; j <= i; ++j) a[i * (i + 1) / 2 + j] -= a[i * (i + 1) / 2 + c] * a[j * (j + 1) / 2 + c];
  }
  // column l of W = L^-1: x_i = (delta_il - sum_{m<i} L_im x_m) / L_ii
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double t = (i == l) ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < i; ++m) t -= a[i * (i + 1) / 2 + m] * x[m];
    x[i] = t * rv[i];
  }
  if (lane < 8) {
#pragma unroll
    for (int m = 0; m < 8; ++m) Wn[toff(m, l)] = -x[m];
    piv[l] = mypiv;
  }
  if (lane == 0 && fail) *bad = 1;
}

__global__ void __launch_bounds__(512, 1) bench(int mode, int smsp3, int iters, long long* out, double* sink, int v2) {
  __shared__ double S[64], W[64], piv[8], buf[4 * 1024];
  __shared__ int bad;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 64) S[tid] = (tid % 9 == 0) ? -10.0 : -0.5;  // −A, A SPD (diag 10, off 0.5)
  if (tid == 0) { bad = 0; done = 0; }
  __syncthreads();
  const int lead = 15;
  if (warp == lead) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (v2 == 2) {
        double c[2] = {S[lane], S[lane + 32]};
#pragma unroll 1
        for (int q = 0; q < 64; ++q) dmma8(c, 1.0000001, 0.5);
        if (lane < 8) W[lane] = c[0] + c[1];
      } else if (v2) factor8v2(S, W, piv, 1e-12, &bad); else factor8(S, W, piv, 1e-12, &bad);
      __syncwarp();
      if (lane < 8) S[toff(lane, lane)] = -10.0 - 1e-9 * it;  // keep a dependency
      __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) { out[blockIdx.x] = (t1 - t0) / iters; done = 1; }
  } else if (mode != 0 && ((warp & 3) != 3 || smsp3)) {
    double acc = 0.0;
    double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    double a = 1.0 + lane, b = 0.5;
    int k = 0;
    while (!done) {
      if (mode == 1) {
#pragma unroll
        for (int q = 0; q < 16; ++q) dmma8(c[q & 3], a, b);
      } else if (mode == 2) {
        double2* p = reinterpret_cast<double2*>(buf) + ((warp * 32 + lane) & 2047);
#pragma unroll
        for (int q = 0; q < 8; ++q) { double2 v = p[(q * 512) & 2047]; acc += v.x; p[((q + 1) * 512) & 2047] = v; }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) acc = fma(acc, 0.999, 1.0);
      }
      ++k;
    }
    sink[blockIdx.x * 512 + tid] = acc + c[0][0] + c[1][1] + c[2][0] + c[3][1] + k;
  }
}

int main() {
  long long* out; double* sink;
  cudaMalloc(&out, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 512 * sizeof(double));
  const char* names[] = {"alone", "dmma", "lds/sts", "dfma"};
  for (int v2 = 0; v2 < 3; ++v2)
  for (int mode = 0; mode < 4; ++mode)
    for (int s3 = 0; s3 < 2; ++s3) {
      if (mode == 0 && s3) continue;
      if (s3 && mode == 1) continue;
      bench<<<148, 512>>>(mode, s3, 200, out, sink, v2);
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
      double m = 0; for (int i = 0; i < 148; ++i) m += h[i]; m /= 148;
      printf("{\"v2\":%d,\"neighbours\":\"%s\",\"on_lead_smsp\":%d,\"cycles_per_factor8\":%.0f}\n", v2, names[mode], s3, m);
    }
  return 0;
}
