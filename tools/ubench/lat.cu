// Dependent-chain latency probes on one warp (cycles per op): DFMA, DADD, DMUL,
// fp64 SHFL (2x32-bit), LDS.64, BAR.SYNC with 8 warps, fp64 division, sqrt.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[256];
  const int t = threadIdx.x;
  sm[t] = a + t;
  __syncthreads();
  double x = a + t * 1e-9, y = b;
  long long c0, c1;
  // DFMA chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    x = fma(x, y, a); x = fma(x, y, a); x = fma(x, y, a); x = fma(x, y, a);
  }
  c1 = clock64();
  if (t == 0) cyc[0] = (c1 - c0);
  // DADD chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) { x = x + y; x = x + a; x = x + y; x = x + a; }
  c1 = clock64();
  if (t == 0) cyc[1] = (c1 - c0);
  // SHFL chain (fp64)
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    x = __shfl_xor_sync(0xffffffff, x, 1); x = __shfl_xor_sync(0xffffffff, x, 2);
    x = __shfl_xor_sync(0xffffffff, x, 4); x = __shfl_xor_sync(0xffffffff, x, 8);
  }
  c1 = clock64();
  if (t == 0) cyc[2] = (c1 - c0);
  // LDS chain (address depends on loaded value)
  int idx = t;
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    idx = (int)sm[idx & 255] & 255; idx = (int)sm[idx] & 255; idx = (int)sm[idx] & 255; idx = (int)sm[idx] & 255;
  }
  c1 = clock64();
  if (t == 0) cyc[3] = (c1 - c0);
  // BAR chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) { __syncthreads(); __syncthreads(); __syncthreads(); __syncthreads(); }
  c1 = clock64();
  if (t == 0) cyc[4] = (c1 - c0);
  // division chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) { x = a / x; x = a / x; x = a / x; x = a / x; }
  c1 = clock64();
  if (t == 0) cyc[5] = (c1 - c0);
  // sqrt chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) { x = sqrt(x + a); x = sqrt(x + a); x = sqrt(x + a); x = sqrt(x + a); }
  c1 = clock64();
  if (t == 0) cyc[6] = (c1 - c0);
  // STS -> BAR -> LDS round trip (cross-warp value exchange)
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    sm[t] = x; __syncthreads(); x = sm[(t + 32) & 255] + 1.0; __syncthreads();
  }
  c1 = clock64();
  if (t == 0) cyc[7] = (c1 - c0);
  // DMUL chain
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) { x = x * y; x = x * y; x = x * y; x = x * y; }
  c1 = clock64();
  if (t == 0) cyc[8] = (c1 - c0);
  out[t] = x + idx;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 256 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const int n = 1000;
  const char* names[] = {"DFMA", "DADD", "SHFL64", "LDS", "BAR(8 warps)", "DDIV", "DSQRT(+DADD)", "STS+BAR+LDS+DADD+BAR", "DMUL"};
  for (int threads : {32, 256}) {
    probe<<<1, threads>>>(out, cyc, 1.0000001, 0.9999999, n);
    cudaDeviceSynchronize();
    probe<<<1, threads>>>(out, cyc, 1.0000001, 0.9999999, n);
    cudaDeviceSynchronize();
    printf("threads=%d\n", threads);
    for (int i = 0; i < 9; ++i) printf("  %-24s %7.1f cycles/op\n", names[i], (double)cyc[i] / (4.0 * n) * (i == 7 ? 4.0 : 1.0));
  }
  return 0;
}
