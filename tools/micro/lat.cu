// Latency microbenchmark (single warp, dependent chains) for the band-solve design.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters, double a, double b) {
  __shared__ double sm[64];
  int lane = threadIdx.x;
  sm[lane] = a + lane; sm[lane + 32] = b;
  __syncwarp();
  double x = a + lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, b, a);            // DFMA chain
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffff, x, (i + 1) & 31);  // SHFL chain (64-bit)
  long long t2 = clock64();
  int idx = lane;
  for (int i = 0; i < iters; ++i) { double v = sm[idx & 63]; idx = (int)v & 63; x += v; }  // LDS chain
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) { double y = __shfl_sync(0xffffffff, x, i & 31); x = fma(y, b, x); }  // shfl+dfma
  long long t4 = clock64();
  float f = (float)x;
  for (int i = 0; i < iters; ++i) f = fmaf(f, (float)b, (float)a);  // FFMA chain
  long long t5 = clock64();
  out[lane] = x + f;
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  int it = 4096;
  k<<<1, 32>>>(o, c, it, 1e-9, 0.999999);
  k<<<1, 32>>>(o, c, it, 1e-9, 0.999999);
  long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  printf("cycles/iter: DFMA %.1f  SHFL64 %.1f  LDS %.1f  SHFL64+DFMA %.1f  FFMA %.1f\n", h[0]/(double)it, h[1]/(double)it, h[2]/(double)it, h[3]/(double)it, h[4]/(double)it);
  return 0;
}
