// FP64 issue-rate microbenchmark: one warp, K independent DFMA chains; and LDS.64 throughput.
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void dfma(double* out, long long* cyc, int iters, double a, double b) {
  double x[K];
  for (int k = 0; k < K; ++k) x[k] = a + threadIdx.x + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = fma(x[k], b, a);
  }
  long long t1 = clock64();
  double s = 0; for (int k = 0; k < K; ++k) s += x[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lds(double* out, long long* cyc, int iters) {
  __shared__ double sm[2048];
  for (int i = threadIdx.x; i < 2048; i += 32) sm[i] = i;
  __syncwarp();
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  const double* p = sm + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    int o = (i & 7) * 128;
    s0 += p[o]; s1 += p[o + 32]; s2 += p[o + 64]; s3 += p[o + 96];
  }
  long long t1 = clock64();
  out[threadIdx.x] = s0 + s1 + s2 + s3;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 64);
  int it = 4096; long long h;
#define RUN(K) dfma<K><<<1, 32>>>(o, c, it, 1e-9, 0.999999); dfma<K><<<1, 32>>>(o, c, it, 1e-9, 0.999999); \
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("1 warp, %2d chains: %.2f cycles per DFMA instr\n", K, h / (double)(it * K));
  RUN(1) RUN(2) RUN(4) RUN(8) RUN(16)
  dfma<16><<<1, 128>>>(o, c, it, 1e-9, 0.999999); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("4 warps x 16 chains: %.2f cycles per DFMA instr per warp\n", h / (double)(it * 16));
  dfma<16><<<1, 512>>>(o, c, it, 1e-9, 0.999999); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("16 warps x 16 chains: %.2f cycles per DFMA instr per warp\n", h / (double)(it * 16));
  lds<<<1, 32>>>(o, c, it); lds<<<1, 32>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("1 warp LDS.64 (+DADD): %.2f cycles per LDS\n", h / (double)(it * 4));
  return 0;
}
