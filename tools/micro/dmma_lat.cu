// DMMA (mma.sync m8n8k4 f64) latency / throughput on one SM: a dependent
// chain in one warp, then k independent chains per warp with w warps.
#include <cstdio>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int K>
__global__ void chains(int iters, double* out, long long* cyc) {
  double acc[K][2];
  for (int k = 0; k < K; ++k) acc[k][0] = acc[k][1] = threadIdx.x * 1e-3;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) dmma(acc[k], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < K; ++k) s += acc[k][0] + acc[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  long long h;
  const int iters = 4096;
  chains<1><<<1, 32>>>(iters, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("1 warp, 1 chain: %.1f cycles per DMMA (latency)\n", (double)h / iters);
  chains<4><<<1, 32>>>(iters, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("1 warp, 4 chains: %.1f cycles per DMMA\n", (double)h / iters / 4);
  chains<8><<<1, 32>>>(iters, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("1 warp, 8 chains: %.1f cycles per DMMA\n", (double)h / iters / 8);
  chains<8><<<1, 128>>>(iters, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("4 warps x 8 chains: %.2f cycles per DMMA per SM\n", (double)h / iters / 32);
  chains<8><<<1, 256>>>(iters, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("8 warps x 8 chains: %.2f cycles per DMMA per SM\n", (double)h / iters / 64);
  chains<8><<<1, 512>>>(iters, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("16 warps x 8 chains: %.2f cycles per DMMA per SM\n", (double)h / iters / 128);
  return 0;
}
