// Does FP64 FMA slow down with subnormal operands/results on this GPU?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters, double a, double b, double x0) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = x0 * (1 + k * 1e-3);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], b, a);
  }
  long long t1 = clock64();
  double s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  long long h; int it = 4096;
  double cases[][3] = {{1e-9, 0.999999, 1.0}, {0.0, 1.0, 1e-310}, {1e-310, 1.0, 1e-310}, {0.0, 0.5, 1e-300}};
  const char* names[] = {"normal", "subnormal x (b=1, a=0)", "subnormal x and a", "decaying to subnormal"};
  for (int q = 0; q < 4; ++q) {
    k<<<1, 32>>>(o, c, it, cases[q][0], cases[q][1], cases[q][2]);
    k<<<1, 32>>>(o, c, it, cases[q][0], cases[q][1], cases[q][2]);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %.2f cycles per DFMA\n", names[q], h / (double)(it * 8));
  }
  return 0;
}
