// Step microbenchmark, round 4: front multipliers explicitly loaded D steps ahead
// (C++ or volatile inline-PTX loads) to take the LDS latency off the pivot chain.
#include <cstdio>
#include <cuda_runtime.h>
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double2 lds2(const double* p) {
  double2 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return r;
}
__device__ __forceinline__ double lds1(const double* p) {
  double r;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return r;
}

template <int R, int KW, int STRIDE, bool BWD, int MODE, int D>
__global__ void k(double* out, long long* cyc, int rounds) {
  extern __shared__ double rec[];
  const int lane = threadIdx.x;
  for (int i = lane; i < 32 * STRIDE; i += 32) rec[i] = 1e-3 * ((i * 7) % 13) - 6e-3;
  for (int s = 0; s < 32; ++s) if (lane == 0) rec[s * STRIDE + KW] = 1.0;
  __syncwarp();
  double v[R];
  for (int r = 0; r < R; ++r) v[r] = 1.0 + lane + r;
  double f[4] = {1, 2, 3, 4};
  const int lim = KW - lane;
  double2 fm01[D + 1];
  double fm2[D + 1], fd[D + 1];
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    auto ld = [&](int s, int slot) {
      const double* rp = rec + s * STRIDE;
      if (MODE == 1) { fm01[slot] = lds2(rp); fm2[slot] = lds1(rp + 2); if (BWD) fd[slot] = lds1(rp + KW); }
      else { fm01[slot] = *reinterpret_cast<const double2*>(rp); fm2[slot] = rp[2]; if (BWD) fd[slot] = rp[KW]; }
    };
#pragma unroll
    for (int s = 0; s < D; ++s) ld(s, s % (D + 1));
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      if (s + D < 32) ld(s + D, (s + D) % (D + 1));
      const int slot = s % (D + 1);
      const int p = s & 3;
      const double* rp = rec + s * STRIDE;
      double bj = f[p];
      if (BWD) { bj *= fd[slot]; if (lane == s) v[0] = bj; }
      f[(p + 1) & 3] = fma(-fm01[slot].x, bj, f[(p + 1) & 3]);
      f[(p + 2) & 3] = fma(-fm01[slot].y, bj, f[(p + 2) & 3]);
      f[(p + 3) & 3] = fma(-fm2[slot], bj, f[(p + 3) & 3]);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = 32 * r + lane - s;
        const bool on = (r == 0 ? (lane > s) : true) && (32 * r - s <= lim);
        v[r] = fma(-(on ? rp[t - 1] : 0.0), bj, v[r]);
      }
      f[p] = __shfl_sync(FULL, v[(s + 4) >> 5], (s + 4) & 31);
    }
    double t = v[0];
    for (int r = 0; r + 1 < R; ++r) v[r] = v[r + 1];
    v[R - 1] = t * 0.5;
  }
  long long t1 = clock64();
  double sacc = f[0] + f[1] + f[2] + f[3];
  for (int r = 0; r < R; ++r) sacc += v[r];
  out[lane] = sacc;
  if (lane == 0) cyc[0] = t1 - t0;
}

template <int R, int KW, int STRIDE, bool BWD, int MODE, int D>
void run(const char* name, double* o, long long* c) {
  int rounds = 200;
  size_t sm = 32 * STRIDE * sizeof(double);
  auto kk = k<R, KW, STRIDE, BWD, MODE, D>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  kk<<<1, 32, sm>>>(o, c, rounds);
  kk<<<1, 32, sm>>>(o, c, rounds);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7.1f cycles/step\n", name, h / (32.0 * rounds));
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  run<4, 72, 74, false, 0, 1>("fwd R=4 C++ loads, D=1", o, c);
  run<4, 72, 74, false, 0, 3>("fwd R=4 C++ loads, D=3", o, c);
  run<4, 72, 74, false, 1, 1>("fwd R=4 asm loads, D=1", o, c);
  run<4, 72, 74, false, 1, 3>("fwd R=4 asm loads, D=3", o, c);
  run<6, 144, 146, true, 0, 3>("bwd R=6 C++ loads, D=3", o, c);
  run<6, 144, 146, true, 1, 3>("bwd R=6 asm loads, D=3", o, c);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
