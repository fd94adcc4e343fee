// Step-structure microbenchmark, round 2: straight-line rounds, prefetched multipliers.
#include <cstdio>
#include <cuda_runtime.h>
constexpr unsigned FULL = 0xffffffffu;

template <int R, int KW, int STRIDE, bool BWD, bool PREF>
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
  double mA[R + 4], mB[R + 4];
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    auto load = [&](double (&m)[R + 4], int s) {
      const double* rp = rec + s * STRIDE;
      m[0] = rp[0]; m[1] = rp[1]; m[2] = rp[2]; m[3] = BWD ? rp[KW] : 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = 32 * r + lane - s;
        const bool on = (r == 0 ? (lane > s) : true) && (32 * r - s <= lim);
        m[4 + r] = on ? rp[t - 1] : 0.0;
      }
    };
    if (PREF) load(mA, 0);
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      const int p = s & 3;
      double* m = (s & 1) ? mB : mA;
      if (PREF) { if (s < 31) load((s & 1) ? mA : mB, s + 1); }
      else load((s & 1) ? mB : mA, s);
      double bj = f[p];
      if (BWD) { bj *= m[3]; if (lane == s) v[0] = bj; }
      f[(p + 1) & 3] = fma(-m[0], bj, f[(p + 1) & 3]);
      f[(p + 2) & 3] = fma(-m[1], bj, f[(p + 2) & 3]);
      f[(p + 3) & 3] = fma(-m[2], bj, f[(p + 3) & 3]);
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = fma(-m[4 + r], bj, v[r]);
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

template <int R, int KW, int STRIDE, bool BWD, bool PREF>
void run(const char* name, double* o, long long* c) {
  int rounds = 200;
  size_t sm = 32 * STRIDE * sizeof(double);
  cudaFuncSetAttribute(k<R, KW, STRIDE, BWD, PREF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<R, KW, STRIDE, BWD, PREF><<<1, 32, sm>>>(o, c, rounds);
  k<R, KW, STRIDE, BWD, PREF><<<1, 32, sm>>>(o, c, rounds);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %7.1f cycles/step\n", name, h / (32.0 * rounds));
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  run<6, 144, 146, true, false>("bwd R=6 select, in-step loads", o, c);
  run<6, 144, 146, true, true>("bwd R=6 select, prefetched", o, c);
  run<4, 72, 74, false, false>("fwd R=4 select, in-step loads", o, c);
  run<4, 72, 74, false, true>("fwd R=4 select, prefetched", o, c);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
