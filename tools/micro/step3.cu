// Step microbenchmark, round 3: front corrections accumulated separately so the
// fetch shuffle has 3 steps of slack; pivot = fetched + corr.
#include <cstdio>
#include <cuda_runtime.h>
constexpr unsigned FULL = 0xffffffffu;

template <int R, int KW, int STRIDE, bool BWD>
__global__ void k(double* out, long long* cyc, int rounds) {
  extern __shared__ double rec[];
  const int lane = threadIdx.x;
  for (int i = lane; i < 32 * STRIDE; i += 32) rec[i] = 1e-3 * ((i * 7) % 13) - 6e-3;
  for (int s = 0; s < 32; ++s) if (lane == 0) rec[s * STRIDE + KW] = 1.0;
  __syncwarp();
  double v[R];
  for (int r = 0; r < R; ++r) v[r] = 1.0 + lane + r;
  // slot q (q = 0..3): fetched value g[q] and correction c[q] of front row j+q (rotating roles)
  double g[4] = {1, 2, 3, 4}, c[4] = {0, 0, 0, 0};
  const int lim = KW - lane;
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      const int p = s & 3;
      const double* rp = rec + s * STRIDE;
      double bj = g[p] + c[p];
      if (BWD) bj *= rp[KW];
      if (lane == s) v[0] = bj;
      c[(p + 1) & 3] = fma(-rp[0], bj, c[(p + 1) & 3]);
      c[(p + 2) & 3] = fma(-rp[1], bj, c[(p + 2) & 3]);
      c[(p + 3) & 3] = fma(-rp[2], bj, c[(p + 3) & 3]);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = 32 * r + lane - s;
        const bool on = (r == 0 ? (lane > s) : true) && (32 * r - s <= lim);
        v[r] = fma(-(on ? rp[t - 1] : 0.0), bj, v[r]);
      }
      // row j+4: distributed value after this step; its later updates go to c[p]
      g[p] = __shfl_sync(FULL, v[(s + 4) >> 5], (s + 4) & 31);
      c[p] = 0.0;
    }
    double t = v[0];
    for (int r = 0; r + 1 < R; ++r) v[r] = v[r + 1];
    v[R - 1] = t * 0.5;
  }
  long long t1 = clock64();
  double sacc = 0;
  for (int q = 0; q < 4; ++q) sacc += g[q] + c[q];
  for (int r = 0; r < R; ++r) sacc += v[r];
  out[lane] = sacc;
  if (lane == 0) cyc[0] = t1 - t0;
}

template <int R, int KW, int STRIDE, bool BWD>
void run(const char* name, double* o, long long* c) {
  int rounds = 200;
  size_t sm = 32 * STRIDE * sizeof(double);
  cudaFuncSetAttribute(k<R, KW, STRIDE, BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<R, KW, STRIDE, BWD><<<1, 32, sm>>>(o, c, rounds);
  k<R, KW, STRIDE, BWD><<<1, 32, sm>>>(o, c, rounds);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %7.1f cycles/step\n", name, h / (32.0 * rounds));
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  run<6, 144, 146, true>("bwd R=6 deferred-front", o, c);
  run<4, 72, 74, false>("fwd R=4 deferred-front", o, c);
  run<2, 24, 26, false>("fwd R=2 deferred-front", o, c);
  run<10, 272, 274, true>("bwd R=10 deferred-front", o, c);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
