// Step microbenchmark, round 5: the candidate production step.  Predicates come
// from per-sweep lane bitmasks (one LOP3 each), only the edge registers are
// masked (r = 0, R-2, R-1; middle registers are always inside the band because
// R = 1 + ceil(kw/32)), predicated LDS + DFMA, LDS.128 for the front.
#include <cstdio>
#include <cuda_runtime.h>
constexpr unsigned FULL = 0xffffffffu;

template <int R, int KW, int STRIDE, bool BWD, bool DEFER>
__global__ void k(double* out, long long* cyc, int rounds) {
  extern __shared__ double rec[];
  const int lane = threadIdx.x;
  for (int i = lane; i < 32 * STRIDE; i += 32) rec[i] = 1e-3 * ((i * 7) % 13) - 6e-3;
  for (int s = 0; s < 32; ++s) if (lane == 0) rec[s * STRIDE + KW] = 1.0;
  __syncwarp();
  const int kw = KW + (int)(out[40] * 0);  // runtime kw like production
  // mask[r] bit s: multiplier t = 32r + lane - s in [1, kw]
  unsigned mask[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    unsigned m = 0;
    for (int s = 0; s < 32; ++s) { int t = 32 * r + lane - s; if (t >= 1 && t <= kw) m |= 1u << s; }
    mask[r] = m;
  }
  double v[R];
  for (int r = 0; r < R; ++r) v[r] = 1.0 + lane + r;
  double f[4] = {1, 2, 3, 4}, c[4] = {0, 0, 0, 0};
  const double* base = rec + lane - 1;
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      const int p = s & 3;
      const double* rp = rec + s * STRIDE;
      double bj = DEFER ? f[p] + c[p] : f[p];
      if (BWD) {
        bj *= rp[kw];
        if (lane == s) v[0] = bj;
      }
      const double2 m01 = *reinterpret_cast<const double2*>(rp);
      const double m2 = rp[2];
      if (DEFER) {
        c[(p + 1) & 3] = fma(-m01.x, bj, c[(p + 1) & 3]);
        c[(p + 2) & 3] = fma(-m01.y, bj, c[(p + 2) & 3]);
        c[(p + 3) & 3] = fma(-m2, bj, c[(p + 3) & 3]);
      } else {
        f[(p + 1) & 3] = fma(-m01.x, bj, f[(p + 1) & 3]);
        f[(p + 2) & 3] = fma(-m01.y, bj, f[(p + 2) & 3]);
        f[(p + 3) & 3] = fma(-m2, bj, f[(p + 3) & 3]);
      }
      const double* bp = base + s * (STRIDE - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool edge = (r == 0) || (r >= R - 2);
        if (!edge || ((mask[r] >> s) & 1u)) v[r] = fma(-bp[32 * r], bj, v[r]);
      }
      f[p] = __shfl_sync(FULL, v[(s + 4) >> 5], (s + 4) & 31);
      if (DEFER) c[p] = 0.0;
    }
    double t = v[0];
    for (int r = 0; r + 1 < R; ++r) v[r] = v[r + 1];
    v[R - 1] = t * 0.5;
  }
  long long t1 = clock64();
  double sacc = f[0] + f[1] + f[2] + f[3] + c[0] + c[1] + c[2] + c[3];
  for (int r = 0; r < R; ++r) sacc += v[r];
  out[lane] = sacc;
  if (lane == 0) cyc[0] = t1 - t0;
}

template <int R, int KW, int STRIDE, bool BWD, bool DEFER>
void run(const char* name, double* o, long long* c) {
  int rounds = 200;
  size_t sm = 32 * STRIDE * sizeof(double);
  auto kk = k<R, KW, STRIDE, BWD, DEFER>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  kk<<<1, 32, sm>>>(o, c, rounds);
  kk<<<1, 32, sm>>>(o, c, rounds);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7.1f cycles/step\n", name, h / (32.0 * rounds));
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 4096); cudaMalloc(&c, 64); cudaMemset(o, 0, 4096);
  run<4, 72, 74, false, false>("fwd R=4 masks", o, c);
  run<4, 72, 74, false, true>("fwd R=4 masks + deferred front", o, c);
  run<6, 144, 146, true, false>("bwd R=6 masks", o, c);
  run<6, 144, 146, true, true>("bwd R=6 masks + deferred front", o, c);
  run<10, 272, 274, true, false>("bwd R=10 masks", o, c);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
