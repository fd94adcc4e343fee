// Microbenchmark of one band-solve sweep step structure (single warp, records
// already in shared memory, no streaming).  Variants isolate the cost of the
// pieces of hg_local.cu's step.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr unsigned FULL = 0xffffffffu;
constexpr int STRIDE = 146;  // bwd record stride of config 5-16 (kv = 144)
constexpr int KW = 144;
constexpr int R = 6;

template <int V>
__global__ void k(double* out, long long* cyc, int rounds, unsigned swapmask, int nsteps) {
  extern __shared__ double rec[];  // 32 records
  const int lane = threadIdx.x;
  for (int i = lane; i < 32 * STRIDE; i += 32) rec[i] = 1e-3 * ((i * 7) % 13) - 6e-3;
  __syncwarp();
  double v[R];
  for (int r = 0; r < R; ++r) v[r] = 1.0 + lane + r;
  double f[4] = {1, 2, 3, 4};
  const int lim = KW - lane;
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      if (V == 6 && s >= nsteps) break;                    // per-step guard
      if ((V == 7 || V == 8) && ((swapmask >> s) & 1u)) {  // never-taken swap branch
        double a = __shfl_sync(FULL, v[0], s);
        v[1] += a;
        f[0] = __shfl_sync(FULL, v[0], s + 1);
      }
      const double* rp = rec + s * STRIDE;
      const int p = s & 3;
      double bj = f[p];
      if (V != 3) bj *= rp[KW];
      if (lane == s) v[0] = bj;
      if (V == 1) {  // front only
        f[(p + 1) & 3] = fma(-rp[0], bj, f[(p + 1) & 3]);
        f[(p + 2) & 3] = fma(-rp[1], bj, f[(p + 2) & 3]);
        f[(p + 3) & 3] = fma(-rp[2], bj, f[(p + 3) & 3]);
        f[p] = __shfl_sync(FULL, v[(s + 4) >> 5], (s + 4) & 31);
        continue;
      }
      f[(p + 1) & 3] = fma(-rp[0], bj, f[(p + 1) & 3]);
      f[(p + 2) & 3] = fma(-rp[1], bj, f[(p + 2) & 3]);
      f[(p + 3) & 3] = fma(-rp[2], bj, f[(p + 3) & 3]);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = 32 * r + lane - s;
        const bool on = (r == 0 ? (lane > s) : true) && (32 * r - s <= lim);
        if (V == 2) {
          v[r] = fma(-(on ? rp[t - 1] : 0.0), bj, v[r]);   // select form
        } else if (V == 4) {
          v[r] = fma(-1e-3, bj, v[r]);                        // no LDS
        } else {
          if (on) v[r] = fma(-rp[t - 1], bj, v[r]);           // predicated form
        }
      }
      if (V == 5) continue;  // no fetch shuffle
      f[p] = __shfl_sync(FULL, v[(s + 4) >> 5], (s + 4) & 31);
    }
    // rotate like the real sweep
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

template <int V>
void run(const char* name, double* o, long long* c) {
  int rounds = 200;
  size_t sm = 32 * STRIDE * sizeof(double);
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<V><<<1, 32, sm>>>(o, c, rounds, 0u, 32);
  k<V><<<1, 32, sm>>>(o, c, rounds, 0u, 32);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7.1f cycles/step\n", name, h / (32.0 * rounds));
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 4096);
  cudaMalloc(&c, 64);
  run<0>("predicated window (current form)", o, c);
  run<2>("select-zero window", o, c);
  run<1>("front only (3 DFMA + shfl)", o, c);
  run<3>("no DMUL", o, c);
  run<4>("window without LDS", o, c);
  run<6>("per-step nsteps guard", o, c);
  run<7>("per-step swap branch (not taken)", o, c);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
