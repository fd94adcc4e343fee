// K3: coarse solve y = B0^{-1} c with the getrf factors of B0
// (schwarz.py:56: scipy.linalg.lu_solve(self.b0_piv, Z^T r)).
//
// Layout (factor.pack_b0_tiles): the triangular solves L x = P c and
// U y = x (the latter in reversed coordinates, where it is lower
// triangular) are cut into panels of P rows.  Per panel t: the explicit
// inverse of its P x P diagonal block and the nonzero P x P tiles T[t, j],
// j < t.  The dense getrf factors of the block-sparse B0 are mostly zero
// outside a skyline, so only ~17% of the dense factor bytes are stored.
//
// Execution: one persistent launch of G CTAs.  Panel g (0..2K-1; L panels
// then U panels) belongs to CTA g % G.  A CTA pulls, in ascending j, each
// tile's contribution acc_t -= T[t, j] x_j as soon as panel j of the same
// phase is published, then x_t = D_t^{-1} acc_t, stores it and publishes
// panel g by advancing a monotone global counter (release / acquire).  The
// result is deterministic: every panel is summed in the same order.  The
// critical path per panel is one P x P tile GEMV + one P x P inverse GEMV +
// a flag round trip through L2; the tile stream of later panels overlaps.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hg_internal.cuh"

namespace hg {

// Timing experiments only (HG_B0_STAMPS=1): per-panel %globaltimer stamps
// {start, tiles done, published}.
constexpr int B0_MAX_STAMPED = 8192;
__device__ int g_b0_stamp_on = 0;
__device__ unsigned long long g_b0_stamps[B0_MAX_STAMPED * 3];

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int P, int THREADS>
__global__ void __launch_bounds__(THREADS) k_b0_tiles(int m, int K, const int* __restrict__ perm,
                                                      const int* __restrict__ col_blk,
                                                      const CblkDesc* __restrict__ descs,
                                                      const double* __restrict__ cpart,
                                                      const double* __restrict__ dinv,
                                                      const long long* __restrict__ tile_ptr,
                                                      const int* __restrict__ tile_col,
                                                      const double* __restrict__ tiles, double* xbuf,
                                                      unsigned long long* done, unsigned long long* ticket,
                                                      double* __restrict__ y,
                                                      const unsigned long long* zt_done,
                                                      unsigned long long n_zt_items, SpinCfg spin) {
  constexpr int TPR = THREADS / P;  // threads per row
  constexpr int CPT = P / TPR;      // columns per thread
  static_assert(TPR >= 1 && TPR <= 32 && (32 % TPR) == 0 && CPT % 2 == 0, "tile mapping");
  __shared__ __align__(16) double accs[P];
  __shared__ unsigned long long s_seen, s_launch;
  const int tid = threadIdx.x, row = tid / TPR, q = tid % TPR, lane = tid & 31;
  const int src = lane - q;  // first lane of this row's group
  bool dead = false;         // thread 0 only: a bounded wait gave up (the host sees the fault word)
  // s_seen: the counter value this CTA has observed (acquire by thread 0,
  // then a barrier so every thread may read the panels it covers).
  auto observe = [&](unsigned long long need) -> unsigned long long {
    if (tid == 0) {
      unsigned long long v = ld_acquire_u64(done);
      SpinGuard sg;
      while (v < need && !dead) {
        if (spin_abort(sg, spin)) dead = true;
        v = ld_acquire_u64(done);
      }
      s_seen = dead ? ~0ull : v;
    }
    __syncthreads();
    return s_seen;
  };
  if (tid == 0) {  // c = Z^T r of this apply complete (the solve may be launched before it)
    s_launch = take_launch_index(ticket, gridDim.x);
    const unsigned long long zt_target = (s_launch + 1) * n_zt_items;
    SpinGuard sg;
    while (ld_acquire_u64(zt_done) < zt_target && !dead)
      if (spin_abort(sg, spin)) dead = true;
  }
  __syncthreads();
  const unsigned long long base = s_launch * 2ull * (unsigned long long)K;  // done counter at this launch's start
  for (int g = blockIdx.x; g < 2 * K; g += gridDim.x) {
    const int ph = g / K, t = g % K;
    const bool stamp = g_b0_stamp_on && tid == 0 && g < B0_MAX_STAMPED;
    if (stamp) g_b0_stamps[3 * g] = gtimer();
    const double* xph = xbuf + (size_t)ph * K * P;
    const unsigned long long pbase = base + (unsigned long long)ph * K;  // counter value of "panel 0 of ph"
    double acc = 0.0;
    unsigned long long seen;
    if (ph == 0) {
      const int i = t * P + row;
      if (q == 0 && i < m) {
        const int col = perm[i];
        const CblkDesc d = descs[col_blk[col]];
        const int l = col - d.col0;
        double c = 0.0;
        for (int ch = 0; ch < d.nchunk; ++ch) c += cpart[d.part_off + (long long)ch * d.m + l];
        acc = c;
      }
      seen = observe(0);
    } else {
      seen = observe(base + K);  // the whole L solve
      if (q == 0) acc = xbuf[(size_t)K * P - 1 - (t * P + row)];
    }
    acc = __shfl_sync(FULL, acc, src);
    const long long e0 = tile_ptr[g], e1 = tile_ptr[g + 1];
    // this panel's inverse diagonal block slice, fetched off the critical path
    double2 dv[CPT / 2];
    {
      const double2* dp = reinterpret_cast<const double2*>(dinv + ((size_t)g * P + row) * P + q * CPT);
#pragma unroll
      for (int c = 0; c < CPT / 2; ++c) dv[c] = __ldg(dp + c);
    }
    // tiles in ascending column panel; contributions subtracted one tile at a
    // time (fixed order, independent of when panels became visible)
    double2 nv[CPT / 2];
    if (e0 < e1) {
      const double2* tp = reinterpret_cast<const double2*>(tiles + ((size_t)e0 * P + row) * P + q * CPT);
#pragma unroll
      for (int c = 0; c < CPT / 2; ++c) nv[c] = __ldg(tp + c);
    }
    for (long long e = e0; e < e1; ++e) {
      const int j = tile_col[e];
      double2 tv[CPT / 2];
#pragma unroll
      for (int c = 0; c < CPT / 2; ++c) tv[c] = nv[c];
      if (e + 1 < e1) {  // prefetch the next tile slice
        const double2* tp = reinterpret_cast<const double2*>(tiles + ((size_t)(e + 1) * P + row) * P + q * CPT);
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) nv[c] = __ldg(tp + c);
      }
      if (seen < pbase + j + 1) seen = observe(pbase + j + 1);  // uniform branch
      const double2* xp = reinterpret_cast<const double2*>(xph + (size_t)j * P + q * CPT);
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < CPT / 2; ++c) {
        const double2 xv = xp[c];
        s = fma(tv[c].x, xv.x, s);
        s = fma(tv[c].y, xv.y, s);
      }
#pragma unroll
      for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
      acc -= s;
    }
    if (stamp) g_b0_stamps[3 * g + 1] = gtimer();
    if (q == 0) accs[row] = acc;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CPT / 2; ++c) {
      s = fma(dv[c].x, accs[q * CPT + 2 * c], s);
      s = fma(dv[c].y, accs[q * CPT + 2 * c + 1], s);
    }
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (q == 0) {
      xbuf[(size_t)ph * K * P + t * P + row] = s;
      if (ph == 1) {
        const int i = K * P - 1 - (t * P + row);
        if (i < m) y[i] = s;
      }
    }
    __syncthreads();
    if (tid == 0) {
      // the release store is cumulative over the CTA's x stores ordered before
      // it by the barrier; publish in panel order (a panel may finish first)
      SpinGuard sg;
      while (ld_acquire_u64(done) < base + g && !dead)
        if (spin_abort(sg, spin)) dead = true;
      st_release_u64(done, base + g + 1);
      if (stamp) g_b0_stamps[3 * g + 2] = gtimer();
    }
  }
}

int preload_b0() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_tiles<64, 256>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_tiles<128, 512>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_tiles<32, 128>));
  return preload_b0_cluster();
}

int launch_coarse_solve(HgPrecond* P, cudaStream_t st) {
  if (P->m == 0) return HG_OK;
  if (P->b0_mode == 1) return launch_coarse_solve_cluster(P, st);
  const int K = P->b0_K;
  const int G = K < P->b0_ctas ? K : P->b0_ctas;
  const unsigned long long nzt = (unsigned long long)P->n_zt_items;
  const SpinCfg spin = spin_cfg(P);
  switch (P->b0_P) {
    case 64:
      k_b0_tiles<64, 256><<<G, 256, 0, st>>>(P->m, K, P->d_b0_perm, P->d_col_blk, P->d_cblk, P->d_cpart,
                                              P->d_b0_dinv, P->d_b0_tile_ptr, P->d_b0_tile_col, P->d_b0_tiles,
                                              P->d_b0_x, P->d_b0_done, P->d_ticket, P->d_y, P->d_zt_done, nzt, spin);
      break;
    case 128:
      k_b0_tiles<128, 512><<<G, 512, 0, st>>>(P->m, K, P->d_b0_perm, P->d_col_blk, P->d_cblk, P->d_cpart,
                                               P->d_b0_dinv, P->d_b0_tile_ptr, P->d_b0_tile_col, P->d_b0_tiles,
                                               P->d_b0_x, P->d_b0_done, P->d_ticket, P->d_y, P->d_zt_done, nzt, spin);
      break;
    case 32:
      k_b0_tiles<32, 128><<<G, 128, 0, st>>>(P->m, K, P->d_b0_perm, P->d_col_blk, P->d_cblk, P->d_cpart,
                                              P->d_b0_dinv, P->d_b0_tile_ptr, P->d_b0_tile_col, P->d_b0_tiles,
                                              P->d_b0_x, P->d_b0_done, P->d_ticket, P->d_y, P->d_zt_done, nzt, spin);
      break;
    default:
      set_error("coarse solve: unsupported panel size");
      return HG_ERR_UNSUPPORTED;
  }
  HG_LAUNCH_CHECK();
  static const bool stamps = getenv("HG_B0_STAMPS") != nullptr;
  if (stamps) {  // timing experiment: dump the panel cadence of this launch
    static bool armed = false;
    if (!armed) {
      int one = 1;
      HG_CUDA_TRY(cudaMemcpyToSymbol(g_b0_stamp_on, &one, sizeof(int)));
      armed = true;
      return HG_OK;  // stamps start with the next launch
    }
    HG_CUDA_TRY(cudaStreamSynchronize(st));
    const int n = 2 * K < B0_MAX_STAMPED ? 2 * K : B0_MAX_STAMPED;
    std::vector<unsigned long long> h(3 * (size_t)n);
    HG_CUDA_TRY(cudaMemcpyFromSymbol(h.data(), g_b0_stamps, sizeof(unsigned long long) * h.size()));
    unsigned long long t0 = h[0];
    for (int g = 0; g < n; ++g) t0 = h[3 * g] < t0 ? h[3 * g] : t0;
    double sum_tiles = 0, sum_tail = 0;
    for (int g = 0; g < n; ++g) {
      sum_tiles += (double)(h[3 * g + 1] - h[3 * g]);
      sum_tail += (double)(h[3 * g + 2] - h[3 * g + 1]);
    }
    fprintf(stderr, "[b0 stamps] K=%d G=%d P=%d: total %.1f us, mean tiles %.2f us, mean dinv+publish %.2f us\n", K, G,
            P->b0_P, (h[3 * (n - 1) + 2] - t0) / 1e3, sum_tiles / n / 1e3, sum_tail / n / 1e3);
    for (int g = 0; g < n; g += (n / 12 > 0 ? n / 12 : 1))
      fprintf(stderr, "   panel %4d: start %8.1f tiles_done %8.1f published %8.1f us\n", g, (h[3 * g] - t0) / 1e3,
              (h[3 * g + 1] - t0) / 1e3, (h[3 * g + 2] - t0) / 1e3);
  }
  return HG_OK;
}

}  // namespace hg
