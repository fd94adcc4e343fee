// Dense coarse mode: y = B0^{-1} c with an explicit inverse (setup computes
// it once and checks it against getrs, factorize / schwarz.py:88-99 — same
// operator, different rounding, bar 1e-11).  Replaces the 2K-panel
// triangular chain of hg_b0c.cu on the apply's critical path by an
// HBM-streaming contraction that overlaps the local solves:
//   k_creduce        c[i] = sum_ch Z^T r partials (fixed chunk order)
//   k_b0_pack        setup: row-major B0^{-1} -> packed DMMA-fragment order
//   k_b0_gemv        y = B0^{-1} c, two warps per 8-row tile, B0^{-1} read once
//   k_creduce_multi  C[i][col] likewise for a batch
//   k_b0_gemm_multi  Y = B0^{-1} C (m x m x 16) on DMMA (mma.sync m8n8k4 f64),
//                    split-K in B0_KSPLIT slices, B0^{-1} read once
//   k_ysum_multi     Y = sum of the slices in fixed order (deterministic)
#include "hg_internal.cuh"

namespace hg {

namespace {
constexpr int MRD = HG_MAX_RHS;

__device__ __forceinline__ void dmma_d(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}
}  // namespace

__global__ void k_creduce(int m, const int* __restrict__ col_blk, const CblkDesc* __restrict__ descs,
                          const double* __restrict__ cpart, double* __restrict__ c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const CblkDesc d = descs[col_blk[i]];
  const int l = i - d.col0;
  double v = 0.0;
  for (int ch = 0; ch < d.nchunk; ++ch) v += cpart[d.part_off + (long long)ch * d.m + l];
  c[i] = v;
}

// B0^{-1} is kept PACKED: 8 x 8 blocks, block (mt, kb) at double2 index (mt KB + kb) 32, lane
// (g = lane / 4, q = lane % 4) holding .x = Binv[8 mt + g][8 kb + q], .y = Binv[8 mt + g][8 kb + 4 + q]
// — the DMMA A fragments of two consecutive k-steps in one 16-byte load, so a warp that owns an
// 8-row tile streams ONE contiguous region, 512 bytes per load instruction (zero padded to
// mp = 8 ceil(m / 8) rows and columns).
__global__ void k_b0_pack(int m, int mp, const double* __restrict__ Binv, double2* __restrict__ Bpk) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int KB = mp >> 3;
  if (e >= (long long)KB * KB * 32) return;
  const int lane = (int)(e & 31), g = lane >> 2, q = lane & 3;
  const long long blk = e >> 5;
  const int kb = (int)(blk % KB), mt = (int)(blk / KB);
  const int row = mt * 8 + g, c0 = kb * 8 + q, c1 = c0 + 4;
  double2 v;
  v.x = (row < m && c0 < m) ? Binv[(size_t)row * m + c0] : 0.0;
  v.y = (row < m && c1 < m) ? Binv[(size_t)row * m + c1] : 0.0;
  Bpk[e] = v;
}

int pack_b0_inverse(int m, const double* d_binv, double** d_packed, int* mp_out) {
  const int mp = (m + 7) / 8 * 8;
  *mp_out = mp;
  HG_CUDA_TRY(cudaMalloc(d_packed, sizeof(double) * (size_t)mp * mp));
  const long long ne = (long long)(mp / 8) * (mp / 8) * 32;
  k_b0_pack<<<(unsigned)ceil_div(ne, 256), 256>>>(m, mp, d_binv, reinterpret_cast<double2*>(*d_packed));
  HG_LAUNCH_CHECK();
  HG_CUDA_TRY(cudaDeviceSynchronize());
  return HG_OK;
}

// y = B0^{-1} c: 8 warps per CTA, 4 row tiles per CTA, two warps per tile (k halves, combined in a
// fixed order through shared memory); c (mp doubles, zero padded) comes through L1
__global__ void __launch_bounds__(256) k_b0_gemv(int m, int mp, const double2* __restrict__ Bpk,
                                                 const double* __restrict__ c, double* __restrict__ y) {
  __shared__ double s_hi[4][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  const int KB = mp >> 3;
  const int mt = blockIdx.x * 4 + (warp >> 1), half = warp & 1;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (mt < KB) {
    const int kh = (KB + 1) >> 1;
    const int ka = half * kh, kb = min(KB, ka + kh);
    const double2* ap = Bpk + ((size_t)mt * KB + ka) * 32 + lane;
    const double* cp = c + (size_t)ka * 8 + q;
    int k = ka;
    for (; k + 4 <= kb; k += 4) {
      const double2 a0 = __ldcs(ap), a1 = __ldcs(ap + 32), a2 = __ldcs(ap + 64), a3 = __ldcs(ap + 96);
      s0 = fma(a0.x, __ldg(cp), s0);
      s0 = fma(a0.y, __ldg(cp + 4), s0);
      s1 = fma(a1.x, __ldg(cp + 8), s1);
      s1 = fma(a1.y, __ldg(cp + 12), s1);
      s2 = fma(a2.x, __ldg(cp + 16), s2);
      s2 = fma(a2.y, __ldg(cp + 20), s2);
      s3 = fma(a3.x, __ldg(cp + 24), s3);
      s3 = fma(a3.y, __ldg(cp + 28), s3);
      ap += 128;
      cp += 32;
    }
    for (; k < kb; ++k) {
      const double2 a0 = __ldcs(ap);
      s0 = fma(a0.x, __ldg(cp), s0);
      s0 = fma(a0.y, __ldg(cp + 4), s0);
      ap += 32;
      cp += 8;
    }
  }
  double s = (s0 + s1) + (s2 + s3);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (half == 1 && q == 0) s_hi[warp >> 1][g] = s;
  __syncthreads();
  const int row = mt * 8 + g;
  if (half == 0 && q == 0 && row < m) y[row] = s + s_hi[warp >> 1][g];
}

int launch_b0_dense(HgPrecond* P, cudaStream_t st) {
  const int m = P->m;
  k_creduce<<<ceil_div(m, 256), 256, 0, st>>>(m, P->d_col_blk, P->d_cblk, P->d_cpart, P->d_c);
  HG_LAUNCH_CHECK();
  k_b0_gemv<<<ceil_div(P->b0_mp / 8, 4), 256, 0, st>>>(m, P->b0_mp, reinterpret_cast<const double2*>(P->d_b0_inv), P->d_c,
                                                     P->d_y);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// C in DMMA B-fragment order: k-step (kb, h) = rows 8 kb + 4 h + q of C; lane (g, q) holds
// {C[row][g], C[row][8 + g]} as one double2 at ((2 kb + h) 32 + lane) — one 16-byte load per lane
// per k-step in the GEMM, 512 contiguous bytes per warp
__global__ void k_creduce_multi(int m, int nrhs, const int* __restrict__ col_blk, const CblkDesc* __restrict__ descs,
                                const double* __restrict__ cpartm, double* __restrict__ Cf) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = e / MRD, col = e % MRD;
  if (i >= m) return;
  double v = 0.0;
  if (col < nrhs) {
    const CblkDesc d = descs[col_blk[i]];
    const int l = i - d.col0;
    for (int ch = 0; ch < d.nchunk; ++ch) v += cpartm[(d.part_off + (long long)ch * d.m + l) * MRD + col];
  }
  const int kb = i >> 3, h = (i >> 2) & 1, q = i & 3, g = col & 7, nt = col >> 3;
  Cf[(((size_t)(kb * 2 + h) * 32 + g * 4 + q) << 1) + nt] = v;
}

// Y_slice[s][rows of this warp] = B0^{-1}[rows, k in slice s] C[k in slice s, :]: a warp owns two 8-row
// tiles (4 DMMA accumulators for the 16 columns), streams their packed fragments and takes the B
// fragments of C (fragment order, zero padded; 2 MB, L1 / L2 resident) straight from global memory —
// no shared memory, no barrier.
__global__ void __launch_bounds__(256, 3) k_b0_gemm_multi(int mp, const double2* __restrict__ Bpk,
                                                       const double* __restrict__ C, double* __restrict__ Yp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  const int KB = mp >> 3;
  const int mt0 = (blockIdx.x * 8 + warp) * 2;
  if (mt0 >= KB) return;
  const bool two = mt0 + 1 < KB;
  const int slice = blockIdx.y;
  const int kbl = (KB + B0_KSPLIT - 1) / B0_KSPLIT;
  const int ka = slice * kbl, kb = min(KB, ka + kbl);
  const double2* a0p = Bpk + ((size_t)mt0 * KB + ka) * 32 + lane;
  const double2* a1p = two ? a0p + (size_t)KB * 32 : a0p;
  const double2* cp = reinterpret_cast<const double2*>(C) + (size_t)ka * 64 + lane;
  double acc[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
  // register double buffer: the A fragments of the next GU k-blocks are in flight while the
  // current GU are multiplied (2 GU 512-byte loads per warp ahead of their use)
  constexpr int GU = 4;
  double2 n0[GU], n1[GU];
  const int last = kb - 1 - ka;  // clamp: loads past the slice re-read its last block (never used)
#pragma unroll
  for (int u = 0; u < GU; ++u) {
    const int o = min(u, last) * 32;
    n0[u] = __ldcs(a0p + o);
    n1[u] = __ldcs(a1p + o);
  }
  for (int k = ka; k < kb; k += GU) {
    double2 c0[GU], c1[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      c0[u] = n0[u];
      c1[u] = n1[u];
    }
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      const int o = min(k - ka + GU + u, last) * 32;
      n0[u] = __ldcs(a0p + o);
      n1[u] = __ldcs(a1p + o);
    }
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      if (k + u < kb) {
        const double2* cu = cp + (size_t)(k - ka + u) * 64;
        const double2 b0 = __ldg(cu), b1 = __ldg(cu + 32);
        dmma_d(acc[0][0], c0[u].x, b0.x);
        dmma_d(acc[0][1], c0[u].x, b0.y);
        dmma_d(acc[1][0], c1[u].x, b0.x);
        dmma_d(acc[1][1], c1[u].x, b0.y);
        dmma_d(acc[0][0], c0[u].y, b1.x);
        dmma_d(acc[0][1], c0[u].y, b1.y);
        dmma_d(acc[1][0], c1[u].y, b1.x);
        dmma_d(acc[1][1], c1[u].y, b1.y);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    if (t == 1 && !two) break;
    double* y = Yp + ((size_t)slice * mp + (mt0 + t) * 8 + g) * MRD;
    *reinterpret_cast<double2*>(y + 2 * q) = make_double2(acc[t][0][0], acc[t][0][1]);
    *reinterpret_cast<double2*>(y + 8 + 2 * q) = make_double2(acc[t][1][0], acc[t][1][1]);
  }
}

__global__ void k_ysum_multi(int m, int mp, const double* __restrict__ Yp, double* __restrict__ Y) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * MRD) return;
  double v = 0.0;
#pragma unroll
  for (int s = 0; s < B0_KSPLIT; ++s) v += Yp[(size_t)s * mp * MRD + e];
  Y[e] = v;
}

int launch_b0_dense_multi(HgPrecond* P, int nrhs, cudaStream_t st) {
  const int m = P->m;
  k_creduce_multi<<<ceil_div((long long)m * MRD, 256), 256, 0, st>>>(m, nrhs, P->d_col_blk, P->d_cblk, P->d_cpartm,
                                                                     P->d_cm);
  HG_LAUNCH_CHECK();
  k_b0_gemm_multi<<<dim3(ceil_div(P->b0_mp / 8, 16), B0_KSPLIT), 256, 0, st>>>(
      P->b0_mp, reinterpret_cast<const double2*>(P->d_b0_inv), P->d_cm, P->d_ypart);
  HG_LAUNCH_CHECK();
  k_ysum_multi<<<ceil_div((long long)m * MRD, 256), 256, 0, st>>>(m, P->b0_mp, P->d_ypart, P->d_ym);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

int preload_b0_dense() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_creduce));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_gemv));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_pack));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_creduce_multi));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_gemm_multi));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_ysum_multi));
  return HG_OK;
}

}  // namespace hg
