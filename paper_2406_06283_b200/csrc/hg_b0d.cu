// Dense coarse mode: y = B0^{-1} c with an explicit inverse (setup computes
// it once and checks it against getrs, factorize / schwarz.py:88-99 — same
// operator, different rounding, bar 1e-11).  Replaces the 2K-panel
// triangular chain of hg_b0c.cu on the apply's critical path by an
// HBM-streaming contraction that overlaps the local solves:
//   k_creduce        c[i] = sum_ch Z^T r partials (fixed chunk order)
//   k_b0_gemv        y = B0^{-1} c, one warp per row, B0^{-1} read once
//   k_creduce_multi  C[i][col] likewise for a batch
//   k_b0_gemm_multi  Y = B0^{-1} C (m x m x 16) on DMMA (mma.sync m8n8k4 f64),
//                    split-K in B0_KSPLIT slices, B0^{-1} read once
//   k_ysum_multi     Y = sum of the slices in fixed order (deterministic)
#include "hg_internal.cuh"

namespace hg {

namespace {
constexpr int MRD = HG_MAX_RHS;
constexpr int SRD = 20;     // smem row stride of 16-column tiles (conflict-free B fragments)
constexpr int KCH = 256;    // k rows of C staged per chunk

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

// one warp per row; 4 independent partial sums in flight per lane
__global__ void __launch_bounds__(256) k_b0_gemv(int m, const double* __restrict__ Binv, const double* __restrict__ c,
                                                 double* __restrict__ y) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const double* a = Binv + (size_t)row * m;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = lane;
  for (; k + 96 < m; k += 128) {
    s0 = fma(__ldg(a + k), __ldg(c + k), s0);
    s1 = fma(__ldg(a + k + 32), __ldg(c + k + 32), s1);
    s2 = fma(__ldg(a + k + 64), __ldg(c + k + 64), s2);
    s3 = fma(__ldg(a + k + 96), __ldg(c + k + 96), s3);
  }
  for (; k < m; k += 32) s0 = fma(__ldg(a + k), __ldg(c + k), s0);
  const double s = warp_sum((s0 + s1) + (s2 + s3));
  if (lane == 0) y[row] = s;
}

int launch_b0_dense(HgPrecond* P, cudaStream_t st) {
  const int m = P->m;
  k_creduce<<<ceil_div(m, 256), 256, 0, st>>>(m, P->d_col_blk, P->d_cblk, P->d_cpart, P->d_c);
  HG_LAUNCH_CHECK();
  k_b0_gemv<<<ceil_div(m, 8), 256, 0, st>>>(m, P->d_b0_inv, P->d_c, P->d_y);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void k_creduce_multi(int m, int nrhs, const int* __restrict__ col_blk, const CblkDesc* __restrict__ descs,
                                const double* __restrict__ cpartm, double* __restrict__ C) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = e / MRD, col = e % MRD;
  if (i >= m) return;
  double v = 0.0;
  if (col < nrhs) {
    const CblkDesc d = descs[col_blk[i]];
    const int l = i - d.col0;
    for (int ch = 0; ch < d.nchunk; ++ch) v += cpartm[(d.part_off + (long long)ch * d.m + l) * MRD + col];
  }
  C[e] = v;
}

// Y_slice[s] (64-row panel of this CTA) = B0^{-1}[rows, k in slice s] * C[k in slice s, :]
// 8 warps x 8 rows, 2 DMMA accumulators (16 columns) per warp.
__global__ void __launch_bounds__(256) k_b0_gemm_multi(int m, const double* __restrict__ Binv,
                                                       const double* __restrict__ C, double* __restrict__ Yp) {
  __shared__ __align__(16) double s_c[KCH * SRD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  const int r0 = blockIdx.x * 64 + warp * 8;
  const int slice = blockIdx.y;
  const int klen = (m + B0_KSPLIT - 1) / B0_KSPLIT;
  const int ka = slice * klen, kb = min(m, ka + klen);
  const int row = r0 + g;
  const double* arow = Binv + (size_t)min(row, m - 1) * m;
  double acc0[2] = {0.0, 0.0}, acc1[2] = {0.0, 0.0};
  for (int kc = ka; kc < kb; kc += KCH) {
    const int kn = min(KCH, kb - kc);
    __syncthreads();
    for (int e = threadIdx.x; e < KCH * MRD; e += 256) {
      const int k = e / MRD, col = e % MRD;
      s_c[k * SRD + col] = k < kn ? C[(size_t)(kc + k) * MRD + col] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int ks = 0; ks < KCH; ks += 4) {
      const int k = ks + q;
      const double a = (row < m && k < kn) ? __ldg(arow + kc + k) : 0.0;
      dmma_d(acc0, a, s_c[k * SRD + g]);
      dmma_d(acc1, a, s_c[k * SRD + 8 + g]);
    }
  }
  if (row < m) {
    double* y = Yp + ((size_t)slice * m + row) * MRD;
    *reinterpret_cast<double2*>(y + 2 * q) = make_double2(acc0[0], acc0[1]);
    *reinterpret_cast<double2*>(y + 8 + 2 * q) = make_double2(acc1[0], acc1[1]);
  }
}

__global__ void k_ysum_multi(int m, const double* __restrict__ Yp, double* __restrict__ Y) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * MRD) return;
  double v = 0.0;
#pragma unroll
  for (int s = 0; s < B0_KSPLIT; ++s) v += Yp[(size_t)s * m * MRD + e];
  Y[e] = v;
}

int launch_b0_dense_multi(HgPrecond* P, int nrhs, cudaStream_t st) {
  const int m = P->m;
  k_creduce_multi<<<ceil_div((long long)m * MRD, 256), 256, 0, st>>>(m, nrhs, P->d_col_blk, P->d_cblk, P->d_cpartm,
                                                                     P->d_cm);
  HG_LAUNCH_CHECK();
  k_b0_gemm_multi<<<dim3(ceil_div(m, 64), B0_KSPLIT), 256, 0, st>>>(m, P->d_b0_inv, P->d_cm, P->d_ypart);
  HG_LAUNCH_CHECK();
  k_ysum_multi<<<ceil_div((long long)m * MRD, 256), 256, 0, st>>>(m, P->d_ypart, P->d_ym);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

int preload_b0_dense() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_creduce));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_gemv));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_creduce_multi));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_gemm_multi));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_ysum_multi));
  return HG_OK;
}

}  // namespace hg
