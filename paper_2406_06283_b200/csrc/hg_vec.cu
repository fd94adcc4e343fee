// FP64 CSR SpMV and the Arnoldi vector kernels (block dots, multi-axpy,
// normalise), all HBM-bound streaming kernels.
//
// SpMV row sums are accumulated in index order with separate multiply and
// add (no FMA contraction), which is exactly what scipy's csr_matvec does
// (sparsetools csr.h), so y = B x / D_k x match the reference bitwise.
// Partial dot products are reduced per CTA in a fixed tree order and then
// across CTAs in a fixed order: results are deterministic run to run.
#include "hg_internal.cuh"

namespace hg {


__global__ void __launch_bounds__(VEC_THREADS) k_spmv(int n, const int* __restrict__ ip,
                                                      const int* __restrict__ ix,
                                                      const double* __restrict__ a,
                                                      const double* __restrict__ x,
                                                      double* __restrict__ y) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  int e1 = ip[i + 1];
  for (int e = ip[i]; e < e1; ++e) s = __dadd_rn(s, __dmul_rn(a[e], __ldg(x + ix[e])));
  y[i] = s;
}

int launch_spmv(const DevCsr& A, const double* vals, const double* x, double* y, cudaStream_t st) {
  if (A.n == 0) return HG_OK;
  k_spmv<<<ceil_div(A.n, VEC_THREADS), VEC_THREADS, 0, st>>>(A.n, A.indptr, A.indices, vals, x, y);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void __launch_bounds__(VEC_THREADS) k_spmv_dots(int n, const int* __restrict__ ip,
                                                           const int* __restrict__ ix,
                                                           const double* __restrict__ a,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ y,
                                                           const double* __restrict__ W, long long ldw,
                                                           int nv, int dot_with_y,
                                                           double* __restrict__ partials) {
  const int width = nv + 1;
  double xv[VEC_ROWS], yv[VEC_ROWS];
  int rows[VEC_ROWS];
  double self = 0.0;
#pragma unroll
  for (int k = 0; k < VEC_ROWS; ++k) {
    int i = blockIdx.x * VEC_TILE + k * VEC_THREADS + threadIdx.x;
    rows[k] = i;
    xv[k] = 0.0;
    yv[k] = 0.0;
    if (i < n) {
      double s = 0.0;
      int e1 = ip[i + 1];
      for (int e = ip[i]; e < e1; ++e) s = __dadd_rn(s, __dmul_rn(a[e], __ldg(x + ix[e])));
      y[i] = s;
      yv[k] = s;
      xv[k] = x[i];
      self = fma(xv[k], s, self);
    }
  }
  // self dot x.y into slot 0
  __shared__ double s_self[VEC_THREADS / 32];
  self = warp_sum(self);
  if ((threadIdx.x & 31) == 0) s_self[threadIdx.x >> 5] = self;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < VEC_THREADS / 32; ++w) t += s_self[w];
    partials[(long long)blockIdx.x * width] = t;
  }
  if (dot_with_y)
    block_dots<VEC_ROWS>(yv, rows, n, W, ldw, nv, partials, width, 1, nullptr);
  else
    block_dots<VEC_ROWS>(xv, rows, n, W, ldw, nv, partials, width, 1, nullptr);
}

int spmv_dots_nblocks(int n) { return ceil_div(n, VEC_TILE); }

int launch_spmv_dots(const DevCsr& A, const double* vals, const double* x, double* y, const double* W,
                     long long ldw, int nv, bool dot_with_y, double* partials, int* nblocks_out,
                     cudaStream_t st) {
  int nb = spmv_dots_nblocks(A.n);
  if (nblocks_out) *nblocks_out = nb;
  if (A.n == 0) return HG_OK;
  k_spmv_dots<<<nb, VEC_THREADS, 0, st>>>(A.n, A.indptr, A.indices, vals, x, y, W, ldw, nv,
                                          dot_with_y ? 1 : 0, partials);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void __launch_bounds__(VEC_THREADS) k_dots(int n, const double* __restrict__ z,
                                                      const double* __restrict__ W, long long ldw,
                                                      int nv, double* __restrict__ partials) {
  const int width = nv + 1;
  double zv[VEC_ROWS];
  int rows[VEC_ROWS];
  double self = 0.0;
#pragma unroll
  for (int k = 0; k < VEC_ROWS; ++k) {
    int i = blockIdx.x * VEC_TILE + k * VEC_THREADS + threadIdx.x;
    rows[k] = i;
    zv[k] = i < n ? z[i] : 0.0;
    self = fma(zv[k], zv[k], self);
  }
  __shared__ double s_self[VEC_THREADS / 32];
  self = warp_sum(self);
  if ((threadIdx.x & 31) == 0) s_self[threadIdx.x >> 5] = self;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < VEC_THREADS / 32; ++w) t += s_self[w];
    partials[(long long)blockIdx.x * width] = t;
  }
  block_dots<VEC_ROWS>(zv, rows, n, W, ldw, nv, partials, width, 1, nullptr);
}

int launch_dots(int n, const double* z, const double* W, long long ldw, int nv, double* partials,
                int* nblocks_out, cudaStream_t st) {
  int nb = ceil_div(n, VEC_TILE);
  if (nblocks_out) *nblocks_out = nb;
  if (n == 0) return HG_OK;
  k_dots<<<nb, VEC_THREADS, 0, st>>>(n, z, W, ldw, nv, partials);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// out[c] = sum_b partials[b*width + c], one CTA per column, fixed tree order.
__global__ void __launch_bounds__(256) k_reduce_cols(const double* __restrict__ partials, int nblocks,
                                                     int width, double* __restrict__ out) {
  __shared__ double s[256];
  int c = blockIdx.x;
  double t = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 256) t += partials[(long long)b * width + c];
  s[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = s[0];
}

int launch_reduce(const double* partials, int nblocks, int width, double* out, cudaStream_t st) {
  if (width == 0) return HG_OK;
  k_reduce_cols<<<width, 256, 0, st>>>(partials, nblocks, width, out);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// mode 1: w -= sum_i coef[i] V[i];  mode 0: w = sum_i coef[i] V[i];
// mode 2: w += sum_i coef[i] V[i]
// The sum over i is sequential, like the reference's one-vector-at-a-time
// update (wgmres.py:135-146).
__global__ void __launch_bounds__(VEC_THREADS) k_axpy_multi(int n, double* __restrict__ w,
                                                            const double* __restrict__ V, long long ldv,
                                                            int nv, const double* __restrict__ coef,
                                                            int mode) {
  __shared__ double s_coef[MAX_NV];
  for (int i = threadIdx.x; i < nv; i += VEC_THREADS) s_coef[i] = coef[i];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < VEC_ROWS; ++k) {
    int d = blockIdx.x * VEC_TILE + k * VEC_THREADS + threadIdx.x;
    if (d >= n) continue;
    double acc = mode ? w[d] : 0.0;
    if (mode == 1) {
      for (int i = 0; i < nv; ++i) acc = fma(-s_coef[i], __ldg(V + (long long)i * ldv + d), acc);
    } else {
      for (int i = 0; i < nv; ++i) acc = fma(s_coef[i], __ldg(V + (long long)i * ldv + d), acc);
    }
    w[d] = acc;
  }
}

int launch_axpy_multi(int n, double* w, const double* V, long long ldv, int nv, const double* coef,
                      int mode, cudaStream_t st) {
  if (n == 0) return HG_OK;
  if (nv > MAX_NV) {
    set_error("axpy_multi: more than 1024 basis vectors");
    return HG_ERR_UNSUPPORTED;
  }
  k_axpy_multi<<<ceil_div(n, VEC_TILE), VEC_THREADS, 0, st>>>(n, w, V, ldv, nv, coef, mode);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void k_scale2(int n, const double* __restrict__ w, const double* __restrict__ ww, double h,
                         double* __restrict__ v_out, double* __restrict__ wv_out) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  v_out[d] = w[d] / h;
  if (wv_out) wv_out[d] = ww[d] / h;
}

int launch_scale2(int n, const double* w, const double* ww, const double* hnorm_host, double* v_out,
                  double* wv_out, cudaStream_t st) {
  if (n == 0) return HG_OK;
  k_scale2<<<ceil_div(n, 256), 256, 0, st>>>(n, w, ww, *hnorm_host, v_out, wv_out);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void k_copy(int n, const double* __restrict__ x, double* __restrict__ y) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) y[d] = x[d];
}

int launch_copy(int n, const double* x, double* y, cudaStream_t st) {
  if (n == 0) return HG_OK;
  k_copy<<<ceil_div(n, 256), 256, 0, st>>>(n, x, y);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void k_sub(int n, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ out) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) out[d] = a[d] - b[d];
}

int launch_sub(int n, const double* a, const double* b, double* out, cudaStream_t st) {
  if (n == 0) return HG_OK;
  k_sub<<<ceil_div(n, 256), 256, 0, st>>>(n, a, b, out);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void k_fill(long long n, double* __restrict__ y, double v) {
  long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) y[d] = v;
}

int preload_vec() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_spmv));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_spmv_dots));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_dots));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_reduce_cols));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_axpy_multi));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_scale2));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_copy));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_sub));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_fill));
  return HG_OK;
}

int launch_fill(long long n, double* y, double val, cudaStream_t st) {
  if (n == 0) return HG_OK;
  k_fill<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, y, val);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

}  // namespace hg
