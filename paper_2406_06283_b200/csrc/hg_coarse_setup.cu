// Coarse operator on the device: B0 = Z^T B Z, its
// symmetrisation, its LU with partial pivoting, and the rank certificate's
// power iterations — the host build_coarse_space / factorize steps
// eigencoarse.py:286-287 (B0 = Z^T (B Z), 0.5 (B0 + B0^T)) and schwarz.py:90
// (lu_factor(B0), LAPACK getrf semantics), restated for one B200.
//
//   k_scatter_zcols   X[c] = E_b Z_b[:, c0 + c]          (16 columns of block b)
//   (k_spmm)          Y = B X                             (hg_multi.cu)
//   k_zty             B0[col0_a + l, col0_b + c0 + c] = Z_a^T Y[c] on idof_a,
//                     for every block a interacting with b (one CTA per a)
//   k_symmetrise      B0 = 0.5 (B0 + B0^T)
//   getrf:            per column j of a 64-column panel: k_lu_pivot (first
//                     index of max |a_ij|, i >= j), k_lu_swap (whole rows, as
//                     getrf's dlaswp), k_lu_panel (multipliers by the
//                     reciprocal pivot, rank-1 update inside the panel); then
//                     k_lu_trsm (U12 = L11^{-1} A12) and k_lu_gemm
//                     (A22 -= L21 U12, FP64 tensor cores, 64 x 64 tiles)
//   certificate:      k_gemv (B0 x) and k_lu_solve_block (blocked triangular
//                     solves with the LU) for the power / inverse iterations
//                     of coarse._sym_extreme_certificate
#include <algorithm>
#include <cmath>
#include <vector>

#include "hg_internal.cuh"

namespace hg {

namespace {
constexpr int CS_NB = 64;   // LU panel width / GEMM tile
constexpr int GSR = 68;     // smem row stride of a 64-wide tile (conflict-free fragments)

__device__ __forceinline__ void dmma_c(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}
}  // namespace

struct CsBlock {  // one coarse block: n interior dofs, m columns from col0
  int n, m, col0, pad;
  long long idx_off, z_off;
};

__global__ void k_scatter_zcols(const CsBlock* __restrict__ blk, int b, int c0, int nc, const int* __restrict__ idx,
                                const double* __restrict__ Z, double* __restrict__ X, long long n) {
  const CsBlock d = blk[b];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.n * nc) return;
  const int k = e / nc, c = e % nc;
  X[(long long)c * n + idx[d.idx_off + k]] = Z[d.z_off + (long long)k * d.m + c0 + c];
}

__global__ void k_clear_zcols(const CsBlock* __restrict__ blk, int b, int nc, const int* __restrict__ idx,
                              double* __restrict__ X, long long n) {
  const CsBlock d = blk[b];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.n * nc) return;
  X[(long long)(e % nc) * n + idx[d.idx_off + e / nc]] = 0.0;
}

constexpr int ZTY_ROWS = 64;   // rows of Z_a per partial-sum CTA
constexpr int ZTY_MAXM = 64;   // coarse columns per block supported by the staged tile

// partial (l, c) = sum_{k in chunk} Z_a[k, l] Y[c][idof_a[k]] for interacting block
// a = nbr[blockIdx.y], rows chunk blockIdx.x; tiles staged in shared memory
__global__ void __launch_bounds__(256) k_zty_part(const CsBlock* __restrict__ blk, const int* __restrict__ nbr,
                                                  const int* __restrict__ idx, const double* __restrict__ Z,
                                                  const double* __restrict__ Y, long long n, int nc,
                                                  double* __restrict__ part, int nchunk_max) {
  __shared__ double sz[ZTY_ROWS][ZTY_MAXM + 1];
  __shared__ double sy[ZTY_ROWS][HG_MAX_RHS + 1];
  const CsBlock d = blk[nbr[blockIdx.y]];
  const int k0 = blockIdx.x * ZTY_ROWS;
  double* out = part + ((long long)blockIdx.y * nchunk_max + blockIdx.x) * (ZTY_MAXM * HG_MAX_RHS);
  if (k0 >= d.n) {
    for (int o = threadIdx.x; o < d.m * nc; o += blockDim.x) out[o] = 0.0;
    return;
  }
  const int rows = min(ZTY_ROWS, d.n - k0);
  for (int e = threadIdx.x; e < rows * d.m; e += blockDim.x) sz[e / d.m][e % d.m] = Z[d.z_off + (long long)(k0 + e / d.m) * d.m + e % d.m];
  for (int e = threadIdx.x; e < rows * nc; e += blockDim.x) {
    const int k = e / nc, c = e % nc;
    sy[k][c] = Y[(long long)c * n + idx[d.idx_off + k0 + k]];
  }
  __syncthreads();
  for (int o = threadIdx.x; o < d.m * nc; o += blockDim.x) {
    const int l = o / nc, c = o % nc;
    double s = 0.0;
    for (int k = 0; k < rows; ++k) s = fma(sz[k][l], sy[k][c], s);
    out[o] = s;
  }
}

// B0[col0_a + l, colb + c] = sum of the chunk partials in chunk order (deterministic)
__global__ void k_zty_reduce(const CsBlock* __restrict__ blk, const int* __restrict__ nbr, int nc, int colb,
                             const double* __restrict__ part, int nchunk_max, double* __restrict__ B0, int m) {
  const CsBlock d = blk[nbr[blockIdx.x]];
  const int nch = (d.n + ZTY_ROWS - 1) / ZTY_ROWS;
  for (int o = threadIdx.x; o < d.m * nc; o += blockDim.x) {
    double s = 0.0;
    for (int ch = 0; ch < nch; ++ch) s += part[((long long)blockIdx.x * nchunk_max + ch) * (ZTY_MAXM * HG_MAX_RHS) + o];
    B0[(long long)(d.col0 + o / nc) * m + colb + o % nc] = s;
  }
}

__global__ void k_symmetrise(double* __restrict__ A, int m) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long i = e / m, j = e % m;
  if (i >= m || j <= i) return;
  const double a = A[i * m + j], b = A[j * m + i];
  const double s = 0.5 * (a + b);  // numpy: 0.5 * (B0 + B0.T)
  A[i * m + j] = s;
  A[j * m + i] = s;
}

// ------------------------------------------------------------------ getrf
__global__ void __launch_bounds__(1024) k_lu_pivot(const double* __restrict__ A, int m, int j, int* __restrict__ piv,
                                                   int* __restrict__ info) {
  __shared__ double sv[32];
  __shared__ int si[32];
  double best = -1.0;
  int bi = j;
  for (int i = j + threadIdx.x; i < m; i += blockDim.x) {
    const double v = fabs(A[(long long)i * m + j]);
    if (v > best) {  // ascending i per thread: first max kept
      best = v;
      bi = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(FULL, best, o);
    const int oi = __shfl_xor_sync(FULL, bi, o);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? sv[lane] : -1.0;
    bi = lane < nw ? si[lane] : m;
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(FULL, best, o);
      const int oi = __shfl_xor_sync(FULL, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) {
      piv[j] = bi;
      if (A[(long long)bi * m + j] == 0.0 && *info == 0) *info = j + 1;
    }
  }
}

__global__ void k_lu_swap(double* __restrict__ A, int m, int j, const int* __restrict__ piv) {
  const int p = piv[j];
  if (p == j) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m; c += gridDim.x * blockDim.x) {
    const double t = A[(long long)j * m + c];
    A[(long long)j * m + c] = A[(long long)p * m + c];
    A[(long long)p * m + c] = t;
  }
}

// rows i > j: l = a_ij / a_jj (by the reciprocal, as dgetf2), a_ic -= l a_jc for c in (j, jend)
__global__ void k_lu_panel(double* __restrict__ A, int m, int j, int jend) {
  const int i = j + 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double piv = A[(long long)j * m + j];
  if (piv == 0.0) return;
  const double l = A[(long long)i * m + j] * (1.0 / piv);
  A[(long long)i * m + j] = l;
  for (int c = j + 1; c < jend; ++c) A[(long long)i * m + c] = fma(-l, A[(long long)j * m + c], A[(long long)i * m + c]);
}

// U12 = L11^{-1} A12 for the panel rows k0..k0+kb-1, columns >= k0+kb (unit lower L11)
__global__ void k_lu_trsm(double* __restrict__ A, int m, int k0, int kb) {
  __shared__ double L[CS_NB][CS_NB + 1];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) L[e / kb][e % kb] = A[(long long)(k0 + e / kb) * m + k0 + e % kb];
  __syncthreads();
  const int c = k0 + kb + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  double x[CS_NB];
  for (int r = 0; r < kb; ++r) {
    double s = A[(long long)(k0 + r) * m + c];
    for (int t = 0; t < r; ++t) s = fma(-L[r][t], x[t], s);
    x[r] = s;
    A[(long long)(k0 + r) * m + c] = s;
  }
}

// A22 -= L21 U12: 64 x 64 output tile per CTA, K = kb (<= 64) in two halves, DMMA
__global__ void __launch_bounds__(256) k_lu_gemm(double* __restrict__ A, int m, int k0, int kb) {
  constexpr int KH = CS_NB / 2;
  __shared__ __align__(16) double sa[CS_NB * (KH + 4)];  // L21 tile [row][k]
  __shared__ __align__(16) double sb[KH * GSR];          // U12 tile [k][col]
  const int s0 = k0 + kb;
  const int i0 = s0 + blockIdx.y * CS_NB, c0 = s0 + blockIdx.x * CS_NB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  double acc[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int r = warp * 8 + g;
  for (int h = 0; h < kb; h += KH) {
    __syncthreads();
    for (int e = threadIdx.x; e < CS_NB * KH; e += 256) {
      const int rr = e / KH, k = e % KH;
      sa[rr * (KH + 4) + k] = (i0 + rr < m && h + k < kb) ? A[(long long)(i0 + rr) * m + k0 + h + k] : 0.0;
      const int kk = e / CS_NB, c = e % CS_NB;
      sb[kk * GSR + c] = (h + kk < kb && c0 + c < m) ? A[(long long)(k0 + h + kk) * m + c0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 2
    for (int ks = 0; ks < KH; ks += 4) {
      const double a = sa[r * (KH + 4) + ks + q];
#pragma unroll
      for (int t = 0; t < 8; ++t) dmma_c(acc[t], a, sb[(ks + q) * GSR + t * 8 + g]);
    }
  }
  const int row = i0 + r;
  if (row < m) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int c = c0 + t * 8 + 2 * q;
      if (c < m) A[(long long)row * m + c] -= acc[t][0];
      if (c + 1 < m) A[(long long)row * m + c + 1] -= acc[t][1];
    }
  }
}

// ------------------------------------------------------------------ certificate kernels
__global__ void __launch_bounds__(256) k_gemv(const double* __restrict__ A, int m, const double* __restrict__ x,
                                              double* __restrict__ y) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= m) return;
  const double* a = A + (long long)row * m;
  double s = 0.0;
  for (int k = lane; k < m; k += 32) s = fma(a[k], x[k], s);
  s = warp_sum(s);
  if (lane == 0) y[row] = s;
}

// off-diagonal part of block t of a triangular solve: x[r0 + i] -= A[r0 + i, done] x[done],
// one warp per (row, 1/8 of the columns) with coalesced row reads; partials summed in order
__global__ void __launch_bounds__(256) k_lu_solve_offdiag(const double* __restrict__ LU, int m, int t, bool upper,
                                                          const double* __restrict__ x, double* __restrict__ part) {
  const int r0 = t * CS_NB, rb = min(CS_NB, m - r0);
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31, seg = blockIdx.y;
  if (row >= rb) return;
  const int k0 = upper ? r0 + rb : 0, k1 = upper ? m : r0;
  const int len = k1 - k0, per = (len + 7) / 8;
  const int a0 = k0 + seg * per, a1 = min(k1, a0 + per);
  const double* a = LU + (long long)(r0 + row) * m;
  double s = 0.0;
  for (int k = a0 + lane; k < a1; k += 32) s = fma(a[k], x[k], s);
  s = warp_sum(s);
  if (lane == 0) part[seg * CS_NB + row] = s;
}

// diagonal block t: x_t = D_t^{-1} (b_t - sum of the 8 partials)
__global__ void __launch_bounds__(256) k_lu_solve_block(const double* __restrict__ LU, int m, int t, bool upper,
                                                        double* __restrict__ x, const double* __restrict__ part) {
  __shared__ double xb[CS_NB];
  const int r0 = t * CS_NB, rb = min(CS_NB, m - r0);
  if (threadIdx.x < CS_NB) {
    const int i = threadIdx.x;
    double s = 0.0;
    for (int g = 0; g < 8; ++g) s += part[g * CS_NB + i];
    xb[i] = i < rb ? x[r0 + i] - s : 0.0;
  }
  __shared__ double D[CS_NB][CS_NB + 1];  // the diagonal block, staged once
  for (int e = threadIdx.x; e < rb * rb; e += blockDim.x) D[e / rb][e % rb] = LU[(long long)(r0 + e / rb) * m + r0 + e % rb];
  __syncthreads();
  // column-oriented substitution: step i finalises x_i, then every row below (L) / above (U) is updated
  if (!upper) {
    for (int i = 0; i < rb; ++i) {
      const double xi = xb[i];
      __syncthreads();
      if (threadIdx.x > i && threadIdx.x < rb) xb[threadIdx.x] = fma(-D[threadIdx.x][i], xi, xb[threadIdx.x]);
      __syncthreads();
    }
  } else {
    for (int i = rb - 1; i >= 0; --i) {
      if (threadIdx.x == 0) xb[i] = xb[i] / D[i][i];
      __syncthreads();
      const double xi = xb[i];
      if (threadIdx.x < i) xb[threadIdx.x] = fma(-D[threadIdx.x][i], xi, xb[threadIdx.x]);
      __syncthreads();
    }
  }
  if (threadIdx.x < rb) x[r0 + threadIdx.x] = xb[threadIdx.x];
}

__global__ void k_gather(const int* __restrict__ perm, int m, const double* __restrict__ x, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) y[i] = x[perm[i]];
}

}  // namespace hg

using namespace hg;

namespace {
template <typename T>
int up(T** d, const T* h, size_t n) {
  HG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(d), sizeof(T) * std::max<size_t>(n, 1)));
  if (h && n) HG_CUDA_TRY(cudaMemcpy(*d, h, sizeof(T) * n, cudaMemcpyHostToDevice));
  return HG_OK;
}

struct Bufs {
  std::vector<void*> p;
  ~Bufs() {
    for (void* x : p) cudaFree(x);
  }
  template <typename T>
  int add(T** d, const T* h, size_t n) {
    HG_TRY(up(d, h, n));
    p.push_back(*d);
    return HG_OK;
  }
};

double host_norm(const std::vector<double>& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
}  // namespace

#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace {
struct PhaseClock {  // HG_SETUP_TIMING=1: seconds per phase on stderr
  bool on = getenv("HG_SETUP_TIMING") && getenv("HG_SETUP_TIMING")[0] == '1';
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void tick(const char* what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[hg_coarse_setup] %-12s %.3f s\n", what, std::chrono::duration<double>(now - t).count());
    t = now;
  }
};
}  // namespace

extern "C" int hg_coarse_setup(const HgPrecondDesc* D, const int32_t* pair_ptr, const int32_t* pair_blk,
                               double* b0_out, double* lu_out, int32_t* piv_out, int32_t* info_out,
                               double* cert_out, int32_t cert_iters) {
  PhaseClock clk;
  if (!D || D->m <= 0 || !D->indptr || !D->z_data || !pair_ptr || !pair_blk) {
    set_error("hg_coarse_setup: bad argument");
    return HG_ERR_ARG;
  }
  const int n = D->n, m = D->m, nb = D->n_cblk;
  Bufs B;
  DevCsr A;
  A.n = n;
  A.nnz = D->nnz;
  HG_TRY(B.add(&A.indptr, D->indptr, (size_t)n + 1));
  HG_TRY(B.add(&A.indices, D->indices, (size_t)D->nnz));
  HG_TRY(B.add(&A.data, D->b_data, (size_t)D->nnz));
  std::vector<CsBlock> blk(nb);
  int col = 0;
  for (int b = 0; b < nb; ++b) {
    blk[b].n = D->cblk_n[b];
    blk[b].m = D->cblk_m[b];
    blk[b].col0 = col;
    blk[b].pad = 0;
    blk[b].idx_off = D->cblk_idx_off[b];
    blk[b].z_off = D->cblk_z_off[b];
    col += blk[b].m;
  }
  if (col != m) {
    set_error("hg_coarse_setup: block widths do not add up to m");
    return HG_ERR_ARG;
  }
  CsBlock* d_blk = nullptr;
  int *d_idx = nullptr, *d_nbr = nullptr;
  double *d_z = nullptr, *d_X = nullptr, *d_Y = nullptr, *d_B0 = nullptr;
  HG_TRY(B.add(&d_blk, blk.data(), blk.size()));
  HG_TRY(B.add(&d_idx, D->cblk_idx, (size_t)D->cblk_idx_off[nb]));
  HG_TRY(B.add(&d_z, D->z_data, (size_t)D->z_len));
  HG_TRY(B.add(&d_nbr, pair_blk, (size_t)pair_ptr[nb]));
  const int CW = HG_MAX_RHS;
  HG_TRY(B.add<double>(&d_X, nullptr, (size_t)n * CW));
  HG_TRY(B.add<double>(&d_Y, nullptr, (size_t)n * CW));
  HG_TRY(B.add<double>(&d_B0, nullptr, (size_t)m * m));
  HG_CUDA_TRY(cudaMemset(d_X, 0, sizeof(double) * (size_t)n * CW));
  HG_CUDA_TRY(cudaMemset(d_B0, 0, sizeof(double) * (size_t)m * m));
  int nchunk_max = 1, nbr_max = 1;
  for (int b = 0; b < nb; ++b) {
    if (blk[b].m > ZTY_MAXM) {
      set_error("hg_coarse_setup: more than 64 coarse columns in one block");
      return HG_ERR_UNSUPPORTED;
    }
    nchunk_max = std::max(nchunk_max, ceil_div(blk[b].n, ZTY_ROWS));
    nbr_max = std::max(nbr_max, pair_ptr[b + 1] - pair_ptr[b]);
  }
  double* d_part = nullptr;
  HG_TRY(B.add<double>(&d_part, nullptr, (size_t)nbr_max * nchunk_max * ZTY_MAXM * HG_MAX_RHS));
  cudaStream_t st = 0;
  // ---- B0 = Z^T (B Z), 16 columns of one block at a time
  for (int b = 0; b < nb; ++b) {
    const int na = pair_ptr[b + 1] - pair_ptr[b];
    for (int c0 = 0; c0 < blk[b].m; c0 += CW) {
      const int nc = std::min(CW, blk[b].m - c0);
      const int ne = blk[b].n * nc;
      k_scatter_zcols<<<ceil_div(ne, 256), 256, 0, st>>>(d_blk, b, c0, nc, d_idx, d_z, d_X, n);
      HG_LAUNCH_CHECK();
      HG_TRY(launch_spmm(A, A.data, d_X, n, d_Y, n, nc, st));
      if (na > 0) {
        k_zty_part<<<dim3(nchunk_max, na), 256, 0, st>>>(d_blk, d_nbr + pair_ptr[b], d_idx, d_z, d_Y, n, nc, d_part,
                                                         nchunk_max);
        HG_LAUNCH_CHECK();
        k_zty_reduce<<<na, 256, 0, st>>>(d_blk, d_nbr + pair_ptr[b], nc, blk[b].col0 + c0, d_part, nchunk_max, d_B0,
                                          m);
        HG_LAUNCH_CHECK();
      }
      k_clear_zcols<<<ceil_div(ne, 256), 256, 0, st>>>(d_blk, b, nc, d_idx, d_X, n);
      HG_LAUNCH_CHECK();
    }
  }
  const long long mm = (long long)m * m;
  k_symmetrise<<<ceil_div(mm, 256), 256, 0, st>>>(d_B0, m);
  HG_LAUNCH_CHECK();
  clk.tick("B0");
  if (b0_out) HG_CUDA_TRY(cudaMemcpy(b0_out, d_B0, sizeof(double) * mm, cudaMemcpyDeviceToHost));
  clk.tick("B0 to host");
  if (!lu_out && !piv_out && !cert_out) return HG_OK;

  // ---- getrf in a copy (B0 is kept for the certificate's power iteration)
  double* d_LU = nullptr;
  int *d_piv = nullptr, *d_info = nullptr;
  HG_TRY(B.add<double>(&d_LU, nullptr, (size_t)mm));
  HG_TRY(B.add<int>(&d_piv, nullptr, (size_t)m));
  HG_TRY(B.add<int>(&d_info, nullptr, 1));
  HG_CUDA_TRY(cudaMemcpy(d_LU, d_B0, sizeof(double) * mm, cudaMemcpyDeviceToDevice));
  HG_CUDA_TRY(cudaMemset(d_info, 0, sizeof(int)));
  for (int k0 = 0; k0 < m; k0 += CS_NB) {
    const int kb = std::min(CS_NB, m - k0);
    for (int j = k0; j < k0 + kb; ++j) {
      k_lu_pivot<<<1, 1024, 0, st>>>(d_LU, m, j, d_piv, d_info);
      k_lu_swap<<<std::max(1, std::min(64, ceil_div(m, 256))), 256, 0, st>>>(d_LU, m, j, d_piv);
      if (j + 1 < m) k_lu_panel<<<ceil_div(m - j - 1, 256), 256, 0, st>>>(d_LU, m, j, k0 + kb);
    }
    HG_LAUNCH_CHECK();
    const int rest = m - k0 - kb;
    if (rest > 0) {
      k_lu_trsm<<<ceil_div(rest, 128), 128, 0, st>>>(d_LU, m, k0, kb);
      HG_LAUNCH_CHECK();
      const dim3 grid(ceil_div(rest, CS_NB), ceil_div(rest, CS_NB));
      k_lu_gemm<<<grid, 256, 0, st>>>(d_LU, m, k0, kb);
      HG_LAUNCH_CHECK();
    }
  }
  HG_CUDA_TRY(cudaDeviceSynchronize());
  clk.tick("getrf");
  int info = 0;
  HG_CUDA_TRY(cudaMemcpy(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost));
  if (info_out) *info_out = info;
  if (lu_out) HG_CUDA_TRY(cudaMemcpy(lu_out, d_LU, sizeof(double) * mm, cudaMemcpyDeviceToHost));
  if (piv_out) HG_CUDA_TRY(cudaMemcpy(piv_out, d_piv, sizeof(int) * m, cudaMemcpyDeviceToHost));
  clk.tick("LU to host");

  // ---- certificate (coarse._sym_extreme_certificate): power iteration on B0
  // for |lambda|_max, inverse iteration through the LU for 1 / |lambda|_min
  if (cert_out && info == 0) {
    const int iters = cert_iters > 0 ? cert_iters : 60;
    double *d_x = nullptr, *d_y = nullptr;
    HG_TRY(B.add<double>(&d_x, nullptr, (size_t)m));
    HG_TRY(B.add<double>(&d_y, nullptr, (size_t)m));
    std::vector<double> hx(m), hy(m);
    unsigned long long s = 12345;
    auto rnd = [&]() {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      return (double)(s >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    };
    for (double& v : hx) v = rnd();
    double lmax = 0.0, inv_max = 0.0;
    for (int it = 0; it < iters; ++it) {
      const double nx = host_norm(hx);
      HG_CUDA_TRY(cudaMemcpy(d_x, hx.data(), sizeof(double) * m, cudaMemcpyHostToDevice));
      k_gemv<<<ceil_div(m, 8), 256, 0, st>>>(d_B0, m, d_x, d_y);
      HG_LAUNCH_CHECK();
      HG_CUDA_TRY(cudaMemcpy(hy.data(), d_y, sizeof(double) * m, cudaMemcpyDeviceToHost));
      const double ny = host_norm(hy);
      lmax = ny / nx;
      for (int i = 0; i < m; ++i) hx[i] = hy[i] / ny;
    }
    clk.tick("power iter");
    std::vector<int> hpiv(m), perm(m);
    HG_CUDA_TRY(cudaMemcpy(hpiv.data(), d_piv, sizeof(int) * m, cudaMemcpyDeviceToHost));
    for (int i = 0; i < m; ++i) perm[i] = i;
    for (int i = 0; i < m; ++i)
      if (hpiv[i] != i) std::swap(perm[i], perm[hpiv[i]]);  // (P b)[i] = b[perm[i]] (getrs row interchanges)
    int* d_perm = nullptr;
    double* d_sp = nullptr;  // 8 x 64 partial sums of one block's off-diagonal rows
    HG_TRY(B.add(&d_perm, perm.data(), (size_t)m));
    HG_TRY(B.add<double>(&d_sp, nullptr, 8 * CS_NB));
    for (double& v : hx) v = rnd();
    const int K = ceil_div(m, CS_NB);
    for (int it = 0; it < iters; ++it) {
      const double nx = host_norm(hx);
      HG_CUDA_TRY(cudaMemcpy(d_x, hx.data(), sizeof(double) * m, cudaMemcpyHostToDevice));
      k_gather<<<ceil_div(m, 256), 256, 0, st>>>(d_perm, m, d_x, d_y);  // getrs: row interchanges first
      for (int t = 0; t < K; ++t) {
        k_lu_solve_offdiag<<<dim3(8, 8), 256, 0, st>>>(d_LU, m, t, false, d_y, d_sp);
        k_lu_solve_block<<<1, 256, 0, st>>>(d_LU, m, t, false, d_y, d_sp);
      }
      for (int t = K - 1; t >= 0; --t) {
        k_lu_solve_offdiag<<<dim3(8, 8), 256, 0, st>>>(d_LU, m, t, true, d_y, d_sp);
        k_lu_solve_block<<<1, 256, 0, st>>>(d_LU, m, t, true, d_y, d_sp);
      }
      HG_LAUNCH_CHECK();
      HG_CUDA_TRY(cudaMemcpy(hy.data(), d_y, sizeof(double) * m, cudaMemcpyDeviceToHost));
      const double ny = host_norm(hy);
      inv_max = ny / nx;
      for (int i = 0; i < m; ++i) hx[i] = hy[i] / ny;
    }
    cert_out[0] = lmax;
    cert_out[1] = inv_max;
    clk.tick("inverse iter");
  }
  return HG_OK;
}
