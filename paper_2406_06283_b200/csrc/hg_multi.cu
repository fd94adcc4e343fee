// Multi-RHS (batched) solve phase — SURVEY §8a row a15: BASELINE config 5's
// 16 seeded right-hand sides solved as one batch.  There is no reference
// function; the oracle is the one-at-a-time path (schwarz.py:51-61 per
// column).  Every kernel here keeps the columns independent (column c of an
// output depends only on column c of the input), so a batch is exactly nrhs
// single solves sharing the operator streams:
//
//  k_spmm        Y = A X for up to 16 columns, the CSR row read once; each
//                column summed in index order without FMA (bitwise equal to
//                scipy's csr_matvec, like k_spmv); optional self dots X.Y.
//  k_zt_multi    C_b = Z_b^T R_b per (block, 256-row chunk) as a dense FP64
//                contraction on the tensor pipe (DMMA m8n8k4): A = Z^T read
//                once from HBM, B = the gathered 256 x 16 R chunk in smem.
//  k_b0_multi    Y = B0^{-1} C with the tiled getrf factors (hg_b0.cu /
//                hg_b0c.cu layout): persistent CTAs, panel t owned by CTA
//                t % G, each 64 x 64 x 16 tile product on DMMA, panels
//                handed over as (value, tag) pairs in L2 (the data is the
//                flag: one round trip per hop).
//  k_zy_multi    U_b = Z_b Y_b (256 rows x m_b x 16) on DMMA.
//  k_assemble_multi  out = coarse + local contributions in the reference's
//                fixed summation order (schwarz.py:52-61), per column.
//  batched Arnoldi helpers (dots / reduce / axpy / scale over a column list).
#include <algorithm>
#include <cstdlib>

#include "hg_internal.cuh"

namespace hg {

constexpr int MR = HG_MAX_RHS;  // layout stride of the [row][rhs] coarse batch arrays
constexpr int SR = 20;          // smem row stride (doubles) of 16-column operand tiles:
                                // conflict-free DMMA B-fragment loads (20 = 4 mod 16)
constexpr int ZROWS = 256;      // rows per Z^T R / Z Y work item (the k_zt chunking)

// D = A B + D, m8n8k4 FP64 (DMMA).  Fragments (lane = 4 g + q):
//   A[g][q], B[q][g], D[g][2q], D[g][2q+1].
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ SpMM
// FULL: all HG_MAX_RHS columns in their natural order (the block solve until columns converge):
// no per-column predicates or column-list lookups, one pointer walk over the columns per nonzero
// (the general path spends ~18 instructions per nonzero and column, this one ~6).
template <bool FULL>
__global__ void __launch_bounds__(256) k_spmm(int n, const int* __restrict__ ip, const int* __restrict__ ix,
                                              const double* __restrict__ a, const double* __restrict__ X,
                                              long long ldx, double* __restrict__ Y, long long ldy, ColList cols,
                                              double* __restrict__ partials, int width, int nb) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int nr = FULL ? MR : cols.n;
  double s[MR];
#pragma unroll
  for (int c = 0; c < MR; ++c) s[c] = 0.0;
  if (i < n) {
    const int e1 = ip[i + 1];
    for (int e = ip[i]; e < e1; ++e) {
      const double av = a[e];
      const int col = ix[e];
      if (FULL) {
        const double* xp = X + col;
#pragma unroll
        for (int c = 0; c < MR; ++c) {
          s[c] = __dadd_rn(s[c], __dmul_rn(av, __ldg(xp)));
          xp += ldx;
        }
      } else {
#pragma unroll
        for (int c = 0; c < MR; ++c)
          if (c < nr) s[c] = __dadd_rn(s[c], __dmul_rn(av, __ldg(X + (long long)cols.c[c] * ldx + col)));
      }
    }
    if (FULL) {
      double* yp = Y + i;
#pragma unroll
      for (int c = 0; c < MR; ++c) {
        *yp = s[c];
        yp += ldy;
      }
    } else {
#pragma unroll
      for (int c = 0; c < MR; ++c)
        if (c < nr) Y[(long long)cols.c[c] * ldy + i] = s[c];
    }
  }
  if (partials) {  // self dots X_c . Y_c, fixed-order block reduction per column
    __shared__ double s_w[8][MR];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < MR; ++c) {
      if (c < nr) {
        double v = i < n ? __ldg(X + (long long)cols.c[c] * ldx + i) * s[c] : 0.0;
        v = warp_sum(v);
        if (lane == 0) s_w[warp][c] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x < nr) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += s_w[w][threadIdx.x];
      partials[((long long)cols.c[threadIdx.x] * nb + blockIdx.x) * width] = t;
    }
  }
}

static ColList all_cols(int nrhs) {
  ColList c{};
  c.n = nrhs;
  for (int k = 0; k < nrhs; ++k) c.c[k] = k;
  return c;
}

static int spmm_impl(const DevCsr& A, const double* vals, const double* X, long long ldx, double* Y, long long ldy,
                     const ColList& cols, double* partials, int width, int* nb_out, cudaStream_t st) {
  const int nb = ceil_div(A.n, 256);
  if (nb_out) *nb_out = nb;
  if (A.n == 0 || cols.n == 0) return HG_OK;
  if (cols.n > MR) {
    set_error("spmm: more than HG_MAX_RHS columns");
    return HG_ERR_ARG;
  }
  bool full = cols.n == MR;
  for (int c = 0; c < MR && full; ++c) full = cols.c[c] == c;
  if (full)
    k_spmm<true><<<nb, 256, 0, st>>>(A.n, A.indptr, A.indices, vals, X, ldx, Y, ldy, cols, partials, width, nb);
  else
    k_spmm<false><<<nb, 256, 0, st>>>(A.n, A.indptr, A.indices, vals, X, ldx, Y, ldy, cols, partials, width, nb);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

int launch_spmm(const DevCsr& A, const double* vals, const double* X, long long ldx, double* Y, long long ldy,
                int nrhs, cudaStream_t st) {
  return spmm_impl(A, vals, X, ldx, Y, ldy, all_cols(nrhs), nullptr, 0, nullptr, st);
}

int launch_spmm_cols(const DevCsr& A, const double* vals, const double* X, long long ldx, double* Y, long long ldy,
                     const ColList& cols, double* partials, int width, int* nb_out, cudaStream_t st) {
  return spmm_impl(A, vals, X, ldx, Y, ldy, cols, partials, width, nb_out, st);
}

int launch_spmm_self(const DevCsr& A, const double* vals, const double* X, long long ldx, double* Y, long long ldy,
                     int nrhs, double* partials, int width, int* nb_out, cudaStream_t st) {
  return spmm_impl(A, vals, X, ldx, Y, ldy, all_cols(nrhs), partials, width, nb_out, st);
}

// ------------------------------------------------------------------ Z^T R
__global__ void k_zt_multi_pk(const int2*, const CblkDesc*, const int*, const long long*, const double2*, const double*,
                              long long, int, double*, unsigned long long*);
struct ZyItem;
__global__ void k_zy_multi_pk(const ZyItem*, int, const double2*, const double*, int, double*, long long);
__global__ void __launch_bounds__(256) k_zt_multi(const int2* __restrict__ items, const CblkDesc* __restrict__ descs,
                                                  const int* __restrict__ idx, const double* __restrict__ Z,
                                                  const double* __restrict__ R, long long ldr, int nrhs,
                                                  double* __restrict__ cpartm,
                                                  unsigned long long* __restrict__ blk_done) {
  __shared__ __align__(16) double s_r[ZROWS * SR];
  const int2 it = items[blockIdx.x];
  const CblkDesc d = descs[it.x];
  const int k0 = it.y * ZROWS, rows = min(ZROWS, d.n - k0);
  const int* ib = idx + d.idx_off + k0;
  for (int e = threadIdx.x; e < ZROWS * MR; e += 256) {  // gather the chunk, zero padded
    const int k = e % ZROWS, c = e / ZROWS;
    double v = 0.0;
    if (k < rows && c < nrhs) v = __ldg(R + (long long)c * ldr + __ldg(ib + k));
    s_r[k * SR + c] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  const double* zb = Z + d.z_off + (long long)k0 * d.m;
  for (int i0 = warp * 8; i0 < d.m; i0 += 64) {  // 8 coarse columns of the block per warp
    const int col = i0 + g;
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
#pragma unroll 8
    for (int ks = 0; ks < ZROWS; ks += 4) {
      const int k = ks + q;
      const double a = (k < rows && col < d.m) ? __ldg(zb + (long long)k * d.m + col) : 0.0;  // A = Z^T
      dmma(c0, a, s_r[k * SR + g]);
      dmma(c1, a, s_r[k * SR + 8 + g]);
    }
    if (col < d.m) {
      double* dst = cpartm + (d.part_off + (long long)it.y * d.m + col) * MR;
      *reinterpret_cast<double2*>(dst + 2 * q) = make_double2(c0[0], c0[1]);
      *reinterpret_cast<double2*>(dst + 8 + 2 * q) = make_double2(c1[0], c1[1]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // chunk complete: the batched coarse solve may be waiting for it
    __threadfence();
    atomicAdd(blk_done + it.x, 1ull);
  }
}

int launch_zt_multi(HgPrecond* P, const double* R, long long ldr, int nrhs, cudaStream_t st) {
  if (P->m == 0 || P->n_zt_items == 0) return HG_OK;
  if (P->skip_zt > 0) {  // fault injection (hg_debug_set)
    --P->skip_zt;
    return HG_OK;
  }
  if (P->d_ztpk)
    k_zt_multi_pk<<<P->n_zt_items, 256, 0, st>>>(P->d_zt_items, P->d_cblk, P->d_cblk_idx, P->d_ztpk_off,
                                                  reinterpret_cast<const double2*>(P->d_ztpk), R, ldr, nrhs,
                                                  P->d_cpartm, P->d_blkm_done);
  else
    k_zt_multi<<<P->n_zt_items, 256, 0, st>>>(P->d_zt_items, P->d_cblk, P->d_cblk_idx, P->d_z, R, ldr, nrhs,
                                               P->d_cpartm, P->d_blkm_done);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// ------------------------------------------------------------------ Z Y
__global__ void __launch_bounds__(256) k_zy_multi(const int2* __restrict__ items, const CblkDesc* __restrict__ descs,
                                                  const double* __restrict__ Z, const double* __restrict__ ym,
                                                  int nrhs, double* __restrict__ zsm, long long zs_len) {
  __shared__ __align__(16) double s_y[64 * SR];
  const int2 it = items[blockIdx.x];
  const CblkDesc d = descs[it.x];
  const int k0 = it.y * ZROWS, rows = min(ZROWS, d.n - k0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  double acc[4][2][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h) acc[t][h][0] = acc[t][h][1] = 0.0;
  const double* zb = Z + d.z_off + (long long)k0 * d.m;
  for (int l0 = 0; l0 < d.m; l0 += 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * MR; e += 256) {
      const int l = e / MR, c = e % MR;
      s_y[l * SR + c] = (l0 + l < d.m && c < nrhs) ? ym[(long long)(d.col0 + l0 + l) * MR + c] : 0.0;
    }
    __syncthreads();
    const int lc = min(64, d.m - l0);
    for (int ks = 0; ks < lc; ks += 4) {
      const int l = ks + q;
      const double b0 = s_y[l * SR + g], b1 = s_y[l * SR + 8 + g];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int row = warp * 32 + t * 8 + g;
        const double a = (row < rows && l0 + l < d.m) ? __ldg(zb + (long long)row * d.m + l0 + l) : 0.0;
        dmma(acc[t][0], a, b0);
        dmma(acc[t][1], a, b1);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int row = warp * 32 + t * 8 + g;
    if (row >= rows) continue;
    double* dst = zsm + d.idx_off + k0 + row;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * h + 2 * q + e;
        if (c < nrhs) dst[(long long)c * zs_len] = acc[t][h][e];
      }
  }
}

int launch_zy_multi(HgPrecond* P, int nrhs, cudaStream_t st) {
  if (P->m == 0 || P->n_zt_items == 0) return HG_OK;
  if (P->d_zypk)
    k_zy_multi_pk<<<ceil_div(P->n_zy_items, 8), 256, 0, st>>>(reinterpret_cast<const ZyItem*>(P->d_zy_items),
                                                               P->n_zy_items,
                                                               reinterpret_cast<const double2*>(P->d_zypk), P->d_ym,
                                                               nrhs, P->d_zsm, P->zs_len);
  else
    k_zy_multi<<<P->n_zt_items, 256, 0, st>>>(P->d_zt_items, P->d_cblk, P->d_z, P->d_ym, nrhs, P->d_zsm, P->zs_len);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// ------------------------------------------------------------------ packed Z (batched applies)
// The batched contractions stream Z in DMMA A-fragment order (8 x 8 blocks, one 16-byte load per
// lane per two k-steps, 512 contiguous bytes per warp load — as B0^{-1} in hg_b0d.cu), built once
// from the row-major blocks on the first batched call:
//   zy copy: block b, row tile mt, k-block kb (coarse columns 8 kb ..) at double2 index
//            zoff[b] / 2 + (mt KB_b + kb) 32 + lane: {Z[8 mt + g][8 kb + q], Z[8 mt + g][8 kb + 4 + q]}
//   zt copy: block b, 256-row chunk ch, coarse-column tile mt, k-block kb (rows 256 ch + 8 kb ..):
//            toff[b] / 2 + ((ch MT_b + mt) 32 + kb) 32 + lane:
//            {Z[r0 + 8 kb + q][8 mt + g], Z[r0 + 8 kb + 4 + q][8 mt + g]}     (A = Z^T)
// both zero padded to whole tiles.
__global__ void k_zpack_zy(const CblkDesc* __restrict__ descs, const long long* __restrict__ zoff,
                           const double* __restrict__ Z, double2* __restrict__ out) {
  const CblkDesc d = descs[blockIdx.y];
  const int KB = (d.m + 7) >> 3, MT = (d.n + 7) >> 3;
  const long long ne = (long long)MT * KB * 32;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(e & 31), g = lane >> 2, q = lane & 3;
    const long long blk = e >> 5;
    const int kb = (int)(blk % KB), mt = (int)(blk / KB);
    const int row = mt * 8 + g, c0 = kb * 8 + q, c1 = c0 + 4;
    double2 v;
    v.x = (row < d.n && c0 < d.m) ? Z[d.z_off + (long long)row * d.m + c0] : 0.0;
    v.y = (row < d.n && c1 < d.m) ? Z[d.z_off + (long long)row * d.m + c1] : 0.0;
    out[(zoff[blockIdx.y] >> 1) + e] = v;
  }
}

__global__ void k_zpack_zt(const CblkDesc* __restrict__ descs, const long long* __restrict__ toff,
                           const double* __restrict__ Z, double2* __restrict__ out) {
  const CblkDesc d = descs[blockIdx.y];
  const int MT = (d.m + 7) >> 3;
  const long long ne = (long long)d.nchunk * MT * 32 * 32;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(e & 31), g = lane >> 2, q = lane & 3;
    long long t = e >> 5;
    const int kb = (int)(t & 31);
    t >>= 5;
    const int mt = (int)(t % MT), ch = (int)(t / MT);
    const int col = mt * 8 + g, r0 = ch * ZROWS + kb * 8 + q, r1 = r0 + 4;
    double2 v;
    v.x = (col < d.m && r0 < d.n) ? Z[d.z_off + (long long)r0 * d.m + col] : 0.0;
    v.y = (col < d.m && r1 < d.n) ? Z[d.z_off + (long long)r1 * d.m + col] : 0.0;
    out[(toff[blockIdx.y] >> 1) + e] = v;
  }
}

// C_b partial of one (block, 256-row chunk): the gathered chunk of R in shared memory (B
// fragments), a warp per 8-column tile of the block streaming its packed Z^T fragments
__global__ void __launch_bounds__(256) k_zt_multi_pk(const int2* __restrict__ items, const CblkDesc* __restrict__ descs,
                                                     const int* __restrict__ idx, const long long* __restrict__ toff,
                                                     const double2* __restrict__ zt, const double* __restrict__ R,
                                                     long long ldr, int nrhs, double* __restrict__ cpartm,
                                                     unsigned long long* __restrict__ blk_done) {
  __shared__ __align__(16) double s_r[ZROWS * SR];
  const int2 it = items[blockIdx.x];
  const CblkDesc d = descs[it.x];
  const int k0 = it.y * ZROWS, rows = min(ZROWS, d.n - k0);
  const int* ib = idx + d.idx_off + k0;
  for (int e = threadIdx.x; e < ZROWS * MR; e += 256) {  // gather the chunk, zero padded
    const int k = e % ZROWS, c = e / ZROWS;
    double v = 0.0;
    if (k < rows && c < nrhs) v = __ldg(R + (long long)c * ldr + __ldg(ib + k));
    s_r[k * SR + c] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  const int MT = (d.m + 7) >> 3;
  const double2* base = zt + (toff[it.x] >> 1) + (size_t)it.y * MT * 1024;
  for (int mt = warp; mt < MT; mt += 8) {
    const double2* ap = base + (size_t)mt * 1024 + lane;
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
#pragma unroll 8
    for (int kb = 0; kb < 32; ++kb) {
      const double2 a = __ldcs(ap + kb * 32);
      const double* b = s_r + (kb * 8 + q) * SR + g;
      dmma(c0, a.x, b[0]);
      dmma(c1, a.x, b[8]);
      dmma(c0, a.y, b[4 * SR]);
      dmma(c1, a.y, b[4 * SR + 8]);
    }
    const int col = mt * 8 + g;
    if (col < d.m) {
      double* dst = cpartm + (d.part_off + (long long)it.y * d.m + col) * MR;
      *reinterpret_cast<double2*>(dst + 2 * q) = make_double2(c0[0], c0[1]);
      *reinterpret_cast<double2*>(dst + 8 + 2 * q) = make_double2(c1[0], c1[1]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // chunk complete: the batched coarse solve may be waiting for it
    __threadfence();
    atomicAdd(blk_done + it.x, 1ull);
  }
}

// U_b rows: a warp owns two 8-row tiles of a block and streams their packed fragments (at most
// 2 x 8 loads, all issued before the first product); Y comes from [coarse column][16] through L1.
// The work item carries everything the warp needs (no dependent descriptor loads before the stream).
struct ZyItem {
  long long a_off;    // double2 index of the pair's first packed tile
  long long dst_off;  // position of the pair's first row in the zs scratch
  int col0, m;        // the block's first coarse column and its width
  int rows, pad;      // rows of the pair that exist (1..16)
};

__global__ void __launch_bounds__(256) k_zy_multi_pk(const ZyItem* __restrict__ items, int nitems,
                                                     const double2* __restrict__ zp, const double* __restrict__ ym,
                                                     int nrhs, double* __restrict__ zsm, long long zs_len) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  const int iw = blockIdx.x * 8 + warp;
  if (iw >= nitems) return;
  const ZyItem it = items[iw];
  const int KB = (it.m + 7) >> 3;
  const bool two = it.rows > 8;
  const double2* a0p = zp + it.a_off + lane;
  const double2* a1p = two ? a0p + (size_t)KB * 32 : a0p;
  const double* cp = ym + ((size_t)it.col0 + q) * MR + g;
  double acc[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
  for (int kb0 = 0; kb0 < KB; kb0 += 8) {
    double2 a0[8], a1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int kb = min(kb0 + u, KB - 1);
      a0[u] = __ldcs(a0p + kb * 32);
      a1[u] = __ldcs(a1p + kb * 32);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int kb = kb0 + u;
      if (kb < KB) {
        const int k = kb * 8 + q;
        const bool v0 = k < it.m, v1 = k + 4 < it.m;
        const double* cu = cp + (size_t)kb * 8 * MR;
        const double b00 = v0 ? __ldg(cu) : 0.0, b01 = v0 ? __ldg(cu + 8) : 0.0;
        const double b10 = v1 ? __ldg(cu + 4 * MR) : 0.0, b11 = v1 ? __ldg(cu + 4 * MR + 8) : 0.0;
        dmma(acc[0][0], a0[u].x, b00);
        dmma(acc[0][1], a0[u].x, b01);
        dmma(acc[1][0], a1[u].x, b00);
        dmma(acc[1][1], a1[u].x, b01);
        dmma(acc[0][0], a0[u].y, b10);
        dmma(acc[0][1], a0[u].y, b11);
        dmma(acc[1][0], a1[u].y, b10);
        dmma(acc[1][1], a1[u].y, b11);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int row = t * 8 + g;
    if (row >= it.rows) continue;
    double* dst = zsm + it.dst_off + row;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * h + 2 * q + e;
        if (c < nrhs) dst[(long long)c * zs_len] = acc[t][h][e];
      }
  }
}

// ------------------------------------------------------------------ B0^{-1}
namespace {
constexpr int BP = 64;
constexpr int BTILE = BP * BP;

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// element (r, c) of a 64 x 64 tile; swizzled tiles (cluster layout,
// factor.swizzle_tile_rows) keep 16-byte chunk c/2 of row r at chunk
// (c/2) ^ ((r & 1) << 2)
__device__ __forceinline__ int tidx(int r, int c, int swz) {
  return r * BP + (swz ? ((((c >> 1) ^ ((r & 1) << 2)) << 1) | (c & 1)) : c);
}

// this lane's 16 A fragments of rows `row` of a tile (scaled by sign)
__device__ __forceinline__ void load_afrag(double (&av)[16], const double* __restrict__ T, int row, int q, int swz,
                                           double sign) {
#pragma unroll
  for (int s = 0; s < 16; ++s) av[s] = sign * __ldg(T + tidx(row, 4 * s + q, swz));
}

// acc (8 x 16 rows of this warp) += A (this warp's 8 tile rows) * X (64 x 16, smem)
__device__ __forceinline__ void mma_tile(double (&acc)[2][2], const double (&av)[16], const double* s_x, int q, int g) {
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    const int k = 4 * s + q;
    dmma(acc[0], av[s], s_x[k * SR + g]);
    dmma(acc[1], av[s], s_x[k * SR + 8 + g]);
  }
}
}  // namespace

struct B0MultiArgs {
  int m, K, nrhs, premul, swz;
  const int* perm;
  const int* col_blk;
  const CblkDesc* descs;
  const double* cpartm;     // [part][MR]
  const double* dinv;       // [2K][64][64]
  const long long* tile_ptr;
  const int* tile_col;
  const double* tiles;      // [ntile][64][64]
  double* xbuf;             // [2K][64][MR] (value, tag) pairs: 2 doubles each
  double* y;                // [m][MR]
  const unsigned long long* blk_done;  // per coarse block Z^T R chunk counters
  unsigned long long* ticket;          // launch index (take_launch_index): launch L reads Z^T R launch L
                                       // (block b complete at (L + 1) nchunk_b) and tags panel g with
                                       // 1 + 2K L + g (unique across launches, exact in a double)
  SpinCfg spin;
};

// 16-byte (value, tag) pair access: written and read as one vector access,
// L1 bypassed on the read side.
__device__ __forceinline__ void st_pair(double* p, double v, double tag) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v), "d"(tag) : "memory");
}
__device__ __forceinline__ double2 ld_pair(const double* p) {
  double2 r;
  asm volatile("ld.volatile.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p) : "memory");
  return r;
}

// Load panel gp (64 x MR values) of this launch into s_x, spinning until every
// pair carries the panel's tag: the data is its own completion flag, so a hop
// costs one L2 round trip (no counter, no fence, no ordered publication).
__device__ __forceinline__ void wait_panel(const double* __restrict__ xbuf, int gp, double tag, double* s_x,
                                           bool reversed, int K, const SpinCfg& spin, bool& dead) {
  // thread t covers pairs t, t + 256, t + 512, t + 768 of the panel (rows r = e / MR)
  const double* base = xbuf + (size_t)gp * BP * MR * 2;
  double v[4];
  bool ok;
  SpinGuard sg;
  do {
    ok = true;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = threadIdx.x + 256 * q;
      const double2 p = ld_pair(base + 2 * e);
      v[q] = p.x;
      ok = ok && (p.y == tag);
    }
    if (!ok && (dead || spin_abort(sg, spin))) {  // bounded: give up on a faulted handle
      dead = true;
      ok = true;
    }
  } while (!ok);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + 256 * q;
    const int r = e / MR, c = e % MR;
    s_x[(reversed ? BP - 1 - r : r) * SR + c] = v[q];
  }
  (void)K;
}

// Panel g (phase ph = g / K: 0 = L solve of P c, 1 = U solve in reversed
// coordinates of the L solution) of 64 rows x nrhs columns; warp w owns
// panel rows 8w..8w+7.  premul (cluster layout): tiles are D_t^{-1} T[t, j]
// and x_t = D_t^{-1} rhs_t - sum_j M[t, j] x_j; otherwise
// x_t = D_t^{-1} (rhs_t - sum_j T[t, j] x_j).  Tiles in ascending j: the
// summation order is fixed, the result deterministic.  Panels are handed
// over as tagged pairs in global memory (wait_panel).
__global__ void __launch_bounds__(256, 1) k_b0_multi(B0MultiArgs a) {
  __shared__ __align__(16) double s_x[BP * SR];
  __shared__ unsigned long long s_launch;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = lane & 3, g8 = lane >> 2;
  const int row = warp * 8 + g8;
  const int K = a.K;
  if (tid == 0) s_launch = take_launch_index(a.ticket, gridDim.x);
  __syncthreads();
  const unsigned long long L = s_launch;
  const double tag0 = 1.0 + 2.0 * (double)K * (double)L;
  bool dead = false;
  for (int g = blockIdx.x; g < 2 * K; g += gridDim.x) {
    const int ph = g / K, t = g % K;
    const double* dinv_g = a.dinv + (size_t)g * BTILE;
    double av[16];
    if (a.premul) load_afrag(av, dinv_g, row, q, a.swz, 1.0);
    __syncthreads();  // s_x free
    if (ph == 0) {
      for (int e = tid; e < BP * MR; e += 256) {
        const int r = e / MR, c = e % MR;
        double v = 0.0;
        const int i = t * BP + r;
        if (c < a.nrhs && i < a.m) {
          // launched before Z^T R: wait for this row's coarse block only
          const int col = a.perm[i];
          const int b = a.col_blk[col];
          const CblkDesc d = a.descs[b];
          const unsigned long long need = (L + 1) * (unsigned long long)d.nchunk;
          SpinGuard sg;
          while (!dead && ld_acq(a.blk_done + b) < need)
            if (spin_abort(sg, a.spin)) dead = true;
          const int l = col - d.col0;
          for (int ch = 0; ch < d.nchunk; ++ch) v += a.cpartm[(d.part_off + (long long)ch * d.m + l) * MR + c];
        }
        s_x[r * SR + c] = v;
      }
    } else {  // the reversed L solution of panel K-1-t
      wait_panel(a.xbuf, K - 1 - t, tag0 + (K - 1 - t), s_x, true, K, a.spin, dead);
    }
    __syncthreads();
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    if (a.premul) {
      mma_tile(acc, av, s_x, q, g8);
    } else {
      acc[0][0] = s_x[row * SR + 2 * q];
      acc[0][1] = s_x[row * SR + 2 * q + 1];
      acc[1][0] = s_x[row * SR + 8 + 2 * q];
      acc[1][1] = s_x[row * SR + 8 + 2 * q + 1];
    }
    const long long e0 = a.tile_ptr[g], e1 = a.tile_ptr[g + 1];
    for (long long e = e0; e < e1; ++e) {
      const int gj = ph * K + a.tile_col[e];
      load_afrag(av, a.tiles + (size_t)e * BTILE, row, q, a.swz, -1.0);  // in flight across the wait
      __syncthreads();  // s_x free
      wait_panel(a.xbuf, gj, tag0 + gj, s_x, false, K, a.spin, dead);
      __syncthreads();
      mma_tile(acc, av, s_x, q, g8);
    }
    if (!a.premul) {  // x_t = D_t^{-1} acc
      load_afrag(av, dinv_g, row, q, a.swz, 1.0);
      __syncthreads();
      *reinterpret_cast<double2*>(s_x + row * SR + 2 * q) = make_double2(acc[0][0], acc[0][1]);
      *reinterpret_cast<double2*>(s_x + row * SR + 8 + 2 * q) = make_double2(acc[1][0], acc[1][1]);
      __syncthreads();
      acc[0][0] = acc[0][1] = acc[1][0] = acc[1][1] = 0.0;
      mma_tile(acc, av, s_x, q, g8);
    }
    // publish: every value with the panel's tag (no fence: each pair is its own flag)
    const double tag = tag0 + g;
    double* xo = a.xbuf + ((size_t)g * BP + row) * MR * 2;
    st_pair(xo + 2 * (2 * q), acc[0][0], tag);
    st_pair(xo + 2 * (2 * q + 1), acc[0][1], tag);
    st_pair(xo + 2 * (8 + 2 * q), acc[1][0], tag);
    st_pair(xo + 2 * (8 + 2 * q + 1), acc[1][1], tag);
    if (ph == 1) {
      const int i = K * BP - 1 - (t * BP + row);
      if (i < a.m) {
        double* yo = a.y + (size_t)i * MR;
        *reinterpret_cast<double2*>(yo + 2 * q) = make_double2(acc[0][0], acc[0][1]);
        *reinterpret_cast<double2*>(yo + 8 + 2 * q) = make_double2(acc[1][0], acc[1][1]);
      }
    }
  }
}

int launch_b0_multi(HgPrecond* P, int nrhs, cudaStream_t st) {
  if (P->m == 0) return HG_OK;
  if (P->b0_P != BP) {
    set_error("batched coarse solve: needs 64-row panels (HG_B0_PANEL=64)");
    return HG_ERR_UNSUPPORTED;
  }
  const int K = P->b0_K;
  static const int env_g = getenv("HG_B0M_CTAS") ? atoi(getenv("HG_B0M_CTAS")) : 0;
  const int G = std::min(K, env_g > 0 ? env_g : 16);
  // tags stay below 2^53 (exact in a double) for ~10^12 launches
  B0MultiArgs a{P->m, K, nrhs, P->b0_mode == 1 ? 1 : 0, P->b0_mode == 1 ? 1 : 0, P->d_b0_perm, P->d_col_blk,
                P->d_cblk, P->d_cpartm, P->d_b0_dinv, P->d_b0_tile_ptr, P->d_b0_tile_col, P->d_b0_tiles,
                P->d_b0m_x, P->d_ym, P->d_blkm_done, P->d_ticket + 1, spin_cfg(P)};
  k_b0_multi<<<G, 256, 0, st>>>(a);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// ------------------------------------------------------------------ assembly
// one thread per dof, all columns: the contributor lists are read once (not
// once per column); per column the sum runs in the reference's fixed order
__global__ void __launch_bounds__(256) k_assemble_multi(int n, const int* __restrict__ cptr,
                                                        const long long* __restrict__ cent,
                                                        const double* __restrict__ zsm, long long zs_len,
                                                        const int* __restrict__ lptr,
                                                        const long long* __restrict__ lent,
                                                        const double* __restrict__ xsm, long long xs_len,
                                                        double* __restrict__ out, long long ldo, int nrhs) {
  const int d = blockIdx.x * 256 + threadIdx.x;
  if (d >= n) return;
  double acc[MR];
#pragma unroll
  for (int c = 0; c < MR; ++c) acc[c] = 0.0;
  if (cptr) {
    for (int e = cptr[d]; e < cptr[d + 1]; ++e) {
      const double* z = zsm + cent[e];
#pragma unroll
      for (int c = 0; c < MR; ++c)
        if (c < nrhs) acc[c] += z[(long long)c * zs_len];
    }
  }
  if (lptr) {
    for (int e = lptr[d]; e < lptr[d + 1]; ++e) {
      const double* x = xsm + lent[e];
#pragma unroll
      for (int c = 0; c < MR; ++c)
        if (c < nrhs) acc[c] += x[(long long)c * xs_len];
    }
  }
#pragma unroll
  for (int c = 0; c < MR; ++c)
    if (c < nrhs) out[(long long)c * ldo + d] = acc[c];
}

int launch_assemble_multi(HgPrecond* P, bool with_coarse, bool with_local, double* OUT, long long ldo, int nrhs,
                          cudaStream_t st) {
  if (P->n == 0 || nrhs == 0) return HG_OK;
  const bool coarse = with_coarse && P->m > 0;
  k_assemble_multi<<<ceil_div(P->n, 256), 256, 0, st>>>(P->n, coarse ? P->d_cptr : nullptr, P->d_cent, P->d_zsm,
                                                        P->zs_len, with_local ? P->d_lptr : nullptr, P->d_lent,
                                                        P->d_xsm, P->xs_len, OUT, ldo, nrhs);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// ------------------------------------------------------------------ batched Arnoldi
__global__ void __launch_bounds__(VEC_THREADS) k_dots_batch(int n, const double* __restrict__ z, long long ldz,
                                                            const double* __restrict__ V, long long ldv,
                                                            long long ldcol, int nv, ColList cols,
                                                            double* __restrict__ partials, int width, int nb) {
  const int c = cols.c[blockIdx.y];
  const double* zc = z + (long long)c * ldz;
  double zv[VEC_ROWS];
  int rows[VEC_ROWS];
  double self = 0.0;
#pragma unroll
  for (int k = 0; k < VEC_ROWS; ++k) {
    const int i = blockIdx.x * VEC_TILE + k * VEC_THREADS + threadIdx.x;
    rows[k] = i;
    zv[k] = i < n ? zc[i] : 0.0;
    self = fma(zv[k], zv[k], self);
  }
  double* pc = partials + (long long)c * nb * width;
  __shared__ double s_self[VEC_THREADS / 32];
  self = warp_sum(self);
  if ((threadIdx.x & 31) == 0) s_self[threadIdx.x >> 5] = self;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < VEC_THREADS / 32; ++w) t += s_self[w];
    pc[(long long)blockIdx.x * width] = t;
  }
  block_dots<VEC_ROWS>(zv, rows, n, V + (long long)c * ldcol, ldv, nv, pc, width, 1, nullptr);
}

int launch_dots_batch(int n, const double* z, long long ldz, const double* V, long long ldv, long long ldcol,
                      int nv, const ColList& cols, double* partials, int width, int* nb_out, cudaStream_t st) {
  const int nb = ceil_div(n, VEC_TILE);
  if (nb_out) *nb_out = nb;
  if (n == 0 || cols.n == 0) return HG_OK;
  k_dots_batch<<<dim3(nb, cols.n), VEC_THREADS, 0, st>>>(n, z, ldz, V, ldv, ldcol, nv, cols, partials, width, nb);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void __launch_bounds__(256) k_reduce_batch(const double* __restrict__ partials, int nb, int width,
                                                      ColList cols, double* __restrict__ out, long long ow) {
  __shared__ double s[256];
  const int k = blockIdx.x, c = cols.c[blockIdx.y];
  const double* pc = partials + (long long)c * nb * width;
  double t = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) t += pc[(long long)b * width + k];
  s[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[(long long)c * ow + k] = s[0];
}

int launch_reduce_batch(const double* partials, int nb, int width, int cnt, const ColList& cols, double* out,
                        long long ow, cudaStream_t st) {
  if (cnt == 0 || cols.n == 0) return HG_OK;
  k_reduce_batch<<<dim3(cnt, cols.n), 256, 0, st>>>(partials, nb, width, cols, out, ow);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void __launch_bounds__(VEC_THREADS) k_axpy_batch(int n, double* __restrict__ w, long long ldw,
                                                            const double* __restrict__ V, long long ldv,
                                                            long long ldcol, int nv, const double* __restrict__ coef,
                                                            long long ldcoef, int mode, ColList cols) {
  __shared__ double s_coef[MAX_NV];
  const int c = cols.c[blockIdx.y];
  const double* cc = coef + (long long)c * ldcoef;
  for (int i = threadIdx.x; i < nv; i += VEC_THREADS) s_coef[i] = cc[i];
  __syncthreads();
  double* wc = w + (long long)c * ldw;
  const double* Vc = V + (long long)c * ldcol;
#pragma unroll
  for (int k = 0; k < VEC_ROWS; ++k) {
    const int d = blockIdx.x * VEC_TILE + k * VEC_THREADS + threadIdx.x;
    if (d >= n) continue;
    double acc = mode ? wc[d] : 0.0;
    if (mode == 1) {
      for (int i = 0; i < nv; ++i) acc = fma(-s_coef[i], __ldg(Vc + (long long)i * ldv + d), acc);
    } else {
      for (int i = 0; i < nv; ++i) acc = fma(s_coef[i], __ldg(Vc + (long long)i * ldv + d), acc);
    }
    wc[d] = acc;
  }
}

int launch_axpy_batch(int n, double* w, long long ldw, const double* V, long long ldv, long long ldcol, int nv,
                      const double* coef, long long ldcoef, int mode, const ColList& cols, cudaStream_t st) {
  if (n == 0 || cols.n == 0) return HG_OK;
  if (nv > MAX_NV) {
    set_error("axpy_batch: more than 1024 basis vectors");
    return HG_ERR_UNSUPPORTED;
  }
  k_axpy_batch<<<dim3(ceil_div(n, VEC_TILE), cols.n), VEC_THREADS, 0, st>>>(n, w, ldw, V, ldv, ldcol, nv, coef,
                                                                             ldcoef, mode, cols);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void k_scale_batch(int n, const double* __restrict__ w, const double* __restrict__ ww, long long ldw,
                              double* __restrict__ V, double* __restrict__ WV, long long ldcol, ColList cols) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const int c = cols.c[blockIdx.y];
  const double h = cols.s[blockIdx.y];
  V[(long long)c * ldcol + d] = w[(long long)c * ldw + d] / h;
  if (WV) WV[(long long)c * ldcol + d] = ww[(long long)c * ldw + d] / h;
}

int launch_scale_batch(int n, const double* w, const double* ww, long long ldw, double* V, double* WV,
                       long long ldcol, const ColList& cols, cudaStream_t st) {
  if (n == 0 || cols.n == 0) return HG_OK;
  k_scale_batch<<<dim3(ceil_div(n, 256), cols.n), 256, 0, st>>>(n, w, ww, ldw, V, WV, ldcol, cols);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void k_fill_batch(int n, double* __restrict__ y, long long ldy, ColList cols) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) y[(long long)cols.c[blockIdx.y] * ldy + d] = 0.0;
}

int launch_fill_batch(int n, double* y, long long ldy, const ColList& cols, cudaStream_t st) {
  if (n == 0 || cols.n == 0) return HG_OK;
  k_fill_batch<<<dim3(ceil_div(n, 256), cols.n), 256, 0, st>>>(n, y, ldy, cols);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// ------------------------------------------------------------------ scratch
int multi_prepare(HgPrecond* P) {
  if (P->multi_ready) return HG_OK;
  auto alloc = [&](double** p, size_t count) -> int {
    if (count == 0) count = 1;
    HG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), sizeof(double) * count));
    P->device_bytes += (long long)(sizeof(double) * count);
    return HG_OK;
  };
  HG_TRY(alloc(&P->d_xsm, (size_t)MR * P->xs_len));
  HG_CUDA_TRY(cudaMemset(P->d_xsm, 0, sizeof(double) * MR * P->xs_len));  // pseudo-block slots are read before written
  HG_TRY(alloc(&P->d_tmpm, (size_t)MR * P->n));
  if (P->m > 0) {
    HG_TRY(alloc(&P->d_zsm, (size_t)MR * P->zs_len));
    HG_TRY(alloc(&P->d_cpartm, (size_t)MR * P->part_len));
    HG_TRY(alloc(&P->d_ym, (size_t)MR * P->m));
    HG_TRY(alloc(&P->d_b0m_x, (size_t)2 * P->b0_K * BP * MR * 2));  // (value, tag) pairs
    HG_CUDA_TRY(cudaMemset(P->d_b0m_x, 0, sizeof(double) * 2 * P->b0_K * BP * MR * 2));  // tag 0 = never
    if (P->d_b0_inv) {
      HG_TRY(alloc(&P->d_cm, (size_t)MR * P->b0_mp));
      HG_CUDA_TRY(cudaMemset(P->d_cm, 0, sizeof(double) * MR * P->b0_mp));  // rows beyond m stay zero
      HG_TRY(alloc(&P->d_ypart, (size_t)B0_KSPLIT * MR * P->b0_mp));
    }
    // packed copies of Z for the batched contractions (HG_Z_PACKED=0: the row-major kernels)
    const char* zenv = getenv("HG_Z_PACKED");
    if (!(zenv && zenv[0] == '0') && P->n_zt_items > 0) {
      std::vector<long long> zoff(P->n_cblk), toff(P->n_cblk);
      std::vector<ZyItem> zit;
      long long zlen = 0, tlen = 0;
      for (int b = 0; b < P->n_cblk; ++b) {
        const CblkDesc& d = P->h_cblk[b];
        const long long KB = (d.m + 7) / 8, MT = (d.n + 7) / 8;
        zoff[b] = zlen;
        toff[b] = tlen;
        zlen += MT * KB * 64;
        tlen += (long long)d.nchunk * KB * 32 * 64;
        if (d.m > 0)
          for (int t = 0; t < (MT + 1) / 2; ++t)
            zit.push_back(ZyItem{zoff[b] / 2 + (long long)t * 2 * KB * 32, d.idx_off + (long long)t * 16, d.col0, d.m,
                                 std::min(16, d.n - t * 16), 0});
      }
      HG_TRY(alloc(&P->d_zypk, (size_t)std::max(zlen, 1LL)));
      HG_TRY(alloc(&P->d_ztpk, (size_t)std::max(tlen, 1LL)));
      HG_CUDA_TRY(cudaMalloc(&P->d_zypk_off, sizeof(long long) * P->n_cblk));
      HG_CUDA_TRY(cudaMalloc(&P->d_ztpk_off, sizeof(long long) * P->n_cblk));
      HG_CUDA_TRY(cudaMemcpy(P->d_zypk_off, zoff.data(), sizeof(long long) * P->n_cblk, cudaMemcpyHostToDevice));
      HG_CUDA_TRY(cudaMemcpy(P->d_ztpk_off, toff.data(), sizeof(long long) * P->n_cblk, cudaMemcpyHostToDevice));
      HG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&P->d_zy_items), sizeof(ZyItem) * std::max<size_t>(zit.size(), 1)));
      HG_CUDA_TRY(cudaMemcpy(P->d_zy_items, zit.data(), sizeof(ZyItem) * zit.size(), cudaMemcpyHostToDevice));
      P->n_zy_items = (int)zit.size();
      k_zpack_zy<<<dim3(64, P->n_cblk), 256>>>(P->d_cblk, P->d_zypk_off, P->d_z, reinterpret_cast<double2*>(P->d_zypk));
      HG_LAUNCH_CHECK();
      k_zpack_zt<<<dim3(64, P->n_cblk), 256>>>(P->d_cblk, P->d_ztpk_off, P->d_z, reinterpret_cast<double2*>(P->d_ztpk));
      HG_LAUNCH_CHECK();
      HG_CUDA_TRY(cudaDeviceSynchronize());
    }
    HG_CUDA_TRY(cudaMalloc(&P->d_blkm_done, sizeof(unsigned long long) * P->n_cblk));
    HG_CUDA_TRY(cudaMemset(P->d_blkm_done, 0, sizeof(unsigned long long) * P->n_cblk));
  }
  HG_CUDA_TRY(cudaDeviceSynchronize());
  P->multi_ready = true;
  return HG_OK;
}

int preload_multi() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_spmm<true>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_spmm<false>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_zt_multi));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_zy_multi));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_zt_multi_pk));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_zy_multi_pk));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_zpack_zy));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_zpack_zt));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_multi));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_assemble_multi));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_dots_batch));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_reduce_batch));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_axpy_batch));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_scale_batch));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_fill_batch));
  return HG_OK;
}

}  // namespace hg

// ------------------------------------------------------------------ DCGS2 Arnoldi kernels
namespace hg {

// Butterfly reduce-scatter of 8 per-lane values over a warp (9 shuffles
// instead of 8 x 5): afterwards lane L holds the warp total of value
// ((L>>4)&1)*4 + ((L>>3)&1)*2 + ((L>>2)&1).
__device__ __forceinline__ double warp_reduce8(double (&v)[8], int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool hi = lane & 16;
    const double send = hi ? v[i] : v[4 + i];
    const double keep = hi ? v[4 + i] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool hi = lane & 8;
    const double send = hi ? v[i] : v[2 + i];
    const double keep = hi ? v[2 + i] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 8);
  }
  {
    const bool hi = lane & 4;
    const double send = hi ? v[0] : v[1];
    const double keep = hi ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(FULL, send, 4);
  }
  double t = v[0] + __shfl_xor_sync(FULL, v[0], 2);
  return t + __shfl_xor_sync(FULL, t, 1);
}

constexpr int D2_CH = 4;  // basis vectors per chunk: 8 sums (4 . a, 4 . u) per lane

// Column c: dots of its basis V_c[0..nv) with a_c and u_c, each V_i read once.
// A thread owns VEC_ROWS rows; a chunk of 4 vectors issues all 16 loads
// before any reduction; per-warp totals by warp_reduce8, per-block totals
// in a fixed order through a double-buffered smem slot (one barrier per
// chunk).  partials value-major: [(c * width + k) * nb + block], k < 2 nv
// (k < nv: V_k . a, nv + k: V_k . u).
__global__ void __launch_bounds__(VEC_THREADS, 3) k_dots2_batch(int n, const double* __restrict__ A, long long lda,
                                                             const double* __restrict__ U, long long ldu,
                                                             const double* __restrict__ V, long long ldv,
                                                             long long ldcol, int nv, ColList cols,
                                                             double* __restrict__ partials, int width, int nb,
                                                             int vsplit) {
  __shared__ double s_p[2][VEC_THREADS / 32][2 * D2_CH];
  const int c = cols.c[blockIdx.y / vsplit];
  // basis vectors [ia, ib) of this block (vsplit blocks share a row tile when
  // the grid would otherwise be a few waves of one column)
  const int per = ((nv + vsplit - 1) / vsplit + D2_CH - 1) / D2_CH * D2_CH;
  const int ia = (blockIdx.y % vsplit) * per, ib = min(nv, ia + per);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double av[VEC_ROWS], uv[VEC_ROWS];
  int rows[VEC_ROWS];
#pragma unroll
  for (int k = 0; k < VEC_ROWS; ++k) {
    const int i = blockIdx.x * VEC_TILE + k * VEC_THREADS + threadIdx.x;
    rows[k] = i < n ? i : -1;
    av[k] = i < n ? A[(long long)c * lda + i] : 0.0;
    uv[k] = i < n ? U[(long long)c * ldu + i] : 0.0;
  }
  const double* Vc = V + (long long)c * ldcol;
  double* pc = partials + (long long)c * width * nb;
  const int my = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  int buf = 0;
  for (int i0 = ia; i0 < ib; i0 += D2_CH, buf ^= 1) {
    double x[D2_CH][VEC_ROWS];
#pragma unroll
    for (int t = 0; t < D2_CH; ++t)
#pragma unroll
      for (int k = 0; k < VEC_ROWS; ++k)
        x[t][k] = (i0 + t < ib && rows[k] >= 0) ? __ldg(Vc + (long long)(i0 + t) * ldv + rows[k]) : 0.0;
    double v[2 * D2_CH];
#pragma unroll
    for (int t = 0; t < D2_CH; ++t) {
      double pa = 0.0, pu = 0.0;
#pragma unroll
      for (int k = 0; k < VEC_ROWS; ++k) {
        pa = fma(x[t][k], av[k], pa);
        pu = fma(x[t][k], uv[k], pu);
      }
      v[t] = pa;
      v[D2_CH + t] = pu;
    }
    const double tot = warp_reduce8(v, lane);
    if (!(lane & 3)) s_p[buf][warp][my] = tot;
    __syncthreads();
    if (threadIdx.x < 2 * D2_CH) {
      const int t = threadIdx.x % D2_CH, which = threadIdx.x / D2_CH;
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < VEC_THREADS / 32; ++w) sum += s_p[buf][w][threadIdx.x];
      if (i0 + t < ib) pc[(long long)(which * nv + i0 + t) * nb + blockIdx.x] = sum;
    }
  }
}

// out[c * ow + k] = sum_b partials[(c * width + k) * nb + b] (contiguous, fixed order)
__global__ void __launch_bounds__(256) k_reduce_vm(const double* __restrict__ partials, int nb, int width,
                                                   ColList cols, double* __restrict__ out, long long ow) {
  __shared__ double s[256];
  const int k = blockIdx.x, c = cols.c[blockIdx.y];
  const double* p = partials + ((long long)c * width + k) * nb;
  double t = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) t += p[b];
  s[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[(long long)c * ow + k] = s[0];
}

int launch_dots2_batch(int n, const double* A, long long lda, const double* U, long long ldu, const double* V,
                       long long ldv, long long ldcol, int nv, const ColList& cols, double* partials, double* out,
                       long long ow, cudaStream_t st) {
  const int nb = ceil_div(n, VEC_TILE);
  if (n == 0 || cols.n == 0) return HG_OK;
  // few columns: split the basis over blocks so the grid is many waves deep
  const int vsplit = (cols.n * nb < 4096 && nv >= 4 * D2_CH) ? 2 : 1;
  k_dots2_batch<<<dim3(nb, cols.n * vsplit), VEC_THREADS, 0, st>>>(n, A, lda, U, ldu, V, ldv, ldcol, nv, cols,
                                                                   partials, 2 * nv, nb, vsplit);
  HG_LAUNCH_CHECK();
  k_reduce_vm<<<dim3(2 * nv, cols.n), 256, 0, st>>>(partials, nb, 2 * nv, cols, out, ow);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// Delayed reorthogonalisation + projection in one read of V_c[0..j):
//   q  = (V_c[j] - sum_{i<j} s_i V_c[i]) * rinv          (q_j re-orthogonalised)
//   w  = w * rinv - sum_{i<j} c_i V_c[i] - c_j q          (w projected)
// coef row of column c: [rinv, s_0..s_{j-1}, c_0..c_j].
__global__ void __launch_bounds__(VEC_THREADS, 4) k_dcgs2_update(int n, double* __restrict__ V, long long ldv,
                                                              long long ldcol, int j, double* __restrict__ w,
                                                              long long ldw, const double* __restrict__ coef,
                                                              long long ldcoef, ColList cols) {
  __shared__ double s_c[2 * MAX_NV + 2];
  const int c = cols.c[blockIdx.y];
  const double* cc = coef + (long long)c * ldcoef;
  for (int i = threadIdx.x; i < 2 * j + 2; i += VEC_THREADS) s_c[i] = cc[i];
  __syncthreads();
  const double rinv = s_c[0];
  const double* sv = s_c + 1;
  const double* cv = s_c + 1 + j;
  double* Vc = V + (long long)c * ldcol;
  double* wc = w + (long long)c * ldw;
  double aq[VEC_ROWS], aw[VEC_ROWS];
  int rows[VEC_ROWS];
#pragma unroll
  for (int k = 0; k < VEC_ROWS; ++k) {
    const int d = blockIdx.x * VEC_TILE + k * VEC_THREADS + threadIdx.x;
    rows[k] = d < n ? d : -1;
    aq[k] = d < n ? Vc[(long long)j * ldv + d] : 0.0;
    aw[k] = d < n ? wc[d] * rinv : 0.0;
  }
  // chunks of 4 vectors: all 16 loads of a chunk issued before its FMAs;
  // per row the sum stays sequential in i (fixed summation order)
  int i = 0;
  for (; i + 4 <= j; i += 4) {
    double x[4][VEC_ROWS];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int k = 0; k < VEC_ROWS; ++k)
        x[t][k] = rows[k] >= 0 ? __ldg(Vc + (long long)(i + t) * ldv + rows[k]) : 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const double si = sv[i + t], ci = cv[i + t];
#pragma unroll
      for (int k = 0; k < VEC_ROWS; ++k) {
        aq[k] = fma(-si, x[t][k], aq[k]);
        aw[k] = fma(-ci, x[t][k], aw[k]);
      }
    }
  }
  for (; i < j; ++i) {
    const double* vi = Vc + (long long)i * ldv;
    const double si = sv[i], ci = cv[i];
#pragma unroll
    for (int k = 0; k < VEC_ROWS; ++k) {
      const double x = rows[k] >= 0 ? __ldg(vi + rows[k]) : 0.0;
      aq[k] = fma(-si, x, aq[k]);
      aw[k] = fma(-ci, x, aw[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < VEC_ROWS; ++k) {
    if (rows[k] < 0) continue;
    const double qn = aq[k] * rinv;
    Vc[(long long)j * ldv + rows[k]] = qn;
    wc[rows[k]] = fma(-cv[j], qn, aw[k]);
  }
}

int launch_dcgs2_update(int n, double* V, long long ldv, long long ldcol, int j, double* w, long long ldw,
                        const double* coef, long long ldcoef, const ColList& cols, cudaStream_t st) {
  if (n == 0 || cols.n == 0) return HG_OK;
  if (j + 1 > MAX_NV) {
    set_error("dcgs2 update: more than 1024 basis vectors");
    return HG_ERR_UNSUPPORTED;
  }
  k_dcgs2_update<<<dim3(ceil_div(n, VEC_TILE), cols.n), VEC_THREADS, 0, st>>>(n, V, ldv, ldcol, j, w, ldw, coef,
                                                                               ldcoef, cols);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// V_c = w_c / h_c and (WQ) Wq_c = ww_c / h_c with h_c = sqrt(max(nrm2[c], 0))
// read on the device (no host round trip before the next operator apply).
__global__ void k_scale_dev_batch(int n, const double* __restrict__ w, const double* __restrict__ ww, long long ldw,
                                  double* __restrict__ V, long long ldcol, double* __restrict__ Wq,
                                  const double* __restrict__ nrm2, ColList cols) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const int c = cols.c[blockIdx.y];
  const double h = sqrt(fmax(nrm2[c], 0.0));
  V[(long long)c * ldcol + d] = w[(long long)c * ldw + d] / h;
  if (Wq) Wq[(long long)c * ldw + d] = ww[(long long)c * ldw + d] / h;
}

int launch_scale_dev_batch(int n, const double* w, const double* ww, long long ldw, double* V, long long ldcol,
                           double* Wq, const double* nrm2, const ColList& cols, cudaStream_t st) {
  if (n == 0 || cols.n == 0) return HG_OK;
  k_scale_dev_batch<<<dim3(ceil_div(n, 256), cols.n), 256, 0, st>>>(n, w, ww, ldw, V, ldcol, Wq, nrm2, cols);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

int preload_dcgs2() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_dots2_batch));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_reduce_vm));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_dcgs2_update));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_scale_dev_batch));
  return HG_OK;
}

}  // namespace hg

namespace hg {
__global__ void k_add(int n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) out[d] = a[d] + b[d];
}

int launch_add(int n, const double* a, const double* b, double* out, cudaStream_t st) {
  if (n == 0) return HG_OK;
  k_add<<<ceil_div(n, 256), 256, 0, st>>>(n, a, b, out);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

int preload_add() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_add));
  return HG_OK;
}
}  // namespace hg
