// Split local blocks (include/helmgpu.h "Split local blocks"): the separator
// and spike stages that follow the chunk solves of a local solve
// (ls.lu.solve, schwarz.py:58-60 — the same operator, eliminated in
// nested-dissection order so that one 18k-row band chain becomes P chains of
// n / P rows on P CTAs):
//   k_sep_solve    x_S = Sigma^{-1} (r_S - F y): grid (split, 64-row group of
//                  Sigma^{-1}); every CTA forms t = r_S - F y for its split
//                  (a few nonzeros per row) in shared memory, then its rows
//                  of the dense product; up to 16 columns
//   k_spike        x_p -= W_p x_S for one right-hand side: a warp owns an
//                  8-row tile of a chunk and streams its packed spike rows
//   k_spike_multi  the same for a batch on DMMA (the packed blocks are the
//                  m8n8k4 A fragments, as for B0^{-1} in hg_b0d.cu)
// Both read W once per apply: HBM streams, fully parallel over all chunks.
#include <algorithm>
#include <vector>

#include "hg_internal.cuh"

namespace hg {

namespace {
constexpr int MRS = HG_MAX_RHS;
constexpr int SEP_ROWS = 64;   // rows of Sigma^{-1} per CTA (8 per warp)
constexpr int TS = MRS + 1;    // shared row stride of t (conflict-free column reads)

__device__ __forceinline__ void dmma_s(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

template <typename T>
int up(T** dptr, const T* host, size_t count, long long* bytes) {
  *dptr = nullptr;
  if (count == 0) return HG_OK;
  HG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dptr), sizeof(T) * count));
  if (host) HG_CUDA_TRY(cudaMemcpy(*dptr, host, sizeof(T) * count, cudaMemcpyDefault));
  if (bytes) *bytes += (long long)(sizeof(T) * count);
  return HG_OK;
}
}  // namespace

// R: right-hand sides (column c at R + c ldr, global dof numbering); xs: local
// solution scratch (column c at xs + c xs_len); xsep: [separator row][16]
// compact copy of x_S for the spike kernels.
template <int NC>
__global__ void __launch_bounds__(256) k_sep_solve(const SplitDesc* __restrict__ splits,
                                                   const long long* __restrict__ fptr,
                                                   const long long* __restrict__ fpos,
                                                   const double* __restrict__ fval,
                                                   const double* __restrict__ sinv_all,
                                                   const int* __restrict__ idx, const double* __restrict__ R,
                                                   long long ldr, double* __restrict__ xs, long long xs_len,
                                                   int nrhs, double* __restrict__ xsep) {
  extern __shared__ double s_t[];  // [nS][NC + 1]
  const SplitDesc d = splits[blockIdx.x];
  const int nS = d.ns;
  const int row0 = blockIdx.y * SEP_ROWS;
  if (row0 >= nS) return;
  constexpr int ST = NC + 1;
  for (int e = threadIdx.x; e < nS * NC; e += blockDim.x) {
    const int k = e / NC, c = e % NC;
    double v = 0.0;
    if (c < nrhs) {
      v = __ldg(R + (long long)c * ldr + __ldg(idx + d.sep_pos + k));
      const double* y = xs + (long long)c * xs_len;
      for (long long j = fptr[d.row0 + k]; j < fptr[d.row0 + k + 1]; ++j) v = fma(-__ldg(fval + j), y[__ldg(fpos + j)], v);
    }
    s_t[k * ST + c] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* sinv = sinv_all + d.sinv_off;
  for (int rr = warp; rr < SEP_ROWS; rr += 8) {
    const int row = row0 + rr;
    if (row >= nS) break;
    const double* a = sinv + (size_t)row * nS;
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    for (int k = lane; k < nS; k += 32) {
      const double av = __ldg(a + k);
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] = fma(av, s_t[k * ST + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = warp_sum(acc[c]);
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (c < nrhs) xs[(long long)c * xs_len + d.sep_pos + row] = acc[c];
        xsep[(size_t)(d.row0 + row) * MRS + c] = c < nrhs ? acc[c] : 0.0;
      }
    }
  }
}

// one right-hand side: item = (spike, 8-row tile); two tiles per warp iteration
__global__ void __launch_bounds__(256) k_spike(const int2* __restrict__ items, int nitems,
                                               const SpikeDesc* __restrict__ spikes,
                                               const double2* __restrict__ data, const double* __restrict__ xsep,
                                               double* __restrict__ xs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  const int it = blockIdx.x * 8 + warp;
  if (it >= nitems) return;
  const int2 item = items[it];
  const SpikeDesc d = spikes[item.x];
  const int KB = d.w >> 3;
  const double2* ap = data + (d.off >> 1) + ((size_t)item.y * KB) * 32 + lane;
  const double* xv = xsep + (size_t)(d.row0 + d.col0) * MRS;  // column 0 of the compact x_S
  double s0 = 0.0, s1 = 0.0;
  int kb = 0;
  for (; kb + 2 <= KB; kb += 2) {
    const double2 a0 = __ldcs(ap), a1 = __ldcs(ap + 32);
    const int k0 = kb * 8 + q;
    s0 = fma(a0.x, k0 < d.wtrue ? __ldg(xv + (size_t)k0 * MRS) : 0.0, s0);
    s0 = fma(a0.y, k0 + 4 < d.wtrue ? __ldg(xv + (size_t)(k0 + 4) * MRS) : 0.0, s0);
    s1 = fma(a1.x, k0 + 8 < d.wtrue ? __ldg(xv + (size_t)(k0 + 8) * MRS) : 0.0, s1);
    s1 = fma(a1.y, k0 + 12 < d.wtrue ? __ldg(xv + (size_t)(k0 + 12) * MRS) : 0.0, s1);
    ap += 64;
  }
  for (; kb < KB; ++kb) {
    const double2 a0 = __ldcs(ap);
    const int k0 = kb * 8 + q;
    s0 = fma(a0.x, k0 < d.wtrue ? __ldg(xv + (size_t)k0 * MRS) : 0.0, s0);
    s0 = fma(a0.y, k0 + 4 < d.wtrue ? __ldg(xv + (size_t)(k0 + 4) * MRS) : 0.0, s0);
    ap += 32;
  }
  double s = s0 + s1;
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  const int row = item.y * 8 + g;
  if (q == 0 && row < d.n) xs[d.pos + row] -= s;
}

// batch: item = (spike, pair of 8-row tiles); 4 DMMA accumulators (2 tiles x 16 columns)
__global__ void __launch_bounds__(256) k_spike_multi(const int2* __restrict__ items, int nitems,
                                                     const SpikeDesc* __restrict__ spikes,
                                                     const double2* __restrict__ data,
                                                     const double* __restrict__ xsep, double* __restrict__ xs,
                                                     long long xs_len, int nrhs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, g = lane >> 2;
  const int it = blockIdx.x * 8 + warp;
  if (it >= nitems) return;
  const int2 item = items[it];
  const SpikeDesc d = spikes[item.x];
  const int KB = d.w >> 3;
  const int MT = (d.n + 7) >> 3;
  const int mt0 = item.y * 2;
  const bool two = mt0 + 1 < MT;
  const double2* a0p = data + (d.off >> 1) + ((size_t)mt0 * KB) * 32 + lane;
  const double2* a1p = two ? a0p + (size_t)KB * 32 : a0p;
  const double* cp = xsep + ((size_t)(d.row0 + d.col0) + q) * MRS + g;
  double acc[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
#pragma unroll 2
  for (int kb = 0; kb < KB; ++kb) {
    const double2 a0 = __ldcs(a0p), a1 = __ldcs(a1p);
    const int k0 = kb * 8 + q;
    const bool v0 = k0 < d.wtrue, v1 = k0 + 4 < d.wtrue;  // padded columns: W is zero there, x_S must not be read
    const double* cu = cp + (size_t)kb * 8 * MRS;
    const double b00 = v0 ? __ldg(cu) : 0.0, b01 = v0 ? __ldg(cu + 8) : 0.0;
    const double b10 = v1 ? __ldg(cu + 4 * MRS) : 0.0, b11 = v1 ? __ldg(cu + 4 * MRS + 8) : 0.0;
    dmma_s(acc[0][0], a0.x, b00);
    dmma_s(acc[0][1], a0.x, b01);
    dmma_s(acc[1][0], a1.x, b00);
    dmma_s(acc[1][1], a1.x, b01);
    dmma_s(acc[0][0], a0.y, b10);
    dmma_s(acc[0][1], a0.y, b11);
    dmma_s(acc[1][0], a1.y, b10);
    dmma_s(acc[1][1], a1.y, b11);
    a0p += 32;
    a1p += 32;
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int row = (mt0 + t) * 8 + g;
    if ((t == 1 && !two) || row >= d.n) continue;
    double* x = xs + d.pos + row;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * h + 2 * q + e;
        if (c < nrhs) x[(long long)c * xs_len] -= acc[t][h][e];
      }
  }
}

// ------------------------------------------------------------------ host side
int split_upload(HgPrecond* P, const HgPrecondDesc* D) {
  P->n_split = 0;
  if (D->n_split <= 0) return HG_OK;
  if (!D->split_blk || !D->split_row_off || !D->split_f_indptr || !D->split_sinv_off || !D->split_sinv ||
      (D->n_spike > 0 && (!D->spike_blk || !D->spike_split || !D->spike_col0 || !D->spike_w || !D->spike_off ||
                          !D->spike_data))) {
    set_error("hg_precond_create: incomplete split-block description");
    return HG_ERR_ARG;
  }
  long long* bytes = &P->device_bytes;
  std::vector<SplitDesc> sd(D->n_split);
  int ns_max = 0;
  for (int s = 0; s < D->n_split; ++s) {
    const int b = D->split_blk[s];
    if (b < 0 || b >= D->n_local || D->local_n[b] != 0) {
      set_error("hg_precond_create: split " + std::to_string(s) + " does not name a separator pseudo block");
      return HG_ERR_ARG;
    }
    SplitDesc& d = sd[s];
    d.row0 = D->split_row_off[s];
    d.ns = (int)(D->split_row_off[s + 1] - D->split_row_off[s]);
    d.sep_pos = D->local_idx_off[b];
    d.sinv_off = D->split_sinv_off[s];
    if (d.ns != D->local_idx_off[b + 1] - D->local_idx_off[b] || d.ns <= 0) {
      set_error("hg_precond_create: separator rows of split " + std::to_string(s) + " do not match its pseudo block");
      return HG_ERR_ARG;
    }
    ns_max = std::max(ns_max, d.ns);
  }
  const long long nrows = D->split_row_off[D->n_split];
  const long long fnnz = D->split_f_indptr[nrows];
  for (long long j = 0; j < fnnz; ++j) {
    if (D->split_f_pos[j] < 0 || D->split_f_pos[j] >= P->xs_len) {
      set_error("hg_precond_create: split F position out of range");
      return HG_ERR_ARG;
    }
  }
  std::vector<SpikeDesc> kd(D->n_spike);
  std::vector<int2> items1, items2;
  for (int i = 0; i < D->n_spike; ++i) {
    const int b = D->spike_blk[i], s = D->spike_split[i];
    if (b < 0 || b >= D->n_local || s < 0 || s >= D->n_split || (D->spike_w[i] & 7) || D->spike_w[i] <= 0 ||
        (D->spike_off[i] & 1) || D->spike_col0[i] < 0 || D->spike_col0[i] >= sd[s].ns) {
      set_error("hg_precond_create: inconsistent spike " + std::to_string(i));
      return HG_ERR_ARG;
    }
    SpikeDesc& d = kd[i];
    d.n = D->local_n[b];
    d.w = D->spike_w[i];
    d.wtrue = std::min(d.w, sd[s].ns - D->spike_col0[i]);
    d.col0 = D->spike_col0[i];
    d.row0 = sd[s].row0;
    d.pos = D->local_idx_off[b];
    d.off = D->spike_off[i];
    const int mt = (d.n + 7) / 8;
    if (d.off + (long long)mt * 8 * d.w > D->spike_len) {
      set_error("hg_precond_create: spike " + std::to_string(i) + " exceeds spike_data");
      return HG_ERR_ARG;
    }
    for (int t = 0; t < mt; ++t) items1.push_back(make_int2(i, t));
    for (int t = 0; t < (mt + 1) / 2; ++t) items2.push_back(make_int2(i, t));
  }
  HG_TRY(up(&P->d_split, sd.data(), sd.size(), bytes));
  HG_TRY(up(&P->d_split_fptr, reinterpret_cast<const long long*>(D->split_f_indptr), (size_t)nrows + 1, bytes));
  HG_TRY(up(&P->d_split_fpos, reinterpret_cast<const long long*>(D->split_f_pos), (size_t)fnnz, bytes));
  HG_TRY(up(&P->d_split_fval, D->split_f_val, (size_t)fnnz, bytes));
  HG_TRY(up(&P->d_split_sinv, D->split_sinv, (size_t)D->split_sinv_len, bytes));
  HG_TRY(up(&P->d_spike, kd.data(), kd.size(), bytes));
  HG_TRY(up(&P->d_spike_data, D->spike_data, (size_t)D->spike_len, bytes));
  HG_TRY(up(&P->d_spike_items1, items1.data(), items1.size(), bytes));
  HG_TRY(up(&P->d_spike_items2, items2.data(), items2.size(), bytes));
  HG_TRY(up<double>(&P->d_xsep, nullptr, (size_t)nrows * MRS, bytes));
  HG_CUDA_TRY(cudaMemset(P->d_xsep, 0, sizeof(double) * nrows * MRS));
  P->n_split = D->n_split;
  P->split_ns_max = ns_max;
  P->n_spike_items1 = (int)items1.size();
  P->n_spike_items2 = (int)items2.size();
  return HG_OK;
}

void split_release(HgPrecond* P) {
  auto rel = [](auto*& p) {
    if (p) cudaFree(p);
    p = nullptr;
  };
  rel(P->d_split);
  rel(P->d_split_fptr);
  rel(P->d_split_fpos);
  rel(P->d_split_fval);
  rel(P->d_split_sinv);
  rel(P->d_spike);
  rel(P->d_spike_data);
  rel(P->d_spike_items1);
  rel(P->d_spike_items2);
  rel(P->d_xsep);
}

// separator + spike stages after the chunk solves wrote xs (single: nrhs = 1, ldr unused)
int launch_split_stages(HgPrecond* P, const double* R, long long ldr, double* xs, long long xs_len, int nrhs,
                        cudaStream_t st) {
  if (P->n_split == 0) return HG_OK;
  const dim3 grid(P->n_split, ceil_div(P->split_ns_max, SEP_ROWS));
  if (nrhs == 1) {
    const size_t smem = sizeof(double) * (size_t)P->split_ns_max * 2;
    HG_TRY(ensure_func_attrs(reinterpret_cast<const void*>(k_sep_solve<1>), smem, false));
    k_sep_solve<1><<<grid, 256, smem, st>>>(P->d_split, P->d_split_fptr, P->d_split_fpos, P->d_split_fval,
                                            P->d_split_sinv, P->d_local_idx, R, ldr, xs, xs_len, 1, P->d_xsep);
    HG_LAUNCH_CHECK();
    if (P->n_spike_items1 > 0) {
      k_spike<<<ceil_div(P->n_spike_items1, 8), 256, 0, st>>>(P->d_spike_items1, P->n_spike_items1, P->d_spike,
                                                              reinterpret_cast<const double2*>(P->d_spike_data),
                                                              P->d_xsep, xs);
      HG_LAUNCH_CHECK();
    }
    return HG_OK;
  }
  const size_t smem = sizeof(double) * (size_t)P->split_ns_max * TS;
  HG_TRY(ensure_func_attrs(reinterpret_cast<const void*>(k_sep_solve<MRS>), smem, false));
  k_sep_solve<MRS><<<grid, 256, smem, st>>>(P->d_split, P->d_split_fptr, P->d_split_fpos, P->d_split_fval,
                                            P->d_split_sinv, P->d_local_idx, R, ldr, xs, xs_len, nrhs, P->d_xsep);
  HG_LAUNCH_CHECK();
  if (P->n_spike_items2 > 0) {
    k_spike_multi<<<ceil_div(P->n_spike_items2, 8), 256, 0, st>>>(
        P->d_spike_items2, P->n_spike_items2, P->d_spike, reinterpret_cast<const double2*>(P->d_spike_data),
        P->d_xsep, xs, xs_len, nrhs);
    HG_LAUNCH_CHECK();
  }
  return HG_OK;
}

int preload_split() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_sep_solve<1>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_sep_solve<MRS>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_spike));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_spike_multi));
  return HG_OK;
}

}  // namespace hg
