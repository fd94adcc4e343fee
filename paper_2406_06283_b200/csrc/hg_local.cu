// K2: one-level Schwarz local solves — gather, pivoted band forward
// substitution (L with row interchanges), band back substitution (U), all
// subdomains in one launch, one CTA per subdomain.
//
// Replaces `out[ls.idof] += ls.lu.solve(r[ls.idof])` (schwarz.py:58-60).
// The factors are LAPACK dgbtrf band factors of B[idof][:, idof] (partial
// pivoting); the solve follows dgbtrs: for j = 0..n-1 swap b_j
// with b_ipiv(j), then b_{j+t} -= l_{j+t,j} b_j (t = 1..kl); then for
// j = n-1..0: x_j = b_j / u_jj, b_{j-t} -= u_{j-t,j} x_j (t = 1..kv).
//
// Execution model (per CTA, 2 warps):
//  * warp 1 lane 0 is the producer: it streams the packed factor records
//    (16 steps per chunk) from HBM into a 4-stage shared-memory ring with
//    cp.async.bulk (TMA bulk copies) completing on mbarriers.  Factors are
//    read exactly once, in order, so the kernel is an HBM stream.
//  * warp 0 is the consumer: the active window of the right-hand side lives
//    in registers, 32 rows per register (R registers = 32R rows; row
//    j0 + 32r + lane sits in register r of `lane` during the round that
//    finalises rows j0..j0+31).  Each step broadcasts the pivot row with one
//    shuffle and every lane applies its multipliers from the staged record
//    (conflict-free 64-bit shared loads).  After 32 steps the finished rows
//    are stored with one coalesced store and the registers rotate; entering
//    rows are prefetched one round ahead.
//  * the backward sweep runs the same machinery on the reversed row order
//    (records are stored reversed), in place on the per-block scratch.
// The output of each block goes to its own scratch segment; overlapping
// contributions are summed later in a fixed order (hg_coarse.cu
// k_assemble), so there are no atomics and the result is deterministic.
#include "hg_internal.cuh"

namespace hg {

constexpr int LS_CH = 16;  // steps per staged chunk
constexpr int LS_NS = 4;   // ring stages
constexpr int LS_THREADS = 64;

template <int R, bool FWD>
__device__ __forceinline__ void ls_step(double (&v)[R], const double* __restrict__ rec, int s, int j,
                                        int j0, int lane, int kw) {
  double bj;
  if (FWD) {
    const int l = __double2int_rn(rec[0]);
    if (l != j) {  // row interchange (warp-uniform, rare)
      const int rl = (l - j0) >> 5, ll = (l - j0) & 31;
      const double a = __shfl_sync(FULL, v[0], s);
      double sel = v[0];
#pragma unroll
      for (int r = 1; r < R; ++r)
        if (r == rl) sel = v[r];
      const double b = __shfl_sync(FULL, sel, ll);
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r == rl && lane == ll) v[r] = a;
      if (lane == s) v[0] = b;
    }
    bj = __shfl_sync(FULL, v[0], s);
  } else {
    bj = __shfl_sync(FULL, v[0], s) * rec[0];
    if (lane == s) v[0] = bj;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int t = 32 * r + lane - s;
    if (t >= 1 && t <= kw) v[r] = fma(-rec[t], bj, v[r]);
  }
}

struct SweepCtx {
  const double* ring;  // smem ring base
  uint64_t* full;
  uint64_t* empty;
  int stage_stride;    // doubles per stage
};

// One sweep over n rows. FWD: input gathered from r[idx[row]], output y[row]
// into xs. !FWD: input y from xs in reverse, output x into xs in reverse.
template <int R, bool FWD>
__device__ void ls_sweep(const SweepCtx& cx, int& chunk, int n, int kw, int stride,
                         const int* __restrict__ idx, const double* __restrict__ rin,
                         double* __restrict__ xs) {
  const int lane = threadIdx.x & 31;
  auto load_in = [&](int row) -> double {
    if (row >= n) return 0.0;
    if (FWD) return __ldg(rin + __ldg(idx + row));
    return xs[n - 1 - row];
  };
  double v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = load_in(32 * r + lane);
  double pre = load_in(32 * R + lane);
  for (int j0 = 0; j0 < n; j0 += 32) {
    const double nxt = load_in(j0 + 32 * R + 32 + lane);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      if (j0 + half * LS_CH < n) {
        const int stage = chunk % LS_NS;
        mbar_wait(&cx.full[stage], (chunk / LS_NS) & 1);
        const double* rec0 = cx.ring + (size_t)stage * cx.stage_stride;
#pragma unroll
        for (int s2 = 0; s2 < LS_CH; ++s2) {
          const int s = half * LS_CH + s2;
          const int j = j0 + s;
          if (j < n) ls_step<R, FWD>(v, rec0 + s2 * stride, s, j, j0, lane, kw);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&cx.empty[stage]);
        ++chunk;
      }
    }
    const int row = j0 + lane;
    if (row < n) {
      if (FWD)
        xs[row] = v[0];
      else
        xs[n - 1 - row] = v[0];
    }
#pragma unroll
    for (int r = 0; r + 1 < R; ++r) v[r] = v[r + 1];
    v[R - 1] = pre;
    pre = nxt;
  }
}

template <int RF, int RB>
__global__ void __launch_bounds__(LS_THREADS) k_local_solve(const LocalDesc* __restrict__ descs,
                                                           const int* __restrict__ idx,
                                                           const double* __restrict__ fwd,
                                                           const double* __restrict__ bwd,
                                                           const double* __restrict__ r,
                                                           double* __restrict__ xs, int stage_stride) {
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[LS_NS], empty[LS_NS];
  const LocalDesc d = descs[blockIdx.x];
  if (threadIdx.x == 0) {
    for (int s = 0; s < LS_NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (d.n == 0) return;
  const int nc = (d.n + LS_CH - 1) / LS_CH;
  if (threadIdx.x >= 32) {
    if (threadIdx.x == 32) {  // producer
      for (int c = 0; c < 2 * nc; ++c) {
        const int stage = c % LS_NS;
        if (c >= LS_NS) mbar_wait(&empty[stage], ((c / LS_NS) - 1) & 1);
        const bool f = c < nc;
        const int cc = f ? c : c - nc;
        const int rows = min(LS_CH, d.n - cc * LS_CH);
        const int stride = f ? d.fstride : d.bstride;
        const double* src = (f ? fwd + d.fwd_off : bwd + d.bwd_off) + (long long)cc * LS_CH * stride;
        const uint32_t bytes = (uint32_t)rows * stride * 8u;
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(ring + (size_t)stage * stage_stride, src, bytes, &full[stage]);
      }
    }
    return;
  }
  SweepCtx cx{ring, full, empty, stage_stride};
  int chunk = 0;
  double* xsb = xs + d.idx_off;
  ls_sweep<RF, true>(cx, chunk, d.n, d.kl, d.fstride, idx + d.idx_off, r, xsb);
  __syncwarp();
  ls_sweep<RB, false>(cx, chunk, d.n, d.kv, d.bstride, nullptr, nullptr, xsb);
}

using LocalKernel = void (*)(const LocalDesc*, const int*, const double*, const double*, const double*,
                             double*, int);

template <int RF, int RB>
static LocalKernel pick2() {
  return k_local_solve<RF, RB>;
}

template <int RF>
static LocalKernel pick_rb(int rb) {
  switch (rb) {
    case 2: return pick2<RF, 2>();
    case 3: return pick2<RF, 3>();
    case 4: return pick2<RF, 4>();
    case 5: return pick2<RF, 5>();
    case 6: return pick2<RF, 6>();
    case 7: return pick2<RF, 7>();
    case 8: return pick2<RF, 8>();
    case 9: return pick2<RF, 9>();
    case 10: return pick2<RF, 10>();
    default: return nullptr;
  }
}

static LocalKernel pick(int rf, int rb) {
  switch (rf) {
    case 2: return pick_rb<2>(rb);
    case 3: return pick_rb<3>(rb);
    case 4: return pick_rb<4>(rb);
    case 5: return pick_rb<5>(rb);
    case 6: return pick_rb<6>(rb);
    default: return nullptr;
  }
}

static int launch_local_grid(HgPrecond* P, const LocalDesc* descs, int nblocks, const double* r,
                             cudaStream_t st) {
  LocalKernel k = pick(P->rf, P->rb);
  if (!k) {
    set_error("local band solve: bandwidth beyond the compiled register tiles (kl <= 160, kv <= 288)");
    return HG_ERR_UNSUPPORTED;
  }
  const int stage_stride = LS_CH * (P->max_fstride > P->max_bstride ? P->max_fstride : P->max_bstride);
  const size_t smem = (size_t)LS_NS * stage_stride * sizeof(double);
  static size_t configured[7][11] = {};
  if (configured[P->rf][P->rb] < smem) {
    HG_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[P->rf][P->rb] = smem;
  }
  k<<<nblocks, LS_THREADS, smem, st>>>(descs, P->d_local_idx, P->d_fwd, P->d_bwd, r, P->d_xs, stage_stride);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

int launch_local_solve(HgPrecond* P, const double* r, cudaStream_t st) {
  if (P->n_local == 0) return HG_OK;
  return launch_local_grid(P, P->d_local, P->n_local, r, st);
}

__global__ void k_scatter_local(int n, const int* __restrict__ idx, const double* __restrict__ src,
                                double* __restrict__ dst) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[idx[k]] = src[k];
}

int launch_local_solve_single(HgPrecond* P, int s, const double* r_local, double* x_local,
                              cudaStream_t st) {
  const LocalDesc& d = P->h_local[s];
  if (d.n == 0) return HG_OK;
  k_scatter_local<<<ceil_div(d.n, 256), 256, 0, st>>>(d.n, P->d_local_idx + d.idx_off, r_local, P->d_tmp);
  HG_LAUNCH_CHECK();
  HG_TRY(launch_local_grid(P, P->d_local + s, 1, P->d_tmp, st));
  HG_CUDA_TRY(cudaMemcpyAsync(x_local, P->d_xs + d.idx_off, sizeof(double) * d.n, cudaMemcpyDeviceToDevice, st));
  return HG_OK;
}

}  // namespace hg
