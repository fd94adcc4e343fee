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
// Execution model (per CTA, 2 warps for one right-hand side):
//  * warp 1 lane 0 is the producer: it streams the packed factor records
//    (16 steps per chunk) from HBM into a shared-memory ring with
//    cp.async.bulk (TMA bulk copies) completing on mbarriers.  Factors are
//    read exactly once, in order, so the kernel is an HBM stream.
//  * warp 0 is the consumer: the active window of the right-hand side lives
//    in registers, 32 rows per register (row j0 + 32r + lane sits in
//    register r of `lane` during the round that finalises rows j0..j0+31).
//    Each lane applies its multipliers from the staged record
//    (conflict-free 64-bit shared loads).  After 32 steps the finished rows
//    are stored with one coalesced store and the registers rotate; entering
//    rows are prefetched one round ahead.
//  * "front": the next F = 4 rows of the window are additionally replicated
//    in every lane and updated redundantly (same fma, same operands, so the
//    copies agree bitwise).  The pivot value of step j is then already in
//    every lane, and the dependency chain of a step is a single DFMA
//    (8 cycles on B200) instead of SHFL -> DFMA (41 cycles measured,
//    tools/micro/lat.cu); the shuffle that feeds row j+F into the front is
//    F-1 steps off the critical path.
//  * the backward sweep runs the same machinery on the reversed row order
//    (records are stored reversed), in place on the per-block scratch.
// The output of each block goes to its own scratch segment; overlapping
// contributions are summed later in a fixed order (hg_coarse.cu
// k_assemble), so there are no atomics and the result is deterministic.
#pragma once
#include <cstdlib>

#include "hg_internal.cuh"

namespace hg {

constexpr int LS_CH = 16;  // steps per staged chunk
constexpr int LS_NS = 6;   // ring stages at most (runtime count: HgPrecond::ls_ns, 4 or 6)
constexpr int LS_THREADS = 64;        // single right-hand side: 1 consumer + 1 producer warp

// Every sweep function is templated on K, the right-hand sides one consumer
// warp carries: each staged multiplier is loaded from shared memory once and
// applied to K windows (K = 1: the single-RHS chain; K = LS_KM: the batched
// kernel, where shared-memory bandwidth and not the chain bounds the step).

// Row interchange of rows j (register 0, lane s) and l (register (l-j0)/32,
// lane (l-j0)%32) in the distributed window; warp-uniform, ~0.2% of steps.
template <int K, int R>
__device__ __forceinline__ void ls_swap(double (&v)[K][R], int s, int l, int j0, int lane) {
  const int rl = (l - j0) >> 5, ll = (l - j0) & 31;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double a = __shfl_sync(FULL, v[k][0], s);
    double sel = v[k][0];
#pragma unroll
    for (int r = 1; r < R; ++r)
      if (r == rl) sel = v[k][r];
    const double b = __shfl_sync(FULL, sel, ll);
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r == rl && lane == ll) v[k][r] = a;
    if (lane == s) v[k][0] = b;
  }
}

template <int R>
__device__ __forceinline__ double ls_fetch(const double (&v)[R], int row_in_round) {
  // value of window row j0 + row_in_round (compile-time) broadcast to all lanes
  return __shfl_sync(FULL, v[row_in_round >> 5], row_in_round & 31);
}

struct SweepCtx {
  const double* ring;  // smem ring base
  int ns;              // ring stages in use
  uint64_t* full;
  uint64_t* empty;
  int stage_stride;    // doubles per stage
};

// One elimination step S (compile-time position in the round) with the
// front f[(S+q)&3] = row j+q, q = 0..3 (roles rotate, values never move).
// Record layout: rec[t-1] = multiplier of row j+t (t = 1..kw), rec[kw] =
// pivot (FWD) or 1/u_jj (BWD).  lim = kw - lane.  Multipliers outside the
// band are skipped by predication (only registers 0, R-2, R-1 can be partly
// outside: R = 1 + ceil(kw_max/32) and every block's records padded to
// kw >= 32 R - 65 keep registers 1..R-3 inside; hg_precond_create checks).
template <int K, int R, bool FWD, int S>
__device__ __forceinline__ void ls_step(double (&v)[K][R], double (&f)[K][4], const double* __restrict__ rec,
                                        int lane, int lim, int kw) {
  constexpr int p = S & 3;
  double bj[K];
#pragma unroll
  for (int k = 0; k < K; ++k) bj[k] = f[k][p];
  if (!FWD) {
    const double dinv = rec[kw];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      bj[k] = f[k][p] * dinv;
      if (lane == S) v[k][0] = bj[k];
    }
  }
  const double2 m01 = *reinterpret_cast<const double2*>(rec);  // 16-byte aligned: even stride
  const double m2 = rec[2];
  // front (every lane): the critical chain is f[p+1] -> next step's pivot
#pragma unroll
  for (int k = 0; k < K; ++k) {
    f[k][(p + 1) & 3] = fma(-m01.x, bj[k], f[k][(p + 1) & 3]);
    f[k][(p + 2) & 3] = fma(-m01.y, bj[k], f[k][(p + 2) & 3]);
    f[k][(p + 3) & 3] = fma(-m2, bj[k], f[k][(p + 3) & 3]);
  }
  // distributed window
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int t = 32 * r + lane - S;
    const bool edge = (r == 0) || (r >= R - 2);
    const bool on = !edge || ((r == 0 ? (lane > S) : true) && (32 * r - S <= lim));
    if (on) {
      const double m = rec[t - 1];
#pragma unroll
      for (int k = 0; k < K; ++k) v[k][r] = fma(-m, bj[k], v[k][r]);
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) f[k][p] = ls_fetch<R>(v[k], S + 4);  // row j+4, includes this step's update
}

// Straight-line round of 32 steps without pivots (the common case).
template <int K, int R, bool FWD, int S>
__device__ __forceinline__ void ls_round_fast(double (&v)[K][R], double (&f)[K][4], const double* rec0,
                                              const double* rec1, int stride, int lane, int lim, int kw) {
  if constexpr (S < 32) {
    ls_step<K, R, FWD, S>(v, f, (S < LS_CH ? rec0 : rec1) + S * stride, lane, lim, kw);
    ls_round_fast<K, R, FWD, S + 1>(v, f, rec0, rec1, stride, lane, lim, kw);
  }
}

// General round: partial (last) round and/or row interchanges.
template <int K, int R, bool FWD, int S>
__device__ __forceinline__ void ls_round_slow(double (&v)[K][R], double (&f)[K][4], const double* rec0,
                                              const double* rec1, int stride, int lane, int lim, int kw,
                                              unsigned swapmask, int pl, int j0, int nsteps) {
  if constexpr (S < 32) {
    if (S < nsteps) {
      if (FWD && ((swapmask >> S) & 1u)) {
        // row interchange: permute the distributed window, refresh the front
        ls_swap<K, R>(v, S, __shfl_sync(FULL, pl, S), j0, lane);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          f[k][S & 3] = ls_fetch<R>(v[k], S);
          f[k][(S + 1) & 3] = ls_fetch<R>(v[k], S + 1);
          f[k][(S + 2) & 3] = ls_fetch<R>(v[k], S + 2);
          f[k][(S + 3) & 3] = ls_fetch<R>(v[k], S + 3);
        }
      }
      ls_step<K, R, FWD, S>(v, f, (S < LS_CH ? rec0 : rec1) + S * stride, lane, lim, kw);
      ls_round_slow<K, R, FWD, S + 1>(v, f, rec0, rec1, stride, lane, lim, kw, swapmask, pl, j0, nsteps);
    }
  }
}

// One sweep over n rows for kc <= K right-hand sides (column k: input
// rin + k * ldr, scratch xs + k * xs_len).  FWD: input gathered from
// r[idx[row]], output y[row] into xs.  !FWD: input y from xs in reverse,
// output x into xs in reverse.
template <int K, int R, bool FWD>
__device__ void ls_sweep(const SweepCtx& cx, int& chunk, int n, int kw, int stride,
                         const int* __restrict__ idx, const double* __restrict__ rin, long long ldr,
                         double* __restrict__ xs, long long xs_len, int kc, int dbg) {
  static_assert(R >= 2, "window must hold row j+4 of every step");
  const int lane = threadIdx.x & 31;
  auto load_in = [&](int k, int row) -> double {
    if (row >= n || k >= kc) return 0.0;
    if (FWD) return __ldg(rin + (long long)k * ldr + __ldg(idx + row));
    return xs[(long long)k * xs_len + n - 1 - row];
  };
  const int lim = kw - lane;
  double v[K][R], f[K][4], pre[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int r = 0; r < R; ++r) v[k][r] = load_in(k, 32 * r + lane);
    pre[k] = load_in(k, 32 * R + lane);
#pragma unroll
    for (int q = 0; q < 4; ++q) f[k][q] = ls_fetch<R>(v[k], q);
  }
  for (int j0 = 0; j0 < n; j0 += 32) {
    double nxt[K];
#pragma unroll
    for (int k = 0; k < K; ++k) nxt[k] = load_in(k, j0 + 32 * R + 32 + lane);
    // the round's records: one or two staged chunks
    const int nch = (min(32, n - j0) + LS_CH - 1) / LS_CH;
    // `chunk` = ring position as stage | parity << 8, advanced without a division (runtime ns)
    const int st0 = chunk & 255, par0 = chunk >> 8;
    if (!(dbg & 1)) mbar_wait(&cx.full[st0], par0);
    const double* rec0 = cx.ring + (size_t)st0 * cx.stage_stride;
    const double* rec1 = rec0;
    int st1 = st0;
    if (nch == 2) {
      st1 = st0 + 1 == cx.ns ? 0 : st0 + 1;
      if (!(dbg & 1)) mbar_wait(&cx.full[st1], st1 == 0 ? par0 ^ 1 : par0);
      rec1 = cx.ring + (size_t)st1 * cx.stage_stride - LS_CH * stride;
    }
    // pivots of the round decoded once: lane s holds ipiv of step j0+s
    unsigned swapmask = 0;
    int pl = 0;
    if (FWD) {
      const int j = j0 + lane;
      pl = j;
      if (j < n) pl = __double2int_rn((lane < LS_CH ? rec0 : rec1)[lane * stride + kw]);
      swapmask = __ballot_sync(FULL, pl != j);
    }
    if (!(dbg & 2)) {
      const int nsteps = min(32, n - j0);
      if (nsteps == 32 && swapmask == 0u)
        ls_round_fast<K, R, FWD, 0>(v, f, rec0, rec1, stride, lane, lim, kw);
      else
        ls_round_slow<K, R, FWD, 0>(v, f, rec0, rec1, stride, lane, lim, kw, swapmask, pl, j0, nsteps);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&cx.empty[st0]);
      if (nch == 2) mbar_arrive(&cx.empty[st1]);
    }
    {
      int st = st0 + nch, par = par0;
      if (st >= cx.ns) {
        st -= cx.ns;
        par ^= 1;
      }
      chunk = st | (par << 8);
    }
    const int row = j0 + lane;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (row < n && k < kc) {
        if (FWD)
          xs[(long long)k * xs_len + row] = v[k][0];
        else
          xs[(long long)k * xs_len + n - 1 - row] = v[k][0];
      }
#pragma unroll
      for (int r = 0; r + 1 < R; ++r) v[k][r] = v[k][r + 1];
      v[k][R - 1] = pre[k];
      pre[k] = nxt[k];
    }
  }
}

constexpr int LS_KM = 2;  // right-hand sides per consumer warp in the batched kernel (4 spills past 255 registers)

// K right-hand sides per consumer warp; consumer warp w solves columns
// w*K .. min(w*K + K, nrhs) - 1 (input r + c * ldr, output xs + c * xs_len)
// against the SAME staged factor records, so the factors stream from HBM
// once for all columns; every consumer warp releases each ring stage (empty
// barrier count = consumer warps).  Two kernels share the body with their
// own launch bounds: the single-RHS chain (64 threads, hg_local.cu) and the
// batched one (HG_MAX_RHS / LS_KM + 1 warps, hg_local_multi.cu).
template <int RF, int RB, int K>
__device__ __forceinline__ void local_solve_body(const LocalDesc* __restrict__ descs, const int* __restrict__ idx,
                                                 const double* __restrict__ fwd, const double* __restrict__ bwd,
                                                 const double* __restrict__ r, double* __restrict__ xs,
                                                 int stage_stride, int dbg, long long ldr, long long xs_len,
                                                 int nrhs, int ns) {
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[LS_NS], empty[LS_NS];
  const LocalDesc d = descs[blockIdx.x];
  const int nw = K == 1 ? 1 : (int)(blockDim.x >> 5) - 1;  // consumer warps
  const int warp = K == 1 ? (threadIdx.x >= 32 ? 1 : 0) : (int)(threadIdx.x >> 5);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nw);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (d.n == 0) return;
  const int nc = (d.n + LS_CH - 1) / LS_CH;
  if (warp == nw) {
    if ((threadIdx.x & 31) == 0 && !(dbg & 1)) {  // producer
      int stage = 0, epar = 1;  // parity of the previous pass over the ring (none yet)
      for (int c = 0; c < 2 * nc; ++c, ++stage) {
        if (stage == ns) {
          stage = 0;
          epar ^= 1;
        }
        if (c >= ns) mbar_wait(&empty[stage], epar);
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
  SweepCtx cx{ring, ns, full, empty, stage_stride};
  int chunk = 0;
  const int c0 = K == 1 ? 0 : warp * K;
  const int kc = K == 1 ? 1 : min(K, nrhs - c0);
  double* xsb = xs + (long long)c0 * xs_len + d.idx_off;
  const double* rin = r + (long long)c0 * ldr;
  const long long t0 = clock64();
  ls_sweep<K, RF, true>(cx, chunk, d.n, d.kl, d.fstride, idx + d.idx_off, rin, ldr, xsb, xs_len, kc, dbg);
  __syncwarp();
  const long long t1 = clock64();
  ls_sweep<K, RB, false>(cx, chunk, d.n, d.kv, d.bstride, nullptr, nullptr, 0, xsb, xs_len, kc, dbg);
  if ((dbg & 4) && blockIdx.x < 2 && threadIdx.x == 0) {
    const long long t2 = clock64();
    printf("block %d n=%d kl=%d kv=%d: fwd %.1f cyc/step, bwd %.1f cyc/step\n", blockIdx.x, d.n, d.kl, d.kv,
           (double)(t1 - t0) / d.n, (double)(t2 - t1) / d.n);
  }
}

template <int RF, int RB, int NWMAX>
__global__ void __launch_bounds__(LS_THREADS) k_local_solve(const LocalDesc* __restrict__ descs,
                                                           const int* __restrict__ idx,
                                                           const double* __restrict__ fwd,
                                                           const double* __restrict__ bwd,
                                                           const double* __restrict__ r, double* __restrict__ xs,
                                                           int stage_stride, int dbg, long long ldr,
                                                           long long xs_len, int nrhs, int ns) {
  local_solve_body<RF, RB, 1>(descs, idx, fwd, bwd, r, xs, stage_stride, dbg, ldr, xs_len, nrhs, ns);
}

template <int RF, int RB>
__global__ void __launch_bounds__(32 * (HG_MAX_RHS / LS_KM + 1), 2) k_local_solve_multi(
    const LocalDesc* __restrict__ descs, const int* __restrict__ idx, const double* __restrict__ fwd,
    const double* __restrict__ bwd, const double* __restrict__ r, double* __restrict__ xs, int stage_stride, int dbg,
    long long ldr, long long xs_len, int nrhs, int ns) {
  local_solve_body<RF, RB, LS_KM>(descs, idx, fwd, bwd, r, xs, stage_stride, dbg, ldr, xs_len, nrhs, ns);
}

using LocalKernel = void (*)(const LocalDesc*, const int*, const double*, const double*, const double*,
                             double*, int, int, long long, long long, int, int);

template <int RF, int RB, int NW>
static LocalKernel pick2() {
  if constexpr (NW == 1)
    return k_local_solve<RF, RB, 1>;
  else
    return k_local_solve_multi<RF, RB>;
}

// compile-time tile actually instantiated for a switch case (cases the
// runtime guard below rejects map onto an instantiated one, never returned)
constexpr int rb_clamp(int rf, int x, int nw) {
  return x < rf ? rf : (nw > 1 && x > 2 * rf + 1 ? 2 * rf + 1 : x);
}

// kv = kl + ku >= kl, so rb >= rf: only those tiles are instantiated; the
// batched kernel only for rb <= 2 rf + 1 (ku <= kl, as for the symmetric
// band patterns of the Helmholtz blocks; anything else fails loudly)
template <int RF, int NW>
static LocalKernel pick_rb(int rb) {
  if (rb < RF || (NW > 1 && rb > 2 * RF + 1)) return nullptr;
  switch (rb) {
    case 2: return pick2<RF, rb_clamp(RF, 2, NW), NW>();
    case 3: return pick2<RF, rb_clamp(RF, 3, NW), NW>();
    case 4: return pick2<RF, rb_clamp(RF, 4, NW), NW>();
    case 5: return pick2<RF, rb_clamp(RF, 5, NW), NW>();
    case 6: return pick2<RF, rb_clamp(RF, 6, NW), NW>();
    case 7: return pick2<RF, rb_clamp(RF, 7, NW), NW>();
    case 8: return pick2<RF, rb_clamp(RF, 8, NW), NW>();
    case 9: return pick2<RF, rb_clamp(RF, 9, NW), NW>();
    case 10: return pick2<RF, rb_clamp(RF, 10, NW), NW>();
    default: return nullptr;
  }
}

// Instantiations are spread over several translation units (hg_local_t*.cu)
// so they compile in parallel; each defines one of these per-rf pickers.
LocalKernel pick_local_single_lo(int rf, int rb);   // rf 2..3
LocalKernel pick_local_single_hi(int rf, int rb);   // rf 4..6
LocalKernel pick_local_multi_lo(int rf, int rb);    // rf 2..3
LocalKernel pick_local_multi_mid(int rf, int rb);   // rf 4
LocalKernel pick_local_multi_hi(int rf, int rb);    // rf 5..6

template <int NW>
static LocalKernel pick_local(int rf, int rb) {
  if (NW == 1) return rf <= 3 ? pick_local_single_lo(rf, rb) : pick_local_single_hi(rf, rb);
  return rf <= 3 ? pick_local_multi_lo(rf, rb) : rf == 4 ? pick_local_multi_mid(rf, rb) : pick_local_multi_hi(rf, rb);
}

// Launch the block solves of `nblocks` descriptors with nrhs consumer warps.
template <int NW>
static int launch_local_grid_t(HgPrecond* P, const LocalDesc* descs, int nblocks, const double* r, cudaStream_t st,
                               int nrhs, long long ldr, double* xs, long long xs_len) {
  LocalKernel k = pick_local<NW>(P->rf, P->rb);
  if (!k) {
    set_error("local band solve: bandwidth beyond the compiled register tiles (kl <= 160, kv <= 288)");
    return HG_ERR_UNSUPPORTED;
  }
  const int stage_stride = LS_CH * (P->max_fstride > P->max_bstride ? P->max_fstride : P->max_bstride);
  const int ns = P->ls_ns >= 2 && P->ls_ns <= LS_NS ? P->ls_ns : LS_NS;
  const size_t smem = (size_t)ns * stage_stride * sizeof(double);
  HG_TRY(ensure_func_attrs(reinterpret_cast<const void*>(k), (size_t)LS_NS * stage_stride * sizeof(double), false));
  static const int dbg = getenv("HG_LOCAL_DEBUG") ? atoi(getenv("HG_LOCAL_DEBUG")) : 0;  // timing experiments only
  const int nwarps = NW == 1 ? 1 : (nrhs + LS_KM - 1) / LS_KM;  // consumer warps
  k<<<nblocks, 32 * (nwarps + 1), smem, st>>>(descs, P->d_local_idx, P->d_fwd, P->d_bwd, r, xs ? xs : P->d_xs,
                                               stage_stride, dbg, ldr, xs_len, nrhs, ns);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

}  // namespace hg
