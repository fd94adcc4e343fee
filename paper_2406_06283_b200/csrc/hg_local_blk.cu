// Blocked multi-RHS local band solve (batched apply, up to 16 columns).
//
// Same operator as k_local_solve (dgbtrs on the packed band-LU records of
// hg_local_impl.cuh), organised for many right-hand sides: per CTA (one
// subdomain) the active rows of all columns live in a shared-memory window;
// each sweep advances in blocks of 32 rows:
//   phase A  the 32-step dependency chain of the block, all 8 warps side by
//            side (lane = block row, warp w = columns 2w, 2w+1; a step is one
//            multiplier load and two shuffle -> FMA chains), updating only the
//            rows inside the block;
//   phase B  the band below the block receives the block's contribution as
//            one dense product  X[below] -= L[below, block] X[block]
//            (kw x 32 x 16) on the FP64 tensor pipe (mma.sync m8n8k4 f64),
//            A fragments read straight from the staged factor records.
// A block containing a row interchange (forward sweep, ~6% of blocks) runs
// the plain step-by-step elimination over the whole band instead.  Factor
// records stream through the TMA ring exactly as in k_local_solve.
#include <algorithm>
#include <cstdlib>

#include "hg_internal.cuh"

namespace hg {

__device__ int blk_timing_on = 0;  // HG_BLK_TIMING=1: per-phase cycle counts of CTA 0 (diagnosis)

namespace {
constexpr int BK = 32;     // rows per block
constexpr int BSR = 20;    // window row stride (16 columns + pad: conflict-free DMMA B fragments)
constexpr int BNS = 4;     // record ring stages
constexpr int BCH = 16;    // records per stage (as LS_CH)
constexpr int BTHREADS = 256 + 32;

// the producer warp returns early: the 256 consumer threads synchronise on
// named barrier 1 only
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ bool csync_or(bool p) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, 1, 256, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((int)p)
      : "memory");
  return r != 0;
}

__device__ __forceinline__ void dmma_b(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

struct BlkCtx {
  double2* bcast;      // [8 warps][2] step-row broadcast slots
  double* win;         // [wrows][BSR]
  int wrows;
  const double* ring;
  uint64_t* full;
  uint64_t* empty;
  int stage_stride;
};

// one chain step s of a block for this lane's row rw and its warp's two
// columns; the step row's values reach the warp through a shared-memory slot
// (one 16-byte store by lane s, one broadcast load) instead of four shuffles
template <bool FWD>
__device__ __forceinline__ void blk_step(int s, const double* __restrict__ r, int rw, int kw, double& v0,
                                         double& v1, double2* slot) {
  const bool below = rw > s && rw - s <= kw;
  const double m = below ? r[rw - s - 1] : 0.0;
  // double-buffered by step parity: one warp barrier per step (a lane cannot
  // rewrite slot[s & 1] before every lane passed step s+1's barrier)
  double2* sl = slot + (s & 1);
  if (rw == s) *sl = make_double2(v0, v1);
  __syncwarp();
  const double2 xs2 = *sl;
  double x0 = xs2.x, x1 = xs2.y;
  if (!FWD) {
    const double dv = r[kw];
    x0 *= dv;
    x1 *= dv;
    if (rw == s) {
      v0 = x0;
      v1 = x1;
    }
  }
  if (below) {
    v0 = fma(-m, x0, v0);
    v1 = fma(-m, x1, v1);
  }
}

// one sweep (FWD: gathered input, pivoted L; !FWD: reversed U with 1/u_jj)
template <bool FWD>
__device__ void blk_sweep(const BlkCtx& cx, int& chunk, int n, int kw, int stride, const int* __restrict__ idx,
                          const double* __restrict__ R, long long ldr, double* __restrict__ xs, long long xs_len,
                          int nrhs) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W = cx.wrows;
  double* win = cx.win;
  auto in = [&](int row, int c) -> double {
    if (row >= n || c >= nrhs) return 0.0;
    if (FWD) return __ldg(R + (long long)c * ldr + __ldg(idx + row));
    return xs[(long long)c * xs_len + (n - 1 - row)];
  };
  auto out = [&](int row, int c, double v) {
    if (row < n && c < nrhs) xs[(long long)c * xs_len + (FWD ? row : n - 1 - row)] = v;
  };
  for (int e = tid; e < W * 16; e += 256) {
    const int row = e >> 4, c = e & 15;
    win[row * BSR + c] = in(row, c);
  }
  csync();
  long long tw = 0, ta = 0, tb = 0, tr = 0;
  for (int j0 = 0; j0 < n; j0 += BK) {
    const long long c0t = clock64();
    const int nb = min(BK, n - j0);
    const int base = j0 % W;  // ring position of row j0: row j0 + x (0 <= x < W) sits at wr(x)
    auto wr = [&](int x) -> int {
      const int p = base + x;
      return p >= W ? p - W : p;
    };
    const int nch = (nb + BCH - 1) / BCH;
    // rows entering the window after this block (positions of the block's rows), fetched early
    double nxt[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int e = tid + 256 * q, i = e >> 4, c = e & 15;
      nxt[q] = in(j0 + W + i, c);
    }
    const int st0 = chunk % BNS;
    mbar_wait(&cx.full[st0], (chunk / BNS) & 1);
    const double* rec0 = cx.ring + (size_t)st0 * cx.stage_stride;
    const double* rec1 = rec0;
    int st1 = st0;
    if (nch == 2) {
      st1 = (chunk + 1) % BNS;
      mbar_wait(&cx.full[st1], ((chunk + 1) / BNS) & 1);
      rec1 = cx.ring + (size_t)st1 * cx.stage_stride;
    }
    auto rec = [&](int s) -> const double* { return (s < BCH ? rec0 : rec1) + (s & (BCH - 1)) * stride; };
    const long long c1t = clock64();
    tw += c1t - c0t;
    bool piv = false;
    if (FWD) {
      const int p = (tid < nb) ? __double2int_rn(rec(tid)[kw]) : j0 + tid;
      piv = csync_or(tid < nb && p != j0 + tid);
    }
    if (!piv) {
      // ---- phase A: the block's chain; lane = block row, warp w owns columns
      // 2w, 2w+1 (columns are independent: no cross-warp dependency, the 8
      // warps run their chains side by side); a step is one multiplier load
      // and 2 shuffle -> FMA chains per warp
      {
        const int rw = lane;  // block row of this lane
        const int c0 = 2 * warp;
        double2* bslot = cx.bcast + 2 * warp;
        double* wrow = win + wr(rw) * BSR + c0;
        const double2 t2 = *reinterpret_cast<const double2*>(wrow);
        double v0 = t2.x, v1 = t2.y;
        // step s of the block: record rec0 + s*stride (s < 16) / rec1 + (s-16)*stride
        const int n0 = min(nb, BCH);
        const double* r = rec0;
#pragma unroll 4
        for (int s = 0; s < n0; ++s, r += stride) blk_step<FWD>(s, r, rw, kw, v0, v1, bslot);
        r = rec1;
#pragma unroll 4
        for (int s = BCH; s < nb; ++s, r += stride) blk_step<FWD>(s, r, rw, kw, v0, v1, bslot);
        if (rw < nb) {
          *reinterpret_cast<double2*>(wrow) = make_double2(v0, v1);
          out(j0 + rw, c0, v0);
          out(j0 + rw, c0 + 1, v1);
        }
      }
      csync();
      const long long c2t = clock64();
      ta += c2t - c1t;
      // ---- phase B: rows j0+32+r (r < W-32) -= L[below, block] X[block] on DMMA
      const int q = lane & 3, g = lane >> 2;
      const int tiles = (W - BK) >> 3;
      for (int t = warp; t < 2 * tiles; t += 8) {
        const int rt = t >> 1, nh = t & 1;
        const int r0 = rt * 8 + g;  // below-row of this lane's A / C fragments
        double* crow = win + wr(BK + r0) * BSR + nh * 8 + 2 * q;
        double acc[2] = {0.0, 0.0};  // L[below, block] X[block], subtracted once
#pragma unroll
        for (int k0 = 0; k0 < BK; k0 += 4) {
          const int s = k0 + q;
          const int tt = BK + r0 - s;  // row offset from step s (>= 1)
          const double* rs = (k0 < BCH ? rec0 + s * stride : rec1 + (s - BCH) * stride);
          const double a = (s < nb && tt <= kw) ? rs[tt - 1] : 0.0;
          const double b = win[wr(k0 + q) * BSR + nh * 8 + g];
          dmma_b(acc, a, b);
        }
        crow[0] -= acc[0];
        crow[1] -= acc[1];
      }
      csync();
      tb += clock64() - c2t;
    } else {
      // ---- row interchanges in the block: plain elimination over the whole band
      for (int s = 0; s < nb; ++s) {
        const int j = j0 + s;
        const double* r = rec(s);
        const int p = __double2int_rn(r[kw]);
        if (p != j && tid < 16) {
          double* a = win + wr(s) * BSR + tid;
          double* b = win + wr(p - j0) * BSR + tid;
          const double tmp = *a;
          *a = *b;
          *b = tmp;
        }
        csync();
        for (int e = tid; e < kw * 16; e += 256) {
          const int t = (e >> 4) + 1, c = e & 15;
          double* dst = win + wr(s + t) * BSR + c;
          *dst = fma(-r[t - 1], win[wr(s) * BSR + c], *dst);
        }
        csync();
      }
      for (int e = tid; e < nb * 16; e += 256) {
        const int Rw = e >> 4, c = e & 15;
        out(j0 + Rw, c, win[wr(Rw) * BSR + c]);
      }
    }
    csync();  // records and the block's rows consumed
    if (tid == 0) {
      mbar_arrive(&cx.empty[st0]);
      if (nch == 2) mbar_arrive(&cx.empty[st1]);
    }
    chunk += nch;
#pragma unroll
    for (int q2 = 0; q2 < 2; ++q2) {
      const int e = tid + 256 * q2, i = e >> 4, c = e & 15;
      if (i < nb) win[wr(i) * BSR + c] = nxt[q2];
    }
    csync();
    tr += clock64() - c0t;
  }
  if (blk_timing_on && blockIdx.x == 0 && threadIdx.x == 0)
    printf("[blk] %s n=%d kw=%d blocks=%d: per block cycles wait %.0f, phase A %.0f, phase B %.0f, total %.0f\n",
           FWD ? "fwd" : "bwd", n, kw, (n + BK - 1) / BK, (double)tw / ((n + BK - 1) / BK),
           (double)ta / ((n + BK - 1) / BK), (double)tb / ((n + BK - 1) / BK), (double)tr / ((n + BK - 1) / BK));
}
}  // namespace

__global__ void __launch_bounds__(BTHREADS, 2) k_local_blocked(const LocalDesc* __restrict__ descs,
                                                              const int* __restrict__ idx,
                                                              const double* __restrict__ fwd,
                                                              const double* __restrict__ bwd,
                                                              const double* __restrict__ R, long long ldr,
                                                              double* __restrict__ xs, long long xs_len, int nrhs,
                                                              int stage_stride, int wrows) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[BNS], empty[BNS];
  const LocalDesc d = descs[blockIdx.x];
  if (threadIdx.x == 0) {
    for (int s = 0; s < BNS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (d.n == 0) return;
  const int nc = (d.n + BCH - 1) / BCH;
  if (threadIdx.x >= 256) {
    if (threadIdx.x == 256) {  // producer: the same record stream as k_local_solve
      for (int c = 0; c < 2 * nc; ++c) {
        const int stage = c % BNS;
        if (c >= BNS) mbar_wait(&empty[stage], ((c / BNS) - 1) & 1);
        const bool f = c < nc;
        const int cc = f ? c : c - nc;
        const int rows = min(BCH, d.n - cc * BCH);
        const int stride = f ? d.fstride : d.bstride;
        const double* src = (f ? fwd + d.fwd_off : bwd + d.bwd_off) + (long long)cc * BCH * stride;
        const uint32_t bytes = (uint32_t)rows * stride * 8u;
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(sm + (size_t)stage * stage_stride, src, bytes, &full[stage]);
      }
    }
    return;
  }
  // named barrier 0 is used by __syncthreads: the producer warp has returned,
  // so the consumers synchronise among themselves with bar.sync 1, 256
  __shared__ double2 bcast[16];
  BlkCtx cx{bcast, sm + (size_t)BNS * stage_stride, wrows, sm, full, empty, stage_stride};
  int chunk = 0;
  blk_sweep<true>(cx, chunk, d.n, d.kl, d.fstride, idx + d.idx_off, R, ldr, xs + d.idx_off, xs_len, nrhs);
  blk_sweep<false>(cx, chunk, d.n, d.kv, d.bstride, nullptr, nullptr, 0, xs + d.idx_off, xs_len, nrhs);
}

size_t local_blocked_smem(HgPrecond* P, int* wrows_out) {
  int kwmax = 0;
  for (const LocalDesc& d : P->h_local) kwmax = std::max(kwmax, std::max(d.kl, d.kv));
  const int wrows = BK + ((kwmax + 7) / 8) * 8;
  if (wrows_out) *wrows_out = wrows;
  const int stage_stride = BCH * (P->max_fstride > P->max_bstride ? P->max_fstride : P->max_bstride);
  return sizeof(double) * ((size_t)BNS * stage_stride + (size_t)wrows * BSR);
}

int launch_local_blocked(HgPrecond* P, const double* R, long long ldr, int nrhs, cudaStream_t st) {
  if (P->n_local == 0) return HG_OK;
  int wrows = 0;
  const size_t smem = local_blocked_smem(P, &wrows);
  const int stage_stride = BCH * (P->max_fstride > P->max_bstride ? P->max_fstride : P->max_bstride);
  static bool timing_set = false;  // timing experiments only
  if (!timing_set) {
    const char* tm = getenv("HG_BLK_TIMING");
    int on = (tm && tm[0] == '1') ? 1 : 0;
    HG_CUDA_TRY(cudaMemcpyToSymbol(blk_timing_on, &on, sizeof(int)));
    timing_set = true;
  }
  HG_TRY(ensure_func_attrs(reinterpret_cast<const void*>(k_local_blocked), smem, false));
  k_local_blocked<<<P->n_local, BTHREADS, smem, st>>>(P->d_local, P->d_local_idx, P->d_fwd, P->d_bwd, R, ldr,
                                                       P->d_xsm, P->xs_len, nrhs, stage_stride, wrows);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

int preload_local_blocked() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_local_blocked));
  return HG_OK;
}

}  // namespace hg
