// Setup on the device: pivoted band LU of every local
// Dirichlet block, written straight into the record layout the band-solve
// kernels stream (include/helmgpu.h).
//
// Replaces the host factorisation of schwarz._factor_block
// (schwarz.py:104-131, SuperLU there, LAPACK dgbtrf in factor.band_lu).
// Semantics are dgbtrf's unblocked algorithm (dgbtf2), column by column:
//   p   = first index of max |a_{j..j+km, j}|          (idamax)
//   swap rows j and j+p on the trailing band            (dswap)
//   l   = a_{j+1..j+km, j} * (1 / a_jj)                 (dscal by the reciprocal)
//   a_{j+r, j+c} -= l_r u_c  for the band               (dger)
// with INFO = first exactly-zero pivot (elimination skipped there, as
// LAPACK does).  The row interchanges touch the trailing band only; L
// columns keep the order they were computed in — the dgbtrs convention the
// solve kernels follow.
//
// Execution: one CTA per block.  The active window — rows j..j+RPT-1,
// columns j..j+WC-1 (RPT-1 >= kl, WC = RPT + ku) — lives in REGISTERS:
// thread t owns column slot t (global column c sits in slot c mod WC) and
// keeps that column's RPT window rows in registers, shifted up one row per
// step as the window slides (the shift is fused into the rank-1 update, so
// it costs no moves).  Window rows beyond the block's own kl are zero and
// stay zero, so one instance serves every block with kl <= RPT-1 and gives
// dgbtf2's result for each.  Per step: the owner of the pivot column copies
// it to shared memory; warp 0 finds the pivot (warp argmax, lowest index on
// ties), forms the multipliers and writes the forward record; every thread
// swaps (rare: warp-uniform branch), writes its U entry into the backward
// record of its column and updates its column.  Two CTA barriers per step.
#include <algorithm>

#include "hg_internal.cuh"

namespace hg {

struct BandLuArgs {
  const LocalDesc* descs;      // record layout per block (kl/kv = record widths)
  const int* bw;               // true band half-width (kl = ku) per block
  const long long* ptr_base;   // block s's row pointers start at lcsr_indptr + ptr_base[s]
  const long long* indptr;     // absolute into cols / vals
  const int* cols;             // block-local columns
  const double* vals;
  double* fwd;
  double* bwd;
  int* info;                   // per block: 0 or j+1 (first zero pivot)
  double* minpiv;              // per block: min |u_jj|
  int WC;                      // window columns = RPT + max ku
};

template <int RPT>
__global__ void __launch_bounds__(256) k_band_lu(BandLuArgs a) {
  __shared__ double s_col[RPT];
  __shared__ double s_l[RPT];
  __shared__ double s_nr[2][256];  // entering row, double-buffered by row parity
  __shared__ int s_p;
  const LocalDesc d = a.descs[blockIdx.x];
  const int n = d.n;
  if (n == 0) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int WC = a.WC;
  const bool mine = t < WC;
  const long long* ip = a.indptr + a.ptr_base[blockIdx.x];
  double* fwd = a.fwd + d.fwd_off;
  double* bwd = a.bwd + d.bwd_off;
  const int fs = d.fstride, bs = d.bstride, klp = d.kl, kvp = d.kv;
  double v[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) v[r] = 0.0;
  if (mine) s_nr[0][t] = s_nr[1][t] = 0.0;
  __syncthreads();

  // scatter row `row` of the block into s_nr[row & 1] (slot = column mod WC);
  // warp 1.  Double buffering: a late warp may still read / clear the
  // previous row's buffer while this one is filled.
  auto scatter = [&](int row) {
    if (warp == 1 && row < n) {
      const long long e0 = ip[row], e1 = ip[row + 1];
      for (long long e = e0 + lane; e < e1; e += 32) s_nr[row & 1][a.cols[e] % WC] = a.vals[e];
    }
  };
  // prologue: rows 0..RPT-1 enter the window one by one
  for (int row = 0; row < RPT; ++row) {
    scatter(row);
    __syncthreads();
    if (mine) {
#pragma unroll
      for (int r = 0; r < RPT - 1; ++r) v[r] = v[r + 1];
      v[RPT - 1] = s_nr[row & 1][t];
    }
    __syncthreads();
    if (mine) s_nr[row & 1][t] = 0.0;
  }

  int info = 0;
  double minp = INFINITY;
  for (int j = 0; j < n; ++j) {
    const int owner = j % WC;
    const int km = min(RPT - 1, n - 1 - j);
    if (t == owner) {
#pragma unroll
      for (int r = 0; r < RPT; ++r) s_col[r] = v[r];
    }
    scatter(j + RPT);  // the row that enters at the end of this step
    __syncthreads();
    if (warp == 0) {
      // idamax over s_col[0..km]: first index of the largest magnitude
      double best = -1.0;
      int bi = 0;
      for (int r = lane; r <= km; r += 32) {
        const double x = fabs(s_col[r]);
        if (x > best) {
          best = x;
          bi = r;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(FULL, best, o);
        const int oi = __shfl_xor_sync(FULL, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      const int p = bi;
      const double piv = s_col[p];
      const bool zero = piv == 0.0;
      const double rcp = zero ? 0.0 : 1.0 / piv;
      // multipliers of the pivoted column (row p now holds the old row 0)
      for (int r = lane; r < RPT; r += 32) {
        double l = 0.0;
        if (r >= 1 && r <= km && !zero) l = (r == p ? s_col[0] : s_col[r]) * rcp;
        s_l[r] = l;
      }
      // forward record j: [l_{j+1..j+klp, j}, ipiv_j]
      double* fr = fwd + (long long)j * fs;
      for (int r = lane; r < klp; r += 32) {
        double l = 0.0;
        if (r + 1 <= km && r + 1 < RPT && !zero) l = (r + 1 == p ? s_col[0] : s_col[r + 1]) * rcp;
        fr[r] = l;
      }
      if (lane == 0) {
        fr[klp] = (double)(j + p);
        bwd[(long long)(n - 1 - j) * bs + kvp] = 1.0 / piv;  // 1/u_jj (inf on a zero pivot: INFO set)
        s_p = zero ? 0 : p;
        if (zero && info == 0) info = j + 1;
        minp = fmin(minp, fabs(piv));
      }
    }
    __syncthreads();
    const int p = s_p;
    if (mine) {
      if (p != 0) {  // row interchange j <-> j+p on this column (warp-uniform, rare)
        double vp = v[0];
#pragma unroll
        for (int r = 1; r < RPT; ++r)
          if (r == p) vp = v[r];
#pragma unroll
        for (int r = 1; r < RPT; ++r)
          if (r == p) v[r] = v[0];
        v[0] = vp;
      }
      const double nr = s_nr[(j + RPT) & 1][t];
      s_nr[(j + RPT) & 1][t] = 0.0;
      if (t == owner) {  // column j is finished; its slot becomes column j + WC
#pragma unroll
        for (int r = 0; r < RPT - 1; ++r) v[r] = 0.0;
      } else {
        const double u = v[0];  // u_{j, c}
        const int c = j + (t - owner + WC) % WC;
        if (c < n && c - j <= kvp) bwd[(long long)(n - 1 - c) * bs + (c - j - 1)] = u;
        // rank-1 update fused with the one-row shift of the window
#pragma unroll
        for (int r = 0; r < RPT - 1; ++r) v[r] = fma(-s_l[r + 1], u, v[r + 1]);
      }
      v[RPT - 1] = nr;
    }
  }
  if (t == 0) {
    a.info[blockIdx.x] = info;
    a.minpiv[blockIdx.x] = minp;
  }
}

// smallest compiled window height covering kl
static int pick_rpt(int kl) {
  const int opts[] = {32, 48, 64, 80};
  for (int r : opts)
    if (r - 1 >= kl) return r;
  return 0;
}

int band_lu_supported(int kl_max, int ku_max) {
  const int rpt = pick_rpt(kl_max);
  return rpt > 0 && rpt + ku_max <= 256;
}

int launch_band_lu(HgPrecond* P, const int* d_bw, int kl_max, int ku_max, const long long* d_ptr_base,
                   const long long* d_indptr, const int* d_cols, const double* d_vals, int* d_info, double* d_minpiv,
                   cudaStream_t st) {
  if (P->n_local == 0) return HG_OK;
  const int rpt = pick_rpt(kl_max);
  if (rpt == 0 || rpt + ku_max > 256) {
    set_error("device band LU: band half-width " + std::to_string(kl_max) + " beyond the compiled windows (<= 79)");
    return HG_ERR_UNSUPPORTED;
  }
  BandLuArgs a{P->d_local, d_bw, d_ptr_base, d_indptr, d_cols, d_vals, P->d_fwd, P->d_bwd, d_info, d_minpiv,
               rpt + ku_max};
  const int threads = std::max(64, ((a.WC + 31) / 32) * 32);
  switch (rpt) {
    case 32: k_band_lu<32><<<P->n_local, threads, 0, st>>>(a); break;
    case 48: k_band_lu<48><<<P->n_local, threads, 0, st>>>(a); break;
    case 64: k_band_lu<64><<<P->n_local, threads, 0, st>>>(a); break;
    default: k_band_lu<80><<<P->n_local, threads, 0, st>>>(a); break;
  }
  HG_LAUNCH_CHECK();
  return HG_OK;
}

}  // namespace hg
