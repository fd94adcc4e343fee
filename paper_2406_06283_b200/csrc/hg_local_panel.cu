// Batched local solves as 16-row panels on the FP64 tensor pipe (the
// batched apply's one-level part, schwarz.py:58-60, for up to 16 columns).
//
// Same operator as the row-record kernels of hg_local_impl.cuh (dgbtrs on
// the band LU of every block: pivoted L sweep, then U sweep in reversed
// coordinates), blocked so that no step-by-step dependency chain remains:
// per sweep the rows advance 16 at a time and a panel is two small dense
// products of the SAME operand,
//     X          =  D^{-1}       W[panel rows]          (16 x 16 x nrhs)
//     W[trail]  +=  -(T D^{-1})  W[panel rows]          (kw x 16 x nrhs)
// where D is the panel's 16 x 16 diagonal block of L (unit) or of U in
// reversed coordinates (diagonal u_jj), T the band below it, and W the
// window of active right-hand-side rows (shared memory, all columns).  With
// T D^{-1} formed at setup both products are independent: every warp works
// on its tiles at once and a panel costs one CTA barrier.
// Row interchanges (forward sweep, ~0.2% of rows) are moved to the front of
// their panel: the panel's swaps are applied to W first and the multiplier
// columns carry the later in-panel swaps (getrf's convention), which is the
// same elimination reordered.  D^{-1} and T come from a setup conversion of
// the row records (k_panel_convert below), stored in DMMA A-fragment order
// (one coalesced 8-byte load per lane per fragment, T negated), and stream
// through a TMA bulk-copy ring like the row records do.  The explicit 16 x 16
// inverses change the rounding, not the operator: hg_precond_create checks
// the panel solve against the row solve on a seeded batch and keeps the row
// kernel if they differ by more than 1e-11 (hg_precond_stat reports it).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "hg_internal.cuh"

namespace hg {

namespace {
constexpr int PB = 16;        // panel rows
// window row stride for NT column tiles of 8 (+ pad: conflict-free B fragments; (stride q + g) mod 16
// distinct over a half-warp for stride 20 and 12)
template <int NT>
struct PanelCols {
  static constexpr int NC = 8 * NT;
  static constexpr int PSR = NT == 2 ? 20 : 12;
};
constexpr int PNS_MAX = 8;    // ring stages (runtime count ns <= PNS_MAX: PanelArgs::ns)
constexpr int PD = 4;         // panels of look-ahead for the entering rows (a gather is two dependent loads)
constexpr int PTHREADS = 256 + 32;

__device__ __forceinline__ void psync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ bool psync_or(bool p) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, 1, 256, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((int)p)
      : "memory");
  return r != 0;
}

__device__ __forceinline__ void dmma_p(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}
}  // namespace

// panel record: [16 relative pivot rows (forward) / 0..15 (backward)]
//               [D^{-1} fragments: 2 m-tiles x 4 k-steps x 32 lanes]
//               [-(T D^{-1}) fragments: KWP/8 m-tiles x 4 k-steps x 32 lanes]
// in a fixed stride; only the first 272 + 128 mt doubles are streamed, mt =
// the panel's count of nonzero 8-row m-tiles of T (per-panel byte `pmt`):
// U's band reaches kl + ku only below row interchanges, so most backward
// panels need about half of KWP.
constexpr int PREC_HDR = 16 + 256;  // pivots + D^{-1} fragments (doubles)
__host__ __device__ inline long long panel_doubles(int kwp) { return PREC_HDR + 16LL * kwp; }
__host__ __device__ inline long long panel_used(int mt) { return PREC_HDR + 128LL * mt; }

// ------------------------------------------------------------------ setup conversion
// One CTA per block, 128 threads, panels in order.  Lt[(16 + KWP) x 16]: the
// panel's multiplier columns (row r = panel row j0 + r), unit (L) or u_jj
// (U, only its reciprocal is stored) diagonal.
template <bool FWD>
__global__ void __launch_bounds__(128) k_panel_convert(const LocalDesc* __restrict__ descs,
                                                       const double* __restrict__ rec_all,
                                                       const long long* __restrict__ poff, int kwp,
                                                       double* __restrict__ out_all,
                                                       const long long* __restrict__ mtoff,
                                                       unsigned char* __restrict__ mt_all) {
  extern __shared__ double lt[];  // (16 + kwp) x 16, then dinvd[16], then X[16][17]
  const LocalDesc d = descs[blockIdx.x];
  const int n = d.n;
  if (n == 0) return;
  const int kw = FWD ? d.kl : d.kv;
  const int stride = FWD ? d.fstride : d.bstride;
  const double* rec = rec_all + (FWD ? d.fwd_off : d.bwd_off);
  double* out = out_all + poff[blockIdx.x];
  const int rows = PB + kwp;
  double* dinvd = lt + rows * PB;
  double* X = dinvd + PB;
  __shared__ int prel[PB];
  const int tid = threadIdx.x;
  const int np = (n + PB - 1) / PB;
  const long long PS = panel_doubles(kwp);
  for (int p = 0; p < np; ++p) {
    const int j0 = p * PB;
    for (int e = tid; e < rows * PB; e += blockDim.x) lt[e] = 0.0;
    __syncthreads();
    for (int e = tid; e < PB * (kw + 1); e += blockDim.x) {
      const int c = e / (kw + 1), t = e % (kw + 1);  // t = 0: diagonal / pivot slot
      const int j = j0 + c;
      const double* r = rec + (long long)j * stride;
      if (t == 0) {
        if (j < n) {
          if (FWD) {
            lt[c * PB + c] = 1.0;
            prel[c] = __double2int_rn(r[kw]) - j0;
          } else {
            dinvd[c] = r[kw];
            prel[c] = c;
          }
        } else {
          lt[c * PB + c] = 1.0;
          if (!FWD) dinvd[c] = 1.0;
          prel[c] = c;
        }
      } else if (j < n && c + t < rows) {
        lt[(c + t) * PB + c] = r[t - 1];
      }
    }
    __syncthreads();
    if (FWD) {
      // move each swap in front of the panel: swap rows t and p_t of the
      // multiplier columns computed before it (getrf's dlaswp on the left)
      for (int t = 0; t < PB; ++t) {
        const int pt = prel[t];
        if (pt != t && tid < t) {
          const double a = lt[t * PB + tid];
          lt[t * PB + tid] = lt[pt * PB + tid];
          lt[pt * PB + tid] = a;
        }
        __syncthreads();
      }
    }
    // D^{-1}: column c by forward substitution (thread c)
    if (tid < PB) {
      const int c = tid;
      for (int i = 0; i < PB; ++i) {
        double s = (i == c) ? 1.0 : 0.0;
        for (int k = 0; k < i; ++k) s = fma(-lt[i * PB + k], X[k * 17 + c], s);
        X[i * 17 + c] = FWD ? s : s * dinvd[i];
      }
    }
    __syncthreads();
    double* po = out + (long long)p * PS;
    if (tid < PB) po[tid] = (double)prel[tid];
    for (int e = tid; e < 256; e += blockDim.x) {  // D^{-1} fragments
      const int f = e >> 5, lane = e & 31, mt = f >> 2, ks = f & 3;
      po[16 + e] = X[(mt * 8 + (lane >> 2)) * 17 + ks * 4 + (lane & 3)];
    }
    __shared__ int s_mt;
    if (tid == 0) s_mt = 0;
    __syncthreads();
    int mt_hi = 0;  // highest nonzero m-tile of T (+1) seen by this thread
    for (int e = tid; e < 16 * kwp; e += blockDim.x) {  // -(T D^{-1}) fragments
      const int f = e >> 5, lane = e & 31, mt = f >> 2, ks = f & 3;
      const int r = PB + mt * 8 + (lane >> 2), c = ks * 4 + (lane & 3);
      double acc = 0.0;
      for (int k = 0; k < PB; ++k) acc = fma(lt[r * PB + k], X[k * 17 + c], acc);
      po[PREC_HDR + e] = -acc;
      if (lt[r * PB + c] != 0.0) mt_hi = max(mt_hi, mt + 1);  // T's own pattern decides
    }
    atomicMax(&s_mt, mt_hi);
    __syncthreads();
    if (tid == 0) mt_all[mtoff[blockIdx.x] + p] = (unsigned char)s_mt;
    __syncthreads();
  }
}

// ------------------------------------------------------------------ the panel solve
struct PanelArgs {
  const LocalDesc* descs;
  const long long* poff;   // [2 n_local]: forward / backward panel offsets per block
  const int* idx;
  const double* pf;
  const double* pb;
  const double* R;
  long long ldr;
  double* xs;
  long long xs_len;
  int nrhs, kwf, kwb, WR, stage_stride, ns;
  const unsigned char* pmt;  // per panel: nonzero m-tiles of T; block s: forward at mtoff[s], backward after
  const long long* mtoff;
  int np_max;                // most panels of a block (shared-memory copy of the counts)
};

struct PanelSweep {
  const PanelArgs* a;
  const int* idx;
  double* xs;
  double* W;
  const double* ring;
  uint64_t* full;
  uint64_t* empty;
  int n, kwp, WR, mtT;
  int* chunk;
  const unsigned char* mt;   // this sweep's per-panel m-tile counts (shared memory)
  const double* R;           // this CTA's first column of the batch
  int nr;                    // this CTA's column count (<= 8 NT)
};

template <bool FWD>
__device__ __forceinline__ double panel_in(const PanelSweep& S, int row, int c) {
  if (row >= S.n || c >= S.nr) return 0.0;
  if (FWD) return __ldg(S.R + (long long)c * S.a->ldr + __ldg(S.idx + row));
  return S.xs[(long long)c * S.a->xs_len + (S.n - 1 - row)];
}

// the gather split in two: the index (loaded a further PD panels ahead, so
// that the value load never waits on it) and the value
__device__ __forceinline__ int panel_idx(const PanelSweep& S, int row) { return row < S.n ? __ldg(S.idx + row) : -1; }

template <bool FWD>
__device__ __forceinline__ double panel_val(const PanelSweep& S, int row, int c, int gi) {
  if (row >= S.n || c >= S.nr) return 0.0;
  if (FWD) return __ldg(S.R + (long long)c * S.a->ldr + gi);
  return S.xs[(long long)c * S.a->xs_len + (S.n - 1 - row)];
}

// window row (j0 + off) for 0 <= off < WR, given base = j0 mod WR
template <int NT>
__device__ __forceinline__ double* panel_row(const PanelSweep& S, int base, int off) {
  int r = base + off;
  if (r >= S.WR) r -= S.WR;
  return S.W + (size_t)r * PanelCols<NT>::PSR;
}

// One panel p.  `ev` is this panel's slot of the entering-row look-ahead: it
// holds the value loaded PD panels ago (stored into the window here) and is
// refilled for panel p + PD — a fixed register per slot (the caller unrolls
// PD panels), so no in-flight load is ever moved between registers.
template <bool FWD, int NT>
__device__ __forceinline__ void panel_step(const PanelSweep& S, int p, double& ev, int& ei) {
  constexpr int NC = PanelCols<NT>::NC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = lane & 3, g = lane >> 2;
  const int er = tid / NC, ec = tid % NC;
  const bool eact = tid < PB * NC;  // threads that carry an entering-row element
  const int kwp = S.kwp;
  const int j0 = p * PB;
  const int base = j0 % S.WR;
  const double evc = ev;
  const int erow = j0 + PB + kwp + er;
  if (eact) {
    ev = panel_val<FWD>(S, erow + PB * PD, ec, ei);     // value for panel p + PD (its index loaded PD panels ago)
    if (FWD) ei = panel_idx(S, erow + 2 * PB * PD);     // index for panel p + 2 PD
  }
  const int chunk = *S.chunk;
  const int ns = S.a->ns;
  const int stage = chunk % ns;
  mbar_wait(&S.full[stage], (chunk / ns) & 1);
  const double* rec = S.ring + (size_t)stage * S.a->stage_stride;
  const int mtp = S.mt[p];  // nonzero m-tiles of this panel's T
  if (FWD) {  // the panel's row interchanges, moved to its front (every thread reads the same 16 pivots)
    bool any = false;
    const double2* pv = reinterpret_cast<const double2*>(rec);
#pragma unroll
    for (int t = 0; t < PB / 2; ++t) {
      const double2 v = pv[t];
      any |= (v.x != (double)(2 * t)) | (v.y != (double)(2 * t + 1));
    }
    if (any) {
      if (warp == 0) {
        for (int t = 0; t < PB; ++t) {
          const int p2 = __double2int_rn(rec[t]);
          if (p2 != t && lane < NC) {
            double* r1 = panel_row<NT>(S, base, t);
            double* r2 = panel_row<NT>(S, base, p2);
            const double tmp = r1[lane];
            r1[lane] = r2[lane];
            r2[lane] = tmp;
          }
          __syncwarp();
        }
      }
      psync();
    }
  }
  // B fragments: the panel rows (the one operand of both products)
  double b0[4], b1[4];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const double* wr = panel_row<NT>(S, base, ks * 4 + q);
    b0[ks] = wr[g];
    b1[ks] = NT == 2 ? wr[8 + g] : 0.0;
  }
  // tiles (m-tile t / NT, n-tile t % NT): m-tiles 0, 1 = X = D^{-1} W; 2.. = trailing rows
  // += -(T D^{-1}) W.  Warp w takes tiles w, w+8, ... (all of the same n-tile), at most
  // TG of them, k-steps interleaved across its tiles.
  const int ntile = NT * (2 + mtp);
  constexpr int TG = 5;
  const double* bsel = (NT == 2 && (warp & 1)) ? b1 : b0;
  // groups of TG tiles per warp (one group while ntile <= 40, i.e. kw <= 144)
  for (int t0 = warp; t0 < ntile; t0 += 8 * TG) {
    const int nu = min(TG, (ntile - t0 + 7) >> 3);  // tiles of this warp in this group
    double acc[TG][2];
    const double* ap[TG];
    double* crow[TG];
#pragma unroll
    for (int u = 0; u < TG; ++u) {
      const int t = t0 + 8 * u;
      acc[u][0] = acc[u][1] = 0.0;
      crow[u] = nullptr;
      ap[u] = rec + lane;
      if (u < nu) {
        const int tm = t / NT, tn = t % NT;
        if (tm < 2) {
          ap[u] = rec + 16 + tm * 128 + lane;
        } else {
          const int mt = tm - 2;
          ap[u] = rec + PREC_HDR + mt * 128 + lane;
          crow[u] = panel_row<NT>(S, base, PB + mt * 8 + g) + tn * 8 + 2 * q;
          const double2 c2 = *reinterpret_cast<const double2*>(crow[u]);
          acc[u][0] = c2.x;
          acc[u][1] = c2.y;
        }
      }
    }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int u = 0; u < TG; ++u)
        if (u < nu) dmma_p(acc[u], ap[u][ks * 32], bsel[ks]);
    }
#pragma unroll
    for (int u = 0; u < TG; ++u) {
      if (u >= nu) continue;
      const int t = t0 + 8 * u;
      if (t < 2 * NT) {
        const int r = (t / NT) * 8 + g, c = (t % NT) * 8 + 2 * q;
        double* xs = S.xs + (FWD ? (long long)(j0 + r) : (long long)(S.n - 1 - (j0 + r)));
        if (j0 + r < S.n) {
          if (c < S.nr) xs[(long long)c * S.a->xs_len] = acc[u][0];
          if (c + 1 < S.nr) xs[(long long)(c + 1) * S.a->xs_len] = acc[u][1];
        }
      } else {
        *reinterpret_cast<double2*>(crow[u]) = make_double2(acc[u][0], acc[u][1]);
      }
    }
  }
  // entering rows take the slots of the previous panel (finished)
  if (eact) panel_row<NT>(S, base, PB + kwp + er)[ec] = evc;
  psync();
  if (tid == 0) mbar_arrive(&S.empty[stage]);
  *S.chunk = chunk + 1;
}

template <bool FWD, int NT>
__device__ __forceinline__ void panel_sweep(const PanelArgs& a, const LocalDesc& d, double* ring, uint64_t* full,
                                            uint64_t* empty, double* W, int& chunk, int c0) {
  constexpr int NC = PanelCols<NT>::NC;
  const int tid = threadIdx.x;
  const unsigned char* smt = reinterpret_cast<const unsigned char*>(W + (size_t)a.WR * PanelCols<NT>::PSR);
  PanelSweep S{&a, a.idx + d.idx_off, a.xs + d.idx_off + (long long)c0 * a.xs_len, W, ring, full, empty, d.n,
               FWD ? a.kwf : a.kwb, a.WR, 0, &chunk, smt + (FWD ? 0 : (d.n + PB - 1) / PB),
               a.R + (long long)c0 * a.ldr, min(NC, a.nrhs - c0)};
  S.mtT = S.kwp >> 3;
  const int np = (S.n + PB - 1) / PB;
  // prologue: panel 0 and its trailing rows
  for (int e = tid; e < (PB + S.kwp) * NC; e += 256) panel_row<NT>(S, 0, e / NC)[e % NC] = panel_in<FWD>(S, e / NC, e % NC);
  // rows entering at panels 0..PD-1, in flight ahead of their use (this
  // thread's row tid / 16, column tid % 16 of each 16-row group)
  const int er = tid / NC, ec = tid % NC;
  const bool eact = tid < PB * NC;
  const int r0 = PB + S.kwp + er;
  double ev0 = eact ? panel_in<FWD>(S, r0, ec) : 0.0;
  double ev1 = eact ? panel_in<FWD>(S, r0 + PB, ec) : 0.0;
  double ev2 = eact ? panel_in<FWD>(S, r0 + 2 * PB, ec) : 0.0;
  double ev3 = eact ? panel_in<FWD>(S, r0 + 3 * PB, ec) : 0.0;
  int ei0 = 0, ei1 = 0, ei2 = 0, ei3 = 0;  // gather indices of panels 4..7 (forward sweep)
  if (FWD && eact) {
    ei0 = panel_idx(S, r0 + 4 * PB);
    ei1 = panel_idx(S, r0 + 5 * PB);
    ei2 = panel_idx(S, r0 + 6 * PB);
    ei3 = panel_idx(S, r0 + 7 * PB);
  }
  static_assert(PD == 4, "unrolled look-ahead slots");
  psync();
  for (int p = 0; p < np; p += PD) {
    panel_step<FWD, NT>(S, p, ev0, ei0);
    if (p + 1 < np) panel_step<FWD, NT>(S, p + 1, ev1, ei1);
    if (p + 2 < np) panel_step<FWD, NT>(S, p + 2, ev2, ei2);
    if (p + 3 < np) panel_step<FWD, NT>(S, p + 3, ev3, ei3);
  }
}

// NT = 2: one CTA per block, 16 columns.  NT = 1: two CTAs per block, 8 columns each (the columns
// are independent; the second read of the panel records comes from L2) — for decompositions with
// fewer blocks than SMs.
template <int NT>
__global__ void __launch_bounds__(PTHREADS, 2) k_local_panel(PanelArgs a) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[PNS_MAX], empty[PNS_MAX];
  const int ns = a.ns;
  const int blk = NT == 2 ? blockIdx.x : blockIdx.x >> 1;
  const int c0 = NT == 2 ? 0 : 8 * (blockIdx.x & 1);
  if (c0 >= a.nrhs) return;
  const LocalDesc d = a.descs[blk];
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  if (d.n == 0) return;
  const int np = (d.n + PB - 1) / PB;
  // per-panel m-tile counts of both sweeps into shared memory (after the window)
  unsigned char* smt =
      reinterpret_cast<unsigned char*>(sm + (size_t)ns * a.stage_stride + (size_t)a.WR * PanelCols<NT>::PSR);
  for (int e = threadIdx.x; e < 2 * np; e += blockDim.x) smt[e] = a.pmt[a.mtoff[blk] + e];
  __syncthreads();
  if (threadIdx.x >= 256) {
    if (threadIdx.x == 256) {  // producer: forward panels, then backward panels (used part only)
      const long long psf = panel_doubles(a.kwf), psb = panel_doubles(a.kwb);
      for (int c = 0; c < 2 * np; ++c) {
        const int stage = c % ns;
        if (c >= ns) mbar_wait(&empty[stage], ((c / ns) - 1) & 1);
        const bool f = c < np;
        const int pp = f ? c : c - np;
        const double* src = f ? a.pf + a.poff[2 * blk] + pp * psf : a.pb + a.poff[2 * blk + 1] + pp * psb;
        const uint32_t bytes = (uint32_t)(panel_used(smt[c]) * 8);
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(sm + (size_t)stage * a.stage_stride, src, bytes, &full[stage]);
      }
    }
    return;
  }
  double* W = sm + (size_t)ns * a.stage_stride;
  int chunk = 0;
  panel_sweep<true, NT>(a, d, sm, full, empty, W, chunk, c0);
  panel_sweep<false, NT>(a, d, sm, full, empty, W, chunk, c0);
}

// ------------------------------------------------------------------ host side
static int round8(int x) { return (x + 7) / 8 * 8; }

template <typename T>
static int dev_upload(T** dptr, const T* host, size_t count, long long* bytes) {
  HG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dptr), sizeof(T) * std::max<size_t>(count, 1)));
  if (host && count) HG_CUDA_TRY(cudaMemcpy(*dptr, host, sizeof(T) * count, cudaMemcpyHostToDevice));
  if (bytes) *bytes += (long long)(sizeof(T) * count);
  return HG_OK;
}

// batched local solves: panels when prepared and checked, else the row kernel
int launch_local_batch(HgPrecond* P, const double* R, long long ldr, int nrhs, cudaStream_t st) {
  if (P->panel_ok)
    HG_TRY(launch_local_panel(P, R, ldr, nrhs, st));
  else
    HG_TRY(launch_local_solve_multi(P, R, ldr, nrhs, st));
  return launch_split_stages(P, R, ldr, P->d_xsm, P->xs_len, nrhs, st);  // split subdomains: separators, spikes
}

// ring stages: as many as fit beside the window with two CTAs per SM (at least
// 3), HG_PANEL_STAGES overrides (up to PNS_MAX; experiments)
static int panel_stages(const HgPrecond* P) {
  const long long ss = std::max(panel_doubles(P->panel_kwf), panel_doubles(P->panel_kwb)) * 8;
  const long long win = (long long)P->panel_wr * PanelCols<2>::PSR * 8;
  static const int env = getenv("HG_PANEL_STAGES") ? atoi(getenv("HG_PANEL_STAGES")) : 0;
  if (env > 0) return std::min(env, PNS_MAX);
  const long long budget = 113 * 1024 - 256 - 2 * P->panel_np_max;  // two CTAs per SM
  return (int)std::max(3LL, std::min((long long)PNS_MAX, (budget - win) / ss));
}

static size_t panel_smem(const HgPrecond* P) {
  const long long ss = std::max(panel_doubles(P->panel_kwf), panel_doubles(P->panel_kwb));
  return sizeof(double) * ((size_t)panel_stages(P) * ss + (size_t)P->panel_wr * PanelCols<2>::PSR) +
         (size_t)((2 * P->panel_np_max + 15) / 16 * 16);
}

int launch_local_panel(HgPrecond* P, const double* R, long long ldr, int nrhs, cudaStream_t st) {
  if (P->n_local == 0) return HG_OK;
  const size_t smem = panel_smem(P);
  // column split: two CTAs per block (8 columns each) while every CTA still has an SM to itself
  // (measured: two column-split CTAs sharing an SM are slower than one 16-column CTA);
  // HG_PANEL_CSPLIT=0/1 overrides
  static const int env = getenv("HG_PANEL_CSPLIT") ? atoi(getenv("HG_PANEL_CSPLIT")) : -1;
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int nblk = 0;  // blocks with rows (separator pseudo blocks of split subdomains have none)
  for (const LocalDesc& d : P->h_local) nblk += d.n > 0;
  const bool split = nrhs > 8 && (env >= 0 ? env != 0 : 2 * nblk <= sms);
  const void* fn = split ? reinterpret_cast<const void*>(k_local_panel<1>)
                         : reinterpret_cast<const void*>(k_local_panel<2>);
  HG_TRY(ensure_func_attrs(fn, smem, false));
  PanelArgs a{P->d_local, P->d_poff, P->d_local_idx, P->d_pfwd, P->d_pbwd, R, ldr, P->d_xsm, P->xs_len, nrhs,
              P->panel_kwf, P->panel_kwb, P->panel_wr,
              (int)std::max(panel_doubles(P->panel_kwf), panel_doubles(P->panel_kwb)), panel_stages(P),
              P->d_pmt, P->d_mtoff, P->panel_np_max};
  if (split)
    k_local_panel<1><<<2 * P->n_local, PTHREADS, smem, st>>>(a);
  else
    k_local_panel<2><<<P->n_local, PTHREADS, smem, st>>>(a);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

__global__ void k_fill_hash(long long n, double* y, unsigned seed) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull + seed;
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 27;
    y[i] = (double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}

// Build the panel records from the row records (device) and check the panel
// solve against the row solve on a seeded batch; keep it only if they agree
// to 1e-11 (relative to each column's largest entry).
int prepare_local_panel(HgPrecond* P) {
  P->panel_ok = false;
  P->panel_dev = -1.0;
  const char* env = getenv("HG_LOCAL_PANEL");
  if (P->n_local == 0 || (env && env[0] == '0')) return HG_OK;
  int kwf = 0, kwb = 0;
  for (const LocalDesc& d : P->h_local) {
    kwf = std::max(kwf, d.kl);
    kwb = std::max(kwb, d.kv);
  }
  P->panel_kwf = round8(kwf);
  P->panel_kwb = round8(kwb);
  P->panel_wr = 2 * PB + std::max(P->panel_kwf, P->panel_kwb);
  if (panel_smem(P) > 227 * 1024) return HG_OK;  // window too wide for shared memory: row kernel only
  std::vector<long long> poff(2 * P->n_local), mtoff(P->n_local), mtoff_b(P->n_local);
  long long pf = 0, pb = 0, pm = 0;
  P->panel_np_max = 0;
  for (int s = 0; s < P->n_local; ++s) {
    const long long np = (P->h_local[s].n + PB - 1) / PB;
    poff[2 * s] = pf;
    poff[2 * s + 1] = pb;
    mtoff[s] = pm;
    mtoff_b[s] = pm + np;
    pm += 2 * np;
    pf += np * panel_doubles(P->panel_kwf);
    pb += np * panel_doubles(P->panel_kwb);
    P->panel_np_max = std::max(P->panel_np_max, (int)np);
  }
  HG_TRY(dev_upload(&P->d_poff, poff.data(), poff.size(), &P->device_bytes));
  // per-sweep offsets for the two conversion launches (temporaries)
  std::vector<long long> pof(P->n_local), pob(P->n_local);
  for (int s = 0; s < P->n_local; ++s) {
    pof[s] = poff[2 * s];
    pob[s] = poff[2 * s + 1];
  }
  long long *d_pof = nullptr, *d_pob = nullptr;
  HG_TRY(dev_upload(&d_pof, pof.data(), pof.size(), nullptr));
  HG_TRY(dev_upload(&d_pob, pob.data(), pob.size(), nullptr));
  HG_TRY(dev_upload<double>(&P->d_pfwd, nullptr, (size_t)pf, &P->device_bytes));
  HG_TRY(dev_upload<double>(&P->d_pbwd, nullptr, (size_t)pb, &P->device_bytes));
  HG_TRY(dev_upload<unsigned char>(&P->d_pmt, nullptr, (size_t)pm, &P->device_bytes));
  HG_TRY(dev_upload(&P->d_mtoff, mtoff.data(), mtoff.size(), &P->device_bytes));
  long long* d_mtoff_b = nullptr;
  HG_TRY(dev_upload(&d_mtoff_b, mtoff_b.data(), mtoff_b.size(), nullptr));
  const size_t cf = sizeof(double) * ((PB + P->panel_kwf) * PB + PB + PB * 17);
  const size_t cb = sizeof(double) * ((PB + P->panel_kwb) * PB + PB + PB * 17);
  HG_TRY(ensure_func_attrs(reinterpret_cast<const void*>(k_panel_convert<true>), cf, false));
  HG_TRY(ensure_func_attrs(reinterpret_cast<const void*>(k_panel_convert<false>), cb, false));
  k_panel_convert<true><<<P->n_local, 128, cf>>>(P->d_local, P->d_fwd, d_pof, P->panel_kwf, P->d_pfwd, P->d_mtoff,
                                                   P->d_pmt);
  HG_LAUNCH_CHECK();
  k_panel_convert<false><<<P->n_local, 128, cb>>>(P->d_local, P->d_bwd, d_pob, P->panel_kwb, P->d_pbwd, d_mtoff_b,
                                                    P->d_pmt);
  HG_LAUNCH_CHECK();
  HG_CUDA_TRY(cudaDeviceSynchronize());
  cudaFree(d_pof);
  cudaFree(d_pob);
  cudaFree(d_mtoff_b);
  {  // bytes one batched local solve streams (hg_precond_stat)
    std::vector<unsigned char> mt((size_t)pm);
    HG_CUDA_TRY(cudaMemcpy(mt.data(), P->d_pmt, mt.size(), cudaMemcpyDeviceToHost));
    long long used = 0;
    for (unsigned char v : mt) used += panel_used(v);
    P->panel_stream_bytes = 8 * used;
  }

  // guard: panel vs row solve on a seeded 16-column batch
  const int nr = HG_MAX_RHS;
  const long long nn = (long long)nr * P->n;
  double *d_r = nullptr, *d_ref = nullptr;
  HG_CUDA_TRY(cudaMalloc(&d_r, sizeof(double) * nn));
  HG_CUDA_TRY(cudaMalloc(&d_ref, sizeof(double) * (size_t)nr * P->xs_len));
  k_fill_hash<<<ceil_div(nn, 256), 256>>>(nn, d_r, 2406u);
  int s = launch_local_solve_multi(P, d_r, P->n, nr, 0);
  if (s == HG_OK && cudaMemcpy(d_ref, P->d_xsm, sizeof(double) * (size_t)nr * P->xs_len, cudaMemcpyDeviceToDevice) !=
                        cudaSuccess)
    s = HG_ERR_CUDA;
  if (s == HG_OK) s = launch_local_panel(P, d_r, P->n, nr, 0);
  std::vector<double> ref, got;
  if (s == HG_OK) {
    ref.resize((size_t)nr * P->xs_len);
    got.resize(ref.size());
    if (cudaMemcpy(ref.data(), d_ref, sizeof(double) * ref.size(), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(got.data(), P->d_xsm, sizeof(double) * got.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
      s = HG_ERR_CUDA;
  }
  cudaFree(d_r);
  cudaFree(d_ref);
  if (s != HG_OK) {
    set_error("local panel guard failed to run");
    return HG_ERR_CUDA;
  }
  double dev = 0.0;
  for (int c = 0; c < nr; ++c) {
    double mx = 0.0, df = 0.0;
    for (long long i = 0; i < P->xs_len; ++i) {
      const double a = ref[(size_t)c * P->xs_len + i], b = got[(size_t)c * P->xs_len + i];
      mx = std::max(mx, std::fabs(a));
      df = std::max(df, std::fabs(a - b));
      if (std::isnan(b)) df = INFINITY;
    }
    dev = std::max(dev, mx > 0.0 ? df / mx : df);
  }
  P->panel_dev = dev;
  P->panel_ok = dev <= 1e-11;
  return HG_OK;
}

int preload_local_panel() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_local_panel<1>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_local_panel<2>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_panel_convert<true>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_panel_convert<false>));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_fill_hash));
  return HG_OK;
}

}  // namespace hg
