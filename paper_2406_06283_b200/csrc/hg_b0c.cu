// K3 (cluster variant): coarse solve y = B0^{-1} c on ONE thread-block
// cluster of CS <= 16 CTAs with distributed shared memory.
//
// Factors: the tiled getrf factors of factor.pack_b0_tiles with every
// off-diagonal tile premultiplied by its panel's inverse diagonal block,
// M[t, j] = D_t^{-1} T[t, j]  (factor.premultiply_tiles), so that
//     x_t = D_t^{-1} rhs_t - sum_j M[t, j] x_j        (j ascending)
// and every row of a panel finishes on its own: no block-wide reduction sits
// between two panels.  The critical hand-off per panel is one 64x64 tile
// GEMV against the freshly received x_{t-1}.
//
// Hand-off: every CTA keeps a ring of the NR most recent panels in shared
// memory as 16-byte (value, panel tag) pairs.  The row group that finishes
// x_t[row] stores its pair straight into the ring of the owner of panel t+1
// first (st.shared::cluster.v2), then of every other CTA; consumers spin on
// their local copies until the tags read t.  No fences or barriers are on
// the critical path; each 16-byte pair is written and read as one access.
// Panels are published in order (a row is published only after the
// publishing row group has seen all of x_{t-1}), hence a ring slot is
// rewritten only after every panel that could read it is complete (the host
// guarantees NR >= largest tile distance + CS).
// Tiles stream through a TMA bulk-copy ring (producer warp).  Their 16-byte
// chunks are XOR-swizzled by row parity so that the 4-threads-per-row GEMV
// reads shared memory without bank conflicts.
// The L -> U transition (the U right-hand side is the reversed L solution,
// read from global memory) is ordered by one cluster-scope mbarrier.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hg_internal.cuh"

namespace hg {

// timing experiments only (HG_B0_STAMPS=1): per panel {start, x_{t-1} seen,
// -, published} SM cycle stamps
__device__ int g_b0c_stamp_on = 0;
__device__ unsigned long long g_b0c_stamps[8192 * 4];
__device__ __forceinline__ unsigned long long gtimer_b0c() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

namespace {

constexpr int CP = 64;             // panel size
constexpr int CONS = 256;          // consumer threads (64 rows x 4)
constexpr int CTHREADS = CONS + 32;
constexpr int TNS = 4;             // tile ring stages at most (runtime count B0ClusterArgs::tns, 2..4)
constexpr int TILE_DOUBLES = CP * CP;

__device__ __forceinline__ uint32_t mapa(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void st_cluster_f64x2(uint32_t addr, double v, double tag) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v), "d"(tag) : "memory");
}

__device__ __forceinline__ double2 ld_volatile_f64x2(const double* p) {
  double2 r;
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(smem_u32(p)) : "memory");
  return r;
}

__device__ __forceinline__ void arrive_remote(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(CONS) : "memory");
}

// chunk (16 bytes = 2 doubles) c of row r lives at physical chunk c ^ ((r & 1) << 2)
__device__ __forceinline__ int swz(int row, int c) { return c ^ ((row & 1) << 2); }

// Entries 2(q+4k), 2(q+4k)+1 (k = 0..7) of panel g from the tagged ring;
// spins until all 16 tags read g.  The 4 threads of a row group together
// cover all CP entries.
__device__ __forceinline__ void poll_panel(const double* xring, int g, int NR, int q, double (&xv)[16],
                                           const SpinCfg& spin, bool& dead) {
  const double* slot = xring + (size_t)(g % NR) * CP * 2;
  const double tag = (double)g;
  bool ok;
  SpinGuard sg;
  do {
    ok = true;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = 2 * (q + 4 * k);
      const double2 p0 = ld_volatile_f64x2(slot + 2 * e);
      const double2 p1 = ld_volatile_f64x2(slot + 2 * (e + 1));
      xv[2 * k] = p0.x;
      xv[2 * k + 1] = p1.x;
      ok = ok && (p0.y == tag) && (p1.y == tag);
    }
    if (!ok && (dead || spin_abort(sg, spin))) {  // bounded: a faulted handle finishes on garbage
      dead = true;
      ok = true;
    }
  } while (!__all_sync(FULL, ok));
}

// this row's partial of (tile row) . (vector): 4 chains, then the row group's sum
__device__ __forceinline__ double row_dot(const double* trow, int row, int q, const double (&xv)[16]) {
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 tv = *reinterpret_cast<const double2*>(trow + 2 * swz(row, q + 4 * k));
    s4[(2 * k) & 3] = fma(tv.x, xv[2 * k], s4[(2 * k) & 3]);
    s4[(2 * k + 1) & 3] = fma(tv.y, xv[2 * k + 1], s4[(2 * k + 1) & 3]);
  }
  double s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  s += __shfl_xor_sync(FULL, s, 1);
  s += __shfl_xor_sync(FULL, s, 2);
  return s;
}

}  // namespace

struct B0ClusterArgs {
  int m, K, NR, CS;
  int tns;                  // tile ring stages (fewer = less shared memory: a local-solve CTA fits beside)
  const int* perm;
  const int* col_blk;
  const CblkDesc* descs;
  const double* cpart;
  const double* dinv;       // swizzled [2K][P][P]
  const long long* tile_ptr;
  const int* tile_col;
  const double* tiles;      // swizzled, premultiplied [ntile][P][P]
  double* xbuf;             // [2][K*P] global copy of the solved panels
  double* y;
  const unsigned long long* blk_done;  // per coarse block Z^T r chunk counters
  unsigned long long* ticket;          // launch L (take_launch_index) reads Z^T r launch L:
                                       // block b of c is complete at (L + 1) nchunk_b
  SpinCfg spin;
};

__global__ void __launch_bounds__(CTHREADS, 1) k_b0_cluster(B0ClusterArgs a) {
  extern __shared__ __align__(128) double sm[];
  double* tring = sm;                                   // TNS x TILE_DOUBLES
  const int tns = a.tns;
  double* xring = tring + (size_t)tns * TILE_DOUBLES;   // NR x CP (value, tag) pairs
  double* rhs = xring + (size_t)a.NR * CP * 2;          // CP
  uint64_t* tfull = reinterpret_cast<uint64_t*>(rhs + CP);
  uint64_t* tempty = tfull + TNS;
  uint64_t* ldone = tempty + TNS;                       // the whole L solve is in global memory

  __shared__ unsigned long long s_launch;
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_rank();
  const int CS = a.CS, K = a.K, NR = a.NR;
  for (int i = tid; i < NR * CP; i += CTHREADS) xring[2 * i + 1] = -1.0;  // no panel yet
  if (tid == 0) {
    s_launch = take_launch_index(a.ticket, CS);
    for (int s = 0; s < tns; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], CONS / 32);
    }
    mbar_init(ldone, CS);
    fence_mbar_init();
  }
  __syncthreads();
  cluster_sync_all();  // initialised rings and barriers before any remote access

  if (tid >= CONS) {
    // ---- producer warp: per own panel, the inverse block then the tiles
    if (tid == CONS) {
      int c = 0, stage = 0, epar = 1;  // epar: parity of the previous pass over the ring
      for (int g = rank; g < 2 * K; g += CS) {
        const long long e0 = a.tile_ptr[g], e1 = a.tile_ptr[g + 1];
        for (long long e = e0 - 1; e < e1; ++e, ++c, ++stage) {  // e == e0 - 1: the inverse block
          if (stage == tns) {
            stage = 0;
            epar ^= 1;
          }
          if (c >= tns) mbar_wait(&tempty[stage], epar);
          const double* src = (e < e0) ? a.dinv + (size_t)g * TILE_DOUBLES : a.tiles + (size_t)e * TILE_DOUBLES;
          mbar_arrive_expect_tx(&tfull[stage], TILE_DOUBLES * 8u);
          bulk_g2s(tring + (size_t)stage * TILE_DOUBLES, src, TILE_DOUBLES * 8u, &tfull[stage]);
        }
      }
    }
  } else {
    // ---- consumers: 64 rows x 4 threads; thread q owns chunks q + 4k (k = 0..7)
    const int row = tid >> 2, q = tid & 3, lane = tid & 31;
    int stage = 0, fpar = 0;  // tile-stream position: ring stage and its parity (no division: runtime tns)
    auto next_tile = [&]() {
      if (++stage == tns) {
        stage = 0;
        fpar ^= 1;
      }
    };
    bool l_done = false;
    bool dead = false;  // a bounded wait gave up: finish on garbage, the host reports the fault
    const unsigned long long zt_launches = s_launch + 1;
    for (int g = rank; g < 2 * K; g += CS) {
      const int ph = g / K, t = g % K;
      const bool stamp = g_b0c_stamp_on && tid == 0 && g < 8192;
      if (stamp) g_b0c_stamps[4 * g] = clock64();
      // right-hand side of the panel: P c (L phase) or the reversed L solution (U phase)
      consumers_sync();  // rhs[] of the previous panel fully consumed
      if (ph == 0) {
        const int i = t * CP + row;
        if (q == 0) {
          double v = 0.0;
          if (i < a.m) {
            // this kernel is launched before Z^T r: wait for this row's coarse block only
            const int col = a.perm[i];
            const int b = a.col_blk[col];
            const CblkDesc d = a.descs[b];
            const unsigned long long need = zt_launches * (unsigned long long)d.nchunk;
            SpinGuard sg;
            while (!dead && ld_acquire_gpu_u64(a.blk_done + b) < need)
              if (spin_abort(sg, a.spin)) dead = true;
            const int l = col - d.col0;
            for (int ch = 0; ch < d.nchunk; ++ch) v += a.cpart[d.part_off + (long long)ch * d.m + l];
          }
          rhs[row] = v;
        }
      } else {
        if (!l_done) {
          mbar_wait_cluster(ldone, 0);  // every CTA stored its L panels
          l_done = true;
        }
        if (q == 0) rhs[row] = a.xbuf[(size_t)K * CP - 1 - (t * CP + row)];
      }
      consumers_sync();
      double xv[16];
      {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double2 r2 = *reinterpret_cast<const double2*>(rhs + 2 * (q + 4 * k));
          xv[2 * k] = r2.x;
          xv[2 * k + 1] = r2.y;
        }
      }
      mbar_wait(&tfull[stage], fpar);
      double acc = row_dot(tring + (size_t)stage * TILE_DOUBLES + row * CP, row, q, xv);  // D_t^{-1} rhs_t
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[stage]);
      next_tile();
      const long long e0 = a.tile_ptr[g], e1 = a.tile_ptr[g + 1];
      bool saw_prev = (g == 0) || (ph == 1 && t == 0);
      for (long long e = e0; e < e1; ++e, next_tile()) {
        const int gj = ph * K + a.tile_col[e];
        if (stamp && gj == g - 1) g_b0c_stamps[4 * g + 1] = gtimer_b0c();
        poll_panel(xring, gj, NR, q, xv, a.spin, dead);
        if (gj == g - 1) {
          saw_prev = true;
          if (stamp) g_b0c_stamps[4 * g + 2] = gtimer_b0c();
        }
        mbar_wait(&tfull[stage], fpar);
        acc -= row_dot(tring + (size_t)stage * TILE_DOUBLES + row * CP, row, q, xv);
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[stage]);
      }
      // in-order publication: this row group has seen all of x_{g-1}
      if (!saw_prev) poll_panel(xring, g - 1, NR, q, xv, a.spin, dead);
      const uint32_t slot_addr = smem_u32(xring + ((size_t)(g % NR) * CP + row) * 2);
      const uint32_t nxt = (rank + 1) % CS;
      const double tag = (double)g;
      if (q == 0) {
        st_cluster_f64x2(mapa(slot_addr, nxt), acc, tag);
        if (nxt != rank) st_cluster_f64x2(mapa(slot_addr, rank), acc, tag);
      }
      if (stamp) { g_b0c_stamps[4 * g + 3] = clock64(); g_b0c_stamps[4 * g] = gtimer_b0c(); }
      for (int k = q; k < CS - 2; k += 4) st_cluster_f64x2(mapa(slot_addr, (rank + 2 + k) % CS), acc, tag);
      if (q == 0) {
        a.xbuf[(size_t)ph * K * CP + t * CP + row] = acc;
        if (ph == 1) {
          const int i = K * CP - 1 - (t * CP + row);
          if (i < a.m) a.y[i] = acc;
        }
      }
      // after this CTA's last L panel (global copies included): every CTA's ldone
      if (ph == 0 && g + CS >= K) {
        consumers_sync();
        if (tid < CS) arrive_remote(mapa(smem_u32(ldone), tid));
      }
    }
    // stay resident until every panel has been delivered here: the last
    // panel written into every ring slot
    for (int s2 = 0; s2 < NR && s2 < 2 * K; ++s2) {
      const int glast = s2 + ((2 * K - 1 - s2) / NR) * NR;
      double tmp[16];
      poll_panel(xring, glast, NR, q, tmp, a.spin, dead);
    }
  }
  __syncthreads();
  cluster_sync_all();
}

size_t b0_cluster_smem(int NR, int tns) {
  return sizeof(double) * ((size_t)tns * TILE_DOUBLES + (size_t)NR * CP * 2 + CP) +
         sizeof(uint64_t) * (2 * TNS + 1);
}

static int launch_chain(const B0ClusterArgs& a, cudaStream_t st) {
  const size_t smem = b0_cluster_smem(a.NR, a.tns);
  HG_TRY(ensure_func_attrs(reinterpret_cast<const void*>(k_b0_cluster), b0_cluster_smem(a.NR, TNS), true));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.CS);
  cfg.blockDim = dim3(CTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HG_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_b0_cluster, a));
  HG_LAUNCH_CHECK();
  return HG_OK;
}

// ---- bisected coarse solve (helmgpu.h "Bisected coarse solve"): separator stage, one warp per row
namespace {
__device__ __forceinline__ double warp_dot(const double* __restrict__ a, const double* __restrict__ x, int n, int lane) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = lane;
  for (; k + 96 < n; k += 128) {
    s0 = fma(__ldcs(a + k), __ldg(x + k), s0);
    s1 = fma(__ldcs(a + k + 32), __ldg(x + k + 32), s1);
    s2 = fma(__ldcs(a + k + 64), __ldg(x + k + 64), s2);
    s3 = fma(__ldcs(a + k + 96), __ldg(x + k + 96), s3);
  }
  for (; k < n; k += 32) s0 = fma(__ldcs(a + k), __ldg(x + k), s0);
  return warp_sum((s0 + s1) + (s2 + s3));
}
}  // namespace

// t = c_S - F [y[a - wl, a); y[a + ns, a + ns + wr)]; c_S from the Z^T r partials (fixed chunk order)
__global__ void __launch_bounds__(256) k_b0s_t(int ns, int wl, int wr, int a, const double* __restrict__ F,
                                               const double* __restrict__ y, const int* __restrict__ col_blk,
                                               const CblkDesc* __restrict__ descs, const double* __restrict__ cpart,
                                               double* __restrict__ t) {
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= ns) return;
  const double* f = F + (size_t)k * (wl + wr);
  const double s = warp_dot(f, y + a - wl, wl, lane) + warp_dot(f + wl, y + a + ns, wr, lane);
  if (lane == 0) {
    const CblkDesc d = descs[col_blk[a + k]];
    const int l = a + k - d.col0;
    double c = 0.0;
    for (int ch = 0; ch < d.nchunk; ++ch) c += cpart[d.part_off + (long long)ch * d.m + l];
    t[k] = c - s;
  }
}

// x_S = Sigma^{-1} t, written to y[a ..)
__global__ void __launch_bounds__(256) k_b0s_x(int ns, const double* __restrict__ Sinv, const double* __restrict__ t,
                                               double* __restrict__ ys) {
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= ns) return;
  const double s = warp_dot(Sinv + (size_t)k * ns, t, ns, lane);
  if (lane == 0) ys[k] = s;
}

// y_H -= W x_S (row r of W belongs to coarse unknown r for r < a, r + ns beyond)
__global__ void __launch_bounds__(256) k_b0s_w(int m, int ns, int a, const double* __restrict__ W, double* __restrict__ y) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= m - ns) return;
  const double s = warp_dot(W + (size_t)r * ns, y + a, ns, lane);
  const int i = r < a ? r : r + ns;
  if (lane == 0) y[i] -= s;
}

static B0ClusterArgs half_args(HgPrecond* P, int h) {
  const HgPrecond::B0Half& c = P->b0h[h];
  const int tns = P->b0_tns >= 2 && P->b0_tns <= TNS ? P->b0_tns : TNS;
  return B0ClusterArgs{c.m, c.K, c.nr, c.cs, tns, c.perm, P->d_col_blk, P->d_cblk, P->d_cpart, c.dinv,
                       c.tile_ptr, c.tile_col, c.tiles, c.xbuf, P->d_y + c.off,
                       P->d_blk_done, P->d_ticket + 2 + h, spin_cfg(P)};
}

// both half chains side by side (half 1 on the handle's second side stream), joined on st
int launch_coarse_chains_split(HgPrecond* P, cudaStream_t st) {
  HG_CUDA_TRY(cudaEventRecord(P->ev_c0, st));
  HG_CUDA_TRY(cudaStreamWaitEvent(P->aux2, P->ev_c0, 0));
  HG_TRY(launch_chain(half_args(P, 1), P->aux2));
  HG_CUDA_TRY(cudaEventRecord(P->ev_c1, P->aux2));
  HG_TRY(launch_chain(half_args(P, 0), st));
  HG_CUDA_TRY(cudaStreamWaitEvent(st, P->ev_c1, 0));
  return HG_OK;
}

// separator stage; the caller has ordered st after the whole Z^T r (c_S is read here)
int launch_coarse_sep_split(HgPrecond* P, cudaStream_t st) {
  const int ns = P->b0s_ns, a = P->b0s_a;
  k_b0s_t<<<ceil_div(ns, 8), 256, 0, st>>>(ns, P->b0s_wl, P->b0s_wr, a, P->d_b0s_f, P->d_y, P->d_col_blk, P->d_cblk,
                                           P->d_cpart, P->d_b0s_t);
  HG_LAUNCH_CHECK();
  k_b0s_x<<<ceil_div(ns, 8), 256, 0, st>>>(ns, P->d_b0s_sinv, P->d_b0s_t, P->d_y + a);
  HG_LAUNCH_CHECK();
  k_b0s_w<<<ceil_div(P->m - ns, 8), 256, 0, st>>>(P->m, ns, a, P->d_b0s_w, P->d_y);
  HG_LAUNCH_CHECK();
  return HG_OK;
}

int launch_coarse_solve_cluster(HgPrecond* P, cudaStream_t st) {
  if (P->b0_split_on) {  // serial contexts: Z^T r (or its stand-in) precedes on this stream
    HG_TRY(launch_coarse_chains_split(P, st));
    return launch_coarse_sep_split(P, st);
  }
  const int K = P->b0_K;
  const int CS = P->b0_cs;
  const int tns = P->b0_tns >= 2 && P->b0_tns <= TNS ? P->b0_tns : TNS;
  B0ClusterArgs a{P->m, K, P->b0_nr, CS, tns, P->d_b0_perm, P->d_col_blk, P->d_cblk, P->d_cpart, P->d_b0_dinv,
                  P->d_b0_tile_ptr, P->d_b0_tile_col, P->d_b0_tiles, P->d_b0_x, P->d_y,
                  P->d_blk_done, P->d_ticket, spin_cfg(P)};
  HG_TRY(launch_chain(a, st));
  static const bool stamps = getenv("HG_B0_STAMPS") != nullptr;
  if (stamps) {  // timing experiment: SM-cycle breakdown of the panel hand-off
    static bool armed = false;
    if (!armed) {
      int one = 1;
      HG_CUDA_TRY(cudaMemcpyToSymbol(g_b0c_stamp_on, &one, sizeof(int)));
      armed = true;
      return HG_OK;
    }
    HG_CUDA_TRY(cudaStreamSynchronize(st));
    const int n = 2 * K < 8192 ? 2 * K : 8192;
    std::vector<unsigned long long> h(4 * (size_t)n);
    HG_CUDA_TRY(cudaMemcpyFromSymbol(h.data(), g_b0c_stamps, sizeof(unsigned long long) * h.size()));
    double late = 0, transit = 0, comp = 0;
    int ct = 0;
    for (int g = 1; g < n; ++g) {
      if (h[4 * g + 2] == 0 || h[4 * g + 1] == 0) continue;
      const double pub_prev = (double)h[4 * (g - 1)], poll0 = (double)h[4 * g + 1], seen = (double)h[4 * g + 2];
      late += poll0 > pub_prev ? poll0 - pub_prev : 0.0;  // consumer reached the tile after the publish
      transit += seen - (poll0 > pub_prev ? poll0 : pub_prev);
      comp += (double)h[4 * g] - seen;
      ++ct;
    }
    fprintf(stderr, "[b0c stamps] K=%d CS=%d NR=%d (ns, %d hops): consumer late %.0f, transit %.0f, seen->published %.0f\n",
            K, CS, P->b0_nr, ct, late / ct, transit / ct, comp / ct);
    for (int g = 0; g < n; ++g) h[4 * g + 1] = 0;
    for (int g = 0; g < n; ++g) h[4 * g + 2] = 0;
    for (int g = 0; g < n; ++g) h[4 * g + 1] = 0;
    HG_CUDA_TRY(cudaMemcpyToSymbol(g_b0c_stamps, h.data(), sizeof(unsigned long long) * h.size()));
  }
  return HG_OK;
}

int preload_b0_cluster() {
  cudaFuncAttributes at;
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0_cluster));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0s_t));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0s_x));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_b0s_w));
  return HG_OK;
}

}  // namespace hg
