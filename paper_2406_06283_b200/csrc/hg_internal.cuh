// Internal device-side data structures and kernel launchers.
#pragma once
#include <vector>

#include "hg_common.cuh"

namespace hg {

// Global CSR on device (B and D_k share indptr/indices).
struct DevCsr {
  int n = 0;
  long long nnz = 0;
  int* indptr = nullptr;
  int* indices = nullptr;
  double* data = nullptr;    // B (or the single matrix of a generic op)
  double* data2 = nullptr;   // D_k (may be null)
};

struct LocalDesc {   // one fine subdomain block
  int n, kl, kv, fstride, bstride, pad;
  long long idx_off;   // into local_idx and the xs scratch
  long long fwd_off;   // doubles
  long long bwd_off;   // doubles
};

struct CblkDesc {    // one coarse (Z) block
  int n, m, col0, nchunk;
  long long idx_off;   // into cblk_idx and the zs scratch
  long long z_off;     // doubles
  long long part_off;  // into the Z^T r partials
};

struct SplitDesc {   // one split subdomain (helmgpu.h "Split local blocks")
  long long row0;      // first of its rows in the global separator numbering
  long long sep_pos;   // position of its separator unknowns in local_idx / the xs scratch
  long long sinv_off;  // Sigma^{-1} (ns x ns row-major), doubles
  int ns, pad;
};

struct SpikeDesc {   // spike block W_p of one chunk
  long long pos;       // the chunk's position in the xs scratch
  long long row0;      // first separator row of its split (global separator numbering)
  long long off;       // packed data, doubles
  int n, w, wtrue, col0;  // chunk rows; padded / true separator columns; first separator column
};

}  // namespace hg

struct HgPrecond {
  int n = 0;
  hg::DevCsr A;  // data = B, data2 = D_k

  // one-level part
  int n_local = 0;
  int rf = 0, rb = 0;            // register tiles (rows/32) of the two sweeps
  int ls_ns = 0;                 // ring stages of the row solve (0 = the default 6; hg_debug_set)
  int max_fstride = 0, max_bstride = 0;
  hg::LocalDesc* d_local = nullptr;
  std::vector<hg::LocalDesc> h_local;
  int* d_local_idx = nullptr;
  double* d_fwd = nullptr;
  double* d_bwd = nullptr;
  long long fwd_len = 0, bwd_len = 0;
  // 16-row panel records of the same factors for the batched solve (hg_local_panel.cu)
  long long* d_poff = nullptr;    // [2 n_local] forward / backward panel offsets
  double* d_pfwd = nullptr;
  double* d_pbwd = nullptr;
  int panel_kwf = 0, panel_kwb = 0, panel_wr = 0, panel_np_max = 0;
  unsigned char* d_pmt = nullptr;    // per panel: nonzero 8-row tiles of its trailing block
  long long* d_mtoff = nullptr;      // [n_local]: block s's counts (forward, then backward)
  long long panel_stream_bytes = 0;  // factor bytes one batched local solve streams
  bool panel_ok = false;          // panel records built and checked against the row solve
  double panel_dev = -1.0;        // that check's deviation (-1: not built)
  long long xs_len = 0;
  double* d_xs = nullptr;         // per-block local solutions (scratch)
  // dof -> local contributions (positions in xs), fixed (subdomain) order
  int* d_lptr = nullptr;
  long long* d_lent = nullptr;

  // split local blocks (hg_split.cu)
  int n_split = 0, split_ns_max = 0, n_spike_items1 = 0, n_spike_items2 = 0;
  hg::SplitDesc* d_split = nullptr;
  long long* d_split_fptr = nullptr;
  long long* d_split_fpos = nullptr;
  double* d_split_fval = nullptr;
  double* d_split_sinv = nullptr;
  hg::SpikeDesc* d_spike = nullptr;
  double* d_spike_data = nullptr;
  int2* d_spike_items1 = nullptr;   // (spike, 8-row tile)
  int2* d_spike_items2 = nullptr;   // (spike, pair of 8-row tiles)
  double* d_xsep = nullptr;         // [separator row][HG_MAX_RHS] compact x_S

  // bisected single-RHS coarse solve (hg_b0c.cu, helmgpu.h "Bisected coarse solve")
  struct B0Half {
    int m = 0, K = 0, nr = 0, cs = 0, off = 0;
    int* perm = nullptr;            // chain row -> global coarse column
    double* dinv = nullptr;
    long long* tile_ptr = nullptr;
    int* tile_col = nullptr;
    double* tiles = nullptr;
    double* xbuf = nullptr;
  };
  bool b0_split = false;            // bisected data present
  bool b0_split_on = false;         // ... and in use (hg_debug_set can switch it off)
  int b0_tns = 0;                   // tile ring stages of the chain kernel (0 = the default 4; hg_debug_set)
  B0Half b0h[2];
  int b0s_a = 0, b0s_ns = 0, b0s_wl = 0, b0s_wr = 0;
  double* d_b0s_f = nullptr;
  double* d_b0s_sinv = nullptr;
  double* d_b0s_w = nullptr;
  double* d_b0s_t = nullptr;
  cudaStream_t aux2 = nullptr;
  cudaEvent_t ev_c0 = nullptr, ev_c1 = nullptr, ev_zt = nullptr;

  // coarse part
  int m = 0;
  int n_cblk = 0;
  hg::CblkDesc* d_cblk = nullptr;
  std::vector<hg::CblkDesc> h_cblk;
  int* d_cblk_idx = nullptr;
  double* d_z = nullptr;
  long long part_len = 0;
  double* d_cpart = nullptr;      // Z^T r partial sums
  int* d_col_blk = nullptr;       // coarse column -> block
  int2* d_zt_items = nullptr;     // (block, row chunk) work items of Z^T r and Z y
  int n_zt_items = 0;
  int* d_b0_perm = nullptr;
  int b0_P = 0, b0_K = 0, b0_ctas = 32;   // panel size, panels per phase, persistent CTAs
  int b0_mode = 0;                        // 0: L2-counter kernel (hg_b0.cu), 1: cluster kernel (hg_b0c.cu)
  int b0_cs = 0, b0_nr = 0;               // cluster size, x ring slots (mode 1)
  double* d_b0_dinv = nullptr;            // [2][K][P][P]
  long long* d_b0_tile_ptr = nullptr;     // [2K+1]
  int* d_b0_tile_col = nullptr;
  double* d_b0_tiles = nullptr;           // [ntile][P][P]
  double* d_b0_x = nullptr;               // [2][K*P] phase solutions
  unsigned long long* d_b0_done = nullptr;  // monotone panel completion counter (mode 0: 2K per launch)
  unsigned long long* d_zt_done = nullptr;  // monotone count of finished single-RHS Z^T r chunks
  unsigned long long* d_blk_done = nullptr; // per coarse block: monotone count of its finished single-RHS Z^T r chunks
  unsigned long long* d_blkm_done = nullptr;  // the same for the batched Z^T R
  // device tickets of the coarse solves ([0] single, [1] batched): the L-th
  // coarse launch waits for the (L+1)-th Z^T r launch (take_launch_index);
  // nothing about the pairing lives on the host, so CUDA-graph replays and
  // eager calls interleave safely
  unsigned long long* d_ticket = nullptr;
  // bounded waits: pinned, host-mapped fault word (hg_common.cuh SpinGuard);
  // nonzero = a wait timed out or a launch failed mid-apply: the handle is
  // poisoned and every later call fails with HG_ERR_CUDA
  int* h_fault = nullptr;
  int* d_fault = nullptr;
  int skip_zt = 0;                // fault injection (hg_debug_set): Z^T r launches to drop
  double* d_y = nullptr;          // coarse solution (m)
  double* d_b0_inv = nullptr;     // dense B0^{-1}, packed 8 x 8 fragment blocks (hg_b0d.cu), b0_mp x b0_mp, or null
  int b0_mp = 0;                  // m rounded up to 8
  bool b0_inv_single = true;      // single-RHS applies use it too (else only the batched ones)
  double* d_c = nullptr;          // reduced Z^T r (m), dense mode
  double* d_cm = nullptr;         // [m][16] reduced Z^T R, dense mode
  double* d_ypart = nullptr;      // [B0_KSPLIT][m][16] split-K partials, dense batched mode
  long long zs_len = 0;
  double* d_zs = nullptr;         // per-block Z_b y_b rows (scratch)
  int* d_cptr = nullptr;
  long long* d_cent = nullptr;

  double* d_tmp = nullptr;        // n-vector scratch (B u for apply_T)

  // multi-RHS scratch (allocated on the first batched call, HG_MAX_RHS columns)
  bool multi_ready = false;
  double* d_xsm = nullptr;        // [c][xs_len] local solutions
  double* d_zsm = nullptr;        // [c][zs_len] Z_b Y_b rows
  double* d_cpartm = nullptr;     // [part_len][HG_MAX_RHS] Z^T R partials
  double* d_ym = nullptr;         // [m][HG_MAX_RHS] coarse solution
  // packed copies of Z for the batched contractions (hg_multi.cu "packed Z")
  double* d_zypk = nullptr;
  double* d_ztpk = nullptr;
  long long* d_zypk_off = nullptr;
  long long* d_ztpk_off = nullptr;
  void* d_zy_items = nullptr;     // ZyItem per pair of 8-row tiles (hg_multi.cu)
  int n_zy_items = 0;
  double* d_b0m_x = nullptr;      // [2][K*64][HG_MAX_RHS] phase solutions
  double* d_tmpm = nullptr;       // [c][n] scratch (B U for the batched apply_T)
  cudaStream_t aux = nullptr;     // coarse chain runs here, forked/joined per apply
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  long long device_bytes = 0;
  struct HgOp* op_T = nullptr;    // cached operators of hg_solve_host
  struct HgOp* op_W = nullptr;
};

namespace hg {

constexpr int VEC_THREADS = 256;
constexpr int VEC_ROWS = 4;                 // rows per thread
constexpr int VEC_TILE = VEC_THREADS * VEC_ROWS;
constexpr int MAX_NV = 1024;                // max vectors in one fused dot

// Block-level partial dots of z against nv vectors W[i] (stride ldw) for the
// rows this block owns; `zv` holds the thread's VEC_ROWS values of z.
// Writes partials[blockIdx.x * width + off + i].
template <int ROWS>
__device__ __forceinline__ void block_dots(const double (&zv)[ROWS], const int (&rows)[ROWS], int n,
                                           const double* __restrict__ W, long long ldw, int nv,
                                           double* __restrict__ partials, int width, int off,
                                           double* /*unused*/) {
  __shared__ double s_warp[VEC_THREADS / 32][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i0 = 0; i0 < nv; i0 += 64) {
    int cnt = min(64, nv - i0);
    for (int ii = 0; ii < cnt; ++ii) {
      const double* wi = W + (long long)(i0 + ii) * ldw;
      double p = 0.0;
#pragma unroll
      for (int k = 0; k < ROWS; ++k)
        if (rows[k] < n) p = fma(__ldg(wi + rows[k]), zv[k], p);
      p = warp_sum(p);
      if (lane == 0) s_warp[warp][ii] = p;
    }
    __syncthreads();
    if (threadIdx.x < cnt) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < VEC_THREADS / 32; ++w) t += s_warp[w][threadIdx.x];
      partials[(long long)blockIdx.x * width + off + i0 + threadIdx.x] = t;
    }
    __syncthreads();
  }
}


// ---- launchers (return HG_OK or an error code) ----
int launch_spmv(const DevCsr& A, const double* vals, const double* x, double* y, cudaStream_t st);
// y = A x with fused partial dots: self_part[b] = sum x.y over block b;
// dot_part[b*nv + i] = sum_d W[i][d] * z[d] where z = (dot_with_y ? y : x).
int launch_spmv_dots(const DevCsr& A, const double* vals, const double* x, double* y, const double* W,
                     long long ldw, int nv, bool dot_with_y, double* partials, int* nblocks_out,
                     cudaStream_t st);
int spmv_dots_nblocks(int n);

int launch_local_solve(HgPrecond* P, const double* r, cudaStream_t st);
int launch_local_solve_multi(HgPrecond* P, const double* R, long long ldr, int nrhs, cudaStream_t st);
// 16-row panel local solves on DMMA (hg_local_panel.cu)
int prepare_local_panel(HgPrecond* P);
int launch_local_panel(HgPrecond* P, const double* R, long long ldr, int nrhs, cudaStream_t st);
int launch_local_batch(HgPrecond* P, const double* R, long long ldr, int nrhs, cudaStream_t st);
int preload_local_panel();
int launch_local_solve_single(HgPrecond* P, int s, const double* r_local, double* x_local, cudaStream_t st);
// device band LU of every local block into P->d_fwd / P->d_bwd (hg_factor.cu)
int band_lu_supported(int kl_max, int ku_max);
int launch_band_lu(HgPrecond* P, const int* d_bw, int kl_max, int ku_max, const long long* d_ptr_base,
                   const long long* d_indptr, const int* d_cols, const double* d_vals, int* d_info, double* d_minpiv,
                   cudaStream_t st);
int launch_zt(HgPrecond* P, const double* r, cudaStream_t st);
// zt_target: value of the Z^T r chunk counter the solve waits for before reading c
// the solve waits (bounded, device side) for the Z^T r launch it pairs with
int launch_coarse_solve(HgPrecond* P, cudaStream_t st);
int launch_coarse_solve_cluster(HgPrecond* P, cudaStream_t st);
// bisected coarse solve: the two half chains (joined on st), then the separator stage
int launch_coarse_chains_split(HgPrecond* P, cudaStream_t st);
int launch_coarse_sep_split(HgPrecond* P, cudaStream_t st);
SpinCfg spin_cfg(const HgPrecond* P);
// per (kernel, device) dynamic shared memory / cluster attributes (thread safe)
int ensure_func_attrs(const void* func, size_t smem, bool nonportable_cluster);
size_t b0_cluster_smem(int NR, int tns = 4);
// force-load kernels at handle creation (see preload_local in hg_local.cu)
int preload_local(HgPrecond* P);
int preload_local_multi(HgPrecond* P);
int preload_coarse();
int preload_assemble();
int preload_b0();
int preload_b0_cluster();
int preload_vec();
int launch_zy(HgPrecond* P, cudaStream_t st);
// out = coarse + local contributions; optional fused partial dots W[i].out
int launch_assemble(HgPrecond* P, bool with_coarse, bool with_local, double* out, const double* W,
                    long long ldw, int nv, double* partials, int* nblocks_out, cudaStream_t st);
int assemble_nblocks(int n);

struct ColList {
  int n;
  int c[HG_MAX_RHS];
  double s[HG_MAX_RHS];   // per-column scalar (h norms for scale)
};

// ---- multi-RHS (hg_multi.cu); batches are column c at base + c * ld
int multi_prepare(HgPrecond* P);
int preload_multi();
int launch_spmm(const DevCsr& A, const double* vals, const double* X, long long ldx, double* Y, long long ldy,
                int nrhs, cudaStream_t st);
// Y = A X with per-column self dots X_c . Y_c into partials[(c * nb + b) * width]
int launch_spmm_cols(const DevCsr& A, const double* vals, const double* X, long long ldx, double* Y, long long ldy,
                     const ColList& cols, double* partials, int width, int* nb_out, cudaStream_t st);
int launch_spmm_self(const DevCsr& A, const double* vals, const double* X, long long ldx, double* Y,
                     long long ldy, int nrhs, double* partials, int width, int* nblocks_out, cudaStream_t st);
int launch_zt_multi(HgPrecond* P, const double* R, long long ldr, int nrhs, cudaStream_t st);
int launch_b0_multi(HgPrecond* P, int nrhs, cudaStream_t st);
// dense coarse mode (hg_b0d.cu): c = reduce(Z^T r partials), y = B0^{-1} c
int launch_b0_dense(HgPrecond* P, cudaStream_t st);
int launch_b0_dense_multi(HgPrecond* P, int nrhs, cudaStream_t st);
int preload_b0_dense();
int split_upload(HgPrecond* P, const HgPrecondDesc* D);
void split_release(HgPrecond* P);
int launch_split_stages(HgPrecond* P, const double* R, long long ldr, double* xs, long long xs_len, int nrhs,
                        cudaStream_t st);
int preload_split();
int pack_b0_inverse(int m, const double* d_binv, double** d_packed, int* mp_out);
constexpr int B0_KSPLIT = 8;
int launch_zy_multi(HgPrecond* P, int nrhs, cudaStream_t st);
int launch_assemble_multi(HgPrecond* P, bool with_coarse, bool with_local, double* OUT, long long ldo, int nrhs,
                          cudaStream_t st);

// Batched Arnoldi kernels over a list of columns (cols: device, ncols
// entries).  Column c's vectors: z + c * ldz; its basis vector i:
// V + c * ldcol + i * ldv.  Partials: [(c * nb + b) * width + slot].

int launch_dots_batch(int n, const double* z, long long ldz, const double* V, long long ldv, long long ldcol,
                      int nv, const ColList& cols, double* partials, int width, int* nblocks_out, cudaStream_t st);
// out[c * ow + k] = sum_b partials[(c * nb + b) * width + k], k < cnt, for the listed columns
int launch_reduce_batch(const double* partials, int nb, int width, int cnt, const ColList& cols, double* out,
                        long long ow, cudaStream_t st);
// mode 0: w = V coef ; 1: w -= V coef ; 2: w += V coef ; coef of column c at coef + c * ldcoef (+ coef_off)
int launch_axpy_batch(int n, double* w, long long ldw, const double* V, long long ldv, long long ldcol, int nv,
                      const double* coef, long long ldcoef, int mode, const ColList& cols, cudaStream_t st);
// V_c = w_c / s_c, WV_c = ww_c / s_c for the listed columns
int launch_scale_batch(int n, const double* w, const double* ww, long long ldw, double* V, double* WV,
                       long long ldcol, const ColList& cols, cudaStream_t st);
int launch_fill_batch(int n, double* y, long long ldy, const ColList& cols, cudaStream_t st);
// DCGS2 Arnoldi (hg_multi.cu): dots of V_c[0..nv) with A_c and U_c in one basis read
// (partials [(c * nb + b) * width + {i, nv + i}]); the fused delayed
// reorthogonalisation / projection update; device-normalised append.
// (reduced into out[c * ow + k], k < 2 nv: V_k . A_c then V_k . U_c)
int launch_dots2_batch(int n, const double* A, long long lda, const double* U, long long ldu, const double* V,
                       long long ldv, long long ldcol, int nv, const ColList& cols, double* partials, double* out,
                       long long ow, cudaStream_t st);
int launch_dcgs2_update(int n, double* V, long long ldv, long long ldcol, int j, double* w, long long ldw,
                        const double* coef, long long ldcoef, const ColList& cols, cudaStream_t st);
int launch_scale_dev_batch(int n, const double* w, const double* ww, long long ldw, double* V, long long ldcol,
                           double* Wq, const double* nrm2, const ColList& cols, cudaStream_t st);
int preload_dcgs2();
int preload_add();
int launch_add(int n, const double* a, const double* b, double* out, cudaStream_t st);  // out = a + b

// Arnoldi helpers
int launch_dots(int n, const double* z, const double* W, long long ldw, int nv, double* partials,
                int* nblocks_out, cudaStream_t st);
int launch_reduce(const double* partials, int nblocks, int width, double* out, cudaStream_t st);
// mode 0: w = V c ; 1: w -= V c ; 2: w += V c  (sequential over the nv vectors)
int launch_axpy_multi(int n, double* w, const double* V, long long ldv, int nv, const double* coef,
                      int mode, cudaStream_t st);
int launch_sub(int n, const double* a, const double* b, double* out, cudaStream_t st);  // out = a - b
int launch_scale2(int n, const double* w, const double* ww, const double* hnorm_dev, double* v_out,
                  double* wv_out, cudaStream_t st);
int launch_copy(int n, const double* x, double* y, cudaStream_t st);
int launch_fill(long long n, double* y, double val, cudaStream_t st);

}  // namespace hg
