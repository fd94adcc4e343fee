/*
 * helmgpu.h — C ABI of the B200 solve phase of the two-level Schwarz /
 * H_k-GenEO preconditioned weighted GMRES (arXiv 2406.06283, reference
 * package `helmdd`).
 *
 * Every entry point is plain C: integers, doubles, pointers and sizes.  No
 * torch or CUDA C++ types appear; a cudaStream_t is passed as `void*`
 * (NULL = legacy default stream).  Pointers documented as "device" must be
 * CUDA device (or managed) memory; "host" pointers are ordinary or pinned
 * host memory.  All functions return 0 on success and a nonzero HG_ERR_*
 * code otherwise; hg_last_error() then holds a message.
 *
 * Reference interfaces replaced (all under /root/reference/pkg/src/helmdd):
 *   hg_precond_create   <- schwarz.factorize            (schwarz.py:74-101)
 *                          consumes the setup products: forms.helmholtz /
 *                          forms.dk (assembly.py:123-145), fine idof lists
 *                          (decomp.py:238-248), per-block LU factors
 *                          (schwarz.py:104-131), Z (eigencoarse.py:259-284),
 *                          lu_factor(B0) (schwarz.py:88-99)
 *   hg_precond_apply    <- TwoLevelPreconditioner.apply (schwarz.py:51-61)
 *   hg_precond_apply_T  <- TwoLevelPreconditioner.apply_T (schwarz.py:63-65)
 *   hg_precond_apply_coarse <- TwoLevelPreconditioner.apply_coarse (schwarz.py:67-71)
 *   hg_local_solve      <- LocalSolver.lu.solve        (schwarz.py:26-34, 60)
 *   hg_op_*             <- the `op` / `weight` arguments of weighted_gmres
 *                          (wgmres.py:74-100, _as_operator wgmres.py:57-60)
 *   hg_gmres            <- wgmres.weighted_gmres        (wgmres.py:74-203)
 *   hg_solve_host       <- the solve block of cli.run_single
 *                          (cli.py:297-307): rhs_p = M^{-1} f,
 *                          x = weighted_gmres(M^{-1} B, rhs_p, weight=D_k)
 *
 * Threading: a handle is used from one host thread at a time (the reference
 * loop is single threaded).  Results are bitwise deterministic
 * run to run: every reduction and every overlapping scatter-add is summed
 * in a fixed order, no floating-point atomics (schwarz.py:52).
 */
#ifndef HELMGPU_H
#define HELMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_OK 0
#define HG_ERR_CUDA 1
#define HG_ERR_ARG 2
#define HG_ERR_UNSUPPORTED 3
#define HG_ERR_NOMEM 4

#define HG_ABI_VERSION 1

typedef struct HgPrecond HgPrecond; /* opaque: device-resident preconditioner */
typedef struct HgOp HgOp;           /* opaque: device linear operator */

/* Host-side description of everything the solve phase consumes.  All arrays
 * are host memory, copied to the device by hg_precond_create (the caller may
 * free them afterwards). */
typedef struct {
  int32_t n; /* global number of dofs */

  /* Global CSR of B = A - k^2 S and D_k = A + k^2 S (same pattern). */
  int64_t nnz;
  const int32_t* indptr;  /* n+1 */
  const int32_t* indices; /* nnz, ascending within a row */
  const double* b_data;   /* nnz */
  const double* dk_data;  /* nnz, may be NULL */

  /* One-level part: n_local fine subdomains in reference order
   * (dec.fine_flat()).  Block s acts on idof_s = local_idx[local_idx_off[s]
   * .. local_idx_off[s+1]) (ascending).  Its pivoted band LU (LAPACK dgbtrf
   * semantics, lower bandwidth kl, U bandwidth kv = kl + ku) is packed as two
   * record streams of fixed stride per block:
   *   forward  record j (j = 0..n_s-1):  [l_{j+1,j}, ..., l_{j+kl,j}, ipiv_j, pad]
   *   backward record r (r = 0..n_s-1, j = n_s-1-r):
   *                                      [u_{j-1,j}, ..., u_{j-kv,j}, 1/u_jj, pad]
   * with local_fstride / local_bstride doubles per record (even), zeros past
   * the end of the block, ipiv stored as an exact double (0-based). */
  int32_t n_local;
  const int32_t* local_n;
  const int32_t* local_kl;
  const int32_t* local_kv;
  const int32_t* local_fstride;
  const int32_t* local_bstride;
  const int64_t* local_idx_off; /* n_local+1 */
  const int32_t* local_idx;
  const int64_t* local_fwd_off; /* n_local, in doubles, even */
  int64_t local_fwd_len;
  const double* local_fwd;
  const int64_t* local_bwd_off; /* n_local, in doubles, even */
  int64_t local_bwd_len;
  const double* local_bwd;

  /* Coarse part (m = 0: one-level preconditioner).  Z is held as n_cblk
   * dense row-major blocks Z_b (cblk_n[b] x cblk_m[b]) over the index sets
   * cblk_idx[cblk_idx_off[b] ..]; columns are numbered block after block
   * (the reference's column order, eigencoarse.py:259-266).
   * B0 = P^T L U (LAPACK getrf); (P c)[i] = c[b0_perm[i]].  The two
   * triangular solves (L; then U in reversed coordinates, where it is lower
   * triangular) are cut into b0_npanel panels of b0_panel rows each (m padded
   * with identity rows).  Panel g = phase*K + t has the explicit inverse of
   * its diagonal block at b0_dinv[g*P*P] (row-major) and the nonzero
   * off-diagonal tiles b0_tiles[e*P*P] for e in [b0_tile_ptr[g],
   * b0_tile_ptr[g+1]), column panel b0_tile_col[e] ascending. */
  int32_t m;
  int32_t n_cblk;
  const int32_t* cblk_n;
  const int32_t* cblk_m;
  const int64_t* cblk_idx_off; /* n_cblk+1 */
  const int32_t* cblk_idx;
  const int64_t* cblk_z_off; /* n_cblk, in doubles */
  int64_t z_len;
  const double* z_data;
  const int32_t* b0_perm;
  int32_t b0_panel;     /* P: 32, 64 or 128 */
  int32_t b0_npanel;    /* K = ceil(m / P) */
  const double* b0_dinv;        /* 2*K*P*P */
  const int64_t* b0_tile_ptr;   /* 2*K+1 */
  const int32_t* b0_tile_col;   /* ntile */
  int64_t b0_ntile;
  const double* b0_tiles;       /* ntile*P*P */
  int32_t b0_ctas;      /* persistent CTAs of the coarse solve (0 = default 32) */
  /* b0_mode 0: persistent-CTA solve synchronised through an L2 counter;
   * b0_mode 1: single thread-block cluster of b0_cluster (<= 16) CTAs, panels
   * handed over through distributed shared memory (ring of b0_ring panels;
   * requires P = 64, b0_ring >= max tile distance + b0_cluster, and tiles /
   * inverse blocks with 16-byte chunks XOR-swizzled by row parity:
   * chunk c of row r stored at chunk c ^ ((r & 1) << 2)). */
  int32_t b0_mode;
  int32_t b0_cluster;
  int32_t b0_ring;
} HgPrecondDesc;

/* ---- library ---- */
int hg_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* hg_last_error(void);
/* Number of this library's kernels launched since load (counter). */
int64_t hg_kernel_launches(void);
int hg_device_sync(void);

/* ---- preconditioner (schwarz.factorize / TwoLevelPreconditioner) ---- */
int hg_precond_create(const HgPrecondDesc* desc, HgPrecond** out);
int hg_precond_destroy(HgPrecond* p);
/* device bytes held by the handle */
int64_t hg_precond_device_bytes(const HgPrecond* p);
/* out = M^{-1} r ; r, out: device, length n; out fully overwritten. */
int hg_precond_apply(HgPrecond* p, const double* r, double* out, void* stream);
/* out = M^{-1} (B u) */
int hg_precond_apply_T(HgPrecond* p, const double* u, double* out, void* stream);
/* out = Z B0^{-1} Z^T r (zeros without a coarse space) */
int hg_precond_apply_coarse(HgPrecond* p, const double* r, double* out, void* stream);
/* y = B x (which = 0) or y = D_k x (which = 1) */
int hg_precond_spmv(HgPrecond* p, int which, const double* x, double* y, void* stream);
/* Local solve of block s alone: x_local = B_s^{-1} r_local, both device,
 * length local_n[s] (LocalSolver.lu.solve). */
int hg_local_solve(HgPrecond* p, int s, const double* r_local, double* x_local, void* stream);

/* Stage timing of the apply (no reference analogue; measurement hook used by
 * bench.py): runs `iters` applies with the stages serialised on `stream`
 * and CUDA events between them; stage_ms (host, HG_NSTAGES doubles) gets the
 * mean device time per stage: {Z^T r, B0 solve, Z y, local band solves,
 * assembly}. */
#define HG_NSTAGES 5
int hg_precond_profile(HgPrecond* p, const double* r, double* out, int32_t iters, double* stage_ms,
                       void* stream);

/* ---- operators for GMRES ---- */
/* General square CSR operator uploaded from host arrays. */
int hg_op_create_csr(int32_t n, int64_t nnz, const int32_t* indptr, const int32_t* indices,
                     const double* data, HgOp** out);
/* mode 0: v -> M^{-1} v ; mode 1: v -> M^{-1} B v (the left-preconditioned
 * operator of cli.py:298) ; mode 2: v -> B v ; mode 3: v -> D_k v.
 * The operator borrows the handle (destroy the op first). */
int hg_op_create_precond(HgPrecond* p, int mode, HgOp** out);
int hg_op_destroy(HgOp* op);
int hg_op_apply(HgOp* op, const double* x, double* y, void* stream);

/* ---- weighted GMRES (wgmres.weighted_gmres) ----
 * Full (unrestarted) GMRES on `op` in the <u,v>_W = v^T W u inner product
 * (weight NULL = Euclidean).  rhs, x0 (may be NULL = zero) and x are device
 * vectors of length n.  history (host, >= maxit+1 doubles) receives the
 * weighted residual norms; info (host, 4 ints) receives
 * {iterations, converged, breakdown, reorth_passes}. */
int hg_gmres(HgOp* op, HgOp* weight, const double* rhs, const double* x0, double* x, double rtol,
             int32_t maxit, double* history, int32_t* info, void* stream);

/* End-to-end solve with HOST buffers (the drop-in for cli.py:297-307):
 * f (host, n) -> x (host, n); rhs_p = M^{-1} f ; x = GMRES(M^{-1}B, rhs_p,
 * weight D_k).  H2D and D2H copies are inside the call. */
int hg_solve_host(HgPrecond* p, const double* f_host, double* x_host, double rtol, int32_t maxit,
                  double* history, int32_t* info, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HELMGPU_H */
