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
 *   hg_precond_apply_multi, hg_op_apply_multi, hg_gmres_batch,
 *   hg_solve_host_batch <- no reference function: the
 *                          reference solves config 5's 16 right-hand sides
 *                          one at a time; these run nrhs independent solves
 *                          (own Krylov space, own stopping test per column)
 *                          through shared operator applies, so the factors,
 *                          Z and B0 stream from HBM once per batched apply.
 *                          Column c of a batch is parity-checked against the
 *                          one-at-a-time call.
 *
 * Batches: nrhs <= HG_MAX_RHS vectors of length n; column c of a batch X
 * with leading dimension ldx is X + c * ldx (ldx >= n).
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

#define HG_ABI_VERSION 5

/* Most right-hand sides one batched call handles (BASELINE config 5's
 * batch of 16 seeded load vectors). */
#define HG_MAX_RHS 16

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
   * the end of the block, ipiv stored as an exact double (0-based).  With
 * R_f = max(2, 1 + ceil(max_s kl_s / 32)) (R_b likewise from kv), every
 * non-empty block needs kl_s >= 32 R_f - 65 and kv_s >= 32 R_b - 65: pad
 * narrower blocks with zero multipliers (hg_precond_create checks). */
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
  /* Optional dense B0^{-1} (m x m, row-major, host or device memory; NULL =
   * none).  When given, the
   * coarse solve is y = B0^{-1} c as an HBM-streaming GEMV (one right-hand
   * side) / FP64 tensor-core GEMM (batches) that runs beside the local
   * solves instead of the 2K-panel triangular chain.  The caller checks it
   * against getrs (factorize does, bar 1e-11) — same operator, different
   * rounding. */
  const double* b0_inv;

  /* Device factorisation of the local blocks.  When
   * local_fwd and local_bwd are NULL, hg_precond_create builds the records
   * itself: block s is given as a block-local CSR (its rows at
   * lcsr_indptr[local_idx_off[s] + s .. + n_s], absolute offsets into
   * lcsr_cols / lcsr_vals; columns block-local, ascending) with band
   * half-width local_bw[s] (kl = ku), and is factored on the device with
   * LAPACK dgbtrf semantics (partial pivoting within the band, multipliers
   * by the reciprocal pivot; schwarz.py:104-131 _factor_block) straight into
   * the record layout above (local_kl / local_kv / strides / offsets still
   * describe it; local_fwd_len / local_bwd_len size it).  factor_info[s]
   * (host out) receives dgbtrf's INFO (0, or j+1 for the first exactly-zero
   * pivot) and factor_min_pivot[s] (host out) min_j |u_jj|, for the
   * caller's singular-block test.  hg_precond_read returns the records. */
  const int32_t* local_bw;
  const int64_t* lcsr_indptr;
  const int32_t* lcsr_cols;
  const double* lcsr_vals;
  int64_t lcsr_nnz;
  int32_t* factor_info;
  double* factor_min_pivot;
  /* With b0_inv given: 0 = every apply uses it; 1 = only batched applies
   * (the single-RHS apply keeps the panel chain, which is shorter there). */
  int32_t b0_inv_batched_only;

  /* Split local blocks (optional; n_split = 0: none).  A fine subdomain whose
   * band solve is one long dependency chain (few, large blocks: config 5 at
   * 8 x 8) may be given as P chunks of consecutive band rows separated by P-1
   * separators of kl rows each (rows i < a and j >= a + kl of a band matrix
   * do not couple).  Its local solve (ls.lu.solve, schwarz.py:58-60 — the same
   * operator B_s^{-1}, eliminated in nested-dissection order) is then
   *   y_p = A_p^{-1} r_p            every chunk: an ordinary local block above
   *   x_S = Sigma^{-1} (r_S - F y)  Sigma = A_SS - sum_p F_p A_p^{-1} E_p
   *   x_p = y_p - W_p x_S           W_p = A_p^{-1} E_p (the chunk's spikes)
   * so the chain is 1/P as long and P times as many CTAs work.  Each chunk is
   * a local block; the separators of split s are ONE pseudo block split_blk[s]
   * with local_n = 0 whose index range (local_idx_off) lists the separator
   * dofs (separator after separator).  Separator rows of all splits are
   * numbered consecutively: split s owns rows split_row_off[s] ..
   * split_row_off[s+1].  F (separator rows x chunk unknowns) is a CSR over
   * those rows whose column entries are POSITIONS in the local solution
   * scratch (local_idx_off[block] + row within the block).  Sigma^{-1} of
   * split s is row-major nS x nS at split_sinv[split_sinv_off[s]].  Spike i
   * belongs to chunk block spike_blk[i] of split spike_split[i]; it couples
   * to separator rows spike_col0[i] .. + spike_w[i] of that split (spike_w a
   * multiple of 8, zero padded) and is stored at spike_data[spike_off[i]] in
   * 8 x 8 fragment blocks: block (mt, kb) at doubles (mt KB + kb) 64, element
   * (lane = 4 g + q, h) at 2 lane + h = W[8 mt + g][8 kb + 4 h + q], rows
   * zero padded to a multiple of 8 (KB = spike_w / 8). */
  int32_t n_split;
  const int32_t* split_blk;       /* n_split */
  const int64_t* split_row_off;   /* n_split+1 */
  const int64_t* split_f_indptr;  /* total separator rows + 1 */
  const int64_t* split_f_pos;
  const double* split_f_val;
  const int64_t* split_sinv_off;  /* n_split, in doubles */
  int64_t split_sinv_len;
  const double* split_sinv;
  int32_t n_spike;
  const int32_t* spike_blk;       /* n_spike */
  const int32_t* spike_split;
  const int32_t* spike_col0;
  const int32_t* spike_w;
  const int64_t* spike_off;       /* n_spike, in doubles */
  int64_t spike_len;
  const double* spike_data;

  /* Bisected coarse solve (optional; b0_split = 0: none).  The single-RHS
   * coarse solve y = B0^{-1} c (lu_solve, schwarz.py:56) is a chain of 2K
   * panel hand-offs; B0 is banded (subdomains couple to their neighbours
   * only), so — like a split local block — its unknowns are cut into two
   * halves H0 = [0, a), H1 = [a + ns, m) and a separator S = [a, a + ns)
   * (ns >= B0's bandwidth): the halves' chains (their own getrf tiles, in
   * the layout of b0_* above; cluster mode only) run side by side on two
   * clusters, then x_S = Sigma^{-1} (c_S - F y_H), y_H -= W x_S with
   * Sigma = B0_SS - sum_h B0_SHh B0_HhHh^{-1} B0_HhS, F = [B0[S, a-wl..a),
   * B0[S, a+ns..a+ns+wr)] (ns x (wl + wr), row-major: everything B0_SH is
   * nonzero on) and W = [B0_H0H0^{-1} B0_H0S; B0_H1H1^{-1} B0_H1S]
   * ((m - ns) x ns, row-major).  Same operator, different elimination
   * order; the caller checks it against getrs (bar 1e-11).  Batched applies
   * are not affected (they use b0_inv). */
  int32_t b0_split;
  int32_t b0s_a, b0s_ns, b0s_wl, b0s_wr;
  int32_t b0h0_npanel, b0h0_ring, b0h0_cluster;
  int64_t b0h0_ntile;
  const int32_t* b0h0_perm;      /* a */
  const double* b0h0_dinv;
  const int64_t* b0h0_tile_ptr;
  const int32_t* b0h0_tile_col;
  const double* b0h0_tiles;
  int32_t b0h1_npanel, b0h1_ring, b0h1_cluster;
  int64_t b0h1_ntile;
  const int32_t* b0h1_perm;      /* m - a - ns */
  const double* b0h1_dinv;
  const int64_t* b0h1_tile_ptr;
  const int32_t* b0h1_tile_col;
  const double* b0h1_tiles;
  const double* b0s_f;
  const double* b0s_sinv;
  const double* b0s_w;
} HgPrecondDesc;

/* ---- library ---- */
int hg_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* hg_last_error(void);
/* Number of this library's kernels launched since load (counter). */
int64_t hg_kernel_launches(void);
int hg_device_sync(void);
/* Process exit: later destroy calls return without touching the device
 * (the CUDA driver may already be torn down when a host language's
 * finalizers run; the Python binding registers this with atexit). */
int hg_shutdown(void);

/* ---- setup on the device ---- */
/* Coarse operator: B0 = 0.5 (Z^T B Z + (Z^T B Z)^T) (eigencoarse.py:286-287)
 * from the desc's global CSR of B and its Z blocks (n, nnz, indptr, indices,
 * b_data, m, n_cblk, cblk_*, z_len, z_data; nothing else is read), with the
 * block interaction lists pair_ptr[n_cblk+1] / pair_blk (blocks a whose
 * dofs couple to block b through B, for b in order); then its LU with partial
 * pivoting (LAPACK getrf semantics, schwarz.py:90: 64-column panels, row
 * interchanges over whole rows, multipliers by the reciprocal pivot) and the
 * rank certificate of coarse._sym_extreme_certificate: cert_out[0] =
 * |lambda|_max estimate (power iteration on B0), cert_out[1] = ||B0^{-1}||
 * estimate (inverse iteration through the LU), cert_iters steps each.  Any
 * host output may be NULL: b0_out, lu_out (m*m row-major), piv_out (m,
 * 0-based), info_out (getrf INFO), cert_out (2). */
int hg_coarse_setup(const HgPrecondDesc* desc, const int32_t* pair_ptr, const int32_t* pair_blk, double* b0_out,
                    double* lu_out, int32_t* piv_out, int32_t* info_out, double* cert_out, int32_t cert_iters);

/* ---- preconditioner (schwarz.factorize / TwoLevelPreconditioner) ---- */
int hg_precond_create(const HgPrecondDesc* desc, HgPrecond** out);
/* Fault state of a handle (no synchronisation).  The coarse solve is
 * launched on a side stream ahead of the Z^T r it consumes and waits for it
 * on the device; every such wait is bounded (default 10 s, hg_debug_set).  A
 * timed-out wait, or a launch that fails part-way through an apply, poisons
 * the handle: this and every later call on it return HG_ERR_CUDA with a
 * message (destroy and recreate it).  The reference's apply never raises
 * (SPEC.md:359); a device fault is the one exception. */
int hg_precond_status(HgPrecond* p);
int hg_precond_destroy(HgPrecond* p);
/* device bytes held by the handle */
int64_t hg_precond_device_bytes(const HgPrecond* p);
/* Copy a device-resident array of the handle to host memory (e.g. the
 * records of a device factorisation, for the on-disk setup cache):
 * field HG_FIELD_LOCAL_FWD / HG_FIELD_LOCAL_BWD, `count` doubles (the
 * desc's local_fwd_len / local_bwd_len). */
#define HG_FIELD_LOCAL_FWD 1
#define HG_FIELD_LOCAL_BWD 2
int hg_precond_read(HgPrecond* p, int32_t field, double* host, int64_t count);
/* Numbers about a handle (no synchronisation; NAN for an unknown key):
 *   HG_STAT_PANEL_ACTIVE     1 if batched applies run the 16-row panel local
 *                            solve (DMMA; built at create from the band
 *                            records, HG_LOCAL_PANEL=0 disables), else 0
 *   HG_STAT_PANEL_DEVIATION  its check against the row solve on a seeded
 *                            16-column batch: max over columns of
 *                            max|x_panel - x_row| / max|x_row| (must be
 *                            <= 1e-11 to be active; -1 = not built)
 *   HG_STAT_PANEL_BYTES      panel-record bytes one batched local solve
 *                            streams (each panel's nonzero part only) */
#define HG_STAT_PANEL_ACTIVE 1
#define HG_STAT_PANEL_DEVIATION 2
#define HG_STAT_PANEL_BYTES 3  /* factor bytes one batched local solve streams */
double hg_precond_stat(HgPrecond* p, int32_t key);
/* out = M^{-1} r ; r, out: device, length n; out fully overwritten. */
int hg_precond_apply(HgPrecond* p, const double* r, double* out, void* stream);
/* out = M^{-1} (B u) */
int hg_precond_apply_T(HgPrecond* p, const double* u, double* out, void* stream);
/* y = B0^{-1} c on the device's panel chain (c, y: device, length m): the
 * coarse solve alone (lu_solve(b0_piv, c), schwarz.py:56), for the check
 * factorize runs against getrs and for tests. */
int hg_precond_coarse_solve(HgPrecond* p, const double* c, double* y, void* stream);
/* out = Z B0^{-1} Z^T r (zeros without a coarse space) */
int hg_precond_apply_coarse(HgPrecond* p, const double* r, double* out, void* stream);
/* y = B x (which = 0) or y = D_k x (which = 1) */
int hg_precond_spmv(HgPrecond* p, int which, const double* x, double* y, void* stream);
/* Local solve of block s alone: x_local = B_s^{-1} r_local, both device,
 * length local_n[s] (LocalSolver.lu.solve). */
int hg_local_solve(HgPrecond* p, int s, const double* r_local, double* x_local, void* stream);
/* The one-level part before assembly: every block's local solution
 * x_s = B_s^{-1} R_s r for a global residual r (device, n), written block
 * after block to xs (device, local_idx_off[n_local] doubles; block s at
 * local_idx_off[s]).  Includes the separator and spike stages of split
 * blocks, whose solution is spread over their chunk blocks and their
 * separator pseudo block — this is how LocalSolver.lu.solve of a split block
 * is served (schwarz.py:26-34, 60). */
int hg_precond_local_solutions(HgPrecond* p, const double* r, double* xs, void* stream);

/* Stage timing of the apply (no reference analogue; measurement hook used by
 * bench.py): runs `iters` applies with the stages serialised on `stream`
 * and CUDA events between them; stage_ms (host, HG_NSTAGES doubles) gets the
 * mean device time per stage: {Z^T r, B0 solve, Z y, local band solves,
 * assembly}. */
#define HG_NSTAGES 5
int hg_precond_profile(HgPrecond* p, const double* r, double* out, int32_t iters, double* stage_ms,
                       void* stream);

/* OUT[:, c] = M^{-1} R[:, c] for c < nrhs (one batched apply: local solves
 * with one warp per column on a shared factor stream, Z^T R and Z Y as dense
 * FP64 tensor-core (DMMA) contractions, one coarse solve for all columns). */
int hg_precond_apply_multi(HgPrecond* p, const double* R, int64_t ldr, double* OUT, int64_t ldo, int32_t nrhs,
                           void* stream);
/* Stage timing of the batched apply (as hg_precond_profile). */
int hg_precond_profile_multi(HgPrecond* p, const double* R, int64_t ldr, double* OUT, int64_t ldo, int32_t nrhs,
                             int32_t iters, double* stage_ms, void* stream);

/* ---- operators for GMRES ---- */
/* General square CSR operator uploaded from host arrays. */
int hg_op_create_csr(int32_t n, int64_t nnz, const int32_t* indptr, const int32_t* indices,
                     const double* data, HgOp** out);
/* mode 0: v -> M^{-1} v ; mode 1: v -> M^{-1} B v (the left-preconditioned
 * operator of cli.py:298) ; mode 2: v -> B v ; mode 3: v -> D_k v.
 * The operator borrows the handle (destroy the op first). */
int hg_op_create_precond(HgPrecond* p, int mode, HgOp** out);
int hg_op_destroy(HgOp* op);
/* Release the operator's Krylov bases and GMRES workspaces (the op stays
 * usable; the next solve maps them again).  hg_op_basis is unavailable until
 * then.  Memory plan: a solve whose worst-case basis (nrhs (maxit+1) n
 * doubles) does not fit the free device memory first releases the idle
 * bases of the other ops of the process, then solves its batch in
 * sub-batches of columns. */
int hg_op_release(HgOp* op);
int hg_op_apply(HgOp* op, const double* x, double* y, void* stream);
/* Y[:, c] = op(X[:, c]), c < nrhs (batched SpMM / batched apply). */
int hg_op_apply_multi(HgOp* op, const double* X, int64_t ldx, double* Y, int64_t ldy, int32_t nrhs, void* stream);

/* ---- weighted GMRES (wgmres.weighted_gmres) ----
 * Full (unrestarted) GMRES on `op` in the <u,v>_W = v^T W u inner product
 * (weight NULL = Euclidean).  rhs, x0 (may be NULL = zero) and x are device
 * vectors of length n.  history (host, >= maxit+1 doubles) receives the
 * weighted residual norms; info (host, 4 ints) receives
 * {iterations, converged, breakdown, reorth_passes}. */
int hg_gmres(HgOp* op, HgOp* weight, const double* rhs, const double* x0, double* x, double rtol,
             int32_t maxit, double* history, int32_t* info, void* stream);

/* nrhs independent weighted GMRES solves (x0 = 0) advanced in lock step:
 * every iteration applies `op` once to the batch of current Krylov vectors;
 * orthogonalisation, the measured second pass, Givens rotations and the
 * stopping test are per column exactly as in hg_gmres; a converged column
 * drops out of the Arnoldi kernels.  rhs / x: device batches (ldr, ldx).
 * history: host, nrhs * (maxit+1) doubles (column c at c*(maxit+1));
 * info: host, nrhs * 4 ints (as hg_gmres, column c at 4c).  The Krylov
 * bases live in a virtual reservation that is backed by device memory only
 * as far as the iterations actually reach.  maxit is capped at 1024 (the
 * basis kernels keep their coefficients in shared memory): a larger
 * min(maxit, n) returns HG_ERR_UNSUPPORTED before any work (hg_gmres too). */
int hg_gmres_batch(HgOp* op, HgOp* weight, const double* rhs, int64_t ldr, double* x, int64_t ldx, int32_t nrhs,
                   double rtol, int32_t maxit, double* history, int32_t* info, void* stream);

/* Orthogonalisation of hg_gmres / hg_gmres_batch (process-wide setting):
 * HG_ORTH_MEASURED mirrors wgmres.py:130-156 decision for decision — a
 *   classical pass, the measurement corr = (W V)^T w, and a second pass when
 *   max|corr| > 1e-12 ||w||_W (at config 5 it fires on ~80% of iterations);
 * HG_ORTH_DCGS2 (default) always reorthogonalises, one iteration late
 *   (delayed classical Gram-Schmidt twice): the reorthogonalisation dots of
 *   q_j share one basis read with the projection dots of A q_j, and the
 *   correction of q_j shares one basis read with the projection update, so
 *   an iteration reads the basis twice instead of three to four times.
 *   Same Krylov space, CGS2-level orthogonality; the parity bars (iterations
 *   +-1, solution 1e-8) are tested against the reference for both modes. */
#define HG_ORTH_MEASURED 0
#define HG_ORTH_DCGS2 1
/* per host thread (the bindings set it around one call) */
int hg_set_orthogonalization(int mode);
int hg_get_orthogonalization(void);
/* DCGS2 safety: when rho^2 = a_j - s.s <= 1e-8 a_j (cancellation: q_j
 * nearly in span Q), that column takes an explicit pass instead (q_j -= Q s
 * on the device, rho measured as ||q_j||_W directly).  Process-wide count of
 * such passes; each also counts in the column's info[3]. */
int64_t hg_dcgs2_explicit_passes(void);

/* Test hooks (no reference analogue).  Keys:
 *   HG_DEBUG_SPIN_LIMIT_MS     process-wide bound of device-side waits, ms
 *                              (0 = unbounded; default 10000)
 *   HG_DEBUG_SKIP_ZT           drop the next `value` Z^T r launches of handle
 *                              p (fault injection: the paired coarse solve
 *                              must time out and poison p, not hang)
 *   HG_DEBUG_FORCE_EXPLICIT_RHO  DCGS2 takes the explicit rho pass on every
 *                              column and iteration (value != 0) */
#define HG_DEBUG_SPIN_LIMIT_MS 1
#define HG_DEBUG_SKIP_ZT 2
#define HG_DEBUG_FORCE_EXPLICIT_RHO 3
/* 0: the single-RHS coarse solve runs the full panel chain even when the handle has the bisected one */
#define HG_DEBUG_B0_SPLIT 4
/* ring stages of the single-RHS local solve (4..6; fewer stages = less shared memory = more CTAs
 * per SM beside the coarse chains) */
#define HG_DEBUG_LOCAL_STAGES 5
/* tile ring stages of the cluster coarse chain (2..4; 2 leaves room for a local-solve CTA on its SMs) */
#define HG_DEBUG_B0_TILE_STAGES 6
int hg_debug_set(HgPrecond* p, int32_t key, int64_t value);

/* Krylov basis of the last hg_gmres / hg_gmres_batch solve on `op`
 * (inspection hook, mirrors test_wgmres.py:35-52): copies basis vectors
 * 0..nv-1 of column `col` into out (device, nv x n, vector i at out + i*n).
 * nv must not exceed the vectors the solve produced (its iterations). */
int hg_op_basis(HgOp* op, int32_t col, int32_t nv, double* out, void* stream);

/* Phase timing of hg_gmres / hg_gmres_batch (measurement hook, used by
 * bench.py to time kernels live inside its timed region).  While enabled,
 * each phase of each iteration is bracketed by CUDA events on the solve's
 * stream; the elapsed device times are summed when the solve synchronises.
 * Phases: 0 operator apply (B SpMV + preconditioner, with the fused
 * projection dots of the single-RHS measured path), 1 projection dots
 * h = (W V)^T w, 2 CGS update w -= V h, 3 measurement (corr dots + W SpMV +
 * norm), 4 second pass, 5 append V_{j+1}, W V_{j+1}, 6 the W w SpMV feeding
 * the dots.  In DCGS2 mode 1 = the fused reorthogonalisation/projection dots
 * (k_dots2_batch + its reduction), 2 = the fused update (k_dcgs2_update),
 * 3 = W SpMV + norm of the projected vector, 4 unused. */
#define HG_NPHASES 7
int hg_stats_enable(int on);
/* ms, count: host arrays of HG_NPHASES; reset != 0 clears the accumulators. */
int hg_stats_read(double* ms, int64_t* count, int reset);

/* End-to-end solve with HOST buffers (the drop-in for cli.py:297-307):
 * f (host, n) -> x (host, n); rhs_p = M^{-1} f ; x = GMRES(M^{-1}B, rhs_p,
 * weight D_k).  H2D and D2H copies are inside the call. */
int hg_solve_host(HgPrecond* p, const double* f_host, double* x_host, double rtol, int32_t maxit,
                  double* history, int32_t* info, void* stream);

/* Batched end-to-end solve with HOST buffers: F (host, column c at F + c*n)
 * -> X (host, same layout); rhs_p = M^{-1} F and the batched GMRES. */
int hg_solve_host_batch(HgPrecond* p, const double* F_host, double* X_host, int32_t nrhs, double rtol,
                        int32_t maxit, double* history, int32_t* info, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HELMGPU_H */
