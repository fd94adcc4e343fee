// C ABI of the solve phase: handle construction (upload of the setup
// products), preconditioner applies, device operators and the weighted GMRES
// driver (Arnoldi on the device, Givens rotations and the stopping test on
// the host, as the north star prescribes).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "hg_internal.cuh"

namespace hg {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
void count_launch(int n) { g_launches += n; }

template <typename T>
static int upload(T** dptr, const T* host, size_t count, long long* bytes) {
  *dptr = nullptr;
  if (count == 0) return HG_OK;
  HG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dptr), sizeof(T) * count));
  if (host) HG_CUDA_TRY(cudaMemcpy(*dptr, host, sizeof(T) * count, cudaMemcpyHostToDevice));
  if (bytes) *bytes += (long long)(sizeof(T) * count);
  return HG_OK;
}

template <typename T>
static void release(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

}  // namespace hg

using namespace hg;

// ------------------------------------------------------------------ operators
struct Workspace {
  int n = 0, cap = 0;          // basis capacity (vectors)
  bool weighted = false;
  double* V = nullptr;
  double* WV = nullptr;
  double* w = nullptr;
  double* ww = nullptr;
  double* partials = nullptr;
  long long partials_len = 0;
  double* dh = nullptr;        // reduced [self, dots...] after the op
  double* dc = nullptr;        // reduced [w.Ww, corr...]
  double* dy = nullptr;        // solution coefficients
  double* hbuf = nullptr;      // pinned host mirror
  ~Workspace() {
    release(V);
    release(WV);
    release(w);
    release(ww);
    release(partials);
    release(dh);
    release(dc);
    release(dy);
    if (hbuf) cudaFreeHost(hbuf);
  }
};

struct HgOp {
  int kind = 0;  // 0: owned CSR; 1: preconditioner-backed
  int n = 0;
  DevCsr csr;
  HgPrecond* P = nullptr;
  int mode = 0;
  Workspace ws;
};

// True under CUDA tool injection (Nsight Compute sets NV_NSIGHT_INJECTION_*,
// the sanitizer NV_SANITIZER_*, others CUDA_INJECTION64_PATH), with
// CUDA_LAUNCH_BLOCKING=1, or HG_SERIAL_APPLY=1: such tools serialise kernels.
extern "C" char** environ;
static bool serial_kernels() {
  static const bool s = [] {
    const char* b = getenv("CUDA_LAUNCH_BLOCKING");
    const char* c = getenv("HG_SERIAL_APPLY");
    if ((b && b[0] == '1') || (c && c[0] == '1')) return true;
    for (char** e = environ; e && *e; ++e) {
      if (!strncmp(*e, "NV_NSIGHT_INJECTION", 19) || !strncmp(*e, "NV_SANITIZER", 12) ||
          !strncmp(*e, "CUDA_INJECTION64_PATH=", 22) || !strncmp(*e, "NV_TPS_LAUNCH_TOKEN", 19))
        return true;
    }
    return false;
  }();
  return s;
}

static int precond_apply_core(HgPrecond* P, const double* r, double* out, const double* W, long long ldw,
                              int nv, double* partials, int* nb, cudaStream_t st) {
  if (P->m > 0) {
    HG_CUDA_TRY(cudaEventRecord(P->ev_fork, st));
    HG_CUDA_TRY(cudaStreamWaitEvent(P->aux, P->ev_fork, 0));
    if (serial_kernels()) {
      // tools that serialise kernels (profilers, sanitizers, blocking launches):
      // no kernel may wait on a later one
      HG_TRY(launch_zt(P, r, P->aux));
      HG_TRY(launch_coarse_solve(P, P->aux, P->zt_epoch));
    } else {
      // The latency-bound coarse solve is launched FIRST (side stream) so that
      // it holds its SMs before the local solves fill the GPU; it starts its
      // work when this apply's Z^T r chunks are all counted (device-side wait).
      HG_TRY(launch_coarse_solve(P, P->aux, P->zt_epoch + (unsigned long long)P->n_zt_items));
    }
    HG_TRY(launch_zy(P, P->aux));
    HG_CUDA_TRY(cudaEventRecord(P->ev_join, P->aux));
    if (!serial_kernels()) HG_TRY(launch_zt(P, r, st));
  }
  HG_TRY(launch_local_solve(P, r, st));
  if (P->m > 0) HG_CUDA_TRY(cudaStreamWaitEvent(st, P->ev_join, 0));
  return launch_assemble(P, true, true, out, W, ldw, nv, partials, nb, st);
}

// y = op(x); when partials != null also the fused dots of y against W[0..nv)
// (slot 0 = y.y for precond ops / x.y for CSR ops; slots 1.. = W_i.y).
static int op_apply_dots(HgOp* op, const double* x, double* y, const double* W, long long ldw, int nv,
                         double* partials, int* nb, cudaStream_t st) {
  if (op->kind == 0) {
    if (!partials) return launch_spmv(op->csr, op->csr.data, x, y, st);
    return launch_spmv_dots(op->csr, op->csr.data, x, y, W, ldw, nv, true, partials, nb, st);
  }
  HgPrecond* P = op->P;
  switch (op->mode) {
    case 0:
      return precond_apply_core(P, x, y, W, ldw, nv, partials, nb, st);
    case 1:
      HG_TRY(launch_spmv(P->A, P->A.data, x, P->d_tmp, st));
      return precond_apply_core(P, P->d_tmp, y, W, ldw, nv, partials, nb, st);
    case 2:
    case 3: {
      const double* vals = op->mode == 2 ? P->A.data : P->A.data2;
      if (!vals) {
        set_error("operator needs D_k but the handle was created without it");
        return HG_ERR_ARG;
      }
      if (!partials) return launch_spmv(P->A, vals, x, y, st);
      return launch_spmv_dots(P->A, vals, x, y, W, ldw, nv, true, partials, nb, st);
    }
    default:
      set_error("bad operator mode");
      return HG_ERR_ARG;
  }
}

// y = W x with fused self dot (x.y) and dots of x against Wb[0..nv)
static int weight_apply_dots(HgOp* wop, const double* x, double* y, const double* Wb, long long ldw, int nv,
                             double* partials, int* nb, cudaStream_t st) {
  const DevCsr* A;
  const double* vals;
  if (wop->kind == 0) {
    A = &wop->csr;
    vals = wop->csr.data;
  } else if (wop->mode == 2 || wop->mode == 3) {
    A = &wop->P->A;
    vals = wop->mode == 2 ? wop->P->A.data : wop->P->A.data2;
  } else {
    set_error("weight must be a matrix operator (CSR, B or D_k)");
    return HG_ERR_ARG;
  }
  if (!vals) {
    set_error("weight operator has no values");
    return HG_ERR_ARG;
  }
  return launch_spmv_dots(*A, vals, x, y, Wb, ldw, nv, false, partials, nb, st);
}

static int ws_reserve(Workspace& ws, int n, int cap, bool weighted) {
  if (ws.n == n && ws.cap >= cap && ws.weighted == weighted) return HG_OK;
  ws.~Workspace();
  new (&ws) Workspace();
  ws.n = n;
  ws.cap = cap;
  ws.weighted = weighted;
  const size_t nv = (size_t)n;
  HG_CUDA_TRY(cudaMalloc(&ws.V, sizeof(double) * nv * cap));
  if (weighted) HG_CUDA_TRY(cudaMalloc(&ws.WV, sizeof(double) * nv * cap));
  HG_CUDA_TRY(cudaMalloc(&ws.w, sizeof(double) * nv));
  HG_CUDA_TRY(cudaMalloc(&ws.ww, sizeof(double) * nv));
  const int nb = std::max(spmv_dots_nblocks(n), assemble_nblocks(n));
  ws.partials_len = (long long)nb * (cap + 2);
  HG_CUDA_TRY(cudaMalloc(&ws.partials, sizeof(double) * ws.partials_len));
  HG_CUDA_TRY(cudaMalloc(&ws.dh, sizeof(double) * (cap + 2)));
  HG_CUDA_TRY(cudaMalloc(&ws.dc, sizeof(double) * (cap + 2)));
  HG_CUDA_TRY(cudaMalloc(&ws.dy, sizeof(double) * (cap + 2)));
  HG_CUDA_TRY(cudaMallocHost(&ws.hbuf, sizeof(double) * 2 * (cap + 2)));
  return HG_OK;
}

extern "C" {

int hg_abi_version(void) { return HG_ABI_VERSION; }
const char* hg_last_error(void) { return g_err.c_str(); }
int64_t hg_kernel_launches(void) { return g_launches.load(); }
int hg_device_sync(void) {
  HG_CUDA_TRY(cudaDeviceSynchronize());
  return HG_OK;
}

int hg_precond_destroy(HgPrecond* P) {
  if (!P) return HG_OK;
  release(P->A.indptr);
  release(P->A.indices);
  release(P->A.data);
  release(P->A.data2);
  release(P->d_local);
  release(P->d_local_idx);
  release(P->d_fwd);
  release(P->d_bwd);
  release(P->d_xs);
  release(P->d_lptr);
  release(P->d_lent);
  release(P->d_cblk);
  release(P->d_cblk_idx);
  release(P->d_z);
  release(P->d_cpart);
  release(P->d_col_blk);
  release(P->d_zt_items);
  release(P->d_b0_perm);
  release(P->d_b0_dinv);
  release(P->d_b0_tile_ptr);
  release(P->d_b0_tile_col);
  release(P->d_b0_tiles);
  release(P->d_b0_x);
  release(P->d_b0_done);
  release(P->d_zt_done);
  release(P->d_y);
  release(P->d_zs);
  release(P->d_cptr);
  release(P->d_cent);
  release(P->d_tmp);
  if (P->aux) cudaStreamDestroy(P->aux);
  if (P->ev_fork) cudaEventDestroy(P->ev_fork);
  if (P->ev_join) cudaEventDestroy(P->ev_join);
  delete P->op_T;
  delete P->op_W;
  delete P;
  return HG_OK;
}

static int build_contrib(int n, int nblk, const int64_t* off, const int32_t* idx, std::vector<int>& ptr,
                         std::vector<long long>& ent) {
  ptr.assign((size_t)n + 1, 0);
  const long long total = off[nblk];
  for (long long e = 0; e < total; ++e) {
    const int d = idx[e];
    if (d < 0 || d >= n) {
      set_error("subdomain index out of range");
      return HG_ERR_ARG;
    }
    ptr[d + 1]++;
  }
  for (int d = 0; d < n; ++d) ptr[d + 1] += ptr[d];
  ent.assign((size_t)total, 0);
  std::vector<int> fill(ptr.begin(), ptr.end() - 1);
  for (int b = 0; b < nblk; ++b)  // block order = fixed summation order
    for (long long e = off[b]; e < off[b + 1]; ++e) ent[fill[idx[e]]++] = e;
  return HG_OK;
}

static int precond_create_impl(const HgPrecondDesc* D, HgPrecond* P) {
  long long* bytes = &P->device_bytes;
  const int n = D->n;
  P->n = n;
  if (n <= 0 || !D->indptr || !D->indices || !D->b_data) {
    set_error("hg_precond_create: missing global CSR");
    return HG_ERR_ARG;
  }
  P->A.n = n;
  P->A.nnz = D->nnz;
  HG_TRY(upload(&P->A.indptr, D->indptr, (size_t)n + 1, bytes));
  HG_TRY(upload(&P->A.indices, D->indices, (size_t)D->nnz, bytes));
  HG_TRY(upload(&P->A.data, D->b_data, (size_t)D->nnz, bytes));
  if (D->dk_data) HG_TRY(upload(&P->A.data2, D->dk_data, (size_t)D->nnz, bytes));
  HG_TRY(upload<double>(&P->d_tmp, nullptr, (size_t)n, bytes));

  // ---- local blocks
  P->n_local = D->n_local;
  int max_kl = 0, max_kv = 0;
  P->h_local.resize(D->n_local);
  for (int s = 0; s < D->n_local; ++s) {
    LocalDesc& d = P->h_local[s];
    d.n = D->local_n[s];
    d.kl = D->local_kl[s];
    d.kv = D->local_kv[s];
    d.fstride = D->local_fstride[s];
    d.bstride = D->local_bstride[s];
    d.pad = 0;
    d.idx_off = D->local_idx_off[s];
    d.fwd_off = D->local_fwd_off[s];
    d.bwd_off = D->local_bwd_off[s];
    if (d.n != D->local_idx_off[s + 1] - D->local_idx_off[s] || d.fstride < d.kl + 1 ||
        d.bstride < d.kv + 1 || (d.fstride & 1) || (d.bstride & 1) || (d.fwd_off & 1) || (d.bwd_off & 1)) {
      set_error("hg_precond_create: inconsistent local block descriptor " + std::to_string(s));
      return HG_ERR_ARG;
    }
    max_kl = std::max(max_kl, d.kl);
    max_kv = std::max(max_kv, d.kv);
    P->max_fstride = std::max(P->max_fstride, d.fstride);
    P->max_bstride = std::max(P->max_bstride, d.bstride);
  }
  P->rf = std::max(2, 1 + (max_kl + 31) / 32);
  P->rb = std::max(2, 1 + (max_kv + 31) / 32);
  if (D->n_local > 0 && (P->rf > 6 || P->rb > 10)) {
    set_error("hg_precond_create: local bandwidth kl=" + std::to_string(max_kl) + ", kv=" +
              std::to_string(max_kv) + " beyond compiled tiles (kl <= 160, kv <= 288)");
    return HG_ERR_UNSUPPORTED;
  }
  if (D->n_local > 0) {
    const long long nidx = D->local_idx_off[D->n_local];
    P->xs_len = nidx;
    HG_TRY(upload(&P->d_local, P->h_local.data(), P->h_local.size(), bytes));
    HG_TRY(upload(&P->d_local_idx, D->local_idx, (size_t)nidx, bytes));
    HG_TRY(upload(&P->d_fwd, D->local_fwd, (size_t)D->local_fwd_len, bytes));
    HG_TRY(upload(&P->d_bwd, D->local_bwd, (size_t)D->local_bwd_len, bytes));
    HG_TRY(upload<double>(&P->d_xs, nullptr, (size_t)nidx, bytes));
    std::vector<int> ptr;
    std::vector<long long> ent;
    HG_TRY(build_contrib(n, D->n_local, D->local_idx_off, D->local_idx, ptr, ent));
    HG_TRY(upload(&P->d_lptr, ptr.data(), ptr.size(), bytes));
    HG_TRY(upload(&P->d_lent, ent.data(), ent.size(), bytes));
  }

  // ---- coarse part
  P->m = D->m;
  P->n_cblk = D->n_cblk;
  if (P->m > 0) {
    std::vector<CblkDesc> cb(D->n_cblk);
    std::vector<int> col_blk(P->m);
    std::vector<int2> items;
    int col = 0;
    long long part = 0;
    for (int b = 0; b < D->n_cblk; ++b) {
      CblkDesc& d = cb[b];
      d.n = D->cblk_n[b];
      d.m = D->cblk_m[b];
      d.col0 = col;
      d.nchunk = d.m > 0 ? (d.n + 255) / 256 : 0;
      d.idx_off = D->cblk_idx_off[b];
      d.z_off = D->cblk_z_off[b];
      d.part_off = part;
      if (d.n != D->cblk_idx_off[b + 1] - D->cblk_idx_off[b]) {
        set_error("hg_precond_create: inconsistent coarse block " + std::to_string(b));
        return HG_ERR_ARG;
      }
      for (int l = 0; l < d.m; ++l) col_blk[col + l] = b;
      for (int c = 0; c < d.nchunk; ++c) items.push_back(make_int2(b, c));
      col += d.m;
      part += (long long)d.nchunk * d.m;
    }
    if (col != P->m) {
      set_error("hg_precond_create: coarse block widths do not add up to m");
      return HG_ERR_ARG;
    }
    P->h_cblk = cb;
    P->part_len = part;
    P->n_zt_items = (int)items.size();
    const long long nidx = D->cblk_idx_off[D->n_cblk];
    P->zs_len = nidx;
    HG_TRY(upload(&P->d_cblk, cb.data(), cb.size(), bytes));
    HG_TRY(upload(&P->d_cblk_idx, D->cblk_idx, (size_t)nidx, bytes));
    HG_TRY(upload(&P->d_z, D->z_data, (size_t)D->z_len, bytes));
    HG_TRY(upload<double>(&P->d_cpart, nullptr, (size_t)std::max(part, 1LL), bytes));
    HG_TRY(upload(&P->d_col_blk, col_blk.data(), col_blk.size(), bytes));
    HG_TRY(upload(&P->d_zt_items, items.data(), items.size(), bytes));
    HG_TRY(upload(&P->d_b0_perm, D->b0_perm, (size_t)P->m, bytes));
    const int bp = D->b0_panel, bk = D->b0_npanel;
    if ((bp != 32 && bp != 64 && bp != 128) || (long long)bk * bp < P->m || (long long)(bk - 1) * bp >= P->m ||
        !D->b0_dinv || !D->b0_tile_ptr || D->b0_tile_ptr[2 * bk] != D->b0_ntile) {
      set_error("hg_precond_create: inconsistent coarse tile description");
      return HG_ERR_ARG;
    }
    P->b0_P = bp;
    P->b0_K = bk;
    P->b0_ctas = D->b0_ctas > 0 ? D->b0_ctas : 32;
    P->b0_mode = D->b0_mode;
    if (P->b0_mode == 1) {
      P->b0_cs = D->b0_cluster;
      P->b0_nr = D->b0_ring;
      if (bp != 64 || P->b0_cs < 1 || P->b0_cs > 16 || P->b0_nr < P->b0_cs + 1 ||
          b0_cluster_smem(P->b0_nr) > 227 * 1024) {
        set_error("hg_precond_create: invalid cluster coarse-solve parameters");
        return HG_ERR_ARG;
      }
    }
    HG_TRY(upload(&P->d_b0_dinv, D->b0_dinv, (size_t)2 * bk * bp * bp, bytes));
    HG_TRY(upload(&P->d_b0_tile_ptr, reinterpret_cast<const long long*>(D->b0_tile_ptr), (size_t)2 * bk + 1, bytes));
    if (D->b0_ntile > 0) {
      HG_TRY(upload(&P->d_b0_tile_col, D->b0_tile_col, (size_t)D->b0_ntile, bytes));
      HG_TRY(upload(&P->d_b0_tiles, D->b0_tiles, (size_t)D->b0_ntile * bp * bp, bytes));
    }
    HG_TRY(upload<double>(&P->d_b0_x, nullptr, (size_t)2 * bk * bp, bytes));
    HG_TRY(upload<unsigned long long>(&P->d_b0_done, nullptr, 1, bytes));
    HG_CUDA_TRY(cudaMemset(P->d_b0_done, 0, sizeof(unsigned long long)));
    HG_TRY(upload<unsigned long long>(&P->d_zt_done, nullptr, 1, bytes));
    HG_CUDA_TRY(cudaMemset(P->d_zt_done, 0, sizeof(unsigned long long)));
    P->zt_epoch = 0;
    P->b0_epoch = 0;
    HG_TRY(upload<double>(&P->d_y, nullptr, (size_t)P->m, bytes));
    HG_TRY(upload<double>(&P->d_zs, nullptr, (size_t)std::max(nidx, 1LL), bytes));
    std::vector<int> ptr;
    std::vector<long long> ent;
    HG_TRY(build_contrib(n, D->n_cblk, D->cblk_idx_off, D->cblk_idx, ptr, ent));
    HG_TRY(upload(&P->d_cptr, ptr.data(), ptr.size(), bytes));
    HG_TRY(upload(&P->d_cent, ent.data(), ent.size(), bytes));
  }
  HG_TRY(preload_local(P));
  HG_TRY(preload_coarse());
  HG_TRY(preload_assemble());
  HG_TRY(preload_b0());
  HG_TRY(preload_vec());
  HG_CUDA_TRY(cudaStreamCreateWithFlags(&P->aux, cudaStreamNonBlocking));
  HG_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
  HG_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming));
  HG_CUDA_TRY(cudaDeviceSynchronize());
  return HG_OK;
}

int hg_precond_create(const HgPrecondDesc* desc, HgPrecond** out) {
  if (!desc || !out) {
    set_error("hg_precond_create: null argument");
    return HG_ERR_ARG;
  }
  HgPrecond* P = new HgPrecond();
  int s = precond_create_impl(desc, P);
  if (s != HG_OK) {
    hg_precond_destroy(P);
    *out = nullptr;
    return s;
  }
  *out = P;
  return HG_OK;
}

int64_t hg_precond_device_bytes(const HgPrecond* P) { return P ? P->device_bytes : 0; }

int hg_precond_apply(HgPrecond* P, const double* r, double* out, void* stream) {
  if (!P || !r || !out) {
    set_error("hg_precond_apply: null argument");
    return HG_ERR_ARG;
  }
  return precond_apply_core(P, r, out, nullptr, 0, 0, nullptr, nullptr, (cudaStream_t)stream);
}

int hg_precond_apply_T(HgPrecond* P, const double* u, double* out, void* stream) {
  if (!P || !u || !out) {
    set_error("hg_precond_apply_T: null argument");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  HG_TRY(launch_spmv(P->A, P->A.data, u, P->d_tmp, st));
  return precond_apply_core(P, P->d_tmp, out, nullptr, 0, 0, nullptr, nullptr, st);
}

int hg_precond_apply_coarse(HgPrecond* P, const double* r, double* out, void* stream) {
  if (!P || !r || !out) {
    set_error("hg_precond_apply_coarse: null argument");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (P->m == 0) return launch_fill(P->n, out, 0.0, st);
  HG_TRY(launch_zt(P, r, st));
  HG_TRY(launch_coarse_solve(P, st, P->zt_epoch));
  HG_TRY(launch_zy(P, st));
  return launch_assemble(P, true, false, out, nullptr, 0, 0, nullptr, nullptr, st);
}

int hg_precond_profile(HgPrecond* P, const double* r, double* out, int32_t iters, double* stage_ms,
                       void* stream) {
  if (!P || !r || !out || !stage_ms || iters <= 0) {
    set_error("hg_precond_profile: bad argument");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t ev[HG_NSTAGES + 1];
  for (auto& e : ev) HG_CUDA_TRY(cudaEventCreate(&e));
  double acc[HG_NSTAGES] = {0, 0, 0, 0, 0};
  int status = HG_OK;
  for (int it = 0; it < iters && status == HG_OK; ++it) {
    cudaEventRecord(ev[0], st);
    if ((status = launch_zt(P, r, st)) != HG_OK) break;
    cudaEventRecord(ev[1], st);
    if ((status = launch_coarse_solve(P, st, P->zt_epoch)) != HG_OK) break;
    cudaEventRecord(ev[2], st);
    if ((status = launch_zy(P, st)) != HG_OK) break;
    cudaEventRecord(ev[3], st);
    if ((status = launch_local_solve(P, r, st)) != HG_OK) break;
    cudaEventRecord(ev[4], st);
    if ((status = launch_assemble(P, true, true, out, nullptr, 0, 0, nullptr, nullptr, st)) != HG_OK) break;
    cudaEventRecord(ev[5], st);
    if (cudaEventSynchronize(ev[5]) != cudaSuccess) {
      set_error("hg_precond_profile: event sync failed");
      status = HG_ERR_CUDA;
      break;
    }
    for (int s = 0; s < HG_NSTAGES; ++s) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[s], ev[s + 1]);
      acc[s] += ms;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int s = 0; s < HG_NSTAGES; ++s) stage_ms[s] = acc[s] / iters;
  return status;
}

int hg_precond_spmv(HgPrecond* P, int which, const double* x, double* y, void* stream) {
  if (!P || !x || !y || (which != 0 && which != 1)) {
    set_error("hg_precond_spmv: bad argument");
    return HG_ERR_ARG;
  }
  const double* vals = which == 0 ? P->A.data : P->A.data2;
  if (!vals) {
    set_error("hg_precond_spmv: D_k not uploaded");
    return HG_ERR_ARG;
  }
  return launch_spmv(P->A, vals, x, y, (cudaStream_t)stream);
}

int hg_local_solve(HgPrecond* P, int s, const double* r_local, double* x_local, void* stream) {
  if (!P || s < 0 || s >= P->n_local || !r_local || !x_local) {
    set_error("hg_local_solve: bad argument");
    return HG_ERR_ARG;
  }
  return launch_local_solve_single(P, s, r_local, x_local, (cudaStream_t)stream);
}

int hg_op_create_csr(int32_t n, int64_t nnz, const int32_t* indptr, const int32_t* indices, const double* data,
                     HgOp** out) {
  if (!out || n <= 0 || !indptr || (nnz > 0 && (!indices || !data))) {
    set_error("hg_op_create_csr: bad argument");
    return HG_ERR_ARG;
  }
  HgOp* op = new HgOp();
  op->kind = 0;
  op->n = n;
  op->csr.n = n;
  op->csr.nnz = nnz;
  int s = HG_OK;
  if ((s = upload(&op->csr.indptr, indptr, (size_t)n + 1, nullptr)) != HG_OK ||
      (s = upload(&op->csr.indices, indices, (size_t)nnz, nullptr)) != HG_OK ||
      (s = upload(&op->csr.data, data, (size_t)nnz, nullptr)) != HG_OK) {
    hg_op_destroy(op);
    return s;
  }
  *out = op;
  return HG_OK;
}

int hg_op_create_precond(HgPrecond* P, int mode, HgOp** out) {
  if (!P || !out || mode < 0 || mode > 3) {
    set_error("hg_op_create_precond: bad argument");
    return HG_ERR_ARG;
  }
  HgOp* op = new HgOp();
  op->kind = 1;
  op->n = P->n;
  op->P = P;
  op->mode = mode;
  *out = op;
  return HG_OK;
}

int hg_op_destroy(HgOp* op) {
  if (!op) return HG_OK;
  if (op->kind == 0) {
    release(op->csr.indptr);
    release(op->csr.indices);
    release(op->csr.data);
  }
  delete op;
  return HG_OK;
}

int hg_op_apply(HgOp* op, const double* x, double* y, void* stream) {
  if (!op || !x || !y) {
    set_error("hg_op_apply: null argument");
    return HG_ERR_ARG;
  }
  return op_apply_dots(op, x, y, nullptr, 0, 0, nullptr, nullptr, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ GMRES
// Restates wgmres.weighted_gmres (wgmres.py:74-203): classical Gram-Schmidt
// with the reference's measured, conditional second pass (the measurement
// corr = (W V)^T w is always taken, as wgmres.py:142), W-norm via one weight
// SpMV fused with the measurement, Givens rotations and the stopping rule on
// the host with the reference's exact arithmetic.
int hg_gmres(HgOp* op, HgOp* weight, const double* rhs, const double* x0, double* x, double rtol, int32_t maxit,
             double* history, int32_t* info, void* stream) {
  if (!op || !rhs || !x || !history || !info) {
    set_error("hg_gmres: null argument");
    return HG_ERR_ARG;
  }
  if (weight && weight->n != op->n) {
    set_error("hg_gmres: weight dimension mismatch");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n = op->n;
  maxit = std::max(0, std::min(maxit, n));
  Workspace& ws = op->ws;
  const bool weighted = weight != nullptr;
  HG_TRY(ws_reserve(ws, n, maxit + 1, weighted));
  double* V = ws.V;
  double* WV = weighted ? ws.WV : ws.V;
  const long long ld = n;
  double* hb = ws.hbuf;
  int nb = 0;
  info[0] = info[1] = info[2] = info[3] = 0;

  // r0 = rhs - op(x0) (or rhs), wr0 = W r0, beta = sqrt(r0 . wr0)
  if (x0) {
    HG_TRY(op_apply_dots(op, x0, ws.w, nullptr, 0, 0, nullptr, nullptr, st));
    HG_TRY(launch_sub(n, rhs, ws.w, V, st));
  } else {
    HG_CUDA_TRY(cudaMemcpyAsync(V, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  if (weighted)
    HG_TRY(weight_apply_dots(weight, V, WV, nullptr, 0, 0, ws.partials, &nb, st));
  else
    HG_TRY(launch_dots(n, V, nullptr, 0, 0, ws.partials, &nb, st));
  HG_TRY(launch_reduce(ws.partials, nb, 1, ws.dc, st));
  HG_CUDA_TRY(cudaMemcpyAsync(hb, ws.dc, sizeof(double), cudaMemcpyDeviceToHost, st));
  HG_CUDA_TRY(cudaStreamSynchronize(st));
  const double beta = std::sqrt(hb[0]);
  if (beta == 0.0) {
    if (x0)
      HG_CUDA_TRY(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    else
      HG_TRY(launch_fill(n, x, 0.0, st));
    history[0] = 0.0;
    info[0] = 0;
    info[1] = 1;
    HG_CUDA_TRY(cudaStreamSynchronize(st));
    return HG_OK;
  }
  HG_TRY(launch_scale2(n, V, WV, &beta, V, weighted ? WV : nullptr, st));

  std::vector<double> H((size_t)(maxit + 1) * std::max(maxit, 1), 0.0);  // column-major (maxit+1) x maxit
  std::vector<double> cs(maxit, 0.0), sn(maxit, 0.0), g(maxit + 1, 0.0), col(maxit + 2, 0.0);
  g[0] = beta;
  int hist_len = 1;
  history[0] = beta;
  bool converged = false, breakdown = false;
  int reorth = 0;
  const double REORTH_TOL = 1e-12, BREAKDOWN_RTOL = 1e-14;

  for (int j = 0; j < maxit; ++j) {
    const int nv = j + 1;
    double* w = ws.w;
    // w = op(V_j), fused h_i = (W V_i) . w
    HG_TRY(op_apply_dots(op, V + (long long)j * ld, w, WV, ld, nv, ws.partials, &nb, st));
    HG_TRY(launch_reduce(ws.partials, nb, nv + 1, ws.dh, st));
    // classical GS pass: w -= V h
    HG_TRY(launch_axpy_multi(n, w, V, ld, nv, ws.dh + 1, 1, st));
    // ww = W w with w.ww and the measurement corr_i = (W V_i) . w
    if (weighted)
      HG_TRY(weight_apply_dots(weight, w, ws.ww, WV, ld, nv, ws.partials, &nb, st));
    else
      HG_TRY(launch_dots(n, w, V, ld, nv, ws.partials, &nb, st));
    HG_TRY(launch_reduce(ws.partials, nb, nv + 1, ws.dc, st));
    HG_CUDA_TRY(cudaMemcpyAsync(hb, ws.dh + 1, sizeof(double) * nv, cudaMemcpyDeviceToHost, st));
    HG_CUDA_TRY(cudaMemcpyAsync(hb + nv, ws.dc, sizeof(double) * (nv + 1), cudaMemcpyDeviceToHost, st));
    HG_CUDA_TRY(cudaStreamSynchronize(st));
    for (int i = 0; i < nv; ++i) col[i] = hb[i];
    double hnorm = std::sqrt(std::max(hb[nv], 0.0));
    double cmax = 0.0;
    for (int i = 0; i < nv; ++i) cmax = std::max(cmax, std::fabs(hb[nv + 1 + i]));
    if (cmax > REORTH_TOL * std::max(hnorm, 1e-300)) {
      for (int i = 0; i < nv; ++i) col[i] += hb[nv + 1 + i];
      HG_TRY(launch_axpy_multi(n, w, V, ld, nv, ws.dc + 1, 1, st));
      if (weighted)
        HG_TRY(weight_apply_dots(weight, w, ws.ww, nullptr, 0, 0, ws.partials, &nb, st));
      else
        HG_TRY(launch_dots(n, w, nullptr, 0, 0, ws.partials, &nb, st));
      HG_TRY(launch_reduce(ws.partials, nb, 1, ws.dc, st));
      HG_CUDA_TRY(cudaMemcpyAsync(hb, ws.dc, sizeof(double), cudaMemcpyDeviceToHost, st));
      HG_CUDA_TRY(cudaStreamSynchronize(st));
      hnorm = std::sqrt(std::max(hb[0], 0.0));
      ++reorth;
    }
    col[j + 1] = hnorm;
    double cscale = 0.0;
    for (int i = 0; i <= j + 1; ++i) cscale = std::max(cscale, std::fabs(col[i]));
    if (hnorm <= BREAKDOWN_RTOL * std::max(cscale, 1e-300)) {
      breakdown = true;
    } else {
      HG_TRY(launch_scale2(n, w, weighted ? ws.ww : w, &hnorm, V + (long long)(j + 1) * ld,
                           weighted ? WV + (long long)(j + 1) * ld : nullptr, st));
    }
    // Givens update of the new Hessenberg column (wgmres.py:158-171)
    for (int i = 0; i < j; ++i) {
      const double t = cs[i] * col[i] - sn[i] * col[i + 1];
      col[i + 1] = sn[i] * col[i] + cs[i] * col[i + 1];
      col[i] = t;
    }
    const double denom = std::hypot(col[j], col[j + 1]);
    if (denom == 0.0) {
      cs[j] = 1.0;
      sn[j] = 0.0;
    } else {
      cs[j] = col[j] / denom;
      sn[j] = -col[j + 1] / denom;
    }
    col[j] = cs[j] * col[j] - sn[j] * col[j + 1];
    col[j + 1] = 0.0;
    for (int i = 0; i <= j + 1; ++i) H[(size_t)j * (maxit + 1) + i] = col[i];
    g[j + 1] = sn[j] * g[j];
    g[j] = cs[j] * g[j];
    history[hist_len++] = std::fabs(g[j + 1]);
    if (history[hist_len - 1] <= rtol * beta) {
      converged = true;
      break;
    }
    if (breakdown) {
      converged = true;
      break;
    }
  }
  const int m = hist_len - 1;
  // y = H[:m,:m]^{-1} g[:m] (upper triangular back substitution, host)
  std::vector<double> y(m, 0.0);
  for (int i = m - 1; i >= 0; --i) {
    double s = g[i];
    for (int k = i + 1; k < m; ++k) s -= H[(size_t)k * (maxit + 1) + i] * y[k];
    y[i] = s / H[(size_t)i * (maxit + 1) + i];
  }
  if (x0)
    HG_CUDA_TRY(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  if (m > 0) {
    for (int i = 0; i < m; ++i) hb[i] = y[i];
    HG_CUDA_TRY(cudaMemcpyAsync(ws.dy, hb, sizeof(double) * m, cudaMemcpyHostToDevice, st));
    HG_TRY(launch_axpy_multi(n, x, V, ld, m, ws.dy, x0 ? 2 : 0, st));
  } else if (!x0) {
    HG_TRY(launch_fill(n, x, 0.0, st));
  }
  HG_CUDA_TRY(cudaStreamSynchronize(st));
  info[0] = m;
  info[1] = converged ? 1 : 0;
  info[2] = breakdown ? 1 : 0;
  info[3] = reorth;
  return HG_OK;
}

int hg_solve_host(HgPrecond* P, const double* f_host, double* x_host, double rtol, int32_t maxit,
                  double* history, int32_t* info, void* stream) {
  if (!P || !f_host || !x_host) {
    set_error("hg_solve_host: null argument");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n = P->n;
  if (!P->op_T) {
    HgOp* t = new HgOp();
    t->kind = 1;
    t->n = n;
    t->P = P;
    t->mode = 1;
    HgOp* w = new HgOp();
    w->kind = 1;
    w->n = n;
    w->P = P;
    w->mode = 3;
    P->op_T = t;
    P->op_W = w;
  }
  double *d_f = nullptr, *d_rhs = nullptr, *d_x = nullptr;
  HG_CUDA_TRY(cudaMallocAsync(&d_f, sizeof(double) * n, st));
  HG_CUDA_TRY(cudaMallocAsync(&d_rhs, sizeof(double) * n, st));
  HG_CUDA_TRY(cudaMallocAsync(&d_x, sizeof(double) * n, st));
  HG_CUDA_TRY(cudaMemcpyAsync(d_f, f_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  HG_TRY(precond_apply_core(P, d_f, d_rhs, nullptr, 0, 0, nullptr, nullptr, st));
  int s = hg_gmres(P->op_T, P->A.data2 ? P->op_W : nullptr, d_rhs, nullptr, d_x, rtol, maxit, history, info,
                   stream);
  if (s == HG_OK) {
    HG_CUDA_TRY(cudaMemcpyAsync(x_host, d_x, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(d_f, st);
  cudaFreeAsync(d_rhs, st);
  cudaFreeAsync(d_x, st);
  HG_CUDA_TRY(cudaStreamSynchronize(st));
  return s;
}

}  // extern "C"
