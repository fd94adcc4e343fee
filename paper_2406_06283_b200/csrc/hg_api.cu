// C ABI of the solve phase: handle construction (upload of the setup
// products), preconditioner applies, device operators and the weighted GMRES
// driver (Arnoldi on the device, Givens rotations and the stopping test on
// the host, as the north star prescribes).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>

#include <map>
#include <mutex>
#include <set>

#include "hg_internal.cuh"

namespace hg {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
void count_launch(int n) { g_launches += n; }

// ---- bounded waits and fault injection (hg_debug_set)
static std::atomic<long long> g_spin_limit_ms{10000};  // a coarse-solve wait longer than this is a fault
static std::atomic<int> g_force_explicit_rho{0};      // DCGS2: always take the explicit rho pass
static std::atomic<long long> g_explicit_rho_passes{0};

SpinCfg spin_cfg(const HgPrecond* P) {
  SpinCfg c;
  c.fault = P->d_fault;
  const long long ms = g_spin_limit_ms.load();
  c.limit_ns = ms > 0 ? (unsigned long long)ms * 1000000ull : 0ull;
  return c;
}

// cudaFuncSetAttribute is per device: remember what each (kernel, device)
// was configured with instead of a process-wide static
int ensure_func_attrs(const void* func, size_t smem, bool nonportable_cluster) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  HG_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[std::make_pair(func, dev)];
  if (have >= smem && have != 0) return HG_OK;
  HG_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nonportable_cluster) HG_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  // kernels built around a shared-memory ring ask for the largest carve-out, so that CTAs of two such
  // kernels (a coarse chain and a local solve) can share an SM whenever their rings fit together
  if (smem >= 64 * 1024)
    HG_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
  have = smem > 0 ? smem : 1;
  return HG_OK;
}

template <typename T>
static int upload(T** dptr, const T* host, size_t count, long long* bytes) {
  *dptr = nullptr;
  if (count == 0) return HG_OK;
  HG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dptr), sizeof(T) * count));
  // cudaMemcpyDefault: descriptor arrays may be host or device memory (unified addressing)
  if (host) HG_CUDA_TRY(cudaMemcpy(*dptr, host, sizeof(T) * count, cudaMemcpyDefault));
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

// Device memory that grows on demand inside one virtual reservation (CUDA
// VMM): the batched Krylov bases are reserved for maxit+1 vectors per column
// (up to ~270 GB of address space at config 5) but backed by HBM only as far
// as the iterations reach, so 16 full-GMRES bases fit the 180 GB device.
struct VmBuf {
  CUdeviceptr base = 0;
  size_t reserved = 0, mapped = 0, gran = 0;
  bool plain = false;  // HG_VMM=0: one cudaMalloc of the whole reservation (tools without VMM support)
  std::vector<CUmemGenericAllocationHandle> handles;
  std::vector<size_t> sizes;
  int dev = 0;
  double* ptr() const { return reinterpret_cast<double*>(base); }
  int reserve(size_t bytes);
  int ensure(size_t bytes);
  void free_all();
  ~VmBuf() { free_all(); }
};

struct DrvApi {
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  bool ok = false;
};

static const DrvApi& drv() {
  static DrvApi d = [] {
    DrvApi a;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn != nullptr;
    };
    a.ok = get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&a.granularity)) &&
           get("cuMemAddressReserve", reinterpret_cast<void**>(&a.reserve)) &&
           get("cuMemAddressFree", reinterpret_cast<void**>(&a.addr_free)) &&
           get("cuMemCreate", reinterpret_cast<void**>(&a.create)) &&
           get("cuMemRelease", reinterpret_cast<void**>(&a.release)) &&
           get("cuMemMap", reinterpret_cast<void**>(&a.map)) &&
           get("cuMemUnmap", reinterpret_cast<void**>(&a.unmap)) &&
           get("cuMemSetAccess", reinterpret_cast<void**>(&a.set_access));
    return a;
  }();
  return d;
}

static CUmemAllocationProp vm_prop(int dev) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = dev;
  return p;
}

int VmBuf::reserve(size_t bytes) {
  free_all();
  static const bool no_vmm = getenv("HG_VMM") && getenv("HG_VMM")[0] == '0';
  if (no_vmm) {
    void* p = nullptr;
    HG_CUDA_TRY(cudaMalloc(&p, bytes));
    base = reinterpret_cast<CUdeviceptr>(p);
    reserved = mapped = bytes;
    plain = true;
    return HG_OK;
  }
  const DrvApi& d = drv();
  if (!d.ok) {
    set_error("CUDA virtual memory management entry points unavailable");
    return HG_ERR_UNSUPPORTED;
  }
  HG_CUDA_TRY(cudaGetDevice(&dev));
  CUmemAllocationProp p = vm_prop(dev);
  if (d.granularity(&gran, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || gran == 0) {
    set_error("cuMemGetAllocationGranularity failed");
    return HG_ERR_CUDA;
  }
  reserved = (bytes + gran - 1) / gran * gran;
  if (d.reserve(&base, reserved, 0, 0, 0) != CUDA_SUCCESS) {
    base = 0;
    reserved = 0;
    set_error("cuMemAddressReserve failed");
    return HG_ERR_NOMEM;
  }
  return HG_OK;
}

int VmBuf::ensure(size_t bytes) {
  if (bytes <= mapped) return HG_OK;
  if (bytes > reserved) {
    set_error("VmBuf: request beyond the reservation");
    return HG_ERR_ARG;
  }
  const DrvApi& d = drv();
  const size_t chunk_min = (std::max<size_t>((size_t)256 << 20, reserved / 16) + gran - 1) / gran * gran;
  while (mapped < bytes) {
    size_t sz = std::max(chunk_min, (bytes - mapped + gran - 1) / gran * gran);
    sz = std::min(sz, reserved - mapped);
    CUmemAllocationProp p = vm_prop(dev);
    CUmemGenericAllocationHandle h;
    if (d.create(&h, sz, &p, 0) != CUDA_SUCCESS) {
      set_error("cuMemCreate failed (device memory exhausted by the Krylov bases?)");
      return HG_ERR_NOMEM;
    }
    if (d.map(base + mapped, sz, 0, h, 0) != CUDA_SUCCESS) {
      d.release(h);
      set_error("cuMemMap failed");
      return HG_ERR_CUDA;
    }
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (d.set_access(base + mapped, sz, &acc, 1) != CUDA_SUCCESS) {
      d.unmap(base + mapped, sz);
      d.release(h);
      set_error("cuMemSetAccess failed");
      return HG_ERR_CUDA;
    }
    handles.push_back(h);
    sizes.push_back(sz);
    mapped += sz;
  }
  return HG_OK;
}

static bool g_shutdown = false;  // hg_shutdown: the process is exiting, skip device frees

void VmBuf::free_all() {
  if (!base) return;
  if (g_shutdown) {  // the driver may already be torn down at interpreter exit: leak, the process ends
    base = 0;
    return;
  }
  if (plain) {
    cudaFree(reinterpret_cast<void*>(base));
    base = 0;
    reserved = mapped = 0;
    plain = false;
    return;
  }
  const DrvApi& d = drv();
  cudaDeviceSynchronize();
  size_t off = 0;
  for (size_t i = 0; i < handles.size(); ++i) {
    d.unmap(base + off, sizes[i]);
    d.release(handles[i]);
    off += sizes[i];
  }
  d.addr_free(base, reserved);
  handles.clear();
  sizes.clear();
  base = 0;
  reserved = mapped = 0;
}

// Batched GMRES workspace.  Basis layout [i][c][n]: vector i of column c at
// V + (i * nrhs + c) * n, so the op input of iteration j is one contiguous
// batch (ld n) and the bases grow contiguously.
struct BatchWs {
  int n = 0, nrhs = 0, cap = 0;
  bool weighted = false;
  VmBuf V, WV;
  double* w = nullptr;          // [c][n] op output / Krylov candidate
  double* ww = nullptr;         // [c][n] W w
  double* partials = nullptr;   // [c][nb][cap + 2]
  double* pself = nullptr;      // [c][nb] self-dot partials of the weight SpMM
  double* dh = nullptr;         // [c][cap + 2]
  double* dc = nullptr;         // [c][cap + 2]
  double* dy = nullptr;         // [c][cap + 2]
  double* hbuf = nullptr;       // pinned [2][c][cap + 2]
  ~BatchWs() { clear(); }
  void clear() {
    release(w);
    release(ww);
    release(partials);
    release(pself);
    release(dh);
    release(dc);
    release(dy);
    if (hbuf) cudaFreeHost(hbuf);
    hbuf = nullptr;
    V.free_all();
    WV.free_all();
    n = nrhs = cap = 0;
  }
};

// DCGS2 workspace (single and batched solves).  Basis Q as in BatchWs; no
// cached W Q: the dots read Q against W w (SpMV) and W q_j (kept from the
// previous normalisation), so the basis costs one vector per iteration.
struct DcWs {
  int n = 0, nrhs = 0, cap = 0;
  bool weighted = false;
  VmBuf Q;
  double* w = nullptr;          // [c][n] op output, then the projected vector
  double* u = nullptr;          // [c][n] W w
  double* ww = nullptr;         // [c][n] W w after projection
  double* wq = nullptr;         // [c][n] W q_j (of the not yet reorthogonalised q_j)
  double* partials = nullptr;   // [c][nb][2 (cap + 2)]
  double* pself = nullptr;      // [c][nb256]
  double* dots = nullptr;       // [c][2 (cap + 2)]
  double* nrm2 = nullptr;       // [c] ||w||_W^2 of the last projected vector
  double* coef = nullptr;       // [c][2 (cap + 2)] rinv, s, c
  double* dy = nullptr;         // [c][cap + 2]
  double* hbuf = nullptr;       // pinned: dots [c][2(cap+2)], nrm2 [c], coef [c][2(cap+2)]
  ~DcWs() { clear(); }
  void clear() {
    release(w);
    release(u);
    release(ww);
    release(wq);
    release(partials);
    release(pself);
    release(dots);
    release(nrm2);
    release(coef);
    release(dy);
    if (hbuf) cudaFreeHost(hbuf);
    hbuf = nullptr;
    Q.free_all();
    n = nrhs = cap = 0;
  }
};

struct HgOp {
  int kind = 0;  // 0: owned CSR; 1: preconditioner-backed
  int n = 0;
  DevCsr csr;
  HgPrecond* P = nullptr;
  int mode = 0;
  Workspace ws;
  BatchWs bws;
  DcWs dws;    // one right-hand side
  DcWs dwsb;   // batches
  // basis of the last solve (hg_op_basis): vector i of column c at base + c*ldcol + i*ldv
  const double* basis = nullptr;
  long long basis_ldv = 0, basis_ldcol = 0;
  int basis_cols = 0, basis_nv = 0;
  std::atomic<int> busy{0};  // inside a solve: its workspaces may not be released by another op's memory plan
};

// ---- memory plan of the Krylov bases
// Every op keeps its last solve's basis mapped (hg_op_basis); a solve whose
// worst-case basis does not fit the free device memory first releases the
// idle bases of the other ops of this process, then splits its batch.
static std::mutex g_ops_mu;
static std::set<HgOp*> g_ops;

static size_t op_ws_bytes(const HgOp* op) {
  size_t b = op->dws.Q.mapped + op->dwsb.Q.mapped + op->bws.V.mapped + op->bws.WV.mapped;
  if (op->ws.V) b += sizeof(double) * (size_t)op->ws.n * op->ws.cap * (op->ws.weighted ? 2 : 1);
  return b;
}

static void op_release_ws(HgOp* op) {
  op->ws.~Workspace();
  new (&op->ws) Workspace();
  op->bws.clear();
  op->dws.clear();
  op->dwsb.clear();
  op->basis = nullptr;
  op->basis_cols = op->basis_nv = 0;
}

// release the idle workspaces of every other op; returns the bytes freed
static size_t release_idle_ops(const HgOp* self) {
  std::lock_guard<std::mutex> lk(g_ops_mu);
  size_t freed = 0;
  for (HgOp* o : g_ops) {
    if (o == self || o->busy.load()) continue;
    const size_t b = op_ws_bytes(o);
    if (b == 0) continue;
    op_release_ws(o);
    freed += b;
  }
  return freed;
}

struct BusyScope {
  HgOp* op;
  explicit BusyScope(HgOp* o) : op(o) { if (op) op->busy.fetch_add(1); }
  ~BusyScope() { if (op) op->busy.fetch_sub(1); }
};

// Orthogonalisation scheme of hg_gmres / hg_gmres_batch (hg_set_orthogonalization).
static thread_local int g_orth = HG_ORTH_DCGS2;  // per host thread (set around one call by the bindings)

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

// ---- phase timing (hg_stats_*): event pairs per phase, summed at solve end
namespace {
struct PhaseStats {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<int, size_t>> open;  // (phase, index of the start event)
  double ms[HG_NPHASES] = {0};
  long long count[HG_NPHASES] = {0};
};
PhaseStats g_stats;

cudaEvent_t stats_event() {
  if (g_stats.used == g_stats.pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_stats.pool.push_back(e);
  }
  return g_stats.pool[g_stats.used++];
}

// phase bracket: start on construction, stop on destruction (same stream)
struct Phase {
  cudaStream_t st;
  int ph;
  size_t i0 = 0;
  bool on;
  Phase(cudaStream_t s, int p) : st(s), ph(p), on(g_stats.on) {
    if (on) {
      i0 = g_stats.used;
      cudaEventRecord(stats_event(), st);
    }
  }
  ~Phase() {
    if (on) {
      cudaEventRecord(stats_event(), st);
      g_stats.open.emplace_back(ph, i0);
    }
  }
};

// called after the solve's final synchronisation
void stats_collect() {
  if (!g_stats.on) return;
  for (auto& pr : g_stats.open) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, g_stats.pool[pr.second], g_stats.pool[pr.second + 1]) == cudaSuccess) {
      g_stats.ms[pr.first] += t;
      g_stats.count[pr.first] += 1;
    }
  }
  g_stats.open.clear();
  g_stats.used = 0;
}
}  // namespace

// Under stream capture the graph would run the pre-launched coarse solve and
// Z^T r as independent nodes: capture the serial order instead.
static bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

static bool serial_order(cudaStream_t st) { return serial_kernels() || capturing(st); }

// ---- handle faults: a timed-out device wait (fault word 1) or a failed launch
// in the middle of an apply (2) poisons the handle
static int precond_fault(const HgPrecond* P) {
  if (!P || !P->h_fault) return HG_OK;
  const int f = *reinterpret_cast<volatile const int*>(P->h_fault);
  if (f == 0) return HG_OK;
  set_error(f == 1 ? "a device-side wait of the coarse solve timed out (its Z^T r never arrived: failed or starved "
                     "launch); the preconditioner handle is poisoned, destroy and recreate it"
                   : "an earlier apply failed part-way through its launches; the preconditioner handle is "
                     "poisoned, destroy and recreate it");
  return HG_ERR_CUDA;
}

static int poison(HgPrecond* P, int status) {
  if (status == HG_ERR_CUDA && P && P->h_fault && *reinterpret_cast<volatile int*>(P->h_fault) == 0)
    *reinterpret_cast<volatile int*>(P->h_fault) = 2;
  return status;
}

static int op_fault(const HgOp* op) { return op && op->kind == 1 ? precond_fault(op->P) : HG_OK; }

// stream synchronisation of a solve loop + the handle's fault word
static int sync_check(cudaStream_t st, const HgOp* op, const HgOp* weight) {
  HG_CUDA_TRY(cudaStreamSynchronize(st));
  HG_TRY(op_fault(op));
  return op_fault(weight);
}

static int precond_apply_core_impl(HgPrecond* P, const double* r, double* out, const double* W, long long ldw,
                                   int nv, double* partials, int* nb, cudaStream_t st);

static int precond_apply_core(HgPrecond* P, const double* r, double* out, const double* W, long long ldw,
                              int nv, double* partials, int* nb, cudaStream_t st) {
  HG_TRY(precond_fault(P));
  return poison(P, precond_apply_core_impl(P, r, out, W, ldw, nv, partials, nb, st));
}

static int precond_apply_core_impl(HgPrecond* P, const double* r, double* out, const double* W, long long ldw,
                                   int nv, double* partials, int* nb, cudaStream_t st) {
  if (P->m > 0 && P->d_b0_inv && P->b0_inv_single) {
    // dense coarse mode: Z^T r, then (side stream) c -> B0^{-1} c -> Z y beside the local solves
    HG_TRY(launch_zt(P, r, st));
    HG_CUDA_TRY(cudaEventRecord(P->ev_fork, st));
    HG_CUDA_TRY(cudaStreamWaitEvent(P->aux, P->ev_fork, 0));
    HG_TRY(launch_b0_dense(P, P->aux));
    HG_TRY(launch_zy(P, P->aux));
    HG_CUDA_TRY(cudaEventRecord(P->ev_join, P->aux));
  } else if (P->m > 0) {
    HG_CUDA_TRY(cudaEventRecord(P->ev_fork, st));
    HG_CUDA_TRY(cudaStreamWaitEvent(P->aux, P->ev_fork, 0));
    const bool ser = serial_order(st);
    bool zt_launched = false;
    if (ser) {
      // tools that serialise kernels (profilers, sanitizers, blocking launches)
      // and graph capture: no kernel may wait on a later one
      HG_TRY(launch_zt(P, r, P->aux));
      HG_TRY(launch_coarse_solve(P, P->aux));
    } else if (P->b0_split_on && P->b0_mode == 1) {
      // bisected coarse solve: the two half chains first (they hold their SMs and wait, bounded,
      // for their rows' Z^T r chunks); the separator stage reads c_S, i.e. needs ALL of Z^T r
      HG_TRY(launch_coarse_chains_split(P, P->aux));
      HG_TRY(launch_zt(P, r, st));
      HG_CUDA_TRY(cudaEventRecord(P->ev_zt, st));
      HG_CUDA_TRY(cudaStreamWaitEvent(P->aux, P->ev_zt, 0));
      HG_TRY(launch_coarse_sep_split(P, P->aux));
      zt_launched = true;
    } else {
      // The latency-bound coarse solve is launched FIRST (side stream) so that
      // it holds its SMs before the local solves fill the GPU; it starts its
      // work when the Z^T r launch it pairs with (device ticket) has counted
      // its chunks — a bounded device-side wait (hg_common.cuh SpinGuard).
      HG_TRY(launch_coarse_solve(P, P->aux));
    }
    HG_TRY(launch_zy(P, P->aux));
    HG_CUDA_TRY(cudaEventRecord(P->ev_join, P->aux));
    if (!ser && !zt_launched) HG_TRY(launch_zt(P, r, st));
  }
  HG_TRY(launch_local_solve(P, r, st));
  if (P->m > 0) HG_CUDA_TRY(cudaStreamWaitEvent(st, P->ev_join, 0));
  return launch_assemble(P, true, true, out, W, ldw, nv, partials, nb, st);
}

// coarse solve of the current Z^T r partials on one stream (apply_coarse, profiling)
static int coarse_solve_serial(HgPrecond* P, cudaStream_t st) {
  if (P->d_b0_inv && P->b0_inv_single) return launch_b0_dense(P, st);
  return launch_coarse_solve(P, st);
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

static int precond_apply_multi_core_impl(HgPrecond* P, const double* R, long long ldr, double* OUT, long long ldo,
                                         int nrhs, cudaStream_t st);

static int precond_apply_multi_core(HgPrecond* P, const double* R, long long ldr, double* OUT, long long ldo,
                                    int nrhs, cudaStream_t st) {
  HG_TRY(precond_fault(P));
  return poison(P, precond_apply_multi_core_impl(P, R, ldr, OUT, ldo, nrhs, st));
}

static int precond_apply_multi_core_impl(HgPrecond* P, const double* R, long long ldr, double* OUT, long long ldo,
                                         int nrhs, cudaStream_t st) {
  if (nrhs < 1 || nrhs > HG_MAX_RHS) {
    set_error("batched apply: nrhs must be in [1, HG_MAX_RHS]");
    return HG_ERR_ARG;
  }
  HG_TRY(multi_prepare(P));
  if (P->m > 0 && P->d_b0_inv) {
    // dense coarse: no kernel waits on another, so the long local solve is
    // issued FIRST and takes its SMs; Z^T R -> B0^{-1} -> Z Y fill the rest
    HG_CUDA_TRY(cudaEventRecord(P->ev_fork, st));
    HG_CUDA_TRY(cudaStreamWaitEvent(P->aux, P->ev_fork, 0));
    HG_TRY(launch_local_batch(P, R, ldr, nrhs, st));
    HG_TRY(launch_zt_multi(P, R, ldr, nrhs, P->aux));
    HG_TRY(launch_b0_dense_multi(P, nrhs, P->aux));
    HG_TRY(launch_zy_multi(P, nrhs, P->aux));
    HG_CUDA_TRY(cudaEventRecord(P->ev_join, P->aux));
    HG_CUDA_TRY(cudaStreamWaitEvent(st, P->ev_join, 0));
    return launch_assemble_multi(P, true, true, OUT, ldo, nrhs, st);
  } else if (P->m > 0) {
    HG_CUDA_TRY(cudaEventRecord(P->ev_fork, st));
    HG_CUDA_TRY(cudaStreamWaitEvent(P->aux, P->ev_fork, 0));
    const bool ser = serial_order(st);
    if (ser) {
      HG_TRY(launch_zt_multi(P, R, ldr, nrhs, P->aux));
      HG_TRY(launch_b0_multi(P, nrhs, P->aux));
    } else {
      // as the single-RHS apply: the persistent coarse solve first (holds its
      // SMs), released by the chunk counters of the Z^T R launch it pairs with
      HG_TRY(launch_b0_multi(P, nrhs, P->aux));
    }
    HG_TRY(launch_zy_multi(P, nrhs, P->aux));
    HG_CUDA_TRY(cudaEventRecord(P->ev_join, P->aux));
    if (!ser) HG_TRY(launch_zt_multi(P, R, ldr, nrhs, st));
  }
  HG_TRY(launch_local_batch(P, R, ldr, nrhs, st));
  if (P->m > 0) HG_CUDA_TRY(cudaStreamWaitEvent(st, P->ev_join, 0));
  return launch_assemble_multi(P, true, true, OUT, ldo, nrhs, st);
}

// Y[:, c] = op(X[:, c])
static int op_apply_multi(HgOp* op, const double* X, long long ldx, double* Y, long long ldy, int nrhs,
                          cudaStream_t st) {
  if (op->kind == 0) return launch_spmm(op->csr, op->csr.data, X, ldx, Y, ldy, nrhs, st);
  HgPrecond* P = op->P;
  switch (op->mode) {
    case 0:
      return precond_apply_multi_core(P, X, ldx, Y, ldy, nrhs, st);
    case 1:
      HG_TRY(multi_prepare(P));
      HG_TRY(launch_spmm(P->A, P->A.data, X, ldx, P->d_tmpm, P->n, nrhs, st));
      return precond_apply_multi_core(P, P->d_tmpm, P->n, Y, ldy, nrhs, st);
    case 2:
    case 3: {
      const double* vals = op->mode == 2 ? P->A.data : P->A.data2;
      if (!vals) {
        set_error("operator needs D_k but the handle was created without it");
        return HG_ERR_ARG;
      }
      return launch_spmm(P->A, vals, X, ldx, Y, ldy, nrhs, st);
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

int hg_stats_enable(int on) {
  g_stats.on = on != 0;
  g_stats.open.clear();
  g_stats.used = 0;
  return HG_OK;
}

int hg_stats_read(double* ms, int64_t* count, int reset) {
  for (int p = 0; p < HG_NPHASES; ++p) {
    if (ms) ms[p] = g_stats.ms[p];
    if (count) count[p] = g_stats.count[p];
    if (reset) {
      g_stats.ms[p] = 0.0;
      g_stats.count[p] = 0;
    }
  }
  return HG_OK;
}
const char* hg_last_error(void) { return g_err.c_str(); }
int64_t hg_kernel_launches(void) { return g_launches.load(); }
int hg_device_sync(void) {
  HG_CUDA_TRY(cudaDeviceSynchronize());
  return HG_OK;
}

int hg_shutdown(void) {
  g_shutdown = true;
  return HG_OK;
}

int hg_precond_destroy(HgPrecond* P) {
  if (!P || g_shutdown) return HG_OK;
  release(P->A.indptr);
  release(P->A.indices);
  release(P->A.data);
  release(P->A.data2);
  release(P->d_local);
  release(P->d_local_idx);
  release(P->d_fwd);
  release(P->d_bwd);
  release(P->d_poff);
  release(P->d_pfwd);
  release(P->d_pbwd);
  release(P->d_pmt);
  release(P->d_mtoff);
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
  release(P->d_blk_done);
  release(P->d_y);
  release(P->d_b0_inv);
  split_release(P);
  release(P->d_c);
  release(P->d_cm);
  release(P->d_ypart);
  release(P->d_zs);
  release(P->d_cptr);
  release(P->d_cent);
  release(P->d_tmp);
  release(P->d_xsm);
  release(P->d_zsm);
  release(P->d_zypk);
  release(P->d_ztpk);
  release(P->d_zypk_off);
  release(P->d_ztpk_off);
  release(P->d_zy_items);
  release(P->d_cpartm);
  release(P->d_ym);
  release(P->d_b0m_x);
  release(P->d_blkm_done);
  release(P->d_ticket);
  if (P->h_fault) cudaFreeHost(P->h_fault);
  P->h_fault = nullptr;
  P->d_fault = nullptr;
  release(P->d_tmpm);
  if (P->aux) cudaStreamDestroy(P->aux);
  if (P->aux2) cudaStreamDestroy(P->aux2);
  for (cudaEvent_t e : {P->ev_c0, P->ev_c1, P->ev_zt})
    if (e) cudaEventDestroy(e);
  for (auto& c : P->b0h) {
    release(c.perm);
    release(c.dinv);
    release(c.tile_ptr);
    release(c.tile_col);
    release(c.tiles);
    release(c.xbuf);
  }
  release(P->d_b0s_f);
  release(P->d_b0s_sinv);
  release(P->d_b0s_w);
  release(P->d_b0s_t);
  if (P->ev_fork) cudaEventDestroy(P->ev_fork);
  if (P->ev_join) cudaEventDestroy(P->ev_join);
  hg_op_destroy(P->op_T);
  hg_op_destroy(P->op_W);
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

// Device factorisation of the local blocks (desc without records): band LU
// straight into the zeroed record arrays (hg_factor.cu), INFO and the
// smallest pivot per block back to the caller.
static int device_factor_local(HgPrecond* P, const HgPrecondDesc* D) {
  if (!D->local_bw || !D->lcsr_indptr || !D->lcsr_cols || !D->lcsr_vals || !D->factor_info ||
      !D->factor_min_pivot) {
    set_error("hg_precond_create: no local records and no block CSR to factor");
    return HG_ERR_ARG;
  }
  const int nl = D->n_local;
  int kl_max = 0;
  for (int s = 0; s < nl; ++s) kl_max = std::max(kl_max, (int)D->local_bw[s]);
  for (int s = 0; s < nl; ++s) {
    const LocalDesc& d = P->h_local[s];
    if (d.kl < D->local_bw[s] || d.kv < 2 * D->local_bw[s]) {
      set_error("hg_precond_create: record widths narrower than the band of block " + std::to_string(s));
      return HG_ERR_ARG;
    }
  }
  if (!band_lu_supported(kl_max, kl_max)) {
    set_error("hg_precond_create: device band LU supports half-widths <= 79 (got " + std::to_string(kl_max) +
              "); pass host records");
    return HG_ERR_UNSUPPORTED;
  }
  HG_CUDA_TRY(cudaMemset(P->d_fwd, 0, sizeof(double) * (size_t)D->local_fwd_len));
  HG_CUDA_TRY(cudaMemset(P->d_bwd, 0, sizeof(double) * (size_t)D->local_bwd_len));
  std::vector<long long> base(nl);
  for (int s = 0; s < nl; ++s) base[s] = (long long)D->local_idx_off[s] + s;
  const long long nptr = (long long)D->local_idx_off[nl] + nl;
  int *d_bw = nullptr, *d_cols = nullptr, *d_info = nullptr;
  long long *d_base = nullptr, *d_ip = nullptr;
  double *d_vals = nullptr, *d_minp = nullptr;
  int s = HG_OK;
  if ((s = upload(&d_bw, D->local_bw, (size_t)nl, nullptr)) == HG_OK &&
      (s = upload(&d_base, base.data(), (size_t)nl, nullptr)) == HG_OK &&
      (s = upload(&d_ip, reinterpret_cast<const long long*>(D->lcsr_indptr), (size_t)nptr, nullptr)) == HG_OK &&
      (s = upload(&d_cols, D->lcsr_cols, (size_t)D->lcsr_nnz, nullptr)) == HG_OK &&
      (s = upload(&d_vals, D->lcsr_vals, (size_t)D->lcsr_nnz, nullptr)) == HG_OK &&
      (s = upload<int>(&d_info, nullptr, (size_t)nl, nullptr)) == HG_OK &&
      (s = upload<double>(&d_minp, nullptr, (size_t)nl, nullptr)) == HG_OK) {
    s = launch_band_lu(P, d_bw, kl_max, kl_max, d_base, d_ip, d_cols, d_vals, d_info, d_minp, 0);
    if (s == HG_OK && cudaDeviceSynchronize() != cudaSuccess) {
      set_error(std::string("device band LU: ") + cudaGetErrorString(cudaGetLastError()));
      s = HG_ERR_CUDA;
    }
    if (s == HG_OK && (cudaMemcpy(D->factor_info, d_info, sizeof(int) * nl, cudaMemcpyDeviceToHost) != cudaSuccess ||
                       cudaMemcpy(D->factor_min_pivot, d_minp, sizeof(double) * nl, cudaMemcpyDeviceToHost) !=
                           cudaSuccess)) {
      set_error("device band LU: reading INFO back failed");
      s = HG_ERR_CUDA;
    }
  }
  release(d_bw);
  release(d_base);
  release(d_ip);
  release(d_cols);
  release(d_vals);
  release(d_info);
  release(d_minp);
  return s;
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
  HG_TRY(upload<unsigned long long>(&P->d_ticket, nullptr, 4, bytes));
  HG_CUDA_TRY(cudaMemset(P->d_ticket, 0, 4 * sizeof(unsigned long long)));
  HG_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&P->h_fault), sizeof(int), cudaHostAllocMapped));
  *P->h_fault = 0;
  HG_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&P->d_fault), P->h_fault, 0));

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
    // d.n = 0 with a non-empty index range: the separator pseudo block of a split subdomain
    if ((d.n != D->local_idx_off[s + 1] - D->local_idx_off[s] && !(d.n == 0 && D->n_split > 0)) ||
        d.fstride < d.kl + 1 ||
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
  // registers 1..R-3 of the sweep window are applied without a band test:
  // every block's records must cover them (factor.record_floor pads)
  for (int s = 0; s < D->n_local; ++s) {
    const LocalDesc& d = P->h_local[s];
    if (d.n > 0 && (d.kl < 32 * P->rf - 65 || d.kv < 32 * P->rb - 65)) {
      set_error("hg_precond_create: block " + std::to_string(s) + " records narrower than the launch's floor (kl " +
                std::to_string(d.kl) + " < " + std::to_string(32 * P->rf - 65) + " or kv " + std::to_string(d.kv) +
                " < " + std::to_string(32 * P->rb - 65) + "); zero pad them (factor.record_floor)");
      return HG_ERR_ARG;
    }
  }
  if (D->n_local > 0 && (P->rf > 6 || P->rb > 10)) {
    set_error("hg_precond_create: local bandwidth kl=" + std::to_string(max_kl) + ", kv=" +
              std::to_string(max_kv) + " beyond compiled tiles (kl <= 160, kv <= 288)");
    return HG_ERR_UNSUPPORTED;
  }
  if (D->n_local > 0) {
    const long long nidx = D->local_idx_off[D->n_local];
    P->xs_len = nidx;
    P->fwd_len = D->local_fwd_len;
    P->bwd_len = D->local_bwd_len;
    HG_TRY(upload(&P->d_local, P->h_local.data(), P->h_local.size(), bytes));
    HG_TRY(upload(&P->d_local_idx, D->local_idx, (size_t)nidx, bytes));
    HG_TRY(upload(&P->d_fwd, D->local_fwd, (size_t)D->local_fwd_len, bytes));
    HG_TRY(upload(&P->d_bwd, D->local_bwd, (size_t)D->local_bwd_len, bytes));
    if (!D->local_fwd || !D->local_bwd) HG_TRY(device_factor_local(P, D));
    HG_TRY(upload<double>(&P->d_xs, nullptr, (size_t)nidx, bytes));
    HG_CUDA_TRY(cudaMemset(P->d_xs, 0, sizeof(double) * (size_t)nidx));
    HG_TRY(split_upload(P, D));
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
    HG_TRY(upload<unsigned long long>(&P->d_blk_done, nullptr, (size_t)D->n_cblk, bytes));
    HG_CUDA_TRY(cudaMemset(P->d_blk_done, 0, sizeof(unsigned long long) * D->n_cblk));
    HG_TRY(upload<double>(&P->d_y, nullptr, (size_t)P->m, bytes));
    if (D->b0_split) {  // bisected single-RHS coarse solve
      const int a = D->b0s_a, ns = D->b0s_ns;
      if (P->b0_mode != 1 || a <= 0 || ns <= 0 || a + ns >= P->m || D->b0s_wl < 0 || D->b0s_wl > a ||
          D->b0s_wr < 0 || a + ns + D->b0s_wr > P->m || !D->b0s_f || !D->b0s_sinv || !D->b0s_w || !D->b0h0_perm ||
          !D->b0h1_perm || !D->b0h0_dinv || !D->b0h1_dinv || !D->b0h0_tile_ptr || !D->b0h1_tile_ptr) {
        set_error("hg_precond_create: inconsistent bisected coarse solve (needs the cluster mode)");
        return HG_ERR_ARG;
      }
      const int hm[2] = {a, P->m - a - ns}, hoff[2] = {0, a + ns};
      const int hk[2] = {D->b0h0_npanel, D->b0h1_npanel}, hr[2] = {D->b0h0_ring, D->b0h1_ring};
      const int hc[2] = {D->b0h0_cluster, D->b0h1_cluster};
      const long long hnt[2] = {D->b0h0_ntile, D->b0h1_ntile};
      const int32_t* hperm[2] = {D->b0h0_perm, D->b0h1_perm};
      const double* hdinv[2] = {D->b0h0_dinv, D->b0h1_dinv};
      const int64_t* hptr[2] = {D->b0h0_tile_ptr, D->b0h1_tile_ptr};
      const int32_t* hcol[2] = {D->b0h0_tile_col, D->b0h1_tile_col};
      const double* htiles[2] = {D->b0h0_tiles, D->b0h1_tiles};
      for (int h = 0; h < 2; ++h) {
        HgPrecond::B0Half& c = P->b0h[h];
        c.m = hm[h];
        c.off = hoff[h];
        c.K = hk[h];
        c.nr = hr[h];
        c.cs = hc[h];
        if (c.K != (c.m + 63) / 64 || c.cs < 1 || c.cs > 16 || c.nr < c.cs + 1 ||
            b0_cluster_smem(c.nr) > 227 * 1024 || (hnt[h] > 0 && (!hcol[h] || !htiles[h]))) {
          set_error("hg_precond_create: invalid half-chain parameters of the bisected coarse solve");
          return HG_ERR_ARG;
        }
        std::vector<int> gperm(c.m);  // chain row -> global coarse column
        for (int i = 0; i < c.m; ++i) {
          if (hperm[h][i] < 0 || hperm[h][i] >= c.m) {
            set_error("hg_precond_create: half-chain permutation out of range");
            return HG_ERR_ARG;
          }
          gperm[i] = c.off + hperm[h][i];
        }
        HG_TRY(upload(&c.perm, gperm.data(), gperm.size(), bytes));
        HG_TRY(upload(&c.dinv, hdinv[h], (size_t)2 * c.K * 64 * 64, bytes));
        HG_TRY(upload(&c.tile_ptr, reinterpret_cast<const long long*>(hptr[h]), (size_t)2 * c.K + 1, bytes));
        if (hnt[h] > 0) {
          HG_TRY(upload(&c.tile_col, hcol[h], (size_t)hnt[h], bytes));
          HG_TRY(upload(&c.tiles, htiles[h], (size_t)hnt[h] * 64 * 64, bytes));
        }
        HG_TRY(upload<double>(&c.xbuf, nullptr, (size_t)2 * c.K * 64, bytes));
      }
      P->b0s_a = a;
      P->b0s_ns = ns;
      P->b0s_wl = D->b0s_wl;
      P->b0s_wr = D->b0s_wr;
      HG_TRY(upload(&P->d_b0s_f, D->b0s_f, (size_t)ns * (D->b0s_wl + D->b0s_wr), bytes));
      HG_TRY(upload(&P->d_b0s_sinv, D->b0s_sinv, (size_t)ns * ns, bytes));
      HG_TRY(upload(&P->d_b0s_w, D->b0s_w, (size_t)(P->m - ns) * ns, bytes));
      HG_TRY(upload<double>(&P->d_b0s_t, nullptr, (size_t)ns, bytes));
      HG_CUDA_TRY(cudaStreamCreateWithFlags(&P->aux2, cudaStreamNonBlocking));
      HG_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_c0, cudaEventDisableTiming));
      HG_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_c1, cudaEventDisableTiming));
      HG_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_zt, cudaEventDisableTiming));
      P->b0_split = P->b0_split_on = true;
    }
    if (D->b0_inv) {
      // row-major in (host or device memory), kept packed in DMMA-fragment order
      double* rowmajor = nullptr;
      cudaPointerAttributes pa{};
      const bool on_dev = cudaPointerGetAttributes(&pa, D->b0_inv) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
      cudaGetLastError();
      if (!on_dev) HG_TRY(upload(&rowmajor, D->b0_inv, (size_t)P->m * P->m, nullptr));
      const int ps = pack_b0_inverse(P->m, on_dev ? D->b0_inv : rowmajor, &P->d_b0_inv, &P->b0_mp);
      release(rowmajor);
      HG_TRY(ps);
      if (bytes) *bytes += (long long)sizeof(double) * P->b0_mp * P->b0_mp;
      P->b0_inv_single = D->b0_inv_batched_only == 0;
      HG_TRY(upload<double>(&P->d_c, nullptr, (size_t)P->b0_mp, bytes));
      HG_CUDA_TRY(cudaMemset(P->d_c, 0, sizeof(double) * P->b0_mp));
    }
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
  HG_TRY(preload_multi());
  HG_TRY(preload_dcgs2());
  HG_TRY(preload_add());
  HG_TRY(preload_b0_dense());
  HG_TRY(preload_split());
  HG_CUDA_TRY(cudaStreamCreateWithFlags(&P->aux, cudaStreamNonBlocking));
  HG_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
  HG_CUDA_TRY(cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming));
  HG_CUDA_TRY(cudaDeviceSynchronize());
  if (P->n_local > 0) {  // batched solves on 16-row panels (checked against the row solve)
    HG_TRY(multi_prepare(P));
    HG_TRY(prepare_local_panel(P));
  }
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

int hg_precond_read(HgPrecond* P, int32_t field, double* host, int64_t count) {
  if (!P || !host || count < 0) {
    set_error("hg_precond_read: bad argument");
    return HG_ERR_ARG;
  }
  const double* src = nullptr;
  long long len = 0;
  if (field == HG_FIELD_LOCAL_FWD) {
    src = P->d_fwd;
    len = P->fwd_len;
  } else if (field == HG_FIELD_LOCAL_BWD) {
    src = P->d_bwd;
    len = P->bwd_len;
  } else {
    set_error("hg_precond_read: unknown field");
    return HG_ERR_ARG;
  }
  if (count != len) {
    set_error("hg_precond_read: count " + std::to_string(count) + " != field length " + std::to_string(len));
    return HG_ERR_ARG;
  }
  if (len) HG_CUDA_TRY(cudaMemcpy(host, src, sizeof(double) * (size_t)len, cudaMemcpyDeviceToHost));
  return HG_OK;
}

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
  HG_TRY(precond_fault(P));
  HG_TRY(launch_spmv(P->A, P->A.data, u, P->d_tmp, st));
  return precond_apply_core(P, P->d_tmp, out, nullptr, 0, 0, nullptr, nullptr, st);
}

int hg_precond_apply_coarse(HgPrecond* P, const double* r, double* out, void* stream) {
  if (!P || !r || !out) {
    set_error("hg_precond_apply_coarse: null argument");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  HG_TRY(precond_fault(P));
  if (P->m == 0) return launch_fill(P->n, out, 0.0, st);
  int s = launch_zt(P, r, st);
  if (s == HG_OK) s = coarse_solve_serial(P, st);
  if (s == HG_OK) s = launch_zy(P, st);
  if (s == HG_OK) s = launch_assemble(P, true, false, out, nullptr, 0, 0, nullptr, nullptr, st);
  return poison(P, s);
}

int hg_precond_profile(HgPrecond* P, const double* r, double* out, int32_t iters, double* stage_ms,
                       void* stream) {
  if (!P || !r || !out || !stage_ms || iters <= 0) {
    set_error("hg_precond_profile: bad argument");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  HG_TRY(precond_fault(P));
  cudaEvent_t ev[HG_NSTAGES + 1];
  for (auto& e : ev) HG_CUDA_TRY(cudaEventCreate(&e));
  double acc[HG_NSTAGES] = {0, 0, 0, 0, 0};
  int status = HG_OK;
  for (int it = 0; it < iters && status == HG_OK; ++it) {
    cudaEventRecord(ev[0], st);
    if ((status = launch_zt(P, r, st)) != HG_OK) break;
    cudaEventRecord(ev[1], st);
    if ((status = coarse_solve_serial(P, st)) != HG_OK) break;
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
  if (status == HG_OK) status = precond_fault(P);
  return poison(P, status);
}

int hg_precond_apply_multi(HgPrecond* P, const double* R, int64_t ldr, double* OUT, int64_t ldo, int32_t nrhs,
                           void* stream) {
  if (!P || !R || !OUT || ldr < P->n || ldo < P->n) {
    set_error("hg_precond_apply_multi: bad argument");
    return HG_ERR_ARG;
  }
  return precond_apply_multi_core(P, R, ldr, OUT, ldo, nrhs, (cudaStream_t)stream);
}

int hg_precond_profile_multi(HgPrecond* P, const double* R, int64_t ldr, double* OUT, int64_t ldo, int32_t nrhs,
                             int32_t iters, double* stage_ms, void* stream) {
  if (!P || !R || !OUT || !stage_ms || iters <= 0 || nrhs < 1 || nrhs > HG_MAX_RHS || ldr < P->n || ldo < P->n) {
    set_error("hg_precond_profile_multi: bad argument");
    return HG_ERR_ARG;
  }
  HG_TRY(precond_fault(P));
  HG_TRY(multi_prepare(P));
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t ev[HG_NSTAGES + 1];
  for (auto& e : ev) HG_CUDA_TRY(cudaEventCreate(&e));
  double acc[HG_NSTAGES] = {0, 0, 0, 0, 0};
  int status = HG_OK;
  for (int it = 0; it < iters && status == HG_OK; ++it) {
    cudaEventRecord(ev[0], st);
    if ((status = launch_zt_multi(P, R, ldr, nrhs, st)) != HG_OK) break;
    cudaEventRecord(ev[1], st);
    if ((status = (P->d_b0_inv ? launch_b0_dense_multi(P, nrhs, st) : launch_b0_multi(P, nrhs, st))) != HG_OK)
      break;
    cudaEventRecord(ev[2], st);
    if ((status = launch_zy_multi(P, nrhs, st)) != HG_OK) break;
    cudaEventRecord(ev[3], st);
    if ((status = launch_local_batch(P, R, ldr, nrhs, st)) != HG_OK) break;
    cudaEventRecord(ev[4], st);
    if ((status = launch_assemble_multi(P, true, true, OUT, ldo, nrhs, st)) != HG_OK) break;
    cudaEventRecord(ev[5], st);
    if (cudaEventSynchronize(ev[5]) != cudaSuccess) {
      set_error("hg_precond_profile_multi: event sync failed");
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
  if (status == HG_OK) status = precond_fault(P);
  return poison(P, status);
}

int hg_precond_status(HgPrecond* P) {
  if (!P) {
    set_error("hg_precond_status: null handle");
    return HG_ERR_ARG;
  }
  return precond_fault(P);
}

int hg_debug_set(HgPrecond* P, int32_t key, int64_t value) {
  switch (key) {
    case HG_DEBUG_SPIN_LIMIT_MS:
      g_spin_limit_ms = value;
      return HG_OK;
    case HG_DEBUG_SKIP_ZT:
      if (!P) break;
      P->skip_zt = (int)value;
      return HG_OK;
    case HG_DEBUG_FORCE_EXPLICIT_RHO:
      g_force_explicit_rho = value != 0;
      return HG_OK;
    case HG_DEBUG_LOCAL_STAGES:
      if (!P) break;
      if (value != 0 && (value < 2 || value > 6)) {
        set_error("hg_debug_set: local stages must be 0 (default) or 2..6");
        return HG_ERR_ARG;
      }
      P->ls_ns = (int)value;
      return HG_OK;
    case HG_DEBUG_B0_TILE_STAGES:
      if (!P) break;
      if (value != 0 && (value < 2 || value > 4)) {
        set_error("hg_debug_set: tile stages must be 0 (default) or 2..4");
        return HG_ERR_ARG;
      }
      P->b0_tns = (int)value;
      return HG_OK;
    case HG_DEBUG_B0_SPLIT: {
      if (!P) break;
      if (!P->b0_split) return HG_OK;  // nothing to switch
      // the chains pair with Z^T r launches through device tickets: bring the tickets of the
      // chains that sat out up to the number of Z^T r launches so far
      HG_CUDA_TRY(cudaDeviceSynchronize());
      unsigned long long done = 0;
      int b0 = -1;
      for (int b = 0; b < P->n_cblk && b0 < 0; ++b)
        if (P->h_cblk[b].nchunk > 0) b0 = b;
      if (b0 >= 0) {
        HG_CUDA_TRY(cudaMemcpy(&done, P->d_blk_done + b0, sizeof(done), cudaMemcpyDeviceToHost));
        const unsigned long long launches = done / (unsigned long long)P->h_cblk[b0].nchunk;
        const unsigned long long t[3] = {launches * (unsigned long long)P->b0_cs,
                                         launches * (unsigned long long)P->b0h[0].cs,
                                         launches * (unsigned long long)P->b0h[1].cs};
        HG_CUDA_TRY(cudaMemcpy(P->d_ticket, &t[0], sizeof(unsigned long long), cudaMemcpyHostToDevice));
        HG_CUDA_TRY(cudaMemcpy(P->d_ticket + 2, &t[1], 2 * sizeof(unsigned long long), cudaMemcpyHostToDevice));
      }
      P->b0_split_on = value != 0;
      return HG_OK;
    }
    default:
      break;
  }
  set_error("hg_debug_set: unknown key or missing handle");
  return HG_ERR_ARG;
}

int64_t hg_dcgs2_explicit_passes(void) { return g_explicit_rho_passes.load(); }

double hg_precond_stat(HgPrecond* P, int32_t key) {
  if (!P) return NAN;
  switch (key) {
    case HG_STAT_PANEL_ACTIVE:
      return P->panel_ok ? 1.0 : 0.0;
    case HG_STAT_PANEL_DEVIATION:
      return P->panel_dev;
    case HG_STAT_PANEL_BYTES:
      return (double)P->panel_stream_bytes;
    default:
      return NAN;
  }
}

// Z^T r partials that reduce to c (chunk 0 of each block = its part of c)
__global__ void k_set_cpart(int m, const int* __restrict__ col_blk, const CblkDesc* __restrict__ descs,
                            const double* __restrict__ c, double* __restrict__ cpart) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const CblkDesc d = descs[col_blk[i]];
  const int l = i - d.col0;
  for (int ch = 0; ch < d.nchunk; ++ch) cpart[d.part_off + (long long)ch * d.m + l] = ch == 0 ? c[i] : 0.0;
}

// the completion counts one Z^T r launch leaves behind (what the paired coarse solve waits for)
__global__ void k_count_zt(int nblk, const CblkDesc* __restrict__ descs, unsigned long long* blk_done,
                           unsigned long long* zt_done, unsigned long long nitems) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nblk) atomicAdd(blk_done + b, (unsigned long long)descs[b].nchunk);
  if (b == 0) atomicAdd(zt_done, nitems);
}

int hg_precond_coarse_solve(HgPrecond* P, const double* c, double* y, void* stream) {
  if (!P || !c || !y || P->m == 0) {
    set_error("hg_precond_coarse_solve: bad argument (or no coarse space)");
    return HG_ERR_ARG;
  }
  HG_TRY(precond_fault(P));
  cudaStream_t st = (cudaStream_t)stream;
  int s = HG_OK;
  k_set_cpart<<<ceil_div(P->m, 256), 256, 0, st>>>(P->m, P->d_col_blk, P->d_cblk, c, P->d_cpart);
  if (cudaGetLastError() != cudaSuccess) s = HG_ERR_CUDA;
  if (s == HG_OK) {
    k_count_zt<<<ceil_div(P->n_cblk, 256), 256, 0, st>>>(P->n_cblk, P->d_cblk, P->d_blk_done, P->d_zt_done,
                                                         (unsigned long long)P->n_zt_items);
    if (cudaGetLastError() != cudaSuccess) s = HG_ERR_CUDA;
  }
  if (s == HG_OK) s = launch_coarse_solve(P, st);  // the panel chain, whatever the apply mode
  if (s == HG_OK && cudaMemcpyAsync(y, P->d_y, sizeof(double) * P->m, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    s = HG_ERR_CUDA;
  if (s == HG_ERR_CUDA && hg::g_err.empty()) set_error("hg_precond_coarse_solve: launch failed");
  return poison(P, s);
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
  HG_TRY(precond_fault(P));
  return launch_spmv(P->A, vals, x, y, (cudaStream_t)stream);
}

int hg_local_solve(HgPrecond* P, int s, const double* r_local, double* x_local, void* stream) {
  if (!P || s < 0 || s >= P->n_local || !r_local || !x_local) {
    set_error("hg_local_solve: bad argument");
    return HG_ERR_ARG;
  }
  HG_TRY(precond_fault(P));
  return launch_local_solve_single(P, s, r_local, x_local, (cudaStream_t)stream);
}

int hg_precond_local_solutions(HgPrecond* P, const double* r, double* xs, void* stream) {
  if (!P || !r || !xs) {
    set_error("hg_precond_local_solutions: null argument");
    return HG_ERR_ARG;
  }
  HG_TRY(precond_fault(P));
  if (P->n_local == 0 || P->xs_len == 0) return HG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  HG_TRY(launch_local_solve(P, r, st));
  HG_CUDA_TRY(cudaMemcpyAsync(xs, P->d_xs, sizeof(double) * (size_t)P->xs_len, cudaMemcpyDeviceToDevice, st));
  return HG_OK;
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
  {
    std::lock_guard<std::mutex> lk(g_ops_mu);
    g_ops.insert(op);
  }
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
  {
    std::lock_guard<std::mutex> lk(g_ops_mu);
    g_ops.insert(op);
  }
  *out = op;
  return HG_OK;
}

int hg_op_release(HgOp* op) {
  if (!op) {
    set_error("hg_op_release: null operator");
    return HG_ERR_ARG;
  }
  if (g_shutdown) return HG_OK;
  op_release_ws(op);
  return HG_OK;
}

int hg_op_destroy(HgOp* op) {
  if (!op || g_shutdown) return HG_OK;
  {
    std::lock_guard<std::mutex> lk(g_ops_mu);
    g_ops.erase(op);
  }
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
  HG_TRY(op_fault(op));
  return op_apply_dots(op, x, y, nullptr, 0, 0, nullptr, nullptr, (cudaStream_t)stream);
}

int hg_op_apply_multi(HgOp* op, const double* X, int64_t ldx, double* Y, int64_t ldy, int32_t nrhs, void* stream) {
  if (!op || !X || !Y || nrhs < 1 || nrhs > HG_MAX_RHS || ldx < op->n || ldy < op->n) {
    set_error("hg_op_apply_multi: bad argument");
    return HG_ERR_ARG;
  }
  HG_TRY(op_fault(op));
  return op_apply_multi(op, X, ldx, Y, ldy, nrhs, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ GMRES
static int gmres_dcgs2(HgOp* op, HgOp* weight, const double* rhs, long long ldr, double* x, long long ldx, int nrhs,
                       double rtol, int maxit, double* history, int32_t* info, cudaStream_t st);

// The basis kernels (fused dots / updates / x = V y) hold their coefficients
// in shared memory: at most MAX_NV basis vectors.  Refused up front rather
// than after ~MAX_NV device iterations.
static int check_maxit(int maxit) {
  if (maxit > MAX_NV) {
    set_error("weighted GMRES: maxit = " + std::to_string(maxit) + " exceeds the " + std::to_string(MAX_NV) +
              "-vector Krylov basis this library supports (full GMRES keeps every vector)");
    return HG_ERR_UNSUPPORTED;
  }
  return HG_OK;
}

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
  HG_TRY(check_maxit(maxit));
  HG_TRY(op_fault(op));
  HG_TRY(op_fault(weight));
  BusyScope busy(op);
  if (g_orth == HG_ORTH_DCGS2) {
    if (!x0) return gmres_dcgs2(op, weight, rhs, n, x, n, 1, rtol, maxit, history, info, st);
    // r0 = rhs - op(x0); x = x0 + GMRES(r0)
    double* r0 = nullptr;
    HG_CUDA_TRY(cudaMallocAsync(&r0, sizeof(double) * n, st));
    int s = op_apply_dots(op, x0, x, nullptr, 0, 0, nullptr, nullptr, st);
    if (s == HG_OK) s = launch_sub(n, rhs, x, r0, st);
    if (s == HG_OK) s = gmres_dcgs2(op, weight, r0, n, x, n, 1, rtol, maxit, history, info, st);
    if (s == HG_OK) s = launch_add(n, x, x0, x, st);
    cudaFreeAsync(r0, st);
    HG_TRY(sync_check(st, op, weight));
    return s;
  }
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
  HG_TRY(sync_check(st, op, weight));
  const double beta = std::sqrt(hb[0]);
  if (beta == 0.0) {
    if (x0)
      HG_CUDA_TRY(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    else
      HG_TRY(launch_fill(n, x, 0.0, st));
    history[0] = 0.0;
    info[0] = 0;
    info[1] = 1;
    HG_TRY(sync_check(st, op, weight));
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
    {  // w = op(V_j), fused h_i = (W V_i) . w
      Phase ph(st, 0);
      HG_TRY(op_apply_dots(op, V + (long long)j * ld, w, WV, ld, nv, ws.partials, &nb, st));
    }
    {
      Phase ph(st, 1);
      HG_TRY(launch_reduce(ws.partials, nb, nv + 1, ws.dh, st));
    }
    {  // classical GS pass: w -= V h
      Phase ph(st, 2);
      HG_TRY(launch_axpy_multi(n, w, V, ld, nv, ws.dh + 1, 1, st));
    }
    {  // ww = W w with w.ww and the measurement corr_i = (W V_i) . w
      Phase ph(st, 3);
      if (weighted)
        HG_TRY(weight_apply_dots(weight, w, ws.ww, WV, ld, nv, ws.partials, &nb, st));
      else
        HG_TRY(launch_dots(n, w, V, ld, nv, ws.partials, &nb, st));
      HG_TRY(launch_reduce(ws.partials, nb, nv + 1, ws.dc, st));
    }
    HG_CUDA_TRY(cudaMemcpyAsync(hb, ws.dh + 1, sizeof(double) * nv, cudaMemcpyDeviceToHost, st));
    HG_CUDA_TRY(cudaMemcpyAsync(hb + nv, ws.dc, sizeof(double) * (nv + 1), cudaMemcpyDeviceToHost, st));
    HG_TRY(sync_check(st, op, weight));
    for (int i = 0; i < nv; ++i) col[i] = hb[i];
    double hnorm = std::sqrt(std::max(hb[nv], 0.0));
    double cmax = 0.0;
    for (int i = 0; i < nv; ++i) cmax = std::max(cmax, std::fabs(hb[nv + 1 + i]));
    if (cmax > REORTH_TOL * std::max(hnorm, 1e-300)) {
      Phase ph(st, 4);
      for (int i = 0; i < nv; ++i) col[i] += hb[nv + 1 + i];
      HG_TRY(launch_axpy_multi(n, w, V, ld, nv, ws.dc + 1, 1, st));
      if (weighted)
        HG_TRY(weight_apply_dots(weight, w, ws.ww, nullptr, 0, 0, ws.partials, &nb, st));
      else
        HG_TRY(launch_dots(n, w, nullptr, 0, 0, ws.partials, &nb, st));
      HG_TRY(launch_reduce(ws.partials, nb, 1, ws.dc, st));
      HG_CUDA_TRY(cudaMemcpyAsync(hb, ws.dc, sizeof(double), cudaMemcpyDeviceToHost, st));
      HG_TRY(sync_check(st, op, weight));
      hnorm = std::sqrt(std::max(hb[0], 0.0));
      ++reorth;
    }
    col[j + 1] = hnorm;
    double cscale = 0.0;
    for (int i = 0; i <= j + 1; ++i) cscale = std::max(cscale, std::fabs(col[i]));
    if (hnorm <= BREAKDOWN_RTOL * std::max(cscale, 1e-300)) {
      breakdown = true;
    } else {
      Phase ph(st, 5);
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
  HG_TRY(sync_check(st, op, weight));
  stats_collect();
  op->basis = V;
  op->basis_ldv = ld;
  op->basis_ldcol = 0;
  op->basis_cols = 1;
  op->basis_nv = m;
  info[0] = m;
  info[1] = converged ? 1 : 0;
  info[2] = breakdown ? 1 : 0;
  info[3] = reorth;
  return HG_OK;
}

static int ensure_solve_ops(HgPrecond* P) {
  if (!P->op_T) {
    HgOp *t = nullptr, *w = nullptr;
    HG_TRY(hg_op_create_precond(P, 1, &t));
    HG_TRY(hg_op_create_precond(P, 3, &w));
    P->op_T = t;
    P->op_W = w;
  }
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
  HG_TRY(precond_fault(P));
  HG_TRY(ensure_solve_ops(P));
  double *d_f = nullptr, *d_rhs = nullptr, *d_x = nullptr;
  HG_CUDA_TRY(cudaMallocAsync(&d_f, sizeof(double) * n, st));
  HG_CUDA_TRY(cudaMallocAsync(&d_rhs, sizeof(double) * n, st));
  HG_CUDA_TRY(cudaMallocAsync(&d_x, sizeof(double) * n, st));
  HG_CUDA_TRY(cudaMemcpyAsync(d_f, f_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  int s = precond_apply_core(P, d_f, d_rhs, nullptr, 0, 0, nullptr, nullptr, st);
  if (s == HG_OK) s = hg_gmres(P->op_T, P->A.data2 ? P->op_W : nullptr, d_rhs, nullptr, d_x, rtol, maxit, history, info,
                   stream);
  if (s == HG_OK) {
    HG_CUDA_TRY(cudaMemcpyAsync(x_host, d_x, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(d_f, st);
  cudaFreeAsync(d_rhs, st);
  cudaFreeAsync(d_x, st);
  HG_CUDA_TRY(cudaStreamSynchronize(st));
  if (s == HG_OK) s = precond_fault(P);
  return s;
}

}  // extern "C"

// ------------------------------------------------------------------ DCGS2 driver
// Full weighted GMRES (wgmres.py:74-203 semantics: x0 = 0 here, left
// operator given, D_k inner product, stop when |g_{j+1}| <= rtol beta or on
// breakdown, maxit = min(maxit, n)) with delayed classical Gram-Schmidt
// twice (Hernandez/Swirydowicz-Bielich "DCGS2" Arnoldi):
//   iteration j:  w = A q_j                              (q_j projected once)
//                 [s; alpha] = Q_{0:j}^T W q_j, z = Q_{0:j}^T W w   (ONE basis read)
//                 rho = sqrt(alpha - s.s); column j-1 corrected: H[:j, j-1] += beta s,
//                 H[j, j-1] = beta rho  -> Givens, history, stopping test on the host
//                 z'_j = (z_j - s.z)/rho; Hs = H s; h = (z' - Hs)/rho
//                 q_j <- (q_j - Q s)/rho ; w <- w/rho - Q (Hs/rho + h)   (ONE basis read)
//                 beta = ||w||_W (W SpMV), q_{j+1} = w/beta on the device.
// nrhs columns advance in lock step with their own bases and host state;
// nrhs == 1 runs the single-RHS operator kernels.
static int dws_reserve(DcWs& ws, int n, int nrhs, int cap, bool weighted) {
  if (ws.n == n && ws.nrhs == nrhs && ws.cap >= cap && ws.weighted == weighted) return HG_OK;
  ws.clear();
  ws.n = n;
  ws.nrhs = nrhs;
  ws.cap = cap;
  ws.weighted = weighted;
  HG_TRY(ws.Q.reserve(sizeof(double) * (size_t)n * nrhs * cap));
  const size_t nn = (size_t)n * nrhs;
  const size_t W2 = 2 * (size_t)(cap + 2);
  HG_CUDA_TRY(cudaMalloc(&ws.w, sizeof(double) * nn));
  HG_CUDA_TRY(cudaMalloc(&ws.u, sizeof(double) * nn));
  HG_CUDA_TRY(cudaMalloc(&ws.ww, sizeof(double) * nn));
  HG_CUDA_TRY(cudaMalloc(&ws.wq, sizeof(double) * nn));
  HG_CUDA_TRY(cudaMalloc(&ws.partials, sizeof(double) * (size_t)ceil_div(n, VEC_TILE) * W2 * nrhs));
  HG_CUDA_TRY(cudaMalloc(&ws.pself, sizeof(double) * (size_t)ceil_div(n, 256) * nrhs));
  HG_CUDA_TRY(cudaMalloc(&ws.dots, sizeof(double) * W2 * nrhs));
  HG_CUDA_TRY(cudaMalloc(&ws.nrm2, sizeof(double) * nrhs));
  HG_CUDA_TRY(cudaMalloc(&ws.coef, sizeof(double) * W2 * nrhs));
  HG_CUDA_TRY(cudaMalloc(&ws.dy, sizeof(double) * (size_t)(cap + 2) * nrhs));
  HG_CUDA_TRY(cudaMallocHost(&ws.hbuf, sizeof(double) * (2 * W2 * nrhs + nrhs + (size_t)(cap + 2) * nrhs)));
  return HG_OK;
}

static int weight_csr(HgOp* wop, const DevCsr** A, const double** vals) {
  if (wop->kind == 0) {
    *A = &wop->csr;
    *vals = wop->csr.data;
  } else if (wop->mode == 2 || wop->mode == 3) {
    *A = &wop->P->A;
    *vals = wop->mode == 2 ? wop->P->A.data : wop->P->A.data2;
  } else {
    set_error("weight must be a matrix operator (CSR, B or D_k)");
    return HG_ERR_ARG;
  }
  if (!*vals) {
    set_error("weight operator has no values");
    return HG_ERR_ARG;
  }
  return HG_OK;
}

// HG_HOST_TIMING=1: report the host's share of the DCGS2 loop (diagnosis)
static bool host_timing() {
  static const bool on = getenv("HG_HOST_TIMING") && getenv("HG_HOST_TIMING")[0] == '1';
  return on;
}
static double g_host_wait = 0.0, g_host_work = 0.0;

static int gmres_dcgs2_run(HgOp* op, HgOp* weight, const double* rhs, long long ldr, double* x, long long ldx,
                           int nrhs, double rtol, int maxit, double* history, int32_t* info, cudaStream_t st);

// Memory plan: the worst-case basis is nrhs (maxit + 1) n doubles.  If it
// does not fit the free device memory (plus what this op already holds),
// the idle bases of the other ops are released first; if it still does not
// fit, the batch is solved in sub-batches of columns (columns are
// independent, so only the throughput changes).  The basis is mapped on
// demand, so a solve that converges early never touches the worst case.
static int gmres_dcgs2(HgOp* op, HgOp* weight, const double* rhs, long long ldr, double* x, long long ldx, int nrhs,
                       double rtol, int maxit, double* history, int32_t* info, cudaStream_t st) {
  const size_t per_col = sizeof(double) * (size_t)op->n * (size_t)(maxit + 1);
  const size_t margin = (size_t)2 << 30;  // workspaces, the operator's scratch, allocator slack
  auto fits = [&](int cols, size_t& free_b) -> bool {
    size_t total = 0;
    free_b = 0;
    if (cudaMemGetInfo(&free_b, &total) != cudaSuccess) {
      cudaGetLastError();
      return true;  // cannot tell: map on demand
    }
    const size_t have = op_ws_bytes(op);
    return per_col * (size_t)cols + margin <= free_b + have;
  };
  size_t free_b = 0;
  if (!fits(nrhs, free_b)) {
    release_idle_ops(op);
    if (!fits(nrhs, free_b) && nrhs > 1) {
      const size_t have = op_ws_bytes(op);
      const size_t avail = free_b + have > margin ? free_b + have - margin : 0;
      const int sub = std::max(1, std::min(nrhs - 1, (int)(avail / std::max(per_col, (size_t)1))));
      for (int c0 = 0; c0 < nrhs; c0 += sub) {
        const int k = std::min(sub, nrhs - c0);
        HG_TRY(gmres_dcgs2_run(op, weight, rhs + (long long)c0 * ldr, ldr, x + (long long)c0 * ldx, ldx, k, rtol,
                               maxit, history + (long long)c0 * (maxit + 1), info + 4 * c0, st));
      }
      op->basis = nullptr;  // several sub-bases: not inspectable as one
      op->basis_cols = op->basis_nv = 0;
      return HG_OK;
    }
  }
  return gmres_dcgs2_run(op, weight, rhs, ldr, x, ldx, nrhs, rtol, maxit, history, info, st);
}

static int gmres_dcgs2_run(HgOp* op, HgOp* weight, const double* rhs, long long ldr, double* x, long long ldx,
                           int nrhs, double rtol, int maxit, double* history, int32_t* info, cudaStream_t st) {
  const int n = op->n;
  const auto t_start = std::chrono::steady_clock::now();
  g_host_wait = g_host_work = 0.0;
  const bool weighted = weight != nullptr;
  const DevCsr* WA = nullptr;
  const double* wvals = nullptr;
  if (weighted) HG_TRY(weight_csr(weight, &WA, &wvals));
  // Y = W X for the listed columns (+ self dots X.Y into pself[c][nb] when given);
  // one column runs the single-vector SpMV kernels
  auto wspmv = [&](const double* X, double* Y, const ColList& cols, double* pself, int* nbs) -> int {
    if (nrhs == 1) {
      if (cols.n == 0) return HG_OK;
      if (pself) return launch_spmv_dots(*WA, wvals, X, Y, nullptr, 0, 0, false, pself, nbs, st);
      return launch_spmv(*WA, wvals, X, Y, st);
    }
    return launch_spmm_cols(*WA, wvals, X, n, Y, n, cols, pself, pself ? 1 : 0, nbs, st);
  };
  DcWs& ws = nrhs == 1 ? op->dws : op->dwsb;
  HG_TRY(dws_reserve(ws, n, nrhs, maxit + 1, weighted));
  const long long W2 = 2LL * (ws.cap + 2), Y2 = ws.cap + 2;
  const long long vstride = (long long)nrhs * n;
  const size_t vbytes = sizeof(double) * (size_t)n;
  // basis growth; on exhaustion release the other ops' idle bases once and retry
  auto grow = [&](size_t bytes) -> int {
    int r = ws.Q.ensure(bytes);
    if (r == HG_ERR_NOMEM && release_idle_ops(op) > 0) r = ws.Q.ensure(bytes);
    return r;
  };
  HG_TRY(grow(vbytes * nrhs));
  double* Q = ws.Q.ptr();
  auto qv = [&](int i) { return Q + (long long)i * vstride; };
  double* hdots = ws.hbuf;
  double* hnrm = hdots + W2 * nrhs;
  double* hcoef = hnrm + nrhs;
  double* hy = hcoef + W2 * nrhs;
  const int stride_h = maxit + 1;
  for (int c = 0; c < nrhs; ++c) info[4 * c] = info[4 * c + 1] = info[4 * c + 2] = info[4 * c + 3] = 0;
  ColList all{};
  all.n = nrhs;
  for (int c = 0; c < nrhs; ++c) all.c[c] = c;
  int nb = 0, nbs = 0;

  // q_0 = r0 / ||r0||_W (wgmres.py:102-115)
  HG_CUDA_TRY(cudaMemcpy2DAsync(Q, vbytes, rhs, sizeof(double) * ldr, vbytes, nrhs, cudaMemcpyDeviceToDevice, st));
  if (weighted) {
    HG_TRY(wspmv(Q, ws.wq, all, ws.pself, &nbs));
    HG_TRY(launch_reduce_batch(ws.pself, nbs, 1, 1, all, ws.nrm2, 1, st));
  } else {
    HG_TRY(launch_dots_batch(n, Q, n, nullptr, 0, 0, 0, all, ws.partials, 1, &nb, st));
    HG_TRY(launch_reduce_batch(ws.partials, nb, 1, 1, all, ws.nrm2, 1, st));
  }
  HG_CUDA_TRY(cudaMemcpyAsync(hnrm, ws.nrm2, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, st));
  HG_TRY(sync_check(st, op, weight));

  struct ColState {
    double beta = 0.0;
    std::vector<std::vector<double>> Hraw, Hrot;  // unrotated / rotated Hessenberg columns
    std::vector<double> cs, sn, g;
    int hist_len = 1;
    bool converged = false, breakdown = false;
    int explicit_passes = 0;
  };
  std::vector<ColState> cst(nrhs);
  ColList act{}, zero{};
  for (int c = 0; c < nrhs; ++c) {
    ColState& S = cst[c];
    S.beta = std::sqrt(hnrm[c]);
    history[(long long)c * stride_h] = S.beta;
    if (S.beta == 0.0 || maxit == 0) {
      S.converged = S.beta == 0.0;
      zero.c[zero.n++] = c;
    } else {
      S.g.assign(1, S.beta);
      act.c[act.n++] = c;
    }
  }
  HG_TRY(launch_fill_batch(n, x, ldx, zero, st));
  HG_TRY(launch_fill_batch(n, Q, n, zero, st));
  HG_TRY(launch_scale_dev_batch(n, Q, ws.wq, n, Q, n, weighted ? ws.wq : nullptr, ws.nrm2, act, st));
  const double BREAKDOWN_RTOL = 1e-14;

  // Givens rotation of the final column k (wgmres.py:158-184); true = stop
  auto finalize = [&](int c, int k) -> bool {
    ColState& S = cst[c];
    std::vector<double> col = S.Hraw[k];
    for (int i = 0; i < k; ++i) {
      const double t = S.cs[i] * col[i] - S.sn[i] * col[i + 1];
      col[i + 1] = S.sn[i] * col[i] + S.cs[i] * col[i + 1];
      col[i] = t;
    }
    const double denom = std::hypot(col[k], col[k + 1]);
    double csk = 1.0, snk = 0.0;
    if (denom != 0.0) {
      csk = col[k] / denom;
      snk = -col[k + 1] / denom;
    }
    S.cs.push_back(csk);
    S.sn.push_back(snk);
    col[k] = csk * col[k] - snk * col[k + 1];
    col[k + 1] = 0.0;
    S.Hrot.push_back(col);
    const double gk = S.g[k];
    S.g.push_back(snk * gk);
    S.g[k] = csk * gk;
    const double res = std::fabs(S.g[k + 1]);
    history[(long long)c * stride_h + S.hist_len++] = res;
    if (res <= rtol * S.beta || S.breakdown) {
      S.converged = true;
      return true;
    }
    return false;
  };

  for (int j = 0; act.n > 0; ++j) {
    const int nv = j + 1;
    if (nrhs > 1 && act.n < nrhs) {
      // finished columns ride along in the batched operator apply: feed them
      // zeros (their slot j of the on-demand basis was never written)
      ColList idle{};
      bool on[HG_MAX_RHS] = {false};
      for (int k = 0; k < act.n; ++k) on[act.c[k]] = true;
      for (int c = 0; c < nrhs; ++c)
        if (!on[c]) idle.c[idle.n++] = c;
      HG_TRY(launch_fill_batch(n, qv(j), n, idle, st));
    }
    {
      Phase ph(st, 0);
      if (nrhs == 1)
        HG_TRY(op_apply_dots(op, qv(j), ws.w, nullptr, 0, 0, nullptr, nullptr, st));
      else
        HG_TRY(op_apply_multi(op, qv(j), n, ws.w, n, nrhs, st));
    }
    const double* U = ws.w;
    if (weighted) {
      Phase ph(st, 6);
      HG_TRY(wspmv(ws.w, ws.u, act, nullptr, nullptr));
      U = ws.u;
    }
    {
      Phase ph(st, 1);
      // compact [c][2 nv] rows: one contiguous D2H per iteration
      HG_TRY(launch_dots2_batch(n, weighted ? ws.wq : qv(j), n, U, n, Q, vstride, n, nv, act, ws.partials, ws.dots,
                                2 * nv, st));
    }
    HG_CUDA_TRY(cudaMemcpyAsync(hdots, ws.dots, sizeof(double) * 2 * nv * nrhs, cudaMemcpyDeviceToHost, st));
    HG_CUDA_TRY(cudaMemcpyAsync(hnrm, ws.nrm2, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, st));
    const auto th0 = std::chrono::steady_clock::now();
    HG_TRY(sync_check(st, op, weight));
    const auto th1 = std::chrono::steady_clock::now();

    // DCGS2 safety: rho^2 = a_j - s.s loses its digits to cancellation when
    // q_j is nearly in span(Q) (rho^2 <= 1e-8 a_j leaves < 4 digits in rho).
    // Those columns take an explicit pass instead: q_j -= Q s on the device,
    // rho^2 = ||q_j||_W^2 measured directly (one more basis read + W SpMV for
    // them), and the update then skips the (already applied) correction.
    double rho2x[HG_MAX_RHS];
    bool expl[HG_MAX_RHS] = {false};
    if (j > 0) {
      ColList ex{};
      const bool force = g_force_explicit_rho.load() != 0;
      for (int k = 0; k < act.n; ++k) {
        const int c = act.c[k];
        const double* a = hdots + (long long)c * 2 * nv;
        const std::vector<double>& col = cst[c].Hraw[j - 1];
        const double beta = std::sqrt(std::max(hnrm[c], 0.0));
        double cscale = beta;
        for (int i = 0; i < j; ++i) cscale = std::max(cscale, std::fabs(col[i]));
        if (beta <= BREAKDOWN_RTOL * std::max(cscale, 1e-300)) continue;  // breakdown: no rho needed
        double ss = 0.0;
        for (int i = 0; i < j; ++i) ss += a[i] * a[i];
        if (force || !(a[j] - ss > 1e-8 * a[j])) {
          ex.c[ex.n++] = c;
          expl[c] = true;
          for (int i = 0; i < j; ++i) hcoef[(long long)c * j + i] = a[i];
        }
      }
      if (ex.n > 0) {
        HG_CUDA_TRY(cudaMemcpyAsync(ws.coef, hcoef, sizeof(double) * j * nrhs, cudaMemcpyHostToDevice, st));
        HG_TRY(launch_axpy_batch(n, qv(j), n, Q, vstride, n, j, ws.coef, j, 1, ex, st));  // q_j -= Q s
        if (weighted) {
          HG_TRY(wspmv(qv(j), ws.wq, ex, ws.pself, &nbs));
          HG_TRY(launch_reduce_batch(ws.pself, nbs, 1, 1, ex, ws.dy, 1, st));
        } else {
          HG_TRY(launch_dots_batch(n, qv(j), n, nullptr, 0, 0, 0, ex, ws.partials, 1, &nb, st));
          HG_TRY(launch_reduce_batch(ws.partials, nb, 1, 1, ex, ws.dy, 1, st));
        }
        HG_CUDA_TRY(cudaMemcpyAsync(hy, ws.dy, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, st));
        HG_TRY(sync_check(st, op, weight));
        for (int k = 0; k < ex.n; ++k) {
          rho2x[ex.c[k]] = hy[ex.c[k]];
          ++cst[ex.c[k]].explicit_passes;
        }
        g_explicit_rho_passes += ex.n;
      }
    }
    ColList keep{}, done{};
    int stopped[HG_MAX_RHS];
    // columns are independent: their host work (Givens, H s) runs in parallel
#pragma omp parallel for schedule(static, 1) num_threads(act.n) if (act.n >= 4)
    for (int k = 0; k < act.n; ++k) {
      const int c = act.c[k];
      stopped[k] = 0;
      ColState& S = cst[c];
      const double* a = hdots + (long long)c * 2 * nv;  // Q_i . W q_j
      const double* z = a + nv;                         // Q_i . W w
      double rho = 1.0;
      std::vector<double> s(j, 0.0);
      bool stop = false;
      if (j > 0) {
        std::vector<double>& col = S.Hraw[j - 1];
        const double beta = std::sqrt(std::max(hnrm[c], 0.0));
        double cscale = beta;
        for (int i = 0; i < j; ++i) cscale = std::max(cscale, std::fabs(col[i]));
        if (beta <= BREAKDOWN_RTOL * std::max(cscale, 1e-300)) {  // lucky breakdown (wgmres.py:151-156)
          col[j] = beta;
          S.breakdown = true;
          stop = finalize(c, j - 1);
        } else {
          double ss = 0.0;
          for (int i = 0; i < j; ++i) {
            s[i] = a[i];
            ss += s[i] * s[i];
          }
          // explicit pass: rho measured on the corrected vector (0 -> breakdown below)
          const double rho2 = expl[c] ? rho2x[c] : a[j] - ss;
          rho = std::sqrt(std::max(rho2, 0.0));
          for (int i = 0; i < j; ++i) col[i] += beta * s[i];
          col[j] = beta * rho;
          cscale = 0.0;
          for (int i = 0; i <= j; ++i) cscale = std::max(cscale, std::fabs(col[i]));
          if (col[j] <= BREAKDOWN_RTOL * std::max(cscale, 1e-300)) S.breakdown = true;
          stop = finalize(c, j - 1);
        }
      }
      if (!stop && j == maxit) stop = true;  // maxit columns finalised, not converged
      if (stop) {
        stopped[k] = 1;
        continue;
      }
      // projection of A q_j (q_j corrected) onto Q_{0:j}
      std::vector<double> col(j + 2, 0.0);
      double* cf = hcoef + (long long)c * (2 * j + 2);  // compact rows: one contiguous H2D
      cf[0] = 1.0 / rho;
      double sz = 0.0;
      for (int i = 0; i < j; ++i) {
        cf[1 + i] = expl[c] ? 0.0 : s[i];  // explicit pass: q_j already corrected on the device
        sz += s[i] * z[i];
      }
      // (H s)_i over the corrected columns 0..j-1, column by column (contiguous
      // inner loops; summed in ascending column order for every row)
      std::vector<double> hs(j + 1, 0.0);
      for (int kk = 0; kk < j; ++kk) {
        const double sk = s[kk];
        const double* hk = S.Hraw[kk].data();
        for (int i = 0; i <= kk + 1; ++i) hs[i] += hk[i] * sk;
      }
      for (int i = 0; i <= j; ++i) {
        const double zp = (i < j) ? z[i] : (z[j] - sz) / rho;
        const double h = (zp - hs[i]) / rho;
        col[i] = h;
        cf[1 + j + i] = hs[i] / rho + h;
      }
      S.Hraw.push_back(col);
    }
    for (int k = 0; k < act.n; ++k) {
      if (stopped[k])
        done.c[done.n++] = act.c[k];
      else
        keep.c[keep.n++] = act.c[k];
    }
    if (keep.n > 0 || done.n > 0) HG_TRY(grow(vbytes * nrhs * std::min(j + 2, ws.cap)));
    const auto th2 = std::chrono::steady_clock::now();
    if (host_timing()) {
      g_host_wait += std::chrono::duration<double>(th1 - th0).count();
      g_host_work += std::chrono::duration<double>(th2 - th1).count();
    }
    if (keep.n > 0) {
      HG_CUDA_TRY(cudaMemcpyAsync(ws.coef, hcoef, sizeof(double) * (2 * j + 2) * nrhs, cudaMemcpyHostToDevice, st));
      {
        Phase ph(st, 2);
        HG_TRY(launch_dcgs2_update(n, Q, vstride, n, j, ws.w, n, ws.coef, 2 * j + 2, keep, st));
      }
      {
        Phase ph(st, 3);
        if (weighted) {
          HG_TRY(wspmv(ws.w, ws.ww, keep, ws.pself, &nbs));
          HG_TRY(launch_reduce_batch(ws.pself, nbs, 1, 1, keep, ws.nrm2, 1, st));
        } else {
          HG_TRY(launch_dots_batch(n, ws.w, n, nullptr, 0, 0, 0, keep, ws.partials, 1, &nb, st));
          HG_TRY(launch_reduce_batch(ws.partials, nb, 1, 1, keep, ws.nrm2, 1, st));
        }
      }
      {
        Phase ph(st, 5);
        HG_TRY(launch_scale_dev_batch(n, ws.w, ws.ww, n, qv(j + 1), n, weighted ? ws.wq : nullptr, ws.nrm2, keep,
                                      st));
      }
    }
    act = keep;
  }
  // x_c = Q_c y_c with y_c = R_c^{-1} g_c (wgmres.py:186-192)
  std::vector<int> mlist(nrhs, 0);
  for (int c = 0; c < nrhs; ++c) {
    ColState& S = cst[c];
    const int m = S.hist_len - 1;
    mlist[c] = m;
    double* y = hy + c * Y2;
    for (int i = m - 1; i >= 0; --i) {
      double sacc = S.g[i];
      for (int k = i + 1; k < m; ++k) sacc -= S.Hrot[k][i] * y[k];
      y[i] = sacc / S.Hrot[i][i];
    }
  }
  HG_CUDA_TRY(cudaMemcpyAsync(ws.dy, hy, sizeof(double) * Y2 * nrhs, cudaMemcpyHostToDevice, st));
  for (int c = 0; c < nrhs; ++c) {
    ColList one{};
    one.n = 1;
    one.c[0] = c;
    if (mlist[c] > 0)
      HG_TRY(launch_axpy_batch(n, x, ldx, Q, vstride, n, mlist[c], ws.dy, Y2, 0, one, st));
    else if (cst[c].beta != 0.0)
      HG_TRY(launch_fill_batch(n, x, ldx, one, st));
  }
  HG_TRY(sync_check(st, op, weight));
  stats_collect();
  op->basis = Q;
  op->basis_ldv = vstride;
  op->basis_ldcol = n;
  op->basis_cols = nrhs;
  op->basis_nv = 0;
  for (int c = 0; c < nrhs; ++c) op->basis_nv = std::max(op->basis_nv, mlist[c]);
  if (host_timing()) {
    const double tot = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    fprintf(stderr, "[dcgs2 host] nrhs %d: total %.1f ms, waiting at the per-iteration sync %.1f ms, host work "
            "after it %.1f ms\n", nrhs, tot * 1e3, g_host_wait * 1e3, g_host_work * 1e3);
  }
  for (int c = 0; c < nrhs; ++c) {
    info[4 * c] = mlist[c];
    info[4 * c + 1] = cst[c].converged ? 1 : 0;
    info[4 * c + 2] = cst[c].breakdown ? 1 : 0;
    // every column is reorthogonalised once (delayed), plus its explicit rho passes
    info[4 * c + 3] = (mlist[c] > 0 ? mlist[c] - 1 : 0) + cst[c].explicit_passes;
  }
  return HG_OK;
}

extern "C" int hg_set_orthogonalization(int mode) {
  if (mode != HG_ORTH_MEASURED && mode != HG_ORTH_DCGS2) {
    set_error("hg_set_orthogonalization: unknown mode");
    return HG_ERR_ARG;
  }
  g_orth = mode;
  return HG_OK;
}

extern "C" int hg_get_orthogonalization(void) { return g_orth; }

// ------------------------------------------------------------------ batched GMRES
// WW[:, c] = W X[:, c] for the listed columns, self dots X_c . WW_c into pself[c][nb]
static int weight_apply_batch(HgOp* wop, const double* X, long long ldx, double* Y, long long ldy,
                              const ColList& cols, double* pself, int* nb, cudaStream_t st) {
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
  return launch_spmm_cols(*A, vals, X, ldx, Y, ldy, cols, pself, 1, nb, st);
}

static int bws_reserve(BatchWs& ws, int n, int nrhs, int cap, bool weighted) {
  if (ws.n == n && ws.nrhs == nrhs && ws.cap >= cap && ws.weighted == weighted) return HG_OK;
  ws.clear();
  ws.n = n;
  ws.nrhs = nrhs;
  ws.cap = cap;
  ws.weighted = weighted;
  const size_t vbytes = sizeof(double) * (size_t)n * nrhs * cap;
  HG_TRY(ws.V.reserve(vbytes));
  if (weighted) HG_TRY(ws.WV.reserve(vbytes));
  const size_t nn = (size_t)n * nrhs;
  HG_CUDA_TRY(cudaMalloc(&ws.w, sizeof(double) * nn));
  HG_CUDA_TRY(cudaMalloc(&ws.ww, sizeof(double) * nn));
  const size_t nb = (size_t)ceil_div(n, VEC_TILE);
  HG_CUDA_TRY(cudaMalloc(&ws.partials, sizeof(double) * nb * (cap + 2) * nrhs));
  HG_CUDA_TRY(cudaMalloc(&ws.pself, sizeof(double) * (size_t)ceil_div(n, 256) * nrhs));
  HG_CUDA_TRY(cudaMalloc(&ws.dh, sizeof(double) * (size_t)(cap + 2) * nrhs));
  HG_CUDA_TRY(cudaMalloc(&ws.dc, sizeof(double) * (size_t)(cap + 2) * nrhs));
  HG_CUDA_TRY(cudaMalloc(&ws.dy, sizeof(double) * (size_t)(cap + 2) * nrhs));
  HG_CUDA_TRY(cudaMallocHost(&ws.hbuf, sizeof(double) * 2 * (size_t)(cap + 2) * nrhs));
  return HG_OK;
}

extern "C" int hg_gmres_batch(HgOp* op, HgOp* weight, const double* rhs, int64_t ldr, double* x, int64_t ldx,
                              int32_t nrhs, double rtol, int32_t maxit, double* history, int32_t* info,
                              void* stream) {
  if (!op || !rhs || !x || !history || !info || nrhs < 1 || nrhs > HG_MAX_RHS || ldr < op->n || ldx < op->n) {
    set_error("hg_gmres_batch: bad argument");
    return HG_ERR_ARG;
  }
  if (weight && weight->n != op->n) {
    set_error("hg_gmres_batch: weight dimension mismatch");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n = op->n;
  maxit = std::max(0, std::min(maxit, n));
  HG_TRY(check_maxit(maxit));
  HG_TRY(op_fault(op));
  HG_TRY(op_fault(weight));
  BusyScope busy(op);
  if (g_orth == HG_ORTH_DCGS2) return gmres_dcgs2(op, weight, rhs, ldr, x, ldx, nrhs, rtol, maxit, history, info, st);
  const bool weighted = weight != nullptr;
  BatchWs& ws = op->bws;
  HG_TRY(bws_reserve(ws, n, nrhs, maxit + 1, weighted));
  const long long W2 = ws.cap + 2;                 // row pitch of dh / dc / dy / hbuf
  const long long vstride = (long long)nrhs * n;   // basis vector i -> i+1 of one column
  const size_t vec_bytes = sizeof(double) * (size_t)n;
  HG_TRY(ws.V.ensure(vec_bytes * nrhs));
  if (weighted) HG_TRY(ws.WV.ensure(vec_bytes * nrhs));
  double* V = ws.V.ptr();
  double* WV = weighted ? ws.WV.ptr() : V;
  auto vec = [&](double* B, int i) { return B + (long long)i * vstride; };  // column 0 of basis vector i
  double* hb = ws.hbuf;
  double* hb2 = ws.hbuf + W2 * nrhs;
  const int stride_h = maxit + 1;
  for (int c = 0; c < nrhs; ++c) info[4 * c] = info[4 * c + 1] = info[4 * c + 2] = info[4 * c + 3] = 0;

  ColList all{};
  all.n = nrhs;
  for (int c = 0; c < nrhs; ++c) all.c[c] = c;
  int nb = 0, nbs = 0;
  // r0 = rhs (x0 = 0), beta_c = ||r0_c||_W
  HG_CUDA_TRY(cudaMemcpy2DAsync(V, vec_bytes, rhs, sizeof(double) * ldr, vec_bytes, nrhs, cudaMemcpyDeviceToDevice, st));
  if (weighted) {
    HG_TRY(weight_apply_batch(weight, V, n, WV, n, all, ws.pself, &nbs, st));
    HG_TRY(launch_reduce_batch(ws.pself, nbs, 1, 1, all, ws.dc, W2, st));
  } else {
    HG_TRY(launch_dots_batch(n, V, n, nullptr, 0, 0, 0, all, ws.partials, 1, &nb, st));
    HG_TRY(launch_reduce_batch(ws.partials, nb, 1, 1, all, ws.dc, W2, st));
  }
  HG_CUDA_TRY(cudaMemcpy2DAsync(hb, sizeof(double), ws.dc, sizeof(double) * W2, sizeof(double), nrhs,
                                cudaMemcpyDeviceToHost, st));
  HG_TRY(sync_check(st, op, weight));

  struct ColState {
    double beta = 0.0;
    std::vector<std::vector<double>> H;  // Givens-rotated Hessenberg columns
    std::vector<double> cs, sn, g;
    int hist_len = 1;
    bool converged = false, breakdown = false;
    int reorth = 0;
  };
  std::vector<ColState> cst(nrhs);
  ColList act{}, zero{};
  for (int c = 0; c < nrhs; ++c) {
    ColState& S = cst[c];
    S.beta = std::sqrt(hb[c]);
    history[(long long)c * stride_h] = S.beta;
    if (S.beta == 0.0) {
      S.converged = true;
      zero.c[zero.n++] = c;
    } else {
      S.g.assign(1, S.beta);
      act.s[act.n] = S.beta;
      act.c[act.n++] = c;
    }
  }
  HG_TRY(launch_fill_batch(n, x, ldx, zero, st));
  HG_TRY(launch_fill_batch(n, V, n, zero, st));  // finite op inputs for finished columns
  HG_TRY(launch_scale_batch(n, V, WV, n, V, weighted ? WV : nullptr, n, act, st));
  const double REORTH_TOL = 1e-12, BREAKDOWN_RTOL = 1e-14;
  std::vector<double> col(maxit + 2, 0.0);

  for (int j = 0; j < maxit && act.n > 0; ++j) {
    const int nv = j + 1;
    HG_TRY(ws.V.ensure(vec_bytes * nrhs * (j + 2)));
    if (weighted) HG_TRY(ws.WV.ensure(vec_bytes * nrhs * (j + 2)));
    {  // w_c = op(V_c[j]) for the whole batch (finished columns carry zeros)
      Phase ph(st, 0);
      HG_TRY(op_apply_multi(op, vec(V, j), n, ws.w, n, nrhs, st));
    }
    {  // classical pass: h_c = (W V_c)^T w_c ; w_c -= V_c h_c
      Phase ph(st, 1);
      HG_TRY(launch_dots_batch(n, ws.w, n, WV, vstride, n, nv, act, ws.partials, nv + 1, &nb, st));
      HG_TRY(launch_reduce_batch(ws.partials, nb, nv + 1, nv + 1, act, ws.dh, W2, st));
    }
    {
      Phase ph(st, 2);
      HG_TRY(launch_axpy_batch(n, ws.w, n, V, vstride, n, nv, ws.dh + 1, W2, 1, act, st));
    }
    {  // measurement corr_c = (W V_c)^T w_c, then ww_c = W w_c with w_c . ww_c (slot 0)
      Phase ph(st, 3);
      HG_TRY(launch_dots_batch(n, ws.w, n, WV, vstride, n, nv, act, ws.partials, nv + 1, &nb, st));
      HG_TRY(launch_reduce_batch(ws.partials, nb, nv + 1, nv + 1, act, ws.dc, W2, st));
      if (weighted) {
        HG_TRY(weight_apply_batch(weight, ws.w, n, ws.ww, n, act, ws.pself, &nbs, st));
        HG_TRY(launch_reduce_batch(ws.pself, nbs, 1, 1, act, ws.dc, W2, st));
      }
    }
    HG_CUDA_TRY(cudaMemcpy2DAsync(hb, sizeof(double) * W2, ws.dh, sizeof(double) * W2, sizeof(double) * (nv + 1),
                                  nrhs, cudaMemcpyDeviceToHost, st));
    HG_CUDA_TRY(cudaMemcpy2DAsync(hb2, sizeof(double) * W2, ws.dc, sizeof(double) * W2, sizeof(double) * (nv + 1),
                                  nrhs, cudaMemcpyDeviceToHost, st));
    HG_TRY(sync_check(st, op, weight));
    std::vector<std::vector<double>> cols(nrhs);
    std::vector<double> hnorm(nrhs, 0.0);
    ColList ro{};
    for (int k = 0; k < act.n; ++k) {
      const int c = act.c[k];
      const double* h = hb + c * W2 + 1;
      const double* dcc = hb2 + c * W2;
      std::vector<double>& cc = cols[c];
      cc.assign(j + 2, 0.0);
      for (int i = 0; i < nv; ++i) cc[i] = h[i];
      hnorm[c] = std::sqrt(std::max(dcc[0], 0.0));
      double cmax = 0.0;
      for (int i = 0; i < nv; ++i) cmax = std::max(cmax, std::fabs(dcc[1 + i]));
      if (cmax > REORTH_TOL * std::max(hnorm[c], 1e-300)) {  // wgmres.py:142-148
        for (int i = 0; i < nv; ++i) cc[i] += dcc[1 + i];
        ro.c[ro.n++] = c;
        ++cst[c].reorth;
      }
    }
    if (ro.n > 0) {
      Phase ph(st, 4);
      HG_TRY(launch_axpy_batch(n, ws.w, n, V, vstride, n, nv, ws.dc + 1, W2, 1, ro, st));
      if (weighted) {
        HG_TRY(weight_apply_batch(weight, ws.w, n, ws.ww, n, ro, ws.pself, &nbs, st));
        HG_TRY(launch_reduce_batch(ws.pself, nbs, 1, 1, ro, ws.dc, W2, st));
      } else {
        HG_TRY(launch_dots_batch(n, ws.w, n, nullptr, 0, 0, 0, ro, ws.partials, 1, &nb, st));
        HG_TRY(launch_reduce_batch(ws.partials, nb, 1, 1, ro, ws.dc, W2, st));
      }
      HG_CUDA_TRY(cudaMemcpy2DAsync(hb2, sizeof(double), ws.dc, sizeof(double) * W2, sizeof(double), nrhs,
                                    cudaMemcpyDeviceToHost, st));
      HG_TRY(sync_check(st, op, weight));
      for (int k = 0; k < ro.n; ++k) hnorm[ro.c[k]] = std::sqrt(std::max(hb2[ro.c[k]], 0.0));
    }
    ColList scl{}, done{}, keep{};
    for (int k = 0; k < act.n; ++k) {
      const int c = act.c[k];
      ColState& S = cst[c];
      std::vector<double>& cc = cols[c];
      cc[j + 1] = hnorm[c];
      double cscale = 0.0;
      for (int i = 0; i <= j + 1; ++i) cscale = std::max(cscale, std::fabs(cc[i]));
      if (hnorm[c] <= BREAKDOWN_RTOL * std::max(cscale, 1e-300)) {
        S.breakdown = true;
      } else {
        scl.s[scl.n] = hnorm[c];
        scl.c[scl.n++] = c;
      }
      // Givens update (wgmres.py:158-171)
      for (int i = 0; i < j; ++i) {
        const double t = S.cs[i] * cc[i] - S.sn[i] * cc[i + 1];
        cc[i + 1] = S.sn[i] * cc[i] + S.cs[i] * cc[i + 1];
        cc[i] = t;
      }
      const double denom = std::hypot(cc[j], cc[j + 1]);
      double csj = 1.0, snj = 0.0;
      if (denom != 0.0) {
        csj = cc[j] / denom;
        snj = -cc[j + 1] / denom;
      }
      S.cs.push_back(csj);
      S.sn.push_back(snj);
      cc[j] = csj * cc[j] - snj * cc[j + 1];
      cc[j + 1] = 0.0;
      S.H.push_back(cc);
      const double gj = S.g[j];
      S.g.push_back(snj * gj);
      S.g[j] = csj * gj;
      const double res = std::fabs(S.g[j + 1]);
      history[(long long)c * stride_h + S.hist_len++] = res;
      if (res <= rtol * S.beta || S.breakdown) {
        S.converged = true;
        done.c[done.n++] = c;
      } else {
        keep.s[keep.n] = act.s[k];
        keep.c[keep.n++] = c;
      }
    }
    {
      Phase ph(st, 5);
      HG_TRY(launch_scale_batch(n, ws.w, ws.ww, n, vec(V, j + 1), weighted ? vec(WV, j + 1) : nullptr, n, scl,
                                st));
      HG_TRY(launch_fill_batch(n, vec(V, j + 1), n, done, st));  // finished columns feed zeros to the op
    }
    act = keep;
  }
  // x_c = V_c y_c, y_c = H_c^{-1} g_c (host back substitution, wgmres.py:186-192)
  std::vector<int> mlist(nrhs, 0);
  for (int c = 0; c < nrhs; ++c) {
    ColState& S = cst[c];
    const int m = S.hist_len - 1;
    mlist[c] = m;
    double* y = hb + c * W2;
    for (int i = m - 1; i >= 0; --i) {
      double s = S.g[i];
      for (int k = i + 1; k < m; ++k) s -= S.H[k][i] * y[k];
      y[i] = s / S.H[i][i];
    }
  }
  HG_CUDA_TRY(cudaMemcpyAsync(ws.dy, hb, sizeof(double) * W2 * nrhs, cudaMemcpyHostToDevice, st));
  for (int c = 0; c < nrhs; ++c) {
    ColList one{};
    one.n = 1;
    one.c[0] = c;
    if (mlist[c] > 0)
      HG_TRY(launch_axpy_batch(n, x, ldx, V, vstride, n, mlist[c], ws.dy, W2, 0, one, st));
    else if (cst[c].beta != 0.0)
      HG_TRY(launch_fill_batch(n, x, ldx, one, st));
  }
  HG_TRY(sync_check(st, op, weight));
  stats_collect();
  op->basis = V;
  op->basis_ldv = vstride;
  op->basis_ldcol = n;
  op->basis_cols = nrhs;
  op->basis_nv = 0;
  for (int c = 0; c < nrhs; ++c) op->basis_nv = std::max(op->basis_nv, mlist[c]);
  for (int c = 0; c < nrhs; ++c) {
    info[4 * c] = mlist[c];
    info[4 * c + 1] = cst[c].converged ? 1 : 0;
    info[4 * c + 2] = cst[c].breakdown ? 1 : 0;
    info[4 * c + 3] = cst[c].reorth;
  }
  return HG_OK;
}

extern "C" int hg_solve_host_batch(HgPrecond* P, const double* F_host, double* X_host, int32_t nrhs, double rtol,
                                   int32_t maxit, double* history, int32_t* info, void* stream) {
  if (!P || !F_host || !X_host || nrhs < 1 || nrhs > HG_MAX_RHS) {
    set_error("hg_solve_host_batch: bad argument");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n = P->n;
  HG_TRY(precond_fault(P));
  HG_TRY(ensure_solve_ops(P));
  const size_t bytes = sizeof(double) * (size_t)n * nrhs;
  double *d_f = nullptr, *d_rhs = nullptr, *d_x = nullptr;
  HG_CUDA_TRY(cudaMallocAsync(&d_f, bytes, st));
  HG_CUDA_TRY(cudaMallocAsync(&d_rhs, bytes, st));
  HG_CUDA_TRY(cudaMallocAsync(&d_x, bytes, st));
  HG_CUDA_TRY(cudaMemcpyAsync(d_f, F_host, bytes, cudaMemcpyHostToDevice, st));
  int s = precond_apply_multi_core(P, d_f, n, d_rhs, n, nrhs, st);
  if (s == HG_OK)
    s = hg_gmres_batch(P->op_T, P->A.data2 ? P->op_W : nullptr, d_rhs, n, d_x, n, nrhs, rtol, maxit, history, info,
                       stream);
  if (s == HG_OK) HG_CUDA_TRY(cudaMemcpyAsync(X_host, d_x, bytes, cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(d_f, st);
  cudaFreeAsync(d_rhs, st);
  cudaFreeAsync(d_x, st);
  HG_CUDA_TRY(cudaStreamSynchronize(st));
  if (s == HG_OK) s = precond_fault(P);
  return s;
}

extern "C" int hg_op_basis(HgOp* op, int32_t col, int32_t nv, double* out, void* stream) {
  if (!op || !out || !op->basis || col < 0 || col >= op->basis_cols || nv < 0 || nv > op->basis_nv) {
    set_error("hg_op_basis: no such basis (solve first; col / nv out of range)");
    return HG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t vb = sizeof(double) * (size_t)op->n;
  if (nv > 0)
    HG_CUDA_TRY(cudaMemcpy2DAsync(out, vb, op->basis + (long long)col * op->basis_ldcol, sizeof(double) * op->basis_ldv,
                                  vb, nv, cudaMemcpyDeviceToDevice, st));
  HG_CUDA_TRY(cudaStreamSynchronize(st));
  return HG_OK;
}
