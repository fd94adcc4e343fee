// Shared device helpers: error plumbing, mbarrier / bulk-copy PTX wrappers,
// warp reductions.  sm_100a only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/helmgpu.h"

namespace hg {

void set_error(const std::string& msg);
void count_launch(int n = 1);

#define HG_CUDA_TRY(expr)                                                                     \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) {                                                                  \
      ::hg::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" __FILE__ ":" + \
                      std::to_string(__LINE__));                                              \
      return HG_ERR_CUDA;                                                                     \
    }                                                                                         \
  } while (0)

#define HG_LAUNCH_CHECK()                                                                      \
  do {                                                                                         \
    ::hg::count_launch();                                                                      \
    cudaError_t _e = cudaGetLastError();                                                       \
    if (_e != cudaSuccess) {                                                                   \
      ::hg::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e) + " @" __FILE__ \
                      ":" + std::to_string(__LINE__));                                         \
      return HG_ERR_CUDA;                                                                      \
    }                                                                                          \
  } while (0)

#define HG_TRY(expr)              \
  do {                            \
    int _s = (expr);              \
    if (_s != HG_OK) return _s;   \
  } while (0)

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// TMA bulk (non-tensor) copy global -> shared, completion counted on `bar`.
// bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// ---- bounded spin waits
// Every cross-CTA / cross-kernel wait in this library polls through a
// SpinGuard: each 256 failed polls it reads the handle's fault word (host
// mapped, so the host sees it without an API call) and %globaltimer; past
// `limit_ns` it raises the fault and the wait gives up.  A kernel whose wait
// gave up finishes its loops on garbage (it never leaves a barrier its peers
// wait on), and every later wait on a faulted handle gives up at once; the
// host turns the fault into HG_ERR_CUDA and poisons the handle.
struct SpinCfg {
  volatile int* fault;          // device alias of the handle's pinned fault word
  unsigned long long limit_ns;  // 0 = no limit
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct SpinGuard {
  unsigned long long t0 = 0;
  unsigned n = 0;
};

// true = stop waiting (timeout raised here, or the handle already faulted)
__device__ __forceinline__ bool spin_abort(SpinGuard& g, const SpinCfg& cfg) {
  if ((++g.n & 255u) != 0u) return false;
  if (cfg.fault && *cfg.fault) return true;
  const unsigned long long t = global_ns();
  if (g.t0 == 0) {
    g.t0 = t;
    return false;
  }
  if (cfg.limit_ns && t - g.t0 > cfg.limit_ns) {
    if (cfg.fault) {
      *cfg.fault = 1;
      __threadfence_system();
    }
    return true;
  }
  return false;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Launch index of a coarse solve from its device ticket counter: every CTA
// of a launch takes one ticket, launches on a handle are stream ordered, so
// CTAs of launch L hold tickets [L * ctas, (L + 1) * ctas).  The t-th coarse
// solve pairs with the t-th Z^T r launch (whose chunks bump the per-block
// counters), also under CUDA-graph replay — no host-side epoch is baked in.
__device__ __forceinline__ unsigned long long take_launch_index(unsigned long long* ticket, unsigned ctas) {
  return atomicAdd(ticket, 1ull) / ctas;
}

}  // namespace hg
