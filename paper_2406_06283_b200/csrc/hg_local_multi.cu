// Multi-RHS instantiations of the local band solve (one consumer warp per
// right-hand side on a shared factor stream), compiled separately so that
// their register budget (544-thread blocks) does not constrain the
// single-RHS kernel of hg_local.cu.
#include "hg_local_impl.cuh"

namespace hg {

int launch_local_solve_multi(HgPrecond* P, const double* R, long long ldr, int nrhs, cudaStream_t st) {
  if (P->n_local == 0) return HG_OK;
  if (nrhs < 1 || nrhs > HG_MAX_RHS) {
    set_error("local band solve: nrhs out of range");
    return HG_ERR_ARG;
  }
  return launch_local_grid_t<HG_MAX_RHS>(P, P->d_local, P->n_local, R, st, nrhs, ldr, P->d_xsm, P->xs_len);
}

int preload_local_multi(HgPrecond* P) {
  cudaFuncAttributes at;
  LocalKernel k = pick_local<HG_MAX_RHS>(P->rf, P->rb);
  if (k) HG_CUDA_TRY(cudaFuncGetAttributes(&at, k));
  return preload_local_panel();
}

}  // namespace hg
