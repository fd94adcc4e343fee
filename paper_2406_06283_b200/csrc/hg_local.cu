#include "hg_local_impl.cuh"

namespace hg {

static int launch_local_grid(HgPrecond* P, const LocalDesc* descs, int nblocks, const double* r,
                             cudaStream_t st) {
  return launch_local_grid_t<1>(P, descs, nblocks, r, st, 1, 0, nullptr, 0);
}

__global__ void k_scatter_local(int n, const int* __restrict__ idx, const double* __restrict__ src,
                                double* __restrict__ dst);

// CUDA lazy loading would load a kernel at its first launch, which waits for
// running kernels — a deadlock when the spinning coarse solve is resident.
// Every kernel the handle uses is loaded at creation instead.
int preload_local(HgPrecond* P) {
  cudaFuncAttributes at;
  LocalKernel k = pick_local<1>(P->rf, P->rb);
  if (k) HG_CUDA_TRY(cudaFuncGetAttributes(&at, k));
  HG_TRY(preload_local_multi(P));
  HG_CUDA_TRY(cudaFuncGetAttributes(&at, k_scatter_local));
  return HG_OK;
}

int launch_local_solve(HgPrecond* P, const double* r, cudaStream_t st) {
  if (P->n_local == 0) return HG_OK;
  HG_TRY(launch_local_grid(P, P->d_local, P->n_local, r, st));
  return launch_split_stages(P, r, 0, P->d_xs, 0, 1, st);  // split subdomains: separators, spikes
}

__global__ void k_scatter_local(int n, const int* __restrict__ idx, const double* __restrict__ src,
                                double* __restrict__ dst) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[idx[k]] = src[k];
}

int launch_local_solve_single(HgPrecond* P, int s, const double* r_local, double* x_local,
                              cudaStream_t st) {
  const LocalDesc& d = P->h_local[s];
  if (d.n == 0) return HG_OK;
  k_scatter_local<<<ceil_div(d.n, 256), 256, 0, st>>>(d.n, P->d_local_idx + d.idx_off, r_local, P->d_tmp);
  HG_LAUNCH_CHECK();
  HG_TRY(launch_local_grid(P, P->d_local + s, 1, P->d_tmp, st));
  HG_CUDA_TRY(cudaMemcpyAsync(x_local, P->d_xs + d.idx_off, sizeof(double) * d.n, cudaMemcpyDeviceToDevice, st));
  return HG_OK;
}

}  // namespace hg
