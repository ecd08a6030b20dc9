// registry_col.cuh — column-engine instances (Cholesky, n <= 64).
#pragma once
#include <atomic>

#include "colengine.cuh"
#include "registry.cuh"

namespace lagen {

struct ColEntry {
  int n, b, variant;
  int smem;
  LaunchFn launch;
};

template <int N, int B, int VAR>
cudaError_t launch_col(const LaunchArgs& a, cudaStream_t s) {
  using P = col::ColPolicy<N>;
  static std::atomic<unsigned long long> configured{0};
  static std::atomic<int> ctas_per_sm{0};
  static std::atomic<int> sm_count{0};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const unsigned long long bit = 1ull << (dev & 63);
  auto kern = col::chol_col_kernel<N, B, VAR>;
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM);
    if (err != cudaSuccess) return err;
    int occ = 0, sms = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, P::WARPS * 32, P::SMEM);
    if (err != cudaSuccess) return err;
    err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err != cudaSuccess) return err;
    ctas_per_sm.store(occ > 0 ? occ : 1);
    sm_count.store(sms);
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  if (a.batch <= 0) return cudaSuccess;
  const long long per_cta = (long long)P::WARPS * P::GPW;
  const long long need = (a.batch + per_cta - 1) / per_cta;
  const long long resident = (long long)ctas_per_sm.load() * sm_budget(sm_count.load());
  const long long grid = need < resident ? need : resident;
  kern<<<(unsigned)grid, P::WARPS * 32, P::SMEM, s>>>(a.in[0], a.X, a.info, a.batch);
  return cudaGetLastError();
}

#define LAGEN_COL_ENTRY(N, B, VI) \
  { N, B, VI, col::ColPolicy<N>::SMEM, &launch_col<N, B, VI> }

}  // namespace lagen
