// registry_rows.cuh — rows-engine instances (Cholesky v1, packed row-major X).
#pragma once
#include <atomic>
#include <cstdlib>

#include "chol_rows.cuh"
#include "registry.cuh"

namespace lagen {

struct RowsEntry {
  int n, b, variant;
  int smem;
  LaunchFn launch;
};

template <int N, int B>
cudaError_t launch_rows(const LaunchArgs& a, cudaStream_t s) {
  using P = eng::WPolicy<0, N>;
  static std::atomic<unsigned long long> configured{0};
  static std::atomic<int> ctas_per_sm{0};
  static std::atomic<int> sm_count{0};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const unsigned long long bit = 1ull << (dev & 63);
  auto kern = cr::chol_rows_kernel<N, B>;
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
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
  const long long need = (a.batch + P::P - 1) / P::P;
  const long long resident = (long long)ctas_per_sm.load() * sm_count.load();
  const long long grid = need < resident ? need : resident;
  // mode = k-split (bits 0-1) | work split (bits 2-3); LAGEN_ROWS_MODE
  // overrides the tuned default (tuning runs only)
  static const int mode = [] {
    const char* e = std::getenv("LAGEN_ROWS_MODE");
    return e ? std::atoi(e) : cr::default_mode(N, B);
  }();
  kern<<<(unsigned)grid, P::WARPS * 32, P::SMEM, s>>>(a.in[0], a.X, a.info, a.batch, mode);
  return cudaGetLastError();
}

#define LAGEN_ROWS_ENTRY(N, B) \
  { N, B, 1, (int)eng::WPolicy<0, N>::SMEM, &launch_rows<N, B> }

}  // namespace lagen
