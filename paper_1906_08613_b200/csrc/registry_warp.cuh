// registry_warp.cuh — warp-engine instances: (equation, n, b, variant) with
// the variant's statement list compiled in.
#pragma once
#include <atomic>

#include "engine.cuh"
#include "registry.cuh"
#include "variants_ct.cuh"

namespace lagen {

struct WarpEntry {
  int eq, n, b, variant;
  int warps;
  int smem;
  LaunchFn launch;
};

template <int EQ, int N, int B, class VAR>
cudaError_t launch_warp(const LaunchArgs& a, cudaStream_t s) {
  using P = eng::WPolicy<EQ, N>;
  static std::atomic<unsigned long long> configured{0};
  static std::atomic<int> ctas_per_sm{0};
  static std::atomic<int> sm_count{0};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const unsigned long long bit = 1ull << (dev & 63);
  auto kern = eng::warp_kernel<EQ, N, B, VAR>;
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
  const long long resident = (long long)ctas_per_sm.load() * sm_budget(sm_count.load());
  const long long grid = need < resident ? need : resident;
  kern<<<(unsigned)grid, P::WARPS * 32, P::SMEM, s>>>(a.in[0], a.in[1], a.in[2], a.X, a.info, a.batch, a.prof);
  return cudaGetLastError();
}

#define LAGEN_WARP_ENTRY(EQ, N, B, VI, VAR) \
  { EQ, N, B, VI, eng::WPolicy<EQ, N>::WARPS, (int)eng::WPolicy<EQ, N>::SMEM, &launch_warp<EQ, N, B, VAR> }

}  // namespace lagen
