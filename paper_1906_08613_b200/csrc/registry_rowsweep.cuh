// registry_rowsweep.cuh — rowsweep-engine instances (Lyapunov / Sylvester,
// n <= 32, one lane per row; see rowsweep.cuh).  One kernel per (equation, n).
#pragma once
#include <atomic>

#include "registry.cuh"
#include "rowsweep.cuh"

namespace lagen {

struct RowSweepEntry {
  int eq, n;
  LaunchFn launch;
};

template <int EQ, int N>
cudaError_t launch_rowsweep(const LaunchArgs& a, cudaStream_t s) {
  using P = rsw::RCfg<EQ, N>;
  static std::atomic<unsigned long long> configured{0};
  static std::atomic<int> ctas_per_sm{0};
  static std::atomic<int> sm_count{0};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const unsigned long long bit = 1ull << (dev & 63);
  auto kern = rsw::rowsweep_kernel<EQ, N>;
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    if (err != cudaSuccess) return err;
    int occ = 0, sms = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, P::THREADS, P::SMEM);
    if (err != cudaSuccess) return err;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err != cudaSuccess) return err;
    ctas_per_sm.store(occ);
    sm_count.store(sms);
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  if (a.batch <= 0) return cudaSuccess;
  const long long per_cta = (long long)P::W * P::PPW;
  const long long need = (a.batch + per_cta - 1) / per_cta;
  const long long resident = (long long)ctas_per_sm.load() * sm_budget(sm_count.load());
  const long long grid = need < resident ? need : resident;
  const double* L = a.in[0];
  const double* U = EQ == 2 ? a.in[1] : a.in[0];
  const double* C = EQ == 2 ? a.in[2] : a.in[1];
  kern<<<(unsigned)grid, P::THREADS, P::SMEM, s>>>(L, U, C, a.X, a.info, a.batch);
  return cudaGetLastError();
}

#define LAGEN_ROWSWEEP_ENTRY(EQ, N) \
  { EQ, N, &launch_rowsweep<EQ, N> }

struct RowSweepTable {
  const RowSweepEntry* e;
  const int* n;
};

}  // namespace lagen
