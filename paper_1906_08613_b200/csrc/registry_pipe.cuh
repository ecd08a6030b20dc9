// registry_pipe.cuh — pipe-engine instances (Lyapunov v5 / Sylvester v13
// order, 8x8 tiles; see pipe.cuh).  One kernel per (equation, n); for
// T = ceil(n / 8) <= 4 both modes (split roles / one warp per problem) are
// instantiated and the measured faster one is the default
// (LAGEN_PIPE_MODE=0|1 forces one for A/B runs).
#pragma once
#include <atomic>
#include <cstdlib>

#include "pipe.cuh"
#include "registry.cuh"

namespace lagen {

struct PipeEntry {
  int eq, n;
  LaunchFn launch;
};

// default mode per tile count
// solo (one warp per problem) for T <= 2, and for Sylvester T = 4 where it beats
// both the split roles and the rowsweep engine (profiles/r02_pipe_solo.txt)
constexpr int pipe_default_mode(int eq, int t) { return (t <= 2 || (eq == 2 && t == 4)) ? 1 : 0; }

template <int EQ, int N, int MODE>
cudaError_t launch_pipe_mode(const LaunchArgs& a, cudaStream_t s) {
  using P = pipe::PCfg<EQ, N, MODE>;
  static std::atomic<unsigned long long> configured{0};
  static std::atomic<int> ctas_per_sm{0};
  static std::atomic<int> sm_count{0};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const unsigned long long bit = 1ull << (dev & 63);
  auto kern = pipe::pipe_kernel<EQ, N, MODE>;
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
  const long long need = (a.batch + P::PP - 1) / P::PP;
  const long long resident = (long long)ctas_per_sm.load() * sm_budget(sm_count.load());
  const long long grid = need < resident ? need : resident;
  // _signature order: lyapunov (L, S), sylvester (L, U, C)
  const double* L = a.in[0];
  const double* U = EQ == 2 ? a.in[1] : a.in[0];
  const double* C = EQ == 2 ? a.in[2] : a.in[1];
  kern<<<(unsigned)grid, P::THREADS, P::SMEM, s>>>(L, U, C, a.X, a.info, a.batch, a.prof);
  return cudaGetLastError();
}

template <int EQ, int N>
cudaError_t launch_pipe(const LaunchArgs& a, cudaStream_t s) {
  constexpr int T = (N + 7) / 8;
  constexpr int maxm = EQ == 2 ? T : (T + 1) / 2;
  static const int forced = [] {
    const char* e = std::getenv("LAGEN_PIPE_MODE");
    return e ? std::atoi(e) : -1;
  }();
  if constexpr (maxm <= 4) {
    const int mode = forced >= 0 ? forced : pipe_default_mode(EQ, T);
    if (mode == 1) return launch_pipe_mode<EQ, N, 1>(a, s);
  }
  return launch_pipe_mode<EQ, N, 0>(a, s);
}

#define LAGEN_PIPE_ENTRY(EQ, N) \
  { EQ, N, &launch_pipe<EQ, N> }

struct PipeTable {
  const PipeEntry* e;
  const int* n;
};

}  // namespace lagen
