// registry.cuh — size-specialised kernel instances and their launchers.
// One entry per (equation, n, b): the generator's size specialisation
// (lowering.py:952 bakes n into every kernel) mirrored as
// template instantiations; the variant itself is a runtime statement list.
#pragma once
#include <atomic>

#include "solver.cuh"

namespace lagen {

struct LaunchArgs {
  StmtList sl;
  const double* in[3];
  double* X;
  int* info;
  long long batch;
  unsigned long long* prof;  // warp-engine cycle accounting (profiling only), usually null
};

typedef cudaError_t (*LaunchFn)(const LaunchArgs&, cudaStream_t);

// SMs the persistent engines may fill (the calling thread's reservation, 0 by
// default): the host pipeline leaves a few SMs to its zero-copy transfer
// kernels, which otherwise could not start while a persistent solve holds
// every SM
inline thread_local int t_sm_reserve = 0;
inline long long sm_budget(int sms) { return sms - t_sm_reserve < 1 ? 1 : sms - t_sm_reserve; }

struct KernelEntry {
  int eq, n, b;
  int G, P, threads;
  int smem;
  LaunchFn launch;
};

template <int EQ, int N, int B>
cudaError_t launch_solve(const LaunchArgs& a, cudaStream_t s) {
  using Pol = Policy<EQ, N>;
  static std::atomic<unsigned long long> configured{0};  // bit per device
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    err = cudaFuncSetAttribute(solve_kernel<EQ, N, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Pol::SMEM);
    if (err != cudaSuccess) return err;
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  if (a.batch <= 0) return cudaSuccess;
  const long long grid = (a.batch + Pol::P - 1) / Pol::P;
  solve_kernel<EQ, N, B><<<(unsigned)grid, Pol::THREADS, Pol::SMEM, s>>>(a.sl, a.in[0], a.in[1], a.in[2], a.X,
                                                                        a.info, a.batch);
  return cudaGetLastError();
}

#define LAGEN_ENTRY(EQ, N, B)                                                                             \
  {                                                                                                       \
    EQ, N, B, Policy<EQ, N>::G, Policy<EQ, N>::P, Policy<EQ, N>::THREADS, (int)Policy<EQ, N>::SMEM, \
        &launch_solve<EQ, N, B>                                                                          \
  }

}  // namespace lagen
