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

template <int N, int B, int WG, int NR = N, bool F4 = false>
cudaError_t launch_rows_wg(const LaunchArgs& a, cudaStream_t s, int mode) {
  using P = cr::RPolicy<N, WG>;
  static std::atomic<unsigned long long> configured{0};
  static std::atomic<int> ctas_per_sm{0};
  static std::atomic<int> sm_count{0};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const unsigned long long bit = 1ull << (dev & 63);
  auto kern = cr::chol_rows_kernel<N, B, WG, NR, F4>;
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    if (err != cudaSuccess) return err;
    int occ = 0, sms = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, P::WARPS * 32, P::SMEM);
    if (err != cudaSuccess) return err;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err != cudaSuccess) return err;
    ctas_per_sm.store(occ);
    sm_count.store(sms);
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  if (a.batch <= 0) return cudaSuccess;
  const long long need = (a.batch + P::P - 1) / P::P;
  const long long resident = (long long)ctas_per_sm.load() * sm_budget(sm_count.load());
  const long long grid = need < resident ? need : resident;
  kern<<<(unsigned)grid, P::WARPS * 32, P::SMEM, s>>>(a.in[0], a.X, a.info, a.batch, mode);
  return cudaGetLastError();
}

// mode = k-split (bits 0-1) | work split (bits 2-3); LAGEN_ROWS_MODE /
// LAGEN_ROWS_WG override the measured per-size defaults (tuning runs only)
template <int N, int B>
cudaError_t launch_rows(const LaunchArgs& a, cudaStream_t s) {
  static const int mode = [] {
    const char* e = std::getenv("LAGEN_ROWS_MODE");
    return e ? std::atoi(e) : cr::default_mode(N, B);
  }();
  static const int wg = [] {
    const char* e = std::getenv("LAGEN_ROWS_WG");
    return e ? std::atoi(e) : cr::rows_wg(N, B);
  }();
  if (wg == 1) return launch_rows_wg<N, B, 1>(a, s, mode);
  if (wg == 2) return launch_rows_wg<N, B, 2>(a, s, mode);
  return launch_rows_wg<N, B, 4>(a, s, mode);
}

// n = 4 (mod 8): the b = 8 kernel of size n + 4 on the identity-padded
// problem (diag(A, I) = diag(X, I)^T diag(X, I), exact), reading and writing
// only the real n x n entries — the b = 8 schedule is the faster one
// (half the iterations of b = 4) at every measured size
template <int NR, int N = NR + 4>
cudaError_t launch_rows_pad(const LaunchArgs& a, cudaStream_t s) {
  static_assert(N > NR && N % 8 == 0 && NR % 4 == 0, "padding to a multiple of 8");
  static const int mode = [] {
    const char* e = std::getenv("LAGEN_ROWS_MODE");
    return e ? std::atoi(e) : cr::pad_mode(NR);
  }();
  static const int wg = [] {
    const char* e = std::getenv("LAGEN_ROWS_WG");
    return e ? std::atoi(e) : cr::pad_wg(NR);
  }();
  if (wg == 1) return launch_rows_wg<N, 8, 1, NR>(a, s, mode);
  if (wg == 2) return launch_rows_wg<N, 8, 2, NR>(a, s, mode);
  return launch_rows_wg<N, 8, 4, NR>(a, s, mode);
}

// n = 4 (mod 8), mixed blocks: a first 4 x 4 block row, then the b = 8
// schedule (chol_rows.cuh, F4) — no padding, the problem's own footprint
template <int N>
cudaError_t launch_rows_mix(const LaunchArgs& a, cudaStream_t s) {
  static const int mode = [] {
    const char* e = std::getenv("LAGEN_ROWS_MODE");
    return e ? std::atoi(e) : cr::mix_mode(N);
  }();
  static const int wg = [] {
    const char* e = std::getenv("LAGEN_ROWS_WG");
    return e ? std::atoi(e) : cr::mix_wg(N);
  }();
  if (wg == 1) return launch_rows_wg<N, 8, 1, N, true>(a, s, mode);
  if (wg == 2) return launch_rows_wg<N, 8, 2, N, true>(a, s, mode);
  return launch_rows_wg<N, 8, 4, N, true>(a, s, mode);
}

#define LAGEN_ROWS_MIX_ENTRY(N) \
  { N, 4, 1, (int)cr::RPolicy<N, 2>::SMEM, &launch_rows_mix<N> }

#define LAGEN_ROWS_PAD_ENTRY(NR, NP) \
  { NR, 4, 1, (int)cr::RPolicy<NP, 2>::SMEM, &launch_rows_pad<NR, NP> }

#define LAGEN_ROWS_ENTRY(N, B) \
  { N, B, 1, (int)cr::RPolicy<N, 2>::SMEM, &launch_rows<N, B> }

}  // namespace lagen
