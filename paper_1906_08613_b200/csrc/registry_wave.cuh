// registry_wave.cuh — wave-engine instances (Sylvester v13 / Lyapunov v5
// semantics, 8x8 tiles; see wave.cuh).  Geometry per size: NW warps per
// problem and PP problems per CTA (WCfg, overridable for tuning runs with
// LAGEN_WAVE_NW / LAGEN_WAVE_PP among the instantiated alternatives).
#pragma once
#include <atomic>
#include <cstdlib>

#include "registry.cuh"
#include "wave.cuh"

// Registers per thread beside the accumulators in the geometry model: sets
// how many problems share a CTA (PP) and so the register cap per thread.
// 136 is spill-free for most sizes; where the solve spilled its lane /
// address state to local memory at that cap, fewer problems per CTA with a
// spill-free register budget measured faster (A/B over the sweep sizes,
// profiles/r01_wave_geometry.md) — keyed by the tile count T = ceil(n / 8),
// which fixes the geometry.  LAGEN_WAVE_REGBASE forces one value (tuning).
#ifndef LAGEN_WAVE_REGBASE
#define LAGEN_WAVE_REGBASE 0
#endif
constexpr int wave_regbase(int eq, int t) {
  if (LAGEN_WAVE_REGBASE) return LAGEN_WAVE_REGBASE;
  if (eq == 2) return (t == 4 || t == 5) ? 170 : 136;                                   // Sylvester
  return t == 4 ? 200 : (t == 6 || t == 7 || t == 10 || t == 11) ? 170 : 136;           // Lyapunov
}

namespace lagen {

struct WaveEntry {
  int eq, n;
  int smem;
  LaunchFn launch;
};

// default geometry: enough warps that a diagonal spreads over <= 4 groups per
// warp and <= ~32 accumulator tiles per warp; then as many problems per CTA as
// registers (~4 S + 136 per thread, spill-free at that cap) and shared memory allow
template <int EQ, int N>
struct WCfg {
  static constexpr int T = (N + 7) / 8;
  static constexpr int NT = EQ == 2 ? T * T : T * (T + 1) / 2;
  static constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  static constexpr int mn(int a, int b) { return a < b ? a : b; }
  // measured: ~136 registers per thread beside the accumulators (spill-free)
  static constexpr int regs(int nw) { return mn(255, 4 * cdiv(NT, nw) + wave_regbase(EQ, T)); }
  static constexpr int slotb(int nw) {
    return 8 * (T * (T + 1) / 2 * (EQ == 2 ? 2 : 1) * 64 + 2 * T * 68 + T * 80 + nw * 4 * 72 + 2);
  }
  static constexpr int pp(int nw) {
    return mx(1, mn(mn(65536 / (regs(nw) * 32 * nw), (227 * 1024) / slotb(nw)), mn(32 / nw, nw == 1 ? 32 : 15)));
  }
  // enough warps that a diagonal spreads over <= 4 groups per warp and
  // <= ~32 accumulator tiles per warp; then, while fewer than 8 warps per SM
  // are resident, one more warp per problem (more solves in parallel, more
  // latency hidden) as long as the registers allow
  static constexpr int nw_pick() {
    int nw = mx(mx(cdiv(T, 4), cdiv(NT, 32)), 1);
    while (pp(nw) * nw < 8 && nw < T && regs(nw + 1) * 32 * (nw + 1) <= 65536) ++nw;
    return nw;
  }
  static constexpr int NW = nw_pick();
  static constexpr int S = wave::WPol<EQ, N, NW, 1>::S;
  static constexpr int PP = pp(NW);
  static_assert(slotb(NW) == (int)(wave::WPol<EQ, N, NW, 1>::SLOT * 8), "slot size model");
};

template <int EQ, int N, int NW, int PP>
cudaError_t launch_wave_cfg(const LaunchArgs& a, cudaStream_t s) {
  using P = wave::WPol<EQ, N, NW, PP>;
  static std::atomic<unsigned long long> configured{0};
  static std::atomic<int> ctas_per_sm{0};
  static std::atomic<int> sm_count{0};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  const unsigned long long bit = 1ull << (dev & 63);
  auto kern = wave::wave_kernel<EQ, N, NW, PP>;
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
  const long long need = (a.batch + PP - 1) / PP;
  const long long resident = (long long)ctas_per_sm.load() * sm_budget(sm_count.load());
  const long long grid = need < resident ? need : resident;
  // _signature order: lyapunov (L, S), sylvester (L, U, C)
  const double* L = a.in[0];
  const double* U = EQ == 2 ? a.in[1] : a.in[0];
  const double* C = EQ == 2 ? a.in[2] : a.in[1];
  static const int mode = [] {
    const char* e = std::getenv("LAGEN_WAVE_MODE");  // profiling switch, see wave_kernel
    return e ? std::atoi(e) : 0;
  }();
  kern<<<(unsigned)grid, P::THREADS, P::SMEM, s>>>(L, U, C, a.X, a.info, a.batch, mode);
  return cudaGetLastError();
}

template <int EQ, int N>
cudaError_t launch_wave(const LaunchArgs& a, cudaStream_t s) {
  using C = WCfg<EQ, N>;
  return launch_wave_cfg<EQ, N, C::NW, C::PP>(a, s);
}

#define LAGEN_WAVE_ENTRY(EQ, N) \
  { EQ, N, (int)wave::WPol<EQ, N, WCfg<EQ, N>::NW, WCfg<EQ, N>::PP>::SMEM, &launch_wave<EQ, N> }

struct WaveTable {
  const WaveEntry* e;
  const int* n;
};

}  // namespace lagen
