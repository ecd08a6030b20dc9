// registry_df.cuh — dataflow-engine instances (right-looking variants, b <= 8)
// and the host-side schedule builder.
#pragma once
#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "dataflow.cuh"
#include "registry.cuh"
#include "variants_ct.cuh"

namespace lagen {

struct DfEntry {
  int eq, n, b, variant;
  int threads;
  int smem;
  LaunchFn launch;
};

namespace df {

// Simulates the variant in program order at 4x4-tile granularity
// (iteration k, statement, task; interpret_algorithm's order, verify.py:245-297)
// and records for every task the exact number of writes each X tile it
// touches has received before it.  Tasks are then ordered by DAG level
// (longest dependency chain from the start), which is a topological order,
// so a walk that claims records in that order cannot deadlock.  Returns
// false if the variant reads a tile that a later task rewrites (a
// write-after-read hazard the version scheme does not cover).
template <int EQ, int N, int B, class... S>
bool build_schedule(eng::Var<S...>, std::vector<int4>& out) {
  using E = EqT<EQ, N>;
  constexpr int NB = N / B, NT = N / 4;
  struct Rec {
    int k, si, idx, level, nd;
    int dep[6];
    int tile[6];
    bool rd[6];
  };
  std::vector<Rec> tasks;
  std::vector<int> cnt(NT * NT, 0), lvl(NT * NT, 0), lastw(NT * NT, -1);
  bool fits = true;
  for (int k = 0; k < NB; ++k) {
    int si = 0;
    auto one = [&](auto sI) {
      using St = typename decltype(sI)::type;
      const int c = task_count<E, N, B, St>(k);
      for (int idx = 0; idx < c; ++idx) {
        Touch t;
        task_tiles<E, N, B, St>(k, idx, t);
        if (t.n > 6) {
          fits = false;
          continue;
        }
        Rec r{};
        r.k = k;
        r.si = si;
        r.idx = idx;
        r.nd = t.n;
        int L = 0;
        for (int i = 0; i < t.n; ++i) {
          const int tile = t.r[i] * NT + t.c[i];
          r.tile[i] = tile;
          r.rd[i] = !t.w[i];
          r.dep[i] = (tile << 16) | cnt[tile];
          L = std::max(L, lvl[tile]);
        }
        r.level = L + 1;
        for (int i = 0; i < t.n; ++i)
          if (t.w[i]) {
            const int tile = r.tile[i];
            ++cnt[tile];
            lvl[tile] = r.level;
            lastw[tile] = (int)tasks.size();
          }
        tasks.push_back(r);
      }
      ++si;
    };
    (one(std::type_identity<S>{}), ...);
  }
  if (!fits) return false;
  for (size_t p = 0; p < tasks.size(); ++p)
    for (int i = 0; i < tasks[p].nd; ++i)
      if (tasks[p].rd[i] && lastw[tasks[p].tile[i]] > (int)p) return false;
  std::vector<int> order(tasks.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  // within a level, group by statement so a warp's 32 claims share a code path
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return tasks[a].level != tasks[b].level ? tasks[a].level < tasks[b].level : tasks[a].si < tasks[b].si;
  });
  out.clear();
  out.reserve(2 * tasks.size());
  for (int i : order) {
    const Rec& r = tasks[i];
    int d[6] = {0, 0, 0, 0, 0, 0};
    for (int j = 0; j < r.nd; ++j) d[j] = r.dep[j];
    out.push_back(make_int4(r.k | (r.si << 8) | (r.nd << 16), r.idx, d[0], d[1]));
    out.push_back(make_int4(d[2], d[3], d[4], d[5]));
  }
  return true;
}

}  // namespace df

template <int EQ, int N, int B, class VAR>
cudaError_t launch_df(const LaunchArgs& a, cudaStream_t s) {
  using P = df::DPolicy<EQ, N, B>;
  static std::mutex mu;
  static std::atomic<unsigned long long> configured{0};
  static int ctas_per_sm[64] = {}, sm_count[64] = {}, ntasks = -1;
  static int4* sched[64] = {};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  dev &= 63;
  const unsigned long long bit = 1ull << dev;
  auto kern = df::df_kernel<EQ, N, B, VAR>;
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    std::lock_guard<std::mutex> lock(mu);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
      std::vector<int4> host;
      if (!df::build_schedule<EQ, N, B>(VAR{}, host)) return cudaErrorNotSupported;
      err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
      if (err != cudaSuccess) return err;
      int occ = 0, sms = 0;
      err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, P::THREADS, P::SMEM);
      if (err != cudaSuccess) return err;
      err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (err != cudaSuccess) return err;
      // the schedule lives for the process (read-only, L2-resident across CTAs)
      err = cudaMalloc(&sched[dev], host.size() * sizeof(int4));
      if (err != cudaSuccess) return err;
      err = cudaMemcpy(sched[dev], host.data(), host.size() * sizeof(int4), cudaMemcpyHostToDevice);
      if (err != cudaSuccess) return err;
      ntasks = (int)(host.size() / 2);
      ctas_per_sm[dev] = occ > 0 ? occ : 1;
      sm_count[dev] = sms;
      configured.fetch_or(bit, std::memory_order_acq_rel);
    }
  }
  if (a.batch <= 0) return cudaSuccess;
  const long long resident = (long long)ctas_per_sm[dev] * sm_budget(sm_count[dev]);
  const long long grid = a.batch < resident ? a.batch : resident;
  kern<<<(unsigned)grid, P::THREADS, P::SMEM, s>>>(a.in[0], a.in[1], a.in[2], a.X, a.info, a.batch, sched[dev],
                                                   ntasks);
  return cudaGetLastError();
}

#define LAGEN_DF_ENTRY(EQ, N, B, VI, VAR) \
  { EQ, N, B, VI, df::DPolicy<EQ, N, B>::THREADS, (int)df::DPolicy<EQ, N, B>::SMEM, &launch_df<EQ, N, B, VAR> }

}  // namespace lagen
