// Standalone check + timing of one gang-engine instance (development aid):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -DGN=128 -DGNR=128 -DGP=3 -DGQ=3 -DGMINB=1 \
//        -Ipaper_1906_08613_b200/csrc tools/gang_bench.cu -o tools/gang_bench_128
//   ./tools/gang_bench_128 [batch]
// Inputs: symmetric diagonally dominant matrices (SPD); the result is compared
// with a plain CPU upper Cholesky on a sample of problems.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "chol_gang.cuh"

#ifndef GNR
#define GNR GN
#endif
#ifndef GMINB
#define GMINB 1
#endif

__global__ void gen(double* A, long long batch, int n) {
  const long long total = batch * n * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / (n * n);
    const int r = (int)((i / n) % n), c = (int)(i % n);
    const int lo = r < c ? r : c, hi = r < c ? c : r;
    unsigned long long h = (unsigned long long)p * 1000003ull + lo * 131ull + hi * 7919ull + 12345ull;
    h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
    const double u = (double)(h >> 11) / 9007199254740992.0 * 2.0 - 1.0;
    A[i] = r == c ? 2.0 * n + u : u;
  }
}

static void cpu_chol(const double* A, double* X, int n) {
  std::vector<double> t(A, A + n * n);
  for (int i = 0; i < n * n; ++i) X[i] = 0.0;
  for (int i = 0; i < n; ++i) {
    const double d = std::sqrt(t[i * n + i]);
    X[i * n + i] = d;
    for (int c = i + 1; c < n; ++c) X[i * n + c] = t[i * n + c] / d;
    for (int r = i + 1; r < n; ++r)
      for (int c = r; c < n; ++c) t[r * n + c] -= X[i * n + r] * X[i * n + c];
  }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

int main(int argc, char** argv) {
  constexpr int N = GN, NR = GNR;
  using C = lagen::gang::GCfg<N, GP, GQ, GMINB>;
  const long long batch = argc > 1 ? atoll(argv[1]) : (1ll << 28) / (8ll * NR * NR);
  const int reps = argc > 2 ? atoi(argv[2]) : 5;
  double *A, *X;
  int* info;
  const size_t bytes = (size_t)batch * NR * NR * 8;
  CK(cudaMalloc(&A, bytes));
  CK(cudaMalloc(&X, bytes));
  CK(cudaMalloc(&info, batch * 4));
  gen<<<1184, 256>>>(A, batch, NR);
  CK(cudaMemset(X, 0xff, bytes));
  auto kern = lagen::gang::chol_gang_kernel<N, NR, GP, GQ, GMINB>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long need = (batch + GP - 1) / GP;
  const long long grid = need < (long long)occ * sms ? need : (long long)occ * sms;
  printf("n=%d nr=%d P=%d Q=%d threads=%d smem=%zu occ=%d grid=%lld batch=%lld\n", N, NR, GP, GQ, C::THREADS, C::SMEM, occ, grid, batch);
  if (occ < 1) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int i = 0; i < reps + 2; ++i) {
    cudaEventRecord(e0);
    kern<<<(unsigned)grid, C::THREADS, C::SMEM>>>(A, X, info, batch);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (i >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  const double byt = (12.0 * NR * NR + 4.0 * NR) * batch;
  printf("time %.4f ms  %.1f GB/s (algorithmic)  frac of 6553 = %.3f  gflops(n^3/3) = %.1f\n", best, byt / best / 1e6,
         byt / best / 1e6 / 6553.0, (double)NR * NR * NR / 3.0 * batch / best / 1e6);
#ifdef GANG_PROF
  {
    unsigned long long hp[64];
    CK(cudaMemcpyFromSymbol(hp, lagen::gang::gang_prof, sizeof(hp)));
    const double r = reps + 2;
    const char* names[3][8] = {{"load_issue", "wait_row", "T1", "T3_leaf", "bar_wait", "tail", "-", "-"},
                               {"load_issue", "B1_trsm", "wait_panel", "B3_bulk", "bar_wait", "tail", "barwait+stores", "wait_row"},
                               {"load_issue", "wait_row", "T1", "T3_leaf", "bar_wait", "tail", "-", "-"}};
    const char* who[3] = {"leaf warp 0", "bulk warp 1", "panel warp 4"};
    for (int w = 0; w < 3; ++w) {
      printf("%s:", who[w]);
      for (int i = 0; i < 8; ++i) printf(" %s=%.0f", names[w][i], hp[16 * w + i] / r);
      printf("\n");
    }
  }
#endif
  // verify a sample
  std::vector<long long> sample;
  for (long long p = 0; p < batch && p < 6; ++p) sample.push_back(p);
  for (long long p = batch > 6 ? batch - 6 : 0; p < batch; ++p) sample.push_back(p);
  for (int i = 0; i < 20; ++i) sample.push_back((long long)((i * 2654435761ull) % (unsigned long long)batch));
  std::vector<double> hA(NR * NR), hX(NR * NR), ref(NR * NR);
  double worst = 0.0;
  int badinfo = 0;
  for (long long p : sample) {
    CK(cudaMemcpy(hA.data(), A + p * NR * NR, NR * NR * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hX.data(), X + p * NR * NR, NR * NR * 8, cudaMemcpyDeviceToHost));
    int hi;
    CK(cudaMemcpy(&hi, info + p, 4, cudaMemcpyDeviceToHost));
    badinfo += hi != 0;
    cpu_chol(hA.data(), ref.data(), NR);
    double num = 0, den = 0;
    for (int i = 0; i < NR * NR; ++i) {
      const double d = hX[i] - ref[i];
      num += d * d;
      den += ref[i] * ref[i];
      if (!(hX[i] == hX[i])) num = 1e300;
    }
    const double e = std::sqrt(num / den);
    if (e > worst) worst = e;
  }
  // info of all problems
  std::vector<int> hinfo(batch);
  CK(cudaMemcpy(hinfo.data(), info, batch * 4, cudaMemcpyDeviceToHost));
  long long nbad = 0;
  for (long long p = 0; p < batch; ++p) nbad += hinfo[p] != 0;
  printf("max rel diff vs CPU on %zu problems: %.3e; info != 0: %lld of %lld  %s\n", sample.size(), worst, nbad, batch,
         (worst < 1e-12 && nbad == 0) ? "OK" : "FAIL");
  return (worst < 1e-12 && nbad == 0) ? 0 : 2;
}
