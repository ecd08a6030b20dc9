// Standalone timing + residual check of one rows-engine (Cholesky v1) instance
// (development aid; the product path is the library):
//   nvcc ... -DPN=48 -DPB=8 -DPWG=1 -DPF4=0 [-DLAGEN_ROWS_MAXW=24] tools/experiments/rows_bench.cu
// A = n I + symmetric noise in [-1, 1] (SPD by diagonal dominance); checks
// ||X^T X - A||_F / ||A||_F on a sample of problems and info == 0.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "chol_rows.cuh"

#ifndef PF4
#define PF4 0
#endif
#ifndef PMODE
#define PMODE 1
#endif

__device__ __forceinline__ double hash01(unsigned long long h) {
  h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
  return (double)(h >> 11) / 9007199254740992.0;
}
__global__ void gen(double* M, long long batch, int n) {
  const long long total = batch * n * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / (n * n);
    int r = (int)((i / n) % n), c = (int)(i % n);
    if (r > c) { const int t = r; r = c; c = t; }
    const double u = hash01((unsigned long long)p * 1000003ull + r * 131ull + c * 7919ull + 5);
    M[i] = r == c ? n + u : 2.0 * u - 1.0;
  }
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

int main(int argc, char** argv) {
  constexpr int N = PN, B = PB, WG = PWG;
  using P = lagen::cr::RPolicy<N, WG>;
  const long long batch = (argc > 1 && atoll(argv[1]) > 0) ? atoll(argv[1]) : (1ll << 28) / (8ll * N * N);
  const int mode = argc > 2 ? atoi(argv[2]) : PMODE;
  const size_t bytes = (size_t)batch * N * N * 8;
  double *A, *X;
  int* info;
  CK(cudaMalloc(&A, bytes));
  CK(cudaMalloc(&X, bytes));
  CK(cudaMalloc(&info, batch * 4));
  gen<<<1184, 256>>>(A, batch, N);
  CK(cudaMemset(X, 0xff, bytes));
  auto kern = lagen::cr::chol_rows_kernel<N, B, WG, N, PF4 != 0>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
  int occ = 0, sms = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, P::WARPS * 32, P::SMEM));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long need = (batch + P::P - 1) / P::P;
  const long long grid = need < (long long)occ * sms ? need : (long long)occ * sms;
  printf("n=%d b=%d wg=%d f4=%d mode=%d P=%d warps=%d smem=%zu occ=%d grid=%lld batch=%lld\n", N, B, WG, PF4, mode, P::P, P::WARPS,
         P::SMEM, occ, grid, batch);
  if (occ < 1) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int i = 0; i < 7; ++i) {
    cudaEventRecord(e0);
    kern<<<(unsigned)grid, P::WARPS * 32, P::SMEM>>>(A, X, info, batch, mode);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (i >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  const double byt = (12.0 * N * N + 4.0 * N) * batch;
  printf("time %.4f ms  GB/s = %.1f  roofline frac = %.3f\n", best, byt / best / 1e6, byt / 6553e9 * 1e3 / best);
#ifdef LAGEN_ROWS_PROF
  {
    unsigned long long hp[16];
    CK(cudaMemcpyFromSymbol(hp, lagen::cr::prof_buf, sizeof(hp)));
    const double runs = 7.0;  // kernel launches above
    printf("phase cycles per launch (CTA 0, group 0): leaf warp A=%.0f barrier=%.0f trsm=%.0f barrier=%.0f | panel warp A=%.0f barrier=%.0f trsm=%.0f barrier=%.0f\n",
           hp[0] / runs, hp[1] / runs, hp[2] / runs, hp[3] / runs, hp[8] / runs, hp[9] / runs, hp[10] / runs, hp[11] / runs);
  }
#endif
  std::vector<long long> sample;
  for (long long p = 0; p < batch && p < 4; ++p) sample.push_back(p);
  for (long long p = batch > 4 ? batch - 4 : 0; p < batch; ++p) sample.push_back(p);
  for (int i = 0; i < 8; ++i) sample.push_back((long long)((i * 2654435761ull) % (unsigned long long)batch));
  std::vector<double> hA(N * N), hX(N * N);
  double worst = 0.0;
  for (long long p : sample) {
    CK(cudaMemcpy(hA.data(), A + p * N * N, N * N * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hX.data(), X + p * N * N, N * N * 8, cudaMemcpyDeviceToHost));
    double num = 0, den = 0;
    for (int r = 0; r < N; ++r)
      for (int c = 0; c < N; ++c) {
        double acc = 0;
        for (int k = 0; k < N; ++k) acc += hX[k * N + r] * hX[k * N + c];
        const double d = acc - hA[r * N + c];
        num += d * d;
        den += hA[r * N + c] * hA[r * N + c];
        if (!(hX[r * N + c] == hX[r * N + c]) || (r > c && hX[r * N + c] != 0.0)) num = 1e300;
      }
    const double e = std::sqrt(num / den);
    if (e > worst) worst = e;
  }
  std::vector<int> hinfo(batch);
  CK(cudaMemcpy(hinfo.data(), info, batch * 4, cudaMemcpyDeviceToHost));
  long long nbad = 0;
  for (long long p = 0; p < batch; ++p) nbad += hinfo[p] != 0;
  const double tol = 10.0 * N * 2.2e-16;
  printf("max residual on %zu problems: %.3e (tol %.1e); info != 0: %lld  %s\n", sample.size(), worst, tol, nbad,
         (worst <= tol && nbad == 0) ? "OK" : "FAIL");
  return (worst <= tol && nbad == 0) ? 0 : 2;
}
