// Standalone check + timing + per-step clocks of one pipe-engine instance
// (development aid; the product path is the library):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -DPEQ=2 -DPN=64 -DPMODE=0 \
//        -Iinclude -Ipaper_1906_08613_b200/csrc tools/experiments/pipe_bench.cu -o tools/experiments/pipe_bin/p_2_64
// Inputs: L lower / U upper triangular with diagonal in [1, 2] and off-diagonal
// entries in [-1, 1] / n, dense right-hand side in [-1, 1] (symmetric for
// Lyapunov); the result is checked by the residual of a sample of problems.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pipe.cuh"

#ifndef PMODE
#define PMODE 0
#endif

__device__ __forceinline__ double hash01(unsigned long long h) {
  h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
  return (double)(h >> 11) / 9007199254740992.0;
}

// kind 0: lower triangular, 1: upper triangular, 2: dense, 3: symmetric
__global__ void gen(double* M, long long batch, int n, int kind, unsigned long long salt) {
  const long long total = batch * n * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / (n * n);
    int r = (int)((i / n) % n), c = (int)(i % n);
    if (kind == 3 && r > c) { const int t = r; r = c; c = t; }
    const double u = hash01((unsigned long long)p * 1000003ull + r * 131ull + c * 7919ull + salt);
    double v;
    if (kind <= 1) {
      const bool keep = kind == 0 ? c <= r : c >= r;
      v = r == c ? 1.0 + u : (keep ? (2.0 * u - 1.0) / n : 0.0);
    } else {
      v = 2.0 * u - 1.0;
    }
    M[i] = v;
  }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

int main(int argc, char** argv) {
  constexpr int EQ = PEQ, N = PN;
  using P = lagen::pipe::PCfg<EQ, N, PMODE>;
  const long long batch = argc > 1 ? atoll(argv[1]) : (1ll << 28) / (8ll * N * N);
  const int reps = 5;
  const size_t bytes = (size_t)batch * N * N * 8;
  double *L, *U, *C, *X;
  int* info;
  unsigned long long* prof;
  CK(cudaMalloc(&L, bytes));
  CK(cudaMalloc(&U, bytes));
  CK(cudaMalloc(&C, bytes));
  CK(cudaMalloc(&X, bytes));
  CK(cudaMalloc(&info, batch * 4));
  CK(cudaMalloc(&prof, 512 * 8));
  gen<<<1184, 256>>>(L, batch, N, 0, 11);
  gen<<<1184, 256>>>(U, batch, N, 1, 23);
  gen<<<1184, 256>>>(C, batch, N, EQ == 1 ? 3 : 2, 37);
  CK(cudaMemset(X, 0xff, bytes));
  CK(cudaMemset(prof, 0, 512 * 8));
  auto kern = lagen::pipe::pipe_kernel<EQ, N, PMODE>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM));
  int occ = 0, sms = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, P::THREADS, P::SMEM));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long need = (batch + P::PP - 1) / P::PP;
  const long long grid = need < (long long)occ * sms ? need : (long long)occ * sms;
  printf("eq=%d n=%d mode=%d threads=%d (NU=%d NS=%d) smem=%zu occ=%d grid=%lld batch=%lld\n", EQ, N, PMODE, P::THREADS, P::NU,
         P::NS, P::SMEM, occ, grid, batch);
  if (occ < 1) return 1;
  const double* Uarg = EQ == 2 ? U : L;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int i = 0; i < reps + 2; ++i) {
    cudaEventRecord(e0);
    kern<<<(unsigned)grid, P::THREADS, P::SMEM>>>(L, Uarg, C, X, info, batch, i == reps + 1 ? prof : nullptr);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (i >= 2 && i <= reps && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  const double flops = 2.0 * N * N * N * batch;
  const double byt = (EQ == 2 ? 24.0 * N * N + 8.0 * N : 16.0 * N * N + 8.0 * N) * batch;
  const double falg = (EQ == 2 ? 2.0 * N * N * N : (double)N * N * (N + 1)) * batch;
  const double troof = fmax(byt / 6553e9, falg / 37.1e12);
  printf("time %.4f ms  gflops(2n^3) = %.1f  roofline frac = %.3f\n", best, flops / best / 1e6, troof * 1e3 / best);
  {
    unsigned long long hp[512];
    CK(cudaMemcpy(hp, prof, sizeof(hp), cudaMemcpyDeviceToHost));
    constexpr int T = (N + 7) / 8;
    double sw = 0, ss = 0, so = 0, su = 0;
    int cnt = 0;
    for (int d = 0; d < 2 * T - 1; ++d) {
      const unsigned long long* s = hp + 4 * (d + 1);
      const unsigned long long* u = hp + 256 + 2 * (d + 1);
      if (s[0] && s[1] && s[2] && s[3]) { sw += s[1] - s[0]; ss += s[2] - s[1]; so += s[3] - s[2]; ++cnt; }
      if (u[0] && u[1]) su += u[1] - u[0];
    }
    const unsigned long long* s0 = hp + 4, *sl = hp + 4 * (2 * T - 1);
    if (cnt)
      printf("steps=%d per step: wait=%.0f solve=%.0f out=%.0f | upd=%.0f | problem=%.0f cycles\n", 2 * T - 1, sw / cnt, ss / cnt,
             so / cnt, su / (2 * T - 1), (double)(sl[3] - s0[0]));
    else
      printf("steps=%d (no per-step clocks: built without LAGEN_PIPE_PROF)\n", 2 * T - 1);
  }
  // residual of a sample
  std::vector<long long> sample;
  for (long long p = 0; p < batch && p < 4; ++p) sample.push_back(p);
  for (long long p = batch > 4 ? batch - 4 : 0; p < batch; ++p) sample.push_back(p);
  for (int i = 0; i < 8; ++i) sample.push_back((long long)((i * 2654435761ull) % (unsigned long long)batch));
  std::vector<double> hL(N * N), hU(N * N), hC(N * N), hX(N * N);
  double worst = 0.0;
  for (long long p : sample) {
    CK(cudaMemcpy(hL.data(), L + p * N * N, N * N * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hU.data(), U + p * N * N, N * N * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hC.data(), C + p * N * N, N * N * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hX.data(), X + p * N * N, N * N * 8, cudaMemcpyDeviceToHost));
    double num = 0, den = 0;
    for (int r = 0; r < N; ++r)
      for (int c = 0; c < N; ++c) {
        double acc = 0;
        for (int k = 0; k < N; ++k) {
          acc += hL[r * N + k] * hX[k * N + c];
          acc += hX[r * N + k] * (EQ == 2 ? hU[k * N + c] : hL[c * N + k]);
        }
        const double d = acc - hC[r * N + c];
        num += d * d;
        den += hC[r * N + c] * hC[r * N + c];
        if (!(hX[r * N + c] == hX[r * N + c])) num = 1e300;
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
