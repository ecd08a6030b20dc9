// Probe: H2D / D2H of the upper triangle of a batch of row-major n x n fp64
// matrices as K row bands (one cudaMemcpy3DAsync per band), vs full copies.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
static double run(int n, long long batch, int K, bool h2d, double* h, double* d, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int rep = 0; rep < 3; ++rep) {
    if (K == 0) {
      size_t bytes = (size_t)batch * n * n * 8;
      cudaMemcpyAsync(h2d ? (void*)d : (void*)h, h2d ? (void*)h : (void*)d, bytes, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s);
    } else {
      for (int j = 0; j < K; ++j) {
        int r0 = j * n / K, r1 = (j + 1) * n / K;
        int c0 = r0 & ~1;
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr(h2d ? (void*)h : (void*)d, (size_t)n * 8, (size_t)n, (size_t)n);
        p.dstPtr = make_cudaPitchedPtr(h2d ? (void*)d : (void*)h, (size_t)n * 8, (size_t)n, (size_t)n);
        p.srcPos = make_cudaPos((size_t)c0 * 8, r0, 0);
        p.dstPos = make_cudaPos((size_t)c0 * 8, r0, 0);
        p.extent = make_cudaExtent((size_t)(n - c0) * 8, r1 - r0, batch);
        p.kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
        cudaError_t e = cudaMemcpy3DAsync(&p, s);
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return -1; }
      }
    }
  }
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 3;
}
int main() {
  for (int n : {16, 32, 64, 128}) {
    long long batch = (1ll << 28) / (8ll * n * n);
    size_t bytes = (size_t)batch * n * n * 8;
    double *h, *d;
    cudaHostAlloc(&h, bytes, 0); cudaMalloc(&d, bytes);
    cudaStream_t s; cudaStreamCreate(&s);
    for (int dir = 0; dir < 2; ++dir)
      for (int K : {0, 2, 4, 8}) {
        double ms = run(n, batch, K, dir == 0, h, d, s);
        double frac = 0;
        if (K) for (int j = 0; j < K; ++j) { int r0 = j * n / K, r1 = (j + 1) * n / K; frac += (double)(r1 - r0) * (n - (r0 & ~1)) / ((double)n * n); }
        else frac = 1;
        printf("n=%d %s K=%d: %.3f ms  (bytes frac %.3f, eff %.1f GB/s, full-equiv %.1f GB/s)\n", n, dir == 0 ? "H2D" : "D2H", K, ms, frac, frac * bytes / ms / 1e6, bytes / ms / 1e6);
      }
    cudaFreeHost(h); cudaFree(d);
  }
}
