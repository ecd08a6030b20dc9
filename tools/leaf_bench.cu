// Latency of one 8x8 register CHOL leaf (chol_leaf_reg) on one warp.
#include <cstdio>
#include "engine.cuh"
using namespace lagen::eng;
__global__ void k(double* p, long long* cyc) {
  __shared__ double sm[2176 + 128];
  __shared__ double pristine[2176];
  TV<TM<16, UPPER>, false, false> v; v.base = sm; v.r0 = 8; v.c0 = 8;
  for (int i = threadIdx.x; i < 2176; i += 32) pristine[i] = p[i];
  __syncwarp();
  if (threadIdx.x < 8) {  // SPD block: strong diagonal
    TV<TM<16, UPPER>, false, false> pv; pv.base = pristine; pv.r0 = 8; pv.c0 = 8;
    pv.ref(threadIdx.x, threadIdx.x) = 50.0;
  }
  __syncwarp();
  long long acc = 0;
  for (int rep = 0; rep < 16; ++rep) {
    for (int i = threadIdx.x; i < 2176; i += 32) sm[i] = pristine[i];
    __syncwarp();
    int f = 0;
    long long t0 = clock64();
    chol_leaf_reg<8>(v, 8, &f, sm + 2176);
    __syncwarp();
    long long t1 = clock64();
    acc += t1 - t0;
  }
  if (threadIdx.x == 0) cyc[0] = acc / 16;
  for (int i = threadIdx.x; i < 2176; i += 32) p[i] = sm[i];
}
__global__ void krs(double* p, long long* cyc) {  // rsqrt dependent-chain latency
  double x = p[threadIdx.x] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < 64; ++i) x = rsqrt(x) + 1.0;
  long long t1 = clock64();
  p[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / 64;
  double y = p[threadIdx.x + 32];
  t0 = clock64();
  for (int i = 0; i < 64; ++i) y = fma(y, 1.0000001, 1e-9);
  t1 = clock64();
  p[threadIdx.x + 32] = y;
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / 64;
}
int main() {
  double* p; long long* c;
  cudaMalloc(&p, 8 * 8192); cudaMalloc(&c, 64);
  double h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = (i % 17 == 0) ? 50.0 : 0.01 * (i % 7);
  cudaMemcpy(p, h, sizeof(h), cudaMemcpyHostToDevice);
  k<<<1, 32>>>(p, c);
  krs<<<1, 32>>>(p, c);
  long long hc[3]; cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
  printf("leaf8 cycles %lld  rsqrt+add latency %lld  dfma latency %lld\n", hc[0], hc[1], hc[2]);
  return 0;
}
