// Dependent-chain latencies on B200 (cycles per iteration, one warp):
// the building blocks of the wavefront / substitution steps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/chain_lat tools/chain_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void chain(double* out, long long* cyc, int iters, double a, double b) {
  double x = a + threadIdx.x;
  const int src = (threadIdx.x + 31) & 31;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) x = fma(x, a, b);                                         // DFMA
    if (MODE == 1) x = __shfl_sync(0xffffffffu, x, src);                      // SHFL (double = 2)
    if (MODE == 2) x = fma(__shfl_sync(0xffffffffu, x * a, src), b, x);       // DMUL -> SHFL -> DFMA
    if (MODE == 3) { x = x * a; x = fma(x, b, a); }                           // DMUL -> DFMA
    if (MODE == 4) x = __int_as_float(__shfl_sync(0xffffffffu, __float_as_int((float)x), src)); // 32-bit SHFL
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 8);
  const char* names[] = {"dfma", "shfl_f64", "dmul_shfl_dfma", "dmul_dfma", "shfl_b32"};
  const int iters = 4096;
  for (int m = 0; m < 5; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (m) {
        case 0: chain<0><<<1, 32>>>(d, c, iters, 1.0000001, 1e-9); break;
        case 1: chain<1><<<1, 32>>>(d, c, iters, 1.0000001, 1e-9); break;
        case 2: chain<2><<<1, 32>>>(d, c, iters, 1.0000001, 1e-9); break;
        case 3: chain<3><<<1, 32>>>(d, c, iters, 1.0000001, 1e-9); break;
        case 4: chain<4><<<1, 32>>>(d, c, iters, 1.0000001, 1e-9); break;
      }
    }
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-16s %.1f cycles/iter\n", names[m], (double)h / iters);
  }
  return 0;
}
