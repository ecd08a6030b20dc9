// Zero-copy PCIe probe: kernels copying between mapped pinned host memory and
// device memory (16-byte units, warp per 1 KiB row), one direction or both
// at once, for several grid sizes; vs cudaMemcpyAsync.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zc_probe tools/zc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_k(const double2* __restrict__ s, double2* __restrict__ d, long long units, int unroll) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (unroll == 4) {
    for (; i + 3 * stride < units; i += 4 * stride) {
      double2 a = s[i], b = s[i + stride], c = s[i + 2 * stride], e = s[i + 3 * stride];
      d[i] = a; d[i + stride] = b; d[i + 2 * stride] = c; d[i + 3 * stride] = e;
    }
  }
  for (; i < units; i += stride) d[i] = s[i];
}

int main() {
  const size_t bytes = 512ull << 20;
  const long long units = bytes / 16;
  double2 *h1, *h2, *d1, *d2;
  cudaHostAlloc(&h1, bytes, cudaHostAllocMapped);
  cudaHostAlloc(&h2, bytes, cudaHostAllocMapped);
  cudaMalloc(&d1, bytes); cudaMalloc(&d2, bytes);
  cudaMemset(d1, 0, bytes); cudaMemset(d2, 0, bytes);
  double2 *mh1, *mh2;
  cudaHostGetDevicePointer(&mh1, h1, 0);
  cudaHostGetDevicePointer(&mh2, h2, 0);
  cudaStream_t s1, s2;
  cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  cudaEventRecord(a);
  cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1);
  cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2);
  cudaDeviceSynchronize();
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf("memcpy both ways: %.1f GB/s each\n", bytes / ms / 1e6);
  for (int unroll : {1, 4}) {
    for (int grid : {8, 16, 32, 64, 148, 296, 592}) {
      for (int mode = 0; mode < 3; ++mode) {
        cudaEventRecord(a);
        if (mode != 1) copy_k<<<grid, 512, 0, s1>>>(mh1, d1, units, unroll);   // H2D by loads
        if (mode != 0) copy_k<<<grid, 512, 0, s2>>>(d2, mh2, units, unroll);   // D2H by stores
        cudaDeviceSynchronize();
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        const char* nm[] = {"H2D loads ", "D2H stores", "both      "};
        printf("unroll %d grid %4d (x512 thr) %s %.1f GB/s each\n", unroll, grid, nm[mode], bytes / ms / 1e6);
      }
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
