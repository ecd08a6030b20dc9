// Dependent-chain latencies on one warp (clock64): DMMA m8n8k4 f64, DFMA,
// rsqrt(double), LDS.64, and the cost of a 4-warp named barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(long long* out, double* buf, int iters) {
  __shared__ double sm[1024];
  __shared__ int idx[1024];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    sm[i] = 1.0 + 1e-9 * i;
    idx[i] = (i + 33) & 1023;
  }
  __syncthreads();
  double c0 = lane, c1 = 1.0, a = buf[lane], b = buf[lane + 32];
  long long t0, t1;
  if (threadIdx.x < 32) {
    t0 = clock64();
    for (int i = 0; i < iters; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    t1 = clock64();
    if (lane == 0) out[0] = (t1 - t0);
    double x = c0;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, a, b);
    t1 = clock64();
    if (lane == 0) out[1] = (t1 - t0);
    double y = 2.0 + c1;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) y = rsqrt(y) + 1.5;
    t1 = clock64();
    if (lane == 0) out[2] = (t1 - t0);
    int p = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) p = idx[p];
    t1 = clock64();
    if (lane == 0) out[3] = (t1 - t0);
    double z = 0.0;
    int q = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      z += sm[q];
      q = (q + (int)z) & 1023;
    }
    t1 = clock64();
    if (lane == 0) out[4] = (t1 - t0);
    buf[64 + lane] = c0 + c1 + x + y + p + z;
  }
  __syncthreads();
  // named barrier among 4 warps, back to back
  t0 = clock64();
  for (int i = 0; i < iters; ++i) asm volatile("bar.sync 1, 128;" ::: "memory");
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0);
}

int main() {
  long long* d;
  double* buf;
  cudaMalloc(&d, 64 * sizeof(long long));
  cudaMalloc(&buf, 256 * sizeof(double));
  cudaMemset(buf, 0, 256 * sizeof(double));
  const int iters = 4096;
  lat<<<1, 128>>>(d, buf, iters);
  lat<<<1, 128>>>(d, buf, iters);
  long long h[8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"dmma_m8n8k4_f64", "dfma", "rsqrt_f64_plus_add", "lds_int_chase", "lds_f64_dep_chain", "bar_sync_4warps"};
  printf("{");
  for (int i = 0; i < 6; ++i) printf("%s\"%s\": %.1f", i ? ", " : "", names[i], (double)h[i] / iters);
  printf("}\n");
  return 0;
}
