// FP64 pipe microbenchmarks for B200 (sm_100a): DFMA vs DMMA (mma.sync m8n8k4 f64).
// Measures sustained FP64 rate with every SM busy; prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters, double a0, double b0) {
  double c[CHAINS][2];
  double a = a0 + threadIdx.x * 1e-12, b = b0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = k; c[k][1] = -k; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  float best_dfma = 0, best_dmma = 0;
  int best_dfma_cfg = 0, best_dmma_cfg = 0;
  int threads_list[] = {256, 512, 1024};
  for (int t : threads_list) {
    for (int blocksPerSm = 1; blocksPerSm <= 4; blocksPerSm *= 2) {
      if (t * blocksPerSm > 2048) continue;
      int grid = sms * blocksPerSm;
      dfma_kernel<8><<<grid, t>>>(out, 16, 1.0000001, 1e-7);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_kernel<8><<<grid, t>>>(out, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double tf = 2.0 * 8 * iters * (double)grid * t / (ms * 1e-3) / 1e12;
      if (tf > best_dfma) { best_dfma = tf; best_dfma_cfg = t * blocksPerSm; }
      dmma_kernel<4><<<grid, t>>>(out, 16, 1.0000001, 1e-7);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_kernel<4><<<grid, t>>>(out, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      // one m8n8k4 per warp = 256 FMA = 512 flop
      double tf2 = 512.0 * 4 * iters * (double)grid * (t / 32) / (ms * 1e-3) / 1e12;
      if (tf2 > best_dmma) { best_dmma = tf2; best_dmma_cfg = t * blocksPerSm; }
      fprintf(stderr, "threads/SM=%d dfma=%.2f TF/s dmma=%.2f TF/s\n", t * blocksPerSm, tf, tf2);
    }
  }
  printf("{\"sms\": %d, \"clock_mhz\": %d, \"dfma_tflops\": %.2f, \"dfma_threads_per_sm\": %d, "
         "\"dmma_tflops\": %.2f, \"dmma_threads_per_sm\": %d}\n",
         sms, clk / 1000, best_dfma, best_dfma_cfg, best_dmma, best_dmma_cfg);
  return 0;
}
