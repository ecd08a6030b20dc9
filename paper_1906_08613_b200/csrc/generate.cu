// generate.cu — seeded, counter-based batched input generator for the
// BASELINE.json configs.  Every value is a pure function of
// (seed, eq, n, global problem index, operand, element, draw), so any
// sharding of the problem range over GPUs produces identical problems
// (SURVEY §8e).  Distributions (BASELINE.json configs 1-5):
//   cholesky : A = B^T B + n I,  B_ij ~ N(0,1)
//   lyapunov : L lower, diag ~ U[1,2], strict lower ~ N(0,1)/n;  S = (C + C^T)/2, C ~ N(0,1)
//   sylvester: L lower, U upper, diag ~ U[1,2], off-diagonal triangle ~ N(0,1)/n;  C ~ N(0,1)
// N(0,1) by Box-Muller from two splitmix64-finalised counters.  The CPU twin
// is oracle/lagen_oracle.c:oracle_generate (same formulas; libdevice vs glibc
// log/cos may differ in the last ulp).
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "lagen_b200.h"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t gen_key(uint64_t seed, int eq, int n) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ULL + ((uint64_t)eq << 40) + ((uint64_t)n << 20) + 0x632BE59BD9B4E019ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double gen_u01(uint64_t key, uint64_t ctr) {
  const uint64_t h = mix64(key + ctr * 0x9E3779B97F4A7C15ULL);
  return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ uint64_t gen_ctr(long long p, int op, int n, int e, int draw) {
  return (((uint64_t)p * 4u + (uint64_t)op) * (uint64_t)n * (uint64_t)n + (uint64_t)e) * 2u + (uint64_t)draw;
}
__device__ __forceinline__ double gen_normal(uint64_t key, long long p, int op, int n, int e) {
  const double u1 = gen_u01(key, gen_ctr(p, op, n, e, 0));
  const double u2 = gen_u01(key, gen_ctr(p, op, n, e, 1));
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
__device__ __forceinline__ double gen_tri(uint64_t key, long long p, int op, int n, int i, int j, bool lower) {
  const int e = i * n + j;
  if (i == j) return 1.0 + gen_u01(key, gen_ctr(p, op, n, e, 0));
  if ((lower && j < i) || (!lower && j > i)) return gen_normal(key, p, op, n, e) / (double)n;
  return 0.0;
}

// elementwise operands (lyapunov, sylvester): one thread per element
__global__ void gen_elementwise(int eq, int n, uint64_t key, long long first, long long batch, double* o0,
                                double* o1, double* o2) {
  const long long nn = (long long)n * n;
  const long long total = batch * nn;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long q = t / nn;
    const int e = (int)(t - q * nn);
    const int i = e / n, j = e - i * n;
    const long long p = first + q;
    if (eq == LAGEN_LYAPUNOV) {
      o0[t] = gen_tri(key, p, 0, n, i, j, true);
      const double cij = gen_normal(key, p, 1, n, i * n + j);
      const double cji = gen_normal(key, p, 1, n, j * n + i);
      o1[t] = 0.5 * (cij + cji);
    } else {
      o0[t] = gen_tri(key, p, 0, n, i, j, true);
      o1[t] = gen_tri(key, p, 1, n, i, j, false);
      o2[t] = gen_normal(key, p, 2, n, e);
    }
  }
}

// cholesky: one CTA per problem, B staged in shared memory, A = B^T B + n I
__global__ void gen_spd(int n, uint64_t key, long long first, long long batch, double* A) {
  extern __shared__ double Bs[];
  const long long nn = (long long)n * n;
  for (long long q = blockIdx.x; q < batch; q += gridDim.x) {
    const long long p = first + q;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) Bs[e] = gen_normal(key, p, 0, n, e);
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc = fma(Bs[k * n + i], Bs[k * n + j], acc);
      A[q * nn + e] = acc + (i == j ? (double)n : 0.0);
    }
    __syncthreads();
  }
}

}  // namespace

namespace lagen {
int set_error(int code, const std::string& msg);  // lagen_b200.cu
}
using lagen::set_error;

extern "C" int lagen_b200_generate(int eq, int n, unsigned long long seed, long long first, long long batch,
                                   double* const* outputs, void* stream) {
  if (eq < 0 || eq > 2) return set_error(LAGEN_EINVAL, "generate: unknown equation");
  if (n < 1 || n > 128) return set_error(LAGEN_EINVAL, "generate: n must be in 1..128");
  if (batch < 0 || first < 0) return set_error(LAGEN_EINVAL, "generate: negative batch or first index");
  if (!outputs) return set_error(LAGEN_EINVAL, "generate: null output array");
  for (int i = 0; i <= eq; ++i)
    if (!outputs[i]) return set_error(LAGEN_EINVAL, "generate: null output buffer");
  if (batch == 0) return LAGEN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t key = gen_key(seed, eq, n);
  if (eq == LAGEN_CHOLESKY) {
    const int smem = n * n * 8;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(gen_spd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return set_error(LAGEN_ECUDA, std::string("generate: ") + cudaGetErrorString(e));
    }
    long long grid = batch < 148 * 64 ? batch : 148 * 64;
    gen_spd<<<(unsigned)grid, 256, smem, s>>>(n, key, first, batch, outputs[0]);
  } else {
    const long long total = batch * (long long)n * n;
    long long grid = (total + 255) / 256;
    if (grid > 148 * 64) grid = 148 * 64;
    gen_elementwise<<<(unsigned)grid, 256, 0, s>>>(eq, n, key, first, batch, outputs[0], outputs[1],
                                                  eq == LAGEN_SYLVESTER ? outputs[2] : nullptr);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(LAGEN_ECUDA, std::string("generate launch: ") + cudaGetErrorString(e));
  return LAGEN_OK;
}
