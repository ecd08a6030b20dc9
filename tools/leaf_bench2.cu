// Break down the 8x8 register CHOL leaf: loads / factor chain / stores.
#include <cstdio>
__device__ __forceinline__ double my_rsqrt(double x) { return rsqrt(x); }
__global__ void k(const double* p, double* out, long long* cyc) {
  __shared__ double sm[512];
  for (int i = threadIdx.x; i < 512; i += 32) sm[i] = p[i];
  __syncwarp();
  long long c_load = 0, c_fac = 0, c_store = 0;
  for (int rep = 0; rep < 16; ++rep) {
    long long t0 = clock64();
    double t[8][8];
#pragma unroll
    for (int ch = 0; ch < 32; ++ch) {
      const double2 v = *reinterpret_cast<const double2*>(sm + ((ch * 2) ^ (rep & 6)));
      t[(ch >> 2) & 7][2 * (ch & 3)] = v.x;
      t[(ch >> 2) & 7][2 * (ch & 3) + 1] = v.y;
    }
    for (int i = 0; i < 8; ++i) t[i][i] += 20.0;
    long long t1 = clock64();
    double rs[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double piv = t[i][i];
      rs[i] = my_rsqrt(piv);
      t[i][i] = piv * rs[i];
#pragma unroll
      for (int c = i + 1; c < 8; ++c) t[i][c] *= rs[i];
#pragma unroll
      for (int r = i + 1; r < 8; ++r)
#pragma unroll
        for (int c = r; c < 8; ++c) t[r][c] = fma(-t[i][r], t[i][c], t[r][c]);
    }
    long long t2 = clock64();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int r = 0; r <= c; ++r) { sm[256 + r * 8 + c] = t[r][c]; sm[320 + r * 8 + c] = t[r][c]; }
#pragma unroll
      for (int c = 0; c < 8; ++c) sm[400 + c] = rs[c];
    }
    __syncwarp();
    long long t3 = clock64();
    c_load += t1 - t0; c_fac += t2 - t1; c_store += t3 - t2;
  }
  if (threadIdx.x == 0) { cyc[0] = c_load / 16; cyc[1] = c_fac / 16; cyc[2] = c_store / 16; }
  for (int i = threadIdx.x; i < 512; i += 32) out[i] = sm[i];
}
int main() {
  double *p, *o; long long* c;
  cudaMalloc(&p, 8 * 512); cudaMalloc(&o, 8 * 512); cudaMalloc(&c, 64);
  double h[512]; for (int i = 0; i < 512; ++i) h[i] = 0.01 * (i % 13);
  cudaMemcpy(p, h, sizeof(h), cudaMemcpyHostToDevice);
  k<<<1, 32>>>(p, o, c);
  long long hc[3]; cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
  printf("loads %lld  factor %lld  stores %lld cycles\n", hc[0], hc[1], hc[2]);
  return 0;
}
