// bigsolve.cu — the "big" engine: any statement list at sizes beyond the
// shared-memory engines (128 < n <= LAGEN_BIG_MAX_N), X resident in its HBM
// output buffer.
//
// The reference generator stops at n = 128 (PAPER.md:155-156 limitation (2),
// ref:pkg/src/lagen/lowering.py:930-932); its interpreter does not
// (ref:pkg/src/lagen/verify.py:221-303 works at any n with b | n).  This
// engine is that interpreter on the GPU for one problem per CTA: the
// statement list runs iteration by iteration on the 3x3 repartition with the
// block kernels of ref:pkg/src/lagen/kernels.py applied to views of global
// memory (row stride n):
//   GEMM_update          kernels.py:16-34   thread or warp per output element
//                        (upper target on the diagonal blocks of a symmetric
//                        right-hand side)
//   CHOL                 kernels.py:79-97   right-looking, one barrier pair per pivot
//   TRSM_left_transposed kernels.py:47-60   thread per column
//   SYLV                 kernels.py:100-110 anti-diagonal wavefront, warp per
//                        element, lanes split the two dot products
//   LYAP                 kernels.py:113-130 the same on the upper triangle, mirrored
// plus the symmetric gather of a symmetric unknown's diagonal blocks
// (verify.py:254-261), copy-in restricted to X's structure (verify.py:236-241),
// mirror_lower and the NaN / Inf guard (verify.py:299-302).  It is a
// correctness path (latency-bound, no shared-memory staging), not a tuned one;
// DESIGN.md states its measured rate.
#include <cuda_runtime.h>

#include "lagen_b200.h"
#include "registry.cuh"

namespace lagen {
namespace big {

struct View {
  double* p;
  long long rs, cs;
  int rows, cols;
  bool sym;  // read (i, j) from the upper triangle of a symmetric block
  __device__ __forceinline__ double at(int i, int j) const {
    if (sym && i > j) {
      const int t = i;
      i = j;
      j = t;
    }
    return p[i * rs + j * cs];
  }
  __device__ __forceinline__ double* ptr(int i, int j) const { return p + i * rs + j * cs; }
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum_l a(i, l) b(l, j), l < len, lanes of one warp split l
__device__ __forceinline__ double warp_dot(const View& a, int i, const View& b, int j, int len, int lane) {
  double acc = 0.0;
  for (int l = lane; l < len; l += 32) acc = fma(a.at(i, l), b.at(l, j), acc);
  return warp_sum(acc);
}

__device__ void gemm_update(const View& out, const View& a, const View& b, int sign, bool upper) {
  const int m = a.rows, p = a.cols, q = b.cols;
  if (m == 0 || p == 0 || q == 0) return;
  const long long total = (long long)m * q;
  if (p >= 64) {  // warp per element
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (long long e = warp; e < total; e += nw) {
      const int i = (int)(e / q), j = (int)(e - (long long)i * q);
      if (upper && i > j) continue;
      const double acc = warp_dot(a, i, b, j, p, lane);
      if (lane == 0) *out.ptr(i, j) += sign > 0 ? acc : -acc;
    }
  } else {
    for (long long e = threadIdx.x; e < total; e += blockDim.x) {
      const int i = (int)(e / q), j = (int)(e - (long long)i * q);
      if (upper && i > j) continue;
      double acc = 0.0;
      for (int l = 0; l < p; ++l) acc = fma(a.at(i, l), b.at(l, j), acc);
      *out.ptr(i, j) += sign > 0 ? acc : -acc;
    }
  }
}

// returns the first non-positive pivot's index + 1 (0: none), same on every thread
__device__ int chol_leaf(const View& w, int base) {
  const int m = w.rows;
  int bad = 0;
  for (int i = 0; i < m; ++i) {
    __syncthreads();
    const double piv = w.at(i, i);
    if (piv <= 0.0 && !bad) bad = base + i + 1;
    const double d = sqrt(piv);
    __syncthreads();
    if (threadIdx.x == 0) *w.ptr(i, i) = d;
    for (int j = i + 1 + threadIdx.x; j < m; j += blockDim.x) *w.ptr(i, j) /= d;
    __syncthreads();
    const int t = m - i - 1;
    for (int e = threadIdx.x; e < t * t; e += blockDim.x) {
      const int r = i + 1 + e / t, c = i + 1 + e % t;
      if (c >= r) *w.ptr(r, c) -= w.at(i, r) * w.at(i, c);
    }
  }
  __syncthreads();
  return bad;
}

__device__ void trsm_left(const View& t, const View& w) {
  const int m = t.rows, q = w.cols;
  for (int j = threadIdx.x; j < q; j += blockDim.x)
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int l = 0; l < i; ++l) acc = fma(t.at(i, l), w.at(l, j), acc);
      *w.ptr(i, j) = (w.at(i, j) - acc) / t.at(i, i);
    }
}

// L W + W U = W0 in place: element (i, j) on anti-diagonal s = i + j needs
// W(i, k), k < j and W(k, j), k < i — all on earlier anti-diagonals
__device__ void sylv_solve(const View& l, const View& u, const View& w) {
  const int m = w.rows, q = w.cols;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int s = 0; s <= m + q - 2; ++s) {
    const int i0 = s - (q - 1) > 0 ? s - (q - 1) : 0, i1 = s < m - 1 ? s : m - 1;
    for (int i = i0 + warp; i <= i1; i += nw) {
      const int j = s - i;
      const double au = warp_dot(w, i, u, j, j, lane);
      const double al = warp_dot(l, i, w, j, i, lane);
      if (lane == 0) *w.ptr(i, j) = ((w.at(i, j) - au) - al) / (l.at(i, i) + u.at(j, j));
    }
    __syncthreads();
  }
}

// L W + W L^T = W0, W symmetric: upper triangle by anti-diagonals, mirrored as solved
__device__ void lyap_solve(const View& l, const View& w) {
  const int m = w.rows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  View lt = l;  // L^T
  lt.rs = l.cs;
  lt.cs = l.rs;
  for (int s = 0; s <= 2 * m - 2; ++s) {
    const int i0 = s - (m - 1) > 0 ? s - (m - 1) : 0, i1 = s / 2;  // i <= j = s - i
    for (int i = i0 + warp; i <= i1; i += nw) {
      const int j = s - i;
      const double al = warp_dot(l, i, w, j, i, lane);
      const double au = warp_dot(w, i, lt, j, j, lane);
      if (lane == 0) {
        const double x = ((w.at(i, j) - al) - au) / (l.at(i, i) + l.at(j, j));
        *w.ptr(i, j) = x;
        *w.ptr(j, i) = x;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) big_kernel(const __grid_constant__ StmtList sl, int eq, int n, int b,
                                                   const double* __restrict__ in0, const double* __restrict__ in1,
                                                   const double* __restrict__ in2, double* __restrict__ X,
                                                   int* __restrict__ info, long long batch) {
  const long long nn = (long long)n * n;
  const bool sym_target = eq != kEqSylv, x_sym = eq == kEqLyap;
  __shared__ int s_bad;
  for (long long prob = blockIdx.x; prob < batch; prob += gridDim.x) {
    double* x = X + prob * nn;
    const double* rhs = (eq == kEqChol ? in0 : eq == kEqLyap ? in1 : in2) + prob * nn;
    double* mats[3] = {x, const_cast<double*>(in0 + prob * nn), const_cast<double*>(in1 + prob * nn)};
    // copy-in restricted to the unknown's structure (verify.py:236-241)
    for (long long e = threadIdx.x; e < nn; e += blockDim.x) {
      const int i = (int)(e / n), j = (int)(e - (long long)i * n);
      x[e] = (eq == kEqChol && j < i) ? 0.0 : rhs[e];
    }
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    int flag = 0;
    for (int k = 0; k < n / b; ++k) {
      const int st[3] = {0, k * b, (k + 1) * b};
      const int ex[3] = {k * b, b, n - (k + 1) * b};
      for (int s = 0; s < sl.count; ++s) {
        const lagen_stmt& S = sl.s[s];
        View out{x + (long long)st[S.out.r] * n + st[S.out.c], n, 1, ex[S.out.r], ex[S.out.c], false};
        if (out.rows == 0 || out.cols == 0) continue;
        View in[2];
        for (int t = 0; t < 2; ++t) {
          const lagen_view& v = S.in[t];
          if (v.op < 0) continue;
          double* base = mats[v.op] + (long long)st[v.r] * n + st[v.c];
          const int r = ex[v.r], c = ex[v.c];
          if (v.trans) in[t] = View{base, 1, n, c, r, false};
          else in[t] = View{base, n, 1, r, c, false};
          // diagonal block of a symmetric unknown: triu(m) + triu(m, 1)^T (verify.py:254-261)
          if (v.op == 0 && x_sym && v.r == v.c && r > 1) in[t] = View{base, n, 1, r, r, true};
        }
        switch (S.kind) {
          case LAGEN_GEMM_UPDATE:
            gemm_update(out, in[0], in[1], S.sign, sym_target && S.out.r == S.out.c);
            break;
          case LAGEN_CHOL: {
            const int bad = chol_leaf(out, st[S.out.r]);
            if (bad && !flag) flag = bad;
            break;
          }
          case LAGEN_TRSM_LEFT_TRANSPOSED:
            trsm_left(in[0], out);
            break;
          case LAGEN_SYLV:
            sylv_solve(in[0], in[1], out);
            break;
          case LAGEN_LYAP:
            lyap_solve(in[0], out);
            break;
          default:
            break;
        }
        __syncthreads();
      }
    }
    // mirror_lower (kernels.py:133-138), then the NaN / Inf guard over all of X
    bool nonfinite = false;
    for (long long e = threadIdx.x; e < nn; e += blockDim.x) {
      const int i = (int)(e / n), j = (int)(e - (long long)i * n);
      double v = x[e];
      if (x_sym && j < i) {
        v = x[(long long)j * n + i];
        x[e] = v;
      }
      nonfinite = nonfinite || !isfinite(v);
    }
    if (nonfinite) s_bad = 1;
    __syncthreads();
    if (threadIdx.x == 0 && info) info[prob] = flag ? flag : (s_bad ? -1 : 0);
    __syncthreads();
  }
}

}  // namespace big

// host side: called by lagen_b200_execute_* for n > 128
cudaError_t launch_big(const StmtList& sl, int eq, int n, int b, const double* const* in, double* X, int* info,
                       long long batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (err != cudaSuccess) return err;
  const long long resident = 4ll * sm_budget(sms);  // 4 CTAs of 256 threads per SM
  const unsigned grid = (unsigned)(batch < resident ? batch : resident);
  const double* i0 = in[0];
  const double* i1 = eq >= 1 ? in[1] : in[0];
  const double* i2 = eq == 2 ? in[2] : in[0];
  big::big_kernel<<<grid, 256, 0, s>>>(sl, eq, n, b, i0, i1, i2, X, info, batch);
  return cudaGetLastError();
}

}  // namespace lagen
