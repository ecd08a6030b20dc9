// rowsweep.cuh — the "rowsweep engine": triangular Sylvester (L X + X U = C)
// and Lyapunov (L X + X L^T = S) for small n (<= 32), one lane per row.
//
// Math: column by column (the Bartels-Stewart order of the PME's last
// column block, ref:pkg/tests/test_invariants.py:25-32), column c of X solves
//     (L + u_cc I) x_c = c_c - X[:, :c] U[:c, c]
// — the SYLV leaf of ref:pkg/src/lagen/kernels.py:100-110 applied to the whole
// matrix (its `W[:, j] -= W[:, :j] U[:j, j]` then forward substitution with
// `(l_ii + u_jj)` divisors), Lyapunov with U = L^T (kernels.py:113-130) and the
// result mirrored from the upper triangle (verify.py:299-300).  Results agree
// with the statement-list executor to rounding (parity tests <= 1e-10).
//
// Mapping: a group of LP lanes (LP = next power of two >= n, >= 4) owns one
// problem, lane r = row r; 32 / LP problems per warp run in lockstep.  Lane r
// keeps row r of the right-hand side / solution in registers (y[0..n-1],
// static indices), so the X U part of every column is lane-local; the forward
// substitution down column c is n steps of (x_k in lane k, shuffled to the
// group, z_r -= (l_rk piv_r) x_k on the pivot-scaled value z_r = piv_r y_r):
// the dependent chain per step is SHFL -> DFMA.  L is staged in shared memory as a square with a zero
// upper triangle and zero diagonal (lane r reads l_rk at a per-lane base plus a
// compile-time offset; pitch n + 1 keeps the lanes on distinct banks); U's
// rows are read as broadcasts (Sylvester: packed upper rows; Lyapunov: the
// columns of the same L square).
#pragma once
#include <cuda_runtime.h>

#include "engine.cuh"

#ifndef LAGEN_RSW_SYMK
#define LAGEN_RSW_SYMK 1
#endif

namespace lagen {
namespace rsw {

__device__ __forceinline__ double recip(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}

template <int EQ, int N>
struct RCfg {
  static_assert(EQ == 1 || EQ == 2, "rowsweep engine: Lyapunov (1) or Sylvester (2)");
  static_assert(N >= 1 && N <= 32, "rowsweep engine: n <= 32");
  static constexpr int LP = N <= 4 ? 4 : N <= 8 ? 8 : N <= 16 ? 16 : 32;  // lanes per problem
  static constexpr int PPW = 32 / LP;                                      // problems per warp
  static constexpr int W = 4;                                              // warps per CTA
  static constexpr int PITCH = N + 1;                                      // L square row pitch (odd)
  static constexpr int LSQ = N * PITCH;
  static constexpr int UPK = EQ == 2 ? N * (N + 1) / 2 : 0;                // packed upper rows of U
  static constexpr int PSZ = (LSQ + UPK + 1) & ~1;                         // doubles per problem (16 B aligned)
  static constexpr int THREADS = W * 32;
  static constexpr size_t SMEM = (size_t)W * PPW * PSZ * 8;
  // CTAs per SM and the substitution form, measured per (equation, n) over
  // MINB in 2..8 x {scaled, unscaled} at the BASELINE batches
  // (tools/experiments/rsw_bench.cu, profiles/r02_rowsweep_sweep.txt; Lyapunov
  // re-swept with the symmetric shortcut, r02_rowsweep_symk.txt): more
  // CTAs hide the substitution chain's latency even where the row of y then
  // spills a few registers; the scaled form (a DFMA less on the chain, n - 1
  // more products live) wins where registers allow.  Index n / 4.
  static constexpr int mn(int a, int b) { return a < b ? a : b; }
  static constexpr int kMinb[2][9] = {{0, 8, 8, 5, 4, 4, 3, 3, 3}, {0, 8, 8, 6, 5, 5, 5, 4, 4}};
  static constexpr bool kScaled[2][9] = {{0, 0, 0, 1, 1, 0, 1, 1, 0}, {0, 0, 0, 1, 0, 0, 0, 0, 0}};
  static constexpr int RMIN = N > 16 ? 168 : N > 8 ? 96 : 64;
  static constexpr int MINB_FIT = mn(mn((227 * 1024) / (int)SMEM, 2048 / THREADS), 65536 / (THREADS * RMIN));
  static constexpr int MINB0 = N % 4 == 0 ? mn(kMinb[EQ - 1][N / 4], mn((227 * 1024) / (int)SMEM, 2048 / THREADS)) : MINB_FIT;
#ifdef LAGEN_RSW_SCALED
  static constexpr bool SCALED = LAGEN_RSW_SCALED;
#else
  static constexpr bool SCALED = N % 4 == 0 ? kScaled[EQ - 1][N / 4] : false;
#endif
#ifdef LAGEN_RSW_MINB
  static constexpr int MINB = LAGEN_RSW_MINB;
#else
  static constexpr int MINB = MINB0 < 1 ? 1 : MINB0;
#endif
};

__host__ __device__ constexpr int urow(int N, int j) { return j * N - j * (j - 1) / 2; }  // packed upper row j start

template <int EQ, int N>
__global__ void __launch_bounds__(RCfg<EQ, N>::THREADS, RCfg<EQ, N>::MINB)
    rowsweep_kernel(const double* __restrict__ Lg, const double* __restrict__ Ug, const double* __restrict__ Cg,
                    double* __restrict__ X, int* __restrict__ info, long long batch) {
  using P = RCfg<EQ, N>;
  constexpr int LP = P::LP, PPW = P::PPW, PITCH = P::PITCH;
  constexpr long long NN = (long long)N * N;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LP, r = lane % LP;  // problem slot in the warp, row
  const int gbase = grp * LP;
  double* Ls = smem + (size_t)(warp * PPW + grp) * P::PSZ;  // L square, zero upper triangle and diagonal
  double* Us = Ls + P::LSQ;                                  // Sylvester: packed upper rows of U
  const bool real = r < N;

  const long long slots = (long long)gridDim.x * P::W * PPW;
  for (long long base = ((long long)blockIdx.x * P::W + warp) * PPW; base < batch; base += slots) {
    const long long prob = base + grp;
    const bool live = prob < batch;
    const long long pc = live ? prob : base;  // dead slots recompute a live problem, store nothing
    const double* Lp = Lg + pc * NN;
    const double* Cp = Cg + pc * NN;
    // stage L (lower part, zero diagonal) and U's upper rows; each lane of the
    // group takes whole rows' elements strided by LP
    for (int e = r; e < N * N; e += LP) {
      const int i = e / N, j = e - (e / N) * N;
      Ls[i * PITCH + j] = j < i ? __ldg(Lp + e) : 0.0;
      if constexpr (EQ == 2)
        if (j >= i) Us[urow(N, i) + (j - i)] = __ldg(Ug + pc * NN + e);
    }
    // row r of the right-hand side (Lyapunov: the symmetric S from its upper
    // triangle) and l_rr
    double y[N];
#pragma unroll
    for (int c = 0; c < N; ++c) {
      y[c] = 0.0;
      if (real) y[c] = (EQ == 1 && c < r) ? __ldg(Cp + (long long)c * N + r) : __ldg(Cp + (long long)r * N + c);
    }
    const double lrr = real ? __ldg(Lp + (long long)r * N + r) : 1.0;
    __syncwarp();
    // row r of L in registers (l_rk, 0 for k >= r; padding lanes: row 0, all 0)
    double lr[N > 1 ? N - 1 : 1];
    {
      const double* Lrow = Ls + (real ? r : 0) * PITCH;
#pragma unroll
      for (int k = 0; k < N - 1; ++k) lr[k] = Lrow[k];
    }
    bool bad = false;
#pragma unroll
    for (int c = 0; c < N; ++c) {
      // u_cc: Sylvester U(c, c); Lyapunov L(c, c) (read from global, cached)
      const double ucc = EQ == 2 ? Us[urow(N, c)] : __ldg(Lp + (long long)c * N + c);
      const double piv = real ? recip(lrr + ucc) : 0.0;
      // forward substitution down column c.  SCALED: on the pivot-scaled
      // value z_r = piv_r (y_r - sum_k l_rk x_k) — lane k's z is x_k itself,
      // so the dependent chain per step is SHFL -> DFMA (the scaling
      // l_rk piv_r is off the chain); otherwise DMUL -> SHFL -> DFMA on y
      // (fewer live registers: measured per size, RCfg::SCALED)
      double x;
      // Lyapunov (SYMK): X is symmetric, so x_kc for k < c is already known
      // as x_ck — lane c's finished y[k] — and its broadcast does not wait
      // for this column's chain; only the steps k >= c are dependent
      // (n^2 / 2 chained steps instead of n^2).
      constexpr bool SYMK = EQ == 1 && LAGEN_RSW_SYMK;
      if constexpr (P::SCALED) {
        double z = y[c] * piv;
#pragma unroll
        for (int k = 0; k < N - 1; ++k) {
          const double xk = (SYMK && k < c) ? __shfl_sync(0xffffffffu, y[k], gbase + c)
                                            : __shfl_sync(0xffffffffu, z, gbase + k);
          z = fma(-(lr[k] * piv), xk, z);
        }
        x = z;
      } else {
#pragma unroll
        for (int k = 0; k < N - 1; ++k) {
          const double xk = (SYMK && k < c) ? __shfl_sync(0xffffffffu, y[k], gbase + c)
                                            : __shfl_sync(0xffffffffu, y[c] * piv, gbase + k);
          y[c] = fma(-lr[k], xk, y[c]);
        }
        x = y[c] * piv;
      }
      y[c] = x;
      bad = bad || !isfinite(x);
      // push into the later columns: y_c' -= x u_{c,c'}
#pragma unroll
      for (int c2 = c + 1; c2 < N; ++c2) {
        const double u = EQ == 2 ? Us[urow(N, c) + (c2 - c)] : Ls[c2 * PITCH + c];
        y[c2] = fma(-x, u, y[c2]);
      }
    }
    // Lyapunov: X := upper triangle mirrored (row r takes column r of the
    // rows above it) through the L square's slot, which is free now
    if constexpr (EQ == 1) {
      __syncwarp();
      if (real) {
#pragma unroll
        for (int c = 0; c < N; ++c) Ls[r * PITCH + c] = y[c];
      }
      __syncwarp();
      if (real) {
#pragma unroll
        for (int c = 0; c < N; ++c)
          if (c < r) y[c] = Ls[c * PITCH + r];
      }
    }
    const unsigned gmask = (PPW == 1) ? 0xffffffffu : (((1u << LP) - 1u) << gbase);
    bad = (__ballot_sync(0xffffffffu, bad && real) & gmask) != 0;
    if (live && real) {
      double* Xr = X + prob * NN + (long long)r * N;
#pragma unroll
      for (int c = 0; c + 1 < N; c += 2) __stcs(reinterpret_cast<double2*>(Xr + c), make_double2(y[c], y[c + 1]));
      if (N & 1) __stcs(Xr + N - 1, y[N - 1]);
    }
    if (live && r == 0 && info) info[prob] = bad ? -1 : 0;
    __syncwarp();
  }
}

}  // namespace rsw
}  // namespace lagen
