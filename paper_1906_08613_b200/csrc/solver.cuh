// solver.cuh — sm_100a device library: one blocked variant executed on a batch
// of fixed-size fp64 problems, every problem resident in shared memory.
//
// The per-iteration statement list (the variant) is the reference's
// `Algorithm.statements` (worksheet.py:47-87) in the lagen_stmt encoding; the
// loop structure restates interpret_algorithm (verify.py:221-303):
//   copy-in X := rhs restricted to X's structure   -> cooperative TMA-free
//   for k < n/b: for stmt: dispatch on kind         -> run_problem()
//   mirror / NaN guard                              -> store phase
// Each statement kind is a G-thread cooperative routine whose semantics match
// the reference block kernel it replaces (kernels.py):
//   gemm_tile     <- gemm_update  (kernels.py:16-34)
//   trsm_lt       <- trsm_left    (kernels.py:47-60)
//   chol_leaf     <- chol_leaf    (kernels.py:79-97)
//   sylv_solve    <- sylv_solve   (kernels.py:100-110)
//   lyap_solve    <- lyap_solve   (kernels.py:113-130)
// Summation orders differ from numpy's BLAS (unpinned by the reference, whose
// tests use tolerances); parity is <= 1e-10 relative.
//
// Shared-memory layout per problem (leading dimension LD = N + 1, odd, so
// column walks are bank-conflict free for 8-byte accesses):
//   cholesky : X   [N][LD]  upper triangle used (lower never read)
//   lyapunov : XL  [N][LD]  X upper incl. diag | L strictly lower | L diag in col N
//   sylvester: X   [N][LD]  dense, and (if it fits) LU [N][LD]:
//              L lower incl. diag | U strictly upper | U diag in col N
// so a problem costs N(N+1) doubles per packed pair instead of 2N^2.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lagen_b200.h"

namespace lagen {

constexpr int kEqChol = 0, kEqLyap = 1, kEqSylv = 2;

struct StmtList {
  lagen_stmt s[LAGEN_MAX_STMTS];
  int count;
};

constexpr int cmin(int a, int b) { return a < b ? a : b; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }

// ----------------------------------------------------------------------------
// Launch policy per (equation, n): threads per problem G, problems per CTA P,
// staging of the coefficient operands.  Chosen so that a CTA holds <= ~100 KB
// of problems and <= 256 threads (>= 2 CTAs/SM where they fit).
// ----------------------------------------------------------------------------
template <int EQ, int N>
struct Policy {
  static constexpr int LD = N + 1;
  static constexpr bool STAGE = (EQ != kEqSylv) || (2 * N * LD * 8 <= 200 * 1024);
  static constexpr int NM = (EQ == kEqSylv && STAGE) ? 2 : 1;
  static constexpr int PS = (NM * N * LD) | 1;  // odd problem stride (doubles)
  static constexpr int G = N <= 8 ? 1 : N <= 16 ? 4 : N <= 32 ? 32 : N <= 64 ? 128 : 256;
  static constexpr int PT = G == 1 ? 128 : cmax(1, 256 / G);
  static constexpr int PSM = cmax(1, (100 * 1024) / (PS * 8));
  static constexpr int P0 = cmin(PT, PSM);
  // whole warps: G==1 -> P multiple of 32; G<32 -> P multiple of 32/G
  static constexpr int WARP_P = G >= 32 ? 1 : 32 / G;
  static constexpr int P1 = (P0 / WARP_P) * WARP_P > 0 ? (P0 / WARP_P) * WARP_P : WARP_P;
  static constexpr int P = G > 32 ? cmin(P1, 15) : P1;  // named barriers 1..15
  static constexpr int THREADS = G * P;
  static constexpr size_t SMEM = (size_t)P * PS * 8 + (((size_t)P * sizeof(int) + 15) & ~(size_t)15);  // + per-problem flags
};

// ----------------------------------------------------------------------------
// Group synchronisation: G consecutive threads own one problem.
// ----------------------------------------------------------------------------
template <int G>
struct Group {
  int rank;
  int slot;
  __device__ __forceinline__ void sync() const {
    if constexpr (G == 1) {
    } else if constexpr (G <= 32) {
      const unsigned lane = threadIdx.x & 31u;
      const unsigned mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(unsigned)(G - 1)));
      __syncwarp(mask);
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(slot + 1), "r"(G) : "memory");
    }
  }
};

// A problem operand in shared (or global) memory.
struct Mat {
  double* p;
  int ld;
  int dcol;  // <0: diagonal at (i,i); else diagonal of row i stored at column dcol
};

// A block view: element (i,j) = p[i*rs + j*cs]; diagonal element i = dp[i*ds]
// (meaningful for diagonal blocks used as triangular coefficients).
struct View {
  double* p;
  int rs, cs;
  double* dp;
  int ds;
  int ld;  // storage leading dimension (for symmetric gathers)
  __device__ __forceinline__ double at(int i, int j) const { return p[i * rs + j * cs]; }
  __device__ __forceinline__ double& ref(int i, int j) const { return p[i * rs + j * cs]; }
  __device__ __forceinline__ double d(int i) const { return dp[i * ds]; }
  // symmetric diagonal block stored in its upper triangle (verify.py:254-261)
  __device__ __forceinline__ double sym(int i, int j) const {
    const int a = i < j ? i : j, b = i < j ? j : i;
    return p[a * ld + b];
  }
};

__device__ __forceinline__ const Mat& pick(const Mat* mats, int op) {
  return op == 0 ? mats[0] : (op == 1 ? mats[1] : mats[2]);
}

__device__ __forceinline__ View make_view(const Mat& M, int r0, int c0, int trans) {
  View v;
  v.p = M.p + r0 * M.ld + c0;
  v.ld = M.ld;
  if (trans) {
    v.rs = 1;
    v.cs = M.ld;
  } else {
    v.rs = M.ld;
    v.cs = 1;
  }
  if (M.dcol < 0) {
    v.dp = M.p + r0 * M.ld + r0;
    v.ds = M.ld + 1;
  } else {
    v.dp = M.p + r0 * M.ld + M.dcol;
    v.ds = M.ld;
  }
  return v;
}

// ----------------------------------------------------------------------------
// GEMM_update: O(m x q) += sign * A(m x p) B(p x q)   [kernels.py:16-34]
// 4x4 register tiles; UP = upper target (only i <= j written); SA/SB =
// symmetric-gather operands.  When tiles < G the p-loop is split across S
// lanes of one warp and reduced with shuffles (fixed order: deterministic).
// ----------------------------------------------------------------------------
template <int G, bool SA, bool SB, bool UP>
__device__ __forceinline__ void gemm_tile(const View& O, const View& A, const View& Bm, int m, int p, int q,
                                          double sgn, int rank) {
  const int tq = q >> 2;
  const int ntiles = (m >> 2) * tq;
  int S = 1;
  if constexpr (G > 1) {
    while (S < 32 && S * 2 <= G && S * 2 * ntiles <= G && S * 2 * 4 <= p) S *= 2;
  }
  const int units = ntiles * S;
  for (int u = rank; u < units; u += G) {
    const int t = u / S;
    const int sp = u - t * S;
    const int ti = t / tq, tj = t - ti * tq;
    if (UP && ti > tj) continue;  // whole tile strictly below the diagonal
    const int i0 = ti * 4, j0 = tj * 4;
    const int l0 = (p * sp) / S, l1 = (p * (sp + 1)) / S;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int l = l0; l < l1; ++l) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = SA ? A.sym(i0 + a, l) : A.at(i0 + a, l);
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = SB ? Bm.sym(l, j0 + b) : Bm.at(l, j0 + b);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    if (S > 1) {
      const unsigned lane = threadIdx.x & 31u;
      const unsigned seg = (S == 32) ? 0xffffffffu : (((1u << S) - 1u) << (lane & ~(unsigned)(S - 1)));
      for (int off = S >> 1; off > 0; off >>= 1)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] += __shfl_xor_sync(seg, acc[a][b], off);
      if (sp != 0) continue;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (!UP || i0 + a <= j0 + b) O.ref(i0 + a, j0 + b) = fma(sgn, acc[a][b], O.at(i0 + a, j0 + b));
  }
}

// ----------------------------------------------------------------------------
// TRSM_left_transposed: T W := W, T (m x m) logically lower  [kernels.py:47-60]
// Blocked right-looking over 4-row panels: diagonal 4-row solve (parallel over
// columns), then a rank-4 update of the rows below (parallel over elements).
// ----------------------------------------------------------------------------
template <int G, class Grp>
__device__ __forceinline__ void trsm_lt(const View& T, const View& W, int m, int q, const Grp& g) {
  for (int I = 0; I < m; I += 4) {
    const double d0 = T.d(I), d1 = T.d(I + 1), d2 = T.d(I + 2), d3 = T.d(I + 3);
    const double t10 = T.at(I + 1, I), t20 = T.at(I + 2, I), t21 = T.at(I + 2, I + 1);
    const double t30 = T.at(I + 3, I), t31 = T.at(I + 3, I + 1), t32 = T.at(I + 3, I + 2);
    for (int j = g.rank; j < q; j += G) {
      double w0 = W.at(I, j) / d0;
      double w1 = (W.at(I + 1, j) - t10 * w0) / d1;
      double w2 = (W.at(I + 2, j) - fma(t20, w0, t21 * w1)) / d2;
      double w3 = (W.at(I + 3, j) - fma(t30, w0, fma(t31, w1, t32 * w2))) / d3;
      W.ref(I, j) = w0;
      W.ref(I + 1, j) = w1;
      W.ref(I + 2, j) = w2;
      W.ref(I + 3, j) = w3;
    }
    const int rows = m - I - 4;
    if (rows <= 0) break;
    g.sync();
    const int units = rows * q;
    for (int u = g.rank; u < units; u += G) {
      const int l = I + 4 + u / q, j = u % q;
      double s = T.at(l, I) * W.at(I, j);
      s = fma(T.at(l, I + 1), W.at(I + 1, j), s);
      s = fma(T.at(l, I + 2), W.at(I + 2, j), s);
      s = fma(T.at(l, I + 3), W.at(I + 3, j), s);
      W.ref(l, j) -= s;
    }
    g.sync();
  }
}

// ----------------------------------------------------------------------------
// CHOL leaf: in-place upper Cholesky of a B x B diagonal block [kernels.py:79-97]
// right-looking: sqrt pivot, row scale, rank-1 update of the trailing upper
// triangle.  Non-positive pivot -> *flag = global index + 1 (first one).
// ----------------------------------------------------------------------------
template <int G, int B, class Grp>
__device__ __forceinline__ void chol_leaf(const View& W, int base, int* flag, const Grp& g) {
  for (int i = 0; i < B; ++i) {
    const double piv = W.at(i, i);
    const double d = sqrt(piv);
    g.sync();  // everyone has read the pivot before it is overwritten
    if (g.rank == 0 && !(piv > 0.0)) {
      if (piv <= 0.0 && *flag == 0) *flag = base + i + 1;
    }
    for (int j = i + g.rank; j < B; j += G) W.ref(i, j) = (j == i) ? d : W.at(i, j) / d;
    const int t = B - i - 1;
    if (t == 0) break;
    g.sync();
    for (int u = g.rank; u < t * t; u += G) {
      const int r = i + 1 + u / t, c = i + 1 + u % t;
      if (c >= r) W.ref(r, c) -= W.at(i, r) * W.at(i, c);
    }
    g.sync();
  }
}

// ----------------------------------------------------------------------------
// SYLV: L W + W U = W0 in place, L (m x m) lower, U (q x q) upper
// [kernels.py:100-110].  4x4-tile anti-diagonal wavefront: the tiles of one
// anti-diagonal are solved (one thread each, reference column/row order inside
// the tile), then every later tile in the same tile-row/-column receives the
// rank-4 contributions of the freshly solved tiles (parallel over elements).
// ----------------------------------------------------------------------------
__device__ __forceinline__ void sylv_tile4(const View& Lv, const View& Uv, const View& W, int i0, int j0) {
  double w[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) w[a][b] = W.at(i0 + a, j0 + b);
  double li[4], uj[4], rp[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    li[a] = Lv.d(i0 + a);
    uj[a] = Uv.d(j0 + a);
  }
  // reciprocal shifted pivots, off the substitution chain (<= 1 ulp)
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) rp[a][b] = 1.0 / (li[a] + uj[b]);
#pragma unroll
  for (int b = 0; b < 4; ++b) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < b; ++c) acc = fma(w[a][c], Uv.at(j0 + c, j0 + b), acc);
      w[a][b] -= acc;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < a; ++c) acc = fma(Lv.at(i0 + a, i0 + c), w[c][b], acc);
      w[a][b] = (w[a][b] - acc) * rp[a][b];
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) W.ref(i0 + a, j0 + b) = w[a][b];
}

template <int G, class Grp>
__device__ __forceinline__ void sylv_solve(const View& Lv, const View& Uv, const View& W, int m, int q,
                                           const Grp& g) {
  const int TI = m >> 2, TJ = q >> 2;
  for (int d = 0; d <= TI + TJ - 2; ++d) {
    const int ilo = d - (TJ - 1) > 0 ? d - (TJ - 1) : 0;
    const int ihi = d < TI - 1 ? d : TI - 1;
    for (int t = ilo + g.rank; t <= ihi; t += G) sylv_tile4(Lv, Uv, W, 4 * t, 4 * (d - t));
    if (d == TI + TJ - 2) break;
    g.sync();
    // push contributions of anti-diagonal d into later tiles
    const int units = TI * TJ * 4;
    for (int u = g.rank; u < units; u += G) {
      const int tile = u >> 2, a = u & 3;
      const int I2 = tile / TJ, J2 = tile - I2 * TJ;
      if (I2 + J2 <= d) continue;
      const int I1 = d - J2;  // solved tile in tile-column J2
      const int J1 = d - I2;  // solved tile in tile-row I2
      const bool colc = (I1 >= 0 && I1 < I2);
      const bool rowc = (J1 >= 0 && J1 < J2);
      if (!colc && !rowc) continue;
      const int i = 4 * I2 + a;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = 4 * J2 + b;
        double s = 0.0;
        if (colc) {
#pragma unroll
          for (int c = 0; c < 4; ++c) s = fma(Lv.at(i, 4 * I1 + c), W.at(4 * I1 + c, j), s);
        }
        if (rowc) {
#pragma unroll
          for (int c = 0; c < 4; ++c) s = fma(W.at(i, 4 * J1 + c), Uv.at(4 * J1 + c, j), s);
        }
        W.ref(i, j) -= s;
      }
    }
    g.sync();
  }
}

// ----------------------------------------------------------------------------
// LYAP: L W + W L^T = W0 for symmetric W (m x m) [kernels.py:113-130].
// Reads/writes the upper triangle only (the lower half of the storage may
// hold L).  Element anti-diagonal wavefront, pull model.
// ----------------------------------------------------------------------------
template <int G, class Grp>
__device__ __forceinline__ void lyap_solve(const View& Lv, const View& W, int m, const Grp& g) {
  for (int d = 0; d <= 2 * (m - 1); ++d) {
    const int ilo = d - (m - 1) > 0 ? d - (m - 1) : 0;
    const int ihi = d >> 1;
    for (int i = ilo + g.rank; i <= ihi; i += G) {
      const int j = d - i;
      const double rp = 1.0 / (Lv.d(i) + Lv.d(j));  // off the dot-product chain
      double acc = W.at(i, j);
      double d1 = 0.0, d2 = 0.0;
      for (int l = 0; l < i; ++l) d1 = fma(Lv.at(i, l), W.at(l, j), d1);
      for (int l = 0; l < j; ++l) d2 = fma(W.sym(i, l), Lv.at(j, l), d2);
      acc -= d1;
      acc -= d2;
      W.ref(i, j) = acc * rp;
    }
    g.sync();
  }
}

// ----------------------------------------------------------------------------
// One problem: the k loop over the variant's statements (verify.py:245-297).
// mats[0] = X storage, mats[1], mats[2] = coefficient operands.
// ----------------------------------------------------------------------------
template <int EQ, int N, int B, int G, class Grp>
__device__ __forceinline__ void run_problem(const StmtList& sl, const Mat* mats, int* flag, const Grp& g) {
  constexpr bool SYMT = (EQ != kEqSylv);  // rhs A/S symmetric: diagonal targets upper-only
  constexpr bool SYMX = (EQ == kEqLyap);  // unknown symmetric: diagonal blocks gathered
#pragma unroll 1
  for (int k = 0; k < N / B; ++k) {
    // 3x3 repartition starts / extents (verify.py:246-247), selected without
    // dynamic indexing so they stay in registers
    auto st = [&](int r) { return r == 0 ? 0 : (r == 1 ? k * B : (k + 1) * B); };
    auto ex = [&](int r) { return r == 0 ? k * B : (r == 1 ? B : N - (k + 1) * B); };
#pragma unroll 1
    for (int s = 0; s < sl.count; ++s) {
      const lagen_stmt S = sl.s[s];
      const int m = ex(S.out.r), q = ex(S.out.c);
      if (m == 0 || q == 0) continue;
      const View O = make_view(mats[0], st(S.out.r), st(S.out.c), 0);
      switch (S.kind) {
        case LAGEN_GEMM_UPDATE: {
          const lagen_view a = S.in[0], b = S.in[1];
          const int p = a.trans ? ex(a.r) : ex(a.c);
          if (p == 0) continue;
          const View Av = make_view(pick(mats, a.op), st(a.r), st(a.c), a.trans);
          const View Bv = make_view(pick(mats, b.op), st(b.r), st(b.c), b.trans);
          const bool up = SYMT && S.out.r == S.out.c;
          const bool sa = SYMX && a.op == 0 && a.r == a.c;
          const bool sb = SYMX && b.op == 0 && b.r == b.c;
          const double sgn = S.sign < 0 ? -1.0 : 1.0;
          if constexpr (SYMX) {
            if (sa) {
              if (up) gemm_tile<G, true, false, true>(O, Av, Bv, m, p, q, sgn, g.rank);
              else gemm_tile<G, true, false, false>(O, Av, Bv, m, p, q, sgn, g.rank);
            } else if (sb) {
              if (up) gemm_tile<G, false, true, true>(O, Av, Bv, m, p, q, sgn, g.rank);
              else gemm_tile<G, false, true, false>(O, Av, Bv, m, p, q, sgn, g.rank);
            } else {
              if (up) gemm_tile<G, false, false, true>(O, Av, Bv, m, p, q, sgn, g.rank);
              else gemm_tile<G, false, false, false>(O, Av, Bv, m, p, q, sgn, g.rank);
            }
          } else if constexpr (SYMT) {
            if (up) gemm_tile<G, false, false, true>(O, Av, Bv, m, p, q, sgn, g.rank);
            else gemm_tile<G, false, false, false>(O, Av, Bv, m, p, q, sgn, g.rank);
          } else {
            gemm_tile<G, false, false, false>(O, Av, Bv, m, p, q, sgn, g.rank);
          }
          break;
        }
        case LAGEN_CHOL:
          if constexpr (EQ == kEqChol) chol_leaf<G, B>(O, st(S.out.r), flag, g);
          break;
        case LAGEN_TRSM_LEFT_TRANSPOSED: {
          const lagen_view a = S.in[0];
          const View Tv = make_view(pick(mats, a.op), st(a.r), st(a.c), a.trans);
          trsm_lt<G>(Tv, O, m, q, g);
          break;
        }
        case LAGEN_SYLV: {
          if constexpr (EQ != kEqChol) {
            const lagen_view a = S.in[0], b = S.in[1];
            const View Lv = make_view(pick(mats, a.op), st(a.r), st(a.c), a.trans);
            const View Uv = make_view(pick(mats, b.op), st(b.r), st(b.c), b.trans);
            sylv_solve<G>(Lv, Uv, O, m, q, g);
          }
          break;
        }
        case LAGEN_LYAP: {
          if constexpr (EQ == kEqLyap) {
            const lagen_view a = S.in[0];
            const View Lv = make_view(pick(mats, a.op), st(a.r), st(a.c), a.trans);
            lyap_solve<G>(Lv, O, m, g);
          }
          break;
        }
        default:
          break;
      }
      g.sync();
    }
  }
}

// ----------------------------------------------------------------------------
// The batched kernel.  CTA = P problems x G threads.  Phases: cooperative
// vectorised load of the needed triangles -> per-group variant execution ->
// cooperative vectorised store of all n^2 entries of X (zeros / mirror) with
// the NaN/Inf guard (verify.py:301-302) folded in.
// inputs: chol {A}; lyap {L, S}; sylv {L, U, C}
// ----------------------------------------------------------------------------
template <int EQ, int N, int B>
__global__ void __launch_bounds__(Policy<EQ, N>::THREADS)
    solve_kernel(const __grid_constant__ StmtList sl, const double* __restrict__ in0, const double* __restrict__ in1,
                 const double* __restrict__ in2, double* __restrict__ X, int* __restrict__ info,
                 long long batch) {
  using Pol = Policy<EQ, N>;
  constexpr int G = Pol::G, P = Pol::P, LD = Pol::LD, PS = Pol::PS;
  constexpr int NN = N * N;
  extern __shared__ double smem[];
  int* flags = reinterpret_cast<int*>(smem + (size_t)P * PS);

  const long long first = (long long)blockIdx.x * P;
  const int nprob = (int)((batch - first) < P ? (batch - first) : P);
  if (threadIdx.x < P) flags[threadIdx.x] = 0;

  // ---- load phase: double2 vectors over the CTA's contiguous problem range
  const double* rhs = (EQ == kEqChol) ? in0 : (EQ == kEqLyap ? in1 : in2);
  {
    const long long base = first * NN;
    const int pairs = nprob * (NN / 2);
    for (int e = threadIdx.x; e < pairs; e += blockDim.x) {
      const int pr = e / (NN / 2);
      const int rem = 2 * (e - pr * (NN / 2));
      const int i = rem / N, j = rem - i * N;  // j even, (j, j+1) same row
      double* xs = smem + pr * PS + i * LD + j;
      // rhs: cholesky / lyapunov need the upper triangle only (j >= i)
      if (EQ == kEqSylv || j + 1 >= i) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(rhs + base) + e);
        if (EQ == kEqSylv || j >= i) xs[0] = v.x;
        if (EQ == kEqSylv || j + 1 >= i) xs[1] = v.y;
      }
      if constexpr (EQ == kEqLyap) {
        // L strictly lower -> same array below the diagonal, diag -> column N
        if (j <= i) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(in0 + base) + e);
          double* rowp = smem + pr * PS + i * LD;
          if (j < i) rowp[j] = v.x; else rowp[N] = v.x;
          if (j + 1 < i) rowp[j + 1] = v.y; else if (j + 1 == i) rowp[N] = v.y;
        }
      }
      if constexpr (EQ == kEqSylv && Pol::STAGE) {
        double* rowp = smem + pr * PS + N * LD + i * LD;
        if (j <= i) {  // L lower incl. diagonal
          const double2 v = __ldg(reinterpret_cast<const double2*>(in0 + base) + e);
          rowp[j] = v.x;
          if (j + 1 <= i) rowp[j + 1] = v.y;
        }
        if (j + 1 >= i) {  // U upper: strict part in place, diagonal -> column N
          const double2 v = __ldg(reinterpret_cast<const double2*>(in1 + base) + e);
          if (j > i) rowp[j] = v.x; else if (j == i) rowp[N] = v.x;
          if (j + 1 > i) rowp[j + 1] = v.y; else if (j + 1 == i) rowp[N] = v.y;
        }
      }
    }
  }
  __syncthreads();

  // ---- compute phase
  {
    Group<G> g;
    g.rank = threadIdx.x % G;
    g.slot = threadIdx.x / G;
    if (g.slot < nprob) {
      double* ps = smem + g.slot * PS;
      Mat mats[3];
      mats[0] = Mat{ps, LD, -1};
      if constexpr (EQ == kEqLyap) {
        mats[1] = Mat{ps, LD, N};
        mats[2] = mats[1];
      } else if constexpr (EQ == kEqSylv) {
        if constexpr (Pol::STAGE) {
          mats[1] = Mat{ps + N * LD, LD, -1};  // L: diag at (i,i)
          mats[2] = Mat{ps + N * LD, LD, N};   // U: diag in column N
        } else {
          const long long off = (first + g.slot) * NN;
          mats[1] = Mat{const_cast<double*>(in0) + off, N, -1};
          mats[2] = Mat{const_cast<double*>(in1) + off, N, -1};
        }
      } else {
        mats[1] = mats[0];
        mats[2] = mats[0];
      }
      run_problem<EQ, N, B, G>(sl, mats, &flags[g.slot], g);
    }
  }
  __syncthreads();

  // ---- store phase: all n^2 entries, zeros (chol) / mirror (lyap)
  {
    const long long base = first * NN;
    const int pairs = nprob * (NN / 2);
    for (int e = threadIdx.x; e < pairs; e += blockDim.x) {
      const int pr = e / (NN / 2);
      const int rem = 2 * (e - pr * (NN / 2));
      const int i = rem / N, j = rem - i * N;
      const double* xs = smem + pr * PS;
      double2 v;
      if constexpr (EQ == kEqChol) {
        v.x = (j >= i) ? xs[i * LD + j] : 0.0;
        v.y = (j + 1 >= i) ? xs[i * LD + j + 1] : 0.0;
      } else if constexpr (EQ == kEqLyap) {
        v.x = (j >= i) ? xs[i * LD + j] : xs[j * LD + i];
        v.y = (j + 1 >= i) ? xs[i * LD + j + 1] : xs[(j + 1) * LD + i];
      } else {
        v.x = xs[i * LD + j];
        v.y = xs[i * LD + j + 1];
      }
      if (!isfinite(v.x) || !isfinite(v.y)) atomicCAS(&flags[pr], 0, -1);
      reinterpret_cast<double2*>(X + base)[e] = v;
    }
  }
  if (info) {
    __syncthreads();
    if (threadIdx.x < nprob) info[first + threadIdx.x] = flags[threadIdx.x];
  }
}

}  // namespace lagen
