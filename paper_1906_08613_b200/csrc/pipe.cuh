// pipe.cuh — the "pipe engine": triangular Sylvester (L X + X U = C) and
// triangular Lyapunov (L X + X L^T = S) as an 8x8-tile anti-diagonal
// wavefront whose diagonal-tile solves run on dedicated solver warps while
// updater warps apply the bulk tile updates (DMMA) concurrently.
//
// Math (tile (I, J) of X, 8x8 tiles, T = ceil(n / 8) per side):
//   L_II X_IJ + X_IJ U_JJ = C_IJ - sum_{k<I} L_Ik X_kJ - sum_{k<J} X_Ik U_kJ
// — the 2x2-block recursion every Sylvester variant is derived from
// (ref:pkg/tests/test_invariants.py:25-32 PME), applied at tile granularity
// in the order of the right-looking variants (Sylvester v13, Lyapunov v5):
// tile (I, J) takes the contributions of X_kJ and X_Ik in increasing k; the
// diagonal-block solve is the SYLV leaf (ref:pkg/src/lagen/kernels.py:100-110,
// element (r, c) from row and column predecessors); Lyapunov computes the
// upper tiles only with U = L^T (kernels.py:113-130), its diagonal tiles are
// solved as Sylvester blocks and mirrored, and X is mirrored on the way out
// (verify.py:299-300).  Results agree with the statement-list executor to
// rounding (parity tests: relative difference <= 1e-10).
//
// Schedule (one problem per warp group; step d solves anti-diagonal d):
//   solver warps : tiles of diagonal d (up to 4 per warp, one per 8-lane
//                  group): add the last two contributions (from diagonal
//                  d-1, DMMA), solve in place (lane = column, 15-step element
//                  wavefront), publish -X, stream X to HBM
//   updater warps: every later tile of their columns takes the contributions
//                  of diagonal d-1 (DMMA m8n8k4, accumulators in registers);
//                  tiles of diagonal d+1 are handed to the solvers
//   one group barrier per step.
// The two roles overlap inside a step, so a step costs max(solve latency,
// update throughput) instead of their sum.  Three rotating tile buffers (one
// tile per row on a diagonal): diagonal d-1 (read by both roles), d (solved
// in place), d+1 (written by the updaters).
//
// Ownership: updater warp w owns columns {w, 2NU-1-w, 2NU+w, ...}
// (boustrophedon, balances the per-column work of both equations); its
// accumulators acc[u][I] are static register indices, and every shared-memory
// operand address is a per-step base plus a compile-time offset.  L and U
// tiles live in shared memory as swizzled 8x8 tiles (A, B and C fragments of
// m8n8k4 bank-conflict free).  n not a multiple of 8: padded rows / columns
// get a zero pivot reciprocal, so the padded X entries are exactly 0 and
// never reach a real one.
#pragma once
#include <cuda_runtime.h>

#include "engine.cuh"

namespace lagen {
namespace pipe {

using eng::cp_async16;
using eng::cp_async_commit;
using eng::cp_async_wait;
using eng::dmma;

// element (r, c) of a swizzled 8x8 tile: 16-byte pairs stay together, rows
// 2, 3, 6, 7 swap column halves (m8n8k4 A / B / C fragments conflict-free)
__device__ __forceinline__ int sw(int r, int c) { return r * 8 + (c ^ ((r & 2) << 1)); }
__host__ __device__ constexpr int ltidx(int I, int J) { return I * (I + 1) / 2 + J; }  // I >= J
__host__ __device__ constexpr int utidx(int I, int J) { return J * (J + 1) / 2 + I; }  // I <= J

// 1 / a without the division subroutine: rcp.approx + two Newton steps (~1 ulp)
__device__ __forceinline__ double recip(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}

// MODE 0: split roles (NU updater warps + NS solver warps per problem, one
// problem per CTA); MODE 1: "solo" — one warp per problem runs both roles in
// turn, PP problems per CTA (small T, where problems in flight hide latency)
template <int EQ, int N, int MODE>
struct PCfg {
  static_assert(EQ == 1 || EQ == 2, "pipe engine: Lyapunov (1) or Sylvester (2)");
  static constexpr int T = (N + 7) / 8;
  static_assert(T >= 1 && T <= 16, "n <= 128");
  static_assert(N % 2 == 0, "16-byte row pairs");
  static constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
  // tiles on the longest anti-diagonal (Lyapunov: upper tiles only)
  static constexpr int MAXM = EQ == 2 ? T : cdiv(T, 2);
  // columns per updater warp: pairs (boustrophedon / folded) while several
  // CTAs share an SM; one column per warp where one CTA per SM runs (more
  // warps per problem; Sylvester T = 11, 12: 8-14 % with SOLVE2, Lyapunov
  // T >= 14: 1-11 %, profiles/r02_pipe_solver_ab.txt)
#ifndef LAGEN_PIPE_SYLV_CU1_T
#define LAGEN_PIPE_SYLV_CU1_T 11
#endif
#ifndef LAGEN_PIPE_LYAP_CU1_T
#define LAGEN_PIPE_LYAP_CU1_T 14
#endif
  static constexpr int CU = MODE == 1 ? T : (EQ == 2 ? (T >= LAGEN_PIPE_SYLV_CU1_T ? 1 : 2) : (T >= LAGEN_PIPE_LYAP_CU1_T ? 1 : 2));
  static constexpr int NU = MODE == 1 ? 1 : cdiv(T, CU);
  static constexpr int NS = MODE == 1 ? 0 : cdiv(MAXM, 4);
  static_assert(MODE == 0 || MAXM <= 4, "solo mode: one warp solves at most 4 tiles per step");
  static constexpr int GW = MODE == 1 ? 1 : NU + NS;  // warps per problem
  static constexpr int NLT = T * (T + 1) / 2;
  static constexpr int TILES = EQ == 2 ? 2 * NLT : NLT;
  static constexpr int PS = 68;  // tile-slot pitch: the 4 solve groups' tiles start in different banks
  static constexpr int NSV = MODE == 1 ? 1 : NS;  // warps that solve
  static constexpr int SCR = NSV * 32 * 8;          // per-lane pivot reciprocals of the solve
  static constexpr int QP = 232;                    // solve scratch per group: 22 rows x 10 (+ pad, = 8 mod 16)
  static constexpr int LSH = (8 * T + 14) * 10;     // L_II columns for the solve, 7 zero rows each side
  static constexpr int BFS = 2 * MAXM * PS;         // two diagonals' tile slots (d-1 read, d written)
  static constexpr int SLOT = TILES * 64 + BFS + LSH + 64 + SCR + NSV * 4 * QP + 2;  // doubles (+ flag)
  static constexpr int smem_fit(int pp) { return (227 * 1024) / (pp * SLOT * 8); }
  static constexpr int PP = MODE == 1 ? 4 : 1;  // problems per CTA
  static constexpr int THREADS = PP * GW * 32;
  static constexpr size_t SMEM = (size_t)PP * SLOT * 8;
  static constexpr int mn(int a, int b) { return a < b ? a : b; }
  // tile-solve formulation (sol_step): SOLVE2 keeps only FMA -> FMA -> MUL ->
  // SHFL on the dependent chain and predicates the idle 8-lane groups' shared
  // memory accesses off; measured faster only where one CTA per SM runs with
  // one column per updater warp (Sylvester T >= 11: 2-14 %, Lyapunov T = 14,
  // 15: 2-5 %), slower or neutral elsewhere (profiles/r02_pipe_solver_ab.txt)
  // first solve formulation: shared-memory accesses of the 8-lane groups
  // without a tile predicated off.  The solve is bound by the SM's shared
  // memory / shuffle pipe (about 45 cycles of it per element step and solver
  // warp: 7 LDS.128, 3 LDS.64, STS.64, a 64-bit SHFL at 8.6), so the idle
  // groups' loads cost as much as the live ones'; the predicates cost a few
  // registers, so it is on where measured faster (profiles/r02_pipe_solver_ab.txt)
  static constexpr bool pred_on() {
    if (MODE == 1) return false;
    if (EQ == 2) return T >= 5 && T <= 8;
    return N == 52 || N == 56 || N == 60 || N == 64 || N == 72 || N == 76 || N == 80 || N == 84 || N == 100 || N == 124 ||
           N == 128;
  }
#ifdef LAGEN_PIPE_PRED
  static constexpr bool PRED = LAGEN_PIPE_PRED != 0;
#else
  static constexpr bool PRED = pred_on();
#endif
#ifdef LAGEN_PIPE_PRED_SETUP
  static constexpr bool PRED_SETUP = LAGEN_PIPE_PRED_SETUP != 0;
#else
  static constexpr bool PRED_SETUP = false;
#endif
#ifdef LAGEN_PIPE_SOLVE2
  static constexpr bool SOLVE2 = LAGEN_PIPE_SOLVE2 != 0;
#else
  static constexpr bool SOLVE2 = MODE == 0 && (EQ == 2 ? T >= LAGEN_PIPE_SYLV_CU1_T : (T == 14 || T == 15));
#endif
  // CTAs per SM for __launch_bounds__ (it sets the register budget).  Split
  // roles: measured per tile count over MINB = 1..8 at the BASELINE batches
  // (tools/experiments/pipe_bench.cu, profiles/r02_pipe_minb_sweep.txt) — more
  // CTAs hide the solve's latency until the accumulators spill (Lyapunov holds
  // T + 1 tiles per updater warp: 96 registers spill from T = 9 on).  Solo
  // mode: what shared memory and threads allow with >= 128 registers.
  static constexpr int RMIN = MODE == 1 ? 128 : 96;
  static constexpr int fitb(int b) { return (b <= 1 || 65536 / (THREADS * b) >= RMIN) ? b : fitb(b - 1); }
  static constexpr int MINB_FIT = fitb(mn(smem_fit(PP), 2048 / THREADS));
  static constexpr int kLyapMinb[17] = {1, 1, 1, 1, 7, 7, 6, 4, 4, 3, 2, 2, 2, 2, 1, 1, 1};
  static constexpr int kSylvMinb[17] = {1, 1, 1, 1, 4, 4, 4, 3, 2, 2, 2, 1, 1, 1, 1, 1, 1};
  static constexpr int MINB_TAB = mn(EQ == 1 ? kLyapMinb[T] : kSylvMinb[T], mn(smem_fit(PP), 2048 / THREADS));
  static constexpr int MINB0 = (MODE == 1 || T < 4) ? MINB_FIT : MINB_TAB;
#ifdef LAGEN_PIPE_MINB
  static constexpr int MINB = LAGEN_PIPE_MINB;
#else
  static constexpr int MINB = MINB0 < 1 ? 1 : MINB0;
#endif
};

// rows x 16-byte pairs of an n x n row-major operand into the lower (PART 0)
// or upper (PART 1) tiles; entries outside n are 0 (identity diagonal) — only
// padded X entries ever read them
template <int N, int T, int PART, int G>
__device__ __forceinline__ void load_tri(double* tiles, const double* __restrict__ src, int rank) {
#ifdef LAGEN_PIPE_LOAD_ROWMAJOR
  constexpr int NP = 8 * T, HP = NP / 2;
  for (int u = rank; u < NP * HP; u += G) {
    const int r = u / HP, cp = u - r * HP;
    const int I = r >> 3, J = cp >> 2;
    if (PART == 0 ? J > I : J < I) continue;
    double* dst = tiles + (PART == 0 ? ltidx(I, J) : utidx(I, J)) * 64 + sw(r & 7, 2 * (cp & 3));
    const int c = 2 * cp;
    if (r < N && c < N) {  // N even: the pair is inside
      cp_async16(dst, src + r * N + c);
    } else {
      *reinterpret_cast<double2*>(dst) = make_double2(r == c ? 1.0 : 0.0, r == c + 1 ? 1.0 : 0.0);
    }
  }
#else
  // a warp per tile and pass: lane (r8, p) moves the 16-byte pair (r8, 2 p) of
  // tile t; the tiles are walked in storage order (t = ltidx / utidx), the
  // tile coordinates follow incrementally — no division and no iterations over
  // the other triangle
  constexpr int NWG = G / 32, NT = T * (T + 1) / 2;
  const int wq = rank >> 5, lane = rank & 31;
  const int r8 = lane >> 2, c2 = 2 * (lane & 3);
  const int so = sw(r8, c2);
  int a = 0, bq = wq;  // tile t = a (a + 1) / 2 + bq, bq <= a: (I, J) = (a, bq) lower, (bq, a) upper
  while (bq > a) {
    bq -= a + 1;
    ++a;
  }
  for (int t = wq; t < NT; t += NWG) {
    const int r = 8 * (PART == 0 ? a : bq) + r8, c = 8 * (PART == 0 ? bq : a) + c2;
    double* dst = tiles + t * 64 + so;
    if (r < N && c < N) {  // N even: the pair is inside
      cp_async16(dst, src + r * N + c);
    } else {
      *reinterpret_cast<double2*>(dst) = make_double2(r == c ? 1.0 : 0.0, r == c + 1 ? 1.0 : 0.0);
    }
    bq += NWG;
    while (bq > a) {
      bq -= a + 1;
      ++a;
    }
  }
#endif
}

template <int EQ, int N, int MODE>
__global__ void __launch_bounds__(PCfg<EQ, N, MODE>::THREADS, PCfg<EQ, N, MODE>::MINB)
    pipe_kernel(const double* __restrict__ Lg, const double* __restrict__ Ug, const double* __restrict__ Cg,
                double* __restrict__ X, int* __restrict__ info, long long batch,
                unsigned long long* __restrict__ prof) {
  using P = PCfg<EQ, N, MODE>;
  constexpr int T = P::T, CU = P::CU, NU = P::NU, GW = P::GW, PS = P::PS, G = GW * 32, QP = P::QP;
  constexpr long long NN = (long long)N * N;
  constexpr int SOLT = P::NSV * 32;  // solver threads per problem
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / GW, wi = warp % GW, rank = threadIdx.x % G;
  double* base = smem + (size_t)grp * P::SLOT;
  double* Lt = base;
  double* Ut = base + P::NLT * 64;  // Sylvester only
  double* Bf = base + P::TILES * 64;
  double* Lsh = Bf + P::BFS;
  double* Zt = Lsh + P::LSH;  // a zero tile
  double* Skb = Zt + 64 + P::SCR;  // solve scratches: tile i of the diagonal -> Skb + i QP
  int* flag = reinterpret_cast<int*>(Skb + P::NSV * 4 * QP);
  const bool is_upd = MODE == 1 || wi < NU;
  const int w = MODE == 1 ? 0 : wi;                          // updater index
  const int sv = MODE == 1 ? 0 : (wi >= NU ? wi - NU : 0);  // solver index
  const int srank = MODE == 1 ? lane : rank - NU * 32;
  double* scr = Zt + 64 + sv * 256 + lane;  // pivot reciprocals: row r of the tile at scr[32 r] (conflict-free)
  const int g = lane >> 2, t = lane & 3;
  const int oA0 = sw(g, t), oA1 = sw(g, t + 4), oB0 = sw(t, g), oB1 = sw(t + 4, g);
  const int oR = (7 + g) * 10 + 2 * t;  // C fragment in a solve scratch (row-major, pitch 10, 7 pad rows)
  // step barrier: one warp (solo) or every thread of the CTA; the two roles
  // reach it from different code, so it is the PTX barrier with an explicit
  // count.  Hand-over barrier (split roles): updaters arrive once the
  // diagonal-d right-hand sides are in the solve scratches, solvers wait.
  auto gbar = [&]() {
    if constexpr (MODE == 1) __syncwarp();
    else asm volatile("bar.sync 1, %0;" ::"n"(P::THREADS) : "memory");
  };
  // profiling (tools/pipe_profile.py): clock64 per phase of the first
  // problem of CTA 0, solver warp 0 -> prof[4 (d + 1) + k], updater warp 0 ->
  // prof[256 + 2 (d + 1) + k]
  // (compiled in with -DLAGEN_PIPE_PROF only: the tests cost ~4 % of the
  // kernel's instructions; tools/experiments/pipe_build.sh defines it)
#ifdef LAGEN_PIPE_PROF
  unsigned long long* pr = nullptr;
  auto stamp = [&](int idx) {
    if (pr && lane == 0) pr[idx] = clock64();
  };
#else
  (void)prof;
  auto stamp = [&](int) {};
#endif
  auto i0of = [&](int dd) { return dd - T + 1 > 0 ? dd - T + 1 : 0; };
  // published -X of diagonal dd: buffer dd mod 2, tile (I, dd - I) at row
  // I - i0(dd) (the base is shifted so that row I is base + I * PS)
  auto dbuf = [&](int dd) -> double* { return Bf + ((dd + 2) & 1) * P::MAXM * PS - i0of(dd) * PS; };
  // column of updater slot u (boustrophedon over the NU warps)
  auto colof = [&](int u) { return (u & 1) ? (u + 1) * NU - 1 - w : u * NU + w; };

  // Accumulator slots.  Sylvester (and Lyapunov with one column per warp):
  // slot (u, I) = tile (I, colof(u)).  Lyapunov with column pairs {w, T-1-w}
  // ("folded", FOLD): slot f <= w is tile (f, w), slot f > w is tile
  // (T - f, T-1-w) — the pair's T + 1 upper tiles in T + 1 static slots.
  constexpr bool FOLD = EQ == 1 && CU == 2;
  constexpr int NSLOT = FOLD ? T + 1 : CU * T;
  // per-column step preamble: L X source row k = d-1-J and its B fragments,
  // per-step bases of the L and U operands
  struct Pre {
    int J, k;
    bool lx;
    double b0, b1;
    const double* pL;
    const double* pU;
  };
  auto prep = [&](int d, int J, const double* pv) {
    Pre q;
    q.J = J;
    q.k = d - 1 - J;
    q.lx = q.k >= 0 && (EQ == 2 ? q.k < T : q.k < J);
    q.b0 = q.lx ? pv[q.k * PS + oB0] : 0.0;
    q.b1 = q.lx ? pv[q.k * PS + oB1] : 0.0;
    q.pL = Lt + q.k * 64;                                               // + ltidx(I, 0) * 64
    q.pU = (EQ == 2 ? Ut : Lt) + (J * (J + 1) / 2 + d - 1) * 64;         // - I * 64
    return q;
  };
  // diagonal d-1's contributions into tile (I, q.J) (I static):
  // L_Ik X_kJ (k = d-1-J) and X_Ik U_kJ (k = d-1-I)
  auto tile_upd = [&](int d, const Pre& q, const double* pv, int I, double& c0, double& c1) {
    if (q.lx) {
      const double* A = q.pL + ltidx(I, 0) * 64;
      dmma(c0, c1, A[oA0], q.b0);
      dmma(c0, c1, A[oA1], q.b1);
    }
    const int kp = d - 1 - I;
    if (kp >= 0) {
      const double* B = q.pU - I * 64;
      if constexpr (EQ == 2) {
        const double* A = pv + I * PS;
        dmma(c0, c1, A[oA0], B[oB0]);
        dmma(c0, c1, A[oA1], B[oB1]);
      } else {  // X_Ik: upper tile (I, k) or (k, I)^T;  U_kJ = L_Jk^T
        const bool up = I <= kp;
        const double* A = pv + (up ? I : kp) * PS;
        dmma(c0, c1, A[up ? oA0 : oB0], B[oA0]);
        dmma(c0, c1, A[up ? oA1 : oB1], B[oA1]);
      }
    }
  };
  // visit every slot: fn(slot, I, J, column-preamble index) with I static
  auto for_slots = [&](auto&& fn) {
    if constexpr (FOLD) {
      const int J1 = T - 1 - w;
#pragma unroll
      for (int f = 0; f <= T; ++f) {
        if (f <= w) fn(f, f, w, 0);
        else if (J1 > w) fn(f, T - f, J1, 1);
      }
    } else {
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const int J = colof(u);
        if (J >= T) continue;
#pragma unroll
        for (int I = 0; I < T; ++I) {
          if (EQ == 1 && I > J) continue;
          fn(u * T + I, I, J, u);
        }
      }
    }
  };

  // right-hand side straight into the accumulators (C fragment layout)
  auto upd_init = [&](double (&a0)[NSLOT], double (&a1)[NSLOT], const double* __restrict__ Cp) {
#pragma unroll
    for (int f = 0; f < NSLOT; ++f) a0[f] = a1[f] = 0.0;
    for_slots([&](int f, int I, int J, int) {
      const int r = 8 * I + g, c = 8 * J + 2 * t;
      if (r < N && c < N) {
        if (EQ == 1 && I == J && r > c) {  // symmetric right-hand side: upper triangle only
          a0[f] = __ldg(Cp + (long long)c * N + r);
          a1[f] = r > c + 1 ? __ldg(Cp + (long long)(c + 1) * N + r) : __ldg(Cp + (long long)r * N + c + 1);
        } else {
          const double2 v = __ldg(reinterpret_cast<const double2*>(Cp + (long long)r * N + c));
          a0[f] = v.x;
          a1[f] = v.y;
        }
      }
    });
  };

  // updater step d: diagonal d-1's contributions into the warp's tiles —
  // phase CRIT: the tile of each column on diagonal d, then its right-hand
  // side to the solve scratch; phase BULK: every later tile.  The active tiles
  // of a column are a contiguous row range, entered through a switch whose
  // cases fall through (static register slots, no per-tile tests beyond the
  // range end): L X into rows [lo, hi], X U into rows [lo, min(hi, d-1)].
  auto slotof = [&](int u, int I) { return FOLD ? (u == 0 ? I : T - I) : u * T + I; };
  auto colJ = [&](int u) { return FOLD ? (u == 0 ? w : T - 1 - w) : colof(u); };
  constexpr int NCOL = FOLD ? 2 : CU;
  auto tile_lx = [&](const Pre& q, int I, double& c0, double& c1) {
    const double* A = q.pL + ltidx(I, 0) * 64;
    dmma(c0, c1, A[oA0], q.b0);
    dmma(c0, c1, A[oA1], q.b1);
  };
  auto tile_xu = [&](int d, const Pre& q, const double* pv, int I, double& c0, double& c1) {
    const double* B = q.pU - I * 64;
    if constexpr (EQ == 2) {
      const double* A = pv + I * PS;
      dmma(c0, c1, A[oA0], B[oB0]);
      dmma(c0, c1, A[oA1], B[oB1]);
    } else {  // X_Ik: upper tile (I, k) or (k, I)^T;  U_kJ = L_Jk^T
      const int kp = d - 1 - I;
      const bool up = I <= kp;
      const double* A = pv + (up ? I : kp) * PS;
      dmma(c0, c1, A[up ? oA0 : oB0], B[oA0]);
      dmma(c0, c1, A[up ? oA1 : oB1], B[oA1]);
    }
  };
#define PIPE_I16(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)
  auto upd_crit = [&](int d, double (&a0)[NSLOT], double (&a1)[NSLOT]) {
    const double* pv = dbuf(d - 1);
    const int i0 = i0of(d);
#pragma unroll
    for (int u = 0; u < NCOL; ++u) {
      const int J = colJ(u);
      if (J >= T || (FOLD && u == 1 && J <= w)) continue;
      const int hi = EQ == 2 ? T - 1 : J;
      const int Ic = d - J;
      if (Ic < 0 || Ic > hi) continue;
      const Pre q = prep(d, J, pv);
      switch (Ic) {
#define PIPE_CRIT(i)                                                                  \
  case i:                                                                             \
    if constexpr (i < T) {                                                            \
      const int f = slotof(u, i);                                                     \
      if (q.lx) tile_lx(q, i, a0[f], a1[f]);                                          \
      if (J >= 1) tile_xu(d, q, pv, i, a0[f], a1[f]);                                 \
      *reinterpret_cast<double2*>(Skb + (i - i0) * QP + oR) = make_double2(a0[f], a1[f]); \
    }                                                                                 \
    break;
        PIPE_I16(PIPE_CRIT)
#undef PIPE_CRIT
        default: break;
      }
    }
  };
  auto upd_bulk = [&](int d, double (&a0)[NSLOT], double (&a1)[NSLOT]) {
    const double* pv = dbuf(d - 1);
#pragma unroll
    for (int u = 0; u < NCOL; ++u) {
      const int J = colJ(u);
      if (J >= T || (FOLD && u == 1 && J <= w)) continue;
      const int hi = EQ == 2 ? T - 1 : J;
      const int lo = d + 1 - J > 0 ? d + 1 - J : 0;
      if (lo > hi) continue;
      const Pre q = prep(d, J, pv);
      if (q.lx) {
        switch (lo) {
#define PIPE_LX(i)                        \
  case i:                                 \
    if constexpr (i < T) {                \
      if (i > hi) break;                  \
      const int f = slotof(u, i);         \
      tile_lx(q, i, a0[f], a1[f]);        \
    }                                     \
    [[fallthrough]];
          PIPE_I16(PIPE_LX)
#undef PIPE_LX
          default: break;
        }
      }
      const int hx = hi < d - 1 ? hi : d - 1;
      if (lo <= hx) {
        switch (lo) {
#define PIPE_XU(i)                         \
  case i:                                  \
    if constexpr (i < T) {                 \
      if (i > hx) break;                   \
      const int f = slotof(u, i);          \
      tile_xu(d, q, pv, i, a0[f], a1[f]);  \
    }                                      \
    [[fallthrough]];
          PIPE_I16(PIPE_XU)
#undef PIPE_XU
          default: break;
        }
      }
    }
  };

  // solver step d (d = -1: build Lsh): tile i = 4 sv + q of diagonal d, in
  // scratch Skb + i QP: rows 7..14 of a pitch-10 row-major block with 7 zero
  // rows above and below, so the wavefront element of step s in lane c, (s -
  // c, c), and its row are a per-lane base plus a compile-time offset; the
  // pivot array and Lsh use the same indexing
  auto sol_step = [&](int d, long long prob, bool& bad) {
    if (d < 0) {
      // Lsh row 7 + 8 I + r: L_II(r + e, r) at column e = 1..7 (0 below the
      // tile); 7 zero rows before and after (rows s - c outside the tile)
      for (int u = srank; u < T * 64; u += SOLT) {
        const int I = u >> 6, r = (u >> 3) & 7, e = u & 7;
        Lsh[(7 + 8 * I + r) * 10 + e] = (e >= 1 && r + e < 8) ? Lt[ltidx(I, I) * 64 + sw(r + e, r)] : 0.0;
      }
      return;
    }
    const int i0 = i0of(d);
    const int i1 = EQ == 2 ? (d < T - 1 ? d : T - 1) : d / 2;
    const int m = i1 - i0 + 1;  // tiles on diagonal d
    if (4 * sv >= m) {  // no tile for this warp: still takes part in the hand-over barrier
      if constexpr (MODE == 0) asm volatile("bar.sync 2, %0;" ::"n"(P::THREADS) : "memory");
      return;
    }
    const int qg = lane >> 3, c = lane & 7;
    const bool live = 4 * sv + qg < m;
    const int I = i0 + 4 * sv + (live ? qg : 0), J = d - I;
    double* Sq = Skb + (4 * sv + (live ? qg : 0)) * QP;
    if (sv == 0) stamp(4 * (d + 1));
    // pivot reciprocals of column c, 1 / (l_rr + u_cc) (0 for padding), and
    // column c of U_JJ above the diagonal (Lyapunov: row c of L_JJ) — ahead
    // of the hand-over wait
    const double* Ld = Lt + ltidx(I, I) * 64;
    const double* Ud = EQ == 2 ? Ut + utidx(J, J) * 64 : Lt + ltidx(J, J) * 64;
    auto uat = [&](int k) -> double { return EQ == 2 ? Ud[sw(k, c)] : Ud[sw(c, k)]; };
    if constexpr (!P::SOLVE2) {
      // uo[j] = U_JJ(j, c) for j <= c - 2 (older row values, from the scratch),
      // u1 = U_JJ(c - 1, c) (newest, by shuffle); 0 elsewhere
      double uo[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      double u1 = 0.0;
      if (live || !P::PRED_SETUP) {
        const double ucc = uat(c);
        double dg[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) dg[r] = Ld[sw(r, r)];
#pragma unroll
        for (int r = 0; r < 8; ++r) scr[32 * r] = (8 * I + r < N && 8 * J + c < N) ? recip(dg[r] + ucc) : 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const double v = uat(j);
          uo[j] = j + 2 <= c ? v : 0.0;
        }
        const double u1v = uat(c >= 1 ? c - 1 : 0);
        u1 = c >= 1 ? u1v : 0.0;
      }
      if constexpr (MODE == 0) asm volatile("bar.sync 2, %0;" ::"n"(P::THREADS) : "memory");
      else __syncwarp();
      if (sv == 0) stamp(4 * (d + 1) + 1);
      // solve: lane c owns column c; y / h: circular buffers of 8 over the
      // steps (slot s & 7 = row s - c), static register indices.  The row
      // contribution sum_{j<c} x_rj u_jc takes x_{r,c-1} (one step old) by
      // shuffle and the older ones from the scratch row (written >= 2 steps ago)
      double* Sl = Sq + (7 - c) * 10 + c;             // + 10 s: element (s - c, c)
      const double* Sr = Sq + (7 - c) * 10;           // + 10 s: row s - c
      // pivot of row s - c: scr[32 ((s - c) & 7)] (rows outside the tile wrap around; their x is masked)
      const int pl0 = (8 - c) & 7;
      auto pl = [&](int s) -> double { return scr[32 * ((pl0 + s) & 7)]; };
      const double* Ll = Lsh + (7 + 8 * I - c) * 10;  // + 10 s: L_II column s - c
      const int src1 = (lane & ~7) | (c >= 1 ? c - 1 : c);
      // (letting the groups without a tile skip the solve — no instructions, no
      // wavefronts — measured 5-17 % slower: the divergence costs more registers)
      const unsigned lm = 0xffffffffu;
      const bool lv = live || !P::PRED;  // groups without a tile: no shared-memory traffic
      double y[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) y[s] = lv ? Sl[10 * s] : 0.0;
      // sum_{j <= c-2} x_rj u_jc of step s's row r = s - c, computed one step
      // ahead from the scratch row (its entries were written >= 2 steps before
      // step s, so visible after the previous step's __syncwarp)
      auto rowsum = [&](int s) -> double {
        const double2* rw = reinterpret_cast<const double2*>(Sr + 10 * s);
        double2 r0 = make_double2(0.0, 0.0), r1 = r0, r2 = r0;
        if (lv) r0 = rw[0], r1 = rw[1], r2 = rw[2];  // (columns 6, 7 are never "older": j <= c - 2 <= 5)
        double t0 = r0.x * uo[0];
        double t1 = r0.y * uo[1];
        t0 = fma(r1.x, uo[2], t0);
        t1 = fma(r1.y, uo[3], t1);
        t0 = fma(r2.x, uo[4], t0);
        t1 = fma(r2.y, uo[5], t1);
        return t0 + t1;
      };
      // Program order matters (in-order issue): each step first loads what the
      // next one needs, then runs the dependent chain x(r, c-1) --shfl--> FMA
      // -> MUL -> x, shuffles x on right away, and only then the pushes and
      // the next row sum (whose loads have landed by then)
      double x1 = 0.0;                       // x(r, c-1) of the current step, by shuffle
      double pcur = lv ? pl(0) : 0.0;
      double vpre = y[0] - rowsum(0);        // y - older row contributions of the current step
      // (loaded values persist in the idle groups: predicated loads, no re-zeroing)
      double2 la = make_double2(0.0, 0.0), lb = la, lcc = la, ld = la, r0 = la, r1 = la, r2 = la;
      double pnxt = 0.0, yref = 0.0;
      auto step = [&](int s, int u) {
        const bool act = (unsigned)(s - c) < 8u;
        // loads: this step's L_II column (push), the next step's row / pivot
        const double2* lc = reinterpret_cast<const double2*>(Ll + 10 * s);
        if (lv) la = lc[0], lb = lc[1], lcc = lc[2], ld = lc[3];
        const double2* rw = reinterpret_cast<const double2*>(Sr + 10 * (s + 1));
        if (s < 14 && lv) {
          r0 = rw[0], r1 = rw[1], r2 = rw[2];
          pnxt = pl(s + 1);
        }
        if (s + 8 <= 14 && lv) yref = Sl[10 * (s + 8)];
        // the chain
        const double v = fma(-x1, u1, vpre);
        const double x = act ? v * pcur : 0.0;
        x1 = __shfl_sync(lm, x, src1);
        // push into the next row first (the next step's vpre), then the rest
        y[(u + 1) & 7] = fma(-la.y, x, y[(u + 1) & 7]);
        if (s < 14) {
          double t0 = r0.x * uo[0];
          double t1 = r0.y * uo[1];
          t0 = fma(r1.x, uo[2], t0);
          t1 = fma(r1.y, uo[3], t1);
          t0 = fma(r2.x, uo[4], t0);
          t1 = fma(r2.y, uo[5], t1);
          vpre = y[(u + 1) & 7] - (t0 + t1);
          pcur = pnxt;
        }
        if (lv) Sl[10 * s] = x;  // in place (0 outside the tile)
        const double coef[8] = {0.0, la.y, lb.x, lb.y, lcc.x, lcc.y, ld.x, ld.y};
#pragma unroll
        for (int e = 2; e < 8; ++e) y[(u + e) & 7] = fma(-coef[e], x, y[(u + e) & 7]);
        if (s + 8 <= 14) y[u] = yref;
        __syncwarp(lm);
      };
#pragma unroll
      for (int u = 0; u < 8; ++u) step(u, u);
#pragma unroll
      for (int u = 0; u < 7; ++u) step(8 + u, u);
    } else {
      // uo[j] = U_JJ(j, c) for j <= c - 3 (older row values, from the scratch),
      // u2 = U_JJ(c - 2, c) and u1 = U_JJ(c - 1, c) (the two newest row values,
      // by shuffle); 0 elsewhere
      double uo[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      double u1 = 0.0, u2 = 0.0;
      {
        const double ucc = uat(c);
        double dg[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) dg[r] = Ld[sw(r, r)];
#pragma unroll
        for (int r = 0; r < 8; ++r) scr[32 * r] = (8 * I + r < N && 8 * J + c < N) ? recip(dg[r] + ucc) : 0.0;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          const double v = uat(j);
          uo[j] = j + 3 <= c ? v : 0.0;
        }
        const double u1v = uat(c >= 1 ? c - 1 : 0);
        u1 = c >= 1 ? u1v : 0.0;
        const double u2v = uat(c >= 2 ? c - 2 : 0);
        u2 = c >= 2 ? u2v : 0.0;
      }
      if constexpr (MODE == 0) asm volatile("bar.sync 2, %0;" ::"n"(P::THREADS) : "memory");
      else __syncwarp();
      if (sv == 0) stamp(4 * (d + 1) + 1);
      // solve: lane c owns column c, step s finishes element (r, c), r = s - c.
      //   x_rc = p_rc (y_rc - sum_{k<r} l_rk x_kc - sum_{j<c} x_rj u_jc)
      // The dependent chain of a step is only
      //   x_{r-1,c} --FMA--> t --(shuffled x_{r,c-1}) FMA--> v --MUL--> x_rc --SHFL-->
      // everything else has at least one step of slack: the contributions of
      // rows <= r-2 of the column are pushed into y[] (circular buffer of 8 over
      // the steps, static register indices), x_{r,c-2} arrives by a second
      // shuffle one step earlier, and x_{r,j}, j <= c-3, were written to the
      // scratch row >= 2 steps before their load (visible after __syncwarp).
      // Lanes outside the tile (r < 0 or r > 7) run on garbage that only reaches
      // other lanes outside the tile; their x is stored and pushed as 0.
      double* Sl = Sq + (7 - c) * 10 + c;             // + 10 s: element (s - c, c)
      const double* Sr = Sq + (7 - c) * 10;           // + 10 s: row s - c
      // pivot of row s - c: scr[32 ((s - c) & 7)] (rows outside the tile wrap around; their x is masked)
      const int pl0 = (8 - c) & 7;
      auto pl = [&](int s) -> double { return scr[32 * ((pl0 + s) & 7)]; };
      const double* Ll = Lsh + (7 + 8 * I - c) * 10;  // + 10 s: L_II column s - c
      const int src1 = (lane & ~7) | (c >= 1 ? c - 1 : c);
      const int src2 = (lane & ~7) | (c >= 2 ? c - 2 : c);
      const unsigned lm = 0xffffffffu;
      double y[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) y[s] = live ? Sl[10 * s] : 0.0;
      // sum_{j <= c-3} x_rj u_jc of the row of step s, from the scratch row
      auto rowsum3 = [&](int s) -> double {
        const double2* rw = reinterpret_cast<const double2*>(Sr + 10 * s);
        double2 r0 = make_double2(0.0, 0.0), r1 = r0;
        double r2 = 0.0;
        if (live) {
          r0 = rw[0], r1 = rw[1];
          r2 = Sr[10 * s + 4];
        }
        double t0 = r0.x * uo[0];
        double t1 = r0.y * uo[1];
        t0 = fma(r1.x, uo[2], t0);
        t1 = fma(r1.y, uo[3], t1);
        t0 = fma(r2, uo[4], t0);
        return t0 + t1;
      };
      double xu = 0.0;                 // this lane's previous element (unmasked)
      double x1 = 0.0;                 // x(r, c-1) for the current step, by shuffle
      double x2 = 0.0;                 // x(r+1, c-2) for the next step, by shuffle
      double l1 = 0.0;                 // L_II(r, r-1)
      double pcur = live ? pl(0) : 0.0;
      double base = y[0] - rowsum3(0);
      double rs3 = rowsum3(1);
      double2 ca = make_double2(0.0, 0.0), cb = ca, cc = ca, cd = ca;  // L_II column r below the diagonal (this step's pushes)
      if (live) {
        const double2* lc = reinterpret_cast<const double2*>(Ll);
        ca = lc[0], cb = lc[1], cc = lc[2], cd = lc[3];
      }
      double2 r0 = make_double2(0.0, 0.0), r1 = r0;  // scratch row of step s + 2
      double r2 = 0.0;
      auto step = [&](int s, int u) {
        const bool act = (unsigned)(s - c) < 8u;
        // loads for later steps: the scratch row of step s + 2 (its entries
        // j <= c - 3 were stored before the previous step's __syncwarp)
        if (s < 13 && live) {
          const double2* rw = reinterpret_cast<const double2*>(Sr + 10 * (s + 2));
          r0 = rw[0], r1 = rw[1];
          r2 = Sr[10 * (s + 2) + 4];
        }
        // the chain
        const double t = fma(-l1, xu, base);
        const double v = fma(-u1, x1, t);
        xu = v * pcur;
        x1 = __shfl_sync(lm, xu, src1);
        const double x = act ? xu : 0.0;
        // next step's right-hand side, without the two newest contributions
        base = (y[(u + 1) & 7] - rs3) - u2 * x2;
        x2 = __shfl_sync(lm, x, src2);
        if (live) Sl[10 * s] = x;  // in place (0 outside the tile)
        l1 = ca.y;
        // pushes into rows r+2 .. r+7 of the column
        const double coef[8] = {0.0, ca.y, cb.x, cb.y, cc.x, cc.y, cd.x, cd.y};
#pragma unroll
        for (int e = 2; e < 8; ++e) y[(u + e) & 7] = fma(-coef[e], x, y[(u + e) & 7]);
        if (s + 8 <= 14 && live) y[u] = Sl[10 * (s + 8)];
        if (s < 14 && live) {
          pcur = pl(s + 1);
          const double2* lc = reinterpret_cast<const double2*>(Ll + 10 * (s + 1));
          ca = lc[0], cb = lc[1], cc = lc[2], cd = lc[3];
        }
        if (s < 13) {
          double t0 = r0.x * uo[0];
          double t1 = r0.y * uo[1];
          t0 = fma(r1.x, uo[2], t0);
          t1 = fma(r1.y, uo[3], t1);
          t0 = fma(r2, uo[4], t0);
          rs3 = t0 + t1;
        }
        __syncwarp(lm);
      };
#pragma unroll
      for (int u = 0; u < 8; ++u) step(u, u);
#pragma unroll
      for (int u = 0; u < 7; ++u) step(8 + u, u);
    }
    if (sv == 0) stamp(4 * (d + 1) + 2);
    // column c of X (Lyapunov diagonal tile: lower := mirror of upper) ->
    // the published tile as -X (swizzled), and X -> HBM
    if (live) {
      double v[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        v[r] = Sq[(7 + r) * 10 + c];
        if (EQ == 1 && I == J && r > c) v[r] = Sq[(7 + c) * 10 + r];
      }
      double* Pt = dbuf(d) + I * PS;
#pragma unroll
      for (int r = 0; r < 8; ++r) Pt[sw(r, c)] = -v[r];
      double* Xp = X + prob * NN;
      const int col = 8 * J + c;
      // split roles: the updater warps stream the published tile to HBM during
      // the next step (store_diag), off the solve -> hand-over critical path
      if (MODE == 1 && col < N) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          bad = bad || !isfinite(v[r]);
          if (8 * I + r < N) __stcs(Xp + (long long)(8 * I + r) * N + col, v[r]);
        }
      }
      if (MODE == 1 && EQ == 1 && I != J && 8 * J + c < N) {  // mirror tile (J, I): its row c is column c of this tile
        double* row = Xp + (long long)(8 * J + c) * N + 8 * I;
#pragma unroll
        for (int mm = 0; mm < 4; ++mm)
          if (8 * I + 2 * mm < N) __stcs(reinterpret_cast<double2*>(row + 2 * mm), make_double2(v[2 * mm], v[2 * mm + 1]));
      }
    }
    if (sv == 0) stamp(4 * (d + 1) + 3);
  };

  // split roles: diagonal dd's published tiles (-X, swizzled) -> X in HBM, by
  // the updater warps (tile i of the diagonal -> warp i mod NU; lane (g, t)
  // stores row g, columns 2t, 2t + 1 as one 16-byte store; Lyapunov also the
  // mirror tile's row g from column g of the tile).  Runs one step after the
  // solve, behind the bulk updates.
  auto store_diag = [&](int dd, long long prob, bool& bad) {
    const int i0 = i0of(dd);
    const int i1 = EQ == 2 ? (dd < T - 1 ? dd : T - 1) : dd / 2;
    const double* pv = dbuf(dd);
    double* Xp = X + prob * NN;
    for (int I = i0 + w; I <= i1; I += NU) {
      const int J = dd - I;
      const double* Pt = pv + I * PS;
      const double2 a = *reinterpret_cast<const double2*>(Pt + sw(g, 2 * t));
      bad = bad || !isfinite(a.x) || !isfinite(a.y);
      const int r = 8 * I + g, c = 8 * J + 2 * t;
      if (r < N && c < N) __stcs(reinterpret_cast<double2*>(Xp + (long long)r * N + c), make_double2(-a.x, -a.y));
      if (EQ == 1 && I != J) {
        const int rm = 8 * J + g, cm = 8 * I + 2 * t;
        if (rm < N && cm < N)
          __stcs(reinterpret_cast<double2*>(Xp + (long long)rm * N + cm),
                 make_double2(-Pt[sw(2 * t, g)], -Pt[sw(2 * t + 1, g)]));
      }
    }
  };

  // once: zero tile, the solve scratches' pad rows / pad columns (must read
  // 0) and Lsh's zero rows
  for (int u = threadIdx.x; u < P::PP * P::SLOT; u += blockDim.x) smem[u] = 0.0;
  __syncthreads();

  const long long stride = (long long)gridDim.x * P::PP;
  for (long long prob = (long long)grp * gridDim.x + blockIdx.x; prob < batch; prob += stride) {
    const double* Lp = Lg + prob * NN;
    const double* Up = Ug + prob * NN;
    const double* Cp = Cg + prob * NN;
    load_tri<N, T, 0, G>(Lt, Lp, rank);
    if constexpr (EQ == 2) load_tri<N, T, 1, G>(Ut, Up, rank);
    cp_async_commit();
    if (rank == 0) *flag = 0;
    bool bad = false;
#ifdef LAGEN_PIPE_PROF
    pr = (prof && blockIdx.x == 0 && prob == grp * gridDim.x) ? prof : nullptr;
#endif
    // the roles run separate step loops with the same barrier sequence, so
    // the accumulators are live only in the updater warps' registers
    if (MODE == 1 || is_upd) {
      double a0[NSLOT], a1[NSLOT];
      upd_init(a0, a1, Cp);
      cp_async_wait<0>();
      gbar();
      if constexpr (MODE == 1) sol_step(-1, prob, bad);
      gbar();
#pragma unroll 1
      for (int d = 0; d <= 2 * T - 2; ++d) {
        if (w == 0) stamp(256 + 2 * (d + 1));
        upd_crit(d, a0, a1);
        if constexpr (MODE == 0) {
          asm volatile("bar.arrive 2, %0;" ::"n"(P::THREADS) : "memory");
        } else {
          __syncwarp();
          sol_step(d, prob, bad);
        }
        upd_bulk(d, a0, a1);
        if constexpr (MODE == 0)
          if (d >= 1) store_diag(d - 1, prob, bad);
        if (w == 0) stamp(256 + 2 * (d + 1) + 1);
        gbar();
      }
      if constexpr (MODE == 0) store_diag(2 * T - 2, prob, bad);
    } else {
      cp_async_wait<0>();
      gbar();
      sol_step(-1, prob, bad);
      gbar();
#pragma unroll 1
      for (int d = 0; d <= 2 * T - 2; ++d) {
        sol_step(d, prob, bad);
        gbar();
      }
    }
    if (bad) *flag = -1;
    gbar();
    if (rank == 0 && info) info[prob] = *flag;
  }
}

}  // namespace pipe
}  // namespace lagen
