// wave.cuh — the "wave engine": triangular Sylvester (L X + X U = C) and
// triangular Lyapunov (L X + X L^T = S) as an 8x8-tile anti-diagonal
// wavefront with every cross-tile update on the FP64 tensor path.
//
// Math (tile (I, J) of X, tiles 8x8, T = ceil(n / 8) per side):
//   L_II X_IJ + X_IJ U_JJ = C_IJ - sum_{k<I} L_Ik X_kJ - sum_{k<J} X_Ik U_kJ
// — the 2x2-block recursion every Sylvester variant is derived from
// (ref:pkg/tests/test_invariants.py:25-32 PME), applied at tile granularity
// in the order of the right-looking variant v13 (Sylvester) / v5 (Lyapunov):
// tile (I, J) takes the contributions of X_kJ and X_Ik in increasing k, the
// diagonal-block solve is the SYLV leaf (ref:pkg/src/lagen/kernels.py:100-110,
// column-then-row order) and, for Lyapunov, only upper tiles are computed
// and mirrored at the end (verify.py:299-300) with U = L^T (kernels.py:113-130).
// Results agree with the statement-list executor to rounding (the tile-level
// summation order differs), which the parity tests bound at 1e-10.
//
// Schedule: anti-diagonal d = I + J is solved at step d.  X_{I,k} / X_{k,J}
// on diagonal d-1 are the LAST contributions any unsolved tile needs from
// that diagonal's tiles in the same tile-row / tile-column... and every tile
// of diagonal d-1 is needed only at step d, by exactly the tiles in its
// row and column — so contributions are PULLED at step d from a one-diagonal
// publish buffer (double-buffered), never stored as a full X in shared memory:
//     step d:  (1) critical: tiles on diagonal d take their last two
//                  contributions (4 DMMA) and are written to the publish slot
//              (2) each 8-lane group solves one of the warp's diagonal-d
//                  tiles in place (column-per-lane wavefront, shuffles);
//                  the result (-X) is published and X streamed to HBM
//              (3) bulk: every later tile takes its contributions from
//                  diagonal d-1 (DMMA m8n8k4, accumulators in registers)
//              one CTA-group barrier.
// Residency: NW warps own a problem, accumulators of the unknown's tiles live
// in registers (tile q of the diagonal-major order -> warp q % NW, slot
// q / NW: balanced per diagonal); L (lower tiles) and U (upper tiles) in
// shared memory, swizzled row-major 8x8 tiles so A, B and C fragments of
// m8n8k4 and the solve's column walks are bank-conflict free.  n not a
// multiple of 8 is padded exactly (identity diagonal, zero right-hand side).
#pragma once
#include <cuda_runtime.h>

#include "engine.cuh"

// L2 prefetch of the next problem's whole operands (cp.async.bulk.prefetch):
// measured off — it read the unused triangles too and the prefetched lines
// were partly evicted before use (DRAM traffic 1.4-2.1x the compulsory bytes),
// without a speed-up (profiles/r01_wave_traffic.txt)
#ifndef WAVE_PREFETCH
#define WAVE_PREFETCH 0
#endif
#ifndef WAVE_SOLVE
#define WAVE_SOLVE 1
#endif
namespace lagen {
namespace wave {

using eng::cp_async16;
using eng::cp_async_commit;
using eng::cp_async_wait;
using eng::dmma;
using eng::lane_id;

// element (r, c) of a swizzled 8x8 tile: 16-byte pairs stay together, rows
// 0/1 vs 2/3 (and 4/5 vs 6/7) swap column halves
__device__ __forceinline__ int sw(int r, int c) { return r * 8 + (c ^ ((r & 2) << 1)); }

template <int EQ, int N, int NW_, int PP_>
struct WPol {
  static_assert(EQ == 1 || EQ == 2, "wave engine: Lyapunov (1) or Sylvester (2)");
  static constexpr int T = (N + 7) / 8;
  static constexpr int NT = EQ == 2 ? T * T : T * (T + 1) / 2;  // unknown tiles
  static constexpr int NW = NW_;
  // tile q -> warp (q / BLK) % NW: blocks of BLK consecutive tiles of the
  // diagonal-major order per warp, so the diagonal-d solves land on few warps
  // with full 8-lane groups (fewer solve passes per step)
  static constexpr int BLK = 1;  // 4 measured slower (fewer warps carry the latency-bound solves)
  static constexpr int S = BLK * (((NT + BLK - 1) / BLK + NW - 1) / NW);  // accumulator slots per warp
  static constexpr int PP = PP_;
  static constexpr int NLT = T * (T + 1) / 2;
  static constexpr int NUT = EQ == 2 ? NLT : 0;
  // L, U (64 doubles per tile), publish (2 diagonals, PS doubles per tile)
  // and the L_II columns shifted for the solve (Lsh, 80 doubles per tile)
  static constexpr int PS = 68;  // 544-byte pitch: the 4 groups' tiles start in different banks
  static constexpr int TILES = NLT + NUT;
  static constexpr int PUBD = 2 * T * PS + T * 80;
  static constexpr int SCR = NW * 4 * 72;          // per-group pivot reciprocals (72: groups 1, 3 shift 8 banks)
  static constexpr int SLOT = TILES * 64 + PUBD + SCR + 2;  // doubles (+ flag)
  static constexpr size_t SMEM = (size_t)PP * SLOT * 8;
  static constexpr int THREADS = PP * NW * 32;
  static_assert(T <= 16, "n <= 128");
  static_assert(S <= 40, "accumulator slots per warp");
  static_assert((T + NW - 1) / NW <= 4, "at most 4 diagonal tiles per warp and step");
};

// case list over accumulator slots 0..39 (S <= 40), used as Duff's device
#define LAGEN_WAVE_SLOTS(X)                                                                                   \
  X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) X(18) \
  X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31) X(32) X(33) X(34) X(35)     \
  X(36) X(37) X(38) X(39)

// 1 / a without the division subroutine (whose call would make the compiler
// save the accumulator registers): rcp.approx + two Newton steps (~1 ulp)
__device__ __forceinline__ double recip(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ int ltidx(int I, int J) { return I * (I + 1) / 2 + J; }  // I >= J
__device__ __forceinline__ int utidx(int I, int J) { return J * (J + 1) / 2 + I; }  // I <= J

// tile q of the diagonal-major order (diagonals ascending, I ascending)
template <int EQ, int T>
__device__ __forceinline__ int tile_of(int q) {
  for (int d = 0; d <= 2 * T - 2; ++d) {
    const int i0 = d - T + 1 > 0 ? d - T + 1 : 0;
    const int i1 = EQ == 2 ? (d < T - 1 ? d : T - 1) : d / 2;
    const int m = i1 - i0 + 1;
    if (q < m) return ((i0 + q) << 4) | (d - i0 - q);
    q -= m;
  }
  return 0xff;
}

// rows x 16-byte pairs of an n x n row-major operand into the lower (PART 0)
// or upper (PART 1) tiles; pad units (outside n) get the identity
template <int N, int T, int PART, int G>
__device__ __forceinline__ void load_tri(double* tiles, const double* __restrict__ src, int rank) {
  constexpr int NP = 8 * T, HP = NP / 2;
  for (int u = rank; u < NP * HP; u += G) {
    const int r = u / HP, cp = u - r * HP;
    const int I = r >> 3, J = cp >> 2;
    if (PART == 0 ? J > I : J < I) continue;
    double* dst = tiles + (PART == 0 ? ltidx(I, J) : utidx(I, J)) * 64 + sw(r & 7, 2 * (cp & 3));
    const int c = 2 * cp;
    if (r < N && c < N) {
      cp_async16(dst, src + r * N + c);
    } else {
      *reinterpret_cast<double2*>(dst) = make_double2(r == c ? 1.0 : 0.0, r == c + 1 ? 1.0 : 0.0);
    }
  }
}

template <int EQ, int N, int NW, int PP>
__global__ void __launch_bounds__(WPol<EQ, N, NW, PP>::THREADS, 1)
    wave_kernel(const double* __restrict__ Lg, const double* __restrict__ Ug, const double* __restrict__ Cg,
                double* __restrict__ X, int* __restrict__ info, long long batch, int mode) {
  // mode (profiling only; results are wrong when set): bit 0 skips the
  // diagonal solves, bit 1 the bulk contributions, bit 2 the critical ones
  using P = WPol<EQ, N, NW, PP>;
  constexpr int T = P::T, S = P::S, G = NW * 32;
  constexpr long long NN = (long long)N * N;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int grp = warp / NW, w = warp % NW, rank = threadIdx.x % G;
  double* base = smem + (size_t)grp * P::SLOT;
  double* Lt = base;
  double* Ut = base + P::NLT * 64;
  double* pub = base + (P::NLT + P::NUT) * 64;
  constexpr int PS = P::PS;
  double* Lsh = pub + 2 * T * PS;
  double* scr = base + P::TILES * 64 + P::PUBD + w * 288 + (lane >> 3) * 72 + (lane & 7) * 8;
  int* flag = reinterpret_cast<int*>(base + P::TILES * 64 + P::PUBD + P::SCR);
  const int g = lane >> 2, t = lane & 3;
  const int oA0 = sw(g, t), oA1 = sw(g, t + 4), oB0 = sw(t, g), oB1 = sw(t + 4, g), oC = sw(g, 2 * t);
  auto gbar = [&]() {
    if constexpr (NW == 1) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(G) : "memory");
  };

  // this warp's tiles: slot s -> packed (I << 4 | J) of tile qof(s) of the
  // diagonal-major order; slots past NT (a suffix) are empty
  constexpr int BLK = P::BLK;
  auto qof = [&](int s) { return ((s / BLK) * NW + w) * BLK + s % BLK; };
  // number of this warp's tiles among q < x
  auto cnt = [&](int x) {
    const int B = x / BLK;
    return BLK * ((B - w + NW - 1) / NW) + ((B % NW == w) ? x % BLK : 0);
  };
  unsigned tab[(S + 3) / 4];
#pragma unroll
  for (int i = 0; i < (S + 3) / 4; ++i) tab[i] = 0u;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int q = qof(s);
    const unsigned ij = q < P::NT ? (unsigned)tile_of<EQ, T>(q) : 0u;
    tab[s >> 2] |= ij << (8 * (s & 3));
  }
  auto valid = [&](int s) { return qof(s) < P::NT; };
  auto tij = [&](int s) -> int { return (int)((tab[s >> 2] >> (8 * (s & 3))) & 0xff); };

  const long long stride = (long long)gridDim.x * PP;
  // slot-major problem order (as in chol_rows.cuh): a partial last round is
  // spread over every SM instead of filling the slots of a few
#ifndef LAGEN_WAVE_SPREAD
#define LAGEN_WAVE_SPREAD 1
#endif
  const long long first = LAGEN_WAVE_SPREAD ? (long long)grp * gridDim.x + blockIdx.x : (long long)blockIdx.x * PP + grp;
  for (long long prob = first; prob < batch; prob += stride) {
    const double* Lp = Lg + prob * NN;
    const double* Up = Ug + prob * NN;
    const double* Cp = Cg + prob * NN;
    // coefficients -> shared memory (cp.async), right-hand side -> registers
    load_tri<N, T, 0, G>(Lt, Lp, rank);
    if constexpr (EQ == 2) load_tri<N, T, 1, G>(Ut, Up, rank);
    cp_async_commit();
    if (rank == 0) {
      *flag = 0;
      const long long nxt = prob + stride;
      if (WAVE_PREFETCH && nxt < batch) {  // next problem's operands -> L2 while this one runs
        const unsigned bytes = (unsigned)(NN * 8);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Lg + nxt * NN), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Cg + nxt * NN), "r"(bytes) : "memory");
        if constexpr (EQ == 2)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Ug + nxt * NN), "r"(bytes) : "memory");
      }
    }
    double a0[S], a1[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      a0[s] = a1[s] = 0.0;
      if (!valid(s)) continue;
      const int ij = tij(s);
      const int I = ij >> 4, J = ij & 15;
      const int r = 8 * I + g, c = 8 * J + 2 * t;
      if (r < N && c < N) {
        if (EQ == 1 && I == J && r > c) {  // symmetric right-hand side: upper triangle only
          a0[s] = __ldg(Cp + (long long)c * N + r);
          a1[s] = r > c + 1 ? __ldg(Cp + (long long)(c + 1) * N + r) : __ldg(Cp + (long long)r * N + c + 1);
        } else {
          const double2 v = __ldg(reinterpret_cast<const double2*>(Cp + (long long)r * N + c));
          a0[s] = v.x;
          a1[s] = v.y;
        }
      }
    }
    cp_async_wait<0>();
    gbar();
    // Lsh[I][10 r + e] = L_II(r + e, r), e = 1..7 (0 below the tile): the solve
    // reads one column of the diagonal block per step as 4 16-byte loads; the
    // 80-byte row pitch puts the 8 lanes' rows on disjoint banks
    for (int u = rank; u < T * 64; u += G) {
      const int I = u >> 6, r = (u >> 3) & 7, e = u & 7;
      Lsh[I * 80 + r * 10 + e] = (e >= 1 && r + e < 8) ? Lt[ltidx(I, I) * 64 + sw(r + e, r)] : 0.0;
    }
    gbar();
    bool bad = false;

    int q0 = 0;  // tiles on diagonals < d
#pragma unroll 1
    for (int d = 0; d <= 2 * T - 2; ++d) {
      const int i0 = d - T + 1 > 0 ? d - T + 1 : 0;
      const int m = (EQ == 2 ? (d < T - 1 ? d : T - 1) : d / 2) - i0 + 1;  // tiles on diagonal d
      const int sc0 = cnt(q0), sc1 = cnt(q0 + m);  // this warp's slots of diagonal d
      const double* pv = pub + ((d + 1) & 1) * T * PS;  // diagonal d-1 (-X)
      double* pc = pub + (d & 1) * T * PS;              // diagonal d
      // contributions of diagonal d-1 into tile (I, J) (I + J >= d)
      auto contrib = [&](double& c0, double& c1, int I, int J) {
        if (J < d) {  // L_Ik X_kJ, k = d-1-J < I
          const int k = d - 1 - J;
          const double* A = Lt + ltidx(I, k) * 64;
          const double* B = pv + k * PS;
          dmma(c0, c1, A[oA0], B[oB0]);
          dmma(c0, c1, A[oA1], B[oB1]);
        }
        if (I < d) {  // X_Ik U_kJ, k = d-1-I < J
          const int k = d - 1 - I;
          if constexpr (EQ == 2) {
            const double* A = pv + I * PS;
            const double* B = Ut + utidx(k, J) * 64;
            dmma(c0, c1, A[oA0], B[oB0]);
            dmma(c0, c1, A[oA1], B[oB1]);
          } else {
            // X_Ik: upper tile (I, k) or the transpose of (k, I); U_kJ = L_Jk^T
            const double* A = pv + (I <= k ? I : k) * PS;
            const int o0 = I <= k ? oA0 : oB0, o1 = I <= k ? oA1 : oB1;
            const double* B = Lt + ltidx(J, k) * 64;
            dmma(c0, c1, A[o0], B[oA0]);
            dmma(c0, c1, A[o1], B[oA1]);
          }
        }
      };
      // (1) critical tiles of diagonal d: slot s <-> tile q = s NW + w,
      //     position q - q0 along the diagonal
      // (jump straight to slot sc0: a switch with fall-through over the
      // unrolled slots, no per-slot tests for the slots already solved)
#define LAGEN_WAVE_CRIT(k)                                                  \
  case k:                                                                   \
    if constexpr (k < S) {                                                  \
      if (k >= sc1) break;                                                  \
      const int I = i0 + qof(k) - q0, J = d - I;                            \
      contrib(a0[k], a1[k], I, J);                                          \
      *reinterpret_cast<double2*>(pc + I * PS + oC) = make_double2(a0[k], a1[k]); \
    }                                                                       \
    [[fallthrough]];
      if (!(mode & 4)) switch (sc0) { LAGEN_WAVE_SLOTS(LAGEN_WAVE_CRIT) default: break; }
#undef LAGEN_WAVE_CRIT
      __syncwarp();
      // (2) solve: group q of 8 lanes takes the q-th of them; lane c owns column c
      const int ncrit = sc1 - sc0;
      if (WAVE_SOLVE && ncrit > 0 && !(mode & 1)) {
        const int qg = lane >> 3, c = lane & 7;
        const bool live = qg < ncrit;
        const int I = i0 + qof(sc0 + (live ? qg : 0)) - q0, J = d - I;
        double* Pt = pc + I * PS;
        const double* Ld = Lt + ltidx(I, I) * 64;
        const double* Ls = Lsh + I * 80;
        // U_JJ (k, c):  sylvester U tile, lyapunov L_JJ^T
        const double* Ud = EQ == 2 ? Ut + utidx(J, J) * 64 : Lt + ltidx(J, J) * 64;
        auto uat = [&](int k) -> double { return EQ == 2 ? Ud[sw(k, c)] : Ud[sw(c, k)]; };
        // y: column c of the right-hand side with row r = s - c handled at step
        // s; y and the history h of computed values are circular buffers of 8
        // (slot s & 7), so the step loop runs as 2 x 8 unrolled steps with
        // static register indices and bounded live state.  y[s] is loaded
        // when slot s & 7 frees up (step s - 8); rows outside 0..7 are 0.
        auto yload = [&](int s) -> double {
          const int r = s - c;
          return (r >= 0 && r < 8) ? Pt[sw(r < 0 ? 0 : (r > 7 ? 7 : r), c)] : 0.0;
        };
        double y[8], h[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          y[s] = yload(s);
          h[s] = 0.0;
        }
        // setup with independent loads issued first (the compiler must keep a
        // shared load after any earlier shared store, so load -> compute ->
        // store order is explicit; divergent selects instead of branches)
        double uc[8], dg[8];
        uc[0] = 0.0;
#pragma unroll
        for (int j = 1; j < 8; ++j) uc[j] = uat(c >= j ? c - j : 0);
        const double ucc = uat(c);
#pragma unroll
        for (int r = 0; r < 8; ++r) dg[r] = Ld[sw(r, r)];
#pragma unroll
        for (int j = 1; j < 8; ++j) uc[j] = j <= c ? uc[j] : 0.0;
#pragma unroll
        for (int r = 0; r < 8; ++r) dg[r] = recip(dg[r] + ucc);
#pragma unroll
        for (int r = 0; r < 8; ++r) scr[r] = dg[r];
        __syncwarp();
        // per-step coefficients (pivot reciprocal, column r of L_II below the
        // diagonal), loaded one step ahead so no load waits behind a store
        struct Co {
          double piv;
          double2 a, b, cc, d;
        };
        auto coload = [&](int s) -> Co {
          const int r = s - c;
          const int rc = r < 0 ? 0 : (r > 7 ? 7 : r);
          const double2* lc = reinterpret_cast<const double2*>(Ls + 10 * rc);
          Co o;
          o.piv = (r >= 0 && r < 8) ? scr[rc] : 0.0;
          o.a = lc[0];
          o.b = lc[1];
          o.cc = lc[2];
          o.d = lc[3];
          return o;
        };
        Co cur = coload(0);
        // one wavefront step; the dependence on the previous step is kept to
        // shfl(x(r, c-1)) -> FMA -> MUL and push(x(r-1, c)) -> ADD -> FMA -> MUL:
        // contributions of values >= 2 steps old are summed off that chain
        auto step = [&](int s, int u) {
          const int r = s - c;
          const bool act = r >= 0 && r < 8;
          const Co nxt = coload(s + 1 <= 14 ? s + 1 : 14);
          const double ynew = yload(s + 8);
          // row contributions: x(r, c - j) from lane c - j, computed j steps ago
          double t0 = 0.0, t1 = 0.0;
#pragma unroll
          for (int j = 2; j < 8; ++j) {
            const int src = (lane & ~7) | (c >= j ? c - j : c);
            const double xv = __shfl_sync(0xffffffffu, h[(u - j) & 7], src);
            if (j & 1) t1 = fma(xv, uc[j], t1);
            else t0 = fma(xv, uc[j], t0);
          }
          const double x1 = __shfl_sync(0xffffffffu, h[(u - 1) & 7], (lane & ~7) | (c >= 1 ? c - 1 : c));
          double v = y[u] - (t0 + t1);
          v = fma(-x1, uc[1], v);
          const double x = v * cur.piv;
          h[u] = x;
          // own column: rows r + e take L(r + e, r) x (row r + 1 first: next step)
          const double coef[8] = {0.0, cur.a.y, cur.b.x, cur.b.y, cur.cc.x, cur.cc.y, cur.d.x, cur.d.y};
#pragma unroll
          for (int e = 1; e < 8; ++e) y[(u + e) & 7] = fma(-coef[e], x, y[(u + e) & 7]);
          y[u] = ynew;
          if (act && live) Pt[sw(r, c)] = -x;
          cur = nxt;
        };
#pragma unroll
        for (int u = 0; u < 8; ++u) step(u, u);
#pragma unroll
        for (int u = 0; u < 7; ++u) step(8 + u, u);
        __syncwarp();
        if (EQ == 1 && live && I == J) {  // symmetric diagonal tile: lower := mirror of upper
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (r > c) Pt[sw(r, c)] = Pt[sw(c, r)];  // upper entries are not written here
        }
        __syncwarp();
        // stream X (= -published) to HBM: lane c writes row c of the tile
        if (live) {
          const int r = 8 * I + c;
          double* Xp = X + prob * NN;
#pragma unroll
          for (int mm = 0; mm < 4; ++mm) {
            const int col = 8 * J + 2 * mm;
            if (r < N && col < N) {
              const double2 v = *reinterpret_cast<const double2*>(Pt + sw(c, 2 * mm));
              bad = bad || !isfinite(v.x) || !isfinite(v.y);
              __stcs(reinterpret_cast<double2*>(Xp + (long long)r * N + col), make_double2(-v.x, -v.y));
            }
          }
          if (EQ == 1 && I != J) {  // mirror tile (J, I): its row c is column c of this tile
            const int r2 = 8 * J + c;
#pragma unroll
            for (int mm = 0; mm < 4; ++mm) {
              const int col = 8 * I + 2 * mm;
              if (r2 < N && col < N)
                __stcs(reinterpret_cast<double2*>(Xp + (long long)r2 * N + col),
                       make_double2(-Pt[sw(2 * mm, c)], -Pt[sw(2 * mm + 1, c)]));
            }
          }
        }
      }
      // (3) bulk: every later tile takes diagonal d-1's contributions
      if (d > 0 && !(mode & 2)) {
        // opaque per step: keeps the compiler from hoisting S decoded tile
        // coordinates / addresses out of the loop (register pressure)
#pragma unroll
        for (int i = 0; i < (S + 3) / 4; ++i) asm volatile("mov.b32 %0, %0;" : "+r"(tab[i]));
#define LAGEN_WAVE_BULK(k)                                  \
  case k:                                                   \
    if constexpr (k < S) {                                  \
      if (!valid(k)) break;                                 \
      const int ij = tij(k);                                \
      contrib(a0[k], a1[k], ij >> 4, ij & 15);              \
    }                                                       \
    [[fallthrough]];
        switch (sc1) { LAGEN_WAVE_SLOTS(LAGEN_WAVE_BULK) default: break; }
#undef LAGEN_WAVE_BULK
      }
      q0 += m;
      gbar();
    }
    if (bad) *flag = -1;
    gbar();
    if (rank == 0 && info) info[prob] = *flag;
  }
}

}  // namespace wave
}  // namespace lagen
