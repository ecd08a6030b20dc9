// engine.cuh — the "warp engine": one warp per problem, the whole problem
// resident in shared memory in a 4x4-tiled, XOR-swizzled fp64 layout, the
// variant's statement list compiled in (template type list generated from
// the reference's enumerate_algorithms() output, variants_ct.cuh), GEMM
// updates on the FP64 tensor path (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4),
// warp-synchronous everything else (no CTA barriers), and the next problem
// prefetched with cp.async while the current one is solved.
//
// Semantics per statement kind follow the reference block kernels
// (kernels.py:16-130) exactly as solver.cuh documents; only the schedule and
// summation order differ (parity <= 1e-10, BASELINE north_star).  Pivots use
// x_ii = a_ii * rsqrt(a_ii), x_ij = a_ij * rsqrt(a_ii) and the triangular
// solves multiply by precomputed reciprocals (<= 2 ulp from sqrt / divide).
//
// Tile layout (per matrix): n x n split into T x T tiles of 4x4 doubles
// (128 B = one full bank sweep).  Element (r, c) of tile (R, C) lives at
//   tile_index(R, C) * 16 + ((chunk ^ ((R ^ C) & 7)) << 1 | (c & 1)),
//   chunk = (r & 3) * 2 + (c & 3) / 2   (16-byte chunk inside the tile)
// DMMA fragments (16 lanes per tile, either orientation), lane-per-row,
// lane-per-column and lane-per-tile walks are all conflict-free, and 16-byte
// cp.async chunks keep (c, c+1) pairs adjacent.
// tile_index: DENSE R*T+C; UPPER (C >= R) packed rows; LOWER (C <= R).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

#include "lagen_b200.h"

namespace lagen {
namespace eng {

enum { DENSE = 0, UPPER = 1, LOWER = 2 };
enum { K_GEMM = 0, K_CHOL = 1, K_TRSM = 2, K_SYLV = 3, K_LYAP = 4 };

__device__ __forceinline__ int swz(int r, int c, int key) {
  return (((((r & 3) << 1) | ((c & 3) >> 1)) ^ key) << 1) | (c & 1);
}

// offset inside a tile whose base (tile_index * 16) and key ((R ^ C) & 7) are known
__device__ __forceinline__ int tile_off(int tbase, int key, int r, int c) {
  return tbase + ((((((r & 3) << 1) | ((c & 3) >> 1)) ^ key) & 7) << 1) + (c & 1);
}

template <int T, int LY>
struct TM {
  static constexpr bool GLOBAL = false;
  static constexpr int LDN = 0;
  static constexpr int TILES = LY == DENSE ? T * T : T * (T + 1) / 2;
  static constexpr int DOUBLES = TILES * 16;
  __device__ static __forceinline__ int tidx(int R, int C) {
    if constexpr (LY == DENSE) return R * T + C;
    else if constexpr (LY == UPPER) return R * T - ((R * (R - 1)) >> 1) + (C - R);
    else return ((R * (R + 1)) >> 1) + C;
  }
  // tile-index step when R -> R + 1 at fixed C
  __device__ static __forceinline__ int dR(int R) {
    if constexpr (LY == DENSE) return T;
    else if constexpr (LY == UPPER) return T - R - 1;
    else return R + 1;
  }
  __device__ static __forceinline__ int off(int r, int c) {
    const int R = r >> 2, C = c >> 2;
    return (tidx(R, C) << 4) + swz(r, c, (R ^ C) & 7);
  }
};

// Row-major global-memory operand (coefficients that do not fit on chip).
template <int N>
struct GM {
  static constexpr bool GLOBAL = true;
  static constexpr int LDN = N;
  static constexpr int TILES = 0;
  static constexpr int DOUBLES = 0;
  __device__ static __forceinline__ int off(int r, int c) { return r * N + c; }
};

// k-walker: address of element (r, c) advanced by 4 rows (ADV_R) or 4
// columns per step, with O(1) integer work per step.
template <class M, bool ADV_R>
struct KW {
  int tp, R, C, e;
  __device__ __forceinline__ void init(int r, int c) {
    R = r >> 2;
    C = c >> 2;
    tp = M::tidx(R, C) << 4;
    e = (((r & 3) << 1) | ((c & 3) >> 1)) | ((c & 1) << 8);
  }
  __device__ __forceinline__ int addr() const { return tp + ((((e & 7) ^ ((R ^ C) & 7)) << 1) | (e >> 8)); }
  __device__ __forceinline__ void step() {
    if constexpr (ADV_R) {
      tp += M::dR(R) << 4;
      ++R;
    } else {
      tp += 16;
      ++C;
    }
  }
};
template <int N, bool ADV_R>
struct KW<GM<N>, ADV_R> {
  int tp;
  __device__ __forceinline__ void init(int r, int c) { tp = r * N + c; }
  __device__ __forceinline__ int addr() const { return tp; }
  __device__ __forceinline__ void step() { tp += ADV_R ? 4 * N : 4; }
};

// A block view over a tiled matrix: element (i, j) of the view.
// TR: transposed view; SY: symmetric diagonal block stored as its upper
// triangle (the reference's gather, verify.py:254-261).
template <class M, bool TR, bool SY>
struct TV {
  using Mat = M;
  static constexpr bool tr = TR, sy = SY;
  double* base;
  int r0, c0;
  __device__ __forceinline__ int off(int i, int j) const {
    int r = TR ? r0 + j : r0 + i;
    int c = TR ? c0 + i : c0 + j;
    if (SY) {
      const int a = min(r, c), b = max(r, c);
      r = a;
      c = b;
    }
    return M::off(r, c);
  }
  __device__ __forceinline__ double at(int i, int j) const { return base[off(i, j)]; }
  __device__ __forceinline__ double& ref(int i, int j) const { return base[off(i, j)]; }
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// In-group index of the warp that carries a problem group's serial chain
// (CHOL leaf): groups of WG consecutive warps would otherwise put every
// group's leaf warp on the same SM sub-partition (warp % 4), where the
// leaves' FP64 / MUFU work queues behind each other; this picks a distinct
// sub-partition per group where the group size allows.
__host__ __device__ constexpr int lead_warp(int g, int WG) {
  return WG == 4 ? g % 4 : WG == 2 ? (g / 2) % 2 : WG == 3 ? (2 * g) % 4 : 0;
}

// A problem is owned by a group of WG warps (G = 32 * WG threads).
struct Grp {
  int rank;     // 0 .. G-1
  int wig;      // warp in group
  int id;       // group index in the CTA (named barrier id - 1)
  double* rsb;  // per-group: reciprocal pivots of the last CHOL leaf [0, 16) and
                //            its factor, row-major B x B, at [16, 16 + B*B)
  double* scr;  // per-group split-K scratch ((WG - 1) * 256 doubles)
  int subbar;   // named barrier of warps 1 .. WG-1 (0: none)
  unsigned long long* prof;  // cycle accounting buffer (profiling launches only)
};
// The warps / threads executing one statement: the whole group, or (when a
// CHOL leaf occupies warp 0 in the same dependency level) warps 1 .. WG-1.
struct Sub {
  int w, nw;        // warp index within the subset, subset size (warps)
  int rank, nthr;   // thread index within the subset, subset size (threads)
  bool full;        // whole group (group barriers allowed)
};

template <int WG>
__device__ __forceinline__ void gsync(const Grp& g) {
  if constexpr (WG == 1) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(g.id + 1), "r"(WG * 32) : "memory");
}

// Operand streams along k for the DMMA loop.  A: element (i, k), B: (k, j).
// Symmetric gathers (Lyapunov X_00 / X_11) pick, per lane and step, between
// the upper element and its mirror.
template <class AV>
struct AStream {
  KW<typename AV::Mat, AV::tr> w;
  KW<typename AV::Mat, !AV::tr> wm;  // mirror walker (SY only)
  int i_abs, k_abs;
  __device__ __forceinline__ void init(const AV& v, int i, int kofs = 0) {
    const int t = (lane_id() & 3) + kofs;
    if constexpr (AV::sy) {
      i_abs = v.r0 + i;
      k_abs = v.c0 + t;
      w.init(v.r0 + i, v.c0 + t);   // upper element (i, k): advance C
      wm.init(v.c0 + t, v.r0 + i);  // mirror (k, i): advance R
    } else if constexpr (AV::tr) {
      w.init(v.r0 + t, v.c0 + i);
    } else {
      w.init(v.r0 + i, v.c0 + t);
    }
  }
  __device__ __forceinline__ double load(const double* base) const {
    if constexpr (AV::sy) return base[(i_abs <= k_abs) ? w.addr() : wm.addr()];
    else return base[w.addr()];
  }
  __device__ __forceinline__ void step() {
    w.step();
    if constexpr (AV::sy) {
      wm.step();
      k_abs += 4;
    }
  }
};

template <class BV>
struct BStream {
  KW<typename BV::Mat, !BV::tr> w;
  KW<typename BV::Mat, BV::tr> wm;
  int j_abs, k_abs;
  __device__ __forceinline__ void init(const BV& v, int j, int kofs = 0) {
    const int t = (lane_id() & 3) + kofs;
    if constexpr (BV::sy) {
      j_abs = v.c0 + j;
      k_abs = v.r0 + t;
      w.init(v.r0 + t, v.c0 + j);   // upper element (k, j): advance R
      wm.init(v.c0 + j, v.r0 + t);  // mirror (j, k): advance C
    } else if constexpr (BV::tr) {
      w.init(v.r0 + j, v.c0 + t);
    } else {
      w.init(v.r0 + t, v.c0 + j);
    }
  }
  __device__ __forceinline__ double load(const double* base) const {
    if constexpr (BV::sy) return base[(k_abs <= j_abs) ? w.addr() : wm.addr()];
    else return base[w.addr()];
  }
  __device__ __forceinline__ void step() {
    w.step();
    if constexpr (BV::sy) {
      wm.step();
      k_abs += 4;
    }
  }
};

// ----------------------------------------------------------------------------
// GEMM_update on the DMMA path: O(m x q) += sgn * A(m x p) B(p x q).
// 16x16 warp blocks of 2x2 m8n8k4 tiles; m, p, q multiples of 4; partial
// 8-row/col tiles read clamped (valid) rows and discard them on write.
// UP: upper target (only i <= j written; tiles strictly below skipped).
// ----------------------------------------------------------------------------
// m <= 8 (block-row updates of the left-looking variants): 8 x 32 warp
// blocks, one A fragment feeds four independent DMMA accumulators per k-step.
// With fewer blocks than warps (late iterations: long k, few columns) the k
// range is split across the warps and the partial accumulators are reduced
// in fixed order through the group's scratch (deterministic).
template <bool UP, class OV, class AV, class BV>
__device__ __forceinline__ void row8_block(const AV& A, const BV& Bm, int m, int q, int j0, int kb, int ke,
                                           bool v[4], double c0[4], double c1[4]) {
  const int lane = lane_id();
  const int g = lane >> 2;
  const int ra = (g < m) ? g : (g & 3);
  int cb[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int jt = j0 + 8 * u;
    v[u] = jt < q && !(UP && 0 >= jt + 8);
    cb[u] = (jt + g < q) ? jt + g : (jt < q ? jt + (g & 3) : j0 + (g & 3));
  }
  AStream<AV> as;
  BStream<BV> bs[4];
  as.init(A, ra, kb);
#pragma unroll
  for (int u = 0; u < 4; ++u) bs[u].init(Bm, cb[u], kb);
  // two accumulator sets (even / odd k-steps): eight independent DMMA
  // chains per warp hide the DMMA latency
  double e0[4] = {0, 0, 0, 0}, e1[4] = {0, 0, 0, 0};
#pragma unroll
  for (int u = 0; u < 4; ++u) c0[u] = c1[u] = 0.0;
  int k0 = kb;
  for (; k0 + 8 <= ke; k0 += 8) {
    const double a = as.load(A.base);
    double bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) bv[u] = v[u] ? bs[u].load(Bm.base) : 0.0;
    as.step();
#pragma unroll
    for (int u = 0; u < 4; ++u) bs[u].step();
    const double a2 = as.load(A.base);
    double bw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) bw[u] = v[u] ? bs[u].load(Bm.base) : 0.0;
    as.step();
#pragma unroll
    for (int u = 0; u < 4; ++u) bs[u].step();
    // unconditional MMAs (invalid tiles multiply zeros): a predicated
    // mma.sync costs a WARPSYNC per instruction
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(c0[u], c1[u], a, bv[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(e0[u], e1[u], a2, bw[u]);
  }
  if (k0 < ke) {
    const double a = as.load(A.base);
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(c0[u], c1[u], a, v[u] ? bs[u].load(Bm.base) : 0.0);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    c0[u] += e0[u];
    c1[u] += e1[u];
  }
}

template <bool UP, class OV>
__device__ __forceinline__ void row8_write(const OV& O, int m, int q, int j0, double sgn, const bool v[4],
                                           const double c0[4], const double c1[4]) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (!v[u]) continue;
    const int i = g, j = j0 + 8 * u + 2 * t;
    if (i < m && j < q && (!UP || i <= j)) {
      double& o0 = O.ref(i, j);
      o0 = fma(sgn, c0[u], o0);
    }
    if (i < m && j + 1 < q && (!UP || i <= j + 1)) {
      double& o1 = O.ref(i, j + 1);
      o1 = fma(sgn, c1[u], o1);
    }
  }
}

template <bool UP, int WG, class OV, class AV, class BV>
__device__ __forceinline__ void gemm_row8(const OV& O, const AV& A, const BV& Bm, int m, int p, int q, double sgn,
                                          const Grp& gr, const Sub& sb) {
  const int nblk = (q + 31) >> 5;
  // k-split factor: idle warps take slices of k (needs scratch and a barrier
  // covering exactly the executing warps)
  const bool can_split = WG > 1 && gr.scr != nullptr && (sb.full || gr.subbar != 0);
  const int ks = (can_split && nblk < sb.nw) ? min(sb.nw / nblk, p / 16) : 1;
  if (ks <= 1) {
    for (int bk = sb.w; bk < nblk; bk += sb.nw) {
      bool v[4];
      double c0[4], c1[4];
      row8_block<UP, OV>(A, Bm, m, q, bk << 5, 0, p, v, c0, c1);
      row8_write<UP>(O, m, q, bk << 5, sgn, v, c0, c1);
    }
    return;
  }
  auto bar = [&]() {
    if (sb.full) gsync<WG>(gr);
    else asm volatile("bar.sync %0, %1;" ::"r"(gr.subbar), "r"(sb.nthr) : "memory");
  };
  const int item = sb.w, blk = item % nblk, sl = item / nblk;  // slice sl of block blk
  const bool active = item < nblk * ks;
  bool v[4];
  double c0[4], c1[4];
  const int lane = lane_id();
  if (active) {
    const int ksteps = p >> 2;
    const int kb = 4 * ((ksteps * sl) / ks), ke = 4 * ((ksteps * (sl + 1)) / ks);
    row8_block<UP, OV>(A, Bm, m, q, blk << 5, kb, ke, v, c0, c1);
    if (sl > 0) {
      double* sp = gr.scr + ((sl - 1) * nblk + blk) * 256 + lane * 8;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sp[2 * u] = c0[u];
        sp[2 * u + 1] = c1[u];
      }
    }
  }
  bar();
  if (active && sl == 0) {
    for (int s2 = 1; s2 < ks; ++s2) {
      const double* sp = gr.scr + ((s2 - 1) * nblk + blk) * 256 + lane * 8;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c0[u] += sp[2 * u];
        c1[u] += sp[2 * u + 1];
      }
    }
    row8_write<UP>(O, m, q, blk << 5, sgn, v, c0, c1);
  }
  bar();  // scratch free for the next split GEMM of this (sub-)group
}

// single 8x8 output tile (m, q <= 8) on one warp: four independent
// accumulator chains over the k-steps (latency-bound otherwise)
template <bool UP, class OV, class AV, class BV>
__device__ __forceinline__ void gemm_tile8(const OV& O, const AV& A, const BV& Bm, int m, int p, int q, double sgn) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int ra = (g < m) ? g : (g & 3);
  const int cb = (g < q) ? g : (g & 3);
  AStream<AV> as;
  BStream<BV> bs;
  as.init(A, ra, 0);
  bs.init(Bm, cb, 0);
  double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
  int k0 = 0;
  for (; k0 + 16 <= p; k0 += 16) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = as.load(A.base);
      b[u] = bs.load(Bm.base);
      as.step();
      bs.step();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(c0[u], c1[u], a[u], b[u]);
  }
  for (int u = 0; k0 < p; k0 += 4, ++u) {
    const double a = as.load(A.base), b = bs.load(Bm.base);
    as.step();
    bs.step();
    dmma(c0[0], c1[0], a, b);
  }
  const double x0 = (c0[0] + c0[1]) + (c0[2] + c0[3]);
  const double x1 = (c1[0] + c1[1]) + (c1[2] + c1[3]);
  const int i = g, j = 2 * t;
  if (i < m && j < q && (!UP || i <= j)) {
    double& o0 = O.ref(i, j);
    o0 = fma(sgn, x0, o0);
  }
  if (i < m && j + 1 < q && (!UP || i <= j + 1)) {
    double& o1 = O.ref(i, j + 1);
    o1 = fma(sgn, x1, o1);
  }
}

template <bool UP, int WG, class OV, class AV, class BV>
__device__ __forceinline__ void gemm(const OV& O, const AV& A, const BV& Bm, int m, int p, int q, double sgn,
                                     const Grp& gr, const Sub& sb) {
  if (m <= 8 && q <= 8 && !(sb.full && WG > 1)) {
    if (sb.w == 0) gemm_tile8<UP>(O, A, Bm, m, p, q, sgn);
    return;
  }
  if (m <= 8 && q > 8) {
    gemm_row8<UP, WG>(O, A, Bm, m, p, q, sgn, gr, sb);
    return;
  }
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int nbj = (q + 15) >> 4;
  const int nblk = ((m + 15) >> 4) * nbj;
  // a single output block and idle warps: split the k loop over the group
  // and reduce the partial accumulators through shared memory (fixed order)
  const bool splitk = (WG > 1) && sb.full && (nblk == 1) && (p >= 16 * WG) && (gr.scr != nullptr);
  const int nks = p >> 2;
  for (int bk = splitk ? 0 : sb.w; bk < nblk; bk += splitk ? 1 : sb.nw) {
    {
      const int i0 = (bk / nbj) << 4, j0 = (bk % nbj) << 4;
      if (UP && i0 >= j0 + 16) continue;
      const bool vi1 = i0 + 8 < m, vj1 = j0 + 8 < q;
      const bool v00 = !(UP && i0 >= j0 + 8);
      const bool v01 = vj1;
      const bool v10 = vi1 && !(UP && i0 + 8 >= j0 + 8);
      const bool v11 = vi1 && vj1 && !(UP && i0 + 8 >= j0 + 16);
      const int ra0 = i0 + ((i0 + g < m) ? g : (g & 3));
      const int ra1 = vi1 ? i0 + 8 + ((i0 + 8 + g < m) ? g : (g & 3)) : ra0;
      const int cb0 = j0 + ((j0 + g < q) ? g : (g & 3));
      const int cb1 = vj1 ? j0 + 8 + ((j0 + 8 + g < q) ? g : (g & 3)) : cb0;
      const int ks0 = splitk ? (nks * gr.wig) / WG : 0;
      const int ks1 = splitk ? (nks * (gr.wig + 1)) / WG : nks;
      AStream<AV> a0s, a1s;
      BStream<BV> b0s, b1s;
      a0s.init(A, ra0, 4 * ks0);
      a1s.init(A, ra1, 4 * ks0);
      b0s.init(Bm, cb0, 4 * ks0);
      b1s.init(Bm, cb1, 4 * ks0);
      double c00a = 0, c00b = 0, c01a = 0, c01b = 0, c10a = 0, c10b = 0, c11a = 0, c11b = 0;
      for (int ks = ks0; ks < ks1; ++ks) {
        const double a0 = a0s.load(A.base);
        const double b0 = b0s.load(Bm.base);
        const double a1 = a1s.load(A.base);
        const double b1 = b1s.load(Bm.base);
        // unconditional (clamped operands are finite; invalid tiles are
        // discarded at write-back): no WARPSYNC per predicated mma.sync
        dmma(c00a, c00b, a0, b0);
        dmma(c01a, c01b, a0, b1);
        dmma(c10a, c10b, a1, b0);
        dmma(c11a, c11b, a1, b1);
        a0s.step();
        a1s.step();
        b0s.step();
        b1s.step();
      }
      if (splitk) {
        double* sp = gr.scr + (gr.wig - 1) * 256 + lane * 8;
        if (gr.wig > 0) {
          sp[0] = c00a; sp[1] = c00b; sp[2] = c01a; sp[3] = c01b;
          sp[4] = c10a; sp[5] = c10b; sp[6] = c11a; sp[7] = c11b;
        }
        gsync<WG>(gr);
        if (gr.wig != 0) continue;
#pragma unroll
        for (int w = 1; w < WG; ++w) {
          const double* q8 = gr.scr + (w - 1) * 256 + lane * 8;
          c00a += q8[0]; c00b += q8[1]; c01a += q8[2]; c01b += q8[3];
          c10a += q8[4]; c10b += q8[5]; c11a += q8[6]; c11b += q8[7];
        }
      }
      auto wb = [&](int ib, int jb, double x0, double x1) {
        const int i = ib + g, j = jb + 2 * t;
        if (i < m && j < q && (!UP || i <= j)) {
          double& o0 = O.ref(i, j);
          o0 = fma(sgn, x0, o0);
        }
        if (i < m && j + 1 < q && (!UP || i <= j + 1)) {
          double& o1 = O.ref(i, j + 1);
          o1 = fma(sgn, x1, o1);
        }
      };
      if (v00) wb(i0, j0, c00a, c00b);
      if (v01) wb(i0, j0 + 8, c01a, c01b);
      if (v10) wb(i0 + 8, j0, c10a, c10b);
      if (v11) wb(i0 + 8, j0 + 8, c11a, c11b);
    }
  }
}

// ----------------------------------------------------------------------------
// TRSM_left_transposed: T W := W, T logically lower (m x m)  [kernels.py:47-60]
// ----------------------------------------------------------------------------
// general m (Cholesky v0: coefficient X_00^T, m = kb): lanes own columns.
template <int WG, class TVt, class WV>
__device__ __forceinline__ void trsm(const TVt& Tm, const WV& W, int m, int q, const Grp& gr, const Sub& sb) {
  for (int j = sb.rank; j < q; j += sb.nthr) {
    for (int i = 0; i < m; ++i) {
      double s = W.at(i, j);
      for (int l = 0; l < i; ++l) s = fma(-Tm.at(i, l), W.at(l, j), s);
      W.ref(i, j) = s / Tm.at(i, i);
    }
  }
}

// compile-time m = B <= 16: column in registers, reciprocal pivots.
template <int B, int WG, class TVt, class WV>
__device__ __forceinline__ void trsm_b(const TVt& Tm, const WV& W, int q, const Grp& gr, const Sub& sb) {
  if (sb.rank >= q) return;
  using M = typename WV::Mat;
  if constexpr (B <= 8 && !WV::tr && !WV::sy) {
    // coefficient = factor of this iteration's CHOL leaf (rsb: reciprocal
    // pivots, then the factor row-major): T(i, l) = X(l, i) = fac[l][i]
    const double* fac = gr.rsb + 16;
    const int R0 = W.r0 >> 2;
    for (int j = sb.rank; j < q; j += sb.nthr) {
      const int c = W.c0 + j, C = c >> 2;
      int tb[B / 4], ky[B / 4];
#pragma unroll
      for (int i = 0; i < B / 4; ++i) {
        tb[i] = M::tidx(R0 + i, C) << 4;
        ky[i] = ((R0 + i) ^ C) & 7;
      }
      double w[B];
#pragma unroll
      for (int i = 0; i < B; ++i) w[i] = W.base[tile_off(tb[i / 4], ky[i / 4], i, c)];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        double v = w[i];
#pragma unroll
        for (int l = 0; l < i; ++l) v = fma(-fac[l * B + i], w[l], v);
        w[i] = v * gr.rsb[i];
      }
#pragma unroll
      for (int i = 0; i < B; ++i) W.base[tile_off(tb[i / 4], ky[i / 4], i, c)] = w[i];
    }
  } else {
    double rd[B];
#pragma unroll
    for (int i = 0; i < B; ++i) rd[i] = 1.0 / Tm.at(i, i);
    for (int j = sb.rank; j < q; j += sb.nthr) {
      double w[B];
#pragma unroll
      for (int i = 0; i < B; ++i) w[i] = W.at(i, j);
#pragma unroll
      for (int i = 0; i < B; ++i) {
        double v = w[i];
#pragma unroll
        for (int l = 0; l < i; ++l) v = fma(-Tm.at(i, l), w[l], v);
        w[i] = v * rd[i];
      }
#pragma unroll
      for (int i = 0; i < B; ++i) W.ref(i, j) = w[i];
    }
  }
}

// ----------------------------------------------------------------------------
// CHOL leaf (B x B upper, in place) [kernels.py:79-97]: lane j < B owns
// column j in registers; pivots and row entries travel by shuffle.
// ----------------------------------------------------------------------------
template <int B, class XV>
__device__ __forceinline__ void chol_leaf(const XV& W, int base, int* flag) {
  const int lane = lane_id();
  const int j = lane < B ? lane : B - 1;
  double col[B];
#pragma unroll
  for (int r = 0; r < B; ++r) col[r] = (r <= j) ? W.at(r, j) : 0.0;
#pragma unroll
  for (int i = 0; i < B; ++i) {
    const double piv = __shfl_sync(0xffffffffu, col[i], i);
    if (lane == 0 && piv <= 0.0 && *flag == 0) *flag = base + i + 1;
    const double rs = rsqrt(piv);
    if (j == i) col[i] = piv * rs;
    else if (j > i) col[i] = col[i] * rs;
#pragma unroll
    for (int r = i + 1; r < B; ++r) {
      const double xir = __shfl_sync(0xffffffffu, col[i], r);
      if (j >= r) col[r] = fma(-xir, col[i], col[r]);
    }
  }
  if (lane < B) {
#pragma unroll
    for (int r = 0; r < B; ++r)
      if (r <= lane) W.ref(r, lane) = col[r];
  }
}

// B <= 8: every lane of the warp factors the B x B block redundantly in
// registers (no shuffles on the pivot chain); lane j < B writes column j back
// and the reciprocal pivots 1/x_ii = rsqrt(a_ii) go to rsb for the TRSM.
template <int B, class XV>
__device__ __forceinline__ void chol_leaf_reg(const XV& W, int base, int* flag, double* rsb) {
  using M = typename XV::Mat;
  constexpr int TB = B / 4;
  const int lane = lane_id();
  // tile bases / keys of the diagonal block (r0 == c0, multiple of 4)
  const int K = W.r0 >> 2;
  int tb[TB][TB], ky[TB][TB];
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int j = i; j < TB; ++j) {
      tb[i][j] = M::tidx(K + i, K + j) << 4;
      ky[i][j] = ((K + i) ^ (K + j)) & 7;
    }
  // whole tiles as 16-byte chunks (uniform addresses -> broadcast loads)
  double t[B][B];
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int j = i; j < TB; ++j)
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const double2 v = *reinterpret_cast<const double2*>(W.base + tb[i][j] + (((ch ^ ky[i][j]) & 7) << 1));
        const int r = 4 * i + (ch >> 1), c = 4 * j + 2 * (ch & 1);
        t[r][c] = v.x;
        t[r][c + 1] = v.y;
      }
  double rs[B];
  bool bad = false;
  int badi = 0;
#pragma unroll
  for (int i = 0; i < B; ++i) {
    const double piv = t[i][i];
    if (!bad && piv <= 0.0) {
      bad = true;
      badi = i;
    }
    rs[i] = rsqrt(piv);
    t[i][i] = piv * rs[i];
#pragma unroll
    for (int c = i + 1; c < B; ++c) t[i][c] *= rs[i];
#pragma unroll
    for (int r = i + 1; r < B; ++r)
#pragma unroll
      for (int c = r; c < B; ++c) t[r][c] = fma(-t[i][r], t[i][c], t[r][c]);
  }
  if (lane == 0 && bad && *flag == 0) *flag = base + badi + 1;
  // lane r < B takes row r of the (lane-uniform) factor with selects (no
  // branches) and stores it: into the tiles (upper part), the row-major
  // factor and the reciprocal pivot for this iteration's TRSM — B lanes store
  // in parallel instead of one lane storing everything
  double row[B];
  double rsr = 0.0;
#pragma unroll
  for (int c = 0; c < B; ++c) row[c] = 0.0;
#pragma unroll
  for (int r = 0; r < B; ++r) {
    const bool me = (lane == r);
#pragma unroll
    for (int c = r; c < B; ++c) row[c] = me ? t[r][c] : row[c];
    rsr = me ? rs[r] : rsr;
  }
  if (lane < B) {
    const int r = lane;
    const int R = K + (r >> 2);
    int tbr[TB], kyr[TB];
#pragma unroll
    for (int J = 0; J < TB; ++J) {
      const int C = K + J;
      tbr[J] = (C >= R) ? (M::tidx(R, C) << 4) : 0;
      kyr[J] = (R ^ C) & 7;
    }
    // whole rows (zeros left of the diagonal): only the tile-level predicate
    // remains, so the stores need no divergent branches
#pragma unroll
    for (int c = 0; c < B; ++c) {
      rsb[16 + r * B + c] = row[c];
      if ((c >> 2) >= (r >> 2)) W.base[tile_off(tbr[c / 4], kyr[c / 4], r, c)] = row[c];
    }
    rsb[r] = rsr;
  }
}

// ----------------------------------------------------------------------------
// SYLV: L W + W U = W0, L (m x m) lower, U (q x q) upper [kernels.py:100-110]
// 4x4-tile anti-diagonal wavefront: a lane solves each tile of the current
// anti-diagonal (reference column/row order inside the tile), then all lanes
// push the fresh tiles' rank-4 contributions into later tiles of the same
// tile-row / tile-column.
// ----------------------------------------------------------------------------
// whole 4x4 tiles of a matrix / view (tiled: 8 x 16-byte chunks; global:
// 4 rows of 32 bytes), in view orientation
template <class M>
__device__ __forceinline__ void mat_tile_load(const double* base, int R, int C, double t[4][4]) {
  if constexpr (M::GLOBAL) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double2* p = reinterpret_cast<const double2*>(base + (4 * R + r) * M::LDN + 4 * C);
      const double2 a = p[0], b = p[1];
      t[r][0] = a.x;
      t[r][1] = a.y;
      t[r][2] = b.x;
      t[r][3] = b.y;
    }
  } else {
    const int tb = M::tidx(R, C) << 4, key = (R ^ C) & 7;
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      const double2 v = *reinterpret_cast<const double2*>(base + tb + (((ch ^ key) & 7) << 1));
      t[ch >> 1][2 * (ch & 1)] = v.x;
      t[ch >> 1][2 * (ch & 1) + 1] = v.y;
    }
  }
}
template <class V>
__device__ __forceinline__ void view_tile_load(const V& v, int I, int J, double t[4][4]) {
  using M = typename V::Mat;
  if constexpr (!V::tr) {
    mat_tile_load<M>(v.base, (v.r0 >> 2) + I, (v.c0 >> 2) + J, t);
  } else {
    double u[4][4];
    mat_tile_load<M>(v.base, (v.r0 >> 2) + J, (v.c0 >> 2) + I, u);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) t[a][b] = u[b][a];
  }
}
template <class V>
__device__ __forceinline__ void view_tile_store(const V& v, int I, int J, const double t[4][4]) {
  using M = typename V::Mat;
  static_assert(!V::tr && !M::GLOBAL, "stores go to the tiled unknown");
  const int R = (v.r0 >> 2) + I, C = (v.c0 >> 2) + J;
  const int tb = M::tidx(R, C) << 4, key = (R ^ C) & 7;
#pragma unroll
  for (int ch = 0; ch < 8; ++ch)
    *reinterpret_cast<double2*>(v.base + tb + (((ch ^ key) & 7) << 1)) =
        make_double2(t[ch >> 1][2 * (ch & 1)], t[ch >> 1][2 * (ch & 1) + 1]);
}

// one 4x4 tile of SYLV (reference column/row order inside the tile,
// kernels.py:100-110), reciprocal shifted pivots off the substitution chain
template <class LV, class UV, class WV>
__device__ __forceinline__ void sylv_tile(const LV& Lv, const UV& Uv, const WV& W, int I, int J) {
  double w[4][4], l[4][4], u[4][4];
  view_tile_load(W, I, J, w);
  view_tile_load(Lv, I, I, l);
  view_tile_load(Uv, J, J, u);
  double rp[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) rp[a][b] = 1.0 / (l[a][a] + u[b][b]);
#pragma unroll
  for (int b = 0; b < 4; ++b) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < b; ++c) acc = fma(w[a][c], u[c][b], acc);
      w[a][b] -= acc;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < a; ++c) acc = fma(l[a][c], w[c][b], acc);
      w[a][b] = (w[a][b] - acc) * rp[a][b];
    }
  }
  view_tile_store(W, I, J, w);
}

// SYLV: L W + W U = W0, L (m x m) lower, U (q x q) upper [kernels.py:100-110]
// 4x4-tile anti-diagonal wavefront: the tiles of anti-diagonal d are solved
// (one thread each), then every later tile of the same tile-row / tile-column
// receives the rank-4 contributions of the fresh tiles (one thread per
// target tile, whole-tile loads).
template <int WG, class LV, class UV, class WV>
__device__ __forceinline__ void sylv(const LV& Lv, const UV& Uv, const WV& W, int m, int q, const Grp& gr) {
  const int rank = gr.rank;
  constexpr int G = 32 * WG;
  const int TI = m >> 2, TJ = q >> 2;
  const int ntile = TI * TJ;
  // step d: every tile not yet solved takes the rank-4 contributions of the
  // tiles solved at step d-1 in its tile-row / tile-column, and the tiles of
  // anti-diagonal d are then solved by the thread that owns them — one group
  // barrier per step.
  for (int d = 0; d <= TI + TJ - 2; ++d) {
    for (int tile = rank; tile < ntile; tile += G) {
      const int I2 = tile / TJ, J2 = tile - I2 * TJ;
      if (I2 + J2 < d) continue;
      const int I1 = d - 1 - J2, J1 = d - 1 - I2;
      const bool colc = (d > 0 && I1 >= 0 && I1 < I2);
      const bool rowc = (d > 0 && J1 >= 0 && J1 < J2);
      const bool solve = (I2 + J2 == d);
      if (!colc && !rowc && !solve) continue;
      double w[4][4], a[4][4], x[4][4];
      view_tile_load(W, I2, J2, w);
      if (colc) {
        view_tile_load(Lv, I2, I1, a);
        view_tile_load(W, I1, J2, x);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double sacc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) sacc = fma(a[r][k], x[k][c], sacc);
            w[r][c] -= sacc;
          }
      }
      if (rowc) {
        view_tile_load(W, I2, J1, x);
        view_tile_load(Uv, J1, J2, a);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double sacc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) sacc = fma(x[r][k], a[k][c], sacc);
            w[r][c] -= sacc;
          }
      }
      if (solve) {
        double l[4][4], u[4][4], rp[4][4];
        view_tile_load(Lv, I2, I2, l);
        view_tile_load(Uv, J2, J2, u);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) rp[r][c] = 1.0 / (l[r][r] + u[c][c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < c; ++k) acc = fma(w[r][k], u[k][c], acc);
            w[r][c] -= acc;
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < r; ++k) acc = fma(l[r][k], w[k][c], acc);
            w[r][c] = (w[r][c] - acc) * rp[r][c];
          }
        }
      }
      view_tile_store(W, I2, J2, w);
    }
    gsync<WG>(gr);
  }
}

// ----------------------------------------------------------------------------
// B <= 8 diagonal-block leaves in registers, run by one warp (lane 0 stores):
// LYAP (kernels.py:113-130, reference (j, i <= j) order) and SYLV
// (kernels.py:100-110, column-then-row order).
// ----------------------------------------------------------------------------
template <int B, class LV, class WV>
__device__ __forceinline__ void lyap_leaf_reg(const LV& Lv, const WV& W) {
  constexpr int TB = B / 4;
  double l[B][B], x[B][B];
#pragma unroll
  for (int I = 0; I < TB; ++I)
#pragma unroll
    for (int J = 0; J < TB; ++J) {
      double t[4][4];
      if (J <= I) {
        view_tile_load(Lv, I, J, t);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) l[4 * I + a][4 * J + b] = t[a][b];
      }
      if (I <= J) {
        view_tile_load(W, I, J, t);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) x[4 * I + a][4 * J + b] = t[a][b];
      }
    }
#pragma unroll
  for (int j = 0; j < B; ++j)
#pragma unroll
    for (int i = 0; i <= j; ++i) {
      const double rp = 1.0 / (l[i][i] + l[j][j]);
      double acc = x[i][j], d1 = 0.0, d2 = 0.0;
#pragma unroll
      for (int q = 0; q < i; ++q) d1 = fma(l[i][q], x[q][j], d1);
#pragma unroll
      for (int q = 0; q < j; ++q) d2 = fma(q < i ? x[q][i] : x[i][q], l[j][q], d2);
      acc -= d1;
      acc -= d2;
      x[i][j] = acc * rp;
    }
  if (lane_id() == 0) {
#pragma unroll
    for (int I = 0; I < TB; ++I)
#pragma unroll
      for (int J = I; J < TB; ++J) {
        double t[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int r = 4 * I + a, c = 4 * J + b;
            t[a][b] = r <= c ? x[r][c] : x[c][r];
          }
        view_tile_store(W, I, J, t);
      }
  }
}

template <int B, class LV, class UV, class WV>
__device__ __forceinline__ void sylv_leaf_reg(const LV& Lv, const UV& Uv, const WV& W) {
  constexpr int TB = B / 4;
  double l[B][B], u[B][B], x[B][B];
#pragma unroll
  for (int I = 0; I < TB; ++I)
#pragma unroll
    for (int J = 0; J < TB; ++J) {
      double t[4][4];
      view_tile_load(W, I, J, t);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) x[4 * I + a][4 * J + b] = t[a][b];
      if (J <= I) {
        view_tile_load(Lv, I, J, t);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) l[4 * I + a][4 * J + b] = t[a][b];
      }
      if (I <= J) {
        view_tile_load(Uv, I, J, t);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) u[4 * I + a][4 * J + b] = t[a][b];
      }
    }
#pragma unroll
  for (int j = 0; j < B; ++j) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < j; ++c) acc = fma(x[i][c], u[c][j], acc);
      x[i][j] -= acc;
    }
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const double rp = 1.0 / (l[i][i] + u[j][j]);
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < i; ++c) acc = fma(l[i][c], x[c][j], acc);
      x[i][j] = (x[i][j] - acc) * rp;
    }
  }
  if (lane_id() == 0) {
#pragma unroll
    for (int I = 0; I < TB; ++I)
#pragma unroll
      for (int J = 0; J < TB; ++J) {
        double t[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) t[a][b] = x[4 * I + a][4 * J + b];
        view_tile_store(W, I, J, t);
      }
  }
}

// ----------------------------------------------------------------------------
// LYAP leaf (symmetric, upper stored) [kernels.py:113-130]: element
// anti-diagonal wavefront, pull model; writes the upper triangle only.
// ----------------------------------------------------------------------------
template <int WG, class LV, class WV, class WSV>
__device__ __forceinline__ void lyap(const LV& Lv, const WV& W, const WSV& Ws, int m, const Grp& gr) {
  const int lane = gr.rank;
  for (int d = 0; d <= 2 * (m - 1); ++d) {
    const int ilo = d - (m - 1) > 0 ? d - (m - 1) : 0;
    const int ihi = d >> 1;
    for (int i = ilo + lane; i <= ihi; i += 32 * WG) {
      const int j = d - i;
      const double rp = 1.0 / (Lv.at(i, i) + Lv.at(j, j));  // off the dot-product chain
      double acc = W.at(i, j);
      double d1 = 0.0, d2 = 0.0;
      for (int l = 0; l < i; ++l) d1 = fma(Lv.at(i, l), W.at(l, j), d1);
      for (int l = 0; l < j; ++l) d2 = fma(Ws.at(i, l), Lv.at(j, l), d2);
      acc -= d1;
      acc -= d2;
      W.ref(i, j) = acc * rp;
    }
    gsync<WG>(gr);
  }
}

// ----------------------------------------------------------------------------
// Compile-time statement encoding (generated: variants_ct.cuh)
// ----------------------------------------------------------------------------
template <int OP, int R, int C, int TRN>
struct V {
  static constexpr int op = OP, r = R, c = C, tr = TRN;
};
struct NoV {
  static constexpr int op = -1, r = 0, c = 0, tr = 0;
};
template <int KIND, int SIGN, class OUT, class IN0 = NoV, class IN1 = NoV>
struct St {
  static constexpr int kind = KIND, sign = SIGN;
  using out = OUT;
  using in0 = IN0;
  using in1 = IN1;
};
template <class... S>
struct Var {};

// Equation traits: storage layout of each operand code.
template <int EQ, int N>
struct EqT;
template <int N>
struct EqT<0, N> {  // cholesky: X upper
  static constexpr int T = N / 4;
  static constexpr bool STAGE = true;
  using M0 = TM<T, UPPER>;
  using M1 = M0;
  using M2 = M0;
  static constexpr bool SYMT = true, SYMX = false;
  static constexpr int SLOT = M0::DOUBLES;
};
template <int N>
struct EqT<1, N> {  // lyapunov: X upper (symmetric), L lower
  static constexpr int T = N / 4;
  static constexpr bool STAGE = true;
  using M0 = TM<T, UPPER>;
  using M1 = TM<T, LOWER>;
  using M2 = M1;
  static constexpr bool SYMT = true, SYMX = true;
  static constexpr int SLOT = M0::DOUBLES + M1::DOUBLES;
};
template <int N>
struct EqT<2, N> {  // sylvester: X dense, L lower, U upper (global if too big)
  static constexpr int T = N / 4;
  static constexpr bool STAGE = (T * T + T * (T + 1)) * 128 <= 220 * 1024;
  using M0 = TM<T, DENSE>;
  using M1 = typename std::conditional<STAGE, TM<T, LOWER>, GM<N>>::type;
  using M2 = typename std::conditional<STAGE, TM<T, UPPER>, GM<N>>::type;
  static constexpr bool SYMT = false, SYMX = false;
  static constexpr int SLOT = M0::DOUBLES + M1::DOUBLES + M2::DOUBLES;
};

template <class E, int OP>
struct MatOf {
  using type = typename E::M0;
};
template <class E>
struct MatOf<E, 1> {
  using type = typename E::M1;
};
template <class E>
struct MatOf<E, 2> {
  using type = typename E::M2;
};

struct Slot {
  double* p[3];
};

template <int N, int B>
struct Rep {
  int k;
  __device__ __forceinline__ int st(int r) const { return r == 0 ? 0 : (r == 1 ? k * B : (k + 1) * B); }
  __device__ __forceinline__ int ex(int r) const { return r == 0 ? k * B : (r == 1 ? B : N - (k + 1) * B); }
};

template <class E, class Vw, bool SY>
__device__ __forceinline__ TV<typename MatOf<E, Vw::op>::type, Vw::tr != 0, SY> mkv(const Slot& s, int r0, int c0) {
  TV<typename MatOf<E, Vw::op>::type, Vw::tr != 0, SY> v;
  v.base = s.p[Vw::op < 0 ? 0 : Vw::op];
  v.r0 = r0;
  v.c0 = c0;
  return v;
}

template <int EQ, int N, int B, int WG, class S>
__device__ __forceinline__ void exec(const Slot& s, const Rep<N, B>& rp, int* flag, const Grp& gr, const Sub& sb) {
  using E = EqT<EQ, N>;
  using O = typename S::out;
  const int m = rp.ex(O::r), q = rp.ex(O::c);
  if (m == 0 || q == 0) return;
  const auto Ov = mkv<E, O, false>(s, rp.st(O::r), rp.st(O::c));
  if constexpr (S::kind == K_GEMM) {
    using A = typename S::in0;
    using Bv = typename S::in1;
    const int p = A::tr ? rp.ex(A::r) : rp.ex(A::c);
    if (p == 0) return;
    constexpr bool UP = E::SYMT && O::r == O::c;
    constexpr bool SA = E::SYMX && A::op == 0 && A::r == A::c;
    constexpr bool SB = E::SYMX && Bv::op == 0 && Bv::r == Bv::c;
    const auto Av = mkv<E, A, SA>(s, rp.st(A::r), rp.st(A::c));
    const auto Bw = mkv<E, Bv, SB>(s, rp.st(Bv::r), rp.st(Bv::c));
    gemm<UP, WG>(Ov, Av, Bw, m, p, q, S::sign < 0 ? -1.0 : 1.0, gr, sb);
  } else if constexpr (S::kind == K_CHOL) {
    if (gr.wig == 0) {
      if constexpr (B <= 8) chol_leaf_reg<B>(Ov, rp.st(O::r), flag, gr.rsb);
      else chol_leaf<B>(Ov, rp.st(O::r), flag);
    }
  } else if constexpr (S::kind == K_TRSM) {
    using A = typename S::in0;
    const auto Tv = mkv<E, A, false>(s, rp.st(A::r), rp.st(A::c));
    if constexpr (O::r == 1) trsm_b<B, WG>(Tv, Ov, q, gr, sb);  // m == B
    else trsm<WG>(Tv, Ov, m, q, gr, sb);
  } else if constexpr (S::kind == K_SYLV) {
    using A = typename S::in0;
    using Bv = typename S::in1;
    const auto Lv = mkv<E, A, false>(s, rp.st(A::r), rp.st(A::c));
    const auto Uv = mkv<E, Bv, false>(s, rp.st(Bv::r), rp.st(Bv::c));
    if constexpr (O::r == O::c && B <= 4) {
      if (gr.wig == 0) sylv_leaf_reg<B>(Lv, Uv, Ov);  // m == q == B
    } else {
      sylv<WG>(Lv, Uv, Ov, m, q, gr);
    }
  } else if constexpr (S::kind == K_LYAP) {
    using A = typename S::in0;
    const auto Lv = mkv<E, A, false>(s, rp.st(A::r), rp.st(A::c));
    const auto Ws = mkv<E, O, true>(s, rp.st(O::r), rp.st(O::c));
    if constexpr (B <= 8) {
      if (gr.wig == 0) lyap_leaf_reg<B>(Lv, Ov);
    } else {
      lyap<WG>(Lv, Ov, Ws, m, gr);
    }
  }
}

// ----------------------------------------------------------------------------
// Per-iteration schedule (compile time).  Statements are grouped into
// dependency levels (as-late-as-possible, so an independent update floats
// next to the statement that needs it last); statements of one level touch
// disjoint blocks, so they run back to back without a barrier, and a CHOL
// leaf (one warp) shares its level with the other statements running on the
// remaining warps.  Results are bitwise those of program order.
// ----------------------------------------------------------------------------
struct SD {
  int kind, oop, orr, oc;
  int iop[2], ir[2], ic[2];
};
template <class S>
constexpr SD make_sd() {
  return SD{S::kind, S::out::op, S::out::r, S::out::c,
            {S::in0::op, S::in1::op}, {S::in0::r, S::in1::r}, {S::in0::c, S::in1::c}};
}
constexpr bool sd_reads(const SD& a, int op, int r, int c) {
  if (a.oop == op && a.orr == r && a.oc == c) return true;  // read-modify-write
  for (int t = 0; t < 2; ++t)
    if (a.iop[t] == op && a.ir[t] == r && a.ic[t] == c) return true;
  return false;
}
constexpr bool sd_dep(const SD& a, const SD& b) {  // b (later) depends on a
  return sd_reads(b, a.oop, a.orr, a.oc) || sd_reads(a, b.oop, b.orr, b.oc);
}
template <int M, int B>
struct Sched {
  int level[M > 0 ? M : 1];
  int nlevels;
  int leaf_level_has_leaf[M > 0 ? M : 1];
  int prefix[M > 0 ? M : 1];  // GEMM updates of a leaf's block run by the leaf warp right before it
  // single-warp statements: CHOL leaves, and LYAP / diagonal SYLV leaves for B <= 8
  static constexpr bool is_leaf(const SD& s) {
    return s.kind == K_CHOL || (B <= 8 && s.kind == K_LYAP) || (B <= 4 && s.kind == K_SYLV && s.orr == s.oc);
  }
  constexpr Sched(const SD* d) : level{}, nlevels(0), leaf_level_has_leaf{} {
    int asap[M > 0 ? M : 1] = {};
    for (int j = 0; j < M; ++j) {
      asap[j] = 0;
      for (int i = 0; i < j; ++i)
        if (sd_dep(d[i], d[j]) && asap[i] + 1 > asap[j]) asap[j] = asap[i] + 1;
    }
    int depth = 0;
    for (int j = 0; j < M; ++j)
      if (asap[j] + 1 > depth) depth = asap[j] + 1;
    // as late as possible
    for (int j = M - 1; j >= 0; --j) {
      int l = depth - 1;
      for (int k = j + 1; k < M; ++k)
        if (sd_dep(d[j], d[k]) && level[k] - 1 < l) l = level[k] - 1;
      level[j] = l;
    }
    nlevels = depth;
    // leaf prefixes: a GEMM whose output is a leaf's block and that nothing
    // but the leaf depends on moves into the leaf's level, executed by the
    // leaf warp right before the leaf (no group barrier in between)
    for (int j = 0; j < M; ++j) prefix[j] = 0;
    for (int l = 0; l < M; ++l) {
      if (!is_leaf(d[l])) continue;
      for (int j = 0; j < l; ++j) {
        if (d[j].kind != K_GEMM || d[j].orr != d[l].orr || d[j].oc != d[l].oc || d[j].oop != d[l].oop) continue;
        bool only_leaf = true;
        for (int k = j + 1; k < M; ++k)
          if (k != l && sd_dep(d[j], d[k]) && level[k] <= level[l] &&
              !(d[k].kind == K_GEMM && d[k].orr == d[l].orr && d[k].oc == d[l].oc))
            only_leaf = false;  // a dependent that would run no later than the leaf
        if (only_leaf) {
          prefix[j] = 1;
          level[j] = level[l];
        }
      }
    }
    // compact the level numbers (a level may have emptied)
    int remap[M > 0 ? M : 1] = {};
    for (int L = 0; L < M; ++L) remap[L] = -1;
    int nl = 0;
    for (int L = 0; L < depth; ++L) {
      bool used = false;
      for (int j = 0; j < M; ++j)
        if (level[j] == L) used = true;
      if (used) remap[L] = nl++;
    }
    for (int j = 0; j < M; ++j) level[j] = remap[level[j]];
    nlevels = nl;
    for (int j = 0; j < M; ++j) leaf_level_has_leaf[j] = 0;
    for (int j = 0; j < M; ++j)
      if (is_leaf(d[j])) leaf_level_has_leaf[level[j]] = 1;
  }
};

template <int B, class... S>
struct VarInfo {
  static constexpr int M = sizeof...(S);
  static constexpr SD d[M] = {make_sd<S>()...};
  static constexpr Sched<M, B> sch{d};
};

template <int EQ, int N, int B, int WG, int L, class INFO, class S, int I>
__device__ __forceinline__ void exec_if(const Slot& s, const Rep<N, B>& rp, int* flag, const Grp& gr) {
  if constexpr (INFO::sch.level[I] == L) {
    constexpr bool is_prefix = INFO::sch.prefix[I] != 0;
    constexpr bool shared_level =
        (WG > 1) && INFO::sch.leaf_level_has_leaf[L] && !INFO::sch.is_leaf(make_sd<S>()) && !is_prefix;
    Sub sb;
    if constexpr (is_prefix && WG > 1) {
      if (gr.wig != 0) return;  // the leaf warp runs its block's updates
      sb.w = 0;
      sb.nw = 1;
      sb.rank = gr.rank;
      sb.nthr = 32;
      sb.full = false;
    } else if constexpr (shared_level) {
      if (gr.wig == 0) return;  // warp 0 runs the leaf of this level
      sb.w = gr.wig - 1;
      sb.nw = WG - 1;
      sb.rank = gr.rank - 32;
      sb.nthr = 32 * (WG - 1);
      sb.full = false;
    } else {
      sb.w = gr.wig;
      sb.nw = WG;
      sb.rank = gr.rank;
      sb.nthr = 32 * WG;
      sb.full = true;
    }
    const long long t0 = gr.prof ? clock64() : 0;
    exec<EQ, N, B, WG, S>(s, rp, flag, gr, sb);
    // per statement, per warp (warp 0 -> [12 + I], warp 1 -> [22 + I])
    if (gr.prof && I < 10) gr.prof[(gr.wig == 0 ? 12 : 22) + I] += clock64() - t0;
  }
}

// Optional cycle accounting (tools/phase_profile.py): when the launch passes
// a profile buffer, thread 0 of group 0 in CTA 0 adds the cycles of each
// schedule level ([4 + L]) and phase ([0] wait, [1] compute, [2] store,
// [3] problems) to it.
template <int EQ, int N, int B, int WG, int L, class INFO, class... S, size_t... I>
__device__ __forceinline__ void run_level(const Slot& s, const Rep<N, B>& rp, int* flag, const Grp& gr,
                                          std::index_sequence<I...>) {
  const long long t0 = clock64();
  (exec_if<EQ, N, B, WG, L, INFO, S, (int)I>(s, rp, flag, gr), ...);
  gsync<WG>(gr);
  if (gr.prof && gr.wig == 0) gr.prof[4 + L] += clock64() - t0;
}

template <int EQ, int N, int B, int WG, class INFO, class... S, int... Ls>
__device__ __forceinline__ void run_iter(const Slot& s, const Rep<N, B>& rp, int* flag, const Grp& gr,
                                         std::integer_sequence<int, Ls...>) {
  (run_level<EQ, N, B, WG, Ls, INFO, S...>(s, rp, flag, gr, std::index_sequence_for<S...>{}), ...);
}

// Cholesky variants whose iteration k finalises block row k (those with an
// "X12 := ..." statement: v1, v2) stream that block row to HBM right after
// the iteration, overlapping the output writes with later iterations.
template <class... S>
struct RowFinal {
#ifdef LAGEN_NO_ROW_STREAM
  static constexpr bool value = false;
#else
  static constexpr bool value = ((S::out::r == 1 && S::out::c == 2) || ...);
#endif
};

template <int N, class M, int G>
__device__ __forceinline__ bool store_chol_rows(double* __restrict__ dst, const double* xs, int r0, int r1, int rank) {
  constexpr int T = N / 4;
  bool finite = true;
  const int units = (r1 - r0) * T;  // (row, tile column) units of 4 doubles
  for (int u = rank; u < units; u += G) {
    const int r = r0 + u / T, C = u % T, c = 4 * C, R = r >> 2;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (C >= R) {
      const double2 p0 = *reinterpret_cast<const double2*>(xs + M::off(r, c));
      const double2 p1 = *reinterpret_cast<const double2*>(xs + M::off(r, c + 2));
      v[0] = (c >= r) ? p0.x : 0.0;
      v[1] = (c + 1 >= r) ? p0.y : 0.0;
      v[2] = (c + 2 >= r) ? p1.x : 0.0;
      v[3] = (c + 3 >= r) ? p1.y : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) finite = finite && isfinite(v[e]);
    double2* gp = reinterpret_cast<double2*>(dst + r * N + c);
    __stcs(gp, make_double2(v[0], v[1]));
    __stcs(gp + 1, make_double2(v[2], v[3]));
  }
  return finite;
}

template <int EQ, int N, int B, int WG, class... S>
__device__ __forceinline__ bool run_variant(Var<S...>, const Slot& s, int* flag, const Grp& gr, double* xout) {
  using INFO = VarInfo<B, S...>;
  bool finite = true;
#pragma unroll 1
  for (int k = 0; k < N / B; ++k) {
    Rep<N, B> rp{k};
    run_iter<EQ, N, B, WG, INFO, S...>(s, rp, flag, gr, std::make_integer_sequence<int, INFO::sch.nlevels>{});
    if constexpr (EQ == 0 && RowFinal<S...>::value)
      finite = store_chol_rows<N, typename EqT<EQ, N>::M0, 32 * WG>(xout, s.p[0], k * B, (k + 1) * B, gr.rank) &&
               finite;
  }
  return finite;
}

template <class VAR>
struct StreamsRows;
template <class... S>
struct StreamsRows<Var<S...>> {
  static constexpr bool value = RowFinal<S...>::value;
};

// ----------------------------------------------------------------------------
// global -> tiled shared memory (cp.async, 16 B chunks), one warp per problem
// part: 0 = all tiles, 1 = upper tiles (C >= R), 2 = lower tiles (C <= R)
// ----------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NLEFT>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NLEFT) : "memory");
}

template <class M, int N, int PART, int G>
__device__ __forceinline__ void load_tiles_async(double* dst, const double* __restrict__ src, int rank) {
  constexpr int T = N / 4;
  // unit = (R, rr, C, half): 16 consecutive bytes of one tile row
  constexpr int UNITS = T * 4 * T * 2;
  for (int u = rank; u < UNITS; u += G) {
    const int h = u & 1;
    const int C = (u >> 1) % T;
    const int rr = ((u >> 1) / T) & 3;
    const int R = (u >> 1) / (4 * T);
    if (PART == 1 && C < R) continue;
    if (PART == 2 && C > R) continue;
    const int r = 4 * R + rr, c = 4 * C + 2 * h;
    double* tp = dst + (M::tidx(R, C) << 4) + swz(r, c, (R ^ C) & 7);
    cp_async16(tp, src + r * N + c);
  }
}

// store all n^2 entries of X; EQ decides zeros (chol) / mirror (lyap)
template <int EQ, class M, int N, int G>
__device__ __forceinline__ bool store_x(double* __restrict__ dst, const double* xs, int rank) {
  constexpr int T = N / 4;
  constexpr int UNITS = T * 4 * T;
  bool finite = true;
#pragma unroll 4
  for (int u = rank; u < UNITS; u += G) {
    const int C = u % T;
    const int rr = (u / T) & 3;
    const int R = u / (4 * T);
    const int r = 4 * R + rr, c = 4 * C;
    double v[4];
    if constexpr (EQ == 2) {
      const double2 p0 = *reinterpret_cast<const double2*>(xs + M::off(r, c));
      const double2 p1 = *reinterpret_cast<const double2*>(xs + M::off(r, c + 2));
      v[0] = p0.x;
      v[1] = p0.y;
      v[2] = p1.x;
      v[3] = p1.y;
    } else if constexpr (EQ == 0) {
      if (C < R) {
        v[0] = v[1] = v[2] = v[3] = 0.0;
      } else {
        const double2 p0 = *reinterpret_cast<const double2*>(xs + M::off(r, c));
        const double2 p1 = *reinterpret_cast<const double2*>(xs + M::off(r, c + 2));
        v[0] = (c >= r) ? p0.x : 0.0;
        v[1] = (c + 1 >= r) ? p0.y : 0.0;
        v[2] = (c + 2 >= r) ? p1.x : 0.0;
        v[3] = (c + 3 >= r) ? p1.y : 0.0;
      }
    } else {
      if (C > R) {
        const double2 p0 = *reinterpret_cast<const double2*>(xs + M::off(r, c));
        const double2 p1 = *reinterpret_cast<const double2*>(xs + M::off(r, c + 2));
        v[0] = p0.x;
        v[1] = p0.y;
        v[2] = p1.x;
        v[3] = p1.y;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int cc = c + e;
          v[e] = (cc >= r) ? xs[M::off(r, cc)] : xs[M::off(cc, r)];
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) finite = finite && isfinite(v[e]);
    double2* gp = reinterpret_cast<double2*>(dst + r * N + c);
    __stcs(gp, make_double2(v[0], v[1]));
    __stcs(gp + 1, make_double2(v[2], v[3]));
  }
  return finite;
}

template <int EQ, int N>
struct WPolicy {
  using E = EqT<EQ, N>;
  static constexpr int SLOT = E::SLOT;  // doubles per problem
  static constexpr int BUDGET = 220 * 1024;
  static constexpr int TARGET_WARPS = 12;
  // problem slots that fit single / double buffered
  static constexpr int S1 = BUDGET / (SLOT * 8 + 640);      // + per-group pivots / factor scratch
  static constexpr int S2 = BUDGET / (2 * SLOT * 8 + 640);
  // double-buffer (prefetch the next problem) when >= 6 problems still fit
  static constexpr int DB = S2 >= 6 ? 2 : 1;
  static constexpr int P0 = DB == 2 ? S2 : (S1 < 1 ? 1 : S1);
  static constexpr int P = P0 > 16 ? 16 : (P0 > 15 && TARGET_WARPS > P0 ? 15 : P0);
  // warps per problem: smallest power of two reaching TARGET_WARPS per CTA
  static constexpr int WG = P >= TARGET_WARPS ? 1 : (2 * P >= TARGET_WARPS ? 2 : (4 * P >= TARGET_WARPS ? 4 : (8 * P >= TARGET_WARPS ? 8 : 16)));
  static constexpr int WARPS = P * WG;
  static constexpr int RSB = 16 + 64;  // reciprocal pivots + B<=8 factor, per group
  static constexpr size_t BASE = (size_t)P * DB * SLOT * 8 + 2 * 16 * sizeof(int) + (size_t)P * RSB * 8;
  // split-K scratch per group (doubles), only where it still fits
  static constexpr int SCR = (BASE + (size_t)P * (WG - 1) * 256 * 8 <= 227 * 1024) ? (WG - 1) * 256 : 0;
  static constexpr size_t SMEM = BASE + (size_t)P * SCR * 8;
};

template <int EQ, int N, int G>
__device__ __forceinline__ void issue_loads(const Slot& s, const double* in0, const double* in1, const double* in2,
                                            long long off, int rank) {
  using E = EqT<EQ, N>;
  if constexpr (EQ == 0) {
    load_tiles_async<typename E::M0, N, 1, G>(s.p[0], in0 + off, rank);
  } else if constexpr (EQ == 1) {
    load_tiles_async<typename E::M1, N, 2, G>(s.p[1], in0 + off, rank);
    load_tiles_async<typename E::M0, N, 1, G>(s.p[0], in1 + off, rank);
  } else {
    if constexpr (E::STAGE) {
      load_tiles_async<typename E::M1, N, 2, G>(s.p[1], in0 + off, rank);
      load_tiles_async<typename E::M2, N, 1, G>(s.p[2], in1 + off, rank);
    }
    load_tiles_async<typename E::M0, N, 0, G>(s.p[0], in2 + off, rank);
  }
  cp_async_commit();
}

// CTA = P problem groups x WG warps; persistent over the batch; each group
// prefetches its next problem (DB == 2) while solving the current one.
template <int EQ, int N, int B, class VAR>
__global__ void __launch_bounds__(WPolicy<EQ, N>::WARPS * 32, 1)
    warp_kernel(const double* __restrict__ in0, const double* __restrict__ in1, const double* __restrict__ in2,
                double* __restrict__ X, int* __restrict__ info, long long batch,
                unsigned long long* __restrict__ prof) {
  using E = EqT<EQ, N>;
  using P = WPolicy<EQ, N>;
  constexpr int WG = P::WG, G = WG * 32;
  extern __shared__ double smem[];
  int* gflag = reinterpret_cast<int*>(smem + (size_t)P::P * P::DB * P::SLOT);
  int* gbad = gflag + 16;
  double* rsb_all = reinterpret_cast<double*>(gbad + 16);
  double* scr_all = rsb_all + P::P * P::RSB;
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  Grp gr;
  gr.id = warp / WG;
  gr.wig = warp % WG;
  gr.rank = threadIdx.x % G;
  gr.rsb = rsb_all + P::RSB * gr.id;
  gr.scr = P::SCR ? scr_all + (size_t)P::SCR * gr.id : nullptr;
  gr.prof = (prof && blockIdx.x == 0 && gr.id == 0 && (gr.rank == 0 || gr.rank == 32)) ? prof : nullptr;
  // warps 1 .. WG-1 of group g synchronise on barrier 1 + P + g (group barriers use 1 .. P)
  gr.subbar = (WG > 2 && 1 + P::P + gr.id <= 15) ? 1 + P::P + gr.id : 0;
  auto slot_at = [&](int d) {
    Slot sl;
    double* base = smem + ((size_t)gr.id * P::DB + (d % P::DB)) * P::SLOT;
    sl.p[0] = base;
    sl.p[1] = base + E::M0::DOUBLES;
    sl.p[2] = (EQ == 2) ? base + E::M0::DOUBLES + E::M1::DOUBLES : sl.p[1];
    return sl;
  };
  constexpr long long NN = (long long)N * N;
  const long long stride = (long long)gridDim.x * P::P;
  long long prob = (long long)blockIdx.x * P::P + gr.id;
  if (prob < batch) issue_loads<EQ, N, G>(slot_at(0), in0, in1, in2, prob * NN, gr.rank);
  int cur = 0;
  for (; prob < batch; prob += stride) {
    const long long off = prob * NN;
    const long long nxt = prob + stride;
    Slot s = slot_at(cur);
    const long long tw0 = clock64();
    if constexpr (P::DB == 2) {
      if (nxt < batch) {
        issue_loads<EQ, N, G>(slot_at(cur ^ 1), in0, in1, in2, nxt * NN, gr.rank);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
    } else {
      cp_async_wait<0>();
    }
    if (gr.rank == 0) {
      gflag[gr.id] = 0;
      gbad[gr.id] = 0;
    }
    gsync<WG>(gr);
    if constexpr (EQ == 2 && !E::STAGE) {
      s.p[1] = const_cast<double*>(in0) + off;
      s.p[2] = const_cast<double*>(in1) + off;
    }
    int flag = 0;
    const long long tw1 = clock64();
    if (gr.prof && gr.wig == 0) gr.prof[0] += tw1 - tw0;  // wait for this problem's tiles
    bool fin = run_variant<EQ, N, B, WG>(VAR{}, s, &flag, gr, X + off);
    const long long tw2 = clock64();
    if (gr.prof && gr.wig == 0) {
      gr.prof[1] += tw2 - tw1;  // compute
      gr.prof[3] += 1;          // problems
    }
    if constexpr (!(EQ == 0 && StreamsRows<VAR>::value))
      fin = store_x<EQ, typename E::M0, N, G>(X + off, s.p[0], gr.rank) && fin;
    const bool allfin = __all_sync(0xffffffffu, fin);
    if (gr.wig == 0 && lane == 0 && flag) gflag[gr.id] = flag;
    if (lane == 0 && !allfin) atomicOr(&gbad[gr.id], 1);
    gsync<WG>(gr);
    if (info && gr.rank == 0) {
      const int f = gflag[gr.id];
      info[prob] = f ? f : (gbad[gr.id] ? -1 : 0);
    }
    if (gr.prof && gr.wig == 0) gr.prof[2] += clock64() - tw2;  // store + guards
    if constexpr (P::DB == 1) {
      gsync<WG>(gr);  // slot reads done before it is refilled
      if (nxt < batch) issue_loads<EQ, N, G>(slot_at(0), in0, in1, in2, nxt * NN, gr.rank);
    } else {
      cur ^= 1;
    }
  }
}

}  // namespace eng
}  // namespace lagen
