// chol_rows.cuh — the "rows engine": Cholesky variant v1 on a packed
// row-major upper layout.
//
// Variant v1 (the reference's enumeration, variants_table.json):
//     S1: X11 -= X01^T X01      (upper target)
//     S2: X11 := CHOL(X11)
//     S3: X12 -= X01^T X02
//     S4: X12 := TRSM(X11^T, X12)                 (verify.py:245-297)
// Both GEMM operands are segments of the rows above the current block row,
// so X lives in shared memory as its upper rows, row-major: row r keeps
// columns [4*floor(r/4), n) (16-byte aligned).  The m8n8k4 DMMA fragments of
// one k-step (4 rows) are then addressed from one per-lane row pointer that
// advances with two integer ops (the tiled layout of the generic engines
// spends ~35% of its instructions on address arithmetic here, measured).
//
// Schedule per iteration (group of WG warps owns a problem, P problems per
// CTA as the warp engine's WPolicy):
//   level A  warp 0: S1 (one 8x8 DMMA tile, 4 accumulator chains), then the
//            CHOL leaf in registers (rsqrt pivots; reciprocals + factor to
//            rsb for S4); warps 1..WG-1 concurrently: S3 in 8x32 DMMA blocks,
//            k split across idle warps with a fixed-order reduction
//   level B  all: S4, lanes own columns
//   then     block row k streams to HBM (zeros left of the diagonal)
// Per element the arithmetic is v1's statements (S3 does not depend on S2).
#pragma once
#include <type_traits>

#include "engine.cuh"

// Residency (measured over the sweep, profiles/r01_rows_db.txt): single
// buffering with up to 16 warps per CTA beats double buffering (prefetch of
// the next problem) at every n — more problems in flight hide more latency
// than the prefetch does; 32 warps per CTA spill registers.
#ifndef LAGEN_ROWS_MAXW
#define LAGEN_ROWS_MAXW 16
#endif
#ifndef LAGEN_ROWS_PCAP
#define LAGEN_ROWS_PCAP 16  // problems per CTA cap (group barriers 1..P, per-group flags: <= 32 with WG = 1)
#endif
// Loads / stores walk warp-per-row when a row's 16-byte pairs fill whole
// warps, and from this many pairs per row on (the partial second pass idles
// fewer lanes than the flattened loop's per-element division costs: 4-5 %
// faster at n = 108..124, 1-9 % slower at n = 68..104; profiles/r01_rowloop_ab.txt)
#ifndef LAGEN_ROWS_ROWLOOP_H
#define LAGEN_ROWS_ROWLOOP_H 54
#endif
// the store's row walk got cheaper in round 2 (row start by an add, unrolled
// passes): it now also wins at n = 68..104
#ifndef LAGEN_ROWS_STORE_ROWLOOP_H
#define LAGEN_ROWS_STORE_ROWLOOP_H 34
#endif
#ifndef LAGEN_ROWS_DBMIN
#define LAGEN_ROWS_DBMIN 1000  // double-buffer when >= this many slots fit twice (off)
#endif

namespace lagen {
namespace cr {

using eng::cp_async16;
using eng::cp_async_commit;
using eng::cp_async_wait;
using eng::dmma;
using eng::Grp;
using eng::gsync;
using eng::lane_id;

// Residency: WG warps own a problem (a template parameter; the launcher picks
// it per size, rows_wg()), as many problems per CTA as shared memory allows,
// double-buffered (next problem prefetched) when >= 6 still fit.
#ifndef LAGEN_ROWS_SPREAD
#define LAGEN_ROWS_SPREAD 1
#endif

// 1 / sqrt(a) for the Cholesky pivots: rsqrt.approx (MUFU.RSQ64H, ~2^-20)
// and two Newton steps y <- y + y (1/2 - (a/2) y^2), 9 instructions instead
// of the ~19 of rsqrt() with its special-case path (13 % of the rows kernel's
// instructions at n = 64); <= 2 ulp for normal a > 0 — a <= 0, NaN and Inf
// pivots are flagged by the callers before the value is used
__device__ __forceinline__ double rsqrt_nr(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  const double h = 0.5 * a;
  double e = fma(-h, y * y, 0.5);
  y = fma(y, e, y);
  e = fma(-h, y * y, 0.5);
  return fma(y, e, y);
}

template <int N, int WG_>
struct RPolicy {
  static constexpr int SLOT = N * N / 2 + 2 * N;
  static constexpr int BUDGET = 220 * 1024;
  static constexpr int WG = WG_;
  static constexpr int S1 = BUDGET / (SLOT * 8 + 640);
  static constexpr int S2 = BUDGET / (2 * SLOT * 8 + 640);
  static constexpr int DB = S2 >= LAGEN_ROWS_DBMIN ? 2 : 1;
  static constexpr int P0 = DB == 2 ? S2 : (S1 < 1 ? 1 : S1);
  static constexpr int PMAX = LAGEN_ROWS_MAXW / WG > LAGEN_ROWS_PCAP ? LAGEN_ROWS_PCAP : LAGEN_ROWS_MAXW / WG;  // warps per CTA cap
  static constexpr int P = P0 > PMAX ? PMAX : P0;
  static constexpr int WARPS = P * WG;
  static constexpr int RSB = 16 + 64;
  static constexpr size_t BASE = (size_t)P * DB * SLOT * 8 + 2 * 16 * sizeof(int) + (size_t)P * RSB * 8;
  static constexpr int SCR = (BASE + (size_t)P * (WG - 1) * 256 * 8 <= 227 * 1024) ? (WG - 1) * 256 : 0;
  static constexpr size_t SMEM = BASE + (size_t)P * SCR * 8;
};

// packed upper rows: row r starts at column 4R (R = r / 4)
template <int N>
struct Rows {
  static constexpr int DOUBLES = N * N / 2 + 2 * N;
  __device__ static __forceinline__ int off(int r) {
    const int R = r >> 2;
    return 4 * N * R - 8 * R * (R - 1) + (r & 3) * (N - 4 * R);
  }
  // address of element (r, c), c >= 4 * floor(r / 4)
  __device__ static __forceinline__ int at(int r, int c) { return off(r) + c - 4 * (r >> 2); }
};

// Row pointer of lane t for the k-step covering rows 4R' .. 4R'+3: element
// (4R' + t, c) is at p + c.  step() moves to R' + 1.
template <int N>
struct KRow {
  int p, d;
  __device__ __forceinline__ void init(int t, int Rk) {
    p = Rows<N>::off(4 * Rk + t) - 4 * Rk;
    d = 4 * N - 4 - 4 * t - 16 * Rk;
  }
  __device__ __forceinline__ void step() {
    p += d;
    d -= 16;
  }
};

// packed offsets of the first stored element of rows r0 .. r0 + B - 1 (r0 a
// multiple of 4): one Rows::off and an add per row instead of B closed forms
// (the per-block-row offsets were ~10 % of the kernel's instructions)
template <int N, int B>
__device__ __forceinline__ void row_starts(int r0, int (&o)[B]) {
  const int w0 = N - r0;  // stored length of rows r0 .. r0 + 3
  const int b0 = Rows<N>::off(r0);
#pragma unroll
  for (int i = 0; i < B; ++i) o[i] = i < 4 ? b0 + i * w0 : b0 + 4 * w0 + (i - 4) * (w0 - 4);
}

// row-major n x n (upper part) -> packed rows, cp.async 16-byte units; full
// rows are walked (division by the compile-time half-width) and the chunks
// left of each row's first stored column are skipped
// NR < N: the real problem is NR x NR (ld NR), padded to N with the identity
// (A_pad = diag(A, I) -> X_pad = diag(X, I), exactly)
template <int N, int G, int NR = N>
__device__ __forceinline__ void load_rows(double* xs, const double* __restrict__ src, int rank) {
  // warps over rows, lanes over the row's 16-byte pairs from its first stored
  // column: no per-element division and no iterations over the lower part
  // (when a row's pair count is not a multiple of 32 above 32, the flattened
  // loop keeps every lane busy instead)
  constexpr int H = N / 2;
  if constexpr (H <= 32 || H % 32 == 0 || H >= LAGEN_ROWS_ROWLOOP_H) {
    constexpr int NWG = G / 32;
    const int w = rank >> 5, lane = rank & 31;
    for (int r = w; r < N; r += NWG) {
      const int c0 = 4 * (r >> 2);
      double* row = xs + Rows<N>::off(r) - c0;
      for (int c = c0 + 2 * lane; c < N; c += 64) {
        if (NR == N || (r < NR && c < NR))
          cp_async16(row + c, src + r * NR + c);
        else
          *reinterpret_cast<double2*>(row + c) = make_double2(r == c ? 1.0 : 0.0, r == c + 1 ? 1.0 : 0.0);
      }
    }
  } else {
    for (int u = rank; u < N * H; u += G) {
      const int r = u / H, c = 2 * (u - r * H);
      if (c >= 4 * (r >> 2)) {
        if (NR == N || (r < NR && c < NR))
          cp_async16(xs + Rows<N>::at(r, c), src + r * NR + c);
        else
          *reinterpret_cast<double2*>(xs + Rows<N>::at(r, c)) = make_double2(r == c ? 1.0 : 0.0, r == c + 1 ? 1.0 : 0.0);
      }
    }
  }
}

// S1 part: X(t0:t0+B, t0:t0+B) (upper) -= sum over rows kk in [4 ks0, 4 ks1)
// of X[kk][t0..]^T X[kk][t0..]; one warp, 4 accumulator chains
template <int N, int B>
__device__ __forceinline__ void s1_tile(double* xs, int t0, int ks0, int ks1) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int ga = (B == 8 || g < B) ? g : (g & 3);
  double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
  KRow<N> kr;
  kr.init(t, ks0);
  int ks = ks0;
  for (; ks + 4 <= ks1; ks += 4) {
    double a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = xs[kr.p + t0 + ga];
      kr.step();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(c0[u], c1[u], a[u], a[u]);
  }
  // remainder (< 4 k-steps) with static accumulator indices: a runtime
  // index (u & 3) put c0 / c1 in local memory for the whole tile
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    if (ks + u < ks1) {
      const double a = xs[kr.p + t0 + ga];
      kr.step();
      dmma(c0[u], c1[u], a, a);
    }
  }
  const double x0 = (c0[0] + c0[1]) + (c0[2] + c0[3]);
  const double x1 = (c1[0] + c1[1]) + (c1[2] + c1[3]);
  const int i = g, j = 2 * t;
  if (i < B && j < B) {
    const int o = Rows<N>::at(t0 + i, t0 + j);
    if (i <= j) xs[o] -= x0;
    if (i <= j + 1 && j + 1 < B) xs[o + 1] -= x1;
  }
}

// S3 block: rows r0..r0+B-1, columns [c0, c0 + 32) of X12 (absolute columns),
// k-steps [ks0, ks1); accumulators returned (even / odd sets folded)
template <int N, int B>
__device__ __forceinline__ void s3_block(const double* xs, int r0, int c0, int cend, int ks0, int ks1, double c0a[4],
                                         double c1a[4]) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int ga = (B == 8 || g < B) ? g : (g & 3);
  double e0[4] = {0, 0, 0, 0}, e1[4] = {0, 0, 0, 0};
#pragma unroll
  for (int u = 0; u < 4; ++u) c0a[u] = c1a[u] = 0.0;
  bool v[4];
  int cb[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = c0 + 8 * u + g;
    v[u] = c < cend;
    cb[u] = v[u] ? c : r0;  // clamped to a valid column (result discarded)
  }
  KRow<N> kr;
  kr.init(t, ks0);
  int ks = ks0;
  for (; ks + 2 <= ks1; ks += 2) {
    const double a = xs[kr.p + r0 + ga];
    double bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) bv[u] = xs[kr.p + cb[u]];
    kr.step();
    const double a2 = xs[kr.p + r0 + ga];
    double bw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) bw[u] = xs[kr.p + cb[u]];
    kr.step();
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(c0a[u], c1a[u], a, bv[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(e0[u], e1[u], a2, bw[u]);
  }
  if (ks < ks1) {
    const double a = xs[kr.p + r0 + ga];
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(c0a[u], c1a[u], a, xs[kr.p + cb[u]]);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    c0a[u] += e0[u];
    c1a[u] += e1[u];
  }
}

template <int N, int B>
__device__ __forceinline__ void s3_write(double* xs, int r0, int c0, int cend, const double c0a[4],
                                         const double c1a[4]) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  if (g >= B) return;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = c0 + 8 * u + 2 * t;
    if (c < cend) {
      double2* p = reinterpret_cast<double2*>(xs + Rows<N>::at(r0 + g, c));
      double2 w = *p;
      w.x -= c0a[u];
      w.y -= c1a[u];
      *p = w;
    }
  }
}

// S3 over warps [w0, w0 + nw) (wi = this warp's index in that set); k split
// across idle warps, partials reduced in fixed order through scratch.
template <int N, int B, int WG>
__device__ __forceinline__ void s3(double* xs, int r0, int wi, int nw, const Grp& gr, int bar_id, int bar_thr,
                                   int split_mode) {
  const int cs = r0 + B, cend = N;
  if (cs >= cend || r0 == 0) return;
  const int nblk = (cend - cs + 31) >> 5;
  const int nks = r0 >> 2;
  int ks = (gr.scr != nullptr && nblk < nw) ? min(nw / nblk, nks / 4) : 1;
  if (split_mode == 0 || (split_mode == 2 && nblk > 1)) ks = 1;
  if (ks <= 1) {
    for (int bk = wi; bk < nblk; bk += nw) {
      double a0[4], a1[4];
      s3_block<N, B>(xs, r0, cs + 32 * bk, cend, 0, nks, a0, a1);
      s3_write<N, B>(xs, r0, cs + 32 * bk, cend, a0, a1);
    }
    return;
  }
  auto bar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_thr) : "memory"); };
  const int blk = wi % nblk, sl = wi / nblk;
  const bool active = wi < nblk * ks;
  const int lane = lane_id();
  double a0[4], a1[4];
  if (active) {
    s3_block<N, B>(xs, r0, cs + 32 * blk, cend, (nks * sl) / ks, (nks * (sl + 1)) / ks, a0, a1);
    if (sl > 0) {
      double* sp = gr.scr + ((sl - 1) * nblk + blk) * 256 + lane * 8;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sp[2 * u] = a0[u];
        sp[2 * u + 1] = a1[u];
      }
    }
  }
  bar();
  if (active && sl == 0) {
    for (int s2 = 1; s2 < ks; ++s2) {
      const double* sp = gr.scr + ((s2 - 1) * nblk + blk) * 256 + lane * 8;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0[u] += sp[2 * u];
        a1[u] += sp[2 * u + 1];
      }
    }
    s3_write<N, B>(xs, r0, cs + 32 * blk, cend, a0, a1);
  }
  bar();
}

// CHOL leaf (B <= 8) on one warp: every lane factors the block in registers;
// lane r < B writes row r (zeros left of the diagonal), its reciprocal pivot
// to rsb[r] and the factor row-major to rsb[16 + r * B + c].
template <int N, int B>
__device__ __forceinline__ void leaf(double* xs, int r0, double* rsb, int* flag) {
  const int lane = lane_id();
  double t[B][B];
  int os[B];
  row_starts<N, B>(r0, os);
#pragma unroll
  for (int r = 0; r < B; ++r) {
    // row r0 + r is stored from column 4 * floor((r0 + r) / 4) = r0 + (r & ~3)
    const int o = os[r];
#pragma unroll
    for (int c = 0; c < B; c += 2) {
      if (c < (r & ~3)) {
        t[r][c] = t[r][c + 1] = 0.0;
        continue;
      }
      const double2 v = *reinterpret_cast<const double2*>(xs + o + c - (r & ~3));
      t[r][c] = c >= r ? v.x : 0.0;
      t[r][c + 1] = c + 1 >= r ? v.y : 0.0;
    }
  }
  double rs[B];
  bool bad = false, nonfinite = false;
  int badi = 0;
#pragma unroll
  for (int i = 0; i < B; ++i) {
    const double piv = t[i][i];
    if (!bad && piv <= 0.0) {
      bad = true;
      badi = i;
    }
    nonfinite = nonfinite || !isfinite(piv);
    rs[i] = rsqrt_nr(piv);
    t[i][i] = piv * rs[i];
#pragma unroll
    for (int c = i + 1; c < B; ++c) t[i][c] *= rs[i];
#pragma unroll
    for (int r = i + 1; r < B; ++r)
#pragma unroll
      for (int c = r; c < B; ++c) t[r][c] = fma(-t[i][r], t[i][c], t[r][c]);
  }
  // first non-positive pivot -> its index + 1 (kernels.py:87-88); a NaN or
  // infinite pivot (which every NaN / Inf of X reaches: each upper entry
  // enters its column's diagonal through S1's square) -> -1 (verify.py:301)
  if (lane == 0 && *flag == 0) *flag = bad ? r0 + badi + 1 : (nonfinite ? -1 : 0);
  double row[B];
  double rsr = 0.0;
#pragma unroll
  for (int c = 0; c < B; ++c) row[c] = 0.0;
#pragma unroll
  for (int r = 0; r < B; ++r) {
    const bool me = lane == r;
#pragma unroll
    for (int c = r; c < B; ++c) row[c] = me ? t[r][c] : row[c];
    rsr = me ? rs[r] : rsr;
  }
  if (lane < B) {
    const int cs = lane & ~3;  // first stored column of this row (relative to r0)
    const int o = Rows<N>::at(r0 + lane, r0 + cs);
#pragma unroll
    for (int c = 0; c < B; c += 2)
      if (c >= cs) *reinterpret_cast<double2*>(xs + o + c - cs) = make_double2(row[c], row[c + 1]);
#pragma unroll
    for (int c = 0; c < B; ++c) rsb[16 + lane * B + c] = row[c];
    rsb[lane] = rsr;
  }
}

// S4: X12 := X11^{-T} X12, threads own columns
template <int N, int B>
__device__ __forceinline__ void trsm(double* xs, int r0, const double* rsb, int rank, int nthr) {
  int o[B];
  row_starts<N, B>(r0, o);
#pragma unroll
  for (int i = 0; i < B; ++i) o[i] -= r0 + (i & ~3);  // -> element (r0 + i, c) at o[i] + c
  for (int c = r0 + B + rank; c < N; c += nthr) {
    double w[B];
#pragma unroll
    for (int i = 0; i < B; ++i) w[i] = xs[o[i] + c];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      double v = w[i];
#pragma unroll
      for (int l = 0; l < i; ++l) v = fma(-rsb[16 + l * B + i], w[l], v);
      w[i] = v * rsb[i];
    }
#pragma unroll
    for (int i = 0; i < B; ++i) xs[o[i] + c] = w[i];
  }
}

// block row [r0, r0 + B) -> X (row-major, zeros left of the diagonal)
template <int N, int B, int NR = N>
__device__ __forceinline__ void store_rows(double* __restrict__ dst, const double* xs, int r0, int rank, int nthr,
                                           int bsz = B) {
  // warps over the block row's rows, lanes over 16-byte pairs (coalesced)
  const int nb = r0 + bsz <= NR ? bsz : NR - r0;  // real rows of this block row
  constexpr int H = NR / 2;
  if constexpr (H <= 32 || H % 32 == 0 || (H >= LAGEN_ROWS_STORE_ROWLOOP_H && H != 42 && H != 36)) {  // (n = 72, 84 measured slower)
    const int w = rank >> 5, nw = nthr >> 5, lane = rank & 31;
    // r0 is a multiple of 4: row r0 + i starts at off(r0) + i (N - r0) - 4 max(i - 4, 0)
    const int b0 = Rows<N>::off(r0), w0 = N - r0;
    for (int i = w; i < nb; i += nw) {
      const int r = r0 + i, c0 = r0 + (i & ~3);
      const int i4 = i > 4 ? i - 4 : 0;
      const double* row = xs + b0 + i * w0 - 4 * i4 - c0;
      double* drow = dst + r * NR;
#pragma unroll
      for (int k = 0; k < (NR + 63) / 64; ++k) {
        const int c = 2 * lane + 64 * k;
        if (64 * k + 64 <= NR || c < NR) {
          double2 v = make_double2(0.0, 0.0);
          if (c >= c0) v = *reinterpret_cast<const double2*>(row + c);
          __stcs(reinterpret_cast<double2*>(drow + c), v);
        }
      }
    }
  } else {
    for (int u = rank; u < nb * H; u += nthr) {
      const int i = u / H, r = r0 + i, c = 2 * (u - i * H);
      double2 v = make_double2(0.0, 0.0);
      if (c >= 4 * (r >> 2)) v = *reinterpret_cast<const double2*>(xs + Rows<N>::at(r, c));
      __stcs(reinterpret_cast<double2*>(dst + r * NR + c), v);
    }
  }
}

#ifdef LAGEN_ROWS_PROF
__device__ unsigned long long prof_buf[16];
#endif

// Measured per size (index n / 4; b = 4 and b = 8): warps per problem and
// launch mode = k-split (1) | work split << 2.  Sweep of WG in {1, 2, 4} x
// modes {1, 5, 9, 13} over n = 36..128 at full 256 MiB batches
// (LAGEN_ROWS_WG / LAGEN_ROWS_MODE + tools/engine_compare.py,
// profiles/r01_rows_wg_modes.txt; the b = 8 row re-measured after the leaf
// warp placement and S1 fixes, profiles/r01_rows_tune.txt, which moved
// n = 56, 64, 72, 80, 112); sizes below 36 use the column engine.
constexpr unsigned char kRowsWG[2][33] = {{1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 1, 1, 2, 1, 1, 2, 1, 2, 2, 2, 2, 2, 2, 2, 2, 2, 4, 4, 4},
                                            {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 1, 2, 1, 2, 1, 2, 1, 2, 1, 4, 1, 4, 1, 4}};
constexpr unsigned char kRowsMode[2][33] = {{1, 1, 1, 1, 1, 1, 1, 1, 1, 13, 1, 13, 13, 9, 5, 5, 13, 1, 13, 5, 1, 5, 5, 5, 5, 5, 5, 5, 5, 5, 13, 13, 13},
                                              {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 5, 1, 5, 1, 5, 1, 5, 1, 9, 1, 9, 1, 9, 1, 9, 1, 9, 1, 13, 1, 13, 1, 13}};
inline int rows_wg(int n, int b) { return kRowsWG[b == 8][n / 4]; }
inline int default_mode(int n, int b) { return kRowsMode[b == 8][n / 4]; }
// padded instances (n = 4 mod 8 on the b = 8 kernel of n + 4) where their own
// sweep (profiles/r01_rowspad_tune.txt) picked a different setting than the
// unpadded size: {n, WG, mode}
constexpr int kRowsPadPick[3][3] = {{60, 2, 9}, {76, 2, 13}, {92, 4, 13}};
inline int pad_wg(int nr) {
  for (const auto& e : kRowsPadPick)
    if (e[0] == nr) return e[1];
  return rows_wg(nr + 4, 8);
}
inline int pad_mode(int nr) {
  for (const auto& e : kRowsPadPick)
    if (e[0] == nr) return e[2];
  return default_mode(nr + 4, 8);
}

// mixed-block instances (n = 4 mod 8): {n, WG, mode} measured over
// WG in {1, 2, 4} x modes {1, 5, 9, 13} at the 256 MiB batches
// (tools/gpu_rowsmix_tune.sh, profiles/r02_rowsmix_tune.txt)
constexpr int kRowsMixPick[15][3] = {{12, 1, 5},  {20, 1, 9},   {28, 1, 13},  {36, 1, 9},   {44, 1, 5},
                                      {52, 1, 1},  {60, 1, 1},   {68, 1, 13},  {76, 2, 13},  {84, 2, 13},
                                      {92, 2, 13}, {100, 2, 9},  {108, 2, 9},  {116, 4, 1},  {124, 4, 13}};
inline int mix_wg(int n) {
  for (const auto& e : kRowsMixPick)
    if (e[0] == n) return e[1];
  return pad_wg(n);
}
inline int mix_mode(int n) {
  for (const auto& e : kRowsMixPick)
    if (e[0] == n) return e[2];
  return pad_mode(n);
}

// F4 ("mixed blocks", n = 4 mod 8): the same statements over the partition
// 4, 8, 8, ..., 8 — a first 4 x 4 block row, then the b = 8 schedule from row
// 4 on (the loop invariant of v1 holds for any partition sequence, so the
// result is v1's to rounding).  It replaces running such sizes as the
// identity-padded n + 4 problem (15-25 % slower than its neighbours: more
// shared memory per problem and (n + 4)^3 work).
template <int N, int B, int WG_, int NR = N, bool F4 = false>
__global__ void __launch_bounds__(RPolicy<N, WG_>::WARPS * 32, 1)
    chol_rows_kernel(const double* __restrict__ A, double* __restrict__ X, int* __restrict__ info,
                     long long batch, int mode) {
  const int split_mode = mode & 3, work_split = (mode >> 2) & 3;
  using P = RPolicy<N, WG_>;
  static_assert(P::SLOT == Rows<N>::DOUBLES, "packed rows and upper tiles have the same size");
  static_assert(!F4 || (B == 8 && N % 8 == 4 && NR == N && N >= 12), "mixed blocks: n = 4 mod 8 on the b = 8 schedule");
  constexpr int WG = P::WG, G = WG * 32, NB = F4 ? 1 + (N - 4) / 8 : N / B;
  extern __shared__ double smem[];
  int* gflag = reinterpret_cast<int*>(smem + (size_t)P::P * P::DB * P::SLOT);
  double* rsb_all = reinterpret_cast<double*>(gflag + 32);
  double* scr_all = rsb_all + P::P * P::RSB;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  Grp gr;
  gr.id = warp / WG;
  gr.wig = (warp % WG + WG - eng::lead_warp(gr.id, WG)) % WG;  // 0: the leaf warp
  gr.rank = gr.wig * 32 + lane;
  gr.rsb = rsb_all + P::RSB * gr.id;
  gr.scr = P::SCR ? scr_all + (size_t)P::SCR * gr.id : nullptr;
  gr.prof = nullptr;
  // warps 1..WG-1 of group g: named barrier 1 + P + g (group barriers: 1 .. P)
  const int subbar = (WG > 2 && 1 + P::P + gr.id <= 15) ? 1 + P::P + gr.id : 0;
  if (!subbar) gr.scr = (WG > 2) ? nullptr : gr.scr;  // split-K needs the sub-group barrier
  auto slot_at = [&](int d) { return smem + ((size_t)gr.id * P::DB + (d % P::DB)) * P::SLOT; };
  constexpr long long NN = (long long)NR * NR;
  const long long stride = (long long)gridDim.x * P::P;
  // slot-major problem order: round t runs problems [t * stride, (t + 1) * stride)
  // with slot g of every CTA before slot g + 1 of any, so a partial last round
  // puts 1-2 problems on every SM (each faster with less contention for the
  // SM's FP64 / DMMA pipes) instead of full slots on a few SMs
  long long prob = LAGEN_ROWS_SPREAD ? (long long)gr.id * gridDim.x + blockIdx.x
                                     : (long long)blockIdx.x * P::P + gr.id;
  if (prob < batch) {
    load_rows<N, G, NR>(slot_at(0), A + prob * NN, gr.rank);
    cp_async_commit();
  }
  int cur = 0;
  for (; prob < batch; prob += stride) {
    const long long off = prob * NN;
    const long long nxt = prob + stride;
    double* xs = slot_at(cur);
    if constexpr (P::DB == 2) {
      if (nxt < batch) {
        load_rows<N, G, NR>(slot_at(cur ^ 1), A + nxt * NN, gr.rank);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
    } else {
      cp_async_wait<0>();
    }
    if (gr.rank == 0) gflag[gr.id] = 0;
    gsync<WG>(gr);
    int flag = 0;
#ifdef LAGEN_ROWS_PROF
    long long tp0 = clock64();
    auto tick = [&](int slot) {
      if (blockIdx.x == 0 && gr.id == 0 && lane == 0 && gr.wig < 2) {
        const long long t1 = clock64();
        atomicAdd(reinterpret_cast<unsigned long long*>(X) + 0, 0ull);  // keep ordering
        prof_buf[gr.wig * 8 + slot] += t1 - tp0;
        tp0 = t1;
      }
    };
#else
    auto tick = [](int) {};
#endif
    // one block row: BB its size (compile time), pB the previous one's
    auto iter = [&](auto bc, const int r0, const int pB) {
      constexpr int BB = decltype(bc)::value;
      if constexpr (WG == 1) {
        if (r0 > 0) s1_tile<N, BB>(xs, r0, 0, r0 >> 2);
        __syncwarp();
        leaf<N, BB>(xs, r0, gr.rsb, &flag);
        s3<N, BB, WG>(xs, r0, 0, 1, gr, 0, 32, split_mode);
        __syncwarp();
        trsm<N, BB>(xs, r0, gr.rsb, gr.rank, G);
        __syncwarp();
        store_rows<N, BB, NR>(X + off, xs, r0, gr.rank, G);
      } else {
        // level A.  warp 0: the last block row's S1 contribution (K = pB; the
        // rows above were applied one iteration ahead), then the leaf.
        // warps 1..WG-1: store block row k-1, S3 of this block row, and the
        // look-ahead S1 part of block k+1 (all rows above r0 are final).
        // who takes the store and the look-ahead beside warp 0's leaf chain
        // (work split, tuned per size: default_mode()) — 0: warps 1..;
        // 1: warp 0; 2: warp 0 stores, warps 1.. look ahead; 3: no look-ahead
        // (warp 0 runs the whole S1), warps 1.. store
        const bool ahead = work_split != 3;
        const bool w0_store = work_split == 1 || work_split == 2, w0_look = work_split == 1;
        if (gr.wig == 0) {
          if (r0 > 0) s1_tile<N, BB>(xs, r0, ahead ? (r0 - pB) >> 2 : 0, r0 >> 2);
          __syncwarp();
          leaf<N, BB>(xs, r0, gr.rsb, &flag);
          if (w0_store && r0 > 0) store_rows<N, B, NR>(X + off, xs, r0 - pB, lane, 32, pB);
          if (ahead && w0_look && r0 + BB < N && r0 > 0) s1_tile<N, B>(xs, r0 + BB, 0, r0 >> 2);
        } else {
          if (!w0_store && r0 > 0) store_rows<N, B, NR>(X + off, xs, r0 - pB, gr.rank - 32, 32 * (WG - 1), pB);
          if constexpr (WG == 2) {
            s3<N, BB, WG>(xs, r0, 0, 1, gr, 0, 32, split_mode);
          } else {
            s3<N, BB, WG>(xs, r0, gr.wig - 1, WG - 1, gr, subbar, 32 * (WG - 1), split_mode);
          }
          if (ahead && !w0_look && r0 + BB < N && r0 > 0 && gr.wig == WG - 1) s1_tile<N, B>(xs, r0 + BB, 0, r0 >> 2);
        }
        tick(0);
        gsync<WG>(gr);
        tick(1);
        trsm<N, BB>(xs, r0, gr.rsb, gr.rank, G);
        tick(2);
        gsync<WG>(gr);
        tick(3);
      }
    };
    if constexpr (F4) {
      iter(std::integral_constant<int, 4>{}, 0, 4);
#pragma unroll 1
      for (int k = 1; k < NB; ++k) iter(std::integral_constant<int, 8>{}, 8 * k - 4, k == 1 ? 4 : 8);
    } else {
#pragma unroll 1
      for (int k = 0; k < NB; ++k) iter(std::integral_constant<int, B>{}, k * B, B);
    }
    if constexpr (WG > 1) store_rows<N, B, NR>(X + off, xs, N - B, gr.rank, G);
    if (gr.wig == 0 && lane == 0 && flag) gflag[gr.id] = flag;
    gsync<WG>(gr);
    if (info && gr.rank == 0) info[prob] = gflag[gr.id];
    if constexpr (P::DB == 1) {
      gsync<WG>(gr);  // slot reads done before it is refilled
      if (nxt < batch) {
        load_rows<N, G, NR>(slot_at(0), A + nxt * NN, gr.rank);
        cp_async_commit();
      }
    } else {
      cur ^= 1;
    }
  }
}

}  // namespace cr
}  // namespace lagen
