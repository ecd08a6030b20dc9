// chol_gang.cuh — the "gang engine": Cholesky variant v1 (left-looking,
// b = 8) on a gang of P problems per CTA that advance in lockstep, with the
// warps of the CTA split by role and by SM sub-partition.
//
// Variant v1 (the reference's enumeration, variants_table.json):
//     S1: X11 -= X01^T X01      (upper target)
//     S2: X11 := CHOL(X11)                        (kernels.py:79-97)
//     S3: X12 -= X01^T X02                        (kernels.py:16-34)
//     S4: X12 := TRSM(X11^T, X12)                 (kernels.py:47-60)
// per block row k of 8 (verify.py:245-297).
//
// Why a gang.  The rows engine (chol_rows.cuh) gives every problem its own
// warp group; its 8x8 CHOL leaf is a ~750-cycle dependent chain that every
// lane of a warp repeats, and on a loaded SM it measured ~2.2k cycles because
// its FP64 instructions queue behind the 16-cycle DMMAs of the update warps
// on the same sub-partition (profiles/r01_chol_lookahead.md).  Here
//   * the P problems of a CTA run the same block row at the same time, so ONE
//     leaf warp factors 4 diagonal blocks at once (8 lanes per problem) —
//     the chain is paid once per 4 problems;
//   * warp w sits on sub-partition w & 3: sub-partition 0 holds only the leaf
//     warps and the store / load warps (LSU work), sub-partitions 1..3 hold
//     the DMMA warps, so the leaf chain never waits for the FP64 pipe;
//   * the bulk updates of all P problems (S3 strips, look-ahead S1 tiles) are
//     one item list dealt over the DMMA warps.
// Inputs arrive by cp.async.bulk (TMA, one copy per matrix row) on one
// mbarrier per block row: block row k is first touched in iteration k, so the
// solve starts as soon as block row 0 has landed and the rest of the load
// overlaps the early iterations.  Finished block rows stream to HBM from the
// store warps while the next iteration runs.
//
// Shared-memory layout of one problem (GL<N>): packed upper rows, row r keeps
// columns [4 floor(r/4), n); the 4 rows of a group share a pitch = 4 (mod 8)
// doubles (4 doubles of padding for every second group), so the m8n8k4
// fragments of a k-step (4 rows x 8 columns) are bank-conflict free.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lagen {
namespace gang {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "GANG_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra GANG_DONE;\n"
      "bra GANG_WAIT;\n"
      "GANG_DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// packed upper rows with conflict-free pitches (N % 8 == 0)
template <int N>
struct GL {
  static_assert(N % 8 == 0 && N >= 8, "gang engine: n padded to a multiple of 8");
  __host__ __device__ static constexpr int pitch(int R) { return N - 4 * R + ((R & 1) ? 0 : 4); }
  __host__ __device__ static constexpr int goff(int R) {
    const int j = R >> 1;
    return 8 * N * j - 32 * j * (j - 1) + ((R & 1) ? 4 * (N - 8 * j + 4) : 0);
  }
  static constexpr int DOUBLES = goff(N / 4);
  // first element of row r (column 4 floor(r/4))
  __host__ __device__ static constexpr int row0(int r) { return goff(r >> 2) + (r & 3) * pitch(r >> 2); }
  // element (r, c), c >= 4 floor(r/4)
  __host__ __device__ static constexpr int at(int r, int c) { return row0(r) + c - 4 * (r >> 2); }
};

// Row pointers of lane t for k-steps 2j (rows 8j + t) and 2j + 1 (rows
// 8j + 4 + t): element (row, c) is at pe + c / po + c.  next() moves to j + 1.
template <int N>
struct KPair {
  int pe, po, de;
  __device__ __forceinline__ void init(int t, int j) {
    const int g = 8 * N * j - 32 * j * (j - 1), w = N - 8 * j + 4;
    pe = g + t * w - 8 * j;
    po = g + 4 * w + t * (w - 8) - 8 * j - 4;
    de = 8 * N - 64 * j - 8 * t - 8;
  }
  __device__ __forceinline__ void next() {
    pe += de;
    po += de - 32;
    de -= 64;
  }
};

// problems per CTA (P), warps per SM sub-partition (Q), CTAs per SM (MINB).
// Sub-partition 0 holds the panel warps (NLEAF of them run the leaves) and NIO
// load / store warps; sub-partitions 1..3 hold the 3 Q bulk (DMMA) warps.
template <int N, int P_, int Q_, int MINB_>
struct GCfg {
  static constexpr int P = P_, Q = Q_, MINB = MINB_;
  static constexpr int NB = N / 8;
  static constexpr int NLEAF = (P + 3) / 4;
  static constexpr int NIO = 0;
  static constexpr int NPW = Q;            // panel warps
  static constexpr int NHELP = Q - NLEAF;  // panel warps without a leaf: they issue the TMA loads / stores
  static_assert(NHELP >= 1, "sub-partition 0 needs a warp beside the leaf warps for the loads / stores");
  static constexpr int LA = 3;             // block rows loaded ahead of the iteration
  static constexpr int NDW = 3 * Q;
  static constexpr int WARPS = 4 * Q;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int SLOT = GL<N>::DOUBLES;
  static constexpr int RSB = 64;  // V = X11^{-1} of one diagonal block
  // slots, V buffers (two per problem: the S4 of block row k-1 runs beside the
  // leaf of block k), mbarriers, flags
  static constexpr size_t SMEM = (size_t)P * SLOT * 8 + (size_t)2 * P * RSB * 8 + (size_t)NB * 8 + 16 * sizeof(int);
  static_assert(SMEM * MINB <= 227 * 1024, "gang does not fit");
};

// 8x8 tile D(r1.., r1..) -= sum over k-step pairs [j0, j1) of X[rows]^T X[rows]
// (upper part written); one warp, 4 accumulator chains
template <int N>
__device__ __forceinline__ void s1_tile(double* xs, int r1, int j0, int j1, int lane) {
  const int g = lane >> 2, t = lane & 3;
  double c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
  KPair<N> kp;
  kp.init(t, j0);
  int j = j0;
  for (; j + 2 <= j1; j += 2) {
    const double a0 = xs[kp.pe + r1 + g], a1 = xs[kp.po + r1 + g];
    kp.next();
    const double a2 = xs[kp.pe + r1 + g], a3 = xs[kp.po + r1 + g];
    kp.next();
    dmma(c0[0], c1[0], a0, a0);
    dmma(c0[1], c1[1], a1, a1);
    dmma(c0[2], c1[2], a2, a2);
    dmma(c0[3], c1[3], a3, a3);
  }
  if (j < j1) {
    const double a0 = xs[kp.pe + r1 + g], a1 = xs[kp.po + r1 + g];
    dmma(c0[0], c1[0], a0, a0);
    dmma(c0[1], c1[1], a1, a1);
  }
  const double x0 = (c0[0] + c0[1]) + (c0[2] + c0[3]);
  const double x1 = (c1[0] + c1[1]) + (c1[2] + c1[3]);
  const int i = g, c = 2 * t;
  double2* p = reinterpret_cast<double2*>(xs + GL<N>::at(r1 + i, r1 + (i & 4)) + c - (i & 4));
  if (c + 1 >= i && c >= (i & 4)) {  // the pair holds an upper entry and is stored
    double2 w = *p;
    if (i <= c) w.x -= x0;
    w.y -= x1;
    *p = w;
  }
}

// S3 block: rows r0..r0+7, NT 8-column tiles from column c0 (< cend) take
// the contributions of the k-step pairs [j0, j1) (rows 8 j0 .. 8 j1 - 1)
template <int N, int NT>
__device__ __forceinline__ void s3_block(double* xs, int r0, int c0, int cend, int j0, int j1, int lane) {
  const int g = lane >> 2, t = lane & 3;
  double ce0[NT], ce1[NT], co0[NT], co1[NT];
  int cb[NT];
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    ce0[u] = ce1[u] = co0[u] = co1[u] = 0.0;
    const int c = c0 + 8 * u + g;
    cb[u] = c < cend ? c : r0;  // clamped to a valid column (result discarded)
  }
  KPair<N> kp;
  kp.init(t, j0);
#pragma unroll 2
  for (int j = j0; j < j1; ++j) {
    const double ae = xs[kp.pe + r0 + g], ao = xs[kp.po + r0 + g];
    double be[NT], bo[NT];
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      be[u] = xs[kp.pe + cb[u]];
      bo[u] = xs[kp.po + cb[u]];
    }
    kp.next();
#pragma unroll
    for (int u = 0; u < NT; ++u) dmma(ce0[u], ce1[u], ae, be[u]);
#pragma unroll
    for (int u = 0; u < NT; ++u) dmma(co0[u], co1[u], ao, bo[u]);
  }
  // row r0 + g of the strip, columns c0 + 8u + 2t, +1
  double* row = xs + GL<N>::at(r0 + g, r0 + (g & 4)) - (r0 + (g & 4));
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    const int c = c0 + 8 * u + 2 * t;
    if (c < cend) {
      double2* p = reinterpret_cast<double2*>(row + c);
      double2 w = *p;
      w.x -= ce0[u] + co0[u];
      w.y -= ce1[u] + co1[u];
      *p = w;
    }
  }
}

// CHOL leaves of up to 4 problems on one warp: lanes 8q..8q+7 factor problem
// q's 8x8 diagonal block redundantly in registers (kernels.py:79-97); lane j
// of the group writes row j (zeros left of the diagonal) and row j of
// V = X11^{-1} (upper, row-major in vb: the S4 coefficient, see trsm_block)
template <int N>
__device__ __forceinline__ void leaf4(double* xs, double* vb, int* flag, int r0, int j, bool act) {
  double t[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const double* row = xs + GL<N>::at(r0 + r, r0 + (r & 4)) - (r & 4);
#pragma unroll
    for (int c = 0; c < 8; c += 2) {
      if (c + 1 < r) {
        t[r][c] = t[r][c + 1] = 0.0;
        continue;
      }
      const double2 v = *reinterpret_cast<const double2*>(row + c);
      t[r][c] = c >= r ? v.x : 0.0;
      t[r][c + 1] = v.y;
    }
  }
  double rs[8];
  bool bad = false, nonfinite = false;
  int badi = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double piv = t[i][i];
    if (!bad && piv <= 0.0) {
      bad = true;
      badi = i;
    }
    nonfinite = nonfinite || !isfinite(piv);
    rs[i] = rsqrt(piv);
    t[i][i] = piv * rs[i];
#pragma unroll
    for (int c = i + 1; c < 8; ++c) t[i][c] *= rs[i];
#pragma unroll
    for (int r = i + 1; r < 8; ++r)
#pragma unroll
      for (int c = r; c < 8; ++c) t[r][c] = fma(-t[i][r], t[i][c], t[r][c]);
  }
  // first non-positive pivot -> index + 1 (kernels.py:87-88); NaN / Inf pivot
  // (every NaN / Inf of X reaches its column's diagonal through S1) -> -1
  // (verify.py:301-302)
  if (act && j == 0 && *flag == 0) *flag = bad ? r0 + badi + 1 : (nonfinite ? -1 : 0);
  // row j of V = T^{-1}: v[c] = 0 (c < j), 1 / t_jj (c = j),
  // -(sum_{m < c} v[m] t[m][c]) / t_cc (c > j); same code in every lane
  double v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double sacc = 0.0;
#pragma unroll
    for (int m = 0; m < c; ++m) sacc = fma(v[m], t[m][c], sacc);
    v[c] = c == j ? rs[c] : -rs[c] * sacc;
  }
  double row[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) row[c] = 0.0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const bool me = j == r;
#pragma unroll
    for (int c = r; c < 8; ++c) row[c] = me ? t[r][c] : row[c];
  }
  if (act) {
    double* dst = xs + GL<N>::at(r0 + j, r0 + (j & 4)) - (j & 4);
#pragma unroll
    for (int c = 0; c < 8; c += 2)
      if (c >= (j & 4)) *reinterpret_cast<double2*>(dst + c) = make_double2(row[c], row[c + 1]);
#pragma unroll
    for (int c = 0; c < 8; c += 2) *reinterpret_cast<double2*>(vb + j * 8 + c) = make_double2(v[c], v[c + 1]);
  }
}

// S4 on NT 8-column tiles of block row kk from column c0 (< cend):
// X12 := X11^{-T} X12 as the product V^T W on the FP64 tensor path, V = X11^{-1}
// from the leaf (kernels.py:47-60 solves the same triangular system by
// substitution; the diagonal blocks are 8x8, so the explicit inverse costs
// 8 more dependent steps once per block instead of 36 FMAs per column)
template <int N, int NT>
__device__ __forceinline__ void trsm_block(double* xs, int kk, int c0, int cend, const double* vb, int lane) {
  const int g = lane >> 2, t = lane & 3;
  KPair<N> kp;
  kp.init(t, kk);
  const double ae = vb[t * 8 + g], ao = vb[(t + 4) * 8 + g];  // A[m = g][k = t] = V[t][g]
  double x0[NT], x1[NT];
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    const int c = c0 + 8 * u + g;
    const int cc = c < cend ? c : c0;
    const double be = xs[kp.pe + cc], bo = xs[kp.po + cc];
    x0[u] = x1[u] = 0.0;
    dmma(x0[u], x1[u], ae, be);
    dmma(x0[u], x1[u], ao, bo);
  }
  double* row = xs + GL<N>::row0(8 * kk + g) - (8 * kk + (g & 4));
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    const int c = c0 + 8 * u + 2 * t;
    if (c < cend) *reinterpret_cast<double2*>(row + c) = make_double2(x0[u], x1[u]);
  }
}

template <int N>
__device__ __forceinline__ void trsm_blocks(double* xs, int kk, int c0, int cend, const double* vb, int lane) {
  const int nt = (cend - c0 + 7) >> 3;
  if (nt >= 4) trsm_block<N, 4>(xs, kk, c0, cend, vb, lane);
  else if (nt == 3) trsm_block<N, 3>(xs, kk, c0, cend, vb, lane);
  else if (nt == 2) trsm_block<N, 2>(xs, kk, c0, cend, vb, lane);
  else trsm_block<N, 1>(xs, kk, c0, cend, vb, lane);
}

template <int N>
__device__ __forceinline__ void s3_blocks(double* xs, int r0, int c0, int cend, int j0, int j1, int lane) {
  const int nt = (cend - c0 + 7) >> 3;
  if (nt >= 4) s3_block<N, 4>(xs, r0, c0, cend, j0, j1, lane);
  else if (nt == 3) s3_block<N, 3>(xs, r0, c0, cend, j0, j1, lane);
  else if (nt == 2) s3_block<N, 2>(xs, r0, c0, cend, j0, j1, lane);
  else s3_block<N, 1>(xs, r0, c0, cend, j0, j1, lane);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// stored part of row r of problem `xs` -> X (row-major NR x NR; the zeros left
// of it are written when the problem is loaded); one warp, the row's 16-byte
// units two per lane in flight
template <int N, int NR>
__device__ __forceinline__ void store_row(double* __restrict__ dst, const double* xs, int r, int lane) {
  const int c0 = 4 * (r >> 2);
  const double* row = xs + GL<N>::row0(r) - c0;
  double* drow = dst + (long long)r * NR;
  for (int c = c0 + 2 * lane; c < NR; c += 128) {
    const int c2 = c + 64;
    const double2 v = *reinterpret_cast<const double2*>(row + c);
    double2 w = make_double2(0.0, 0.0);
    if (c2 < NR) w = *reinterpret_cast<const double2*>(row + c2);
    __stcs(reinterpret_cast<double2*>(drow + c), v);
    if (c2 < NR) __stcs(reinterpret_cast<double2*>(drow + c2), w);
  }
}

// shared -> global bulk copy (bulk async-group of the issuing thread)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

// rows [ra, ra + cnt) of problem `xs` -> X (row-major NR x NR); one warp: lane
// i issues the bulk copy of row ra + i's stored part (one TMA request per
// row), then the warp writes the zeros left of the stored parts
template <int N, int NR>
__device__ __forceinline__ void store_rows_bulk(double* __restrict__ dst, const double* xs, int ra, int cnt, int lane) {
#ifndef GANG_NOBULK
  if (lane < cnt) {
    const int r = ra + lane;
    if (r >= 0 && r < NR) {
      const int c0 = 4 * (r >> 2);
      bulk_s2g(dst + (long long)r * NR + c0, xs + GL<N>::row0(r), (uint32_t)((NR - c0) * 8));
    }
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
#endif
#ifdef GANG_NOZERO
  return;
#endif
  for (int i = 0; i < cnt; ++i) {
    const int r = ra + i;
    if (r < 0 || r >= NR) continue;
    const int c0 = 4 * (r >> 2);
    double* drow = dst + (long long)r * NR;
    for (int c = 2 * lane; c < c0; c += 64) {
#ifdef GANG_STWB
      *reinterpret_cast<double2*>(drow + c) = make_double2(0.0, 0.0);
#else
      __stcs(reinterpret_cast<double2*>(drow + c), make_double2(0.0, 0.0));
#endif
    }
  }
}

#ifdef GANG_PROF
__device__ unsigned long long gang_prof[64];
#define GANG_TICK(slot)                                              \
  do {                                                               \
    const long long t1_ = clock64();                                 \
    pacc_[slot] += t1_ - tp_;                                        \
    tp_ = t1_;                                                       \
  } while (0)
#else
#define GANG_TICK(slot) do {} while (0)
#endif

// Schedule of iteration k (block row k, r0 = 8k; one CTA barrier per iteration):
//   panel warps (sub-partition 0):
//     T1  S4 of block row k-1 on the 8 columns of block k, then that tile's
//         contribution to the diagonal block k (S1, last K = 8)  -> arrive(2)
//     T3  CHOL leaves of block k (leaf warps)
//   io warp (sub-partition 0): stores block row k-2
//   bulk warps (sub-partitions 1..3), concurrently:
//     B1  S4 of block row k-1 on the columns right of block k     -> sync(2)
//     B3  S3 of block row k (K = 8k) and the look-ahead part of S1 for block
//         k+1 (rows [0, 8k))
// so the CHOL chain of block k overlaps the bulk update of block row k, and
// every S4 / update a later step needs is complete at the barrier before it.
template <int N, int NR, int P, int Q, int MINB>
__global__ void __launch_bounds__(GCfg<N, P, Q, MINB>::THREADS, MINB)
    chol_gang_kernel(const double* __restrict__ A, double* __restrict__ X, int* __restrict__ info, long long batch) {
  using C = GCfg<N, P, Q, MINB>;
  static_assert(NR <= N && NR > N - 8 && NR % 4 == 0, "real size padded to the next multiple of 8");
  constexpr int NB = C::NB, SLOT = C::SLOT, NT = C::THREADS;
  static_assert(NB >= 2, "gang engine: n >= 16");
  constexpr int NPW = C::NPW, NPT = NPW * 32;  // panel warps / threads
  constexpr long long NN = (long long)NR * NR;
  extern __shared__ __align__(16) double smem[];
  double* vb_all = smem + (size_t)P * SLOT;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(vb_all + 2 * P * C::RSB);
  int* flags = reinterpret_cast<int*>(mbar + NB);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sp = warp & 3, wq = warp >> 2;
  const bool is_panel = sp == 0 && wq < NPW;
  const bool is_leaf = is_panel && wq < C::NLEAF;
    const int bw = wq * 3 + (sp - 1);             // bulk warp index (neighbours on different sub-partitions)

  if (tid == 0) {
    for (int k = 0; k < NB; ++k) mbar_init(mbar + k, 1);  // the loader's expect_tx arrive
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < P) flags[tid] = 0;
  // padding columns (never written: every loop stops at NR) read as 0
  if constexpr (NR < N) {
    for (int u = tid; u < P * SLOT; u += NT) smem[u] = 0.0;
  }
  __syncthreads();

#ifdef GANG_STAGGER
  {  // de-phase the CTAs (they run identical rounds, so they would hit HBM in bursts)
    const long long until = clock64() + (long long)(blockIdx.x % GANG_STAGGER_M) * GANG_STAGGER;
    while (clock64() < until) {}
  }
#endif
  auto bar_panel = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(NPT) : "memory"); };
  auto vbuf = [&](int p, int k) { return vb_all + (2 * p + (k & 1)) * C::RSB; };

  const long long grid = gridDim.x;
  for (long long t = 0;; ++t) {
    // slot-major order: problem of slot p in round t
#ifdef GANG_CTAMAJOR
    const long long first = (t * grid + blockIdx.x) * P, pstride = 1;
#else
    const long long first = (t * P) * grid + blockIdx.x, pstride = grid;
#endif
    if (first >= batch) break;
    int nv = 0;
#pragma unroll
    for (int p = 0; p < P; ++p) nv += (first + (long long)p * pstride < batch) ? 1 : 0;
    const uint32_t parity = (uint32_t)(t & 1);
#ifdef GANG_PROF
    // warp 0 (leaf), warp 1 (bulk), the first io warp; second round of CTA 0
    const bool profme = blockIdx.x == 0 && t == 1 && (warp == 0 || warp == 1 || warp == 4);
    const int pbase = warp == 0 ? 0 : (warp == 1 ? 16 : 32);
    long long pacc_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tp_ = clock64();
#endif

    // ---- loads: one bulk copy (TMA) per matrix row, issued by the loader
    // warp LA block rows ahead; block row k completes on mbarrier k
    const bool is_loader = sp == 0 && wq == Q - 1;
    const bool is_storer = sp == 0 && wq == (C::NHELP >= 2 ? Q - 2 : Q - 1);
    auto load_block_row = [&](int kb) {
      for (int u = lane; u < nv * 8; u += 32) {
        const int p = u >> 3, r = 8 * kb + (u & 7);
        if (r < NR) {
          const int c0 = 4 * (r >> 2);
          bulk_g2s(smem + (size_t)p * SLOT + GL<N>::row0(r),
                   A + (first + (long long)p * pstride) * NN + (long long)r * NR + c0, (uint32_t)((NR - c0) * 8),
                   mbar + kb);
        }
      }
    };
    auto store_block_rows = [&](int ra, int cnt) {  // rows [ra, ra + cnt) of every problem, stored parts
      for (int u = lane; u < nv * cnt; u += 32) {
        const int p = u / cnt, r = ra + (u - p * cnt);
        if (r >= 0 && r < NR) {
          const int c0 = 4 * (r >> 2);
          bulk_s2g(X + (first + (long long)p * pstride) * NN + (long long)r * NR + c0,
                   smem + (size_t)p * SLOT + GL<N>::row0(r), (uint32_t)((NR - c0) * 8));
        }
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    };
    auto zero_block_rows = [&](int ra, int cnt, int w, int nw) {  // X's zeros left of the stored parts
      for (int u = w; u < nv * cnt; u += nw) {
        const int p = u / cnt, r = ra + (u - p * cnt);
        if (r >= 0 && r < NR) {
          double* xrow = X + (first + (long long)p * pstride) * NN + (long long)r * NR;
          for (int c = 2 * lane; c < 4 * (r >> 2); c += 64) __stcs(reinterpret_cast<double2*>(xrow + c), make_double2(0.0, 0.0));
        }
      }
    };
    if constexpr (NR < N) {
      // the padded tail of the last block row: zeros right of the real
      // columns, identity on the padded diagonal (rewritten every round: a
      // failed problem leaves NaN there)
      for (int u = tid; u < nv * 32; u += NT) {
        const int p = u >> 5, i = (u >> 2) & 7, c = NR + (u & 3), r = N - 8 + i;
        if (c >= 4 * (r >> 2)) smem[(size_t)p * SLOT + GL<N>::at(r, c)] = r == c ? 1.0 : 0.0;
      }
    }
    if (is_loader) {
      if (lane < NB) {  // block row `lane`: rows 8k..8k+3 keep NR - 8k columns, rows 8k+4.. four fewer
        const int w = NR - 8 * lane;
        const int bytes = (4 * w + (w > 4 ? 4 * (w - 4) : 0)) * 8;
        mbar_expect_tx(mbar + lane, (uint32_t)(bytes * nv));
      }
      __syncwarp();
      for (int kb = 0; kb < C::LA && kb < NB; ++kb) load_block_row(kb);
    }
    GANG_TICK(0);  // load issue

#pragma unroll 1
    for (int k = 0; k < NB; ++k) {
      const int r0 = 8 * k;
      if (is_panel) {
        mbar_wait(mbar + k, parity);
        GANG_TICK(1);  // wait for block row k
#ifndef GANG_IOONLY
        if (k > 0) {
          // T1: S4 of block row k-1 on the columns of block k, then the
          // diagonal block k -= X(k-1, k)^T X(k-1, k)
          for (int p = wq; p < nv; p += NPW) {
            double* xs = smem + (size_t)p * SLOT;
            trsm_block<N, 1>(xs, k - 1, r0, NR, vbuf(p, k - 1), lane);
            __syncwarp();
            s1_tile<N>(xs, r0, k - 1, k, lane);
          }
        }
#endif
        asm volatile("bar.arrive 2, %0;" ::"n"(NT - 32 * C::NIO) : "memory");
        bar_panel();
        GANG_TICK(2);  // T1
#ifndef GANG_IOONLY
        if (is_leaf && 4 * wq < nv) {
          const int q = lane >> 3, j = lane & 7;
          const bool act = 4 * wq + q < nv;
          const int p = act ? 4 * wq + q : 4 * wq;
          leaf4<N>(smem + (size_t)p * SLOT, vbuf(p, k), flags + p, r0, j, act);
        }
#endif
        if (!is_leaf) {
          if (is_loader && k + C::LA < NB) load_block_row(k + C::LA);
          if (is_storer && k >= 2) store_block_rows(r0 - 16, 8);  // final (and fenced) since the last barrier
        }
        GANG_TICK(3);  // T3 (leaf / loads / stores)
      } else {
        if (k >= 2) zero_block_rows(r0 - 16, 8, bw, C::NDW);
        GANG_TICK(6);  // barrier wait (deferred) + zero prefixes
#ifndef GANG_IOONLY
        if (k > 0) {
          mbar_wait(mbar + k, parity);
          GANG_TICK(7);  // wait for block row k
          // B1: S4 of block row k-1 right of block k
          const int cs = r0 + 8;
          const int nblk = cs < NR ? (NR - cs + 31) >> 5 : 0;
          for (int it = bw; it < nv * nblk; it += C::NDW) {
            const int p = it / nblk, i = it - p * nblk;
            trsm_blocks<N>(smem + (size_t)p * SLOT, k - 1, cs + 32 * i, NR, vbuf(p, k - 1), lane);
          }
        }
#endif
        GANG_TICK(1);  // B1
        asm volatile("bar.sync 2, %0;" ::"n"(NT - 32 * C::NIO) : "memory");
        GANG_TICK(2);  // wait for the panel's columns
#ifndef GANG_IOONLY
        if (k > 0) {
          // B3: S3 of block row k; rows [0, 8k) into the diagonal block k+1
          const int cs = r0 + 8;
          const int nblk = cs < NR ? (NR - cs + 31) >> 5 : 0;
          const bool la = k + 1 < NB;
          if (la) mbar_wait(mbar + k + 1, parity);
          const int ipp = nblk + (la ? 1 : 0);
          // offset by k so the short diagonal-tile items do not always land on the same warps
          for (int it = (bw + C::NDW - (k % C::NDW)) % C::NDW; it < nv * ipp; it += C::NDW) {
            const int p = it / ipp, i = it - p * ipp;
            double* xs = smem + (size_t)p * SLOT;
            if (i < nblk) s3_blocks<N>(xs, r0, cs + 32 * i, NR, 0, k, lane);
            else s1_tile<N>(xs, r0 + 8, 0, k, lane);
          }
        }
#endif
        GANG_TICK(3);  // B3
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      GANG_TICK(4);  // wait at the iteration barrier
    }
    // last two block rows, info
    if (is_storer) {
      store_block_rows(N - 16, 16);
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the slots are refilled next
    } else if (!is_panel) {
      zero_block_rows(N - 16, 16, bw, C::NDW);
    }
    if (tid < P) {
      if (info && tid < nv) info[first + (long long)tid * pstride] = flags[tid];
      flags[tid] = 0;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    GANG_TICK(5);  // tail
#ifdef GANG_PROF
    if (profme && lane == 0)
      for (int i = 0; i < 8; ++i) gang_prof[pbase + i] += pacc_[i];
#endif
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace gang
}  // namespace lagen
