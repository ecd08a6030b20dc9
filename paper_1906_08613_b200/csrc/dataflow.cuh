// dataflow.cuh — the "dataflow engine": a blocked variant executed as a DAG
// of 4x4-tile tasks instead of statement by statement.
//
// Every statement of every iteration is split into tile tasks, enumerated in
// program order (k, statement, task).  Thread t of the CTA runs tasks
// t, t + G, t + 2G, ... in that order.  Each tile of the unknown X carries a
// version = number of completed writes; a task waits until every X tile it
// reads or updates has exactly the number of writes that precede the task in
// program order, computes, then bumps the version of the tiles it wrote.
// The result is therefore identical, per tile and per update, to executing
// the statements in program order (interpret_algorithm, verify.py:245-297),
// while panels, leaves and trailing updates of different iterations overlap
// as their data become ready.  Deadlock-free: the earliest unfinished task in
// program order always has all its inputs.
//
// Scope: the right-looking variants (every statement writes a block with
// indices in {1, 2}: Cholesky v2, Lyapunov v5, Sylvester v13), b in {4, 8}.
// Statement semantics as in the reference block kernels (kernels.py):
//   GEMM_update   one task per output tile (upper tiles / elements i <= j
//                 for diagonal blocks of a symmetric right-hand side)
//   CHOL, LYAP    one task for the whole b x b block (registers)
//   TRSM          one task per column tile of the block row
//   SYLV          m <= q: column tiles, SOLVE(J) then UPD(J -> J') for J' > J
//                 (right-looking over the long dimension); m > q: row tiles.
#pragma once
#include "engine.cuh"

namespace lagen {
namespace df {

using eng::EqT;
using eng::MatOf;
using eng::Slot;
using eng::TV;
using eng::view_tile_load;
using eng::view_tile_store;
using eng::K_GEMM;
using eng::K_CHOL;
using eng::K_TRSM;
using eng::K_SYLV;
using eng::K_LYAP;

// ---------------------------------------------------------------------------
// tile geometry of one iteration (in tiles): block starts / extents
// ---------------------------------------------------------------------------
template <int N, int B>
struct TRep {
  static constexpr int BT = B / 4, NT = N / 4;
  int k;
  __host__ __device__ __forceinline__ int st(int r) const { return r == 0 ? 0 : (r == 1 ? k * BT : (k + 1) * BT); }
  __host__ __device__ __forceinline__ int ex(int r) const { return r == 0 ? k * BT : (r == 1 ? BT : NT - (k + 1) * BT); }
};

// iteration at which row / column tile R lies in block 1
template <int B>
__device__ __forceinline__ int kblk(int R) { return R / (B / 4); }

// ---------------------------------------------------------------------------
// task counts per statement and iteration
// ---------------------------------------------------------------------------
template <class E, int N, int B, class S>
__host__ __device__ __forceinline__ int task_count(int k) {
  using O = typename S::out;
  TRep<N, B> rp{k};
  const int mt = rp.ex(O::r), qt = rp.ex(O::c);
  if (mt == 0 || qt == 0) return 0;
  if constexpr (S::kind == K_GEMM) {
    using A = typename S::in0;
    const int pt = A::tr ? rp.ex(A::r) : rp.ex(A::c);
    if (pt == 0) return 0;
    if (E::SYMT && O::r == O::c) return mt * (mt + 1) / 2;
    return mt * qt;
  } else if constexpr (S::kind == K_CHOL || S::kind == K_LYAP) {
    return 1;
  } else if constexpr (S::kind == K_TRSM) {
    return qt;
  } else {  // SYLV: SOLVE + UPD tasks along the long side
    const int L = mt <= qt ? qt : mt;
    return L + L * (L - 1) / 2;
  }
}

// SYLV task index -> SOLVE(j0) as (j0, -1) or UPD(j0 -> j1) as (j0, j1);
// order: SOLVE(0), UPD(0->1..L-1), SOLVE(1), UPD(1->2..L-1), ...
__host__ __device__ __forceinline__ void sylv_decode(int L, int idx, int& j0, int& j1) {
  int start = 0;
  for (j0 = 0; j0 < L; ++j0) {
    const int len = L - j0;
    if (idx < start + len) {
      const int o = idx - start;
      j1 = o == 0 ? -1 : j0 + o;
      return;
    }
    start += len;
  }
  j0 = L - 1;
  j1 = -1;
}

// GEMM task index -> output tile (I, J): upper tiles row-major for a
// symmetric diagonal target, else row-major
__host__ __device__ __forceinline__ void gemm_decode(bool up, int mt, int qt, int idx, int& I, int& J) {
  if (up) {
    int rem = idx;
    I = 0;
    while (rem >= mt - I) {
      rem -= mt - I;
      ++I;
    }
    J = I + rem;
  } else {
    I = idx / qt;
    J = idx - I * qt;
  }
}

// X-tile coordinates (tile units) of tile (I, J) of a block view
template <class Vw, bool SY, int N, int B>
__host__ __device__ __forceinline__ void vtile(const TRep<N, B>& rp, int I, int J, int& R, int& C) {
  const int r0 = rp.st(Vw::r), c0 = rp.st(Vw::c);
  if (Vw::tr) {
    R = r0 + J;
    C = c0 + I;
  } else {
    R = r0 + I;
    C = c0 + J;
  }
  if (SY && R > C) {
    const int t = R;
    R = C;
    C = t;
  }
}

// X tiles a task reads (w = false) or updates (w = true) — the host-side
// mirror of run_task, used to build the schedule
struct Touch {
  int r[8], c[8];
  bool w[8];
  int n = 0;
  void add(int R, int C, bool wr) {
    for (int i = 0; i < n; ++i)
      if (r[i] == R && c[i] == C) {
        w[i] = w[i] || wr;
        return;
      }
    r[n] = R;
    c[n] = C;
    w[n] = wr;
    ++n;
  }
};

template <class E, int N, int B, class S>
inline void task_tiles(int k, int idx, Touch& t) {
  using O = typename S::out;
  constexpr int BT = B / 4;
  TRep<N, B> rp{k};
  const int R0 = rp.st(O::r), C0 = rp.st(O::c), mt = rp.ex(O::r), qt = rp.ex(O::c);
  if constexpr (S::kind == K_GEMM) {
    using A = typename S::in0;
    using Bv = typename S::in1;
    constexpr bool UP = E::SYMT && O::r == O::c;
    constexpr bool SA = E::SYMX && A::op == 0 && A::r == A::c;
    constexpr bool SB = E::SYMX && Bv::op == 0 && Bv::r == Bv::c;
    const int pt = A::tr ? rp.ex(A::r) : rp.ex(A::c);
    int I, J, R, C;
    gemm_decode(UP, mt, qt, idx, I, J);
    t.add(R0 + I, C0 + J, true);
    for (int q = 0; q < pt; ++q) {
      if (A::op == 0) {
        vtile<A, SA>(rp, I, q, R, C);
        t.add(R, C, false);
      }
      if (Bv::op == 0) {
        vtile<Bv, SB>(rp, q, J, R, C);
        t.add(R, C, false);
      }
    }
  } else if constexpr (S::kind == K_CHOL || S::kind == K_LYAP) {
    for (int I = 0; I < BT; ++I)
      for (int J = I; J < BT; ++J) t.add(R0 + I, C0 + J, true);
  } else if constexpr (S::kind == K_TRSM) {
    using A = typename S::in0;
    for (int I = 0; I < BT; ++I) {
      t.add(R0 + I, C0 + idx, true);
      for (int Q = 0; Q <= I; ++Q) {
        int R, C;
        vtile<A, false>(rp, I, Q, R, C);
        t.add(R, C, false);
      }
    }
  } else {
    const bool bycol = mt <= qt;
    int j0, j1;
    sylv_decode(bycol ? qt : mt, idx, j0, j1);
    for (int s = 0; s < BT; ++s) {
      if (bycol) {
        if (j1 < 0) {
          t.add(R0 + s, C0 + j0, true);
        } else {
          t.add(R0 + s, C0 + j0, false);
          t.add(R0 + s, C0 + j1, true);
        }
      } else {
        if (j1 < 0) {
          t.add(R0 + j0, C0 + s, true);
        } else {
          t.add(R0 + j0, C0 + s, false);
          t.add(R0 + j1, C0 + s, true);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// tile versions (shared memory)
// ---------------------------------------------------------------------------
struct Ver {
  int* v;
  int nt;
  __device__ __forceinline__ void bump(int R, int C) const {
    __threadfence_block();
    atomicAdd(v + R * nt + C, 1);
  }
};

__device__ __forceinline__ void mm_sub(double w[4][4], const double a[4][4], const double b[4][4]) {
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) s = fma(a[r][q], b[q][c], s);
      w[r][c] -= s;
    }
}

// tile (I, J) of a view; symmetric diagonal blocks are stored as upper tiles
template <class V>
__device__ __forceinline__ void load_vt(const V& v, int I, int J, double t[4][4]) {
  if constexpr (V::sy) {
    TV<typename V::Mat, false, false> u;
    u.base = v.base;
    u.r0 = v.r0;
    u.c0 = v.c0;
    if (I <= J) {
      view_tile_load(u, I, J, t);
      if (I == J) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < a; ++b) t[a][b] = t[b][a];
      }
    } else {
      double s[4][4];
      view_tile_load(u, J, I, s);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) t[a][b] = s[b][a];
    }
  } else {
    view_tile_load(v, I, J, t);
  }
}

// X tile coordinates of view tile (I, J)
template <class V>
__device__ __forceinline__ void xcoord(const V& v, int I, int J, int& R, int& C) {
  if constexpr (V::tr) {
    R = (v.r0 >> 2) + J;
    C = (v.c0 >> 2) + I;
  } else {
    R = (v.r0 >> 2) + I;
    C = (v.c0 >> 2) + J;
  }
  if constexpr (V::sy) {
    if (R > C) {
      const int t = R;
      R = C;
      C = t;
    }
  }
}

// Runs task idx of statement S at iteration k; the caller has checked that
// every X tile it touches holds its program-order version.
template <int EQ, int N, int B, class S>
__device__ __forceinline__ bool run_task(const Slot& sl, const Ver& ver, int k, int idx, int* flag) {
  using E = EqT<EQ, N>;
  using O = typename S::out;
  TRep<N, B> rp{k};
  constexpr int BT = B / 4;
  auto mkv = [&](auto vw, auto sy) {
    using Vw = decltype(vw);
    constexpr bool SY = decltype(sy)::value;
    TV<typename MatOf<E, Vw::op>::type, Vw::tr != 0, SY> v;
    v.base = sl.p[Vw::op < 0 ? 0 : Vw::op];
    v.r0 = 4 * rp.st(Vw::r);
    v.c0 = 4 * rp.st(Vw::c);
    return v;
  };
  const auto Ov = mkv(O{}, std::false_type{});
  const int R0 = rp.st(O::r), C0 = rp.st(O::c), mt = rp.ex(O::r), qt = rp.ex(O::c);
  auto need = [](int, int, int) { return true; };  // (checked from the schedule)

  if constexpr (S::kind == K_GEMM) {
    using A = typename S::in0;
    using Bv = typename S::in1;
    constexpr bool UP = E::SYMT && O::r == O::c;
    constexpr bool SA = E::SYMX && A::op == 0 && A::r == A::c;
    constexpr bool SB = E::SYMX && Bv::op == 0 && Bv::r == Bv::c;
    const auto Av = mkv(A{}, std::integral_constant<bool, SA>{});
    const auto Bw = mkv(Bv{}, std::integral_constant<bool, SB>{});
    const int pt = A::tr ? rp.ex(A::r) : rp.ex(A::c);
    int I, J;
    gemm_decode(UP, mt, qt, idx, I, J);
    if (!need(R0 + I, C0 + J, 0)) return false;
    for (int q = 0; q < pt; ++q) {
      int R, C;
      if constexpr (A::op == 0) {
        xcoord(Av, I, q, R, C);
        if (!need(R, C, 0)) return false;
      }
      if constexpr (Bv::op == 0) {
        xcoord(Bw, q, J, R, C);
        if (!need(R, C, 0)) return false;
      }
    }
    double w[4][4], acc[4][4] = {};
    view_tile_load(Ov, I, J, w);
    for (int q = 0; q < pt; ++q) {
      double a[4][4], b[4][4];
      load_vt(Av, I, q, a);
      load_vt(Bw, q, J, b);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int z = 0; z < 4; ++z) acc[r][c] = fma(a[r][z], b[z][c], acc[r][c]);
    }
    const double sgn = S::sign < 0 ? -1.0 : 1.0;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (!UP || I != J || r <= c) w[r][c] = fma(sgn, acc[r][c], w[r][c]);
    view_tile_store(Ov, I, J, w);
    ver.bump(R0 + I, C0 + J);
  } else if constexpr (S::kind == K_CHOL) {
    static_assert(B <= 8, "dataflow CHOL leaf: b <= 8");
#pragma unroll
    for (int I = 0; I < BT; ++I)
#pragma unroll
      for (int J = I; J < BT; ++J)
        if (!need(R0 + I, C0 + J, 0)) return false;
    double t[B][B];
#pragma unroll
    for (int I = 0; I < BT; ++I)
#pragma unroll
      for (int J = I; J < BT; ++J) {
        double x[4][4];
        view_tile_load(Ov, I, J, x);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) t[4 * I + a][4 * J + b] = x[a][b];
      }
    int bad = 0;
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const double piv = t[i][i];
      if (piv <= 0.0 && bad == 0) bad = 4 * R0 + i + 1;
      const double rs = rsqrt(piv);
      t[i][i] = piv * rs;
#pragma unroll
      for (int c = i + 1; c < B; ++c) t[i][c] *= rs;
#pragma unroll
      for (int r = i + 1; r < B; ++r)
#pragma unroll
        for (int c = r; c < B; ++c) t[r][c] = fma(-t[i][r], t[i][c], t[r][c]);
    }
    if (bad) atomicMin(flag, bad);
#pragma unroll
    for (int I = 0; I < BT; ++I)
#pragma unroll
      for (int J = I; J < BT; ++J) {
        double x[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) x[a][b] = (4 * I + a <= 4 * J + b) ? t[4 * I + a][4 * J + b] : 0.0;
        view_tile_store(Ov, I, J, x);
        ver.bump(R0 + I, C0 + J);
      }
  } else if constexpr (S::kind == K_LYAP) {
    static_assert(B <= 8, "dataflow LYAP leaf: b <= 8");
    using A = typename S::in0;
    const auto Lv = mkv(A{}, std::false_type{});
#pragma unroll
    for (int I = 0; I < BT; ++I)
#pragma unroll
      for (int J = I; J < BT; ++J)
        if (!need(R0 + I, C0 + J, 0)) return false;
    double l[B][B], x[B][B];
#pragma unroll
    for (int I = 0; I < BT; ++I)
#pragma unroll
      for (int J = 0; J < BT; ++J) {
        double t[4][4];
        if (J <= I) {
          view_tile_load(Lv, I, J, t);
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) l[4 * I + a][4 * J + b] = t[a][b];
        }
        if (I <= J) {
          view_tile_load(Ov, I, J, t);
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) x[4 * I + a][4 * J + b] = t[a][b];
        }
      }
    // upper triangle, column by column (kernels.py LYAP block kernel)
#pragma unroll
    for (int j = 0; j < B; ++j)
#pragma unroll
      for (int i = 0; i <= j; ++i) {
        double d1 = 0.0, d2 = 0.0;
#pragma unroll
        for (int q = 0; q < i; ++q) d1 = fma(l[i][q], x[q][j], d1);
#pragma unroll
        for (int q = 0; q < j; ++q) d2 = fma(q < i ? x[q][i] : x[i][q], l[j][q], d2);
        x[i][j] = (x[i][j] - d1 - d2) * __drcp_rn(l[i][i] + l[j][j]);
      }
#pragma unroll
    for (int I = 0; I < BT; ++I)
#pragma unroll
      for (int J = I; J < BT; ++J) {
        double t[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int r = 4 * I + a, c = 4 * J + b;
            t[a][b] = r <= c ? x[r][c] : x[c][r];
          }
        view_tile_store(Ov, I, J, t);
        ver.bump(R0 + I, C0 + J);
      }
  } else if constexpr (S::kind == K_TRSM) {
    static_assert(B <= 8, "dataflow TRSM: b <= 8");
    using A = typename S::in0;  // X11^T, logically lower
    const auto Tv = mkv(A{}, std::false_type{});
    const int J = idx;
#pragma unroll
    for (int I = 0; I < BT; ++I) {
      if (!need(R0 + I, C0 + J, 0)) return false;
#pragma unroll
      for (int Q = 0; Q <= I; ++Q) {
        int R, C;
        xcoord(Tv, I, Q, R, C);
        if (!need(R, C, 0)) return false;
      }
    }
    double t[B][B], w[B][4];
#pragma unroll
    for (int I = 0; I < BT; ++I) {
      double x[4][4];
#pragma unroll
      for (int Q = 0; Q <= I; ++Q) {
        view_tile_load(Tv, I, Q, x);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) t[4 * I + a][4 * Q + b] = x[a][b];
      }
      view_tile_load(Ov, I, J, x);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) w[4 * I + a][b] = x[a][b];
    }
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const double rd = __drcp_rn(t[i][i]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double v = w[i][c];
#pragma unroll
        for (int l = 0; l < i; ++l) v = fma(-t[i][l], w[l][c], v);
        w[i][c] = v * rd;
      }
    }
#pragma unroll
    for (int I = 0; I < BT; ++I) {
      double x[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) x[a][b] = w[4 * I + a][b];
      view_tile_store(Ov, I, J, x);
      ver.bump(R0 + I, C0 + J);
    }
  } else {  // SYLV (the short side is always one block: b rows or b columns)
    static_assert(B <= 8, "dataflow SYLV: b <= 8");
    using A = typename S::in0;
    using U = typename S::in1;
    const auto Lv = mkv(A{}, std::false_type{});
    const auto Uv = mkv(U{}, std::false_type{});
    const bool bycol = mt <= qt;
    int j0, j1;
    sylv_decode(bycol ? qt : mt, idx, j0, j1);
    if (bycol) {
      // column tiles of W (b x 4); rows coupled by L (b x b)
      if (j1 < 0) {
        // SOLVE(j0): every UPD(j -> j0), j < j0, has landed
#pragma unroll
        for (int I = 0; I < BT; ++I)
          if (!need(R0 + I, C0 + j0, j0)) return false;
        double w[B][4], l[B][B], u[4][4];
#pragma unroll
        for (int I = 0; I < BT; ++I) {
          double x[4][4];
          view_tile_load(Ov, I, j0, x);
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) w[4 * I + a][b] = x[a][b];
#pragma unroll
          for (int Q = 0; Q <= I; ++Q) {
            view_tile_load(Lv, I, Q, x);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) l[4 * I + a][4 * Q + b] = x[a][b];
          }
        }
        view_tile_load(Uv, j0, j0, u);
        double rp[B][4];  // shifted pivots, off the substitution chain
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) rp[i][c] = __drcp_rn(l[i][i] + u[c][c]);
        // reference column order (kernels.py:100-110)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
          for (int i = 0; i < B; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < c; ++q) acc = fma(w[i][q], u[q][c], acc);
            w[i][c] -= acc;
          }
#pragma unroll
          for (int i = 0; i < B; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < i; ++q) acc = fma(l[i][q], w[q][c], acc);
            w[i][c] = (w[i][c] - acc) * rp[i][c];
          }
        }
#pragma unroll
        for (int I = 0; I < BT; ++I) {
          double x[4][4];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) x[a][b] = w[4 * I + a][b];
          view_tile_store(Ov, I, j0, x);
          ver.bump(R0 + I, C0 + j0);
        }
      } else {
        // UPD(j0 -> j1): W[:, j1] -= X[:, j0] U[j0, j1]
#pragma unroll
        for (int I = 0; I < BT; ++I) {
          if (!need(R0 + I, C0 + j0, j0 + 1)) return false;
          if (!need(R0 + I, C0 + j1, j0)) return false;
        }
        double u[4][4];
        view_tile_load(Uv, j0, j1, u);
#pragma unroll
        for (int I = 0; I < BT; ++I) {
          double x[4][4], w[4][4];
          view_tile_load(Ov, I, j0, x);
          view_tile_load(Ov, I, j1, w);
          mm_sub(w, x, u);
          view_tile_store(Ov, I, j1, w);
          ver.bump(R0 + I, C0 + j1);
        }
      }
    } else {
      // row tiles of W (4 x b); columns coupled by U (b x b)
      if (j1 < 0) {
#pragma unroll
        for (int J = 0; J < BT; ++J)
          if (!need(R0 + j0, C0 + J, j0)) return false;
        double w[4][B], u[B][B], l[4][4];
#pragma unroll
        for (int J = 0; J < BT; ++J) {
          double x[4][4];
          view_tile_load(Ov, j0, J, x);
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) w[a][4 * J + b] = x[a][b];
#pragma unroll
          for (int Q = 0; Q <= J; ++Q) {
            view_tile_load(Uv, Q, J, x);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) u[4 * Q + a][4 * J + b] = x[a][b];
          }
        }
        view_tile_load(Lv, j0, j0, l);
        double rp[4][B];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < B; ++c) rp[a][c] = __drcp_rn(l[a][a] + u[c][c]);
#pragma unroll
        for (int c = 0; c < B; ++c) {
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            double acc = 0.0;
#pragma unroll
            for (int z = 0; z < c; ++z) acc = fma(w[a][z], u[z][c], acc);
            w[a][c] -= acc;
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            double acc = 0.0;
#pragma unroll
            for (int z = 0; z < a; ++z) acc = fma(l[a][z], w[z][c], acc);
            w[a][c] = (w[a][c] - acc) * rp[a][c];
          }
        }
#pragma unroll
        for (int J = 0; J < BT; ++J) {
          double x[4][4];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) x[a][b] = w[a][4 * J + b];
          view_tile_store(Ov, j0, J, x);
          ver.bump(R0 + j0, C0 + J);
        }
      } else {
        // UPD(j0 -> j1): W[j1, :] -= L[j1, j0] X[j0, :]
#pragma unroll
        for (int J = 0; J < BT; ++J) {
          if (!need(R0 + j0, C0 + J, j0 + 1)) return false;
          if (!need(R0 + j1, C0 + J, j0)) return false;
        }
        double lt[4][4];
        view_tile_load(Lv, j1, j0, lt);
#pragma unroll
        for (int J = 0; J < BT; ++J) {
          double x[4][4], w[4][4];
          view_tile_load(Ov, j0, J, x);
          view_tile_load(Ov, j1, J, w);
          mm_sub(w, lt, x);
          view_tile_store(Ov, j1, J, w);
          ver.bump(R0 + j1, C0 + J);
        }
      }
    }
  }
  return true;
}

// statement dispatch by runtime index
template <int EQ, int N, int B, int I, class S0, class... Ss>
__device__ __forceinline__ void exec_at(int si, const Slot& sl, const Ver& ver, int k, int idx, int* flag) {
  if (si == I) {
    run_task<EQ, N, B, S0>(sl, ver, k, idx, flag);
    return;
  }
  if constexpr (sizeof...(Ss) > 0) exec_at<EQ, N, B, I + 1, Ss...>(si, sl, ver, k, idx, flag);
}

// Schedule record (built once on the host, registry_df.cuh): 2 x int4 per
// task, x = k | si << 8 | ndeps << 16, y = task index within the statement,
// then up to 6 dependencies (tile << 16 | required version).
//
// Warp-synchronous walk with continuous refill: every round, lanes without a
// task claim the next records (one warp-aggregated atomic; schedule order =
// DAG level, so claims follow the critical path), then every lane whose
// tiles hold the required versions runs its task.  Waiting is warp-uniform
// (no lane spins alone), a waiting lane never holds up its warp's other
// lanes, and every dependency lies earlier in the schedule, so the walk
// cannot deadlock: the earliest claimed unfinished task is always runnable.
template <int EQ, int N, int B, class... S>
__device__ __forceinline__ bool run_dataflow(eng::Var<S...>, const Slot& sl, const Ver& ver,
                                             const int4* __restrict__ sched, int total, int* next_task, int* abort,
                                             int* flag) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  bool have = false, exhausted = false;
  int k = 0, si = 0, nd = 0, idx = 0;
  int dep[6] = {0, 0, 0, 0, 0, 0};
  unsigned idle = 0;
  for (;;) {
    const unsigned want = __ballot_sync(0xffffffffu, !have && !exhausted);
    if (want) {
      const int leader = __ffs(want) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(next_task, __popc(want));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (!have && !exhausted) {
        const int task = base + __popc(want & lt_mask);
        if (task >= total) {
          exhausted = true;
        } else {
          const int4 a = __ldg(sched + 2 * task), b = __ldg(sched + 2 * task + 1);
          k = a.x & 255;
          si = (a.x >> 8) & 255;
          nd = a.x >> 16;
          idx = a.y;
          dep[0] = a.z;
          dep[1] = a.w;
          dep[2] = b.x;
          dep[3] = b.y;
          dep[4] = b.z;
          dep[5] = b.w;
          have = true;
        }
      }
    }
    if (!__any_sync(0xffffffffu, have)) break;  // every lane exhausted
    bool ran = false;
    if (have) {
      bool ok = true;
#pragma unroll
      for (int d = 0; d < 6; ++d)
        if (d < nd) ok = ok && *reinterpret_cast<volatile int*>(ver.v + (dep[d] >> 16)) >= (dep[d] & 0xffff);
      if (ok) {
        __threadfence_block();
        exec_at<EQ, N, B, 0, S...>(si, sl, ver, k, idx, flag);
        have = false;
        ran = true;
      }
    }
    if (__any_sync(0xffffffffu, ran)) {
      idle = 0;
    } else {
      // nothing ready: yield the issue slots to the warps on the critical path
      __nanosleep(32);
      if (++idle > (1u << 24) || *reinterpret_cast<volatile int*>(abort)) {  // lost dependency: fail, never hang
        *reinterpret_cast<volatile int*>(abort) = 1;
        return false;
      }
    }
  }
  return true;
}

template <int EQ, int N, int B>
struct DPolicy {
  using E = EqT<EQ, N>;
  static constexpr int SLOT = E::SLOT;
  static constexpr int NT = N / 4;
  static constexpr size_t SMEM = (size_t)SLOT * 8 + (size_t)NT * NT * 4 + 64;
  // problems per SM that shared memory allows; the DAG walk is latency-bound,
  // so concurrent problems beat more threads per problem once two fit
  static constexpr int FIT = (int)((227 * 1024) / SMEM);
  static constexpr int THREADS = N <= 32 ? 64 : (FIT >= 2 ? 128 : (B == 4 ? 512 : 256));
};

// one problem per CTA at a time (several CTAs per SM), persistent over the batch
template <int EQ, int N, int B, class VAR>
__global__ void __launch_bounds__(DPolicy<EQ, N, B>::THREADS)
    df_kernel(const double* __restrict__ in0, const double* __restrict__ in1, const double* __restrict__ in2,
              double* __restrict__ X, int* __restrict__ info, long long batch,
              const int4* __restrict__ sched, int ntasks) {
  using E = EqT<EQ, N>;
  using P = DPolicy<EQ, N, B>;
  constexpr int G = P::THREADS;
  constexpr int NT = N / 4;
  extern __shared__ double smem[];
  Slot sl;
  sl.p[0] = smem;
  sl.p[1] = smem + E::M0::DOUBLES;
  sl.p[2] = (EQ == 2) ? smem + E::M0::DOUBLES + E::M1::DOUBLES : sl.p[1];
  int* vers = reinterpret_cast<int*>(smem + P::SLOT);
  int* misc = vers + NT * NT;  // [0] abort, [1] flag, [2] non-finite, [3] task counter
  Ver ver{vers, NT};
  const int rank = threadIdx.x;
  constexpr long long NN = (long long)N * N;
  for (long long prob = blockIdx.x; prob < batch; prob += gridDim.x) {
    const long long off = prob * NN;
    for (int i = rank; i < NT * NT; i += G) vers[i] = 0;
    if (rank < 4) misc[rank] = rank == 1 ? 0x7fffffff : 0;
    eng::issue_loads<EQ, N, G>(sl, in0, in1, in2, off, rank);
    eng::cp_async_wait<0>();
    __syncthreads();
    Slot s = sl;
    if constexpr (EQ == 2 && !E::STAGE) {
      s.p[1] = const_cast<double*>(in0) + off;
      s.p[2] = const_cast<double*>(in1) + off;
    }
    run_dataflow<EQ, N, B>(VAR{}, s, ver, sched, ntasks, &misc[3], &misc[0], &misc[1]);
    __syncthreads();
    const bool fin = eng::store_x<EQ, typename E::M0, N, G>(X + off, s.p[0], rank);
    if (!fin) atomicOr(&misc[2], 1);
    __syncthreads();
    if (info && rank == 0) info[prob] = misc[0] ? -2 : (misc[1] != 0x7fffffff ? misc[1] : (misc[2] ? -1 : 0));
    __syncthreads();
  }
}

}  // namespace df
}  // namespace lagen
