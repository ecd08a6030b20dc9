// colengine.cuh — the "column engine" for upper Cholesky, n <= 64.
//
// A group of W lanes (W = 4..32) owns one problem; lane l holds column l (and,
// for n > 32, column l + 32) of the unknown in REGISTERS, fully unrolled for
// the compile-time (n, b).  The variant's statements (worksheet listings,
// SURVEY appendix A) are executed block by block exactly as in
// interpret_algorithm (verify.py:221-303); operands that live in other lanes'
// columns are published once per statement to a small shared-memory buffer
// and read back as warp-wide broadcasts (LDS.128), so each statement costs
// ~(flops / lanes) DFMA plus one broadcast load per two products:
//
//   v1 (left-looking):  X11 -= X01^T X01;  X11 := CHOL(X11);
//                       X12 -= X01^T X02;  X12 := TRSM(X11^T, X12)
//   v2 (right-looking): X11 := CHOL(X11);  X12 := TRSM(X11^T, X12);
//                       X22 -= X12^T X12
//
// Block kernels restated: gemm_update (kernels.py:16-34, upper target on the
// diagonal block), chol_leaf (kernels.py:79-97), trsm_left (kernels.py:47-60).
// Pivots use rsqrt (x_ii = a_ii * rsqrt(a_ii), row scale by rsqrt) and the
// TRSM multiplies by reciprocal pivots: <= 2 ulp from sqrt / divide.
//
// Global traffic: only the upper triangle of A is read (coalesced row
// segments), all n^2 entries of X are written (zeros below the diagonal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace lagen {
namespace col {

// 1 / sqrt(a) for the Cholesky pivots: rsqrt.approx (MUFU.RSQ64H, ~2^-20)
// and two Newton steps y <- y + y (1/2 - (a/2) y^2), 9 instructions instead
// of the ~19 of rsqrt() with its special-case path (see chol_rows.cuh); <= 2 ulp for normal a > 0 — a <= 0, NaN and Inf
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

template <int N>
struct ColPolicy {
  static constexpr int W = N <= 4 ? 4 : N <= 8 ? 8 : N <= 16 ? 16 : 32;  // lanes per problem
  static constexpr int CPL = N <= 32 ? 1 : 2;                            // columns per lane
  static constexpr int GPW = 32 / W;                                     // problems per warp
#ifndef LAGEN_COL_WIDE
#define LAGEN_COL_WIDE 1
#endif
  // n = 28 / 32 as 3 CTAs of 4 warps (12 warps/SM, <= 168 registers): at the
  // 128-register cap of 16 warps/SM they spilled ~108 bytes per thread;
  // measured 3-4 % faster (v1) / 11-12 % (v2), profiles/r01_col_wide_ab.txt
  static constexpr bool WIDE = LAGEN_COL_WIDE && (N == 28 || N == 32);
  static constexpr int WARPS = WIDE ? 4 : N <= 32 ? 8 : 4;                // warps per CTA
// n <= 12 fits 3 CTAs of 8 warps (24 warps/SM, <= 85 registers) spill-free:
// 5-10 % faster at n = 8, 12 (profiles/r01_col_wide_ab.txt)
#ifndef LAGEN_COL_SMALL3
#define LAGEN_COL_SMALL3 1
#endif
  static constexpr int MINB = WIDE ? 3 : (LAGEN_COL_SMALL3 && N <= 12) ? 3 : N <= 32 ? 2 : 1;  // >= 16 warps/SM for n <= 32 (<= 128 regs)
  static constexpr int PUB_LD = 18;  // publish buffer: <= 16 rows per column; even -> LDS.128 pairs
  static constexpr int PUB = PUB_LD * (N < 32 ? N : 32);  // <= 32 columns per publish
  static constexpr int SMEM = WARPS * GPW * PUB * 8;
};

template <int N, int CPL>
struct Cols {
  double c0[N <= 32 ? N : 32];
  double c1[CPL == 2 ? N : 1];
};

// element (r, own column #s) accessors with compile-time r
#define COLV(cs, s, r) ((s) == 0 ? (cs).c0[(r) < 32 ? (r) : 0] : (cs).c1[(r)])

template <int N, int B, int VARIANT>
struct Chol {
  using Pol = ColPolicy<N>;
  static constexpr int W = Pol::W, CPL = Pol::CPL;

  // owner lane (within group) and slot of column j
  __device__ static constexpr int own_lane(int j) { return j & 31; }
  __device__ static constexpr int own_slot(int j) { return j >> 5; }

  template <int R, int S>
  __device__ static __forceinline__ double& cv(Cols<N, CPL>& cs) {
    if constexpr (S == 0) {
      static_assert(R < 32, "slot 0 holds rows < 32 of columns < 32");
      return cs.c0[R];
    } else {
      return cs.c1[R];
    }
  }

  // broadcast X(r, j) (held by the owner lane of column j) to the group
  template <int R, int J>
  __device__ static __forceinline__ double bcast(Cols<N, CPL>& cs, unsigned mask) {
    return __shfl_sync(mask, cv<R, own_slot(J)>(cs), own_lane(J), W);
  }
};

// Static for-loop helper
template <int I, int E, class F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (I < E) {
    f(std::integral_constant<int, I>{});
    sfor<I + 1, E>(f);
  }
}

template <int N, int B, int VARIANT>
__global__ void __launch_bounds__(ColPolicy<N>::WARPS * 32, ColPolicy<N>::MINB)
    chol_col_kernel(const double* __restrict__ A, double* __restrict__ X, int* __restrict__ info, long long batch) {
  using Pol = ColPolicy<N>;
  using K = Chol<N, B, VARIANT>;
  constexpr int W = Pol::W, CPL = Pol::CPL, GPW = Pol::GPW;
  constexpr int NB = N / B;
  constexpr int LD = Pol::PUB_LD;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gl = lane % W;   // lane within group
  const int grp = lane / W;  // group within warp
  const unsigned gmask = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << (grp * W));
  double* pub = smem + (size_t)(warp * GPW + grp) * Pol::PUB;
  const long long stride = (long long)gridDim.x * Pol::WARPS * GPW;
  constexpr long long NN = (long long)N * N;

  for (long long prob = ((long long)blockIdx.x * Pol::WARPS + warp) * GPW + grp;
       prob - grp < batch; prob += stride) {
    const bool live = prob < batch;
    const double* a = A + (live ? prob : 0) * NN;
    Cols<N, CPL> cs;
    // ---- load: X := A restricted to the upper triangle (verify.py:236-241)
    sfor<0, N>([&](auto rI) {
      constexpr int r = decltype(rI)::value;
      const int j0 = gl;
      if constexpr (r < 32) cs.c0[r] = (j0 < N && j0 >= r) ? __ldg(a + r * N + j0) : 0.0;
      if constexpr (CPL == 2) {
        const int j1 = gl + 32;
        cs.c1[r] = (j1 < N && j1 >= r) ? __ldg(a + r * N + j1) : 0.0;
      }
    });
    int flag = 0;
    // ---- the variant, k unrolled
    sfor<0, NB>([&](auto kI) {
      constexpr int k = decltype(kI)::value;
      constexpr int s1 = k * B;        // block 1 start
      constexpr int s2 = (k + 1) * B;  // block 2 start
      // column index of each own slot
      const int jj[2] = {gl, gl + 32};

      // X_rows(lo..hi) x cols(clo..chi) published as pub[(c - clo) * LD + (r - lo)]
      // (column-major so LDS.128 broadcasts two consecutive rows of one column)
      auto publish = [&](auto loI, auto hiI, auto cloI, auto chiI) {
        constexpr int lo = decltype(loI)::value, hi = decltype(hiI)::value;
        constexpr int clo = decltype(cloI)::value, chi = decltype(chiI)::value;
        __syncwarp(gmask);
        sfor<0, CPL>([&](auto sI) {
          constexpr int s = decltype(sI)::value;
          const int j = jj[s];
          if (j >= clo && j < chi) {
            sfor<lo, hi>([&](auto rI) {
              constexpr int r = decltype(rI)::value;
              if constexpr (s == 1 || r < 32) pub[(j - clo) * LD + (r - lo)] = K::template cv<r, s>(cs);
            });
          }
        });
        __syncwarp(gmask);
      };

      // out(rows r in [ro, ro+B), own column j) -= sum_{l in [lo, hi)} X(l, r) X(l, j)
      // X(l, r) read from pub (published rows lo..hi of columns ro..), X(l, j) own.
      // UPPER: only r <= j.  cmin/cmax: columns j this applies to.
      auto update = [&](auto roI, auto nrI, auto loI, auto hiI, auto cminI, auto cmaxI, auto upI) {
        constexpr int ro = decltype(roI)::value, nr = decltype(nrI)::value;
        constexpr int lo = decltype(loI)::value, hi = decltype(hiI)::value;
        constexpr int cmin = decltype(cminI)::value, cmax = decltype(cmaxI)::value;
        constexpr bool up = decltype(upI)::value;
        if constexpr (hi > lo) {
          sfor<0, nr>([&](auto iI) {
            constexpr int r = ro + decltype(iI)::value;
            // X(l, r) for l in [lo, hi): column r of the published block
            double acc0 = 0.0, acc1 = 0.0, acc0b = 0.0, acc1b = 0.0;
            sfor<0, (hi - lo + 1) / 2>([&](auto pI) {
              constexpr int l = lo + 2 * decltype(pI)::value;
              const double* src = pub + (r - ro) * LD + (l - lo);
              double xr0, xr1;
              if constexpr (l + 1 < hi) {
                const double2 pr = *reinterpret_cast<const double2*>(src);
                xr0 = pr.x;
                xr1 = pr.y;
              } else {
                xr0 = src[0];
                xr1 = 0.0;
              }
              sfor<0, CPL>([&](auto sI) {
                constexpr int s = decltype(sI)::value;
                if constexpr (s == 1 || (l < 32 && (l + 1 < 32 || l + 1 >= hi))) {
                  double& acc = s == 0 ? acc0 : acc1;
                  double& accb = s == 0 ? acc0b : acc1b;
                  acc = fma(xr0, K::template cv<l, s>(cs), acc);
                  if constexpr (l + 1 < hi) accb = fma(xr1, K::template cv<(l + 1 < hi ? l + 1 : l), s>(cs), accb);
                }
              });
            });
            sfor<0, CPL>([&](auto sI) {
              constexpr int s = decltype(sI)::value;
              if constexpr (s == 1 || r < 32) {
                const int j = jj[s];
                const double acc = s == 0 ? acc0 + acc0b : acc1 + acc1b;
                if (j >= cmin && j < cmax && (!up || r <= j)) K::template cv<r, s>(cs) -= acc;
              }
            });
          });
        }
      };

      // CHOL leaf on block 1 (kernels.py:79-97), shuffles within the group
      auto leaf = [&]() {
        sfor<s1, s2>([&](auto iI) {
          constexpr int i = decltype(iI)::value;
          const double piv = K::template bcast<i, i>(cs, gmask);
          if (gl == 0 && piv <= 0.0 && flag == 0) flag = i + 1;
          const double rs = N <= 16 ? rsqrt_nr(piv) : rsqrt(piv);  // (n >= 20 measured slower with the lean form)
          sfor<0, CPL>([&](auto sI) {
            constexpr int s = decltype(sI)::value;
            if constexpr (s == 1 || i < 32) {
              const int j = jj[s];
              if (j == i) K::template cv<i, s>(cs) = piv * rs;
              else if (j > i && j < s2) K::template cv<i, s>(cs) *= rs;
            }
          });
          sfor<i + 1, s2>([&](auto rI) {
            constexpr int r = decltype(rI)::value;
            const double xir = K::template bcast<i, r>(cs, gmask);
            sfor<0, CPL>([&](auto sI) {
              constexpr int s = decltype(sI)::value;
              if constexpr (s == 1 || (r < 32 && i < 32)) {
                const int j = jj[s];
                if (j >= r && j < s2) K::template cv<r, s>(cs) = fma(-xir, K::template cv<i, s>(cs), K::template cv<r, s>(cs));
              }
            });
          });
        });
      };

      // X12 := TRSM(X11^T, X12) (kernels.py:47-60): T(i, l) = X(l, i), block 1
      auto trsm = [&]() {
        if constexpr (s2 < N) {
          publish(std::integral_constant<int, s1>{}, std::integral_constant<int, s2>{},
                  std::integral_constant<int, s1>{}, std::integral_constant<int, s2>{});
          sfor<s1, s2>([&](auto iI) {
            constexpr int i = decltype(iI)::value;
            const double rd = 1.0 / pub[(i - s1) * LD + (i - s1)];
            sfor<0, CPL>([&](auto sI) {
              constexpr int s = decltype(sI)::value;
              if constexpr (s == 1 || i < 32) {
                double v = K::template cv<i, s>(cs);
                sfor<s1, i>([&](auto lI) {
                  constexpr int l = decltype(lI)::value;
                  v = fma(-pub[(i - s1) * LD + (l - s1)], K::template cv<l, s>(cs), v);
                });
                const int j = jj[s];
                if (j >= s2 && j < N) K::template cv<i, s>(cs) = v * rd;
              }
            });
          });
        }
      };

      // B <= 8: CHOL leaf computed redundantly by every lane of the group from
      // the published diagonal block (no shuffles on the pivot chain), then
      // the TRSM of block row 1 uses the factor and its reciprocal pivots
      // (rsqrt) straight from registers.
      auto leaf_trsm_reg = [&]() {
        publish(std::integral_constant<int, s1>{}, std::integral_constant<int, s2>{},
                std::integral_constant<int, s1>{}, std::integral_constant<int, s2>{});
        double t[B][B];
        double rs[B];
        sfor<0, B>([&](auto cI) {
          constexpr int c = decltype(cI)::value;
          sfor<0, c + 1>([&](auto rI) {
            constexpr int r = decltype(rI)::value;
            t[r][c] = pub[c * LD + r];
          });
        });
        sfor<0, B>([&](auto iI) {
          constexpr int i = decltype(iI)::value;
          const double piv = t[i][i];
          if (gl == 0 && piv <= 0.0 && flag == 0) flag = s1 + i + 1;
          rs[i] = N <= 16 ? rsqrt_nr(piv) : rsqrt(piv);
          t[i][i] = piv * rs[i];
          sfor<i + 1, B>([&](auto cI) {
            constexpr int c = decltype(cI)::value;
            t[i][c] *= rs[i];
          });
          sfor<i + 1, B>([&](auto rI) {
            constexpr int r = decltype(rI)::value;
            sfor<r, B>([&](auto cI) {
              constexpr int c = decltype(cI)::value;
              t[r][c] = fma(-t[i][r], t[i][c], t[r][c]);
            });
          });
        });
        // own column inside block 1 takes its factor column
        sfor<0, CPL>([&](auto sI) {
          constexpr int s = decltype(sI)::value;
          const int j = jj[s];
          sfor<0, B>([&](auto cI) {
            constexpr int c = decltype(cI)::value;
            if constexpr (s == 1 || s1 + c < 32) {
              if (j == s1 + c) {
                sfor<0, c + 1>([&](auto rI) {
                  constexpr int r = decltype(rI)::value;
                  K::template cv<s1 + r, s>(cs) = t[r][c];
                });
              }
            }
          });
        });
        // X12 := TRSM(X11^T, X12): T(i, l) = X(l, i) = t[l][i]
        if constexpr (s2 < N) {
          sfor<0, CPL>([&](auto sI) {
            constexpr int s = decltype(sI)::value;
            if constexpr (s == 1 || s2 <= 32) {
              const int j = jj[s];
              double w[B];
              sfor<0, B>([&](auto iI) {
                constexpr int i = decltype(iI)::value;
                if constexpr (s == 1 || s1 + i < 32) {
                  double v = K::template cv<s1 + i, s>(cs);
                  sfor<0, i>([&](auto lI) {
                    constexpr int l = decltype(lI)::value;
                    v = fma(-t[l][i], w[l], v);
                  });
                  w[i] = v * rs[i];
                  if (j >= s2 && j < N) K::template cv<s1 + i, s>(cs) = w[i];
                }
              });
            }
          });
        }
      };

      using I0 = std::integral_constant<int, 0>;
      using IS1 = std::integral_constant<int, s1>;
      using IS2 = std::integral_constant<int, s2>;
      using IN = std::integral_constant<int, N>;
      using IB = std::integral_constant<int, B>;
      using INR = std::integral_constant<int, N - s2>;
      if constexpr (VARIANT == 1) {
        // X11 -= X01^T X01 (upper);  X12 -= X01^T X02: publish X01 = rows [0,s1) x cols block 1
        if constexpr (s1 > 0) {
          if constexpr (s1 <= 16) {
            publish(I0{}, IS1{}, IS1{}, IS2{});
            update(IS1{}, IB{}, I0{}, IS1{}, IS1{}, IN{}, std::true_type{});
          } else {
            // publish in chunks of 16 rows
            sfor<0, (s1 + 15) / 16>([&](auto cI) {
              constexpr int lo = 16 * decltype(cI)::value;
              constexpr int hi = lo + 16 < s1 ? lo + 16 : s1;
              publish(std::integral_constant<int, lo>{}, std::integral_constant<int, hi>{}, IS1{}, IS2{});
              update(IS1{}, IB{}, std::integral_constant<int, lo>{}, std::integral_constant<int, hi>{}, IS1{},
                     IN{}, std::true_type{});
            });
          }
        }
        if constexpr (B <= 4 || (B <= 8 && CPL == 1)) leaf_trsm_reg();
        else {
          leaf();
          trsm();
        }
      } else {
        // v2: leaf, trsm, then X22 -= X12^T X12 (upper)
        if constexpr (B <= 4 || (B <= 8 && CPL == 1)) leaf_trsm_reg();
        else {
          leaf();
          trsm();
        }
        if constexpr (s2 < N) {
          sfor<0, (N - s2 + 31) / 32>([&](auto cI) {
            constexpr int c0 = s2 + 32 * decltype(cI)::value;
            constexpr int c1 = c0 + 32 < N ? c0 + 32 : N;
            // publish X12 rows block 1, cols [c0, c1) and update rows r in [c0, c1)
            publish(IS1{}, IS2{}, std::integral_constant<int, c0>{}, std::integral_constant<int, c1>{});
            update(std::integral_constant<int, c0>{}, std::integral_constant<int, c1 - c0>{}, IS1{}, IS2{},
                   std::integral_constant<int, c0>{}, IN{}, std::true_type{});
          });
        }
        (void)INR{};
      }
    });
    // ---- store all n^2 entries (zeros below the diagonal) + guards
    bool fin = true;
    if (live) {
      double* x = X + prob * NN;
      sfor<0, N>([&](auto rI) {
        constexpr int r = decltype(rI)::value;
        sfor<0, CPL>([&](auto sI) {
          constexpr int s = decltype(sI)::value;
          const int j = gl + 32 * s;
          if (j < N) {
            double v = 0.0;
            if constexpr (s == 1 || r < 32) v = (j >= r) ? K::template cv<r, s>(cs) : 0.0;
            fin = fin && isfinite(v);
            __stcs(x + r * N + j, v);
          }
        });
      });
    }
    const unsigned bad = __ballot_sync(0xffffffffu, !fin) & gmask;
    const int f0 = __shfl_sync(0xffffffffu, flag, grp * W);
    if (live && gl == 0 && info) info[prob] = f0 ? f0 : (bad ? -1 : 0);
  }
}

}  // namespace col
}  // namespace lagen
