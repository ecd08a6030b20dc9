// lagen_b200.cu — the C ABI (include/lagen_b200.h): validation, (eq, n, b)
// dispatch to the size-specialised instances, the host-buffer pipeline and
// the seeded batched generator.  No C++ exception crosses the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>
#include <string>

#include "inst_index.h"
#include "lagen_b200.h"
#include "registry.cuh"
#include "registry_col.cuh"
#include "registry_rows.cuh"
#include "registry_warp.cuh"
#include "registry_pipe.cuh"
#include "registry_rowsweep.cuh"
#include "variants_table.h"

using namespace lagen;

namespace lagen {
// bigsolve.cu
cudaError_t launch_big(const StmtList& sl, int eq, int n, int b, const double* const* in, double* X, int* info,
                       long long batch, cudaStream_t s);
}  // namespace lagen

namespace {
thread_local std::string g_last_error;
}  // namespace

namespace lagen {
// shared with generate.cu: every failing entry point sets the message that
// lagen_b200_last_error() returns
int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
}  // namespace lagen

namespace {

int fail(int code, const std::string& msg) { return lagen::set_error(code, msg); }

int cuda_fail(cudaError_t e, const char* where) {
  return fail(LAGEN_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

const WarpEntry* find_warp(int eq, int n, int b, int variant) {
  if (eq < 0 || eq > 2 || variant < 0) return nullptr;
  for (int p = 0; p < kWarpParts; ++p) {
    const WarpTable& t = kWarpTables[eq][p];
    for (int i = 0; i < *t.n; ++i)
      if (t.e[i].n == n && t.e[i].b == b && t.e[i].variant == variant) return &t.e[i];
  }
  return nullptr;
}

const ColEntry* find_col(int eq, int n, int b, int variant) {
  if (eq != 0 || variant < 0) return nullptr;
  for (int p = 0; p < kColParts; ++p) {
    const ColTable& t = kColTables[p];
    for (int i = 0; i < *t.n; ++i)
      if (t.e[i].n == n && t.e[i].b == b && t.e[i].variant == variant) return &t.e[i];
  }
  return nullptr;
}

const RowsEntry* find_rows(int eq, int n, int b, int variant) {
  if (eq != 0 || variant < 0) return nullptr;
  for (int p = 0; p < kRowsParts; ++p) {
    const RowsTable& t = kRowsTables[p];
    for (int i = 0; i < *t.n; ++i)
      if (t.e[i].n == n && t.e[i].b == b && t.e[i].variant == variant) return &t.e[i];
  }
  return nullptr;
}

// padded rows engine: Cholesky v1 as the b = 8 kernel of a larger size on the
// identity-padded problem (n = 4 mod 8 -> n + 4; 104 -> 112, 120 -> 128)
const RowsEntry* find_rows_pad(int eq, int n, int b, int variant) {
  if (eq != 0 || variant != 1 || (b != 4 && b != 8)) return nullptr;
  for (int p = 0; p < kRowsPadParts; ++p) {
    const RowsPadTable& t = kRowsPadTables[p];
    for (int i = 0; i < *t.n; ++i)
      if (t.e[i].n == n) return &t.e[i];
  }
  return nullptr;
}

// mixed-block rows engine: Cholesky v1, n = 4 mod 8, partition 4, 8, 8, ...
const RowsEntry* find_rows_mix(int eq, int n, int b, int variant) {
  if (eq != 0 || variant != 1 || b != 4) return nullptr;
  for (int p = 0; p < kRowsMixParts; ++p) {
    const RowsPadTable& t = kRowsMixTables[p];
    for (int i = 0; i < *t.n; ++i)
      if (t.e[i].n == n) return &t.e[i];
  }
  return nullptr;
}

// pipe engine: Lyapunov v5 / Sylvester v13 order at 8x8-tile granularity
// (pipe.cuh), any block size the variant runs at
const PipeEntry* find_pipe(int eq, int n, int b, int variant) {
  (void)b;
  if (!((eq == 1 && variant == 5) || (eq == 2 && variant == 13))) return nullptr;
  for (int p = 0; p < kPipeParts; ++p) {
    const PipeTable& t = kPipeTables[p];
    for (int i = 0; i < *t.n; ++i)
      if (t.e[i].eq == eq && t.e[i].n == n) return &t.e[i];
  }
  return nullptr;
}

// rowsweep engine: Lyapunov / Sylvester n <= 32 as the b = n leaf (the SYLV
// / LYAP block kernel on the whole matrix, rowsweep.cuh) — every variant
// reduces to that single statement at b = n
const RowSweepEntry* find_rowsweep(int eq, int n, int b, int variant) {
  if (eq < 1 || eq > 2 || variant < 0 || b != n) return nullptr;
  for (int p = 0; p < kRowSweepParts; ++p) {
    const RowSweepTable& t = kRowSweepTables[p];
    for (int i = 0; i < *t.n; ++i)
      if (t.e[i].eq == eq && t.e[i].n == n) return &t.e[i];
  }
  return nullptr;
}

const lagen_stmt* builtin(int eq, int variant, int* count);

// index of the built-in variant whose statement list equals stmts, or -1
int match_builtin(int eq, const lagen_stmt* stmts, int nstmts) {
  for (int v = 0;; ++v) {
    int count = 0;
    const lagen_stmt* s = builtin(eq, v, &count);
    if (!s) return -1;
    if (count != nstmts) continue;
    bool same = true;
    for (int k = 0; k < count && same; ++k) {
      const lagen_stmt& a = s[k];
      const lagen_stmt& b = stmts[k];
      same = a.kind == b.kind && a.sign == b.sign && a.out.op == b.out.op && a.out.r == b.out.r &&
             a.out.c == b.out.c;
      for (int j = 0; j < 2 && same; ++j)
        same = a.in[j].op == b.in[j].op && (a.in[j].op < 0 || (a.in[j].r == b.in[j].r && a.in[j].c == b.in[j].c &&
                                                              a.in[j].trans == b.in[j].trans));
    }
    if (same) return v;
  }
}

const KernelEntry* find_entry(int eq, int n, int b) {
  if (eq < 0 || eq > 2) return nullptr;
  for (int p = 0; p < kTableParts; ++p) {
    const EntryTable& t = kTables[eq][p];
    for (int i = 0; i < *t.n; ++i)
      if (t.e[i].n == n && t.e[i].b == b) return &t.e[i];
  }
  return nullptr;
}

int eq_ninputs(int eq) { return eq + 1; }
int eq_ncoef(int eq) { return eq; }  // chol 0, lyap 1 (L), sylv 2 (L, U)

// Structural checks mirroring verify.py:263-295 / worksheet.py:47-67.
int validate(int eq, const lagen_stmt* stmts, int nstmts) {
  if (!stmts || nstmts <= 0) return fail(LAGEN_EVARIANT, "empty statement list");
  if (nstmts > LAGEN_MAX_STMTS) return fail(LAGEN_EVARIANT, "more than LAGEN_MAX_STMTS statements");
  static const int arity[5] = {2, 0, 1, 2, 1};
  const int ncoef = eq_ncoef(eq);
  for (int s = 0; s < nstmts; ++s) {
    const lagen_stmt& S = stmts[s];
    if (S.kind < 0 || S.kind > 4) return fail(LAGEN_EVARIANT, "unknown statement kind");
    if (S.out.op != 0) return fail(LAGEN_EVARIANT, "statement writes outside the output");
    if (S.out.trans) return fail(LAGEN_EVARIANT, "transposed output view");
    if (S.out.r < 0 || S.out.r > 2 || S.out.c < 0 || S.out.c > 2)
      return fail(LAGEN_EVARIANT, "block index out of range");
    if (S.kind == LAGEN_CHOL && (eq != LAGEN_CHOLESKY || S.out.r != S.out.c))
      return fail(LAGEN_EVARIANT, "CHOL statement outside a Cholesky diagonal block");
    if (S.kind == LAGEN_LYAP && (eq != LAGEN_LYAPUNOV || S.out.r != S.out.c))
      return fail(LAGEN_EVARIANT, "LYAP statement outside a Lyapunov diagonal block");
    if (S.kind == LAGEN_SYLV && eq == LAGEN_CHOLESKY) return fail(LAGEN_EVARIANT, "SYLV in Cholesky");
    if (S.kind == LAGEN_GEMM_UPDATE && S.sign != 1 && S.sign != -1)
      return fail(LAGEN_EVARIANT, "GEMM sign must be +-1");
    for (int j = 0; j < 2; ++j) {
      const lagen_view& v = S.in[j];
      if (j < arity[S.kind]) {
        if (v.op < 0 || v.op > ncoef) return fail(LAGEN_EVARIANT, "input view operand out of range");
        if (v.r < 0 || v.r > 2 || v.c < 0 || v.c > 2) return fail(LAGEN_EVARIANT, "input block out of range");
        if (v.trans != 0 && v.trans != 1) return fail(LAGEN_EVARIANT, "bad transpose flag");
        // coefficient diagonal blocks are packed (diag in a pad column): GEMM
        // operands from L/U must be off-diagonal blocks (true for every
        // synthesised variant)
        if (S.kind == LAGEN_GEMM_UPDATE && v.op > 0 && v.r == v.c)
          return fail(LAGEN_EVARIANT, "GEMM operand is a diagonal block of a triangular coefficient");
        if ((S.kind == LAGEN_SYLV || S.kind == LAGEN_LYAP || S.kind == LAGEN_TRSM_LEFT_TRANSPOSED) &&
            v.r != v.c)
          return fail(LAGEN_EVARIANT, "triangular coefficient is not a diagonal block");
      } else if (v.op != -1) {
        return fail(LAGEN_EVARIANT, "unexpected input view");
      }
    }
    if (S.kind == LAGEN_TRSM_LEFT_TRANSPOSED) {
      // logically lower coefficient: X^T of the upper factor (kernels.py:47-60)
      const lagen_view& v = S.in[0];
      const bool lower = (v.op == 0) ? (v.trans == 1) : (v.op == 1 ? v.trans == 0 : v.trans == 1);
      if (eq != LAGEN_CHOLESKY || !lower)
        return fail(LAGEN_EVARIANT, "TRSM coefficient must be logically lower");
    }
  }
  return LAGEN_OK;
}

// Sizes without a compiled instance (n not a multiple of 4, or a block size
// the instances do not use, e.g. (7, 7) or (10, 5)) run as the identity-padded
// problem of the next multiple of 4 — exact for all three equations:
//   A_p = diag(A, I)                  ->  X_p = diag(X, I)     (Cholesky)
//   L_p = diag(L, I), S_p = [S 0; 0 0] ->  X_p = [X 0; 0 0]     (Lyapunov)
//   L_p = diag(L, I), U_p = diag(U, I), C_p = [C 0; 0 0] -> X_p = [X 0; 0 0]
// (the unknown's first n rows / columns never read the padded ones: every
// variant is a forward recursion over the leading blocks), with the padded
// size's own block size b' (b itself when it divides n' and has an instance).
// Returns n' (0: none) and sets *bp.
int padded_size(int eq, int n, int b, int* bp) {
  const int np = n < 4 ? 4 : (n + 3) & ~3;
  if (np > 128) return 0;
  const int cands[4] = {b, 8, 4, 16};
  for (int c : cands)
    if (c >= 1 && np % c == 0 && find_entry(eq, np, c)) {
      *bp = c;
      return np;
    }
  return 0;
}

int check_common(int eq, int n, int b, long long batch, bool direct = false) {
  if (eq < 0 || eq > 2) return fail(LAGEN_EINVAL, "unknown equation");
  if (batch < 0) return fail(LAGEN_EINVAL, "negative batch");
  if (n < 1 || b < 1 || n % b) return fail(LAGEN_EUNSUPPORTED, "block size does not divide n");
  if (n > 128) {  // the big engine (bigsolve.cu)
    if (n > LAGEN_BIG_MAX_N)
      return fail(LAGEN_EUNSUPPORTED, "n = " + std::to_string(n) + " exceeds LAGEN_BIG_MAX_N");
    return LAGEN_OK;
  }
  int bp = 0;
  if (!direct && !find_entry(eq, n, b) && !padded_size(eq, n, b, &bp))
    return fail(LAGEN_EUNSUPPORTED, "no sm_100a instance for (n=" + std::to_string(n) + ", b=" +
                                        std::to_string(b) + ")");
  return LAGEN_OK;
}

// problem p, element (r, c) of the n' x n' padded operand.  Padded diagonal:
// 0 for a right-hand side, 1 for the Cholesky A, and for a Lyapunov /
// Sylvester coefficient d = 1 + max |diagonal| over the problem's L (and U),
// so every padded pivot (d + u_jj, l_ii + d, 2d) is nonzero (a fixed 1 gives
// 0 / 0 when a real diagonal entry is -1).
__global__ void pad_kernel(const double* __restrict__ src, double* __restrict__ dst, long long batch, int n, int np,
                           int mode, const double* __restrict__ co0, const double* __restrict__ co1) {
  const long long total = batch * np * np;
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < total;
       u += (long long)gridDim.x * blockDim.x) {
    const long long p = u / (np * np);
    const int e = (int)(u - p * np * np), r = e / np, c = e - r * np;
    double v = 0.0;
    if (r < n && c < n) {
      v = src[(p * n + r) * n + c];
    } else if (r == c && mode == 1) {
      v = 1.0;
    } else if (r == c && mode == 2) {
      double m = 0.0;
      for (int i = 0; i < n; ++i) {
        m = fmax(m, fabs(co0[(p * n + i) * n + i]));
        if (co1) m = fmax(m, fabs(co1[(p * n + i) * n + i]));
      }
      v = 1.0 + m;
    }
    dst[u] = v;
  }
}

__global__ void unpad_kernel(const double* __restrict__ src, double* __restrict__ dst, long long batch, int n,
                             int np) {
  const long long total = batch * n * n;
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < total;
       u += (long long)gridDim.x * blockDim.x) {
    const long long p = u / (n * n);
    const int e = (int)(u - p * n * n), r = e / n, c = e - r * n;
    dst[u] = src[(p * np + r) * np + c];
  }
}

int grid_for(long long total) {
  long long g = (total + 255) / 256;
  return (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

const lagen_stmt* builtin(int eq, int variant, int* count) {
  switch (eq) {
    case LAGEN_CHOLESKY:
      if (variant < 0 || variant >= kNumVariants_cholesky) return nullptr;
      *count = kNumStmts_cholesky[variant];
      return kStmts_cholesky[variant];
    case LAGEN_LYAPUNOV:
      if (variant < 0 || variant >= kNumVariants_lyapunov) return nullptr;
      *count = kNumStmts_lyapunov[variant];
      return kStmts_lyapunov[variant];
    case LAGEN_SYLVESTER:
      if (variant < 0 || variant >= kNumVariants_sylvester) return nullptr;
      *count = kNumStmts_sylvester[variant];
      return kStmts_sylvester[variant];
  }
  return nullptr;
}

}  // namespace

extern "C" {

int lagen_b200_abi_version(void) { return LAGEN_B200_ABI_VERSION; }

const char* lagen_b200_last_error(void) { return g_last_error.c_str(); }

int lagen_b200_num_variants(int eq) {
  switch (eq) {
    case LAGEN_CHOLESKY: return kNumVariants_cholesky;
    case LAGEN_LYAPUNOV: return kNumVariants_lyapunov;
    case LAGEN_SYLVESTER: return kNumVariants_sylvester;
  }
  return fail(LAGEN_EINVAL, "unknown equation");
}

int lagen_b200_variant_stmts(int eq, int variant, lagen_stmt* out, int cap) {
  int count = 0;
  const lagen_stmt* s = builtin(eq, variant, &count);
  if (!s) return fail(LAGEN_EVARIANT, "unknown variant index");
  if (out) {
    if (cap < count) return fail(LAGEN_EINVAL, "output capacity too small");
    std::memcpy(out, s, sizeof(lagen_stmt) * count);
  }
  return count;
}

int lagen_b200_supported(int eq, int n, int b) { return find_entry(eq, n, b) ? 1 : 0; }

int lagen_b200_geometry(int eq, int n, int b, int* g, int* p, int* threads, int* smem) {
  const KernelEntry* e = find_entry(eq, n, b);
  if (!e) return fail(LAGEN_EUNSUPPORTED, "no instance");
  if (g) *g = e->G;
  if (p) *p = e->P;
  if (threads) *threads = e->threads;
  if (smem) *smem = e->smem;
  return LAGEN_OK;
}

int lagen_b200_warp_supported(int eq, int n, int b, int variant) { return find_warp(eq, n, b, variant) ? 1 : 0; }

int lagen_b200_engine_supported(int eq, int n, int b, int variant, int engine) {
  switch (engine) {
    case LAGEN_ENGINE_GENERIC:
      if (n > 128) return (n <= LAGEN_BIG_MAX_N && b >= 1 && n % b == 0 && eq >= 0 && eq <= 2) ? 1 : 0;
      return find_entry(eq, n, b) ? 1 : 0;
    case LAGEN_ENGINE_WARP: return find_warp(eq, n, b, variant) ? 1 : 0;
    case LAGEN_ENGINE_COLUMN: return find_col(eq, n, b, variant) ? 1 : 0;
    case LAGEN_ENGINE_DATAFLOW: return 0;  // removed (never selected by the measured dispatch table)
    case LAGEN_ENGINE_ROWS: return find_rows(eq, n, b, variant) ? 1 : 0;
    case LAGEN_ENGINE_WAVE: return 0;  // superseded by the pipe engine
    case LAGEN_ENGINE_ROWS_PAD: return find_rows_pad(eq, n, b, variant) ? 1 : 0;
    case LAGEN_ENGINE_PIPE: return find_pipe(eq, n, b, variant) ? 1 : 0;
    case LAGEN_ENGINE_ROWSWEEP: return find_rowsweep(eq, n, b, variant) ? 1 : 0;
    case LAGEN_ENGINE_ROWS_MIX: return find_rows_mix(eq, n, b, variant) ? 1 : 0;
  }
  return 0;
}

int lagen_b200_execute(int eq, const lagen_stmt* stmts, int nstmts, int n, int b, long long batch,
                       const double* const* inputs, double* X, int* info, void* stream) {
  return lagen_b200_execute_engine(eq, stmts, nstmts, n, b, batch, inputs, X, info, stream, LAGEN_ENGINE_AUTO);
}

int lagen_b200_execute_engine(int eq, const lagen_stmt* stmts, int nstmts, int n, int b, long long batch,
                              const double* const* inputs, double* X, int* info, void* stream, int engine) {
  return lagen_b200_execute_profile(eq, stmts, nstmts, n, b, batch, inputs, X, info, stream, engine, nullptr);
}

int lagen_b200_execute_profile(int eq, const lagen_stmt* stmts, int nstmts, int n, int b, long long batch,
                               const double* const* inputs, double* X, int* info, void* stream, int engine,
                               unsigned long long* d_prof) {
  if (engine < LAGEN_ENGINE_AUTO || engine > LAGEN_ENGINE_ROWS_MIX) return fail(LAGEN_EINVAL, "unknown engine");
  if (eq < 0 || eq > 2) return fail(LAGEN_EINVAL, "unknown equation");
  if (batch < 0) return fail(LAGEN_EINVAL, "negative batch");
  int rc = validate(eq, stmts, nstmts);
  if (rc) return rc;
  // engines with their own instance for (n, b) that the generic table lacks
  // (rowsweep: b = n) run directly, without padding
  const RowSweepEntry* rs_direct =
      (engine == LAGEN_ENGINE_ROWSWEEP || engine == LAGEN_ENGINE_AUTO) && eq >= 1 && eq <= 2 && b == n
          ? find_rowsweep(eq, n, b, match_builtin(eq, stmts, nstmts))
          : nullptr;
  rc = check_common(eq, n, b, batch, rs_direct != nullptr);
  if (rc) return rc;
  if (batch == 0) return LAGEN_OK;
  if (!inputs || !X) return fail(LAGEN_EINVAL, "null buffer");
  for (int i = 0; i < eq_ninputs(eq); ++i)
    if (!inputs[i]) return fail(LAGEN_EINVAL, "null input buffer");
  if (n > 128) {  // beyond the shared-memory engines: X stays in HBM (bigsolve.cu)
    if (engine != LAGEN_ENGINE_AUTO && engine != LAGEN_ENGINE_GENERIC)
      return fail(LAGEN_EUNSUPPORTED, "n > 128 runs on the big engine only (engine auto or generic)");
    StmtList sl;
    std::memset(&sl, 0, sizeof(sl));
    std::memcpy(sl.s, stmts, sizeof(lagen_stmt) * nstmts);
    sl.count = nstmts;
    cudaError_t berr = launch_big(sl, eq, n, b, inputs, X, info, batch, static_cast<cudaStream_t>(stream));
    if (berr != cudaSuccess) return cuda_fail(berr, "big-engine launch");
    return LAGEN_OK;
  }
  if (!rs_direct && !find_entry(eq, n, b)) {  // identity-padded problem (see padded_size)
    int bp = 0;
    const int np = padded_size(eq, n, b, &bp);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int nin = eq_ninputs(eq);
    const size_t per = (size_t)batch * np * np;
    double* buf = nullptr;
    cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&buf), sizeof(double) * per * (nin + 1), s);
    if (err != cudaSuccess) return cuda_fail(err, "padded buffers");
    const double* pin[3] = {nullptr, nullptr, nullptr};
    // identity on the diagonal of A, a per-problem nonzero-pivot value on the
    // diagonal of L and U, zeros in S and C
    for (int i = 0; i < nin; ++i) {
      const bool rhs = (eq == LAGEN_LYAPUNOV && i == 1) || (eq == LAGEN_SYLVESTER && i == 2);
      const int mode = rhs ? 0 : (eq == LAGEN_CHOLESKY ? 1 : 2);
      pad_kernel<<<grid_for((long long)per), 256, 0, s>>>(inputs[i], buf + per * i, batch, n, np, mode, inputs[0],
                                                          eq == LAGEN_SYLVESTER ? inputs[1] : nullptr);
      pin[i] = buf + per * i;
    }
    double* Xp = buf + per * nin;
    int rc2 = lagen_b200_execute_profile(eq, stmts, nstmts, np, bp, batch, pin, Xp, info, stream, engine, d_prof);
    if (rc2 == LAGEN_OK) {
      unpad_kernel<<<grid_for(batch * n * n), 256, 0, s>>>(Xp, X, batch, n, np);
      err = cudaGetLastError();
      if (err != cudaSuccess) rc2 = cuda_fail(err, "unpad launch");
    }
    cudaFreeAsync(buf, s);
    return rc2;
  }
  LaunchArgs a;
  std::memset(&a, 0, sizeof(a));
  std::memcpy(a.sl.s, stmts, sizeof(lagen_stmt) * nstmts);
  a.sl.count = nstmts;
  for (int i = 0; i < 3; ++i) a.in[i] = i < eq_ninputs(eq) ? inputs[i] : inputs[0];
  a.X = X;
  a.info = info;
  a.batch = batch;
  a.prof = d_prof;
  const KernelEntry* ge = find_entry(eq, n, b);
  if (!ge && !rs_direct) return fail(LAGEN_EUNSUPPORTED, "no sm_100a instance");
  if (engine == LAGEN_ENGINE_GENERIC && !ge) return fail(LAGEN_EUNSUPPORTED, "no generic instance for this (n, b)");
  LaunchFn fn = ge ? ge->launch : rs_direct->launch;
  if (engine != LAGEN_ENGINE_GENERIC) {
    const int v = match_builtin(eq, stmts, nstmts);
    const ColEntry* c = (engine == LAGEN_ENGINE_AUTO || engine == LAGEN_ENGINE_COLUMN) ? find_col(eq, n, b, v) : nullptr;
    const WarpEntry* w = (engine == LAGEN_ENGINE_AUTO || engine == LAGEN_ENGINE_WARP) ? find_warp(eq, n, b, v) : nullptr;
    if (engine == LAGEN_ENGINE_COLUMN && !c)
      return fail(LAGEN_EUNSUPPORTED, "no column-engine instance for this (variant, n, b)");
    if (engine == LAGEN_ENGINE_WARP && !w)
      return fail(LAGEN_EUNSUPPORTED, "no warp-engine instance for this (variant, n, b)");
    if (engine == LAGEN_ENGINE_DATAFLOW || engine == LAGEN_ENGINE_WAVE)
      return fail(LAGEN_EUNSUPPORTED, "the dataflow and wave engines were removed (never the fastest measured path)");
    // AUTO: the rows engine (Cholesky v1, n > 32) is the fastest measured path
    // (dispatch_table.json); the register column engine below that
    const RowsEntry* st =
        (engine == LAGEN_ENGINE_ROWS || (engine == LAGEN_ENGINE_AUTO && n > 32)) ? find_rows(eq, n, b, v) : nullptr;
    if (engine == LAGEN_ENGINE_ROWS && !st)
      return fail(LAGEN_EUNSUPPORTED, "no rows-engine instance for this (variant, n, b)");
    // AUTO: the pipe engine for the right-looking Lyapunov / Sylvester
    // variants (dispatch_table.json measures the rest)
    const PipeEntry* pp =
        (engine == LAGEN_ENGINE_PIPE || engine == LAGEN_ENGINE_AUTO) ? find_pipe(eq, n, b, v) : nullptr;
    if (engine == LAGEN_ENGINE_PIPE && !pp)
      return fail(LAGEN_EUNSUPPORTED, "no pipe-engine instance for this (variant, n, b)");
    // AUTO: the rowsweep engine whenever b = n (n <= 32)
    const RowSweepEntry* rs =
        (engine == LAGEN_ENGINE_ROWSWEEP || engine == LAGEN_ENGINE_AUTO) ? find_rowsweep(eq, n, b, v) : nullptr;
    if (engine == LAGEN_ENGINE_ROWSWEEP && !rs)
      return fail(LAGEN_EUNSUPPORTED, "no rowsweep-engine instance for this (variant, n, b): it runs b = n, n <= 32");
    const RowsEntry* rp = (engine == LAGEN_ENGINE_ROWS_PAD) ? find_rows_pad(eq, n, b, v) : nullptr;
    if (engine == LAGEN_ENGINE_ROWS_PAD && !rp)
      return fail(LAGEN_EUNSUPPORTED, "no padded rows-engine instance for this (variant, n, b)");
    const RowsEntry* rm = (engine == LAGEN_ENGINE_ROWS_MIX) ? find_rows_mix(eq, n, b, v) : nullptr;
    if (engine == LAGEN_ENGINE_ROWS_MIX && !rm)
      return fail(LAGEN_EUNSUPPORTED, "no mixed-block rows-engine instance for this (variant, n, b): Cholesky v1, n = 4 mod 8, b = 4");
    if (rm) fn = rm->launch;
    else if (rp) fn = rp->launch;
    else if (rs) fn = rs->launch;
    else if (pp) fn = pp->launch;
    else if (st) fn = st->launch;
    else if (c) fn = c->launch;
    else if (w) fn = w->launch;
  }
  cudaError_t err = fn(a, static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "solve launch");
  return LAGEN_OK;
}

static int run_variant(int eq, int variant, int n, int b, long long batch, const double* const* in, double* X,
                       int* info, void* stream) {
  int count = 0;
  const lagen_stmt* s = builtin(eq, variant, &count);
  if (!s) return fail(LAGEN_EVARIANT, "unknown variant index");
  return lagen_b200_execute(eq, s, count, n, b, batch, in, X, info, stream);
}

int lagen_b200_cholesky(int variant, int n, int b, long long batch, const double* A, double* X, int* info,
                        void* stream) {
  const double* in[1] = {A};
  return run_variant(LAGEN_CHOLESKY, variant, n, b, batch, in, X, info, stream);
}

int lagen_b200_lyapunov(int variant, int n, int b, long long batch, const double* L, const double* S, double* X,
                        int* info, void* stream) {
  const double* in[2] = {L, S};
  return run_variant(LAGEN_LYAPUNOV, variant, n, b, batch, in, X, info, stream);
}

int lagen_b200_sylvester(int variant, int n, int b, long long batch, const double* L, const double* U,
                         const double* C, double* X, int* info, void* stream) {
  const double* in[3] = {L, U, C};
  return run_variant(LAGEN_SYLVESTER, variant, n, b, batch, in, X, info, stream);
}

// Host-buffer pipeline: chunks of the batch cycle through NS device buffer
// sets on NS streams so the H2D engine, the SMs and the D2H engine all stay
// busy (with 2 sets the H2D of chunk c+2 would wait for the D2H of chunk c).
// Streams and staging buffers persist across calls (per device, grown on
// demand, one caller at a time): a sweep of many sizes pays no per-call
// stream creation / allocation, and no pool release between calls.
namespace {
constexpr int kNS = 4;
// Cholesky moves only row bands of the upper triangle over PCIe: band j =
// rows [r0, r1), columns [c0, n), c0 = r0 rounded down to 8 (covers every
// entry any Cholesky engine reads: columns >= 4 floor(r / 4)); K = n / 16
// bands keep the shortest copied row >= 128 B, where the copy engines still
// run at full rate (tools/band_copy_probe.cu).  Lyapunov / Sylvester return
// a full X, so their D2H bounds the pipeline and they copy whole matrices.
struct Bands {
  int K = 0;
  int r0[16], r1[16], c0[16];
};
Bands host_bands(int eq, int n) {
  Bands b;
  // opt-in (LAGEN_HOST_BANDS=1): measured on the B200 box, the banded copies
  // run below the whole-matrix rate in bidirectional traffic and the host
  // zero-fill costs ~1 ms per 256 MiB, so whole copies win or tie at every n
  // (tools/e2e_probe3.py, profiles/r01_e2e_bands.txt)
  static const int mode = [] {
    const char* e = std::getenv("LAGEN_HOST_BANDS");
    return e ? std::atoi(e) : 0;
  }();
  if (eq != LAGEN_CHOLESKY || n < 32 || mode == 0) return b;
  b.K = n / 16 > 16 ? 16 : n / 16;
  for (int j = 0; j < b.K; ++j) {
    b.r0[j] = j * n / b.K;
    b.r1[j] = (j + 1) * n / b.K;
    b.c0[j] = b.r0[j] & ~7;
  }
  return b;
}
struct HostPipe {
  int dev = -1;
  cudaStream_t st[kNS] = {nullptr};
  double* d_in[kNS][3] = {{nullptr}};
  double* d_X[kNS] = {nullptr};
  int* d_info[kNS] = {nullptr};
  size_t cap_bytes = 0, cap_info = 0;
  long long it = 0;  // chunks issued so far: chunk i runs on stream i mod kNS, across calls
  cudaError_t reserve(size_t bytes, size_t info_bytes) {
    if (bytes <= cap_bytes && info_bytes <= cap_info) return cudaSuccess;
    for (int k = 0; k < kNS; ++k) {
      if (st[k]) cudaStreamSynchronize(st[k]);
      for (int i = 0; i < 3; ++i) cudaFree(d_in[k][i]), d_in[k][i] = nullptr;
      cudaFree(d_X[k]), d_X[k] = nullptr;
      cudaFree(d_info[k]), d_info[k] = nullptr;
    }
    cap_bytes = cap_info = 0;
    cudaError_t err = cudaSuccess;
    for (int k = 0; k < kNS && err == cudaSuccess; ++k) {
      if (!st[k]) err = cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking);
      for (int i = 0; i < 3 && err == cudaSuccess; ++i) {
        err = cudaMalloc(&d_in[k][i], bytes);
        if (err == cudaSuccess) err = cudaMemset(d_in[k][i], 0, bytes);  // never-copied parts read as 0
      }
      if (err == cudaSuccess) err = cudaMalloc(&d_X[k], bytes);
      if (err == cudaSuccess) err = cudaMalloc(&d_info[k], info_bytes);
    }
    if (err == cudaSuccess) {
      cap_bytes = bytes;
      cap_info = info_bytes;
    }
    return err;
  }
};
std::mutex g_pipe_mu;
HostPipe g_pipe[64];

// Zero-copy triangle transfer (LAGEN_HOST_TRIANGLES): kernels read the
// needed part of each input row straight from mapped pinned host memory into
// the device staging buffer, and write X's rows back the same way, so PCIe
// carries only the structurally needed bytes (SURVEY §8d compulsory bytes)
// instead of dense matrices.  Row r of an operand moves columns [c0, c1):
//   part 0 (full)  : [0, n)
//   part 1 (upper) : [8 floor(r / 8), n)      A, S, U; Cholesky X (zeroed host X)
//   part 2 (lower) : [0, min(n, 8 floor(r / 8) + 8))   L
// in 16-byte units (n even).  The parts of the device staging buffer that are
// not copied hold stale finite values (zeroed on allocation); no engine reads
// them (tests: test_unread_triangles_are_ignored).
__host__ __device__ inline void part_cols(int part, int n, int r, int* c0, int* c1) {
  *c0 = part == 1 ? (r & ~7) : 0;
  *c1 = part == 2 ? ((r & ~7) + 8 < n ? (r & ~7) + 8 : n) : n;
}
// rows' 16-byte unit offsets inside one problem: unit u of the problem lies in
// row r with start[r] <= u < start[r + 1], column col0[r] + 2 (u - start[r])
struct TriRows {
  int start[130];
  int col0[129];
};
// A per-unit offset table (16-byte units inside one problem) is built in
// shared memory once per CTA; every thread then keeps four independent
// 16-byte transfers in flight (PCIe reads are latency-bound per request).
__global__ void tri_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, long long cnt, int n,
                                const __grid_constant__ TriRows tr) {
  extern __shared__ unsigned short tri_tab[];  // unit u -> (row * n + column) / 2
  const int U = tr.start[n];                   // units per problem
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const int base = (r * n + tr.col0[r]) >> 1;
    for (int u = tr.start[r]; u < tr.start[r + 1]; ++u) tri_tab[u] = (unsigned short)(base + (u - tr.start[r]));
  }
  __syncthreads();
  const double2* __restrict__ s2 = reinterpret_cast<const double2*>(src);
  double2* __restrict__ d2 = reinterpret_cast<double2*>(dst);
  const long long total = cnt * U, nn2 = (long long)n * n / 2;
  const long long step = (long long)gridDim.x * 4 * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * 4 * blockDim.x + threadIdx.x; i0 < total; i0 += step) {
    double2 v[4];
    long long off[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const long long i = i0 + (long long)k * blockDim.x;
      off[k] = -1;
      if (i < total) {
        const long long p = i / U;
        off[k] = p * nn2 + tri_tab[(int)(i - p * U)];
        v[k] = s2[off[k]];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (off[k] >= 0) d2[off[k]] = v[k];
  }
}
TriRows tri_rows(int part, int n) {
  TriRows t;
  t.start[0] = 0;
  for (int r = 0; r < n; ++r) {
    int c0, c1;
    part_cols(part, n, r, &c0, &c1);
    t.col0[r] = c0;
    t.start[r + 1] = t.start[r] + (c1 - c0) / 2;
  }
  return t;
}
long long part_doubles(int part, int n);
// Hybrid transfer of a triangular part: the half of the rows that is mostly
// needed goes through the copy engines as ONE strided copy per chunk — rows
// [0, s) (upper part) or [s, n) (lower part) of a row-major matrix are
// contiguous, s n doubles per problem, so the 2-D copy has one long row per
// problem — and only the remaining small triangle (rows [s, n) of an upper
// part, rows [0, s) of a lower part) goes through the zero-copy kernel.
// Measured (tools/e2e_probe4.py): the copy engines move 45 GB/s each way
// under bidirectional load, the zero-copy kernels 25, so the bulk belongs on
// the engines.  s = n / 2 rounded down to the 8-column tile grid; 0 (no
// split) below n = 16.  LAGEN_HOST_SPLIT=0 restores all-zero-copy triangles.
int split_row(int n) {
  static const int on = [] {
    const char* e = std::getenv("LAGEN_HOST_SPLIT");
    return e ? std::atoi(e) : 1;
  }();
  if (!on || n < 16) return 0;
  return (n / 2) & ~7;
}
// rows [ra, rb) of a part only
TriRows tri_rows_range(int part, int n, int ra, int rb) {
  TriRows t;
  t.start[0] = 0;
  for (int r = 0; r < n; ++r) {
    int c0, c1;
    part_cols(part, n, r, &c0, &c1);
    if (r < ra || r >= rb) c1 = c0;
    t.col0[r] = c0;
    t.start[r + 1] = t.start[r] + (c1 - c0) / 2;
  }
  return t;
}
// doubles per problem a part moves over PCIe with the split at row s
long long part_doubles_split(int part, int n, int s) {
  if (part == 0) return (long long)n * n;
  if (s <= 0) return part_doubles(part, n);
  long long t = part == 1 ? (long long)s * n : (long long)(n - s) * n;  // the engine-copied rows, full width
  for (int r = (part == 1 ? s : 0); r < (part == 1 ? n : s); ++r) {
    int c0, c1;
    part_cols(part, n, r, &c0, &c1);
    t += c1 - c0;
  }
  return t;
}
int input_part(int eq, int i) {
  if (eq == LAGEN_CHOLESKY) return 1;                 // A: upper
  if (i == 0) return 2;                               // L: lower
  if (eq == LAGEN_LYAPUNOV) return 1;                 // S: upper
  return i == 1 ? 1 : 0;                              // Sylvester U: upper, C: full
}
long long part_doubles(int part, int n) {
  long long t = 0;
  for (int r = 0; r < n; ++r) {
    int c0, c1;
    part_cols(part, n, r, &c0, &c1);
    t += c1 - c0;
  }
  return t;
}
// device address of mapped pinned host memory, or nullptr
const void* mapped(const void* h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
  return a.devicePointer;
}
}  // namespace

int lagen_b200_execute_host(int eq, const lagen_stmt* stmts, int nstmts, int n, int b, long long batch,
                            const double* const* h_inputs, double* h_X, int* h_info) {
  return lagen_b200_execute_host_engine(eq, stmts, nstmts, n, b, batch, h_inputs, h_X, h_info, LAGEN_ENGINE_AUTO);
}

int lagen_b200_execute_host_engine(int eq, const lagen_stmt* stmts, int nstmts, int n, int b, long long batch,
                                   const double* const* h_inputs, double* h_X, int* h_info, int engine) {
  return lagen_b200_execute_host_flags(eq, stmts, nstmts, n, b, batch, h_inputs, h_X, h_info, engine, 0);
}

int lagen_b200_execute_host_flags(int eq, const lagen_stmt* stmts, int nstmts, int n, int b, long long batch,
                                  const double* const* h_inputs, double* h_X, int* h_info, int engine, int flags) {
  if (flags & ~(LAGEN_HOST_TRIANGLES | LAGEN_HOST_X_ZEROED | LAGEN_HOST_ASYNC))
    return fail(LAGEN_EINVAL, "unknown host flags");
  const bool async = (flags & LAGEN_HOST_ASYNC) != 0;
  if (engine < LAGEN_ENGINE_AUTO || engine > LAGEN_ENGINE_ROWS_MIX) return fail(LAGEN_EINVAL, "unknown engine");
  if (eq < 0 || eq > 2) return fail(LAGEN_EINVAL, "unknown equation");
  if (batch < 0) return fail(LAGEN_EINVAL, "negative batch");
  int rc = validate(eq, stmts, nstmts);
  if (rc) return rc;
  // engines with their own instance for (n, b) that the generic table lacks
  // (rowsweep: b = n) run directly, without padding
  const RowSweepEntry* rs_direct =
      (engine == LAGEN_ENGINE_ROWSWEEP || engine == LAGEN_ENGINE_AUTO) && eq >= 1 && eq <= 2 && b == n
          ? find_rowsweep(eq, n, b, match_builtin(eq, stmts, nstmts))
          : nullptr;
  rc = check_common(eq, n, b, batch, rs_direct != nullptr);
  if (rc) return rc;
  if (batch == 0) return LAGEN_OK;
  if (!h_inputs || !h_X) return fail(LAGEN_EINVAL, "null buffer");
  const int nin = eq_ninputs(eq);
  for (int i = 0; i < nin; ++i)
    if (!h_inputs[i]) return fail(LAGEN_EINVAL, "null input buffer");
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return cuda_fail(err, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(LAGEN_EINVAL, "device index out of range");
  const size_t prob_bytes = sizeof(double) * (size_t)n * n;
  // ~16 MiB of input per chunk and operand, at least one problem
  long long chunk = (16ll << 20) / (long long)prob_bytes;
  if (chunk < 1) chunk = 1;
  const Bands bd = host_bands(eq, n);
  std::lock_guard<std::mutex> lock(g_pipe_mu);
  HostPipe& hp = g_pipe[dev];
  // one capacity for every size (a chunk is <= 16 MiB per operand), so a
  // sequence of calls never reallocates under queued work
  err = hp.reserve(std::max((size_t)chunk * prob_bytes, (size_t)16 << 20),
                   std::max((size_t)chunk * sizeof(int), (size_t)1 << 20));
  if (err != cudaSuccess) return cuda_fail(err, "host pipeline setup");
  if (chunk > batch) chunk = batch;
  // zero-copy triangles: every buffer must be mapped pinned memory and n even
  const double* mh_in[3] = {nullptr, nullptr, nullptr};
  double* mh_X = nullptr;
  bool tri = (flags & LAGEN_HOST_TRIANGLES) && n % 2 == 0 && n <= 128;
  for (int i = 0; i < nin && tri; ++i) tri = (mh_in[i] = static_cast<const double*>(mapped(h_inputs[i]))) != nullptr;
  if (tri) tri = (mh_X = static_cast<double*>(const_cast<void*>(mapped(h_X)))) != nullptr;
  if ((flags & LAGEN_HOST_TRIANGLES) && !tri)
    return fail(LAGEN_EINVAL, "LAGEN_HOST_TRIANGLES needs mapped pinned host buffers and an even n");
  const int xpart = (eq == LAGEN_CHOLESKY && (flags & LAGEN_HOST_X_ZEROED)) ? 1 : 0;
  if (tri) {
    int status = LAGEN_OK;
    // the transfer kernels run on SMs the persistent solves leave free
    struct Reserve {
      Reserve() { t_sm_reserve = 8; }
      ~Reserve() { t_sm_reserve = 0; }
    } reserve_guard;
    const int sp = split_row(n);
    // zero-copy regions: the whole part without a split; with it, rows [sp, n)
    // of an upper part and rows [0, sp) of a lower part
    TriRows parts[3] = {tri_rows(0, n), sp ? tri_rows_range(1, n, sp, n) : tri_rows(1, n),
                        sp ? tri_rows_range(2, n, 0, sp) : tri_rows(2, n)};
    // one operand chunk: engine copy of the contiguous half (or of a full
    // part), then the zero-copy kernel for the remaining rows; both on stream
    // st.  src / dst are a mapped-host and a device pointer (either order;
    // unified addressing lets the engines resolve the direction).
    auto tcopy = [&](const double* src, double* dst, long long cnt, int part, cudaStream_t st) {
      if (part == 0) return cudaMemcpyAsync(dst, src, (size_t)cnt * prob_bytes, cudaMemcpyDefault, st);
      if (sp) {
        const size_t row0 = part == 1 ? 0 : (size_t)sp * n;  // first engine-copied element
        const size_t width = (part == 1 ? (size_t)sp : (size_t)(n - sp)) * n * sizeof(double);
        cudaError_t e = cudaMemcpy2DAsync(dst + row0, prob_bytes, src + row0, prob_bytes, width, (size_t)cnt,
                                          cudaMemcpyDefault, st);
        if (e != cudaSuccess) return e;
      }
      const long long units = cnt * parts[part].start[n];
      if (units == 0) return cudaSuccess;
      long long grid = (units + 2047) / 2048;
      if (grid > 32) grid = 32;  // 32 CTAs x 512 threads x 4 transfers keep PCIe busy (tools/zc_probe.cu)
      if (grid < 1) grid = 1;
      tri_copy_kernel<<<(unsigned)grid, 512, (size_t)parts[part].start[n] * sizeof(unsigned short), st>>>(
          src, dst, cnt, n, parts[part]);
      return cudaGetLastError();
    };
    for (long long c0 = 0; status == LAGEN_OK && c0 < batch; c0 += chunk) {
      const int k = (int)(hp.it++ % kNS);
      const long long cnt = (batch - c0) < chunk ? (batch - c0) : chunk;
      for (int i = 0; i < nin && err == cudaSuccess; ++i)
        err = tcopy(mh_in[i] + c0 * n * n, hp.d_in[k][i], cnt, input_part(eq, i), hp.st[k]);
      if (err != cudaSuccess) { status = cuda_fail(err, "triangle gather"); break; }
      const double* ins[3] = {hp.d_in[k][0], hp.d_in[k][1], hp.d_in[k][2]};
      status = lagen_b200_execute_engine(eq, stmts, nstmts, n, b, cnt, ins, hp.d_X[k],
                                         h_info ? hp.d_info[k] : nullptr, hp.st[k], engine);
      if (status != LAGEN_OK) break;
      err = tcopy(hp.d_X[k], mh_X + c0 * n * n, cnt, xpart, hp.st[k]);
      if (err == cudaSuccess && h_info)
        err = cudaMemcpyAsync(h_info + c0, hp.d_info[k], cnt * sizeof(int), cudaMemcpyDeviceToHost, hp.st[k]);
      if (err != cudaSuccess) { status = cuda_fail(err, "triangle scatter"); break; }
    }
    for (int k = 0; k < kNS && (!async || status != LAGEN_OK); ++k) {
      cudaError_t e2 = cudaStreamSynchronize(hp.st[k]);
      if (e2 != cudaSuccess && status == LAGEN_OK) status = cuda_fail(e2, "host pipeline sync");
    }
    return status;
  }
  // Cholesky: the strictly-lower part of X left of each band is zero; the
  // host writes it (threads, overlapped with the copies) instead of PCIe
  std::vector<std::thread> fill;
  static const bool no_fill = std::getenv("LAGEN_HOST_NOFILL") != nullptr;  // measurement only: X left partly unwritten
  if (bd.K > 0 && !no_fill) {
    unsigned nt = std::thread::hardware_concurrency();
    nt = nt < 1 ? 1 : (nt > 16 ? 16 : nt);
    for (unsigned t = 0; t < nt; ++t)
      fill.emplace_back([=]() {
        const long long p0 = batch * t / nt, p1 = batch * (t + 1) / nt;
        for (long long p = p0; p < p1; ++p)
          for (int j = 0; j < bd.K; ++j)
            if (bd.c0[j] > 0)
              for (int r = bd.r0[j]; r < bd.r1[j]; ++r)
                std::memset(h_X + (p * n + r) * (long long)n, 0, sizeof(double) * bd.c0[j]);
      });
  }
  auto copy = [&](double* dst, const double* src, long long cnt, cudaMemcpyKind kind, cudaStream_t st) {
    if (bd.K == 0) return cudaMemcpyAsync(dst, src, cnt * prob_bytes, kind, st);
    for (int j = 0; j < bd.K; ++j) {
      cudaMemcpy3DParms p = {};
      p.srcPtr = make_cudaPitchedPtr(const_cast<double*>(src), sizeof(double) * n, n, n);
      p.dstPtr = make_cudaPitchedPtr(dst, sizeof(double) * n, n, n);
      p.srcPos = make_cudaPos(sizeof(double) * bd.c0[j], bd.r0[j], 0);
      p.dstPos = p.srcPos;
      p.extent = make_cudaExtent(sizeof(double) * (n - bd.c0[j]), bd.r1[j] - bd.r0[j], cnt);
      p.kind = kind;
      cudaError_t e = cudaMemcpy3DAsync(&p, st);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  int status = LAGEN_OK;
  for (long long c0 = 0; status == LAGEN_OK && c0 < batch; c0 += chunk) {
    const int k = (int)(hp.it++ % kNS);
    const long long cnt = (batch - c0) < chunk ? (batch - c0) : chunk;
    for (int i = 0; i < nin && err == cudaSuccess; ++i)
      err = copy(hp.d_in[k][i], h_inputs[i] + c0 * n * n, cnt, cudaMemcpyHostToDevice, hp.st[k]);
    if (err != cudaSuccess) { status = cuda_fail(err, "H2D"); break; }
    const double* ins[3] = {hp.d_in[k][0], hp.d_in[k][1], hp.d_in[k][2]};
    status = lagen_b200_execute_engine(eq, stmts, nstmts, n, b, cnt, ins, hp.d_X[k], h_info ? hp.d_info[k] : nullptr,
                                       hp.st[k], engine);
    if (status != LAGEN_OK) break;
    err = copy(h_X + c0 * n * n, hp.d_X[k], cnt, cudaMemcpyDeviceToHost, hp.st[k]);
    if (err == cudaSuccess && h_info)
      err = cudaMemcpyAsync(h_info + c0, hp.d_info[k], cnt * sizeof(int), cudaMemcpyDeviceToHost, hp.st[k]);
    if (err != cudaSuccess) { status = cuda_fail(err, "D2H"); break; }
  }
  for (int k = 0; k < kNS && (!async || status != LAGEN_OK); ++k) {
    cudaError_t e2 = cudaStreamSynchronize(hp.st[k]);
    if (e2 != cudaSuccess && status == LAGEN_OK) status = cuda_fail(e2, "host pipeline sync");
  }
  for (auto& th : fill) th.join();
  return status;
}

int lagen_b200_host_sync(void) {
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return cuda_fail(err, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(LAGEN_EINVAL, "device index out of range");
  std::lock_guard<std::mutex> lock(g_pipe_mu);
  HostPipe& hp = g_pipe[dev];
  int status = LAGEN_OK;
  for (int k = 0; k < kNS; ++k) {
    if (!hp.st[k]) continue;
    cudaError_t e2 = cudaStreamSynchronize(hp.st[k]);
    if (e2 != cudaSuccess && status == LAGEN_OK) status = cuda_fail(e2, "host pipeline sync");
  }
  return status;
}

int lagen_b200_host_bytes_flags(int eq, int n, long long batch, int flags, long long* h2d, long long* d2h) {
  if (!(flags & LAGEN_HOST_TRIANGLES) || n % 2) return lagen_b200_host_bytes(eq, n, batch, h2d, d2h);
  if (eq < 0 || eq > 2 || n < 1 || batch < 0) return fail(LAGEN_EINVAL, "bad arguments");
  long long in = 0;
  const int sp = n <= 128 ? split_row(n) : 0;
  for (int i = 0; i < eq_ninputs(eq); ++i) in += part_doubles_split(input_part(eq, i), n, sp);
  const int xpart = (eq == LAGEN_CHOLESKY && (flags & LAGEN_HOST_X_ZEROED)) ? 1 : 0;
  if (h2d) *h2d = batch * in * (long long)sizeof(double);
  if (d2h) *d2h = batch * (part_doubles_split(xpart, n, sp) * (long long)sizeof(double) + (long long)sizeof(int));
  return LAGEN_OK;
}

int lagen_b200_host_bytes(int eq, int n, long long batch, long long* h2d, long long* d2h) {
  if (eq < 0 || eq > 2 || n < 1 || batch < 0) return fail(LAGEN_EINVAL, "bad arguments");
  const Bands bd = host_bands(eq, n);
  long long per = (long long)n * n;
  if (bd.K > 0) {
    per = 0;
    for (int j = 0; j < bd.K; ++j) per += (long long)(bd.r1[j] - bd.r0[j]) * (n - bd.c0[j]);
  }
  if (h2d) *h2d = batch * per * (long long)sizeof(double) * eq_ninputs(eq);
  if (d2h) *d2h = batch * (per * (long long)sizeof(double) + (long long)sizeof(int));
  return LAGEN_OK;
}

}  // extern "C"
