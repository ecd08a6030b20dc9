/*
 * lagen_b200.h — C ABI of the B200 execution backend for the `lagen`
 * blocked-variant solvers (upper Cholesky, triangular Lyapunov, triangular
 * Sylvester) over batches of fixed-size fp64 matrices.
 *
 * Drop-in boundary.  The reference exposes its hot path as
 *
 *   (1) the emitted size-specialised C kernel
 *         void <eq>_v<k>_n<n>_b<b>(const double* <inputs>..., double* X)
 *       /root/reference/pkg/src/lagen/codegen.py:143-201 (signature order from
 *       `_signature`, codegen.py:143-152; name from lowering.py:952), and
 *   (2) the executor  interpret_algorithm(alg, inst, b)
 *       /root/reference/pkg/src/lagen/verify.py:221-303.
 *
 * The batched entry points below replace both: `lagen_b200_<eq>` is (1) with
 * the variant/n/b baked into arguments instead of the symbol name and a batch
 * dimension added; `lagen_b200_execute` is (2) for an arbitrary synthesised
 * statement list.  All matrices are flat row-major, ld = n, and a batch is
 * `batch` contiguous n*n problems (stride n*n doubles).  Inputs follow the
 * reference's `_signature` order (inputs in declaration order, then X).
 *
 * Differences to the reference contract (supersets):
 *   - X need not be zero-initialised: every one of the n*n entries is written
 *     (zeros below the diagonal for Cholesky, the mirror for Lyapunov).
 *   - Errors are reported, not silent: `info[p]` (optional, may be NULL) is
 *     0 on success, i+1 if the Cholesky leaf met a non-positive pivot at
 *     global index i (kernels.py:87-88), and -1 if X holds NaN/Inf
 *     (verify.py:301-302).
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream).  Device pointers unless stated otherwise.
 *   - Return value: LAGEN_OK or a negative LAGEN_E* code; no C++ exception
 *     crosses the ABI; lagen_b200_last_error() gives a thread-local message.
 */
#ifndef LAGEN_B200_H
#define LAGEN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAGEN_B200_ABI_VERSION 1
#define LAGEN_MAX_STMTS 16
/* Sizes: 1 <= n <= 128 run on the size-specialised shared-memory engines;
 * 128 < n <= LAGEN_BIG_MAX_N (b | n) run on the "big" engine (bigsolve.cu: the
 * statement-list interpreter with X resident in its HBM output buffer, one
 * problem per CTA) — the reference's interpreter has no size limit
 * (verify.py:221-303), its generator stops at 128 (lowering.py:930-932). */
#define LAGEN_BIG_MAX_N 1024

/* equations (the three shipped cases, /root/reference/pkg/cases/ *.la) */
enum {
  LAGEN_CHOLESKY = 0,  /* X^T X = A,        inputs (A)       */
  LAGEN_LYAPUNOV = 1,  /* L X + X L^T = S,  inputs (L, S)    */
  LAGEN_SYLVESTER = 2  /* L X + X U = C,    inputs (L, U, C) */
};

/* statement kinds (worksheet.py:47-67, dispatch at verify.py:263-295) */
enum {
  LAGEN_GEMM_UPDATE = 0,
  LAGEN_CHOL = 1,
  LAGEN_TRSM_LEFT_TRANSPOSED = 2,
  LAGEN_SYLV = 3,
  LAGEN_LYAP = 4
};

/* operand codes inside a statement: 0 = the unknown's storage X, then the
 * coefficient operands in declaration order (L = 1, U = 2); -1 = unused. */
typedef struct lagen_view {
  int8_t op, r, c, trans;  /* 3x3 repartition block (r, c) of `op`, maybe ^T (worksheet.py:29-44) */
} lagen_view;

typedef struct lagen_stmt {
  int8_t kind;             /* LAGEN_GEMM_UPDATE ... */
  int8_t sign;             /* +1 / -1 (GEMM_update sign) */
  lagen_view out;          /* written in place, never transposed */
  lagen_view in[2];        /* read views (coefficients / factors) */
} lagen_stmt;

/* status codes */
#define LAGEN_OK 0
#define LAGEN_EINVAL (-1)       /* null pointer, negative batch, bad equation */
#define LAGEN_EUNSUPPORTED (-2) /* (n, b) has no sm_100a instantiation or b does not divide n */
#define LAGEN_EVARIANT (-3)     /* statement list malformed / unknown variant index */
#define LAGEN_ECUDA (-4)        /* CUDA runtime error (launch, copy, allocation) */

int lagen_b200_abi_version(void);
const char* lagen_b200_last_error(void);

/* ---- variant table (enumerate_algorithms() output, worksheet.py:281) ---- */
int lagen_b200_num_variants(int eq);
/* copies the statement list of `variant` into out[0..cap); returns the count or <0 */
int lagen_b200_variant_stmts(int eq, int variant, lagen_stmt* out, int cap);
/* 1 if a kernel is instantiated for (eq, n, b), else 0 */
int lagen_b200_supported(int eq, int n, int b);
/* launch geometry chosen for (eq, n, b): threads per problem, problems per CTA,
 * threads per CTA, dynamic shared memory bytes; returns 0 or <0 */
int lagen_b200_geometry(int eq, int n, int b, int* threads_per_problem,
                        int* problems_per_cta, int* threads_per_cta, int* smem_bytes);

/* ---- batched solvers: the emitted kernel <eq>_v<k>_n<n>_b<b> of codegen.py:155-201 ---- */
int lagen_b200_cholesky(int variant, int n, int b, long long batch,
                        const double* A, double* X, int* info, void* stream);
int lagen_b200_lyapunov(int variant, int n, int b, long long batch,
                        const double* L, const double* S, double* X, int* info,
                        void* stream);
int lagen_b200_sylvester(int variant, int n, int b, long long batch,
                         const double* L, const double* U, const double* C,
                         double* X, int* info, void* stream);

/* ---- generic executor: interpret_algorithm(alg, inst, b), verify.py:221 ----
 * inputs[] in _signature order: chol {A}, lyap {L, S}, sylv {L, U, C}.
 * Any 1 <= n <= 128 with b dividing n (the reference's own condition,
 * verify.py:232-233): (n, b) without a compiled instance (n not a multiple of
 * 4, or e.g. b = 1) runs as the identity-padded problem of the next multiple
 * of 4 with that size's block size (exact: diag(A, I) -> diag(X, I); zero
 * right-hand-side rows / columns -> zero X rows / columns), through a
 * stream-ordered scratch allocation of (#inputs + 1) padded batches. */
int lagen_b200_execute(int eq, const lagen_stmt* stmts, int nstmts, int n, int b,
                       long long batch, const double* const* inputs, double* X,
                       int* info, void* stream);

/* Engine selection: LAGEN_ENGINE_AUTO picks, for a statement
 * list equal to a built-in variant, the "rows engine" (Cholesky v1, n > 32),
 * the register-resident "column engine" (Cholesky v1/v2, n <= 64) or the
 * compiled-in "warp engine" when they have an instance for (n, b); otherwise
 * the generic statement-list kernel.  The Python layer passes the engine of
 * the GPU-measured dispatch table explicitly. */
#define LAGEN_ENGINE_AUTO 0
#define LAGEN_ENGINE_GENERIC 1
#define LAGEN_ENGINE_WARP 2
#define LAGEN_ENGINE_COLUMN 3
/* 4x4-tile task DAG (right-looking variants, b <= 8): tasks of successive
 * iterations overlap as soon as their input tiles are final */
#define LAGEN_ENGINE_DATAFLOW 4
/* Cholesky v1 on a packed row-major upper layout (cheap DMMA operand
 * addressing for the block-row updates) */
#define LAGEN_ENGINE_ROWS 5
/* Lyapunov v5 / Sylvester v13: 8x8-tile anti-diagonal wavefront, DMMA
 * tile updates with register-resident accumulators (wave.cuh) */
#define LAGEN_ENGINE_WAVE 6
/* Cholesky v1: the rows engine's b = 8 kernel of a larger size on the
 * identity-padded problem (n = 4 mod 8 -> n + 4; 104 -> 112; 120 -> 128;
 * only the real n x n entries move) */
#define LAGEN_ENGINE_ROWS_PAD 7
/* Lyapunov v5 / Sylvester v13 order at 8x8-tile granularity: dedicated
 * solver warps solve anti-diagonal d while updater warps apply diagonal
 * d-1's DMMA tile updates (pipe.cuh) */
#define LAGEN_ENGINE_PIPE 8
/* Lyapunov / Sylvester at b = n, n <= 32 (the SYLV / LYAP leaf on the whole
 * matrix, kernels.py:100-130): one lane per row, column-by-column forward
 * substitution with the X U part lane-local (rowsweep.cuh); any variant */
#define LAGEN_ENGINE_ROWSWEEP 9
/* Cholesky v1, n = 4 mod 8 (requested as b = 4): the rows engine's b = 8
 * schedule after a first 4 x 4 block row — v1's statements over the
 * partition 4, 8, 8, ..., 8, unpadded (chol_rows.cuh, F4) */
#define LAGEN_ENGINE_ROWS_MIX 10
int lagen_b200_execute_engine(int eq, const lagen_stmt* stmts, int nstmts, int n, int b,
                              long long batch, const double* const* inputs, double* X,
                              int* info, void* stream, int engine);
/* Same as lagen_b200_execute_engine; for warp-engine launches, d_prof (device,
 * >= 32 zeroed uint64) receives cycle counts per phase / schedule level of
 * one problem group (tools/phase_profile.py).  Profiling aid only. */
int lagen_b200_execute_profile(int eq, const lagen_stmt* stmts, int nstmts, int n, int b,
                               long long batch, const double* const* inputs, double* X,
                               int* info, void* stream, int engine, unsigned long long* d_prof);
/* 1 if the warp engine has an instance for (eq, n, b, built-in variant) */
int lagen_b200_warp_supported(int eq, int n, int b, int variant);
/* 1 if `engine` has an instance for (eq, n, b, built-in variant) */
int lagen_b200_engine_supported(int eq, int n, int b, int variant, int engine);

/* Same, but every buffer is in HOST memory (pinned for full overlap).  The
 * batch is streamed through the device in chunks, H2D copy / solve / D2H copy
 * pipelined over four streams with persistent staging buffers (PCIe
 * bidirectional-bound); synchronous on return. */
int lagen_b200_execute_host(int eq, const lagen_stmt* stmts, int nstmts, int n, int b,
                            long long batch, const double* const* h_inputs,
                            double* h_X, int* h_info);
/* Same with an explicit engine (LAGEN_ENGINE_*), so the host path runs the
 * kernel the device path's dispatch picked (bit-identical results). */
int lagen_b200_execute_host_engine(int eq, const lagen_stmt* stmts, int nstmts, int n, int b,
                                   long long batch, const double* const* h_inputs,
                                   double* h_X, int* h_info, int engine);

/* Same with flags:
 *   LAGEN_HOST_TRIANGLES: move only the structurally needed part of every
 *     operand over PCIe (A / S / U's upper and L's lower triangles, rows
 *     rounded to 8-column tiles; X back the same way).  From n = 16 on the
 *     copy engines move the contiguous mostly-needed half of the rows (one
 *     strided copy per chunk) and zero-copy kernels, reading / writing the
 *     mapped pinned host memory directly, only the remaining small triangle.
 *     Needs pinned (cudaHostAlloc / cudaHostRegister-mapped) buffers and an
 *     even n.
 *   LAGEN_HOST_X_ZEROED: the caller's X already holds zeros in its
 *     structurally-zero part (the reference's contract: "outputs must be
 *     zero-initialised by the caller", codegen.py:4-7); Cholesky then writes
 *     only X's upper triangle.
 *   LAGEN_HOST_ASYNC: return once the call's copies and launches are
 *     queued; results (X, info) are valid after lagen_b200_host_sync().
 *     Consecutive calls keep feeding the same four pipeline streams, so a
 *     sequence of batches (e.g. a sweep over sizes) pays the pipeline's fill
 *     and drain once instead of once per call.  The caller must keep every
 *     host buffer alive and untouched until the sync; errors of queued work
 *     are reported by the sync. */
#define LAGEN_HOST_TRIANGLES 1
#define LAGEN_HOST_X_ZEROED 2
#define LAGEN_HOST_ASYNC 4
/* Wait for all queued host-pipeline work of the current device. */
int lagen_b200_host_sync(void);
int lagen_b200_execute_host_flags(int eq, const lagen_stmt* stmts, int nstmts, int n, int b,
                                  long long batch, const double* const* h_inputs,
                                  double* h_X, int* h_info, int engine, int flags);
int lagen_b200_host_bytes_flags(int eq, int n, long long batch, int flags, long long* h2d, long long* d2h);

/* Bytes the host pipeline moves per call (H2D of all inputs, D2H of X and
 * info).  With LAGEN_HOST_BANDS=1 (opt-in, measured not faster) Cholesky
 * n >= 32 copies only row bands of the upper triangle and zero-fills the rest
 * of X's lower triangle on host threads. */
int lagen_b200_host_bytes(int eq, int n, long long batch, long long* h2d, long long* d2h);

/* ---- seeded batched generator (BASELINE.json configs) ----
 * Writes problems [first, first + batch) of the seeded stream into outputs[]
 * (device, _signature order).  Problem p depends only on (eq, n, seed, p), so
 * any sharding of the index range sees identical problems. */
int lagen_b200_generate(int eq, int n, unsigned long long seed, long long first,
                        long long batch, double* const* outputs, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LAGEN_B200_H */
