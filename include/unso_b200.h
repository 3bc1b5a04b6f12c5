/*
 * unso_b200.h -- C ABI of the B200-native UNSO orthogonalization hot path.
 *
 * The reference (arXiv 2602.02500, /root/reference/pkg/src/unso) is a pure
 * Python/numpy package with no FFI; its drop-in boundary is the Python API of
 * `unso.ortho` (re-exported in unso/__init__.py:31-42).  Each entry point below
 * replaces one reference function; the Python host package
 * `paper_2602_02500_b200` binds them with ctypes.
 *
 * Conventions
 *   - Plain pointers and sizes; every call is stream-ordered on `stream`
 *     (a cudaStream_t passed as void*), never synchronises the host, never throws.
 *   - The caller owns all memory (inputs, outputs, workspace; device memory).
 *   - Matrices are strided batches of row-major rows x cols matrices.
 *   - Host-detectable errors are returned as unso_status; data-dependent
 *     errors (zero input / non-finite scale, ortho.py:147-148,164-165) are
 *     written per matrix to the device int32 array `d_status` (may be NULL).
 */
#ifndef UNSO_B200_H
#define UNSO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum unso_status {
  UNSO_OK = 0,
  UNSO_ERR_SHAPE = 1,        /* ShapeError            (errors.py:4-5)          */
  UNSO_ERR_DEGENERATE = 2,   /* DegenerateInputError  (errors.py:12-13)        */
  UNSO_ERR_VALUE = 3,        /* ValueError            (ortho.py:85-110)        */
  UNSO_ERR_CUDA = 4,         /* CUDA launch / driver failure                    */
  UNSO_ERR_UNSUPPORTED = 5,  /* valid request this build does not implement     */
  UNSO_ERR_WORKSPACE = 6     /* workspace smaller than unso_workspace_size()    */
} unso_status;

typedef enum unso_dtype { UNSO_DTYPE_F32 = 0, UNSO_DTYPE_BF16 = 1, UNSO_DTYPE_F64 = 2 } unso_dtype;

/* Arithmetic recipe.
 *   FP32: fp32 I/O, fp64-grade Gram + squaring chain (fp64 tensor cores, DMMA), fp64-accumulated apply;
 *         parity <= 1e-5 against the fp64 reference on every config.
 *   BF16: tcgen05 tensor cores, bf16 operands / f32 accumulation; the h x h chain in
 *         C-form with bf16x3 split products, the apply with a bf16x2 split P;
 *         parity <= 2e-2 against the reference fed the same bf16-rounded input. */
typedef enum unso_precision { UNSO_PREC_FP32 = 0, UNSO_PREC_BF16 = 1 } unso_precision;

/* Scaling (ortho.py:54-57): gram = A/||AA^T||_F^(1/2), plain = A/||A||_F, gelfand. */
typedef enum unso_scaling {
  UNSO_SCALING_GRAM = 0,
  UNSO_SCALING_PLAIN = 1,
  UNSO_SCALING_GELFAND = 2,
  UNSO_SCALING_NONE = 3 /* input already scaled: the bare kernels unso()/muon_ns()/... (ortho.py:171-256) */
} unso_scaling;

/* Kernel families (ortho.py:60-65): UNSO, original cubic NS, and the quintic
 * step family (muon / cesista / external differ only in their (a,b,c) rows). */
typedef enum unso_method { UNSO_METHOD_UNSO = 0, UNSO_METHOD_ORIGINAL_NS = 1, UNSO_METHOD_QUINTIC = 2 } unso_method;

/* flags */
#define UNSO_FLAG_SINGLE_TERM_APPLY 0x1 /* BF16: always apply with one bf16 term of P (faster, less accurate) */
#define UNSO_FLAG_CHAIN_BF16X3 0x4       /* BF16, large h: keep all squarings in bf16x3 (hi*hi + hi*lo + lo*hi)
                                           instead of the default hi*hi (bf16) + e4m3 cross terms */
#define UNSO_FLAG_TWO_TERM_APPLY 0x2    /* BF16: always apply with the bf16x2 (hi + lo) split of P.
                                           Default (neither flag): per matrix, the lo term is dropped on the
                                           device when ||X dR||_F / ||Y||_F <= 2^-9 ||R||_F / sqrt(tr C_1) <= 5e-3
                                           (R = P - d I, d = tr(P)/h; d X is added exactly in the epilogue). */

#define UNSO_FLAG_NS_SINGLE_STATE 0x10 /* NS/Muon, BF16: round the fp32 state to one bf16 term in its
                                          long-side products (1 + 2 instead of 3 + 3 bf16 products per
                                          step; ~1e-2 instead of ~1e-4 from the fp64 result). */
#define UNSO_FLAG_FP32_DMMA 0x20        /* UNSO, FP32, h > 256: run the Gram, the squarings and the apply on the
                                           fp64 DMMA engine instead of the default int8 tensor-core split
                                           (5 int8 digits per operand, 15 exact int8 products per contraction,
                                           fp64 combination; ~1e-7 from the fp64 reference). */
#define UNSO_FLAG_NO_TRUNCATION 0x8     /* UNSO, BF16: run all N-1 squarings.  Default: the persistent chain
                                           (h <= ~1900 per co-resident batch) stops before step k once every
                                           matrix has sum_{j>k}|c_j| * ||I - C_k||_F^2 <= 2^-12 and subtracts
                                           sum_{j>k} c_j * I (the remaining C_j are I to that bound; with
                                           ||X||_2 <= 1 the relative change of Y is at most that bound). */

typedef struct unso_matrix_desc {
  int64_t rows, cols;    /* per matrix, as given (orientation is chosen internally, ortho.py:149-150) */
  int64_t ld;            /* leading dimension in elements, >= cols */
  int64_t batch;         /* number of matrices, >= 1 */
  int64_t batch_stride;  /* elements between consecutive matrices */
  int32_t dtype;         /* unso_dtype of the input and of the output */
  int32_t orientation;   /* 0: auto, long side = rows iff rows > cols (ortho.py:149-150);
                            1: rows are the long side (a row shard of a tall matrix); 2: cols are */
} unso_matrix_desc;

typedef struct unso_method_desc {
  int32_t method;        /* unso_method */
  int32_t scaling;       /* unso_scaling (already resolved: UNSO -> gram, NS -> plain, ortho.py:112-118) */
  int32_t gelfand_power; /* >= 1 (ortho.py:78,85-86) */
  int32_t precision;     /* unso_precision */
  int32_t order;         /* UNSO: N (number of polynomial terms, scalarpoly.py:39-61) */
  int32_t steps;         /* ORIGINAL_NS: iterations; QUINTIC: number of (a,b,c) rows */
  const double* coeffs;  /* host memory. UNSO: N values a_1..a_{N-1}, b (b = derive_b, scalarpoly.py:117-127);
                            QUINTIC: 3*steps values, row-major (a,b,c) (ortho.py:221-231); ORIGINAL: unused */
  int32_t flags;         /* UNSO_FLAG_* */
  int32_t reserved;
} unso_method_desc;

/* Library identity. */
const char* unso_version(void);
const char* unso_status_string(int32_t status);

/* Bytes of device workspace `unso_orthogonalize` / `unso_orthogonalize_from_gram` /
 * `unso_gram` / `unso_ortho_error` need for this problem (0 on invalid input). */
size_t unso_workspace_size(const unso_matrix_desc* x, const unso_method_desc* method);

/* Y = orthogonalize(X): preprocess -> kernel -> restore orientation.
 * Replaces unso.ortho.orthogonalize (ortho.py:267-283) together with
 * preprocess (ortho.py:140-168) and unso / original_ns / _quintic_steps
 * (ortho.py:171-231).  y has x's shape and dtype, contiguous (ld = cols). */
int32_t unso_orthogonalize(const unso_matrix_desc* x, const void* x_ptr, void* y_ptr,
                           const unso_method_desc* method, void* workspace, size_t workspace_bytes,
                           int32_t* d_status, void* stream);

/* Row-sharded path, stage 1: the un-normalised short-side Gram of the local rows
 * (ortho.py:156, 198 without the 1/denom).  g_ptr: batch x h x h, element type
 * unso_gram_dtype(method) (f64 for FP32 precision, f32 for BF16).  The caller sums
 * it over ranks (one all-reduce) before stage 2.  UNSO method only. */
int32_t unso_gram(const unso_matrix_desc* x, const void* x_ptr, void* g_ptr, const unso_method_desc* method,
                  void* workspace, size_t workspace_bytes, void* stream);
int32_t unso_gram_dtype(const unso_method_desc* method);

/* Row-sharded path, stage 2: given the (globally reduced) Gram, scale, form P
 * with the squaring chain (ortho.py:197-204) and apply it to the local rows
 * (ortho.py:205).  Every rank forms the same P redundantly. */
int32_t unso_orthogonalize_from_gram(const unso_matrix_desc* x, const void* x_ptr, const void* g_ptr, void* y_ptr,
                                     const unso_method_desc* method, void* workspace, size_t workspace_bytes,
                                     int32_t* d_status, void* stream);

/* Row-sharded path with the Gram reduction over NVLink peer memory instead of an all-reduce
 * (BF16 precision, one matrix).  Every rank owns three peer-mapped buffers (e.g.
 * torch symmetric memory) whose device addresses on every rank are listed here:
 *   slots  unso_gram_peer_bytes(h, world, splits, 0) bytes: partial Gram tiles pushed to their owner,
 *   g      unso_gram_peer_bytes(h, world, splits, 1) bytes: the reduced dense h x h fp32 Gram,
 *   flags  unso_gram_peer_bytes(h, world, splits, 2) bytes: zero-initialised once, then never reset
 *          (`epoch` must increase by one per call).
 * Per call and rank, in stream order: unso_gram_push (local Gram on the CTA pairs, partial tiles
 * stored straight into the owners' slots, then "pushed" published), unso_gram_reduce (wait for all
 * ranks' pushes, sum the owned tiles in a fixed order, write them into every rank's g, publish),
 * unso_gram_wait (wait until every rank delivered); g then holds the same reduced Gram on every
 * rank and feeds unso_orthogonalize_from_gram.  The three calls are separate so that one GPU can
 * emulate all ranks phase by phase.  `splits` (split-K slices, >= 1, <= local rows / 64) must be
 * equal on every rank. */
#define UNSO_MAX_PEERS 8
typedef struct unso_gram_peers {
  void* slots[UNSO_MAX_PEERS];
  void* g[UNSO_MAX_PEERS];
  uint32_t* flags[UNSO_MAX_PEERS];
} unso_gram_peers;
size_t unso_gram_peer_bytes(int64_t h, int32_t world, int32_t splits, int32_t which);
int32_t unso_gram_push(const unso_matrix_desc* x_local, const void* x_ptr, const unso_method_desc* method,
                       const unso_gram_peers* peers, int32_t rank, int32_t world, int32_t splits, uint32_t epoch,
                       void* workspace, size_t workspace_bytes, void* stream);
int32_t unso_gram_reduce(int64_t h, const unso_gram_peers* peers, int32_t rank, int32_t world, int32_t splits,
                         uint32_t epoch, void* workspace, size_t workspace_bytes, void* stream);
int32_t unso_gram_wait(int64_t h, const unso_gram_peers* peers, int32_t rank, int32_t world, uint32_t epoch,
                       void* stream);

/* The preprocess denominator alone (ortho.py:140-168): d_denom[b] = ||A A^T||_F^(1/2) (gram),
 * ||A||_F (plain) or ||(A A^T)^k||_F^(1/2k) (gelfand), fp64 accumulation; d_status[b] = 2 when the
 * input is zero or the denominator is not positive and finite. Only scaling/gelfand_power are read. */
int32_t unso_scale_denominator(const unso_matrix_desc* x, const void* x_ptr, const unso_method_desc* method,
                               double* d_denom, void* workspace, size_t workspace_bytes, int32_t* d_status,
                               void* stream);

/* ||Y Y^T - I||_F on the short side (bench.py:71-82), fp64 accumulation;
 * writes `batch` doubles to device memory d_err. */
int32_t unso_ortho_error(const unso_matrix_desc* y, const void* y_ptr, double* d_err, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Copy the per-matrix scalars the last call on this workspace produced into device memory
 * d_out (batch x UNSO_SCALARS doubles): [0] trace(G), [1] ||G||_F^2, [2] ||G - I||_F^2, [3] s^2,
 * [4] 1/s, [5] ortho error, [6] d/s identity shift, [7] apply mode (1 = P_lo term skipped),
 * [8] the adaptive bound.  Same descriptors as the call. */
#define UNSO_SCALARS 16
int32_t unso_query_scalars(const unso_matrix_desc* x, const unso_method_desc* method, const void* workspace,
                           double* d_out, void* stream);

/* Elementwise passes of a Muon optimizer step around the orthogonalizer (no
 * reference interface: the reference lists the optimizer as out of scope).  One shape
 * group of n matrices, `numel` elements each, all of `dtype` (F32 or BF16); d_grads / d_bufs /
 * d_params are DEVICE arrays of n <= 65535 pointers, every pointer 16-byte aligned, numel a multiple of 8.
 *   prepare: M_i <- mu M_i + G_i; U_i = G_i + mu M_i (nesterov) or M_i written to stacked + i*numel;
 *            d_maxabs[i] = max |U_i| (n floats, zeroed by the call).
 *   update:  P_i <- decay P_i + alpha O_i, O = ortho + i*numel, skipped (P_i <- decay P_i) when
 *            d_maxabs[i] == 0 (a zero update is a zero step). */
int32_t unso_muon_prepare(int32_t n, const void* d_grads, const void* d_bufs, void* stacked, int64_t numel,
                          int32_t dtype, float mu, int32_t nesterov, float* d_maxabs, void* stream);
int32_t unso_muon_update(int32_t n, const void* d_params, const void* ortho, int64_t numel, int32_t dtype,
                         const float* d_maxabs, float decay, float alpha, void* stream);

/* Number of CUDA kernels launched by the last successful call on this thread. */
int32_t unso_last_launch_count(void);

/* Stage profiling of unso_orthogonalize (UNSO method) with CUDA events recorded on
 * the call's stream at stage boundaries, so a caller can attribute a timed region to
 * kernels without extra syncs.  Stages (UNSO_PROFILE_STAGES):
 *   0 convert (X -> bf16 copy), 1 gram (K1 SYRK), 2 scale+prep (finalize, norms, C_1, P),
 *   3 chain (K2, N-1 launches), 4 finalize P, 5 apply (K3).
 * begin() arms up to max_calls calls (process-wide, not thread-safe); read() synchronises
 * the recorded events and writes max_calls x UNSO_PROFILE_STAGES milliseconds, returning
 * the number of calls recorded; end() releases the events. */
#define UNSO_PROFILE_STAGES 6
int32_t unso_profile_begin(int32_t max_calls);
int32_t unso_profile_read(float* out_ms, int32_t max_calls);
void unso_profile_end(void);

#ifdef __cplusplus
}
#endif

#endif /* UNSO_B200_H */
