// fp64-grade products on the int8 tensor cores (tcgen05.mma kind::i8) for the fp32 mode: an
// Ozaki-style split of both operands into OZ_S signed int8 digits.
//
// Reference contractions carried: the Gram densemat.matmul(a, transpose(a)) (ortho.py:156, 198), the
// squarings B_{k+1} = B_k B_k (ortho.py:201-203, run in the C-form C' = 2C - C^2) and the apply
// P(A) . X (ortho.py:205) -- all computed by the reference in numpy float64.
//
// Split (oz_split_kernel): every operand row r (the contraction runs along the row) is scaled by
// 2^-e_r, e_r = the frexp exponent of the row's max |a|, so |a 2^-e_r| < 1, and written as
//   a = 2^e_r * sum_{s=1..S} d_s 2^-(6 + 7(s-1)),   d_1 = rint(64 r), d_{s+1} = rint(128 (r_s - d_s))
// with every |d_s| <= 64 (the remainder after round-to-nearest is within +-1/2).  The product keeps
// the digit pairs with s + t <= S + 1 (S(S+1)/2 int8 GEMMs, exact int32 sums); pairs with the same
// s + t share one TMEM accumulator, so the epilogue combines S accumulators in fp64:
//   (A B^T)_mn = 2^(e_m + e_n - 12) * sum_{g=0..S-1} acc_g(m, n) 2^(-7 g).
// The dropped pairs bound the error at ~2^-(6 + 7S) relative to (row max x column max x K); S = 5
// keeps the whole UNSO pipeline within 1.5e-7 (configs[1]) / 2.6e-7 (configs[4]-like Pareto
// spectrum) of the fp64 oracle (tools/ozaki_emulation.py, an exact emulation of this scheme).
// int32 bound: a group holds <= S products of |d_s d_t| <= 4096, so K <= OZ_MAX_K per split-K slice.
//
// Engine: persistent CTA pairs (cta_group::2), 256 x 96 output tiles per pair (TMEM: S accumulators
// of 96 columns = 480 of 512), K staged 64 bytes at a time: each CTA loads its 128 A rows and 48 of the
// B rows in all S digit planes with one 4-D TMA box each (SWIZZLE_64B), 3 stages; warp 0 TMA (both
// CTAs), warp 1 of the leader MMA (15 products x 2 k-steps per stage, M = 256 per instruction: the
// i8 MMAs are short, so fewer and larger instructions matter -- issue, not the tensor pipe, bounds
// small-N tiles), warp 2 TMEM, warps 4..7 epilogue (drain + fp64 combination, exponents, coalesced
// block functors) in both CTAs.
#pragma once
#include "common.cuh"
#include "ptx_sm100.cuh"
#include "simt_gemm.cuh"

namespace unso {

constexpr int OZ_S = 5;                        // digits per operand
constexpr int OZ_BM = 256, OZ_BN = 96, OZ_BK = 64;   // CTA-pair tile; BK in int8 elements (= bytes)
constexpr int OZ_HB = OZ_BN / 2;               // B rows staged per CTA
constexpr int OZ_STAGES = 3;
constexpr int OZ_A_TILE = 128 * OZ_BK;         // 8 KB per digit plane (the CTA's 128 A rows)
constexpr int OZ_B_TILE = OZ_HB * OZ_BK;       // 3 KB
constexpr int OZ_STAGE_BYTES = OZ_S * (OZ_A_TILE + OZ_B_TILE);  // per CTA
constexpr int OZ_SMEM = OZ_STAGES * OZ_STAGE_BYTES + 1024 + 1024;  // stages, barriers, alignment slack
constexpr uint32_t OZ_TMEM_COLS = 512;         // OZ_S * OZ_BN = 480 used
constexpr int64_t OZ_MAX_K = 65536;            // 5 * 64 * 64 * 65536 < 2^31
static_assert(OZ_S * OZ_BN <= 512, "tmem");
static_assert(OZ_SMEM <= 227 * 1024, "smem");
static_assert(OZ_STAGE_BYTES % 1024 == 0 && OZ_B_TILE % 512 == 0, "swizzle atom alignment");

// kind::i8: s8 x s8 -> s32 (c_format 2, a/b format 1 = signed), K-major operands.
__host__ __device__ constexpr uint32_t idesc_s8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
// Warp-collective forms: every lane of a converged warp executes the asm, one elected lane issues.
// Descriptors computed in warp-uniform control flow then stay in uniform registers (no per-MMA
// R2UR waterfall around a lane-0-only issue, which cost ~80 cycles per instruction here).
__device__ __forceinline__ void umma_s8_pair_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                  uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(const CUtensorMap* m, uint32_t leader_bar, void* smem_dst, int c0,
                                                 int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// Row scale exponent from the row's max |a| (as the u64 bits of a non-negative double): the frexp
// exponent, so |a| 2^-e < 1.  0 for an all-zero row.  Split kernel and epilogue use the same rule.
__device__ __forceinline__ int oz_exponent(unsigned long long maxbits) {
  const double m = __longlong_as_double(static_cast<long long>(maxbits));
  return m > 0.0 ? ilogb(m) + 1 : 0;
}

// ---------------------------------------------------------------- max |a| per operand row
// Per source row (one warp per row): out[b * out_bs + r] = bits of max_c |src[b][r][c]|.
__global__ void oz_rowmax_kernel(const void* __restrict__ src, int dt, int64_t ld, int64_t bs, int64_t rows,
                                 int64_t cols, int batch, unsigned long long* __restrict__ out, int64_t out_bs) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int b = blockIdx.y;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += nw) {
    double m = 0.0;
    bool bad = false;
    for (int64_t c = lane; c < cols; c += 32) {
      const double v = fabs(load_as_f64(src, b * bs + r * ld + c, dt));
      bad |= !(v <= 1.7976931348623157e308);  // NaN or Inf
      m = fmax(m, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      bad |= __shfl_xor_sync(0xffffffffu, bad ? 1 : 0, o) != 0;
    }
    if (lane == 0) out[b * out_bs + r] = static_cast<unsigned long long>(__double_as_longlong(bad ? __longlong_as_double(0x7FF8000000000000ll) : m));
  }
  (void)batch;
}

// Per source column: out[b * out_bs + c] = bits of max_r |src[b][r][c]| (out zeroed beforehand;
// non-negative doubles order like their bit patterns, NaN 0x7FF8.. above every finite value).
__global__ void oz_colmax_kernel(const void* __restrict__ src, int dt, int64_t ld, int64_t bs, int64_t rows,
                                 int64_t cols, unsigned long long* __restrict__ out, int64_t out_bs, int rows_per_block) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int b = blockIdx.z;
  if (c >= cols) return;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
  const int64_t r1 = r0 + rows_per_block < rows ? r0 + rows_per_block : rows;
  double m = 0.0;
  bool bad = false;
  for (int64_t r = r0; r < r1; ++r) {
    const double v = fabs(load_as_f64(src, b * bs + r * ld + c, dt));
    bad |= !(v <= 1.7976931348623157e308);
    m = fmax(m, v);
  }
  const unsigned long long bits =
      bad ? 0x7FF8000000000000ull : static_cast<unsigned long long>(__double_as_longlong(m));
  atomicMax(out + b * out_bs + c, bits);
}

// ---------------------------------------------------------------- digit planes
// dst[s][b][R][ldd] (plane stride `plane`, batch stride `dbs`), operand row R of K entries.
// transpose = 0: operand row = source row (R = rows, K = cols); 1: operand row = source column.
// Scale exponent of operand row R from maxbits[b * max_bs + R].
__device__ __forceinline__ void oz_digits(double v, int e, int8_t (&d)[OZ_S]) {
  double r = ldexp(v, 6 - e);  // 64 * v * 2^-e, |r| < 64
#pragma unroll
  for (int s = 0; s < OZ_S; ++s) {
    const double q = rint(r);
    d[s] = static_cast<int8_t>(static_cast<int>(q));
    r = (r - q) * 128.0;
  }
}

// 64 x 64 source tiles, 256 threads; every thread digitises 4 consecutive operand-row entries and
// writes them as one 4-byte word per digit plane (ldd % 64 == 0; entries past K are written as 0
// digits and never read: the TMA map's K extent ends at K).
__global__ void __launch_bounds__(256) oz_split_kernel(const void* __restrict__ src, int dt, int64_t ld, int64_t bs,
                                                       int64_t rows, int64_t cols, int transpose,
                                                       const unsigned long long* __restrict__ maxbits, int64_t max_bs,
                                                       int8_t* __restrict__ dst, int64_t ldd, int64_t dbs,
                                                       int64_t plane) {
  __shared__ double tile[64][65];
  const int b = blockIdx.z;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 64, c0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int tq = threadIdx.x & 15, tr = threadIdx.x >> 4;  // 16 x 16
  const char* srcb = static_cast<const char*>(src) + b * bs * dtype_size(dt);
  auto emit = [&](int64_t R, int64_t k, const double (&v)[4], int e) {
    uint32_t w[OZ_S];
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) w[s] = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int8_t d[OZ_S];
      oz_digits(v[q], e, d);
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) w[s] |= static_cast<uint32_t>(static_cast<uint8_t>(d[s])) << (8 * q);
    }
    const int64_t o = b * dbs + R * ldd + k;
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint32_t*>(dst + s * plane + o) = w[s];
  };
  if (!transpose) {
    for (int i = tr; i < 64; i += 16) {
      const int64_t r = r0 + i, c = c0 + 4 * tq;
      if (r >= rows || c >= cols) continue;
      const int e = oz_exponent(maxbits[b * max_bs + r]);
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (c + q < cols) ? load_as_f64(srcb, r * ld + c + q, dt) : 0.0;
      emit(r, c, v, e);
    }
  } else {
    for (int i = tr; i < 64; i += 16) {
      const int64_t r = r0 + i;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t c = c0 + 4 * tq + q;
        tile[i][4 * tq + q] = (r < rows && c < cols) ? load_as_f64(srcb, r * ld + c, dt) : 0.0;
      }
    }
    __syncthreads();
    for (int i = tr; i < 64; i += 16) {
      const int64_t R = c0 + i, k = r0 + 4 * tq;  // operand row = source column c0 + i
      if (R >= cols || k >= rows) continue;
      const int e = oz_exponent(maxbits[b * max_bs + R]);
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = tile[4 * tq + q][i];
      emit(R, k, v, e);
    }
  }
}

// One warp per row r of matrix b, the C-form chain bookkeeping fused with the next squaring's split:
//   mode 0 (C_1):     c = G * (1 / s^2),       P  = alpha I - coef c
//   mode 1 (C_{k+1}): c = 2 C_k - S (S = C_k^2), P -= coef c
// writes c to Cn, then (digits != nullptr) the row max and the row's digit planes (re-reading c).
struct OzStepParams {
  const double* src;    // G (mode 0) or C_k (mode 1)
  const double* S;      // mode 1
  double* Cn;
  double* P;
  const double* scal;   // mode 0: per-matrix scalars (S_S2)
  double alpha, coef;
  int mode, h;
  int64_t ld, bs;
  unsigned long long* maxbits;  // [b * h + r]
  int8_t* digits;               // [s][b][r][ld] planes (plane stride `plane`, batch stride bs)
  int64_t plane;
};
__global__ void __launch_bounds__(256) oz_chain_step_kernel(const OzStepParams p) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const double inv_s2 = p.mode == 0 ? 1.0 / p.scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_S2] : 0.0;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < p.h; r += nw) {
    const int64_t o0 = static_cast<int64_t>(b) * p.bs + r * p.ld;  // 16-byte aligned (ld % 256 == 0)
    double m = 0.0;
    bool bad = false;
    for (int c = 2 * lane; c < p.h; c += 64) {  // two entries per lane: 16-byte accesses
      const int64_t o = o0 + c;
      const bool two = c + 1 < p.h;
      double2 cn, pv;
      if (p.mode == 0) {
        const double2 g = two ? *reinterpret_cast<const double2*>(p.src + o) : make_double2(p.src[o], 0.0);
        cn = make_double2(g.x * inv_s2, g.y * inv_s2);
        pv = make_double2((c == r ? p.alpha : 0.0) - p.coef * cn.x, (c + 1 == r ? p.alpha : 0.0) - p.coef * cn.y);
      } else {
        const double2 cc = two ? *reinterpret_cast<const double2*>(p.src + o) : make_double2(p.src[o], 0.0);
        const double2 ss = two ? *reinterpret_cast<const double2*>(p.S + o) : make_double2(p.S[o], 0.0);
        const double2 pp = two ? *reinterpret_cast<const double2*>(p.P + o) : make_double2(p.P[o], 0.0);
        cn = make_double2(2.0 * cc.x - ss.x, 2.0 * cc.y - ss.y);
        pv = make_double2(pp.x - p.coef * cn.x, pp.y - p.coef * cn.y);
      }
      if (two) {
        *reinterpret_cast<double2*>(p.Cn + o) = cn;
        *reinterpret_cast<double2*>(p.P + o) = pv;
      } else {
        p.Cn[o] = cn.x;
        p.P[o] = pv.x;
        cn.y = 0.0;
      }
      const double a0 = fabs(cn.x), a1 = fabs(cn.y);
      bad |= !(a0 <= 1.7976931348623157e308) || !(a1 <= 1.7976931348623157e308);
      m = fmax(m, fmax(a0, a1));
    }
    if (!p.digits) continue;
#pragma unroll
    for (int q = 16; q > 0; q >>= 1) {
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, q));
      bad |= __shfl_xor_sync(0xffffffffu, bad ? 1 : 0, q) != 0;
    }
    const unsigned long long bits =
        bad ? 0x7FF8000000000000ull : static_cast<unsigned long long>(__double_as_longlong(m));
    if (lane == 0) p.maxbits[static_cast<int64_t>(b) * p.h + r] = bits;
    const int e = oz_exponent(bits);
    __syncwarp();
    for (int c = 4 * lane; c < p.h; c += 128) {  // four entries per lane: one 4-byte word per plane
      const int64_t o = o0 + c;
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (c + q < p.h) ? p.Cn[o + q] : 0.0;
      uint32_t w[OZ_S];
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) w[s] = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int8_t d[OZ_S];
        oz_digits(v[q], e, d);
#pragma unroll
        for (int s = 0; s < OZ_S; ++s) w[s] |= static_cast<uint32_t>(static_cast<uint8_t>(d[s])) << (8 * q);
      }
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint32_t*>(p.digits + s * p.plane + o) = w[s];
    }
  }
}

// ---------------------------------------------------------------- GEMM / SYRK on the digits
struct OzWork {
  int tiles_m, tiles_n, syrk, splits, k_tiles, batch, tiles_per_mat, num_work;
  int dbg;  // timing experiments only (developer builds): 1 = skip the MMAs, 2 = skip the TMA loads
};

// SYRK (square): pair tile (tm, tn) is kept when its columns reach the diagonal block's first row,
// tn >= tn_min(tm) = floor(256 tm / 96); the epilogue drops the elements with n < m.
__host__ __device__ __forceinline__ int oz_tn_min(int tm) { return (OZ_BM * tm) / OZ_BN; }
__device__ __forceinline__ void oz_decode(const OzWork& w, int idx, int& b, int& split, int& tm, int& tn, int& kt0,
                                          int& kt1) {
  int t = idx % w.tiles_per_mat;
  const int r = idx / w.tiles_per_mat;
  split = r % w.splits;
  b = r / w.splits;
  if (w.syrk) {
    tm = 0;
    for (;;) {
      const int n = w.tiles_n - oz_tn_min(tm);
      if (t < n) break;
      t -= n;
      ++tm;
    }
    tn = oz_tn_min(tm) + t;
  } else {
    constexpr int G = 8;  // row-block groups: the tiles in flight share ~G A row blocks
    const int per_group = G * w.tiles_n;
    const int g = t / per_group;
    const int q = t - g * per_group;
    const int rows = min(G, w.tiles_m - g * G);
    tn = q / rows;
    tm = g * G + (q - tn * rows);
  }
  kt0 = static_cast<int>(static_cast<int64_t>(split) * w.k_tiles / w.splits);
  kt1 = static_cast<int>(static_cast<int64_t>(split + 1) * w.k_tiles / w.splits);
}

struct OzScales {
  const unsigned long long* a;  // per A row max bits: a[b * a_bs + m]
  int64_t a_bs;
  const unsigned long long* b;  // per B row max bits
  int64_t b_bs;
  int M, N;
};

// 2^k as an exact double for |k| <= 1022 (ldexp beyond: denormal / overflow ranges).
__device__ __forceinline__ double oz_pow2(int k) {
  if (k >= -1022 && k <= 1023) return __longlong_as_double(static_cast<long long>(k + 1023) << 52);
  return ldexp(1.0, k);
}

// Row functors: the calling thread owns output row `row`, columns n0 .. n0 + 31 (v[j] = D(row, n0 + j)).
// Full in-bounds segments go out as 32-byte vector stores (each lane writes whole sectors of its own
// row: no shared-memory transpose -- the epilogue runs one warp per scheduler and its per-element
// instruction count sets the time of short-K tiles); edges and misaligned rows element by element.
// SYRK keeps n >= row.
__device__ __forceinline__ void oz_store_row_f64(double* dst, int row, int n0, const double (&v)[32], int M, int N,
                                                 bool syrk) {
  if (row >= M) return;
  const bool full = n0 + 32 <= N && !(syrk && n0 < row) && (reinterpret_cast<uintptr_t>(dst) & 31) == 0;
  if (full) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      uint32_t w[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v[j + q]));
        w[2 * q] = static_cast<uint32_t>(u);
        w[2 * q + 1] = static_cast<uint32_t>(u >> 32);
      }
      st_global_v8(dst + j, w);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (n0 + j < N && !(syrk && n0 + j < row)) dst[j] = v[j];
  }
}

// Gram split-K partial (fp64), the layout of EpiPartialF64 / finalize_sum_kernel.
struct OzEpiPartial {
  double* part;
  int64_t bs, ld;
  int batch;
  __device__ void rows(int b, int split, int row, int n0, const double (&v)[32], int M, int N, bool syrk) const {
    double* dst = part + (static_cast<int64_t>(split) * batch + b) * bs + static_cast<int64_t>(row) * ld + n0;
    oz_store_row_f64(dst, row, n0, v, M, N, syrk);
  }
};

// Symmetric product S = C C^T (the squaring): the upper row segment, then the mirror -- for a fixed
// column the 32 lanes of the warp hold 32 consecutive rows, so S[n][row] is one coalesced 256-byte
// store per column.  Stores only; oz_chain_step_kernel consumes S row by row.
struct OzEpiSym {
  double* out;
  int64_t ld, bs;
  __device__ void rows(int b, int, int row, int n0, const double (&v)[32], int M, int N, bool syrk) const {
    double* base = out + static_cast<int64_t>(b) * bs;
    oz_store_row_f64(base + static_cast<int64_t>(row) * ld + n0, row, n0, v, M, N, syrk);
    if (row >= M) return;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = n0 + j;
      if (n > row && n < N) base[static_cast<int64_t>(n) * ld + row] = v[j];
    }
  }
};

// NS quintic operator B = bq G + cq G^2 (ortho.py:226-230 regrouped) from the SYRK of G: upper row
// segment and its mirror (B is symmetric; the mirror reuses G(row, n) = G(n, row)).
struct OzEpiQuinticB {
  const double* G;
  double* Bm;
  int64_t ld, bs;
  double bq, cq;
  __device__ void rows(int b, int, int row, int n0, const double (&v)[32], int M, int N, bool syrk) const {
    if (row >= M) return;
    const int64_t base = static_cast<int64_t>(b) * bs;
    const double* g = G + base + static_cast<int64_t>(row) * ld + n0;
    double o[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = (n0 + j < N) ? fma(bq, __ldg(g + j), cq * v[j]) : 0.0;
    oz_store_row_f64(Bm + base + static_cast<int64_t>(row) * ld + n0, row, n0, o, M, N, syrk);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = n0 + j;
      if (n > row && n < N) Bm[base + static_cast<int64_t>(n) * ld + row] = o[j];
    }
  }
};

// NS state update out = alpha * (X B or B X) + beta * old, fp64 state (ortho.py:215-217, 226-230).
struct OzEpiAxpy {
  double* out;
  const double* old;
  int64_t ld, bs;
  double alpha, beta;
  __device__ void rows(int b, int, int row, int n0, const double (&v)[32], int M, int N, bool) const {
    if (row >= M) return;
    const int64_t o = static_cast<int64_t>(b) * bs + static_cast<int64_t>(row) * ld + n0;
    double r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = (n0 + j < N) ? fma(alpha, v[j], beta * __ldg(old + o + j)) : 0.0;
    oz_store_row_f64(out + o, row, n0, r, M, N, false);
  }
};

// Output in the caller's dtype (the apply).
struct OzEpiOut {
  void* out;
  int dt;
  int64_t ld, bs;
  __device__ void rows(int b, int, int row, int n0, const double (&v)[32], int M, int N, bool) const {
    if (row >= M) return;
    const int64_t o = static_cast<int64_t>(b) * bs + static_cast<int64_t>(row) * ld + n0;
    if (dt == DT_F64) {
      oz_store_row_f64(static_cast<double*>(out) + o, row, n0, v, M, N, false);
      return;
    }
    if (dt == DT_F32) {
      float* dst = static_cast<float*>(out) + o;
      if (n0 + 32 <= N && (reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint32_t w[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) w[q] = __float_as_uint(static_cast<float>(v[j + q]));
          st_global_v8(dst + j, w);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (n0 + j < N) dst[j] = static_cast<float>(v[j]);
      }
      return;
    }
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(out) + o;
    if (n0 + 32 <= N && (reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
#pragma unroll
      for (int j = 0; j < 32; j += 16) {
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          w[q] = pack_bf16x2(static_cast<float>(v[j + 2 * q]), static_cast<float>(v[j + 2 * q + 1]));
        st_global_v8(dst + j, w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) dst[j] = __float2bfloat16_rn(static_cast<float>(v[j]));
    }
  }
};

#ifdef UNSO_EXP_TIMING  // timing experiment only (tools/oz_trace.py): per-tile events of pair 0
__device__ unsigned long long g_oz_trace[2][16][8];
__device__ __forceinline__ void oz_trace(int t, int ev) {
  if ((blockIdx.x >> 1) != 0 || t >= 16) return;
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  g_oz_trace[blockIdx.x & 1][t][ev] = v;
}
#define OZ_TRACE(t, ev) oz_trace(t, ev)
#else
#define OZ_TRACE(t, ev)
#endif

constexpr int OZ_THREADS = 128 + 12 * 32;  // 4 role warps + 12 epilogue warps (3 chunks x 4 lane quarters)

template <class Epi>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const OzWork work, const OzScales sc, const Epi epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OZ_STAGES * OZ_STAGE_BYTES);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* tfull = empty + OZ_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) OZ_TRACE(15, 0);
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * 12);  // every epilogue warp of both CTAs
    fence_mbar_init();
  }
  cluster_sync_all();
  if (warp == 2) tmem_alloc_pair(tmem_slot, OZ_TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) OZ_TRACE(15, 1);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t lbar0 = leader_bar_addr(&full[0]);
      int stage = 0;
      uint32_t phase = 0;
      for (int idx = cluster; idx < work.num_work; idx += nclusters) {
        int b, split, tm, tn, kt0, kt1;
        oz_decode(work, idx, b, split, tm, tn, kt0, kt1);
        const int arow = tm * OZ_BM + static_cast<int>(rank) * 128;
        const int brow = tn * OZ_BN + static_cast<int>(rank) * OZ_HB;
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * OZ_STAGE_BYTES;
          if (work.dbg & 2) {
            if (leader) mbar_arrive(&full[stage]);
          } else {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * OZ_STAGE_BYTES);
            const uint32_t lbar = lbar0 + stage * 8;
            tma_load_4d_pair(&tmA, lbar, st, kt * OZ_BK, arow, b, 0);                       // S planes
            tma_load_4d_pair(&tmB, lbar, st + OZ_S * OZ_A_TILE, kt * OZ_BK, brow, b, 0);
          }
          if (++stage == OZ_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      // MMA issuer (leader CTA): the whole warp walks the loop (uniform control flow), one elected
      // lane issues -- descriptors then stay in uniform registers.
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      const uint32_t IDESC = idesc_s8(OZ_BM, OZ_BN);
      const uint64_t D0 = sdesc_sw64(0, 16, 512);  // descriptor of smem address 0: + (addr >> 4) per operand
      for (int idx = cluster; idx < work.num_work; idx += nclusters) {
        int b, split, tm, tn, kt0, kt1;
        oz_decode(work, idx, b, split, tm, tn, kt0, kt1);
        mbar_wait(tempty, acc_phase ^ 1);
        tc_fence_after();
        if (lane == 0) OZ_TRACE((idx - cluster) / nclusters, 2);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if ((work.dbg & 1) == 0) {
            const uint64_t da = D0 + (smem_u32(smem + stage * OZ_STAGE_BYTES) >> 4);
            const uint64_t db = da + ((OZ_S * OZ_A_TILE) >> 4);
#pragma unroll
            for (int ks = 0; ks < OZ_BK / 32; ++ks) {
#pragma unroll
              for (int g = 0; g < OZ_S; ++g) {      // digit pairs (s, t) with s + t = g (0-based)
#pragma unroll
                for (int s = 0; s <= g; ++s) {
                  const int t = g - s;
                  const uint32_t acc = (kt > kt0 || ks > 0 || s > 0) ? 1u : 0u;
                  umma_s8_pair_warp(tmem_base + static_cast<uint32_t>(g * OZ_BN),
                                    da + static_cast<uint64_t>((s * OZ_A_TILE + ks * 32) >> 4),
                                    db + static_cast<uint64_t>((t * OZ_B_TILE + ks * 32) >> 4), IDESC, acc);
                }
              }
            }
          }
          umma_commit_pair_warp(&empty[stage], 0x3);
          if (++stage == OZ_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair_warp(tfull, 0x3);
        if (lane == 0) OZ_TRACE((idx - cluster) / nclusters, 3);
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // Epilogue: 12 warps, one per (TMEM lane quarter, 32-column chunk) -- it runs at one warp per
    // scheduler per chunk set and its per-element instruction count sets the tile time of short-K
    // tiles, so the three chunks run in parallel.  Each warp drains its chunk's S accumulator groups
    // and combines them exactly in int64 (Q = sum_g acc_g 128^(S-1-g), |Q| < 2^60), releases the TMEM
    // (the S x 96 accumulator columns cannot be double-buffered in 512), then rounds Q once to fp64,
    // scales it by the exact powers of two 2^(e_m - 12 - 7(S-1)) (row) and 2^(e_n) (column; NaN marks
    // a non-finite operand row / column) and hands its row segment to the functor.
    const int ew = warp - 4;
    const int q4 = warp & 3;   // TMEM lane quarter this warp may access
    const int c = ew >> 2;     // 32-column chunk of the tile
    uint32_t acc_phase = 0;
    for (int idx = cluster; idx < work.num_work; idx += nclusters) {
      int b, split, tm, tn, kt0, kt1;
      oz_decode(work, idx, b, split, tm, tn, kt0, kt1);
      // the row / column maxima are loaded before waiting for the accumulator: their latency under the
      // operand stream (several µs) then hides behind the tile's MMAs instead of following the drain
      const int row = tm * OZ_BM + static_cast<int>(rank) * 128 + q4 * 32 + lane;
      const int n0 = tn * OZ_BN + c * 32;
      const unsigned long long ma = row < sc.M ? __ldg(sc.a + b * sc.a_bs + row) : 0ull;
      const unsigned long long mb = n0 + lane < sc.N ? __ldg(sc.b + b * sc.b_bs + n0 + lane) : 0ull;
      mbar_wait(tfull, acc_phase);
      acc_phase ^= 1;
      tc_fence_after();
      if (ew == 0 && lane == 0) OZ_TRACE((idx - cluster) / nclusters, 4);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q4 * 32) << 16) + static_cast<uint32_t>(c * 32);
      long long v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0;
#pragma unroll
      for (int g = 0; g < OZ_S; ++g) {
        uint32_t r[32];
        tmem_ld32(taddr + g * OZ_BN, r);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = v[j] * 128 + static_cast<long long>(static_cast<int32_t>(r[j]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty, 0);  // this warp's accumulator columns are in registers
      if (ew == 0 && lane == 0) OZ_TRACE((idx - cluster) / nclusters, 5);
      const bool a_bad = !(__longlong_as_double(static_cast<long long>(ma)) <= 1.7976931348623157e308);
      const double rowscale = a_bad ? __longlong_as_double(0x7FF8000000000000ll)
                                    : oz_pow2(oz_exponent(ma) - 12 - 7 * (OZ_S - 1));
      const double colscale = !(__longlong_as_double(static_cast<long long>(mb)) <= 1.7976931348623157e308)
                                  ? __longlong_as_double(0x7FF8000000000000ll)
                                  : oz_pow2(oz_exponent(mb));
      if (ew == 0 && lane == 0) OZ_TRACE((idx - cluster) / nclusters, 0);
      double d[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) d[j] = __ll2double_rn(v[j]) * rowscale * __shfl_sync(0xffffffffu, colscale, j);
      if (ew == 0 && lane == 0) OZ_TRACE((idx - cluster) / nclusters, 1);
      epi.rows(b, split, row, n0, d, sc.M, sc.N, work.syrk != 0);
      if (ew == 0 && lane == 0) OZ_TRACE((idx - cluster) / nclusters, 6);
    }
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, OZ_TMEM_COLS);
  }
}

}  // namespace unso
