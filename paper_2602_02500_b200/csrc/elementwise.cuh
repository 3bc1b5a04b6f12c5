// HBM-bound helper kernels around the contractions: dtype conversion, split-K
// finalize (+ symmetric mirror), Gram norm reductions, per-matrix scalars,
// the C-form chain prologue (C_1 = G/s^2, P = alpha I - a_1 C_1) and the
// symmetric P finalisation (scale by 1/s, split for the apply).
#pragma once
#include "common.cuh"

namespace unso {

constexpr int NORM_BLOCKS = 1024;  // max per-matrix partial-reduction blocks (workspace slots)
// Partial-reduction blocks for a matrix of `elems` elements: ~16K elements per block, at most
// NORM_BLOCKS; a pure function of the shape, so the partials (and their fixed-order sum) are
// deterministic.  The producing kernel's grid.x and the scalars_kernel's nblk must both use it.
inline int norm_blocks(int64_t elems) {
  const int64_t n = (elems + 16383) / 16384;
  return static_cast<int>(n < 1 ? 1 : (n > NORM_BLOCKS ? NORM_BLOCKS : n));
}

// scal[b * SCAL_STRIDE + ...]
// S_SHIFT: d/s, the identity shift removed from P before the bf16 split (added back as d/s * X in the
// apply epilogue); S_MODE: 1 = the apply may skip the P_lo term (adaptive bound met); S_BOUND: that bound;
// S_STEPS: squarings the persistent chain executed (< N-1 after truncation), -1 on other routes.
enum ScalSlot : int {
  S_TRACE = 0, S_FRO2 = 1, S_DEV2 = 2, S_S2 = 3, S_INV_S = 4, S_ERR = 5, S_SHIFT = 6, S_MODE = 7, S_BOUND = 8,
  S_STEPS = 9
};
constexpr int SCAL_STRIDE = 16;

// ------------------------------------------------------------------ conversion
// dst[b](r, c) = src[b](r, c) * (scal ? scal[b].inv_s : 1), any dtype -> any dtype.
// One warp per row (grid-stride over batch x rows), lanes along the columns: one 64-bit division per
// row instead of three per element.
__global__ void convert_kernel(const void* __restrict__ src, int sdt, int64_t sld, int64_t sbs, void* __restrict__ dst,
                               int ddt, int64_t dld, int64_t dbs, int64_t rows, int64_t cols, int batch,
                               const double* __restrict__ scal) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t nrows = rows * batch;
  for (int64_t R = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); R < nrows;
       R += nwarps) {
    const int64_t b = R / rows, r = R - b * rows;
    const double sc = scal ? scal[b * SCAL_STRIDE + S_INV_S] : 1.0;
    const int64_t so = b * sbs + r * sld, d0 = b * dbs + r * dld;
    for (int64_t c = lane; c < cols; c += 32) store_from_f64(dst, d0 + c, ddt, load_as_f64(src, so + c, sdt) * sc);
  }
}

// fast path: f32 -> bf16 (row-contiguous source), 4 elements per thread
__global__ void f32_to_bf16_kernel(const float* __restrict__ src, int64_t sld, int64_t sbs,
                                   __nv_bfloat16* __restrict__ dst, int64_t dld, int64_t dbs, int64_t rows,
                                   int64_t cols, int batch) {
  const int64_t cq = cols / 4;
  const int64_t per = rows * cq;
  const int64_t total = per * batch;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / per, rc = i - b * per, r = rc / cq, c = (rc - r * cq) * 4;
    const float4 v = *reinterpret_cast<const float4*>(src + b * sbs + r * sld + c);
    __nv_bfloat162 lo2 = __floats2bfloat162_rn(v.x, v.y);
    __nv_bfloat162 hi2 = __floats2bfloat162_rn(v.z, v.w);
    __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(dst + b * dbs + r * dld + c);
    d[0] = lo2;
    d[1] = hi2;
  }
}

// contiguous f32 -> bf16: 8 elements per thread per iteration, no index arithmetic beyond the stride
__global__ void f32_to_bf16_flat_kernel(const float4* __restrict__ src, uint4* __restrict__ dst, int64_t n8) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 a = __ldcs(src + 2 * i), b = __ldcs(src + 2 * i + 1);
    uint4 o;
    o.x = pack_bf16x2(a.x, a.y);
    o.y = pack_bf16x2(a.z, a.w);
    o.z = pack_bf16x2(b.x, b.y);
    o.w = pack_bf16x2(b.z, b.w);
    dst[i] = o;
  }
}

// ------------------------------------------------------------------ symmetric tiles
// 32x32 upper tiles (ti <= tj) of a batch of h x h matrices; the load functor
// produces tile values, the store functor writes (r, c) in both triangles.
__device__ __forceinline__ void sym_tile_coords(int t, int nt, int& ti, int& tj) {
  int row = 0, len = nt;
  while (t >= len) {
    t -= len;
    ++row;
    --len;
  }
  ti = row;
  tj = row + t;
}

// G[b] = sum_s part[s][b]  (upper values mirrored into the lower triangle); G has its own leading
// dimension / batch stride (the padded workspace layout, or a dense caller buffer).
template <typename T>
__global__ void finalize_sum_kernel(const T* __restrict__ part, int splits, int batch, int h, int64_t ld,
                                    T* __restrict__ G, int64_t gld, int64_t gbs) {
  __shared__ double tile[32][33];
  const int nt = (h + 31) / 32;
  int ti, tj;
  sym_tile_coords(blockIdx.x, nt, ti, tj);
  const int b = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t mat = static_cast<int64_t>(h) * ld;
  for (int r = ty; r < 32; r += 8) {
    const int gr = ti * 32 + r, gc = tj * 32 + tx;
    double s = 0.0;
    if (gr < h && gc < h) {
      for (int sp = 0; sp < splits; ++sp)
        s += static_cast<double>(part[(static_cast<int64_t>(sp) * batch + b) * mat + static_cast<int64_t>(gr) * ld + gc]);
    }
    tile[r][tx] = s;
  }
  __syncthreads();
  T* g = G + static_cast<int64_t>(b) * gbs;
  for (int r = ty; r < 32; r += 8) {
    const int gr = ti * 32 + r, gc = tj * 32 + tx;
    if (gr < h && gc < h) g[static_cast<int64_t>(gr) * gld + gc] = static_cast<T>((ti == tj && r > tx) ? tile[tx][r] : tile[r][tx]);
    if (ti != tj) {
      const int mr = tj * 32 + r, mc = ti * 32 + tx;
      if (mr < h && mc < h) g[static_cast<int64_t>(mr) * gld + mc] = static_cast<T>(tile[tx][r]);
    }
  }
}

// Per-block partial sums over a full symmetric h x h matrix: trace, ||G||_F^2, ||G - I||_F^2.
template <typename T>
__global__ void gram_norms_kernel(const T* __restrict__ G, int h, int64_t ld, double* __restrict__ blk) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const T* g = G + static_cast<int64_t>(b) * h * ld;
  double tr = 0.0, fr = 0.0, dv = 0.0;
  // rows strided over the blocks, columns over the threads: no 64-bit division per element (the
  // flat-index form spent most of its time in the emulated int64 divide)
  for (int r = blockIdx.x; r < h; r += gridDim.x) {
    const T* gr = g + static_cast<int64_t>(r) * ld;
    for (int c = threadIdx.x; c < h; c += blockDim.x) {
      const double v = static_cast<double>(gr[c]);
      const double d = (r == c) ? v - 1.0 : v;
      if (r == c) tr += v;
      fr += v * v;
      dv += d * d;
    }
  }
  tr = block_sum(tr, scratch);
  if (threadIdx.x == 0) blk[(static_cast<int64_t>(b) * gridDim.x + blockIdx.x) * 3 + 0] = tr;
  fr = block_sum(fr, scratch);
  if (threadIdx.x == 0) blk[(static_cast<int64_t>(b) * gridDim.x + blockIdx.x) * 3 + 1] = fr;
  dv = block_sum(dv, scratch);
  if (threadIdx.x == 0) blk[(static_cast<int64_t>(b) * gridDim.x + blockIdx.x) * 3 + 2] = dv;
}

// sum of squares of a rows x cols input (plain scaling, ortho.py:153-154) -> slot 0
__global__ void sumsq_kernel(const void* __restrict__ x, int dt, int64_t rows, int64_t cols, int64_t ld, int64_t bs,
                             double* __restrict__ blk, int round_in = 0) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const int64_t total = rows * cols;
  double s = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    double v = load_as_f64(x, b * bs + r * ld + c, dt);
    if (round_in) v = static_cast<double>(__bfloat162float(__float2bfloat16_rn(static_cast<float>(v))));
    s += v * v;
  }
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) {
    double* o = blk + (static_cast<int64_t>(b) * gridDim.x + blockIdx.x) * 3;
    o[0] = s;
    o[1] = 0.0;
    o[2] = 0.0;
  }
}

// ||A||_F^2 partials for the plain scaling (ortho.py:153-154) on 16-byte chunks: a power-of-two
// group of threads walks each row (no per-element index arithmetic), every element squared in
// fp64.  Requires 16-byte aligned rows whose length is a multiple of the chunk; launch_sumsq falls
// back to sumsq_kernel otherwise.  Fixed grid and assignment -> deterministic partials.
__device__ __forceinline__ double round_bf16_d(double a) {
  return static_cast<double>(__bfloat162float(__float2bfloat16_rn(static_cast<float>(a))));
}
template <int DT, bool ROUND>
__device__ __forceinline__ double sumsq_chunk(const uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  double s = 0.0;
  if constexpr (DT == DT_BF16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double a = bf16_lo_to_f32(w[i]), c = bf16_hi_to_f32(w[i]);
      s = fma(a, a, fma(c, c, s));
    }
  } else if constexpr (DT == DT_F32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double a = __uint_as_float(w[i]);
      if (ROUND) a = round_bf16_d(a);
      s = fma(a, a, s);
    }
  } else {
    double a = __hiloint2double(static_cast<int>(w[1]), static_cast<int>(w[0]));
    double c = __hiloint2double(static_cast<int>(w[3]), static_cast<int>(w[2]));
    if (ROUND) {
      a = round_bf16_d(a);
      c = round_bf16_d(c);
    }
    s = fma(a, a, c * c);
  }
  return s;
}

template <int DT, bool ROUND>
__global__ void sumsq_vec_kernel(const void* __restrict__ x, int64_t rows, int64_t cpr, int64_t ld, int64_t bs,
                                 int tpr, double* __restrict__ blk) {
  __shared__ double scratch[32];
  constexpr int E = DT == DT_F64 ? 8 : (DT == DT_F32 ? 4 : 2);
  const int b = blockIdx.y;
  const char* base = static_cast<const char*>(x) + static_cast<int64_t>(b) * bs * E;
  const int rpi = blockDim.x / tpr, sub = threadIdx.x / tpr, li = threadIdx.x % tpr;
  double s = 0.0;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * rpi + sub; r < rows; r += static_cast<int64_t>(gridDim.x) * rpi) {
    const uint4* row = reinterpret_cast<const uint4*>(base + r * ld * E);
    int64_t c = li;
    for (; c + 3 * tpr < cpr; c += 4 * tpr) {  // four independent 16-byte loads in flight per thread
      const uint4 v0 = __ldcs(row + c), v1 = __ldcs(row + c + tpr), v2 = __ldcs(row + c + 2 * tpr),
                  v3 = __ldcs(row + c + 3 * tpr);
      s += (sumsq_chunk<DT, ROUND>(v0) + sumsq_chunk<DT, ROUND>(v1)) +
           (sumsq_chunk<DT, ROUND>(v2) + sumsq_chunk<DT, ROUND>(v3));
    }
    for (; c < cpr; c += tpr) s += sumsq_chunk<DT, ROUND>(__ldcs(row + c));
  }
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) {
    double* o = blk + (static_cast<int64_t>(b) * gridDim.x + blockIdx.x) * 3;
    o[0] = s;
    o[1] = 0.0;
    o[2] = 0.0;
  }
}

// Plain-scaling partials (norm_blocks(rows * cols) per matrix into blk), vectorized when the layout allows.
// round_in: square the bf16-rounded values (bf16-mode NS path, see launch_ns_init_state).
inline void launch_sumsq(const void* x, int dt, int64_t rows, int64_t cols, int64_t ld, int64_t bs, int64_t batch,
                         double* blk, cudaStream_t st, bool round_in = false) {
  const int e = dt == DT_F64 ? 8 : (dt == DT_F32 ? 4 : 2), v = 16 / e;
  const bool vec = (cols % v) == 0 && ((ld * e) & 15) == 0 && ((bs * e) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const dim3 grid(norm_blocks(rows * cols), static_cast<unsigned>(batch));
  if (!vec) {
    sumsq_kernel<<<grid, 256, 0, st>>>(x, dt, rows, cols, ld, bs, blk, round_in ? 1 : 0);
    return;
  }
  const int64_t cpr = cols / v;
  int tpr = 1;
  while (tpr < cpr && tpr < 256) tpr <<= 1;
  if (dt == DT_BF16)
    sumsq_vec_kernel<DT_BF16, false><<<grid, 256, 0, st>>>(x, rows, cpr, ld, bs, tpr, blk);
  else if (dt == DT_F32)
    (round_in ? sumsq_vec_kernel<DT_F32, true> : sumsq_vec_kernel<DT_F32, false>)<<<grid, 256, 0, st>>>(
        x, rows, cpr, ld, bs, tpr, blk);
  else
    (round_in ? sumsq_vec_kernel<DT_F64, true> : sumsq_vec_kernel<DT_F64, false>)<<<grid, 256, 0, st>>>(
        x, rows, cpr, ld, bs, tpr, blk);
}

enum ScalarsMode : int { SM_GRAM = 0, SM_PLAIN = 1, SM_GELFAND = 2, SM_ERROR = 3, SM_NONE = 4 };

// One block per matrix: fixed-order reduction of the partials, then the scale
// denominator of preprocess (ortho.py:153-165) and the degenerate-input status.
__global__ void scalars_kernel(const double* __restrict__ blk, int nblk, int mode, int gelfand_power,
                               double* __restrict__ scal, int32_t* __restrict__ status) {
  __shared__ double scratch[32];
  const int b = blockIdx.x;
  double t0 = 0.0, t1 = 0.0, t2 = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    const double* p = blk + (static_cast<int64_t>(b) * nblk + i) * 3;
    t0 += p[0];
    t1 += p[1];
    t2 += p[2];
  }
  t0 = block_sum(t0, scratch);
  const double s0 = t0;
  t1 = block_sum(t1, scratch);
  const double s1 = t1;
  t2 = block_sum(t2, scratch);
  const double s2v = t2;
  if (threadIdx.x != 0) return;
  double* o = scal + static_cast<int64_t>(b) * SCAL_STRIDE;
  if (mode == SM_ERROR) {
    o[S_ERR] = sqrt(s2v);
    return;
  }
  if (mode == SM_GELFAND) {
    // s0/s1 are the norms of G^k: denom = ||G^k||_F^(1/2k) -> s^2 = ||G^k||_F^(1/k)
    const double s2 = pow(sqrt(s1), 1.0 / gelfand_power);
    o[S_S2] = s2;
    o[S_INV_S] = 1.0 / sqrt(s2);
    const bool bad = !(s2 > 0.0) || !isfinite(s2) || !isfinite(o[S_INV_S]);
    if (status && bad) status[b] = 2;
    return;
  }
  o[S_TRACE] = s0;
  o[S_FRO2] = s1;
  o[S_DEV2] = s2v;
  o[S_SHIFT] = 0.0;
  o[S_MODE] = 0.0;
  o[S_BOUND] = -1.0;
  o[S_STEPS] = -1.0;
  if (mode == SM_NONE) {  // bare kernel on pre-scaled input: no rescale, no degenerate check
    o[S_S2] = 1.0;
    o[S_INV_S] = 1.0;
    if (status) status[b] = 0;
    return;
  }
  const double s2 = (mode == SM_PLAIN) ? s0 : sqrt(s1);
  o[S_S2] = s2;
  o[S_INV_S] = 1.0 / sqrt(s2);
  // zero input <=> trace(A A^T) = ||A||_F^2 = 0 (ortho.py:147-148); bad denominator (ortho.py:164-165)
  const bool bad = !(s0 > 0.0) || !isfinite(s0) || !(s2 > 0.0) || !isfinite(s2) || !isfinite(o[S_INV_S]);
  if (status) status[b] = bad ? 2 : 0;
}

__global__ void copy_err_kernel(const double* __restrict__ scal, int batch, double* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) out[b] = scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_ERR];
}

__global__ void copy_denom_kernel(const double* __restrict__ scal, int batch, double* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) out[b] = sqrt(scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_S2]);
}

// ------------------------------------------------------------------ chain prologue
// C_1 = G / s^2 (C-form state), P = alpha I - coef1 C_1 with
// alpha = 1 + sum(a) + b.  fp64 variant (FP32 precision) and bf16 hi/lo variant.
template <typename TG>
__global__ void prep_f64_kernel(const TG* __restrict__ G, int h, int64_t ld, const double* __restrict__ scal,
                                double alpha, double coef1, double* __restrict__ C, double* __restrict__ P) {
  const int b = blockIdx.y;
  const int64_t total = static_cast<int64_t>(h) * h;
  const double inv_s2 = 1.0 / scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_S2];
  const int64_t off = static_cast<int64_t>(b) * h * ld;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / h, c = i - r * h, o = off + r * ld + c;
    const double cv = static_cast<double>(G[o]) * inv_s2;
    C[o] = cv;
    P[o] = (r == c ? alpha : 0.0) - coef1 * cv;
  }
}

__global__ void prep_bf16_kernel(const float* __restrict__ G, int h, int64_t ld, const double* __restrict__ scal,
                                 double alpha, double coef1, __nv_bfloat16* __restrict__ Chi,
                                 __nv_bfloat16* __restrict__ Clo, float* __restrict__ P) {
  const int b = blockIdx.y;
  const int64_t total = static_cast<int64_t>(h) * h;
  const double inv_s2 = 1.0 / scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_S2];
  const int64_t off = static_cast<int64_t>(b) * h * ld;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / h, c = i - r * h, o = off + r * ld + c;
    const float cv = static_cast<float>(static_cast<double>(G[o]) * inv_s2);
    __nv_bfloat16 hi, lo;
    split_bf16(cv, hi, lo);
    Chi[o] = hi;
    Clo[o] = lo;
    P[o] = static_cast<float>((r == c ? alpha : 0.0) - coef1 * static_cast<double>(cv));
  }
}

// ------------------------------------------------------------------ P finalisation
// Reads the upper triangle of P (the only part the chain epilogues maintain),
// scales by 1/s (ortho.py:167 folded into the apply) and writes it symmetric.
template <int OUT>  // 0: f64 full, 1: bf16 hi/lo full
__global__ void finalize_p_kernel(const void* __restrict__ Pin, int h, int64_t ld, const double* __restrict__ scal,
                                  void* __restrict__ out0, void* __restrict__ out1) {
  __shared__ double tile[32][33];
  const int nt = (h + 31) / 32;
  int ti, tj;
  sym_tile_coords(blockIdx.x, nt, ti, tj);
  const int b = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t off = static_cast<int64_t>(b) * h * ld;
  const double inv_s = scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_INV_S];
  const double shift = scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_SHIFT];  // d/s (0 unless decided)
  for (int r = ty; r < 32; r += 8) {
    const int gr = ti * 32 + r, gc = tj * 32 + tx;
    double v = 0.0;
    if (gr < h && gc < h) {
      const int64_t o = off + static_cast<int64_t>(gr) * ld + gc;
      v = OUT == 0 ? static_cast<const double*>(Pin)[o] : static_cast<double>(static_cast<const float*>(Pin)[o]);
    }
    tile[r][tx] = v * inv_s - (gr == gc ? shift : 0.0);
  }
  __syncthreads();
  auto put = [&](int gr, int gc, double v) {
    const int64_t o = off + static_cast<int64_t>(gr) * ld + gc;
    if (OUT == 0) {
      static_cast<double*>(out0)[o] = v;
    } else {
      __nv_bfloat16 hi, lo;
      split_bf16(static_cast<float>(v), hi, lo);
      static_cast<__nv_bfloat16*>(out0)[o] = hi;
      static_cast<__nv_bfloat16*>(out1)[o] = lo;
    }
  };
  for (int r = ty; r < 32; r += 8) {
    const int gr = ti * 32 + r, gc = tj * 32 + tx;
    if (gr < h && gc < h) put(gr, gc, (ti == tj && r > tx) ? tile[tx][r] : tile[r][tx]);
    if (ti != tj) {
      const int mr = tj * 32 + r, mc = ti * 32 + tx;
      if (mr < h && mc < h) put(mr, mc, tile[tx][r]);
    }
  }
}

// finalize_p_kernel<1> for the tensor-core path, vectorised: 64 x 64 upper tiles of the f32 P, 16-byte
// loads and 8-byte bf16 hi/lo stores of both the tile and its mirror.  Same values as the scalar form
// (split of float(p / s - shift)).  Requires ld % 4 == 0 and ld >= round_up(h, 64) (the workspace ldc):
// columns in [h, round_up(h, 64)) of the padded rows are written as zeros.
__global__ void __launch_bounds__(256) finalize_p_bf16_kernel(const float* __restrict__ Pin, int h, int64_t ld,
                                                              const double* __restrict__ scal,
                                                              __nv_bfloat16* __restrict__ hi,
                                                              __nv_bfloat16* __restrict__ lo) {
  __shared__ float tile[64][65];
  const int nt = (h + 63) / 64;
  int ti, tj;
  sym_tile_coords(blockIdx.x, nt, ti, tj);
  const int b = blockIdx.y;
  const int64_t off = static_cast<int64_t>(b) * h * ld;
  const double inv_s = scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_INV_S];
  const double shift = scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_SHIFT];
  const int cq = (threadIdx.x & 15) * 4, r0 = threadIdx.x >> 4;
  for (int r = r0; r < 64; r += 16) {
    const int gr = ti * 64 + r, gc = tj * 64 + cq;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (gr < h) v = *reinterpret_cast<const float4*>(Pin + off + static_cast<int64_t>(gr) * ld + gc);
    const float in[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = gc + q;
      tile[r][cq + q] =
          (gr < h && c < h) ? static_cast<float>(static_cast<double>(in[q]) * inv_s - (gr == c ? shift : 0.0)) : 0.f;
    }
  }
  __syncthreads();
  auto put4 = [&](int gr, int gc, const float (&v)[4]) {
    __nv_bfloat16 h4[4], l4[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) split_bf16(v[q], h4[q], l4[q]);
    const int64_t o = off + static_cast<int64_t>(gr) * ld + gc;
    *reinterpret_cast<uint2*>(hi + o) = *reinterpret_cast<const uint2*>(h4);
    *reinterpret_cast<uint2*>(lo + o) = *reinterpret_cast<const uint2*>(l4);
  };
  for (int r = r0; r < 64; r += 16) {
    float v[4];
    if (ti * 64 + r < h) {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (ti == tj && r > cq + q) ? tile[cq + q][r] : tile[r][cq + q];
      put4(ti * 64 + r, tj * 64 + cq, v);
    }
    if (ti != tj && tj * 64 + r < h) {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = tile[cq + q][r];
      put4(tj * 64 + r, ti * 64 + cq, v);
    }
  }
}

}  // namespace unso
