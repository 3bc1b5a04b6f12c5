// Newton-Schulz / Muon comparison path in BF16 precision (ortho.py:208-256), on the
// tensor-core engines.  Recipe: fp32 X state, bf16 X operand for the
// Gram, the h x h step operator B in fp32 and split bf16 hi/lo for the apply:
//   quintic  G = X^T X ; B = b G + c G^2 (bf16x3 SYRK) ; X' = a X + X B   (ortho.py:221-231 regrouped)
//   cubic    G = X^T X ; B = -0.5 G                    ; X' = 1.5 X + X B (ortho.py:208-218)
// (tall orientation shown; wide uses X X^T and B X).
#pragma once
#include "common.cuh"
#include "elementwise.cuh"

namespace unso {

// X state (fp32, ld = cols) and its bf16 operand copy (ld = xld), optionally scaled by 1/s.
__global__ void ns_init_state_kernel(const void* __restrict__ src, int sdt, int64_t sld, int64_t sbs,
                                     const double* __restrict__ scal, float* __restrict__ xf,
                                     __nv_bfloat16* __restrict__ xb, int64_t xld, int64_t rows, int64_t cols,
                                     int batch) {
  const int64_t per = rows * cols, total = per * batch;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / per, rc = i - b * per, r = rc / cols, c = rc - r * cols;
    double v = load_as_f64(src, b * sbs + r * sld + c, sdt);
    if (scal) v *= scal[b * SCAL_STRIDE + S_INV_S];
    const float f = static_cast<float>(v);
    xf[b * per + r * cols + c] = f;
    xb[b * rows * xld + r * xld + c] = __float2bfloat16_rn(f);
  }
}

// out_hi/lo = split(factor * G), full h x h (the cubic step operator B = -0.5 G).
__global__ void split_scaled_kernel(const float* __restrict__ G, int h, int64_t ld, float factor,
                                    __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  const int b = blockIdx.y;
  const int64_t total = static_cast<int64_t>(h) * h, off = static_cast<int64_t>(b) * h * ld;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / h, c = i - r * h, o = off + r * ld + c;
    split_bf16(factor * G[o], hi[o], lo[o]);
  }
}

__global__ void fill_unit_scal_kernel(double* __restrict__ scal, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  for (int k = 0; k < SCAL_STRIDE; ++k) scal[b * SCAL_STRIDE + k] = 0.0;
  scal[b * SCAL_STRIDE + S_S2] = 1.0;
  scal[b * SCAL_STRIDE + S_INV_S] = 1.0;
}

// Quintic operator on the CTA's rows of an upper pair tile: B = bq G + cq (G G^T)  (G symmetric).
struct EpiQuinticBF16 {
  const float* G;
  float* B;
  int64_t ld, bs;
  int h;
  float bq, cq;
  __device__ __forceinline__ void operator()(int b, int, int row, int col0, const float (&v)[32]) const {
    if (row >= h) return;
    const int64_t o = static_cast<int64_t>(b) * bs + static_cast<int64_t>(row) * ld + col0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 g = *reinterpret_cast<const float4*>(G + o + 4 * j);
      *reinterpret_cast<float4*>(B + o + 4 * j) =
          make_float4(bq * g.x + cq * v[4 * j], bq * g.y + cq * v[4 * j + 1], bq * g.z + cq * v[4 * j + 2],
                      bq * g.w + cq * v[4 * j + 3]);
    }
  }
};

// X' = alpha X + acc on the fp32 state, plus the bf16 operand copy for the next Gram.
struct EpiNSUpdate {
  const float* xold;
  float* xnew;
  __nv_bfloat16* xb;
  int64_t xld;            // bf16 copy leading dim
  int64_t rows, cols;     // state is rows x cols, ld = cols
  int M, N;               // output tile bounds (= rows, cols in the matrix's own layout)
  float alpha;
  __device__ __forceinline__ void operator()(int b, int, int row, int col0, const float (&v)[32]) const {
    if (row >= M) return;
    const int64_t o = static_cast<int64_t>(b) * rows * cols + static_cast<int64_t>(row) * cols + col0;
    const int64_t ob = static_cast<int64_t>(b) * rows * xld + static_cast<int64_t>(row) * xld + col0;
    float xn[32];
    const bool vec = col0 + 32 <= N && (cols % 4) == 0 && (xld % 8) == 0;
    if (vec) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 t = *reinterpret_cast<const float4*>(xold + o + 4 * j);
        xn[4 * j] = fmaf(alpha, t.x, v[4 * j]);
        xn[4 * j + 1] = fmaf(alpha, t.y, v[4 * j + 1]);
        xn[4 * j + 2] = fmaf(alpha, t.z, v[4 * j + 2]);
        xn[4 * j + 3] = fmaf(alpha, t.w, v[4 * j + 3]);
        *reinterpret_cast<float4*>(xnew + o + 4 * j) = make_float4(xn[4 * j], xn[4 * j + 1], xn[4 * j + 2], xn[4 * j + 3]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<uint4*>(xb + ob + 8 * j) =
            make_uint4(pack_bf16x2(xn[8 * j], xn[8 * j + 1]), pack_bf16x2(xn[8 * j + 2], xn[8 * j + 3]),
                       pack_bf16x2(xn[8 * j + 4], xn[8 * j + 5]), pack_bf16x2(xn[8 * j + 6], xn[8 * j + 7]));
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (col0 + j < N) {
          const float x = fmaf(alpha, xold[o + j], v[j]);
          xnew[o + j] = x;
          xb[ob + j] = __float2bfloat16_rn(x);
        }
      }
    }
  }
};

}  // namespace unso
