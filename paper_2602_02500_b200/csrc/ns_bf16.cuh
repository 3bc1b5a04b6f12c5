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
                                     int batch, int round_in, __nv_bfloat16* __restrict__ xlo) {
  const int64_t per = rows * cols, total = per * batch;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / per, rc = i - b * per, r = rc / cols, c = rc - r * cols;
    double v = load_as_f64(src, b * sbs + r * sld + c, sdt);
    if (round_in) v = static_cast<double>(__bfloat162float(__float2bfloat16_rn(static_cast<float>(v))));
    if (scal) v *= scal[b * SCAL_STRIDE + S_INV_S];
    const float f = static_cast<float>(v);
    xf[b * per + r * cols + c] = f;
    const __nv_bfloat16 hb = __float2bfloat16_rn(f);
    xb[b * rows * xld + r * xld + c] = hb;
    if (xlo) xlo[b * rows * xld + r * xld + c] = __float2bfloat16_rn(f - __bfloat162float(hb));
  }
}

// Same state initialisation on 8-element chunks (16-byte aligned rows, cols % 8 == 0): a
// power-of-two group of threads per row, no per-element index arithmetic; identical rounding
// (double scale -> float -> bf16 RNE).
template <int SDT>
__global__ void ns_init_state_vec_kernel(const void* __restrict__ src, int64_t sld, int64_t sbs,
                                         const double* __restrict__ scal, float* __restrict__ xf,
                                         __nv_bfloat16* __restrict__ xb, int64_t xld, int64_t rows, int64_t cols,
                                         int batch, int tpr, int round_in, __nv_bfloat16* __restrict__ xlo) {
  constexpr int E = SDT == DT_F64 ? 8 : (SDT == DT_F32 ? 4 : 2);
  const int64_t cpr = cols / 8, nrows = rows * batch;
  const int rpi = blockDim.x / tpr, sub = threadIdx.x / tpr, li = threadIdx.x % tpr;
  for (int64_t R = static_cast<int64_t>(blockIdx.x) * rpi + sub; R < nrows; R += static_cast<int64_t>(gridDim.x) * rpi) {
    const int64_t b = R / rows, r = R - b * rows;
    const double sc = scal ? scal[b * SCAL_STRIDE + S_INV_S] : 1.0;
    const char* srow = static_cast<const char*>(src) + (b * sbs + r * sld) * E;
    float* frow = xf + (b * rows + r) * cols;
    __nv_bfloat16* brow = xb + (b * rows + r) * xld;
    for (int64_t c = li; c < cpr; c += tpr) {
      float f[8];
      if constexpr (SDT == DT_BF16) {
        const uint4 v = *reinterpret_cast<const uint4*>(srow + c * 16);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          f[2 * i] = static_cast<float>(static_cast<double>(bf16_lo_to_f32(w[i])) * sc);
          f[2 * i + 1] = static_cast<float>(static_cast<double>(bf16_hi_to_f32(w[i])) * sc);
        }
      } else if constexpr (SDT == DT_F32) {
        const float4 a = *reinterpret_cast<const float4*>(srow + c * 32);
        const float4 d = *reinterpret_cast<const float4*>(srow + c * 32 + 16);
        const float in[8] = {a.x, a.y, a.z, a.w, d.x, d.y, d.z, d.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float vi = round_in ? __bfloat162float(__float2bfloat16_rn(in[i])) : in[i];
          f[i] = static_cast<float>(static_cast<double>(vi) * sc);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          double vi = reinterpret_cast<const double*>(srow)[c * 8 + i];
          if (round_in) vi = static_cast<double>(__bfloat162float(__float2bfloat16_rn(static_cast<float>(vi))));
          f[i] = static_cast<float>(vi * sc);
        }
      }
      *reinterpret_cast<float4*>(frow + c * 8) = make_float4(f[0], f[1], f[2], f[3]);
      *reinterpret_cast<float4*>(frow + c * 8 + 4) = make_float4(f[4], f[5], f[6], f[7]);
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        hw[e] = pack_bf16x2(f[2 * e], f[2 * e + 1]);
        lw[e] = pack_bf16x2(f[2 * e] - bf16_lo_to_f32(hw[e]), f[2 * e + 1] - bf16_hi_to_f32(hw[e]));
      }
      *reinterpret_cast<uint4*>(brow + c * 8) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      if (xlo) *reinterpret_cast<uint4*>(xlo + (b * rows + r) * xld + c * 8) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
  }
}

// round_in: round every input value to bf16 first (bf16 mode: the path computes on the bf16-rounded
// input, the same values the UNSO path and the parity oracle see).
inline void launch_ns_init_state(const void* src, int sdt, int64_t sld, int64_t sbs, const double* scal, float* xf,
                                 __nv_bfloat16* xb, int64_t xld, int64_t rows, int64_t cols, int batch,
                                 int round_in, cudaStream_t st, __nv_bfloat16* xlo = nullptr) {
  const int e = sdt == DT_F64 ? 8 : (sdt == DT_F32 ? 4 : 2);
  const bool vec = (cols % 8) == 0 && ((sld * e) & 15) == 0 && ((sbs * e) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (xld % 8) == 0 &&
                   (reinterpret_cast<uintptr_t>(xb) & 15) == 0 && (reinterpret_cast<uintptr_t>(xf) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(xlo) & 15) == 0;
  if (!vec) {
    const int64_t total = rows * cols * batch;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    ns_init_state_kernel<<<blocks, 256, 0, st>>>(src, sdt, sld, sbs, scal, xf, xb, xld, rows, cols, batch, round_in, xlo);
    return;
  }
  const int64_t cpr = cols / 8;
  int tpr = 1;
  while (tpr < cpr && tpr < 256) tpr <<= 1;
  const int64_t nrows = rows * batch;
  const int blocks = static_cast<int>(std::min<int64_t>((nrows + 256 / tpr - 1) / (256 / tpr), 148 * 16));
  if (sdt == DT_BF16)
    ns_init_state_vec_kernel<DT_BF16><<<blocks, 256, 0, st>>>(src, sld, sbs, scal, xf, xb, xld, rows, cols, batch, tpr, round_in, xlo);
  else if (sdt == DT_F32)
    ns_init_state_vec_kernel<DT_F32><<<blocks, 256, 0, st>>>(src, sld, sbs, scal, xf, xb, xld, rows, cols, batch, tpr, round_in, xlo);
  else
    ns_init_state_vec_kernel<DT_F64><<<blocks, 256, 0, st>>>(src, sld, sbs, scal, xf, xb, xld, rows, cols, batch, tpr, round_in, xlo);
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
  __nv_bfloat16* xlo = nullptr;  // optional bf16 lo part of the new state (hi/lo products)
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
      for (int j = 0; j < 4; ++j) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hw[e] = pack_bf16x2(xn[8 * j + 2 * e], xn[8 * j + 2 * e + 1]);
          lw[e] = pack_bf16x2(xn[8 * j + 2 * e] - bf16_lo_to_f32(hw[e]), xn[8 * j + 2 * e + 1] - bf16_hi_to_f32(hw[e]));
        }
        *reinterpret_cast<uint4*>(xb + ob + 8 * j) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        if (xlo) *reinterpret_cast<uint4*>(xlo + ob + 8 * j) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (col0 + j < N) {
          const float x = fmaf(alpha, xold[o + j], v[j]);
          xnew[o + j] = x;
          const __nv_bfloat16 hb = __float2bfloat16_rn(x);
          xb[ob + j] = hb;
          if (xlo) xlo[ob + j] = __float2bfloat16_rn(x - __bfloat162float(hb));
        }
      }
    }
  }
};

}  // namespace unso
