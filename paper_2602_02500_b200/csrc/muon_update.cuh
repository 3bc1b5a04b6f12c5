// Elementwise passes of the Muon optimizer step around the batched orthogonalizer (
// the reference lists the optimizer itself as out of scope).  Two multi-tensor kernels
// replace five torch passes per shape group (momentum, Nesterov stacking, zero check, decay, update):
//
//   prepare: for matrix i of the group (device pointer lists, all tensors `numel` elements, one dtype)
//              M_i <- mu M_i + G_i;  U_i = G_i + mu M_i (Nesterov) or M_i, written into the stacked
//              batch;  maxabs[i] = max |U_i| (zero update -> zero step, no host sync)
//   update:  P_i <- decay P_i + alpha O_i   (O_i = 0 when maxabs[i] == 0)
//
// 16-byte vectors, fp32 arithmetic with one rounding per stored value, ~16K elements per CTA.
#pragma once
#include "common.cuh"

namespace unso {

constexpr int MUON_THREADS = 256;

__device__ __forceinline__ float muon_block_max(float v) {
  __shared__ float red[MUON_THREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int w = 1; w < MUON_THREADS / 32; ++w) v = fmaxf(v, red[w]);
  return v;  // valid in thread 0
}

template <typename T> struct MuonVec;
template <> struct MuonVec<float> {
  static constexpr int N = 4;
  __device__ static void load(const float* p, float (&v)[4]) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
  __device__ static void store(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct MuonVec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void load(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 q = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[2 * j] = __uint_as_float(w[j] << 16);
      v[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
    }
  }
  __device__ static void store(__nv_bfloat16* p, const float (&v)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      w[j] = *reinterpret_cast<const uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};

__device__ __forceinline__ float muon_ld(const float* p) { return *p; }
__device__ __forceinline__ float muon_ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void muon_st(float* p, float v) { *p = v; }
__device__ __forceinline__ void muon_st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ float muon_round(float v, float) { return v; }
__device__ __forceinline__ float muon_round(float v, __nv_bfloat16) { return __bfloat162float(__float2bfloat16_rn(v)); }

// grid (ceil(numel / per_block), n); every pointer 16-byte aligned (checked by the host)
template <typename T>
__global__ void __launch_bounds__(MUON_THREADS) muon_prepare_kernel(const uint64_t* grads, const uint64_t* bufs,
                                                                     T* stacked, int64_t numel, int64_t per_block,
                                                                     float mu, int nesterov, float* maxabs) {
  using V = MuonVec<T>;
  const int i = blockIdx.y;
  const T* g = reinterpret_cast<const T*>(grads[i]);
  T* m = reinterpret_cast<T*>(bufs[i]);
  T* u = stacked + static_cast<int64_t>(i) * numel;
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * per_block;
  const int64_t e1 = min(numel, e0 + per_block);
  float mx = 0.f;
  const int64_t v1 = e0 + (e1 - e0) / V::N * V::N;
  for (int64_t e = e0 + static_cast<int64_t>(threadIdx.x) * V::N; e < v1; e += static_cast<int64_t>(blockDim.x) * V::N) {
    float gv[V::N], mv[V::N], uv[V::N];
    V::load(g + e, gv);
    V::load(m + e, mv);
#pragma unroll
    for (int j = 0; j < V::N; ++j) {
      mv[j] = muon_round(fmaf(mu, mv[j], gv[j]), T());
      uv[j] = nesterov ? muon_round(fmaf(mu, mv[j], gv[j]), T()) : mv[j];
      mx = fmaxf(mx, fabsf(uv[j]));
    }
    V::store(m + e, mv);
    V::store(u + e, uv);
  }
  for (int64_t e = v1 + threadIdx.x; e < e1; e += blockDim.x) {  // tail (numel not a multiple of the vector)
    const float gv = muon_ld(g + e);
    const float mv = muon_round(fmaf(mu, muon_ld(m + e), gv), T());
    const float uv = nesterov ? muon_round(fmaf(mu, mv, gv), T()) : mv;
    muon_st(m + e, mv);
    muon_st(u + e, uv);
    mx = fmaxf(mx, fabsf(uv));
  }
  mx = muon_block_max(mx);
  // non-negative floats (and +NaN) order like their bit patterns: one integer atomicMax per CTA
  if (threadIdx.x == 0 && mx != 0.f) atomicMax(reinterpret_cast<int*>(maxabs) + i, __float_as_int(mx));
}

template <typename T>
__global__ void __launch_bounds__(MUON_THREADS) muon_update_kernel(const uint64_t* params, const T* ortho,
                                                                    int64_t numel, int64_t per_block,
                                                                    const float* maxabs, float decay, float alpha) {
  using V = MuonVec<T>;
  const int i = blockIdx.y;
  T* p = reinterpret_cast<T*>(params[i]);
  const T* o = ortho + static_cast<int64_t>(i) * numel;
  const float a = maxabs[i] != 0.f ? alpha : 0.f;  // zero update -> zero step (O may be non-finite)
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * per_block;
  const int64_t e1 = min(numel, e0 + per_block);
  const int64_t v1 = e0 + (e1 - e0) / V::N * V::N;
  for (int64_t e = e0 + static_cast<int64_t>(threadIdx.x) * V::N; e < v1; e += static_cast<int64_t>(blockDim.x) * V::N) {
    float pv[V::N], ov[V::N];
    V::load(p + e, pv);
    if (a != 0.f) V::load(o + e, ov);
#pragma unroll
    for (int j = 0; j < V::N; ++j) pv[j] = a != 0.f ? fmaf(a, ov[j], decay * pv[j]) : decay * pv[j];
    V::store(p + e, pv);
  }
  for (int64_t e = v1 + threadIdx.x; e < e1; e += blockDim.x) {
    const float pv = muon_ld(p + e);
    muon_st(p + e, a != 0.f ? fmaf(a, muon_ld(o + e), decay * pv) : decay * pv);
  }
}

}  // namespace unso
