// Shared device helpers: element loads/stores by dtype, bf16 hi/lo split, reductions.
#pragma once
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace unso {

// Kernel attributes (the dynamic shared-memory opt-in) and occupancy are per device: one flag bit
// per device ordinal, so a process driving several GPUs configures every one of them.
struct PerDeviceFlag {
  std::atomic<unsigned long long> bits{0};
  static int current() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
  }
  bool test(int d) const { return (bits.load(std::memory_order_acquire) >> d) & 1ull; }
  void set(int d) { bits.fetch_or(1ull << d, std::memory_order_acq_rel); }
};

// Developer A/B overrides (routes, recipes) are read from the environment only in builds with
// -DUNSO_DEVELOPER_OVERRIDES; the shipped library ignores them.
inline const char* dev_override(const char* name) {
#ifdef UNSO_DEVELOPER_OVERRIDES
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

enum Dtype : int { DT_F32 = 0, DT_BF16 = 1, DT_F64 = 2 };

__host__ __device__ inline int dtype_size(int dt) { return dt == DT_F32 ? 4 : (dt == DT_BF16 ? 2 : 8); }

__device__ __forceinline__ double load_as_f64(const void* p, int64_t i, int dt) {
  if (dt == DT_F32) return static_cast<double>(static_cast<const float*>(p)[i]);
  if (dt == DT_BF16) return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]));
  return static_cast<const double*>(p)[i];
}
__device__ __forceinline__ void store_from_f64(void* p, int64_t i, int dt, double v) {
  if (dt == DT_F32)
    static_cast<float*>(p)[i] = static_cast<float>(v);
  else if (dt == DT_BF16)
    static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(static_cast<float>(v));
  else
    static_cast<double*>(p)[i] = v;
}

// x ~= hi + lo with hi = bf16(x), lo = bf16(x - hi): 16 significant bits, the operand
// split used by the bf16x3 / bf16x2 tensor-core products.
__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// bf16x2 pack (lo -> bits 0..15, hi -> bits 16..31), round to nearest even; and exact unpack.
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// two e4m3 (RNE, saturating): a -> bits 0..7, b -> bits 8..15
__device__ __forceinline__ uint32_t pack_e4m3x2(float a, float b) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(b), "f"(a));
  return r;
}
// 256-bit global accesses (sm_100: LDG/STG .256): one full 32-byte sector per lane
__device__ __forceinline__ void st_global_v8(void* p, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
// streaming (evict-first) variant for write-once outputs
__device__ __forceinline__ void st_global_cs_v8(void* p, const uint32_t (&w)[8]) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
__device__ __forceinline__ void ld_global_v8(const void* p, uint32_t (&w)[8]) {
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}
__device__ __forceinline__ float bf16_lo_to_f32(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi_to_f32(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum (blockDim.x multiple of 32, <= 1024); result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* scratch /* >= 32 */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? scratch[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

}  // namespace unso
