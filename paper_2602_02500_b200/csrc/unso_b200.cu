// B200-native UNSO orthogonalization: host orchestration + C ABI (include/unso_b200.h).
//
// Reference path (arXiv 2602.02500, /root/reference/pkg/src/unso/ortho.py):
//   preprocess (:140-168) -> unso (:171-205) | original_ns (:208-218) | _quintic_steps (:221-231)
// Device pipeline for UNSO (one stream, no host syncs):
//   [convert]  X -> bf16 copy (BF16 precision with f32 input only)
//   K1  Gram SYRK over the long side, split-K partials        (ortho.py:156/198 computed ONCE)
//       finalize: sum partials, mirror                          (deterministic fixed order)
//       norms + scalars: trace, ||G||_F -> s^2, 1/s, status     (ortho.py:147-165)
//       prep: C_1 = G/s^2, P = alpha I - a_1 C_1                 (C-form of ortho.py:199-202)
//   K2  13 x chain SYRK  C_{k+1} = 2 C_k - C_k^2, P -= c_{k+1} C_{k+1}   (ortho.py:201-204)
//       finalize P: P/s, symmetric, split for the apply          (ortho.py:167 folded)
//   K3  apply Y = X P (tall) or P X (wide), written in the input dtype   (ortho.py:205, :275-276)
#include <cuda.h>
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <vector>

#include "../../include/unso_b200.h"
#include "common.cuh"
#include "elementwise.cuh"
#include "simt_gemm.cuh"
#include "umma_gemm.cuh"
#include "chain_persistent.cuh"
#include "chain_small.cuh"
#include "chain_f64.cuh"
#include "gram_allreduce.cuh"
#include "umma2_gemm.cuh"
#include "chain_pair.cuh"
#include "ns_bf16.cuh"
#include "ozaki_i8.cuh"
#include "multi_chain.cuh"
#include "muon_update.cuh"
#include <cstdlib>

#define UNSO_VERSION_STRING "unso_b200 0.1.0 (sm_100a: tcgen05/TMEM/TMA bf16 path + fp64 DFMA parity path)"

namespace unso {

static thread_local int g_launches = 0;

// Stage profiler (unso_profile_*): CUDA events recorded on the call's stream.
struct Profiler {
  bool on = false;
  int cap = 0, n = 0;
  std::vector<cudaEvent_t> ev;
};
static Profiler g_prof;
static thread_local bool g_prof_call = false;
constexpr int PROF_EV = UNSO_PROFILE_STAGES + 1;
// NVTX ranges (header-only NVTX v3: inert unless a tool such as nsys / ncu --nvtx is attached): one
// range per stage of an orthogonalization, opened and closed at the same marks as the profiler's events.
static nvtxDomainHandle_t nvtx_domain() {
  static nvtxDomainHandle_t d = nvtxDomainCreateA("unso_b200");
  return d;
}
static thread_local nvtxRangeId_t g_nvtx_range = 0;
static void nvtx_stage(int idx) {
  static const char* const names[UNSO_PROFILE_STAGES] = {"unso.convert", "unso.gram", "unso.scale_prep",
                                                         "unso.chain", "unso.finalize_p", "unso.apply"};
  if (g_nvtx_range) nvtxDomainRangeEnd(nvtx_domain(), g_nvtx_range);
  g_nvtx_range = 0;
  if (idx < 0 || idx >= UNSO_PROFILE_STAGES) return;
  nvtxEventAttributes_t a = {};
  a.version = NVTX_VERSION;
  a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
  a.messageType = NVTX_MESSAGE_TYPE_ASCII;
  a.message.ascii = names[idx];
  g_nvtx_range = nvtxDomainRangeStartEx(nvtx_domain(), &a);
}
static void prof_mark(int idx, cudaStream_t st) {
  nvtx_stage(idx);  // mark idx opens stage idx (the profiler's stage idx runs from mark idx to idx + 1)
  if (g_prof_call && g_prof.on && g_prof.n < g_prof.cap) cudaEventRecord(g_prof.ev[g_prof.n * PROF_EV + idx], st);
}

#define UNSO_CHECK_LAUNCH()                          \
  do {                                               \
    ++g_launches;                                    \
    cudaError_t e__ = cudaGetLastError();            \
    if (e__ != cudaSuccess) return UNSO_ERR_CUDA;    \
  } while (0)

#define UNSO_TRY(expr)                               \
  do {                                               \
    int32_t s__ = (expr);                            \
    if (s__ != UNSO_OK) return s__;                  \
  } while (0)

// ==================================================================== tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = []() -> EncodeTiledFn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 3-D SWIZZLE_128B map, memoised per host thread: a map is a pure function of (dtype, base, dims,
// strides, box), and training loops hand the same buffers every step, so most calls skip the
// driver encode (a few microseconds each, several per orthogonalization).
static bool encode_map_3d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, const cuuint64_t (&dims)[3],
                          const cuuint64_t (&strides)[2], cuuint32_t b0, cuuint32_t b1) {
  struct Entry {
    CUtensorMap map;
    const void* base;
    cuuint64_t dims[3], strides[2];
    cuuint32_t b0, b1;
    int dt;
    bool used;
  };
  constexpr int kEntries = 64;
  thread_local Entry cache[kEntries];
  thread_local int next = 0;
  for (Entry& e : cache) {
    if (e.used && e.base == base && e.dt == static_cast<int>(dt) && e.b0 == b0 && e.b1 == b1 &&
        e.dims[0] == dims[0] && e.dims[1] == dims[1] && e.dims[2] == dims[2] && e.strides[0] == strides[0] &&
        e.strides[1] == strides[1]) {
      *m = e.map;
      return true;
    }
  }
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  if (fn(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  Entry& e = cache[next];
  next = (next + 1) % kEntries;
  e.map = *m;
  e.base = base;
  for (int i = 0; i < 3; ++i) e.dims[i] = dims[i];
  e.strides[0] = strides[0];
  e.strides[1] = strides[1];
  e.b0 = b0;
  e.b1 = b1;
  e.dt = static_cast<int>(dt);
  e.used = true;
  return true;
}

static bool make_map(CUtensorMap* m, const void* base, cuuint64_t d0, cuuint64_t d1, cuuint64_t d2, int64_t ld,
                     int64_t bstride, cuuint32_t b0, cuuint32_t b1) {
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(bstride) * 2};
  return encode_map_3d(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, dims, strides, b0, b1);
}

// e4m3 operand maps (byte elements, SWIZZLE_128B, 128-byte TMA rows).
static bool make_map_u8(CUtensorMap* m, const void* base, int64_t d0, int64_t d1, int64_t d2, int64_t ld, int64_t bs,
                        cuuint32_t b0, cuuint32_t b1) {
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d0), static_cast<cuuint64_t>(d1), static_cast<cuuint64_t>(d2)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(d2 <= 1 ? d1 * ld : bs)};
  return encode_map_3d(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, base, dims, strides, b0, b1);
}

bool umma_make_kmajor_map(CUtensorMap* m, const void* base, int64_t rows, int64_t k, int64_t ld, int64_t batch,
                          int64_t bstride, int box_rows) {
  if (batch <= 1) bstride = rows * ld;
  return make_map(m, base, k, rows, batch, ld, bstride, 64, box_rows);
}

bool umma_make_mnmajor_map(CUtensorMap* m, const void* base, int64_t krows, int64_t mn, int64_t ld, int64_t batch,
                           int64_t bstride) {
  if (batch <= 1) bstride = krows * ld;
  return make_map(m, base, mn, krows, batch, ld, bstride, 64, 64);
}

int device_sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  static int cached_dev = -1, cached = 148;
  if (dev != cached_dev) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n;
    cached_dev = dev;
  }
  return cached;
}

// ==================================================================== epilogues
// --- SIMT (per element, n >= m on SYRK) ------------------------------------------
struct EpiPartialF64 {
  double* part;
  int64_t bs;  // per matrix
  int64_t ld;
  int batch;
  __device__ void operator()(int b, int split, int m, int n, double acc) const {
    part[(static_cast<int64_t>(split) * batch + b) * bs + static_cast<int64_t>(m) * ld + n] = acc;
  }
};

// C-form squaring step: C' = 2C - C^2 (the reference's B' = B^2 with B = I - C), P -= coef C'
struct EpiChainF64 {
  const double* cur;
  double* nxt;
  double* P;
  int64_t ld, bs;
  double coef;
  int write_next;
  __device__ void operator()(int b, int, int m, int n, double acc) const {
    const int64_t base = static_cast<int64_t>(b) * bs;
    const int64_t o = base + static_cast<int64_t>(m) * ld + n;
    const double cn = 2.0 * cur[o] - acc;
    if (write_next) {
      nxt[o] = cn;
      nxt[base + static_cast<int64_t>(n) * ld + m] = cn;
    }
    P[o] -= coef * cn;
  }
};

// B = bq G + cq G^2 (quintic step operator, ortho.py:226-230 regrouped), symmetric
struct EpiQuinticB {
  const double* G;
  double* Bm;
  int64_t ld, bs;
  double bq, cq;
  __device__ void operator()(int b, int, int m, int n, double acc) const {
    const int64_t base = static_cast<int64_t>(b) * bs;
    const double v = bq * G[base + static_cast<int64_t>(m) * ld + n] + cq * acc;
    Bm[base + static_cast<int64_t>(m) * ld + n] = v;
    Bm[base + static_cast<int64_t>(n) * ld + m] = v;
  }
};

// out = alpha * acc + beta * old  (old may be null)
struct EpiOut {
  void* out;
  int dt;
  int64_t ld, bs;
  const double* old;
  int64_t old_ld, old_bs;
  double alpha, beta;
  __device__ void operator()(int b, int, int m, int n, double acc) const {
    double v = alpha * acc;
    if (old) v += beta * old[static_cast<int64_t>(b) * old_bs + static_cast<int64_t>(m) * old_ld + n];
    store_from_f64(out, static_cast<int64_t>(b) * bs + static_cast<int64_t>(m) * ld + n, dt, v);
  }
};

// --- tcgen05 (per row, 32 consecutive columns) ---------------------------------------
struct UEpiPartialF32 {
  float* part;
  int64_t bs, ld;
  int batch, h;
  __device__ void operator()(int b, int split, int row, int col0, const float* v) const {
    if (row >= h) return;
    float* dst = part + (static_cast<int64_t>(split) * batch + b) * bs + static_cast<int64_t>(row) * ld + col0;
#pragma unroll
    for (int j = 0; j < 32; j += 8) {  // 256-bit stores (ld is a multiple of 256, col0 of 32)
      uint32_t w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = __float_as_uint(v[j + q]);
      st_global_v8(dst + j, w);
    }
  }
};

struct UEpiChainBF16 {
  const __nv_bfloat16* chi;
  const __nv_bfloat16* clo;
  __nv_bfloat16* nhi;
  __nv_bfloat16* nlo;
  float* P;
  int64_t ld, bs;
  int h;
  float coef;
  int write_next;
  __device__ void operator()(int b, int, int row, int col0, const float* v) const {
    if (row >= h || col0 + 31 < row) return;
    const int64_t base = static_cast<int64_t>(b) * bs;
    const int64_t o = base + static_cast<int64_t>(row) * ld + col0;
    __align__(16) __nv_bfloat16 hi[32];
    __align__(16) __nv_bfloat16 lo[32];
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      *reinterpret_cast<uint4*>(hi + j) = *reinterpret_cast<const uint4*>(chi + o + j);
      *reinterpret_cast<uint4*>(lo + j) = *reinterpret_cast<const uint4*>(clo + o + j);
    }
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const int col = col0 + j;
      if (col < row || col >= h) continue;
      const float c = __bfloat162float(hi[j]) + __bfloat162float(lo[j]);
      const float cn = 2.0f * c - v[j];
      if (write_next) {
        __nv_bfloat16 h2, l2;
        split_bf16(cn, h2, l2);
        nhi[o + j] = h2;
        nlo[o + j] = l2;
        if (col != row) {
          const int64_t t = base + static_cast<int64_t>(col) * ld + row;
          nhi[t] = h2;
          nlo[t] = l2;
        }
      }
      P[o + j] -= coef * cn;
    }
  }
};

struct UEpiOut {
  void* out;
  int dt;  // DT_BF16, DT_F32 or DT_F64
  int64_t ld, bs;
  int M, N;
  // identity shift: Y += scal[b].shift * X (X = the bf16 operand, same indexing as Y)
  const __nv_bfloat16* x = nullptr;
  int64_t xld = 0, xbs = 0;
  const double* scal = nullptr;
  // All indexing below is compile-time (fully unrolled, predicated tails): the 32-value chunk
  // stays in registers (a dynamic index would spill it to local memory, ~18 GB of L1 traffic
  // per cfg4 apply in round-1 ncu).
  __device__ __forceinline__ void add_shift(int b, int row, int col0, float (&v)[32]) const {
    if (!x) return;
    const float sh = static_cast<float>(scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_SHIFT]);
    if (sh == 0.0f) return;
    const __nv_bfloat16* xr = x + static_cast<int64_t>(b) * xbs + static_cast<int64_t>(row) * xld + col0;
    if (col0 + 32 <= N && (reinterpret_cast<uintptr_t>(xr) & 31) == 0) {
#pragma unroll
      for (int j = 0; j < 32; j += 16) {
        uint32_t w[8];
        ld_global_v8(xr + j, w);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          v[j + 2 * q] = fmaf(sh, bf16_lo_to_f32(w[q]), v[j + 2 * q]);
          v[j + 2 * q + 1] = fmaf(sh, bf16_hi_to_f32(w[q]), v[j + 2 * q + 1]);
        }
      }
    } else if (col0 + 32 <= N && (reinterpret_cast<uintptr_t>(xr) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        const uint4 t = *reinterpret_cast<const uint4*>(xr + j);
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[j + 2 * q] = fmaf(sh, bf16_lo_to_f32(w[q]), v[j + 2 * q]);
          v[j + 2 * q + 1] = fmaf(sh, bf16_hi_to_f32(w[q]), v[j + 2 * q + 1]);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < N) v[j] = fmaf(sh, __bfloat162float(xr[j]), v[j]);
    }
  }

  __device__ __forceinline__ void operator()(int b, int, int row, int col0, const float (&vin)[32]) const {
    if (row >= M) return;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = vin[j];
    const bool full = col0 + 32 <= N;
    add_shift(b, row, col0, v);
    const int64_t o = static_cast<int64_t>(b) * bs + static_cast<int64_t>(row) * ld + col0;
    if (dt == DT_BF16) {
      __nv_bfloat16* y = static_cast<__nv_bfloat16*>(out) + o;
      if (full && (reinterpret_cast<uintptr_t>(y) & 31) == 0) {  // two 256-bit stores: whole sectors
#pragma unroll
        for (int j = 0; j < 32; j += 16) {
          uint32_t w[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) w[q] = pack_bf16x2(v[j + 2 * q], v[j + 2 * q + 1]);
          st_global_cs_v8(y + j, w);
        }
      } else if (full && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 8)
          *reinterpret_cast<uint4*>(y + j) =
              make_uint4(pack_bf16x2(v[j], v[j + 1]), pack_bf16x2(v[j + 2], v[j + 3]),
                         pack_bf16x2(v[j + 4], v[j + 5]), pack_bf16x2(v[j + 6], v[j + 7]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) y[j] = __float2bfloat16_rn(v[j]);
      }
    } else if (dt == DT_F32) {
      float* y = static_cast<float*>(out) + o;
      if (full && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(y + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) y[j] = v[j];
      }
    } else {  // f64 I/O on the tensor-core path (the result carries bf16-mode accuracy)
      double* y = static_cast<double*>(out) + o;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < N) y[j] = static_cast<double>(v[j]);
    }
  }
};

// tcgen05 configurations
using CfgGramK = UmmaCfg<128, 1, 1, 1, TERM(0, 0, 0), false, false, 6>;
using CfgGramMN = UmmaCfg<128, 1, 1, 1, TERM(0, 0, 0), true, true, 6>;
// bf16x3: hi*hi + hi*lo + lo*hi
using CfgChain = UmmaCfg<128, 2, 2, 3, TERM(0, 0, 0) | TERM(1, 0, 1) | TERM(2, 1, 0), false, false, 3>;
// tall apply: X * (P_hi + P_lo)
using CfgApplyTall2 = UmmaCfg<128, 1, 2, 2, TERM(0, 0, 0) | TERM(1, 0, 1), false, false, 4>;
using CfgApplyTall1 = UmmaCfg<128, 1, 1, 1, TERM(0, 0, 0), false, false, 6>;
// wide apply: (P_hi + P_lo) * X, X read MN-major
using CfgApplyWide2 = UmmaCfg<128, 2, 1, 2, TERM(0, 0, 0) | TERM(1, 1, 0), false, true, 4>;
using CfgApplyWide1 = UmmaCfg<128, 1, 1, 1, TERM(0, 0, 0), false, true, 6>;
// CTA-pair (cta_group::2) 256 x 256 tiles
using Cfg2GramK = Umma2Cfg<256, 1, 1, 1, TERM(0, 0, 0), false, false, 6>;
using Cfg2GramMN = Umma2Cfg<256, 1, 1, 1, TERM(0, 0, 0), true, true, 6>;
using Cfg2ApplyTall2 = Umma2Cfg<256, 1, 2, 2, TERM(0, 0, 0) | TERM(1, 0, 1), false, false, 4>;
using Cfg2ApplyTall1 = Umma2Cfg<256, 1, 1, 1, TERM(0, 0, 0), false, false, 6>;
using Cfg2ApplyWide2 = Umma2Cfg<256, 2, 1, 2, TERM(0, 0, 0) | TERM(1, 1, 0), false, true, 4>;
using Cfg2ApplyWide1 = Umma2Cfg<256, 1, 1, 1, TERM(0, 0, 0), false, true, 6>;

// Engine selection: CTA pairs by default; UNSO_ENGINE=1cta forces the 1-CTA 128x128 engine (A/B tests).
static bool use_pair_engine() {
  static int v = -1;
  if (v < 0) {
    const char* e = dev_override("UNSO_ENGINE");
    v = (e && std::strcmp(e, "1cta") == 0) ? 0 : 1;
  }
  return v == 1;
}

// ==================================================================== problem + workspace plan
static inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

struct Problem {
  int64_t rows, cols, ld, batch, bs;
  int dt;
  bool tall;
  int64_t h, w;
  int method = 0, scaling = 0, gpow = 1, prec = 0, order = 0, steps = 0, flags = 0;
  std::vector<double> co;
};

static int32_t make_problem(const unso_matrix_desc* x, const unso_method_desc* m, Problem& p, bool need_method = true) {
  if (!x) return UNSO_ERR_VALUE;
  if (x->rows < 1 || x->cols < 1 || x->batch < 1 || x->ld < x->cols) return UNSO_ERR_SHAPE;
  if (x->dtype != UNSO_DTYPE_F32 && x->dtype != UNSO_DTYPE_BF16 && x->dtype != UNSO_DTYPE_F64) return UNSO_ERR_VALUE;
  if (x->rows > (1 << 30) || x->cols > (1 << 30)) return UNSO_ERR_SHAPE;
  p.rows = x->rows;
  p.cols = x->cols;
  p.ld = x->ld;
  p.batch = x->batch;
  p.bs = x->batch > 1 ? x->batch_stride : x->rows * x->ld;
  if (x->batch > 1 && x->batch_stride < x->rows * x->ld) return UNSO_ERR_SHAPE;
  p.dt = x->dtype;
  p.tall = x->rows > x->cols;  // ortho.py:149 (square is not transposed)
  if (x->orientation == 1) p.tall = true;
  if (x->orientation == 2) p.tall = false;
  if (x->orientation < 0 || x->orientation > 2) return UNSO_ERR_VALUE;
  p.h = p.tall ? x->cols : x->rows;
  p.w = p.tall ? x->rows : x->cols;
  if (p.h > 65536) return UNSO_ERR_UNSUPPORTED;
  if (!need_method) return UNSO_OK;
  if (!m) return UNSO_ERR_VALUE;
  p.method = m->method;
  p.scaling = m->scaling;
  p.gpow = m->gelfand_power;
  p.prec = m->precision;
  p.order = m->order;
  p.steps = m->steps;
  p.flags = m->flags;
  if (p.scaling < 0 || p.scaling > 3 || p.gpow < 1) return UNSO_ERR_VALUE;
  if (p.prec != UNSO_PREC_FP32 && p.prec != UNSO_PREC_BF16) return UNSO_ERR_VALUE;
  if (p.method == UNSO_METHOD_UNSO) {
    if (p.order < 1 || !m->coeffs) return UNSO_ERR_VALUE;
    p.co.assign(m->coeffs, m->coeffs + p.order);
  } else if (p.method == UNSO_METHOD_ORIGINAL_NS) {
    if (p.steps < 1) return UNSO_ERR_VALUE;
  } else if (p.method == UNSO_METHOD_QUINTIC) {
    if (p.steps < 1 || !m->coeffs) return UNSO_ERR_VALUE;
    p.co.assign(m->coeffs, m->coeffs + 3 * static_cast<int64_t>(p.steps));
  } else {
    return UNSO_ERR_VALUE;
  }
  for (double v : p.co)
    if (!std::isfinite(v)) return UNSO_ERR_VALUE;
  return UNSO_OK;
}

struct Plan {
  int64_t ldc;    // leading dimension of every h x h workspace matrix
  int64_t hh;     // h * ldc (per matrix)
  int64_t ldx;    // leading dim of the bf16 X copy
  int splits;
  bool xcopy;     // BF16: X needs a bf16 (re-)layout copy
  size_t total = 0;
  size_t xb = 0, part = 0, G = 0, blk = 0, scal = 0;
  size_t C[2] = {0, 0}, P = 0, Pout = 0;          // FP32
  size_t Chi[2] = {0, 0}, Clo[2] = {0, 0}, Phi = 0, Plo = 0;  // BF16 (P reused as f32)
  size_t Gk[2] = {0, 0};                          // gelfand powers
  size_t normbuf = 0, pstat = 0, gbar = 0;        // persistent chain: per-tile norms / P stats, grid barrier
  size_t Xs[2] = {0, 0};                          // NS state (f64 in FP32 mode, f32 in BF16 mode)
  size_t xb2 = 0;                                 // NS BF16: second bf16 operand buffer (ping-pong)
  size_t xl[2] = {0, 0};                          // NS BF16: bf16 lo parts of the state (hi/lo products)
  size_t mnorm = 0, mpstat = 0;                   // multi-launch pipeline: norm / final-P partials
  size_t C8h[2] = {0, 0}, C8l[2] = {0, 0};        // e4m3 operand planes of C_k (2^8 hi, 2^16 lo)
  size_t C8i[2] = {0, 0};                         // e4m3 interleaved [hi8 | lo8] per 64-column block
  size_t ozX = 0, ozC = 0, ozMaxA = 0, ozMaxB = 0;  // FP32 on the int8 tensor cores: digit planes, row maxima
  int64_t ozX_plane = 0, ozC_plane = 0, ozMaxA_bs = 0;
};

static size_t take(Plan& pl, size_t bytes) {
  const size_t off = pl.total;
  pl.total += (bytes + 255) / 256 * 256;
  return off;
}

// Split-K factor: the smallest s whose (tiles x s) work items fill >= 90% of the last wave
// of persistent CTAs (or CTA pairs), keeping >= 4 k-blocks per split.
static int pick_splits(int64_t tiles, int64_t ktiles, int64_t slots) {
  if (tiles >= 2 * slots) return 1;  // >= 2 waves: the tail is small, and no split-K reduction is needed
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 32 && s <= ktiles / 4; ++s) {
    const int64_t items = tiles * s;
    const double eff = static_cast<double>(items) / (static_cast<double>((items + slots - 1) / slots) * slots);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
    if (eff >= 0.9) break;
  }
  return best;
}

// FP32 mode on the int8 tensor cores (ozaki_i8.cuh): UNSO with h > 256 (smaller h runs the
// one-launch fp64 chain, latency-bound) unless UNSO_FLAG_FP32_DMMA asks for the fp64 DMMA engine.
static bool use_oz(const Problem& p) {
  return p.prec == UNSO_PREC_FP32 && p.h > 256 && (p.flags & UNSO_FLAG_FP32_DMMA) == 0;
}
static int64_t oz_syrk_tiles(int64_t h) {  // pair tiles of oz_decode's SYRK order
  const int64_t tm = (h + OZ_BM - 1) / OZ_BM, tn = (h + OZ_BN - 1) / OZ_BN;
  int64_t t = 0;
  for (int64_t i = 0; i < tm; ++i) t += std::max<int64_t>(0, tn - oz_tn_min(static_cast<int>(i)));
  return t;
}

static int gram_splits(const Problem& p, bool for_error = false) {
  if (!for_error && use_oz(p)) {  // every split-K slice within the int32 bound, then fill the last wave
    const int64_t kt = (p.w + OZ_BK - 1) / OZ_BK;
    const int min_s = static_cast<int>((p.w + OZ_MAX_K - 1) / OZ_MAX_K);
    const int s = pick_splits(oz_syrk_tiles(p.h) * p.batch, kt, device_sm_count() / 2);
    return std::max(min_s, s);
  }
  if (p.prec == UNSO_PREC_BF16) {
    const int64_t tm = use_pair_engine() ? 256 : 128;
    const int64_t t = (p.h + tm - 1) / tm;
    const int64_t slots = use_pair_engine() ? 74 : 148;
    return pick_splits(t * (t + 1) / 2 * p.batch, (p.w + 63) / 64, slots);
  }
  const int64_t t = (p.h + SIMT_BM - 1) / SIMT_BM;
  return simt_pick_splits(static_cast<int>(t * (t + 1) / 2), static_cast<int>(p.batch), static_cast<int>(p.w));
}

// int8 digit-engine buffers (fp32 mode, h > 256): X digit planes [S][B][h][round_up(w, 64)] (Gram
// operand) or [S][B][w][round_up(h, 64)] (apply / NS update operand) -- one buffer, used in turn; the
// h x h digit planes (C_k, P, G or the NS operator); per-row maxima of both operands.
static void take_oz(Plan& pl, const Problem& p) {
  const int64_t B = p.batch;
  const int64_t xa = p.h * round_up(p.w, 64), xb = p.w * round_up(p.h, 64);
  pl.ozX_plane = B * std::max(xa, xb);
  pl.ozX = take(pl, static_cast<size_t>(OZ_S * pl.ozX_plane));
  pl.ozC_plane = B * pl.hh;
  pl.ozC = take(pl, static_cast<size_t>(OZ_S * pl.ozC_plane));
  pl.ozMaxA_bs = std::max(p.w, p.h);
  pl.ozMaxA = take(pl, static_cast<size_t>(B * pl.ozMaxA_bs) * 8);
  pl.ozMaxB = take(pl, static_cast<size_t>(B * p.h) * 8);
}

static Plan make_plan(const Problem& p, bool with_gram, bool for_error = false) {
  Plan pl;
  pl.ldc = round_up(p.h, 256);
  pl.hh = p.h * pl.ldc;
  const int64_t B = p.batch;
  const bool bf = !for_error && p.prec == UNSO_PREC_BF16;
  const size_t ge = bf ? 4 : 8;  // Gram element size
  pl.splits = with_gram ? gram_splits(p, for_error) : 1;
  pl.scal = take(pl, static_cast<size_t>(B) * SCAL_STRIDE * 8);  // first: same offset for every plan
  pl.ldx = p.ld;
  pl.xcopy = false;
  if (bf) {
    pl.xcopy = p.dt != UNSO_DTYPE_BF16 || (p.ld % 8) != 0 || (p.batch > 1 && (p.bs % 8) != 0);
    if (pl.xcopy) {
      pl.ldx = round_up(p.cols, 8);
      pl.xb = take(pl, static_cast<size_t>(B * p.rows * pl.ldx) * 2);
    }
  }
  if (with_gram) pl.part = take(pl, static_cast<size_t>(pl.splits) * B * pl.hh * ge);
  pl.G = take(pl, static_cast<size_t>(B * pl.hh) * ge);
  pl.blk = take(pl, static_cast<size_t>(B) * NORM_BLOCKS * 3 * 8);
  if (for_error) return pl;
  if (p.scaling == UNSO_SCALING_GELFAND && p.gpow > 1) {
    pl.Gk[0] = take(pl, static_cast<size_t>(B * pl.hh) * 8);
    pl.Gk[1] = take(pl, static_cast<size_t>(B * pl.hh) * 8);
  }
  if (p.method == UNSO_METHOD_UNSO) {
    if (bf) {
      for (int i = 0; i < 2; ++i) {
        pl.Chi[i] = take(pl, static_cast<size_t>(B * pl.hh) * 2);
        pl.Clo[i] = take(pl, static_cast<size_t>(B * pl.hh) * 2);
      }
      pl.P = take(pl, static_cast<size_t>(B * pl.hh) * 4);
      pl.Phi = take(pl, static_cast<size_t>(B * pl.hh) * 2);
      pl.Plo = take(pl, static_cast<size_t>(B * pl.hh) * 2);
      const int64_t nt = (p.h + 127) / 128;
      pl.normbuf = take(pl, static_cast<size_t>(nt * (nt + 1) / 2 * B) * 2 * 8);
      pl.pstat = take(pl, static_cast<size_t>(nt * (nt + 1) / 2 * B) * 2 * 8);
      // multi-launch pipeline partials: per (pair tile, 32-row group, 32-col chunk), or per 32x32 tile
      const int64_t nt2 = (p.h + 255) / 256, nt32 = (p.h + 31) / 32;
      const int64_t slots = nt2 * (nt2 + 1) / 2 * 64;
      const int64_t nrm = slots > nt32 * (nt32 + 1) / 2 ? slots : nt32 * (nt32 + 1) / 2;
      pl.mnorm = take(pl, static_cast<size_t>(B * nrm) * 3 * 8);
      pl.mpstat = take(pl, static_cast<size_t>(B * slots) * 2 * 8);
      for (int i = 0; i < 2; ++i) {
        pl.C8h[i] = take(pl, static_cast<size_t>(B * pl.hh));
        pl.C8l[i] = take(pl, static_cast<size_t>(B * pl.hh));
        pl.C8i[i] = take(pl, static_cast<size_t>(B * pl.hh) * 2);
      }
      pl.gbar = take(pl, CH_SLOTS * CHAIN_ROUNDS * 8);  // persistent chain: one set of rounds per matrix group
    } else {
      pl.C[0] = take(pl, static_cast<size_t>(B * pl.hh) * 8);
      pl.C[1] = take(pl, static_cast<size_t>(B * pl.hh) * 8);
      pl.P = take(pl, static_cast<size_t>(B * pl.hh) * 8);
      pl.Pout = take(pl, static_cast<size_t>(B * pl.hh) * 8);
      pl.gbar = take(pl, CHAIN_ROUNDS * 8);  // chain_f64_kernel rounds and phase-A partials
      const int64_t nt16 = (p.h + 15) / 16;
      pl.normbuf = take(pl, static_cast<size_t>(nt16 * (nt16 + 1) / 2 * B) * 2 * 8);
      if (use_oz(p)) take_oz(pl, p);
    }
  } else if (bf) {
    // NS in BF16: fp32 state ping-pong + bf16 operand copy (always), G hi/lo, operator B (P), B hi/lo
    if (!pl.xcopy) {
      pl.xcopy = true;
      pl.ldx = round_up(p.cols, 8);
      pl.xb = take(pl, static_cast<size_t>(B * p.rows * pl.ldx) * 2);
    }
    pl.xb2 = take(pl, static_cast<size_t>(B * p.rows * pl.ldx) * 2);
    if ((p.flags & UNSO_FLAG_NS_SINGLE_STATE) == 0) {
      pl.xl[0] = take(pl, static_cast<size_t>(B * p.rows * pl.ldx) * 2);
      pl.xl[1] = take(pl, static_cast<size_t>(B * p.rows * pl.ldx) * 2);
    }
    pl.Xs[0] = take(pl, static_cast<size_t>(B * p.rows * p.cols) * 4);
    pl.Xs[1] = take(pl, static_cast<size_t>(B * p.rows * p.cols) * 4);
    pl.Chi[0] = take(pl, static_cast<size_t>(B * pl.hh) * 2);
    pl.Clo[0] = take(pl, static_cast<size_t>(B * pl.hh) * 2);
    pl.P = take(pl, static_cast<size_t>(B * pl.hh) * 4);
    pl.Phi = take(pl, static_cast<size_t>(B * pl.hh) * 2);
    pl.Plo = take(pl, static_cast<size_t>(B * pl.hh) * 2);
    pl.normbuf = take(pl, static_cast<size_t>(B) * SCAL_STRIDE * 8);  // unit scalars for finalize_p
  } else {
    pl.Xs[0] = take(pl, static_cast<size_t>(B * p.rows * p.cols) * 8);
    pl.Xs[1] = take(pl, static_cast<size_t>(B * p.rows * p.cols) * 8);
    pl.C[0] = take(pl, static_cast<size_t>(B * pl.hh) * 8);  // quintic operator B
    if (use_oz(p)) take_oz(pl, p);
  }
  return pl;
}

template <typename T>
static T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

static int grid_for(int64_t n, int per_block = 256, int max_blocks = 148 * 8) {
  int64_t g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return static_cast<int>(g);
}

// ==================================================================== stages
// Gram partials of X (orientation per p.tall) with fp64 accumulation -> part (f64).
static int32_t gram_simt(const Problem& p, const void* x, int dt, int64_t ld, int64_t bs, const Plan& pl, void* ws,
                         int splits, cudaStream_t st) {
  SimtOperand X{x, ld, bs, dt, p.tall ? 0 : 1};
  EpiPartialF64 epi{at<double>(ws, pl.part), pl.hh, pl.ldc, static_cast<int>(p.batch)};
  if (launch_simt_gemm(X, X, static_cast<int>(p.h), static_cast<int>(p.h), static_cast<int>(p.w),
                       static_cast<int>(p.batch), true, splits, epi, st) != cudaSuccess)
    return UNSO_ERR_CUDA;
  ++g_launches;
  return UNSO_OK;
}

// Split-K partials -> symmetric G, in the padded workspace layout (gld = 0) or a dense (gld, gbs) buffer.
template <typename T>
static int32_t finalize_gram(const Problem& p, const Plan& pl, void* ws, int splits, T* G, cudaStream_t st,
                             int64_t gld = 0, int64_t gbs = 0) {
  const int nt = static_cast<int>((p.h + 31) / 32);
  dim3 grid(nt * (nt + 1) / 2, static_cast<unsigned>(p.batch));
  finalize_sum_kernel<T><<<grid, 256, 0, st>>>(at<T>(ws, pl.part), splits, static_cast<int>(p.batch),
                                                static_cast<int>(p.h), pl.ldc, G, gld ? gld : pl.ldc,
                                                gld ? gbs : pl.hh);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

template <typename T>
static int32_t norms_and_scalars(const Problem& p, const Plan& pl, void* ws, const T* G, int mode, int32_t* status,
                                 cudaStream_t st) {
  const int nb = norm_blocks(p.h * p.h);
  dim3 grid(nb, static_cast<unsigned>(p.batch));
  gram_norms_kernel<T><<<grid, 256, 0, st>>>(G, static_cast<int>(p.h), pl.ldc, at<double>(ws, pl.blk));
  UNSO_CHECK_LAUNCH();
  scalars_kernel<<<static_cast<unsigned>(p.batch), 256, 0, st>>>(at<double>(ws, pl.blk), nb, mode, p.gpow,
                                                                  at<double>(ws, pl.scal), status);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

// Gelfand denominator ||G^k||_F^(1/2k) (ortho.py:158-163): powers on the fp64 engine.
template <typename T>
static int32_t gelfand_scale(const Problem& p, const Plan& pl, void* ws, const T* G, int gdt, int32_t* status,
                             cudaStream_t st) {
  if (p.gpow <= 1) return UNSO_OK;  // k = 1: ||G||_F^(1/2) == gram scaling, already computed
  const int h = static_cast<int>(p.h);
  SimtOperand Gop{G, pl.ldc, pl.hh, gdt, 1};
  const void* prev = G;
  int prev_dt = gdt;
  int cur = 0;
  for (int j = 2; j <= p.gpow; ++j) {
    SimtOperand A{prev, pl.ldc, pl.hh, prev_dt, 1};
    EpiOut epi{at<double>(ws, pl.Gk[cur]), DT_F64, pl.ldc, pl.hh, nullptr, 0, 0, 1.0, 0.0};
    if (launch_simt_gemm(A, Gop, h, h, h, static_cast<int>(p.batch), false, 1, epi, st) != cudaSuccess)
      return UNSO_ERR_CUDA;
    ++g_launches;
    prev = at<double>(ws, pl.Gk[cur]);
    prev_dt = DT_F64;
    cur ^= 1;
  }
  const int nb = norm_blocks(p.h * p.h);
  dim3 grid(nb, static_cast<unsigned>(p.batch));
  gram_norms_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(prev), h, pl.ldc, at<double>(ws, pl.blk));
  UNSO_CHECK_LAUNCH();
  scalars_kernel<<<static_cast<unsigned>(p.batch), 256, 0, st>>>(at<double>(ws, pl.blk), nb, SM_GELFAND,
                                                                  p.gpow, at<double>(ws, pl.scal), status);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

// ---------------------------------------------------------------- FP32 mode: int8 tensor-core engine
// 4-D map over the digit planes: {K, rows, batch, digit}, box {64, box_rows, 1, OZ_S}, SWIZZLE_64B --
// one TMA instruction stages all digit planes of a 64-byte k-block (ozaki_i8.cuh).
static bool oz_map(CUtensorMap* m, const int8_t* base, int64_t k, int64_t rows, int64_t batch, int64_t ld, int64_t bs,
                   int64_t plane, int box_rows) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(batch), static_cast<cuuint64_t>(OZ_S)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(batch > 1 ? bs : rows * ld),
                                 static_cast<cuuint64_t>(plane)};
  const cuuint32_t box[4] = {static_cast<cuuint32_t>(OZ_BK), static_cast<cuuint32_t>(box_rows), 1u,
                             static_cast<cuuint32_t>(OZ_S)};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Digit planes of one operand: operand row = source row (transpose = false) or source column
// (true); maxbuf[b * max_bs + operand row] receives the row's max |a| first.
static int32_t oz_slice(const void* src, int dt, int64_t ld, int64_t bs, int64_t rows, int64_t cols, int64_t batch,
                        bool transpose, unsigned long long* maxbuf, int64_t max_bs, int8_t* dst, int64_t ldd,
                        int64_t dbs, int64_t plane, cudaStream_t st) {
  if (!transpose) {
    dim3 g(static_cast<unsigned>(std::min<int64_t>((rows + 7) / 8, 148 * 16)), static_cast<unsigned>(batch));
    oz_rowmax_kernel<<<g, 256, 0, st>>>(src, dt, ld, bs, rows, cols, static_cast<int>(batch), maxbuf, max_bs);
    UNSO_CHECK_LAUNCH();
  } else {
    if (cudaMemsetAsync(maxbuf, 0, static_cast<size_t>(batch * max_bs) * 8, st) != cudaSuccess) return UNSO_ERR_CUDA;
    const int rpb = 256;
    dim3 g(static_cast<unsigned>((cols + 255) / 256), static_cast<unsigned>((rows + rpb - 1) / rpb),
           static_cast<unsigned>(batch));
    oz_colmax_kernel<<<g, 256, 0, st>>>(src, dt, ld, bs, rows, cols, maxbuf, max_bs, rpb);
    UNSO_CHECK_LAUNCH();
  }
  dim3 g(static_cast<unsigned>((cols + 63) / 64), static_cast<unsigned>((rows + 63) / 64), static_cast<unsigned>(batch));
  oz_split_kernel<<<g, 256, 0, st>>>(src, dt, ld, bs, rows, cols, transpose ? 1 : 0, maxbuf, max_bs, dst, ldd, dbs,
                                     plane);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

struct OzOperand {
  const int8_t* planes;
  int64_t ld, bs, plane;                 // bytes
  const unsigned long long* maxbits;     // per operand row
  int64_t max_bs;
};

// D[b](m, n) = sum_k A[b](m, k) B[b](n, k) through the digit planes; SYRK keeps n >= m.
template <class Epi>
static int32_t oz_gemm(const OzOperand& A, const OzOperand& B, int64_t M, int64_t N, int64_t K, int64_t batch,
                       bool syrk, int splits, const Epi& epi, cudaStream_t st) {
  static PerDeviceFlag configured;
  const int cfg_dev = PerDeviceFlag::current();
  if (!configured.test(cfg_dev)) {
    if (cudaFuncSetAttribute(oz_gemm_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM) != cudaSuccess)
      return UNSO_ERR_CUDA;
    configured.set(cfg_dev);
  }
  OzWork w;
  w.tiles_m = static_cast<int>((M + OZ_BM - 1) / OZ_BM);
  w.tiles_n = static_cast<int>((N + OZ_BN - 1) / OZ_BN);
  w.syrk = syrk ? 1 : 0;
  w.k_tiles = static_cast<int>((K + OZ_BK - 1) / OZ_BK);
  w.splits = std::max(1, std::min(splits, w.k_tiles));
  if ((K + w.splits - 1) / w.splits > OZ_MAX_K) return UNSO_ERR_UNSUPPORTED;  // int32 accumulator bound
  w.batch = static_cast<int>(batch);
  static const int oz_dbg = dev_override("UNSO_OZ_DEBUG") ? std::atoi(dev_override("UNSO_OZ_DEBUG")) : 0;
  w.dbg = oz_dbg;
  w.tiles_per_mat = static_cast<int>(syrk ? oz_syrk_tiles(M) : static_cast<int64_t>(w.tiles_m) * w.tiles_n);
  const int64_t nw = static_cast<int64_t>(w.tiles_per_mat) * w.splits * batch;
  if (nw <= 0) return UNSO_OK;
  if (nw > (1ll << 31) - 1) return UNSO_ERR_UNSUPPORTED;
  w.num_work = static_cast<int>(nw);
  CUtensorMap ta, tb;  // each CTA of a pair stages 128 A rows and OZ_HB B rows
  if (!oz_map(&ta, A.planes, K, M, batch, A.ld, A.bs, A.plane, 128) ||
      !oz_map(&tb, B.planes, K, N, batch, B.ld, B.bs, B.plane, OZ_HB))
    return UNSO_ERR_CUDA;
  OzScales sc{A.maxbits, A.max_bs, B.maxbits, B.max_bs, static_cast<int>(M), static_cast<int>(N)};
  const int pairs = static_cast<int>(std::min<int64_t>(nw, device_sm_count() / 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  cfg.blockDim = dim3(OZ_THREADS);
  cfg.dynamicSmemBytes = OZ_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, oz_gemm_kernel<Epi>, ta, tb, w, sc, epi) != cudaSuccess) return UNSO_ERR_CUDA;
  ++g_launches;
  return UNSO_OK;
}

// Gram split-K partials of X on the int8 engine (the fp64 partial layout of gram_simt); the source
// may be the input (dt, ld, bs of the problem) or an fp64 NS state.
static int32_t gram_oz(const Problem& p, const void* x, const Plan& pl, void* ws, int splits, cudaStream_t st,
                       int dt = -1, int64_t ld = -1, int64_t bs = -1) {
  if (dt < 0) {
    dt = p.dt;
    ld = p.ld;
    bs = p.bs;
  }
  int8_t* planes = at<int8_t>(ws, pl.ozX);
  unsigned long long* mx = at<unsigned long long>(ws, pl.ozMaxA);
  const int64_t ldd = round_up(p.w, 64), dbs = p.h * ldd;
  // operand rows = the h short-side vectors: columns of a tall X, rows of a wide one
  UNSO_TRY(oz_slice(x, dt, ld, bs, p.rows, p.cols, p.batch, p.tall, mx, pl.ozMaxA_bs, planes, ldd, dbs,
                    pl.ozX_plane, st));
  const OzOperand X{planes, ldd, dbs, pl.ozX_plane, mx, pl.ozMaxA_bs};
  OzEpiPartial epi{at<double>(ws, pl.part), pl.hh, pl.ldc, static_cast<int>(p.batch)};
  return oz_gemm(X, X, p.h, p.h, p.w, p.batch, true, splits, epi, st);
}

static int32_t gram_fp32(const Problem& p, const void* x, const Plan& pl, void* ws, int splits, cudaStream_t st) {
  if (use_oz(p)) return gram_oz(p, x, pl, ws, splits, st);
  return gram_simt(p, x, p.dt, p.ld, p.bs, pl, ws, splits, st);
}

static int scal_mode(int scaling) {
  return scaling == UNSO_SCALING_PLAIN ? SM_PLAIN : (scaling == UNSO_SCALING_NONE ? SM_NONE : SM_GRAM);
}

// ---------------------------------------------------------------- UNSO, FP32 precision
// h <= 256: all squarings in one cooperative launch per co-resident batch chunk (chain_f64.cuh).
// Returns false when the problem does not qualify (the caller then runs the per-step launches).
static bool chain_f64_persistent(const Problem& p, const Plan& pl, void* ws, const double* G, int32_t* status,
                                 cudaStream_t st) {
  static const bool no_f64_chain = dev_override("UNSO_NO_F64_CHAIN") != nullptr;  // developer override, read once
  // rows are pulled with 16-byte-granular bulk copies: h must be even
  if (p.h > CF_MAX_H || (p.h & 1) || p.order < 2 || p.order > CHAIN_MAX_ORDER ||
      p.scaling == UNSO_SCALING_GELFAND || no_f64_chain)
    return false;
  const int h = static_cast<int>(p.h);
  const int T = cf_tile(h);
  const int smem = cf_smem_bytes(h, T);
  auto kernel = T == 16 ? chain_f64_kernel<16> : chain_f64_kernel<32>;
  static PerDeviceFlag configured;
  const int cfg_dev = PerDeviceFlag::current();
  if (!configured.test(cfg_dev)) {
    if (cudaFuncSetAttribute(chain_f64_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             cf_smem_bytes(128, 16)) != cudaSuccess ||
        cudaFuncSetAttribute(chain_f64_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             cf_smem_bytes(CF_MAX_H, 32)) != cudaSuccess)
      return false;
    configured.set(cfg_dev);
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 128, smem) != cudaSuccess || per_sm < 1)
    return false;
  ChainF64Params cp;
  std::memset(&cp, 0, sizeof(cp));
  cp.G = G;
  cp.normbuf = at<double>(ws, pl.normbuf);
  cp.status = status;
  cp.scal_mode = scal_mode(p.scaling);
  cp.alpha = 1.0;
  for (double v : p.co) cp.alpha += v;
  cp.C[0] = at<double>(ws, pl.C[0]);
  cp.C[1] = at<double>(ws, pl.C[1]);
  cp.P = at<double>(ws, pl.P);
  cp.ld = pl.ldc;
  cp.mat = pl.hh;
  cp.h = h;
  cp.nt = (h + T - 1) / T;
  cp.tiles_per_mat = cp.nt * (cp.nt + 1) / 2;
  cp.order = p.order;
  cp.gbar = at<unsigned long long>(ws, pl.gbar);
  cp.scal = at<double>(ws, pl.scal);
  cp.trunc_tau = (p.flags & UNSO_FLAG_NO_TRUNCATION) ? 0.0 : std::ldexp(1.0, -30);
  for (int k = 0; k < p.order; ++k) cp.coef[k] = p.co[k];
  for (int k = 0; k <= p.order && k < CHAIN_MAX_ORDER; ++k) {
    for (int j = k + 1; j <= p.order; ++j) {
      cp.tail[k] += p.co[j - 1];
    }
  }
  const int cap = std::min(per_sm * device_sm_count(), CF_MAX_GRID);
  if (cap < cp.tiles_per_mat) return false;
  const int per = cap / cp.tiles_per_mat;
  for (int b0 = 0; b0 < static_cast<int>(p.batch); b0 += per) {
    const int nb = std::min(per, static_cast<int>(p.batch) - b0);
    cp.b0 = b0;
    if (cudaMemsetAsync(cp.gbar, 0, CHAIN_ROUNDS * sizeof(unsigned long long), st) != cudaSuccess) return false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(cp.tiles_per_mat * nb));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kernel, cp) != cudaSuccess) return false;
    ++g_launches;
  }
  return true;
}

static int32_t unso_fp32_from_G(const Problem& p, const Plan& pl, void* ws, const void* x, const double* G, void* y,
                                int32_t* status, cudaStream_t st) {
  const int h = static_cast<int>(p.h);
  const int N = p.order;
  if (chain_f64_persistent(p, pl, ws, G, status, st)) {  // norms, C_1 and the whole chain in one launch
    prof_mark(3, st);
    prof_mark(4, st);
  } else {
  UNSO_TRY(norms_and_scalars<double>(p, pl, ws, G, scal_mode(p.scaling), status, st));
  if (p.scaling == UNSO_SCALING_GELFAND) UNSO_TRY(gelfand_scale<double>(p, pl, ws, G, DT_F64, status, st));
  double alpha = 1.0;
  for (double v : p.co) alpha += v;
  if (use_oz(p)) {
    // int8 engine: per squaring one SYRK on C_k's digit planes writing S = C_k^2 (stores only),
    // then one fused row kernel: C_{k+1} = 2 C_k - S, P -= c_{k+1} C_{k+1}, row max + digit planes.
    OzStepParams sp;
    sp.S = at<double>(ws, pl.Pout);  // scratch for S until finalize_p
    sp.P = at<double>(ws, pl.P);
    sp.scal = at<double>(ws, pl.scal);
    sp.alpha = alpha;
    sp.h = h;
    sp.ld = pl.ldc;
    sp.bs = pl.hh;
    sp.maxbits = at<unsigned long long>(ws, pl.ozMaxB);
    sp.plane = pl.ozC_plane;
    const dim3 rgrid(static_cast<unsigned>(std::min<int64_t>((h + 7) / 8, 148 * 16)), static_cast<unsigned>(p.batch));
    sp.mode = 0;
    sp.src = G;
    sp.Cn = at<double>(ws, pl.C[0]);
    sp.coef = p.co[0];
    sp.digits = N > 1 ? at<int8_t>(ws, pl.ozC) : nullptr;
    oz_chain_step_kernel<<<rgrid, 256, 0, st>>>(sp);
    UNSO_CHECK_LAUNCH();
    prof_mark(3, st);
    const OzOperand C{at<int8_t>(ws, pl.ozC), pl.ldc, pl.hh, pl.ozC_plane, sp.maxbits, h};
    const OzEpiSym se{at<double>(ws, pl.Pout), pl.ldc, pl.hh};
    int cur = 0;
    for (int k = 1; k < N; ++k) {  // produces C_{k+1}
      UNSO_TRY(oz_gemm(C, C, h, h, h, p.batch, true, 1, se, st));
      sp.mode = 1;
      sp.src = at<double>(ws, pl.C[cur]);
      sp.Cn = at<double>(ws, pl.C[cur ^ 1]);
      sp.coef = p.co[k];
      sp.digits = k + 1 < N ? at<int8_t>(ws, pl.ozC) : nullptr;
      oz_chain_step_kernel<<<rgrid, 256, 0, st>>>(sp);
      UNSO_CHECK_LAUNCH();
      cur ^= 1;
    }
  } else {
  {
    dim3 grid(grid_for(static_cast<int64_t>(h) * h, 256, 1024), static_cast<unsigned>(p.batch));
    prep_f64_kernel<double><<<grid, 256, 0, st>>>(G, h, pl.ldc, at<double>(ws, pl.scal), alpha, p.co[0],
                                                  at<double>(ws, pl.C[0]), at<double>(ws, pl.P));
    UNSO_CHECK_LAUNCH();
  }
  prof_mark(3, st);
  int cur = 0;
  for (int k = 1; k < N; ++k) {  // produces C_{k+1}
    EpiChainF64 epi{at<double>(ws, pl.C[cur]), at<double>(ws, pl.C[cur ^ 1]), at<double>(ws, pl.P), pl.ldc, pl.hh,
                    p.co[k], k + 1 < N ? 1 : 0};
    SimtOperand C{at<double>(ws, pl.C[cur]), pl.ldc, pl.hh, DT_F64, 1};
    if (launch_simt_gemm(C, C, h, h, h, static_cast<int>(p.batch), true, 1, epi, st) != cudaSuccess)
      return UNSO_ERR_CUDA;
    ++g_launches;
    cur ^= 1;
  }
  }
  prof_mark(4, st);
  }
  {
    const int nt = (h + 31) / 32;
    dim3 grid(nt * (nt + 1) / 2, static_cast<unsigned>(p.batch));
    finalize_p_kernel<0><<<grid, 256, 0, st>>>(at<double>(ws, pl.P), h, pl.ldc, at<double>(ws, pl.scal),
                                               at<double>(ws, pl.Pout), nullptr);
    UNSO_CHECK_LAUNCH();
  }
  prof_mark(5, st);
  if (use_oz(p)) {  // apply on the int8 engine: tall Y = X P, wide Y = P X (P symmetric: its rows are B's)
    int8_t* pp = at<int8_t>(ws, pl.ozC);
    unsigned long long* pm = at<unsigned long long>(ws, pl.ozMaxB);
    UNSO_TRY(oz_slice(at<double>(ws, pl.Pout), DT_F64, pl.ldc, pl.hh, h, h, p.batch, false, pm, h, pp, pl.ldc, pl.hh,
                      pl.ozC_plane, st));
    const OzOperand Pd{pp, pl.ldc, pl.hh, pl.ozC_plane, pm, h};
    int8_t* xp = at<int8_t>(ws, pl.ozX);
    unsigned long long* xm = at<unsigned long long>(ws, pl.ozMaxA);
    const int64_t ldd = round_up(p.h, 64), dbs = p.w * ldd;
    // operand rows = the w long-side vectors of length h: rows of a tall X, columns of a wide one
    UNSO_TRY(oz_slice(x, p.dt, p.ld, p.bs, p.rows, p.cols, p.batch, !p.tall, xm, pl.ozMaxA_bs, xp, ldd, dbs,
                      pl.ozX_plane, st));
    const OzOperand Xd{xp, ldd, dbs, pl.ozX_plane, xm, pl.ozMaxA_bs};
    OzEpiOut epi{y, p.dt, p.cols, p.rows * p.cols};
    if (p.tall)
      UNSO_TRY(oz_gemm(Xd, Pd, p.w, h, h, p.batch, false, 1, epi, st));
    else
      UNSO_TRY(oz_gemm(Pd, Xd, h, p.w, h, p.batch, false, 1, epi, st));
    prof_mark(6, st);
    return UNSO_OK;
  }
  // apply: tall Y = X P (A = X K-major over w rows), wide Y = P X (B = X MN-major)
  SimtOperand Xop{x, p.ld, p.bs, p.dt, 1};
  SimtOperand Pop{at<double>(ws, pl.Pout), pl.ldc, pl.hh, DT_F64, 1};
  EpiOut epi{y, p.dt, p.cols, p.rows * p.cols, nullptr, 0, 0, 1.0, 0.0};
  cudaError_t e;
  if (p.tall) {
    e = launch_simt_gemm(Xop, Pop, static_cast<int>(p.rows), h, h, static_cast<int>(p.batch), false, 1, epi, st);
  } else {
    Xop.kmajor = 0;
    e = launch_simt_gemm(Pop, Xop, h, static_cast<int>(p.cols), h, static_cast<int>(p.batch), false, 1, epi, st);
  }
  if (e != cudaSuccess) return UNSO_ERR_CUDA;
  ++g_launches;
  prof_mark(6, st);
  return UNSO_OK;
}

// ---------------------------------------------------------------- UNSO, BF16 precision (tcgen05)
// Upper-triangle f32 P -> symmetric bf16 hi/lo (scaled by 1/s, shifted by d) for the apply.
static int32_t finalize_p_bf16(const Problem& p, const Plan& pl, void* ws, const double* scal, cudaStream_t st) {
  const int h = static_cast<int>(p.h);
  const int nt = (h + 63) / 64;
  dim3 grid(nt * (nt + 1) / 2, static_cast<unsigned>(p.batch));
  finalize_p_bf16_kernel<<<grid, 256, 0, st>>>(at<float>(ws, pl.P), h, pl.ldc, scal, at<__nv_bfloat16>(ws, pl.Phi),
                                               at<__nv_bfloat16>(ws, pl.Plo));
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

static int32_t ensure_bf16_x(const Problem& p, const Plan& pl, void* ws, const void* x, const __nv_bfloat16*& xb,
                             int64_t& ldx, int64_t& bsx, cudaStream_t st) {
  if (!pl.xcopy) {
    xb = static_cast<const __nv_bfloat16*>(x);
    ldx = p.ld;
    bsx = p.bs;
    return UNSO_OK;
  }
  __nv_bfloat16* dst = at<__nv_bfloat16>(ws, pl.xb);
  ldx = pl.ldx;
  bsx = p.rows * pl.ldx;
  const int64_t n = p.batch * p.rows * p.cols;
  if (p.dt == UNSO_DTYPE_F32 && p.ld == p.cols && ldx == p.cols && p.bs == p.rows * p.cols && n % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    f32_to_bf16_flat_kernel<<<grid_for(n / 8, 256, 148 * 16), 256, 0, st>>>(static_cast<const float4*>(x),
                                                                             reinterpret_cast<uint4*>(dst), n / 8);
  } else if (p.dt == UNSO_DTYPE_F32 && p.cols % 4 == 0 && p.ld % 4 == 0 && p.bs % 4 == 0 &&
             (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    f32_to_bf16_kernel<<<grid_for(n / 4), 256, 0, st>>>(static_cast<const float*>(x), p.ld, p.bs, dst, ldx, bsx,
                                                          p.rows, p.cols, static_cast<int>(p.batch));
  } else {
    convert_kernel<<<grid_for(n), 256, 0, st>>>(x, p.dt, p.ld, p.bs, dst, DT_BF16, ldx, bsx, p.rows, p.cols,
                                                static_cast<int>(p.batch), nullptr);
  }
  UNSO_CHECK_LAUNCH();
  xb = dst;
  return UNSO_OK;
}

// Gram launches (A and B maps are the same tensor): diagonal tiles share one operand copy (umma2_gemm.cuh).
static UmmaWork gram_work2(int M, int N, int K, int BN, int batch, int splits) {
  UmmaWork w = umma2_make_work(M, N, K, BN, batch, true, splits);
  w.diag_share = 1;
  return w;
}

static int32_t gram_bf16(const Problem& p, const Plan& pl, void* ws, const __nv_bfloat16* xb, int64_t ldx,
                         int64_t bsx, cudaStream_t st) {
  CUtensorMap mx;
  UmmaWork w = umma_make_work(static_cast<int>(p.h), static_cast<int>(p.h), static_cast<int>(p.w), 128,
                              static_cast<int>(p.batch), true, pl.splits);
  UEpiPartialF32 epi{at<float>(ws, pl.part), pl.hh, pl.ldc, static_cast<int>(p.batch), static_cast<int>(p.h)};
  cudaError_t e;
  const bool pair = use_pair_engine();
  const UmmaWork w2 = gram_work2(static_cast<int>(p.h), static_cast<int>(p.h), static_cast<int>(p.w), 256,
                                 static_cast<int>(p.batch), pl.splits);
  if (p.tall) {
    if (!umma_make_mnmajor_map(&mx, xb, p.rows, p.cols, ldx, p.batch, bsx)) return UNSO_ERR_CUDA;
    e = pair ? launch_umma2<Cfg2GramMN>(mx, mx, mx, mx, w2, epi, st) : launch_umma<CfgGramMN>(mx, mx, mx, mx, w, epi, st);
  } else {
    if (!umma_make_kmajor_map(&mx, xb, p.rows, p.cols, ldx, p.batch, bsx, 128)) return UNSO_ERR_CUDA;
    e = pair ? launch_umma2<Cfg2GramK>(mx, mx, mx, mx, w2, epi, st) : launch_umma<CfgGramK>(mx, mx, mx, mx, w, epi, st);
  }
  if (e != cudaSuccess) return UNSO_ERR_CUDA;
  ++g_launches;
  return UNSO_OK;
}

// K1 writing G straight into the chain's bf16 hi/lo state + norm partials (CTA pairs, no split-K).
static int32_t gram_bf16_split(const Problem& p, const Plan& pl, void* ws, const __nv_bfloat16* xb, int64_t ldx,
                               int64_t bsx, cudaStream_t st) {
  CUtensorMap mx;
  const int nt2 = static_cast<int>((p.h + 255) / 256);
  UEpiGramSplit epi{at<__nv_bfloat16>(ws, pl.Chi[0]), at<__nv_bfloat16>(ws, pl.Clo[0]), at<double>(ws, pl.mnorm),
                    pl.ldc, pl.hh, static_cast<int>(p.h), nt2};
  const UmmaWork w2 = gram_work2(static_cast<int>(p.h), static_cast<int>(p.h), static_cast<int>(p.w), 256,
                                 static_cast<int>(p.batch), 1);
  cudaError_t e;
  if (p.tall) {
    if (!umma_make_mnmajor_map(&mx, xb, p.rows, p.cols, ldx, p.batch, bsx)) return UNSO_ERR_CUDA;
    e = launch_umma2<Cfg2GramMN>(mx, mx, mx, mx, w2, epi, st);
  } else {
    if (!umma_make_kmajor_map(&mx, xb, p.rows, p.cols, ldx, p.batch, bsx, 128)) return UNSO_ERR_CUDA;
    e = launch_umma2<Cfg2GramK>(mx, mx, mx, mx, w2, epi, st);
  }
  if (e != cudaSuccess) return UNSO_ERR_CUDA;
  ++g_launches;
  return UNSO_OK;
}

constexpr int CHAIN_HI_ONLY_STEPS = 3;
// developer overrides (A/B timing and precision): cross terms in every squaring; another count
static const bool g_dev_cross_all = dev_override("UNSO_CHAIN_CROSS_ALL") != nullptr;
static const int g_dev_hi_only = dev_override("UNSO_CHAIN_HI_ONLY_STEPS") ? std::atoi(dev_override("UNSO_CHAIN_HI_ONLY_STEPS")) : -1;  // clamped at use

// Multi-launch pipeline for large h (multi_chain.cuh): scalars from the norm partials, N-1 CTA-pair
// squaring steps (the first folds C_1 = G/s^2 and initialises P, the last emits P statistics),
// the adaptive-apply decision and the shifted symmetric P.  Requires C hi/lo[0] = split(G) and
// the partials in pl.mnorm (nnorm per matrix).
static int32_t scale_chain_bf16_glue_free(const Problem& p, const Plan& pl, void* ws, int nnorm, int32_t* status,
                                          cudaStream_t st) {
  const int h = static_cast<int>(p.h);
  const int N = p.order;
  const int nt2 = (h + 255) / 256;
  scalars_kernel<<<static_cast<unsigned>(p.batch), 256, 0, st>>>(at<double>(ws, pl.mnorm), nnorm,
                                                                  scal_mode(p.scaling), p.gpow,
                                                                  at<double>(ws, pl.scal), status);
  UNSO_CHECK_LAUNCH();
  prof_mark(3, st);
  double alpha = 1.0;
  for (double v : p.co) alpha += v;
  const UmmaWork wc2 = umma2_make_work(h, h, h, 256, static_cast<int>(p.batch), true, 1);
  const bool f8 = (p.flags & UNSO_FLAG_CHAIN_BF16X3) == 0;
  // The first CHAIN_HI_ONLY_STEPS squarings of the default (bf16 + e4m3) recipe take the hi*hi
  // product alone (shipped-order chains only): an error there is damped by the later squarings,
  // whereas the last squarings (largest coefficients) need the cross terms
  // (tools/chain_precision_emulation.py: 2.6-2.7e-3 -> 2.7-3.3e-3 on the cfg2/3/5-like spectra;
  // dropping them in the LAST step instead gives 2-7e-2).
  const int hi_only_steps =
      (f8 && N >= 12 && !g_dev_cross_all) ? (g_dev_hi_only >= 0 ? std::min(g_dev_hi_only, N - 1) : CHAIN_HI_ONLY_STEPS) : 0;
  int cur = 0;
  bool p_pending = false;
  for (int k = 1; k < N; ++k) {
    SymMaps maps;
    const void* hi = at<__nv_bfloat16>(ws, pl.Chi[cur]);
    const void* lo = at<__nv_bfloat16>(ws, pl.Clo[cur]);
    if (!umma_make_kmajor_map(&maps.hiK, hi, h, h, pl.ldc, p.batch, pl.hh, 128) ||
        !umma_make_kmajor_map(&maps.loK, lo, h, h, pl.ldc, p.batch, pl.hh, 128) ||
        !umma_make_mnmajor_map(&maps.hiMN, hi, h, h, pl.ldc, p.batch, pl.hh) ||
        !umma_make_mnmajor_map(&maps.loMN, lo, h, h, pl.ldc, p.batch, pl.hh))
      return UNSO_ERR_CUDA;
    const bool last = k + 1 == N;
    EpiChainStep epi{at<__nv_bfloat16>(ws, pl.Chi[cur]), at<__nv_bfloat16>(ws, pl.Clo[cur]),
                     at<__nv_bfloat16>(ws, pl.Chi[cur ^ 1]), at<__nv_bfloat16>(ws, pl.Clo[cur ^ 1]),
                     at<float>(ws, pl.P), pl.ldc, pl.hh, h, nt2, static_cast<float>(p.co[k]), last ? 0 : 1,
                     k == 1 ? 1 : 0, static_cast<float>(p.co[0]), alpha, at<double>(ws, pl.scal),
                     last ? at<double>(ws, pl.mpstat) : nullptr};
    if (f8 && !last) {  // produce the e4m3 operand copies (and the 2^12-scaled bf16 hi) of C_{k+1}
      epi.out_hi_scale = 4096.f;
      if (k + 1 > hi_only_steps) {  // step k + 1 reads them
        epi.n8hi = at<uint8_t>(ws, pl.C8h[cur ^ 1]);
        epi.n8lo = at<uint8_t>(ws, pl.C8l[cur ^ 1]);
        epi.n8i = at<uint8_t>(ws, pl.C8i[cur ^ 1]);
        epi.ld8i = 2 * pl.ldc;
      }
    }
    if (f8 && k > 1) epi.in_hi_scale = 1.f / 4096.f;
    // P is updated every other step (a_k C_k + a_{k+1} C_{k+1} in one read-modify-write)
    epi.write_p = (k == 1 || (k & 1) || last) ? 1 : 0;
    epi.coefk = p_pending ? static_cast<float>(p.co[k - 1]) : 0.f;
    p_pending = epi.write_p == 0;
    cudaError_t le;
    UmmaWork wk = wc2;
    wk.no_cross = k <= hi_only_steps ? 1 : 0;
    if (f8 && k > 1) {  // C_k is scaled (|C| <= 1): hi*hi in bf16 + e4m3 cross terms
      SymMapsF8 m8;
      m8.hiK = maps.hiK;
      m8.hiMN = maps.hiMN;
      const void* h8 = at<uint8_t>(ws, pl.C8h[cur]);
      const void* l8 = at<uint8_t>(ws, pl.C8l[cur]);
      const void* i8 = at<uint8_t>(ws, pl.C8i[cur]);
      if (!make_map_u8(&m8.f8K, i8, 2 * pl.ldc, h, p.batch, 2 * pl.ldc, 2 * pl.hh, 128, 128) ||
          !make_map_u8(&m8.h8MN, h8, h, h, p.batch, pl.ldc, pl.hh, 128, 64) ||
          !make_map_u8(&m8.l8MN, l8, h, h, p.batch, pl.ldc, pl.hh, 128, 64))
        return UNSO_ERR_CUDA;
      le = launch_chain_pair_f8(m8, wk, epi, st);
    } else {
      le = launch_chain_pair(maps, wk, epi, st);
    }
    if (le != cudaSuccess) return UNSO_ERR_CUDA;
    ++g_launches;
    cur ^= 1;
  }
  prof_mark(4, st);
  const int adaptive = ((p.flags & UNSO_FLAG_TWO_TERM_APPLY) == 0 && p.scaling != UNSO_SCALING_NONE) ? 1 : 0;
  apply_decision_kernel<<<static_cast<unsigned>(p.batch), 256, 0, st>>>(at<double>(ws, pl.mpstat),
                                                                         nt2 * (nt2 + 1) / 2 * 64,
                                                                         at<double>(ws, pl.scal), h, adaptive, 5e-3);
  UNSO_CHECK_LAUNCH();
  UNSO_TRY(finalize_p_bf16(p, pl, ws, at<double>(ws, pl.scal), st));
  prof_mark(5, st);
  return UNSO_OK;
}

static int32_t apply_bf16(const Problem& p, const Plan& pl, void* ws, const __nv_bfloat16* xb, int64_t ldx,
                          int64_t bsx, void* y, cudaStream_t st) {
  const int h = static_cast<int>(p.h);
  const bool force1 = (p.flags & UNSO_FLAG_SINGLE_TERM_APPLY) != 0;
  const bool force2 = (p.flags & UNSO_FLAG_TWO_TERM_APPLY) != 0;
  CUtensorMap mx, mph, mpl;
  if (!umma_make_kmajor_map(&mph, at<__nv_bfloat16>(ws, pl.Phi), h, h, pl.ldc, p.batch, pl.hh, 128) ||
      !umma_make_kmajor_map(&mpl, at<__nv_bfloat16>(ws, pl.Plo), h, h, pl.ldc, p.batch, pl.hh, 128))
    return UNSO_ERR_CUDA;
  const int ydt = p.dt;  // unso_dtype and Dtype share their values
  cudaError_t e = cudaSuccess;
  // Tiny problems (a handful of 256-wide pair tiles, e.g. configs[0]) launch faster on the 1-CTA
  // engine (no cluster setup): 12-13 us instead of 17-20 us for 512 x 128.  It has no per-matrix
  // filter, so there the adaptive choice resolves to the (more accurate) bf16x2 term pair.
  const int64_t pair_items = ((std::max(p.rows, p.cols) + 255) / 256) * ((h + 255) / 256) * p.batch;
  const bool pair = use_pair_engine() && pair_items > 8;
  const double* mode = at<double>(ws, pl.scal) + S_MODE;
  // Adaptive (default): two launches, each processing only the matrices whose device-side
  // decision matches it -- a 6-stage single-term kernel and a 4-stage bf16x2 kernel.
  auto filt = [&](UmmaWork w, int want) {
    if (!force1 && !force2) {
      w.mode_flag = mode;
      w.opt_stride = SCAL_STRIDE;
      w.mode_want = want;
    }
    return w;
  };
  if (p.tall) {
    if (!umma_make_kmajor_map(&mx, xb, p.rows, p.cols, ldx, p.batch, bsx, 128)) return UNSO_ERR_CUDA;
    UEpiOut epi{y, ydt, p.cols, p.rows * p.cols, static_cast<int>(p.rows), h, xb, ldx, bsx, at<double>(ws, pl.scal)};
    if (pair) {
      const UmmaWork wa = umma2_make_work(static_cast<int>(p.rows), h, h, 256, static_cast<int>(p.batch), false, 1);
      if (!force2) {
        e = launch_umma2<Cfg2ApplyTall1>(mx, mx, mph, mph, filt(wa, 1), epi, st);
        ++g_launches;
      }
      if (e == cudaSuccess && !force1) e = launch_umma2<Cfg2ApplyTall2>(mx, mx, mph, mpl, filt(wa, 0), epi, st);
    } else {
      const UmmaWork wa = umma_make_work(static_cast<int>(p.rows), h, h, 128, static_cast<int>(p.batch), false, 1);
      e = force1 ? launch_umma<CfgApplyTall1>(mx, mx, mph, mph, wa, epi, st)
                 : launch_umma<CfgApplyTall2>(mx, mx, mph, mpl, wa, epi, st);
    }
  } else {
    if (!umma_make_mnmajor_map(&mx, xb, p.rows, p.cols, ldx, p.batch, bsx)) return UNSO_ERR_CUDA;
    UEpiOut epi{y, ydt, p.cols, p.rows * p.cols, h, static_cast<int>(p.cols), xb, ldx, bsx, at<double>(ws, pl.scal)};
    if (pair) {
      const UmmaWork wa = umma2_make_work(h, static_cast<int>(p.cols), h, 256, static_cast<int>(p.batch), false, 1);
      if (!force2) {
        e = launch_umma2<Cfg2ApplyWide1>(mph, mph, mx, mx, filt(wa, 1), epi, st);
        ++g_launches;
      }
      if (e == cudaSuccess && !force1) e = launch_umma2<Cfg2ApplyWide2>(mph, mpl, mx, mx, filt(wa, 0), epi, st);
    } else {
      const UmmaWork wa = umma_make_work(h, static_cast<int>(p.cols), h, 128, static_cast<int>(p.batch), false, 1);
      e = force1 ? launch_umma<CfgApplyWide1>(mph, mph, mx, mx, wa, epi, st)
                 : launch_umma<CfgApplyWide2>(mph, mpl, mx, mx, wa, epi, st);
    }
  }
  if (e != cudaSuccess) return UNSO_ERR_CUDA;
  ++g_launches;
  prof_mark(6, st);
  return UNSO_OK;
}

// Multi-launch scale + chain from a finalized Gram G (large h, or gelfand scaling).
static int32_t scale_chain_bf16_multi(const Problem& p, const Plan& pl, void* ws, const float* G, int32_t* status,
                                      cudaStream_t st) {
  UNSO_TRY(norms_and_scalars<float>(p, pl, ws, G, scal_mode(p.scaling), status, st));
  if (p.scaling == UNSO_SCALING_GELFAND) UNSO_TRY(gelfand_scale<float>(p, pl, ws, G, DT_F32, status, st));
  const int h = static_cast<int>(p.h);
  const int N = p.order;
  double alpha = 1.0;
  for (double v : p.co) alpha += v;
  {
    dim3 grid(grid_for(static_cast<int64_t>(h) * h, 256, 1024), static_cast<unsigned>(p.batch));
    prep_bf16_kernel<<<grid, 256, 0, st>>>(G, h, pl.ldc, at<double>(ws, pl.scal), alpha, p.co[0],
                                           at<__nv_bfloat16>(ws, pl.Chi[0]), at<__nv_bfloat16>(ws, pl.Clo[0]),
                                           at<float>(ws, pl.P));
    UNSO_CHECK_LAUNCH();
  }
  prof_mark(3, st);
  int cur = 0;
  if (use_pair_engine()) {
    const UmmaWork wc2 = umma2_make_work(h, h, h, 256, static_cast<int>(p.batch), true, 1);
    for (int k = 1; k < N; ++k) {
      SymMaps maps;
      const void* hi = at<__nv_bfloat16>(ws, pl.Chi[cur]);
      const void* lo = at<__nv_bfloat16>(ws, pl.Clo[cur]);
      if (!umma_make_kmajor_map(&maps.hiK, hi, h, h, pl.ldc, p.batch, pl.hh, 128) ||
          !umma_make_kmajor_map(&maps.loK, lo, h, h, pl.ldc, p.batch, pl.hh, 128) ||
          !umma_make_mnmajor_map(&maps.hiMN, hi, h, h, pl.ldc, p.batch, pl.hh) ||
          !umma_make_mnmajor_map(&maps.loMN, lo, h, h, pl.ldc, p.batch, pl.hh))
        return UNSO_ERR_CUDA;
      EpiChainSym epi{at<__nv_bfloat16>(ws, pl.Chi[cur]), at<__nv_bfloat16>(ws, pl.Clo[cur]),
                      at<__nv_bfloat16>(ws, pl.Chi[cur ^ 1]), at<__nv_bfloat16>(ws, pl.Clo[cur ^ 1]),
                      at<float>(ws, pl.P), pl.ldc, pl.hh, h, static_cast<float>(p.co[k]), k + 1 < N ? 1 : 0};
      if (launch_chain_pair(maps, wc2, epi, st) != cudaSuccess) return UNSO_ERR_CUDA;
      ++g_launches;
      cur ^= 1;
    }
  }
  const UmmaWork wc = umma_make_work(h, h, h, 128, static_cast<int>(p.batch), true, 1);
  for (int k = 1; k < N && !use_pair_engine(); ++k) {
    CUtensorMap mh, ml;
    if (!umma_make_kmajor_map(&mh, at<__nv_bfloat16>(ws, pl.Chi[cur]), h, h, pl.ldc, p.batch, pl.hh, 128) ||
        !umma_make_kmajor_map(&ml, at<__nv_bfloat16>(ws, pl.Clo[cur]), h, h, pl.ldc, p.batch, pl.hh, 128))
      return UNSO_ERR_CUDA;
    UEpiChainBF16 epi{at<__nv_bfloat16>(ws, pl.Chi[cur]), at<__nv_bfloat16>(ws, pl.Clo[cur]),
                      at<__nv_bfloat16>(ws, pl.Chi[cur ^ 1]), at<__nv_bfloat16>(ws, pl.Clo[cur ^ 1]),
                      at<float>(ws, pl.P), pl.ldc, pl.hh, h, static_cast<float>(p.co[k]), k + 1 < N ? 1 : 0};
    if (launch_umma<CfgChain>(mh, ml, mh, ml, wc, epi, st) != cudaSuccess) return UNSO_ERR_CUDA;
    ++g_launches;
    cur ^= 1;
  }
  prof_mark(4, st);
  UNSO_TRY(finalize_p_bf16(p, pl, ws, at<double>(ws, pl.scal), st));
  prof_mark(5, st);
  return UNSO_OK;
}

// Can the fused persistent chain run (all tiles co-resident, order and scaling supported)?
static bool chain_persistent_fits(const Problem& p) {
  if (p.order < 1 || p.order > CHAIN_MAX_ORDER || p.scaling == UNSO_SCALING_GELFAND) return false;
  static int max_blocks[64] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
                                -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
                                -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
                                -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
  int& max_blocks_per_sm = max_blocks[PerDeviceFlag::current()];
  if (max_blocks_per_sm < 0) {
    if (cudaFuncSetAttribute(chain_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, CH_SMEM) !=
        cudaSuccess)
      return false;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, chain_persistent_kernel, 256, CH_SMEM) != cudaSuccess)
      return false;
    max_blocks_per_sm = nb;
  }
  const int64_t nt = (p.h + 127) / 128;
  const int64_t tpm = nt * (nt + 1) / 2;
  const int64_t cap = static_cast<int64_t>(max_blocks_per_sm) * device_sm_count();
  if (tpm > cap) return false;
  // batches run in co-resident chunks (up to two tiles per CTA); more than ~4 chunks is better
  // served by the multi-launch pipeline (each launch then covers the whole batch)
  const int64_t per = CH_SLOTS * (cap / tpm);
  return (p.batch + per - 1) / per <= 4;
}

constexpr int CHAIN_PERSISTENT_HI_ONLY = 0;  // A/B in DESIGN §9: 0.5 % of configs[3] for 2.4x the error, not taken

// Parameters shared by the on-chip chain kernels (chain_persistent.cuh, chain_small.cuh).
static ChainParams chain_params(const Problem& p, const Plan& pl, void* ws, const float* part, int splits,
                                int64_t part_ld, int64_t part_mat, int32_t* status) {
  const int h = static_cast<int>(p.h);
  ChainParams cp;
  std::memset(&cp, 0, sizeof(cp));
  cp.part = part;
  cp.part_ld = part_ld;
  cp.part_mat = part_mat;
  cp.splits = splits;
  cp.h = h;
  cp.nt = (h + 127) / 128;
  cp.tiles_per_mat = cp.nt * (cp.nt + 1) / 2;
  cp.batch = static_cast<int>(p.batch);
  cp.ld = pl.ldc;
  cp.mat = pl.hh;
  for (int i = 0; i < 2; ++i) {
    cp.chi[i] = at<__nv_bfloat16>(ws, pl.Chi[i]);
    cp.clo[i] = at<__nv_bfloat16>(ws, pl.Clo[i]);
  }
  cp.phi = at<__nv_bfloat16>(ws, pl.Phi);
  cp.plo = at<__nv_bfloat16>(ws, pl.Plo);
  cp.normbuf = at<double>(ws, pl.normbuf);
  cp.pstat = at<double>(ws, pl.pstat);
  // adaptive P_lo skipping needs ||X||_2 <= 1, i.e. a gram/plain-scaled input
  cp.adaptive = ((p.flags & UNSO_FLAG_TWO_TERM_APPLY) == 0 && p.scaling != UNSO_SCALING_NONE) ? 1 : 0;
  cp.tau = 5e-3;
  cp.scal = at<double>(ws, pl.scal);
  cp.status = status;
  cp.gbar = at<unsigned long long>(ws, pl.gbar);
  cp.order = p.order;
  cp.scal_mode = scal_mode(p.scaling);
  cp.alpha = 1.0;
  for (int k = 0; k < p.order; ++k) {
    cp.alpha += p.co[k];
    cp.coef[k] = static_cast<float>(p.co[k]);
  }
  // truncation (chain_persistent.cuh): tail[k] = sum_{j>k} c_j, c_j = co[j-1]
  cp.trunc_tau = (p.flags & UNSO_FLAG_NO_TRUNCATION) ? 0.0 : std::ldexp(1.0, -12);
  // hi*hi alone in the first squarings (as the large-h route): an error there is damped by the later
  // squarings; shipped-order chains only, UNSO_FLAG_CHAIN_BF16X3 keeps bf16x3 in every step
  {
    static const char* const f = dev_override("UNSO_PCHAIN_HI_ONLY");  // developer override (A/B)
    const int dflt = (p.order >= 12 && (p.flags & UNSO_FLAG_CHAIN_BF16X3) == 0) ? CHAIN_PERSISTENT_HI_ONLY : 0;
    cp.hi_only = f ? std::max(0, std::min(std::atoi(f), p.order - 1)) : dflt;
  }
  for (int k = 0; k <= p.order && k < CHAIN_MAX_ORDER; ++k) {
    double t = 0.0;
    for (int j = k + 1; j <= p.order; ++j) t += p.co[j - 1];
    cp.tail[k] = static_cast<float>(t);
  }
  return cp;
}

static int32_t scale_chain_bf16_persistent(const Problem& p, const Plan& pl, void* ws, const float* part, int splits,
                                           int64_t part_ld, int64_t part_mat, int32_t* status, cudaStream_t st) {
  const int h = static_cast<int>(p.h);
  ChainMaps maps;
  for (int buf = 0; buf < 2; ++buf) {
    const void* base[2] = {at<__nv_bfloat16>(ws, pl.Chi[buf]), at<__nv_bfloat16>(ws, pl.Clo[buf])};
    for (int hl = 0; hl < 2; ++hl) {
      if (!umma_make_kmajor_map(&maps.m[buf][hl][0], base[hl], h, h, pl.ldc, p.batch, pl.hh, 128) ||
          !umma_make_mnmajor_map(&maps.m[buf][hl][1], base[hl], h, h, pl.ldc, p.batch, pl.hh))
        return UNSO_ERR_CUDA;
    }
  }
  ChainParams cp = chain_params(p, pl, ws, part, splits, part_ld, part_mat, status);
  prof_mark(3, st);
  // co-resident chunks of the batch, one cooperative launch each (same stream: the barrier word
  // and per-tile buffers are reused after the previous chunk completes).  A chunk holds up to
  // CH_SLOTS tiles per CTA; chunks are balanced so no launch runs a nearly empty grid.
  int nb_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb_sm, chain_persistent_kernel, 256, CH_SMEM);
  const int cap = nb_sm * device_sm_count();
  const int per_max = std::max(1, CH_SLOTS * (cap / cp.tiles_per_mat));
  const int nchunks = (static_cast<int>(p.batch) + per_max - 1) / per_max;
  const int per = (static_cast<int>(p.batch) + nchunks - 1) / nchunks;
  for (int b0 = 0; b0 < static_cast<int>(p.batch); b0 += per) {
    const int nb = std::min(per, static_cast<int>(p.batch) - b0);
    cp.b0 = b0;
    cp.nb = nb;
    // one wave cannot hold the chunk: two matrix groups, slot s of every CTA in group s (whole matrices
    // per group: each group runs its own barrier rounds, chain_persistent.cuh)
    const int tiles = cp.tiles_per_mat * nb;
    const int grid = tiles <= cap ? tiles : cp.tiles_per_mat * ((nb + 1) / 2);
    if (cudaMemsetAsync(cp.gbar, 0, CH_SLOTS * CHAIN_ROUNDS * sizeof(unsigned long long), st) != cudaSuccess)
      return UNSO_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = CH_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, chain_persistent_kernel, maps, cp) != cudaSuccess) return UNSO_ERR_CUDA;
    ++g_launches;
  }
  prof_mark(4, st);
  prof_mark(5, st);
  return UNSO_OK;
}

// h <= 128: one CTA per matrix, the chain entirely on chip (chain_small.cuh).
static bool chain_small_fits(const Problem& p) {
  static const bool no_small_chain = dev_override("UNSO_NO_SMALL_CHAIN") != nullptr;  // developer override
  return p.h <= 128 && p.order >= 1 && p.order <= CHAIN_MAX_ORDER && p.scaling != UNSO_SCALING_GELFAND &&
         !no_small_chain;
}

// `xb` non-null: the kernel also computes the Gram of the tall bf16 X itself (FUSED_GRAM); `part`
// is then unused.  Otherwise phase A reads the split-K partials (or a dense reduced Gram).
static int32_t scale_chain_bf16_small(const Problem& p, const Plan& pl, void* ws, const float* part, int splits,
                                      int64_t part_ld, int64_t part_mat, int32_t* status, cudaStream_t st,
                                      const __nv_bfloat16* xb = nullptr, int64_t ldx = 0, int64_t bsx = 0) {
  static PerDeviceFlag configured;
  const int cfg_dev = PerDeviceFlag::current();
  if (!configured.test(cfg_dev)) {
    if (cudaFuncSetAttribute(chain_small_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, CS_SMEM) !=
            cudaSuccess ||
        cudaFuncSetAttribute(chain_small_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, CS_SMEM) !=
            cudaSuccess)
      return UNSO_ERR_CUDA;
    configured.set(cfg_dev);
  }
  ChainParams cp = chain_params(p, pl, ws, part, splits, part_ld, part_mat, status);
  SmallGram sg;
  std::memset(&sg, 0, sizeof(sg));
  if (xb) {
    if (!umma_make_mnmajor_map(&sg.x, xb, p.rows, p.cols, ldx, p.batch, bsx)) return UNSO_ERR_CUDA;
    sg.w = static_cast<int>(p.w);
  } else {
    prof_mark(3, st);
  }
  cp.b0 = 0;
  if (xb)
    chain_small_kernel<true><<<static_cast<unsigned>(p.batch), CS_THREADS, CS_SMEM, st>>>(cp, sg);
  else
    chain_small_kernel<false><<<static_cast<unsigned>(p.batch), CS_THREADS, CS_SMEM, st>>>(cp, sg);
  UNSO_CHECK_LAUNCH();
  ++g_launches;
  if (xb) {
    prof_mark(2, st);
    prof_mark(3, st);
  }
  prof_mark(4, st);
  prof_mark(5, st);
  return UNSO_OK;
}

// tall bf16 X with h <= 128 and few enough rows that one CTA per matrix does the Gram too
static bool small_fused_gram(const Problem& p) {
  static const bool no_fused = dev_override("UNSO_NO_FUSED_SMALL_GRAM") != nullptr;  // developer override
  return chain_small_fits(p) && p.tall && p.w <= 8192 && use_pair_engine() &&
         !no_fused;
}

// Which scale+chain implementation a BF16 UNSO problem takes.
enum Bf16Route { ROUTE_SMALL, ROUTE_PERSISTENT, ROUTE_GLUE_FREE, ROUTE_LEGACY };
static Bf16Route bf16_route(const Problem& p) {
  static const char* const route_override = dev_override("UNSO_BF16_ROUTE");  // developer override (A/B timing)
  if (const char* f = route_override) {
    if (!std::strcmp(f, "glue") && use_pair_engine() && p.order >= 2 && p.scaling != UNSO_SCALING_GELFAND)
      return ROUTE_GLUE_FREE;
    if (!std::strcmp(f, "persistent") && chain_persistent_fits(p)) return ROUTE_PERSISTENT;
  }
  if (chain_small_fits(p)) return ROUTE_SMALL;
  if (chain_persistent_fits(p)) return ROUTE_PERSISTENT;
  if (use_pair_engine() && p.order >= 2 && p.scaling != UNSO_SCALING_GELFAND) return ROUTE_GLUE_FREE;
  return ROUTE_LEGACY;
}

// Everything after the Gram: scale, chain, P, apply.  `split_done`: K1 already wrote G as
// bf16 hi/lo + norm partials (glue-free route with one split); otherwise `part` holds split-K
// fp32 partials (or the reduced Gram with splits == 1).
// `dense_ld` > 0: `part` is one dense reduced Gram per matrix (leading dimension dense_ld, used in
// place by the persistent route), otherwise it is in the padded workspace layout.
static int32_t unso_bf16_after_gram(const Problem& p, const Plan& pl, void* ws, const __nv_bfloat16* xb, int64_t ldx,
                                    int64_t bsx, const float* part, int splits, bool split_done, void* y,
                                    int32_t* status, cudaStream_t st, int64_t dense_ld = 0) {
  const Bf16Route route = bf16_route(p);
  if (dense_ld > 0 && route != ROUTE_PERSISTENT && route != ROUTE_SMALL) {  // the others read the padded layout
    float* G = at<float>(ws, pl.G);
    convert_kernel<<<grid_for(p.batch * p.h * p.h), 256, 0, st>>>(part, DT_F32, dense_ld, dense_ld * p.h, G, DT_F32,
                                                                  pl.ldc, pl.hh, p.h, p.h, static_cast<int>(p.batch),
                                                                  nullptr);
    UNSO_CHECK_LAUNCH();
    part = G;
    dense_ld = 0;
  }
  if (route == ROUTE_SMALL) {
    UNSO_TRY(scale_chain_bf16_small(p, pl, ws, part, splits, dense_ld > 0 ? dense_ld : pl.ldc,
                                    dense_ld > 0 ? dense_ld * p.h : pl.hh, status, st));
  } else if (route == ROUTE_PERSISTENT) {
    UNSO_TRY(scale_chain_bf16_persistent(p, pl, ws, part, splits, dense_ld > 0 ? dense_ld : pl.ldc,
                                         dense_ld > 0 ? dense_ld * p.h : pl.hh, status, st));
  } else if (route == ROUTE_GLUE_FREE) {
    int nnorm;
    if (split_done) {
      const int64_t nt2 = (p.h + 255) / 256;
      nnorm = static_cast<int>(nt2 * (nt2 + 1) / 2 * 64);
    } else {
      const int nt = static_cast<int>((p.h + 31) / 32);
      nnorm = nt * (nt + 1) / 2;
      dim3 grid(nnorm, static_cast<unsigned>(p.batch));
      finalize_split_kernel<<<grid, 256, 0, st>>>(part, splits, static_cast<int>(p.batch), static_cast<int>(p.h), pl.ldc,
                                                  at<__nv_bfloat16>(ws, pl.Chi[0]), at<__nv_bfloat16>(ws, pl.Clo[0]),
                                                  at<double>(ws, pl.mnorm));
      UNSO_CHECK_LAUNCH();
    }
    UNSO_TRY(scale_chain_bf16_glue_free(p, pl, ws, nnorm, status, st));
  } else {
    float* G = at<float>(ws, pl.G);
    if (part != G || splits != 1) {
      const int nt = static_cast<int>((p.h + 31) / 32);
      dim3 grid(nt * (nt + 1) / 2, static_cast<unsigned>(p.batch));
      finalize_sum_kernel<float><<<grid, 256, 0, st>>>(part, splits, static_cast<int>(p.batch), static_cast<int>(p.h),
                                                       pl.ldc, G, pl.ldc, pl.hh);
      UNSO_CHECK_LAUNCH();
    }
    UNSO_TRY(scale_chain_bf16_multi(p, pl, ws, G, status, st));
  }
  return apply_bf16(p, pl, ws, xb, ldx, bsx, y, st);
}

// ---------------------------------------------------------------- NS baselines (FP32 precision)
static int32_t ns_fp32(const Problem& p, const Plan& pl, void* ws, const void* x, void* y, int32_t* status,
                       cudaStream_t st) {
  const int64_t B = p.batch;
  const int h = static_cast<int>(p.h);
  const int64_t xsz = p.rows * p.cols;
  // scale (preprocess, ortho.py:140-168)
  const double* xscale = at<double>(ws, pl.scal);
  if (p.scaling == UNSO_SCALING_NONE) {
    xscale = nullptr;
  } else if (p.scaling == UNSO_SCALING_PLAIN) {
    launch_sumsq(x, p.dt, p.rows, p.cols, p.ld, p.bs, B, at<double>(ws, pl.blk), st);
    UNSO_CHECK_LAUNCH();
    scalars_kernel<<<static_cast<unsigned>(B), 256, 0, st>>>(at<double>(ws, pl.blk), norm_blocks(p.rows * p.cols), SM_PLAIN, p.gpow,
                                                            at<double>(ws, pl.scal), status);
    UNSO_CHECK_LAUNCH();
  } else {
    UNSO_TRY(gram_fp32(p, x, pl, ws, pl.splits, st));
    UNSO_TRY(finalize_gram<double>(p, pl, ws, pl.splits, at<double>(ws, pl.G), st));
    UNSO_TRY(norms_and_scalars<double>(p, pl, ws, at<double>(ws, pl.G), SM_GRAM, status, st));
    if (p.scaling == UNSO_SCALING_GELFAND)
      UNSO_TRY(gelfand_scale<double>(p, pl, ws, at<double>(ws, pl.G), DT_F64, status, st));
  }
  convert_kernel<<<grid_for(B * xsz), 256, 0, st>>>(x, p.dt, p.ld, p.bs, at<double>(ws, pl.Xs[0]), DT_F64, p.cols, xsz,
                                                    p.rows, p.cols, static_cast<int>(B), xscale);
  UNSO_CHECK_LAUNCH();
  int cur = 0;
  const int iters = p.steps;
  for (int it = 0; it < iters; ++it) {
    const double* X = at<double>(ws, pl.Xs[cur]);
    if (use_oz(p)) {  // the same three products on the int8 digit engine (fp32 mode, h > 256)
      UNSO_TRY(gram_oz(p, X, pl, ws, pl.splits, st, DT_F64, p.cols, xsz));
      UNSO_TRY(finalize_gram<double>(p, pl, ws, pl.splits, at<double>(ws, pl.G), st));
      int8_t* cp = at<int8_t>(ws, pl.ozC);
      unsigned long long* cm = at<unsigned long long>(ws, pl.ozMaxB);
      const double* Bop = at<double>(ws, pl.G);
      double a_c, alpha;
      if (p.method == UNSO_METHOD_ORIGINAL_NS) {  // X <- 1.5 X - 0.5 G X (ortho.py:215-217)
        a_c = 1.5;
        alpha = -0.5;
      } else {  // X <- a X + (b G + c G^2) X (ortho.py:226-230)
        a_c = p.co[3 * it + 0];
        alpha = 1.0;
        UNSO_TRY(oz_slice(at<double>(ws, pl.G), DT_F64, pl.ldc, pl.hh, h, h, B, false, cm, h, cp, pl.ldc, pl.hh,
                          pl.ozC_plane, st));
        const OzOperand Gd{cp, pl.ldc, pl.hh, pl.ozC_plane, cm, h};
        const OzEpiQuinticB qe{at<double>(ws, pl.G), at<double>(ws, pl.C[0]), pl.ldc, pl.hh, p.co[3 * it + 1],
                               p.co[3 * it + 2]};
        UNSO_TRY(oz_gemm(Gd, Gd, h, h, h, B, true, 1, qe, st));
        Bop = at<double>(ws, pl.C[0]);
      }
      UNSO_TRY(oz_slice(Bop, DT_F64, pl.ldc, pl.hh, h, h, B, false, cm, h, cp, pl.ldc, pl.hh, pl.ozC_plane, st));
      const OzOperand Bd{cp, pl.ldc, pl.hh, pl.ozC_plane, cm, h};
      int8_t* xp = at<int8_t>(ws, pl.ozX);
      unsigned long long* xm = at<unsigned long long>(ws, pl.ozMaxA);
      const int64_t ldd = round_up(p.h, 64), dbs = p.w * ldd;
      // operand rows = the w long-side vectors of the state: rows of a tall X, columns of a wide one
      UNSO_TRY(oz_slice(X, DT_F64, p.cols, xsz, p.rows, p.cols, B, !p.tall, xm, pl.ozMaxA_bs, xp, ldd, dbs,
                        pl.ozX_plane, st));
      const OzOperand Xd{xp, ldd, dbs, pl.ozX_plane, xm, pl.ozMaxA_bs};
      const OzEpiAxpy ae{at<double>(ws, pl.Xs[cur ^ 1]), X, p.cols, xsz, alpha, a_c};
      if (p.tall)
        UNSO_TRY(oz_gemm(Xd, Bd, p.w, h, h, B, false, 1, ae, st));
      else
        UNSO_TRY(oz_gemm(Bd, Xd, h, p.w, h, B, false, 1, ae, st));
      cur ^= 1;
      continue;
    }
    UNSO_TRY(gram_simt(p, X, DT_F64, p.cols, xsz, pl, ws, pl.splits, st));
    UNSO_TRY(finalize_gram<double>(p, pl, ws, pl.splits, at<double>(ws, pl.G), st));
    const double* Bop = at<double>(ws, pl.G);
    double a_c, alpha;
    if (p.method == UNSO_METHOD_ORIGINAL_NS) {  // X <- 1.5 X - 0.5 G X (ortho.py:215-217)
      a_c = 1.5;
      alpha = -0.5;
    } else {  // X <- a X + (b G + c G^2) X (ortho.py:226-230)
      a_c = p.co[3 * it + 0];
      alpha = 1.0;
      SimtOperand Gop{at<double>(ws, pl.G), pl.ldc, pl.hh, DT_F64, 1};
      EpiQuinticB epi{at<double>(ws, pl.G), at<double>(ws, pl.C[0]), pl.ldc, pl.hh, p.co[3 * it + 1],
                      p.co[3 * it + 2]};
      if (launch_simt_gemm(Gop, Gop, h, h, h, static_cast<int>(B), true, 1, epi, st) != cudaSuccess)
        return UNSO_ERR_CUDA;
      ++g_launches;
      Bop = at<double>(ws, pl.C[0]);
    }
    SimtOperand Xop{X, p.cols, xsz, DT_F64, 1};
    SimtOperand Bm{Bop, pl.ldc, pl.hh, DT_F64, 1};
    EpiOut epi{at<double>(ws, pl.Xs[cur ^ 1]), DT_F64, p.cols, xsz, X, p.cols, xsz, alpha, a_c};
    cudaError_t e;
    if (p.tall) {
      e = launch_simt_gemm(Xop, Bm, static_cast<int>(p.rows), h, h, static_cast<int>(B), false, 1, epi, st);
    } else {
      Xop.kmajor = 0;
      e = launch_simt_gemm(Bm, Xop, h, static_cast<int>(p.cols), h, static_cast<int>(B), false, 1, epi, st);
    }
    if (e != cudaSuccess) return UNSO_ERR_CUDA;
    ++g_launches;
    cur ^= 1;
  }
  convert_kernel<<<grid_for(B * xsz), 256, 0, st>>>(at<double>(ws, pl.Xs[cur]), DT_F64, p.cols, xsz, y, p.dt, p.cols,
                                                    xsz, p.rows, p.cols, static_cast<int>(B), nullptr);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

// ---------------------------------------------------------------- NS baselines (BF16 precision, tcgen05)
using Cfg2NSTall = Umma2Cfg<256, 1, 2, 2, TERM(0, 0, 0) | TERM(1, 0, 1), false, false, 4>;
using Cfg2NSWide = Umma2Cfg<256, 2, 1, 2, TERM(0, 0, 0) | TERM(1, 1, 0), false, true, 4>;
// hi/lo state (default): X = X_hi + X_lo in every long-side product, bf16x3 (hi*hi + hi*lo + lo*hi)
constexpr int TERMS_X3 = TERM(0, 0, 0) | TERM(1, 0, 1) | TERM(2, 1, 0);
using Cfg2GramMN3 = Umma2Cfg<256, 2, 2, 3, TERMS_X3, true, true, 3>;
using Cfg2GramK3 = Umma2Cfg<256, 2, 2, 3, TERMS_X3, false, false, 3>;
using Cfg2NSTall3 = Umma2Cfg<256, 2, 2, 3, TERMS_X3, false, false, 3>;
using Cfg2NSWide3 = Umma2Cfg<256, 2, 2, 3, TERMS_X3, false, true, 3>;

// Gram of the NS state from its bf16 hi/lo parts (split-K partials, like gram_bf16).
static int32_t gram_bf16_x3(const Problem& p, const Plan& pl, void* ws, const __nv_bfloat16* xh,
                            const __nv_bfloat16* xl, int64_t ldx, int64_t bsx, cudaStream_t st) {
  CUtensorMap mh, ml;
  UEpiPartialF32 epi{at<float>(ws, pl.part), pl.hh, pl.ldc, static_cast<int>(p.batch), static_cast<int>(p.h)};
  const UmmaWork w2 = gram_work2(static_cast<int>(p.h), static_cast<int>(p.h), static_cast<int>(p.w), 256,
                                 static_cast<int>(p.batch), pl.splits);
  cudaError_t e;
  if (p.tall) {
    if (!umma_make_mnmajor_map(&mh, xh, p.rows, p.cols, ldx, p.batch, bsx) ||
        !umma_make_mnmajor_map(&ml, xl, p.rows, p.cols, ldx, p.batch, bsx))
      return UNSO_ERR_CUDA;
    e = launch_umma2<Cfg2GramMN3>(mh, ml, mh, ml, w2, epi, st);
  } else {
    if (!umma_make_kmajor_map(&mh, xh, p.rows, p.cols, ldx, p.batch, bsx, 128) ||
        !umma_make_kmajor_map(&ml, xl, p.rows, p.cols, ldx, p.batch, bsx, 128))
      return UNSO_ERR_CUDA;
    e = launch_umma2<Cfg2GramK3>(mh, ml, mh, ml, w2, epi, st);
  }
  if (e != cudaSuccess) return UNSO_ERR_CUDA;
  ++g_launches;
  return UNSO_OK;
}

static int32_t ns_bf16(const Problem& p, const Plan& pl, void* ws, const void* x, void* y, int32_t* status,
                       cudaStream_t st) {
  const int64_t B = p.batch;
  const int h = static_cast<int>(p.h);
  const int64_t xsz = p.rows * p.cols;
  __nv_bfloat16* xbs[2] = {at<__nv_bfloat16>(ws, pl.xb), at<__nv_bfloat16>(ws, pl.xb2)};
  __nv_bfloat16* xb = xbs[0];
  // hi/lo state: every long-side product (Gram of X_k, X_k B) uses X_k = hi + lo in bf16x3, so the
  // fp32 state enters the tensor cores at ~2^-17 instead of bf16 rounding (Muon-5: ~1e-2 -> ~1e-4
  // from the fp64 result, at 3 + 3 instead of 1 + 2 bf16 products per step).
  const bool x3 = (p.flags & UNSO_FLAG_NS_SINGLE_STATE) == 0 && use_pair_engine();
  __nv_bfloat16* xls[2] = {x3 ? at<__nv_bfloat16>(ws, pl.xl[0]) : nullptr, x3 ? at<__nv_bfloat16>(ws, pl.xl[1]) : nullptr};
  const int64_t ldx = pl.ldx, bsx = p.rows * pl.ldx;
  double* scal = at<double>(ws, pl.scal);
  double* unit = at<double>(ws, pl.normbuf);
  fill_unit_scal_kernel<<<static_cast<unsigned>((B + 127) / 128), 128, 0, st>>>(unit, static_cast<int>(B));
  UNSO_CHECK_LAUNCH();
  // preprocess scale (ortho.py:140-168): plain = ||A||_F, gram = ||A A^T||_F^(1/2), none = 1
  const double* xscale = scal;
  if (p.scaling == UNSO_SCALING_NONE) {
    xscale = nullptr;
  } else if (p.scaling == UNSO_SCALING_PLAIN) {
    launch_sumsq(x, p.dt, p.rows, p.cols, p.ld, p.bs, B, at<double>(ws, pl.blk), st, /*round_in=*/true);
    UNSO_CHECK_LAUNCH();
    scalars_kernel<<<static_cast<unsigned>(B), 256, 0, st>>>(at<double>(ws, pl.blk), norm_blocks(p.rows * p.cols), SM_PLAIN, p.gpow,
                                                            scal, status);
    UNSO_CHECK_LAUNCH();
  } else {  // gram / gelfand: Gram of the unscaled bf16 input on the tensor cores
    launch_ns_init_state(x, p.dt, p.ld, p.bs, nullptr, at<float>(ws, pl.Xs[0]), xb, ldx, p.rows, p.cols,
                         static_cast<int>(B), /*round_in=*/1, st);
    UNSO_CHECK_LAUNCH();
    UNSO_TRY(gram_bf16(p, pl, ws, xb, ldx, bsx, st));
    UNSO_TRY(finalize_gram<float>(p, pl, ws, pl.splits, at<float>(ws, pl.G), st));
    UNSO_TRY(norms_and_scalars<float>(p, pl, ws, at<float>(ws, pl.G), SM_GRAM, status, st));
    if (p.scaling == UNSO_SCALING_GELFAND)
      UNSO_TRY(gelfand_scale<float>(p, pl, ws, at<float>(ws, pl.G), DT_F32, status, st));
  }
  launch_ns_init_state(x, p.dt, p.ld, p.bs, xscale, at<float>(ws, pl.Xs[0]), xb, ldx, p.rows, p.cols,
                       static_cast<int>(B), /*round_in=*/1, st, xls[0]);
  UNSO_CHECK_LAUNCH();
  const dim3 egrid(grid_for(static_cast<int64_t>(h) * h, 256, 1024), static_cast<unsigned>(B));
  int cur = 0;
  for (int it = 0; it < p.steps; ++it) {
    xb = xbs[cur];  // read this step's operand, write the next one into the other buffer
    if (x3)
      UNSO_TRY(gram_bf16_x3(p, pl, ws, xb, xls[cur], ldx, bsx, st));
    else
      UNSO_TRY(gram_bf16(p, pl, ws, xb, ldx, bsx, st));
    UNSO_TRY(finalize_gram<float>(p, pl, ws, pl.splits, at<float>(ws, pl.G), st));
    const float* G = at<float>(ws, pl.G);
    float a_c;
    if (p.method == UNSO_METHOD_ORIGINAL_NS) {  // B = -0.5 G, X' = 1.5 X + X B
      a_c = 1.5f;
      split_scaled_kernel<<<egrid, 256, 0, st>>>(G, h, pl.ldc, -0.5f, at<__nv_bfloat16>(ws, pl.Phi),
                                                 at<__nv_bfloat16>(ws, pl.Plo));
      UNSO_CHECK_LAUNCH();
    } else {  // B = b G + c G^2 (bf16x3 SYRK), X' = a X + X B
      a_c = static_cast<float>(p.co[3 * it + 0]);
      split_scaled_kernel<<<egrid, 256, 0, st>>>(G, h, pl.ldc, 1.0f, at<__nv_bfloat16>(ws, pl.Chi[0]),
                                                 at<__nv_bfloat16>(ws, pl.Clo[0]));
      UNSO_CHECK_LAUNCH();
      SymMaps maps;
      const void* hi = at<__nv_bfloat16>(ws, pl.Chi[0]);
      const void* lo = at<__nv_bfloat16>(ws, pl.Clo[0]);
      if (!umma_make_kmajor_map(&maps.hiK, hi, h, h, pl.ldc, B, pl.hh, 128) ||
          !umma_make_kmajor_map(&maps.loK, lo, h, h, pl.ldc, B, pl.hh, 128) ||
          !umma_make_mnmajor_map(&maps.hiMN, hi, h, h, pl.ldc, B, pl.hh) ||
          !umma_make_mnmajor_map(&maps.loMN, lo, h, h, pl.ldc, B, pl.hh))
        return UNSO_ERR_CUDA;
      const UmmaWork wq = umma2_make_work(h, h, h, 256, static_cast<int>(B), true, 1);
      EpiQuinticBF16 qe{G, at<float>(ws, pl.P), pl.ldc, pl.hh, h, static_cast<float>(p.co[3 * it + 1]),
                        static_cast<float>(p.co[3 * it + 2])};
      if (launch_chain_pair(maps, wq, qe, st) != cudaSuccess) return UNSO_ERR_CUDA;
      ++g_launches;
      UNSO_TRY(finalize_p_bf16(p, pl, ws, unit, st));
    }
    CUtensorMap mx, mph, mpl;
    if (!umma_make_kmajor_map(&mph, at<__nv_bfloat16>(ws, pl.Phi), h, h, pl.ldc, B, pl.hh, 128) ||
        !umma_make_kmajor_map(&mpl, at<__nv_bfloat16>(ws, pl.Plo), h, h, pl.ldc, B, pl.hh, 128))
      return UNSO_ERR_CUDA;
    const float* xo = at<float>(ws, pl.Xs[cur]);
    float* xn = at<float>(ws, pl.Xs[cur ^ 1]);
    cudaError_t e;
    CUtensorMap mxl;
    if (p.tall) {
      if (!umma_make_kmajor_map(&mx, xb, p.rows, p.cols, ldx, B, bsx, 128)) return UNSO_ERR_CUDA;
      EpiNSUpdate epi{xo, xn, xbs[cur ^ 1], ldx, p.rows, p.cols, static_cast<int>(p.rows), h, a_c, xls[cur ^ 1]};
      const UmmaWork wa = umma2_make_work(static_cast<int>(p.rows), h, h, 256, static_cast<int>(B), false, 1);
      if (x3) {
        if (!umma_make_kmajor_map(&mxl, xls[cur], p.rows, p.cols, ldx, B, bsx, 128)) return UNSO_ERR_CUDA;
        e = launch_umma2<Cfg2NSTall3>(mx, mxl, mph, mpl, wa, epi, st);
      } else {
        e = launch_umma2<Cfg2NSTall>(mx, mx, mph, mpl, wa, epi, st);
      }
    } else {
      if (!umma_make_mnmajor_map(&mx, xb, p.rows, p.cols, ldx, B, bsx)) return UNSO_ERR_CUDA;
      EpiNSUpdate epi{xo, xn, xbs[cur ^ 1], ldx, p.rows, p.cols, h, static_cast<int>(p.cols), a_c, xls[cur ^ 1]};
      const UmmaWork wa = umma2_make_work(h, static_cast<int>(p.cols), h, 256, static_cast<int>(B), false, 1);
      if (x3) {
        if (!umma_make_mnmajor_map(&mxl, xls[cur], p.rows, p.cols, ldx, B, bsx)) return UNSO_ERR_CUDA;
        e = launch_umma2<Cfg2NSWide3>(mph, mpl, mx, mxl, wa, epi, st);
      } else {
        e = launch_umma2<Cfg2NSWide>(mph, mpl, mx, mx, wa, epi, st);
      }
    }
    if (e != cudaSuccess) return UNSO_ERR_CUDA;
    ++g_launches;
    cur ^= 1;
  }
  convert_kernel<<<grid_for(B * xsz), 256, 0, st>>>(at<float>(ws, pl.Xs[cur]), DT_F32, p.cols, xsz, y, p.dt, p.cols,
                                                    xsz, p.rows, p.cols, static_cast<int>(B), nullptr);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

static int32_t check_ws(const Plan& pl, void* ws, size_t bytes) {
  if (bytes < pl.total) return UNSO_ERR_WORKSPACE;
  if (pl.total > 0 && !ws) return UNSO_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return UNSO_ERR_VALUE;
  return UNSO_OK;
}

}  // namespace unso

// ==================================================================== C ABI
using namespace unso;

extern "C" {

const char* unso_version(void) { return UNSO_VERSION_STRING; }

const char* unso_status_string(int32_t s) {
  switch (s) {
    case UNSO_OK: return "ok";
    case UNSO_ERR_SHAPE: return "shape error";
    case UNSO_ERR_DEGENERATE: return "degenerate input";
    case UNSO_ERR_VALUE: return "invalid value";
    case UNSO_ERR_CUDA: return "CUDA error";
    case UNSO_ERR_UNSUPPORTED: return "unsupported";
    case UNSO_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

int32_t unso_last_launch_count(void) { return g_launches; }

size_t unso_workspace_size(const unso_matrix_desc* x, const unso_method_desc* method) {
  Problem p;
  if (make_problem(x, method, p) != UNSO_OK) return 0;
  const Plan a = make_plan(p, true);
  Plan e = make_plan(p, true, true);
  if (p.scaling == UNSO_SCALING_GELFAND && p.gpow > 1) {
    take(e, static_cast<size_t>(p.batch * e.hh) * 8);
    take(e, static_cast<size_t>(p.batch * e.hh) * 8);
  }
  return (a.total > e.total ? a.total : e.total) + 256;
}

int32_t unso_gram_dtype(const unso_method_desc* method) {
  return (method && method->precision == UNSO_PREC_BF16) ? UNSO_DTYPE_F32 : UNSO_DTYPE_F64;
}

int32_t unso_orthogonalize(const unso_matrix_desc* x, const void* x_ptr, void* y_ptr, const unso_method_desc* method,
                           void* workspace, size_t workspace_bytes, int32_t* d_status, void* stream) {
  g_launches = 0;
  Problem p;
  UNSO_TRY(make_problem(x, method, p));
  if (!x_ptr || !y_ptr) return UNSO_ERR_VALUE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p.method != UNSO_METHOD_UNSO) {
    const Plan pl = make_plan(p, true);
    UNSO_TRY(check_ws(pl, workspace, workspace_bytes));
    return p.prec == UNSO_PREC_FP32 ? ns_fp32(p, pl, workspace, x_ptr, y_ptr, d_status, st)
                                    : ns_bf16(p, pl, workspace, x_ptr, y_ptr, d_status, st);
  }
  const Plan pl = make_plan(p, true);
  UNSO_TRY(check_ws(pl, workspace, workspace_bytes));
  struct ProfGuard {
    ProfGuard() { g_prof_call = true; }
    ~ProfGuard() {
      nvtx_stage(-1);  // close the last stage range (also on an early error return)
      if (g_prof.on && g_prof.n < g_prof.cap) ++g_prof.n;
      g_prof_call = false;
    }
  } guard;
  prof_mark(0, st);
  if (p.prec == UNSO_PREC_FP32) {
    prof_mark(1, st);
    UNSO_TRY(gram_fp32(p, x_ptr, pl, workspace, pl.splits, st));
    prof_mark(2, st);
    double* G = at<double>(workspace, pl.G);
    UNSO_TRY(finalize_gram<double>(p, pl, workspace, pl.splits, G, st));
    return unso_fp32_from_G(p, pl, workspace, x_ptr, G, y_ptr, d_status, st);
  }
  const __nv_bfloat16* xb;
  int64_t ldx, bsx;
  UNSO_TRY(ensure_bf16_x(p, pl, workspace, x_ptr, xb, ldx, bsx, st));
  prof_mark(1, st);
  if (p.method == UNSO_METHOD_UNSO && bf16_route(p) == ROUTE_SMALL && small_fused_gram(p)) {
    UNSO_TRY(scale_chain_bf16_small(p, pl, workspace, nullptr, 1, 0, 0, d_status, st, xb, ldx, bsx));
    return apply_bf16(p, pl, workspace, xb, ldx, bsx, y_ptr, st);
  }
  const bool split_out = bf16_route(p) == ROUTE_GLUE_FREE && pl.splits == 1;
  if (split_out)
    UNSO_TRY(gram_bf16_split(p, pl, workspace, xb, ldx, bsx, st));
  else
    UNSO_TRY(gram_bf16(p, pl, workspace, xb, ldx, bsx, st));
  prof_mark(2, st);
  return unso_bf16_after_gram(p, pl, workspace, xb, ldx, bsx, at<float>(workspace, pl.part), pl.splits, split_out,
                              y_ptr, d_status, st);
}

#ifdef UNSO_EXP_TIMING
extern "C" int32_t unso_debug_chain_trace(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, g_chain_trace, sizeof(g_chain_trace)) == cudaSuccess ? UNSO_OK : UNSO_ERR_CUDA;
}
extern "C" int32_t unso_debug_oz_trace(unsigned long long* host_out) {  // 2 x 16 x 8 timestamps
  return cudaMemcpyFromSymbol(host_out, g_oz_trace, sizeof(g_oz_trace)) == cudaSuccess ? UNSO_OK : UNSO_ERR_CUDA;
}
extern "C" int32_t unso_debug_chain_kb(unsigned long long* host_out) {  // 2 x 64 per-k-block timestamps
  return cudaMemcpyFromSymbol(host_out, g_chain_kb, sizeof(g_chain_kb)) == cudaSuccess ? UNSO_OK : UNSO_ERR_CUDA;
}
#endif

int32_t unso_query_scalars(const unso_matrix_desc* x, const unso_method_desc* method, const void* workspace,
                           double* d_out, void* stream) {
  Problem p;
  UNSO_TRY(make_problem(x, method, p));
  if (!workspace || !d_out) return UNSO_ERR_VALUE;
  static_assert(SCAL_STRIDE == UNSO_SCALARS, "scalar block layout");
  const Plan pl = make_plan(p, true);
  if (cudaMemcpyAsync(d_out, static_cast<const char*>(workspace) + pl.scal, sizeof(double) * SCAL_STRIDE * p.batch,
                      cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return UNSO_ERR_CUDA;
  return UNSO_OK;
}

int32_t unso_profile_begin(int32_t max_calls) {
  unso_profile_end();
  if (max_calls < 1) return UNSO_ERR_VALUE;
  g_prof.ev.assign(static_cast<size_t>(max_calls) * PROF_EV, nullptr);
  for (auto& e : g_prof.ev)
    if (cudaEventCreate(&e) != cudaSuccess) return UNSO_ERR_CUDA;
  g_prof.cap = max_calls;
  g_prof.n = 0;
  g_prof.on = true;
  return UNSO_OK;
}

int32_t unso_profile_read(float* out_ms, int32_t max_calls) {
  if (!g_prof.on || !out_ms) return 0;
  const int n = g_prof.n < max_calls ? g_prof.n : max_calls;
  for (int c = 0; c < n; ++c) {
    for (int s = 0; s < UNSO_PROFILE_STAGES; ++s) {
      float ms = 0.f;
      cudaEvent_t a = g_prof.ev[c * PROF_EV + s], b = g_prof.ev[c * PROF_EV + s + 1];
      if (cudaEventSynchronize(b) != cudaSuccess || cudaEventElapsedTime(&ms, a, b) != cudaSuccess) ms = -1.f;
      out_ms[c * UNSO_PROFILE_STAGES + s] = ms;
    }
  }
  return n;
}

void unso_profile_end(void) {
  for (auto& e : g_prof.ev)
    if (e) cudaEventDestroy(e);
  g_prof.ev.clear();
  g_prof.on = false;
  g_prof.cap = g_prof.n = 0;
}

int32_t unso_gram(const unso_matrix_desc* x, const void* x_ptr, void* g_ptr, const unso_method_desc* method,
                  void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  Problem p;
  UNSO_TRY(make_problem(x, method, p));
  if (p.method != UNSO_METHOD_UNSO) return UNSO_ERR_UNSUPPORTED;
  if (!x_ptr || !g_ptr) return UNSO_ERR_VALUE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Plan pl = make_plan(p, true);
  UNSO_TRY(check_ws(pl, workspace, workspace_bytes));
  // g_ptr is dense batch x h x h; finalize into the padded workspace G, then compact
  const int64_t h = p.h;
  if (p.prec == UNSO_PREC_FP32) {
    UNSO_TRY(gram_fp32(p, x_ptr, pl, workspace, pl.splits, st));
    return finalize_gram<double>(p, pl, workspace, pl.splits, static_cast<double*>(g_ptr), st, h, h * h);
  }
  const __nv_bfloat16* xb;
  int64_t ldx, bsx;
  UNSO_TRY(ensure_bf16_x(p, pl, workspace, x_ptr, xb, ldx, bsx, st));
  UNSO_TRY(gram_bf16(p, pl, workspace, xb, ldx, bsx, st));
  return finalize_gram<float>(p, pl, workspace, pl.splits, static_cast<float*>(g_ptr), st, h, h * h);
}

// ---------------------------------------------------------------- Gram reduction over NVLink peers
static bool gar_peers(const unso_gram_peers* in, int32_t world, GarPeers& out) {
  if (!in || world < 1 || world > GAR_MAX_WORLD) return false;
  for (int r = 0; r < world; ++r) {
    if (!in->slots[r] || !in->g[r] || !in->flags[r]) return false;
    out.slots[r] = static_cast<float*>(in->slots[r]);
    out.g[r] = static_cast<float*>(in->g[r]);
    out.flags[r] = in->flags[r];
  }
  return true;
}

size_t unso_gram_peer_bytes(int64_t h, int32_t world, int32_t splits, int32_t which) {
  if (h < 1 || h > (1 << 16) || world < 1 || world > GAR_MAX_WORLD || splits < 1 || splits > 64) return 0;
  if (which == 0)
    return static_cast<size_t>(gar_slot_offset(world, 0, 0, splits, gar_owned_max(static_cast<int>(h), world))) * 4;
  if (which == 1) return static_cast<size_t>(h * h) * 4;
  if (which == 2) return static_cast<size_t>(2 * world) * 4;
  return 0;
}

int32_t unso_gram_push(const unso_matrix_desc* x, const void* x_ptr, const unso_method_desc* method,
                       const unso_gram_peers* peers, int32_t rank, int32_t world, int32_t splits, uint32_t epoch,
                       void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  Problem p;
  UNSO_TRY(make_problem(x, method, p));
  if (p.method != UNSO_METHOD_UNSO || p.prec != UNSO_PREC_BF16 || p.batch != 1 || !use_pair_engine())
    return UNSO_ERR_UNSUPPORTED;
  GarPeers gp;
  if (!x_ptr || !gar_peers(peers, world, gp) || rank < 0 || rank >= world || splits < 1 || splits > 64 ||
      (p.w + 63) / 64 < splits)
    return UNSO_ERR_VALUE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Plan pl = make_plan(p, true);
  UNSO_TRY(check_ws(pl, workspace, workspace_bytes));
  const __nv_bfloat16* xb;
  int64_t ldx, bsx;
  UNSO_TRY(ensure_bf16_x(p, pl, workspace, x_ptr, xb, ldx, bsx, st));
  const int h = static_cast<int>(p.h);
  UEpiPushF32 epi{gp, rank, world, splits, gar_owned_max(h, world), h, (h + GAR_TILE - 1) / GAR_TILE};
  const UmmaWork w2 = gram_work2(h, h, static_cast<int>(p.w), 256, 1, splits);
  CUtensorMap mx;
  cudaError_t e;
  if (p.tall) {
    if (!umma_make_mnmajor_map(&mx, xb, p.rows, p.cols, ldx, 1, bsx)) return UNSO_ERR_CUDA;
    e = launch_umma2<Cfg2GramMN>(mx, mx, mx, mx, w2, epi, st);
  } else {
    if (!umma_make_kmajor_map(&mx, xb, p.rows, p.cols, ldx, 1, bsx, 128)) return UNSO_ERR_CUDA;
    e = launch_umma2<Cfg2GramK>(mx, mx, mx, mx, w2, epi, st);
  }
  if (e != cudaSuccess) return UNSO_ERR_CUDA;
  gar_signal_kernel<<<1, 1, 0, st>>>(gp, rank, world, 0, epoch);
  UNSO_CHECK_LAUNCH();
  g_launches += 2;
  return UNSO_OK;
}

int32_t unso_gram_reduce(int64_t h, const unso_gram_peers* peers, int32_t rank, int32_t world, int32_t splits,
                         uint32_t epoch, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  GarPeers gp;
  if (h < 1 || !gar_peers(peers, world, gp) || rank < 0 || rank >= world || splits < 1 || splits > 64)
    return UNSO_ERR_VALUE;
  if (!workspace || workspace_bytes < sizeof(unsigned)) return UNSO_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned* done = static_cast<unsigned*>(workspace);
  if (cudaMemsetAsync(done, 0, sizeof(unsigned), st) != cudaSuccess) return UNSO_ERR_CUDA;
  const int hh = static_cast<int>(h);
  const int owned = gar_owned_max(hh, world);
  dim3 grid(static_cast<unsigned>(owned), 64);
  gar_reduce_kernel<<<grid, 256, 0, st>>>(gp, rank, world, splits, owned, hh, (hh + GAR_TILE - 1) / GAR_TILE, epoch,
                                          done);
  UNSO_CHECK_LAUNCH();
  g_launches = 1;
  return UNSO_OK;
}

int32_t unso_gram_wait(int64_t h, const unso_gram_peers* peers, int32_t rank, int32_t world, uint32_t epoch,
                       void* stream) {
  g_launches = 0;
  GarPeers gp;
  if (h < 1 || !gar_peers(peers, world, gp) || rank < 0 || rank >= world) return UNSO_ERR_VALUE;
  gar_wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(gp.flags[rank], world, 1, epoch);
  UNSO_CHECK_LAUNCH();
  g_launches = 1;
  return UNSO_OK;
}

int32_t unso_orthogonalize_from_gram(const unso_matrix_desc* x, const void* x_ptr, const void* g_ptr, void* y_ptr,
                                     const unso_method_desc* method, void* workspace, size_t workspace_bytes,
                                     int32_t* d_status, void* stream) {
  g_launches = 0;
  Problem p;
  UNSO_TRY(make_problem(x, method, p));
  if (p.method != UNSO_METHOD_UNSO) return UNSO_ERR_UNSUPPORTED;
  if (!x_ptr || !g_ptr || !y_ptr) return UNSO_ERR_VALUE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Plan pl = make_plan(p, false);
  UNSO_TRY(check_ws(pl, workspace, workspace_bytes));
  const int64_t h = p.h;
  // copy the dense reduced Gram into the padded workspace layout
  if (p.prec == UNSO_PREC_FP32) {
    convert_kernel<<<grid_for(p.batch * h * h), 256, 0, st>>>(g_ptr, DT_F64, h, h * h, at<double>(workspace, pl.G),
                                                              DT_F64, pl.ldc, pl.hh, h, h, static_cast<int>(p.batch),
                                                              nullptr);
    UNSO_CHECK_LAUNCH();
    return unso_fp32_from_G(p, pl, workspace, x_ptr, at<double>(workspace, pl.G), y_ptr, d_status, st);
  }
  const __nv_bfloat16* xb;
  int64_t ldx, bsx;
  UNSO_TRY(ensure_bf16_x(p, pl, workspace, x_ptr, xb, ldx, bsx, st));
  if (h % 4 == 0 && (reinterpret_cast<uintptr_t>(g_ptr) & 15) == 0)  // dense G read in place (float4 rows)
    return unso_bf16_after_gram(p, pl, workspace, xb, ldx, bsx, static_cast<const float*>(g_ptr), 1, false, y_ptr,
                                d_status, st, h);
  convert_kernel<<<grid_for(p.batch * h * h), 256, 0, st>>>(g_ptr, DT_F32, h, h * h, at<float>(workspace, pl.G), DT_F32,
                                                            pl.ldc, pl.hh, h, h, static_cast<int>(p.batch), nullptr);
  UNSO_CHECK_LAUNCH();
  return unso_bf16_after_gram(p, pl, workspace, xb, ldx, bsx, at<float>(workspace, pl.G), 1, false, y_ptr, d_status,
                              st);
}

int32_t unso_scale_denominator(const unso_matrix_desc* x, const void* x_ptr, const unso_method_desc* method,
                               double* d_denom, void* workspace, size_t workspace_bytes, int32_t* d_status,
                               void* stream) {
  g_launches = 0;
  Problem p;
  UNSO_TRY(make_problem(x, nullptr, p, false));
  if (!method || !x_ptr || !d_denom) return UNSO_ERR_VALUE;
  p.prec = UNSO_PREC_FP32;
  p.method = UNSO_METHOD_UNSO;
  p.scaling = method->scaling;
  p.gpow = method->gelfand_power;
  if (p.scaling < 0 || p.scaling > 2 || p.gpow < 1) return UNSO_ERR_VALUE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Plan pl = make_plan(p, true, true);
  Plan plg = pl;
  if (p.scaling == UNSO_SCALING_GELFAND && p.gpow > 1) {  // room for the power ping-pong
    plg.Gk[0] = take(plg, static_cast<size_t>(p.batch * pl.hh) * 8);
    plg.Gk[1] = take(plg, static_cast<size_t>(p.batch * pl.hh) * 8);
  }
  UNSO_TRY(check_ws(plg, workspace, workspace_bytes));
  if (p.scaling == UNSO_SCALING_PLAIN) {
    launch_sumsq(x_ptr, p.dt, p.rows, p.cols, p.ld, p.bs, p.batch, at<double>(workspace, pl.blk), st);
    UNSO_CHECK_LAUNCH();
    scalars_kernel<<<static_cast<unsigned>(p.batch), 256, 0, st>>>(at<double>(workspace, pl.blk), norm_blocks(p.rows * p.cols),
                                                                    SM_PLAIN, 1, at<double>(workspace, pl.scal),
                                                                    d_status);
    UNSO_CHECK_LAUNCH();
  } else {
    UNSO_TRY(gram_simt(p, x_ptr, p.dt, p.ld, p.bs, pl, workspace, pl.splits, st));
    UNSO_TRY(finalize_gram<double>(p, pl, workspace, pl.splits, at<double>(workspace, pl.G), st));
    UNSO_TRY(norms_and_scalars<double>(p, pl, workspace, at<double>(workspace, pl.G), SM_GRAM, d_status, st));
    if (p.scaling == UNSO_SCALING_GELFAND)
      UNSO_TRY(gelfand_scale<double>(p, plg, workspace, at<double>(workspace, pl.G), DT_F64, d_status, st));
  }
  copy_denom_kernel<<<static_cast<unsigned>((p.batch + 127) / 128), 128, 0, st>>>(at<double>(workspace, pl.scal),
                                                                                  static_cast<int>(p.batch), d_denom);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

int32_t unso_ortho_error(const unso_matrix_desc* y, const void* y_ptr, double* d_err, void* workspace,
                         size_t workspace_bytes, void* stream) {
  g_launches = 0;
  Problem p;
  UNSO_TRY(make_problem(y, nullptr, p, false));
  if (!y_ptr || !d_err) return UNSO_ERR_VALUE;
  p.prec = UNSO_PREC_FP32;
  p.method = UNSO_METHOD_UNSO;
  p.scaling = UNSO_SCALING_GRAM;
  p.gpow = 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Plan pl = make_plan(p, true, true);
  UNSO_TRY(check_ws(pl, workspace, workspace_bytes));
  UNSO_TRY(gram_simt(p, y_ptr, p.dt, p.ld, p.bs, pl, workspace, pl.splits, st));
  UNSO_TRY(finalize_gram<double>(p, pl, workspace, pl.splits, at<double>(workspace, pl.G), st));
  const int nb = norm_blocks(p.h * p.h);
  dim3 grid(nb, static_cast<unsigned>(p.batch));
  gram_norms_kernel<double><<<grid, 256, 0, st>>>(at<double>(workspace, pl.G), static_cast<int>(p.h), pl.ldc,
                                                  at<double>(workspace, pl.blk));
  UNSO_CHECK_LAUNCH();
  scalars_kernel<<<static_cast<unsigned>(p.batch), 256, 0, st>>>(at<double>(workspace, pl.blk), nb, SM_ERROR,
                                                                  1, at<double>(workspace, pl.scal), nullptr);
  UNSO_CHECK_LAUNCH();
  copy_err_kernel<<<static_cast<unsigned>((p.batch + 127) / 128), 128, 0, st>>>(at<double>(workspace, pl.scal),
                                                                                static_cast<int>(p.batch), d_err);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

// ---------------------------------------------------------------- Muon optimizer passes
static int64_t muon_per_block(int64_t numel) {
  const int64_t per = 16384;
  return numel < per ? ((numel + 7) / 8) * 8 : per;
}

int32_t unso_muon_prepare(int32_t n, const void* d_grads, const void* d_bufs, void* stacked, int64_t numel,
                          int32_t dtype, float mu, int32_t nesterov, float* d_maxabs, void* stream) {
  if (n < 0 || n > 65535 || numel < 0 || (n > 0 && (!d_grads || !d_bufs || !stacked || !d_maxabs)))
    return UNSO_ERR_VALUE;
  if (dtype != UNSO_DTYPE_F32 && dtype != UNSO_DTYPE_BF16) return UNSO_ERR_UNSUPPORTED;
  g_launches = 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 0) return UNSO_OK;
  if (cudaMemsetAsync(d_maxabs, 0, sizeof(float) * n, st) != cudaSuccess) return UNSO_ERR_CUDA;
  if (numel == 0) return UNSO_OK;
  const int64_t per = muon_per_block(numel);
  dim3 grid(static_cast<unsigned>((numel + per - 1) / per), static_cast<unsigned>(n));
  const uint64_t* g = static_cast<const uint64_t*>(d_grads);
  const uint64_t* m = static_cast<const uint64_t*>(d_bufs);
  if (dtype == UNSO_DTYPE_BF16)
    muon_prepare_kernel<__nv_bfloat16><<<grid, MUON_THREADS, 0, st>>>(g, m, static_cast<__nv_bfloat16*>(stacked),
                                                                     numel, per, mu, nesterov, d_maxabs);
  else
    muon_prepare_kernel<float><<<grid, MUON_THREADS, 0, st>>>(g, m, static_cast<float*>(stacked), numel, per, mu,
                                                             nesterov, d_maxabs);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

int32_t unso_muon_update(int32_t n, const void* d_params, const void* ortho, int64_t numel, int32_t dtype,
                         const float* d_maxabs, float decay, float alpha, void* stream) {
  if (n < 0 || n > 65535 || numel < 0 || (n > 0 && (!d_params || !ortho || !d_maxabs))) return UNSO_ERR_VALUE;
  if (dtype != UNSO_DTYPE_F32 && dtype != UNSO_DTYPE_BF16) return UNSO_ERR_UNSUPPORTED;
  g_launches = 0;
  if (n == 0 || numel == 0) return UNSO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t per = muon_per_block(numel);
  dim3 grid(static_cast<unsigned>((numel + per - 1) / per), static_cast<unsigned>(n));
  const uint64_t* pp = static_cast<const uint64_t*>(d_params);
  if (dtype == UNSO_DTYPE_BF16)
    muon_update_kernel<__nv_bfloat16><<<grid, MUON_THREADS, 0, st>>>(
        pp, static_cast<const __nv_bfloat16*>(ortho), numel, per, d_maxabs, decay, alpha);
  else
    muon_update_kernel<float><<<grid, MUON_THREADS, 0, st>>>(pp, static_cast<const float*>(ortho), numel, per,
                                                            d_maxabs, decay, alpha);
  UNSO_CHECK_LAUNCH();
  return UNSO_OK;
}

}  // extern "C"
