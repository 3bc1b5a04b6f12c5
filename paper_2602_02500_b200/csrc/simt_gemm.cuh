// Reference: densemat.matmul (densemat.py:74-82, numpy/OpenBLAS dgemm) at fp64 accumulation.
// fp64-accumulating GEMM/SYRK engine on the fp64 tensor cores (DMMA, mma.sync m8n8k4 f64):
// the "fp32 mode" of the orthogonalizer (parity <= 1e-5 needs fp64-grade Gram and squaring
// chain on ill-conditioned inputs), the Gelfand scaling products and the
// device-side orthogonality-error Gram.
//
//   D[b](m, n) = sum_k A[b](m, k) * B[b](n, k)        (fp64 products and accumulation)
//
// Each operand is a strided batch of row-major matrices read either K-major (element (i,k)
// at p[i*ld + k]) or MN-major (element (i,k) at p[k*ld + i]), stored as f32 / bf16 / f64 and
// widened to f64 exactly on the way into shared memory.  `syrk` restricts the tile grid to
// tiles whose columns reach the diagonal; the epilogue is only invoked on n >= m there.
// `splits` partitions K; every (tile, split) is one CTA.
// CTA tile 64 x 64, 4 warps of 32 x 32 (4 x 4 DMMA 8x8x4 fragments), k-tile 16, smem double
// buffered with register prefetch; shared layouts [k][m] padded by 8 doubles so the 32 lanes of
// a fragment load hit all banks in the minimum two wavefronts.
#pragma once
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace unso {

struct SimtOperand {
  const void* p;
  int64_t ld;
  int64_t bstride;
  int dtype;
  int kmajor;
};

constexpr int SIMT_BM = 64, SIMT_BN = 64, SIMT_BK = 16, SIMT_PAD = 8;

__device__ __forceinline__ void simt_tile_coords(int t, int tiles_m, int tiles_n, int syrk, int& tm, int& tn) {
  if (!syrk) {
    tm = t / tiles_n;
    tn = t % tiles_n;
    return;
  }
  int row = 0, len = tiles_n;
  while (t >= len) {
    t -= len;
    ++row;
    --len;
  }
  tm = row;
  tn = row + t;
}

__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// 64 rows x 16 k of one operand -> 8 values per thread (coalesced along the contiguous axis).
template <int DT>
__device__ __forceinline__ void simt_fetch(const char* base, const SimtOperand& op, int r0, int k0, int R, int K,
                                           double (&v)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int e = threadIdx.x + 128 * q;
    int i, k;
    if (op.kmajor) { k = e & 15; i = e >> 4; } else { i = e & 63; k = e >> 6; }
    double x = 0.0;
    if (r0 + i < R && k0 + k < K) {
      const int64_t off = op.kmajor ? static_cast<int64_t>(r0 + i) * op.ld + (k0 + k)
                                    : static_cast<int64_t>(k0 + k) * op.ld + (r0 + i);
      if (DT == DT_F32) x = static_cast<double>(reinterpret_cast<const float*>(base)[off]);
      else if (DT == DT_BF16) x = static_cast<double>(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[off]));
      else x = reinterpret_cast<const double*>(base)[off];
    }
    v[q] = x;
  }
}

__device__ __forceinline__ void simt_fetch_any(const char* base, const SimtOperand& op, int r0, int k0, int R, int K,
                                               double (&v)[8]) {
  if (op.dtype == DT_F64) simt_fetch<DT_F64>(base, op, r0, k0, R, K, v);
  else if (op.dtype == DT_F32) simt_fetch<DT_F32>(base, op, r0, k0, R, K, v);
  else simt_fetch<DT_BF16>(base, op, r0, k0, R, K, v);
}

__device__ __forceinline__ void simt_stash(double (*S)[SIMT_BM + SIMT_PAD], const SimtOperand& op,
                                           const double (&v)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int e = threadIdx.x + 128 * q;
    int i, k;
    if (op.kmajor) { k = e & 15; i = e >> 4; } else { i = e & 63; k = e >> 6; }
    S[k][i] = v[q];
  }
}

template <class Epi>
__global__ void __launch_bounds__(128, 4) simt_gemm_kernel(SimtOperand A, SimtOperand B, int M, int N, int K, int syrk,
                                                        int tiles_m, int tiles_n, int splits, Epi epi) {
  __shared__ __align__(16) double As[2][SIMT_BK][SIMT_BM + SIMT_PAD];
  __shared__ __align__(16) double Bs[2][SIMT_BK][SIMT_BN + SIMT_PAD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1, gid = lane >> 2, tig = lane & 3;
  const int split = blockIdx.y, b = blockIdx.z;
  int tm, tn;
  simt_tile_coords(blockIdx.x, tiles_m, tiles_n, syrk, tm, tn);
  const int m0 = tm * SIMT_BM, n0 = tn * SIMT_BN;
  const int ktiles = (K + SIMT_BK - 1) / SIMT_BK;
  const int kt0 = static_cast<int>(static_cast<int64_t>(split) * ktiles / splits);
  const int kt1 = static_cast<int>(static_cast<int64_t>(split + 1) * ktiles / splits);
  const char* pa = static_cast<const char*>(A.p) + static_cast<int64_t>(b) * A.bstride * dtype_size(A.dtype);
  const char* pb = static_cast<const char*>(B.p) + static_cast<int64_t>(b) * B.bstride * dtype_size(B.dtype);

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double va[8], vb[8];
  if (kt0 < kt1) {
    simt_fetch_any(pa, A, m0, kt0 * SIMT_BK, M, K, va);
    simt_fetch_any(pb, B, n0, kt0 * SIMT_BK, N, K, vb);
    simt_stash(As[0], A, va);
    simt_stash(Bs[0], B, vb);
  }
  __syncthreads();
  int buf = 0;
  for (int kt = kt0; kt < kt1; ++kt) {
    const bool more = kt + 1 < kt1;
    if (more) {
      simt_fetch_any(pa, A, m0, (kt + 1) * SIMT_BK, M, K, va);
      simt_fetch_any(pb, B, n0, (kt + 1) * SIMT_BK, N, K, vb);
    }
#pragma unroll
    for (int kk = 0; kk < SIMT_BK / 4; ++kk) {
      double a[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][kk * 4 + tig][wm * 32 + i * 8 + gid];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][kk * 4 + tig][wn * 32 + j * 8 + gid];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_884(acc[i][j], a[i], bv[j]);
    }
    if (more) {
      simt_stash(As[buf ^ 1], A, va);
      simt_stash(Bs[buf ^ 1], B, vb);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + wm * 32 + i * 8 + gid;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = n0 + wn * 32 + j * 8 + 2 * tig + e;
        if (n >= N) continue;
        if (syrk && n < m) continue;
        epi(b, split, m, n, acc[i][j][e]);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// Pipelined variant (operands 16-byte aligned): raw-dtype tiles streamed into shared memory by
// cp.async (3 stages, zero-filled edges), widened to f64 at the fragment load.  No register
// staging, so 4 CTAs (16 warps) fit per SM to hide the DMMA and load latencies.
// Padded strides keep the fragment loads conflict-free (K-major tile [m][16+pk], MN-major
// [k][64+pm]); every row stride is a multiple of 16 bytes for the cp.async destinations.
template <int DT> struct DmmaLayout {
  static constexpr int E = DT == DT_F64 ? 8 : (DT == DT_F32 ? 4 : 2);
  static constexpr int KS = SIMT_BK + (DT == DT_BF16 ? 8 : 4);   // K-major row stride (elements)
  static constexpr int MS = SIMT_BM + (DT == DT_F64 ? 4 : 8);    // MN-major row stride (elements)
  static constexpr int BYTES = (64 * KS > SIMT_BK * MS ? 64 * KS : SIMT_BK * MS) * E;
  static constexpr int EPC = 16 / E;                              // elements per 16-byte chunk
};
// Two stages with 4 CTAs (16 warps) per SM beat three stages with 3 CTAs: the batched chain of
// configs[1] (16 x 36 upper 64x64 tiles = 576 CTAs) then runs in one wave of 592 slots
// (fp32-mode chain 1.86 -> 1.40 ms; cfg5 chain -5 %; Gram / apply unchanged).
constexpr int DMMA_STAGES = 2;

template <int DT>
__device__ __forceinline__ double dmma_lds(const uint8_t* base, int idx) {
  if (DT == DT_F64) return reinterpret_cast<const double*>(base)[idx];
  if (DT == DT_F32) return static_cast<double>(reinterpret_cast<const float*>(base)[idx]);
  return static_cast<double>(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx]));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes) : "memory");
}

// 64 rows x 16 k of one operand, tile origin (r0, k0), into one stage buffer
template <int DT>
__device__ __forceinline__ void dmma_issue(uint8_t* dst, const char* base, const SimtOperand& op, int r0, int k0, int R,
                                           int K) {
  using L = DmmaLayout<DT>;
  if (op.kmajor) {
    constexpr int CPR = SIMT_BK / L::EPC;  // chunks per tile row
    for (int c = threadIdx.x; c < 64 * CPR; c += 128) {
      const int row = c / CPR, kc = (c % CPR) * L::EPC;
      const int gr = r0 + row, gk = k0 + kc;
      const int valid = (gr < R && gk < K) ? min(L::EPC, K - gk) : 0;
      const char* src = base + (static_cast<int64_t>(valid ? gr : 0) * op.ld + (valid ? gk : 0)) * L::E;
      cp_async16(dst + (row * L::KS + kc) * L::E, src, valid * L::E);
    }
  } else {
    constexpr int CPR = SIMT_BM / L::EPC;
    for (int c = threadIdx.x; c < SIMT_BK * CPR; c += 128) {
      const int row = c / CPR, mc = (c % CPR) * L::EPC;
      const int gk = k0 + row, gm = r0 + mc;
      const int valid = (gk < K && gm < R) ? min(L::EPC, R - gm) : 0;
      const char* src = base + (static_cast<int64_t>(valid ? gk : 0) * op.ld + (valid ? gm : 0)) * L::E;
      cp_async16(dst + (row * L::MS + mc) * L::E, src, valid * L::E);
    }
  }
}

template <int DTA, int DTB, class Epi>
__global__ void __launch_bounds__(128, 4) dmma_gemm_kernel(SimtOperand A, SimtOperand B, int M, int N, int K, int syrk,
                                                           int tiles_m, int tiles_n, int splits, Epi epi) {
  using LA = DmmaLayout<DTA>;
  using LB = DmmaLayout<DTB>;
  constexpr int STAGE = LA::BYTES + LB::BYTES;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1, gid = lane >> 2, tig = lane & 3;
  const int split = blockIdx.y, b = blockIdx.z;
  int tm, tn;
  simt_tile_coords(blockIdx.x, tiles_m, tiles_n, syrk, tm, tn);
  const int m0 = tm * SIMT_BM, n0 = tn * SIMT_BN;
  const int ktiles = (K + SIMT_BK - 1) / SIMT_BK;
  const int kt0 = static_cast<int>(static_cast<int64_t>(split) * ktiles / splits);
  const int kt1 = static_cast<int>(static_cast<int64_t>(split + 1) * ktiles / splits);
  const char* pa = static_cast<const char*>(A.p) + static_cast<int64_t>(b) * A.bstride * LA::E;
  const char* pb = static_cast<const char*>(B.p) + static_cast<int64_t>(b) * B.bstride * LB::E;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = kt1 - kt0;
#pragma unroll
  for (int s = 0; s < DMMA_STAGES - 1; ++s) {
    if (s < nk) {
      dmma_issue<DTA>(dsm + s * STAGE, pa, A, m0, (kt0 + s) * SIMT_BK, M, K);
      dmma_issue<DTB>(dsm + s * STAGE + LA::BYTES, pb, B, n0, (kt0 + s) * SIMT_BK, N, K);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; it < nk; ++it) {
    asm volatile("cp.async.wait_group %0;" ::"n"(DMMA_STAGES - 2) : "memory");
    __syncthreads();  // stage it landed for every thread; stage it-1 is free to refill
    const int nxt = it + DMMA_STAGES - 1;
    if (nxt < nk) {
      uint8_t* st = dsm + (nxt % DMMA_STAGES) * STAGE;
      dmma_issue<DTA>(st, pa, A, m0, (kt0 + nxt) * SIMT_BK, M, K);
      dmma_issue<DTB>(st + LA::BYTES, pb, B, n0, (kt0 + nxt) * SIMT_BK, N, K);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const uint8_t* sa = dsm + (it % DMMA_STAGES) * STAGE;
    const uint8_t* sb = sa + LA::BYTES;
#pragma unroll
    for (int kk = 0; kk < SIMT_BK / 4; ++kk) {
      const int k = kk * 4 + tig;
      double a[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + gid;
        a[i] = A.kmajor ? dmma_lds<DTA>(sa, m * LA::KS + k) : dmma_lds<DTA>(sa, k * LA::MS + m);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = wn * 32 + j * 8 + gid;
        bv[j] = B.kmajor ? dmma_lds<DTB>(sb, n * LB::KS + k) : dmma_lds<DTB>(sb, k * LB::MS + n);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_884(acc[i][j], a[i], bv[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + wm * 32 + i * 8 + gid;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = n0 + wn * 32 + j * 8 + 2 * tig + e;
        if (n >= N) continue;
        if (syrk && n < m) continue;
        epi(b, split, m, n, acc[i][j][e]);
      }
    }
  }
}

template <int DTA, int DTB, class Epi>
inline cudaError_t launch_dmma(const SimtOperand& A, const SimtOperand& B, int M, int N, int K, int batch, bool syrk,
                               int splits, const Epi& epi, cudaStream_t stream, int tm, int tn, int tiles) {
  constexpr int smem = DMMA_STAGES * (DmmaLayout<DTA>::BYTES + DmmaLayout<DTB>::BYTES);
  static PerDeviceFlag configured;
  const int cfg_dev = PerDeviceFlag::current();
  if (!configured.test(cfg_dev)) {
    const cudaError_t e =
        cudaFuncSetAttribute(dmma_gemm_kernel<DTA, DTB, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured.set(cfg_dev);
  }
  dim3 grid(tiles, splits, batch);
  dmma_gemm_kernel<DTA, DTB, Epi><<<grid, 128, smem, stream>>>(A, B, M, N, K, syrk ? 1 : 0, tm, tn, splits, epi);
  return cudaGetLastError();
}

inline bool dmma_aligned(const SimtOperand& op) {
  const int e = dtype_size(op.dtype);
  return (reinterpret_cast<uintptr_t>(op.p) & 15) == 0 && (op.ld * e) % 16 == 0 && (op.bstride * e) % 16 == 0;
}

template <class Epi>
inline cudaError_t launch_simt_gemm(const SimtOperand& A, const SimtOperand& B, int M, int N, int K, int batch,
                                    bool syrk, int splits, const Epi& epi, cudaStream_t stream) {
  const int tm = (M + SIMT_BM - 1) / SIMT_BM, tn = (N + SIMT_BN - 1) / SIMT_BN;
  const int tiles = syrk ? tm * (tm + 1) / 2 : tm * tn;
  if (syrk && tm != tn) return cudaErrorInvalidValue;
  if (dmma_aligned(A) && dmma_aligned(B)) {
    const int da = A.dtype, db = B.dtype;
    if (da == DT_F64 && db == DT_F64) return launch_dmma<DT_F64, DT_F64>(A, B, M, N, K, batch, syrk, splits, epi, stream, tm, tn, tiles);
    if (da == DT_F32 && db == DT_F32) return launch_dmma<DT_F32, DT_F32>(A, B, M, N, K, batch, syrk, splits, epi, stream, tm, tn, tiles);
    if (da == DT_BF16 && db == DT_BF16) return launch_dmma<DT_BF16, DT_BF16>(A, B, M, N, K, batch, syrk, splits, epi, stream, tm, tn, tiles);
    if (da == DT_F32 && db == DT_F64) return launch_dmma<DT_F32, DT_F64>(A, B, M, N, K, batch, syrk, splits, epi, stream, tm, tn, tiles);
    if (da == DT_F64 && db == DT_F32) return launch_dmma<DT_F64, DT_F32>(A, B, M, N, K, batch, syrk, splits, epi, stream, tm, tn, tiles);
    if (da == DT_BF16 && db == DT_F64) return launch_dmma<DT_BF16, DT_F64>(A, B, M, N, K, batch, syrk, splits, epi, stream, tm, tn, tiles);
    if (da == DT_F64 && db == DT_BF16) return launch_dmma<DT_F64, DT_BF16>(A, B, M, N, K, batch, syrk, splits, epi, stream, tm, tn, tiles);
  }
  dim3 grid(tiles, splits, batch);
  simt_gemm_kernel<Epi><<<grid, 128, 0, stream>>>(A, B, M, N, K, syrk ? 1 : 0, tm, tn, splits, epi);
  return cudaGetLastError();
}

// Split K until the (tiles x splits x batch) grid covers ~4 CTAs per SM, keeping >= 8 k-tiles per split.
inline int simt_pick_splits(int tiles, int batch, int K) {
  const int ktiles = (K + SIMT_BK - 1) / SIMT_BK;
  int s = 1;
  while (static_cast<int64_t>(tiles) * batch * s < 4 * 148 && ktiles / (2 * s) >= 8 && s < 64) s *= 2;
  return s;
}

}  // namespace unso
