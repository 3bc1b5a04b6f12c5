// fp64-accumulating SIMT (DFMA) GEMM/SYRK engine: the "fp32 mode" of the
// orthogonalizer (parity <= 1e-5 needs fp64-grade Gram and squaring chain on
// ill-conditioned inputs), the Gelfand scaling products and
// the device-side orthogonality-error Gram.
//
//   D[b](m, n) = sum_k A[b](m, k) * B[b](n, k)        (fp64 accumulate)
//
// Each operand is a strided batch of row-major matrices read either K-major
// (element (i,k) at p[i*ld + k]) or MN-major (element (i,k) at p[k*ld + i]),
// stored as f32 / bf16 / f64.  `syrk` restricts the tile grid to tiles whose
// columns reach the diagonal (n >= m); the epilogue is only invoked on n >= m
// there.  `splits` partitions K; every (tile, split) is one CTA.
#pragma once
#include "common.cuh"

namespace unso {

struct SimtOperand {
  const void* p;
  int64_t ld;
  int64_t bstride;
  int dtype;
  int kmajor;
};

constexpr int SIMT_BM = 64, SIMT_BN = 64, SIMT_BK = 16;

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

template <class Epi>
__global__ void __launch_bounds__(256) simt_gemm_kernel(SimtOperand A, SimtOperand B, int M, int N, int K, int syrk,
                                                        int tiles_m, int tiles_n, int splits, Epi epi) {
  __shared__ double As[SIMT_BK][SIMT_BM + 1];
  __shared__ double Bs[SIMT_BK][SIMT_BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int split = blockIdx.y, b = blockIdx.z;
  int tm, tn;
  simt_tile_coords(blockIdx.x, tiles_m, tiles_n, syrk, tm, tn);
  const int m0 = tm * SIMT_BM, n0 = tn * SIMT_BN;
  const int ktiles = (K + SIMT_BK - 1) / SIMT_BK;
  const int kt0 = static_cast<int>(static_cast<int64_t>(split) * ktiles / splits);
  const int kt1 = static_cast<int>(static_cast<int64_t>(split + 1) * ktiles / splits);
  const char* pa = static_cast<const char*>(A.p) + static_cast<int64_t>(b) * A.bstride * dtype_size(A.dtype);
  const char* pb = static_cast<const char*>(B.p) + static_cast<int64_t>(b) * B.bstride * dtype_size(B.dtype);

  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  for (int kt = kt0; kt < kt1; ++kt) {
    const int k0 = kt * SIMT_BK;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + 256 * r;
      int i, k;
      // A tile: 64 rows x 16 k
      if (A.kmajor) { k = e & 15; i = e >> 4; } else { i = e & 63; k = e >> 6; }
      double va = 0.0;
      if (m0 + i < M && k0 + k < K) {
        const int64_t off = A.kmajor ? static_cast<int64_t>(m0 + i) * A.ld + (k0 + k)
                                     : static_cast<int64_t>(k0 + k) * A.ld + (m0 + i);
        va = load_as_f64(pa, off, A.dtype);
      }
      As[k][i] = va;
      if (B.kmajor) { k = e & 15; i = e >> 4; } else { i = e & 63; k = e >> 6; }
      double vb = 0.0;
      if (n0 + i < N && k0 + k < K) {
        const int64_t off = B.kmajor ? static_cast<int64_t>(n0 + i) * B.ld + (k0 + k)
                                     : static_cast<int64_t>(k0 + k) * B.ld + (n0 + i);
        vb = load_as_f64(pb, off, B.dtype);
      }
      Bs[k][i] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SIMT_BK; ++k) {
      double a[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      if (syrk && n < m) continue;
      epi(b, split, m, n, acc[i][j]);
    }
  }
}

template <class Epi>
inline cudaError_t launch_simt_gemm(const SimtOperand& A, const SimtOperand& B, int M, int N, int K, int batch,
                                    bool syrk, int splits, const Epi& epi, cudaStream_t stream) {
  const int tm = (M + SIMT_BM - 1) / SIMT_BM, tn = (N + SIMT_BN - 1) / SIMT_BN;
  const int tiles = syrk ? tm * (tm + 1) / 2 : tm * tn;
  if (syrk && tm != tn) return cudaErrorInvalidValue;
  dim3 grid(tiles, splits, batch);
  simt_gemm_kernel<Epi><<<grid, 256, 0, stream>>>(A, B, M, N, K, syrk ? 1 : 0, tm, tn, splits, epi);
  return cudaGetLastError();
}

// Heuristic: split K until the (tiles x splits x batch) grid covers ~2 waves of 148 SMs,
// keeping >= 8 k-tiles per split.
inline int simt_pick_splits(int tiles, int batch, int K) {
  const int ktiles = (K + SIMT_BK - 1) / SIMT_BK;
  int s = 1;
  while (static_cast<int64_t>(tiles) * batch * s < 296 && ktiles / (2 * s) >= 8 && s < 64) s *= 2;
  return s;
}

}  // namespace unso
