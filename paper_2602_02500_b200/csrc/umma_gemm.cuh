// Reference contractions: as umma2_gemm.cuh (ortho.py:156, 198, 205, 215-230), 1-CTA tiles.
// tcgen05 / TMEM / TMA GEMM-SYRK engine for sm_100a (bf16 operands, f32 accumulate).
//
//   D[b](m, n) = sum_t sum_k A_{a(t)}[b](m, k) * B_{b(t)}[b](n, k)
//
// One persistent CTA per SM, 8 warps, warp-specialised:
//   warp 0 (1 lane)  TMA producer: per k-block loads NA A-tiles (128 x 64) and NB
//                    B-tiles (BN x 64) into one smem stage (SWIZZLE_128B).
//   warp 1 (1 lane)  MMA issuer: NT "terms" (A_i, B_j) per k-step, all into the same
//                    TMEM accumulator -> bf16x3 (hi*hi + hi*lo + lo*hi) and bf16x2
//                    (x*P_hi + x*P_lo) products cost no extra smem traffic.
//   warp 2           TMEM allocator (2 x BN columns: double-buffered accumulator).
//   warps 4..7       epilogue: tcgen05.ld 32 lanes x 32 columns -> functor.
// Operands are K-major (row-major rows x K) or MN-major (row-major K x MN, read
// transposed by the tensor core through the descriptor's major bit) -- the tall
// Gram X^T X therefore needs no transpose pass.
// Work items = (batch, split-K, tile); `syrk` keeps only tiles with tn >= tm (BN == 128).
#pragma once
#include "common.cuh"
#include "ptx_sm100.cuh"
#include "simt_gemm.cuh"

namespace unso {

struct UmmaWork {
  int tiles_m, tiles_n, syrk, splits, k_tiles, batch, tiles_valid, num_work;
  // Optional second operand tile (CTA-pair engine, Cfg::OPT != 0): skipped for matrix b when
  // opt_skip[b * opt_stride] != 0 (device-side decision written by an earlier kernel).
  const double* opt_skip = nullptr;
  int opt_stride = 0;
  // Work filter (CTA-pair engine): when mode_flag is set, only matrices b with
  // (mode_flag[b * opt_stride] != 0) == (mode_want == 1) are processed by this launch.
  const double* mode_flag = nullptr;
  int mode_want = -1;
  // Squaring-chain kernels (chain_pair.cuh): 1 = accumulate the hi*hi product only (no lo / e4m3
  // cross terms, their operand tiles are not loaded) -- the first squarings of the chain.
  int no_cross = 0;
  // SYRK launches whose A and B maps are the same tensor (the Gram X^T X): a diagonal tile's B rows
  // are its A rows, so the pair engine loads one copy and points both descriptors at it.
  int diag_share = 0;
};

// Non-SYRK tile order: groups of UMMA_GROUP_M row blocks, row block fastest within a group, so the
// ~74 tiles in flight touch UMMA_GROUP_M A row blocks and ~74 / UMMA_GROUP_M B column blocks (an
// L2-sized working set when A and B are both large, e.g. the apply of configs[4]: P is then read
// from DRAM once per group instead of once per row block).
constexpr int UMMA_GROUP_M = 8;
__device__ __forceinline__ void umma_grouped_coords(int t, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int per_group = UMMA_GROUP_M * tiles_n;
  const int g = t / per_group;
  const int r = t - g * per_group;
  const int rows = min(UMMA_GROUP_M, tiles_m - g * UMMA_GROUP_M);
  tn = r / rows;
  tm = g * UMMA_GROUP_M + (r - tn * rows);
}

__device__ __forceinline__ void umma_decode(const UmmaWork& w, int idx, int& b, int& split, int& tm, int& tn,
                                            int& kt0, int& kt1) {
  const int t = idx % w.tiles_valid;
  const int r = idx / w.tiles_valid;
  split = r % w.splits;
  b = r / w.splits;
  if (!w.syrk)
    umma_grouped_coords(t, w.tiles_m, w.tiles_n, tm, tn);
  else
    simt_tile_coords(t, w.tiles_m, w.tiles_n, 1, tm, tn);
  kt0 = static_cast<int>(static_cast<int64_t>(split) * w.k_tiles / w.splits);
  kt1 = static_cast<int>(static_cast<int64_t>(split + 1) * w.k_tiles / w.splits);
}

template <int BN_, int NA_, int NB_, int NT_, int TERMS_, bool A_MN_, bool B_MN_, int STAGES_>
struct UmmaCfg {
  static constexpr int BM = 128, BN = BN_, BK = 64;
  static constexpr int NA = NA_, NB = NB_, NT = NT_, TERMS = TERMS_, STAGES = STAGES_;
  static constexpr bool A_MN = A_MN_, B_MN = B_MN_;
  static constexpr int A_TILE = BM * BK * 2;
  static constexpr int B_TILE = BN * BK * 2;
  static constexpr int STAGE_BYTES = NA * A_TILE + NB * B_TILE;
  static constexpr int BAR_BYTES = 256;
  static constexpr int SMEM = STAGES * STAGE_BYTES + BAR_BYTES + 1024;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr uint32_t IDESC = idesc_bf16(BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
  static_assert(BN == 128 || BN == 256, "BN");
  static_assert(SMEM <= 227 * 1024, "smem budget");
  static_assert(TMEM_COLS <= 512, "tmem budget");
};

// term t uses A-tile (TERMS >> 2t) & 1 and B-tile (TERMS >> (2t+1)) & 1
constexpr int TERM(int t, int a, int b) { return (a | (b << 1)) << (2 * t); }

template <bool MN, int ROWS>
__device__ __forceinline__ void load_operand_tile(const CUtensorMap* map, uint64_t* bar, uint8_t* dst, int k0,
                                                  int r0, int b) {
  if constexpr (!MN) {
    tma_load_3d(map, bar, dst, k0, r0, b);  // box {64 (K), ROWS, 1}
  } else {
#pragma unroll
    for (int c = 0; c < ROWS / 64; ++c) tma_load_3d(map, bar, dst + c * 8192, r0 + c * 64, k0, b);  // box {64, 64, 1}
  }
}

template <bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t tile_addr, int ks) {
  // K-major: advance 16 bf16 (32 B) inside the 128 B swizzle row.
  // MN-major: advance 16 K-rows (2 x 1024 B groups); 64-wide MN chunks are 8 KB apart.
  return MN ? sdesc_sw128(tile_addr + ks * 2048, 8192, 1024) : sdesc_sw128(tile_addr + ks * 32, 16, 1024);
}

// e4m3 operand tile of a 128-row block (chain kernels): K-major = one SWIZZLE_128B box of
// 128 rows x [hi8 k0..63 | lo8 k0..63]; MN-major = hi8 plane (64 K-rows x 128 B) then lo8 plane.
// Descriptor of the hi8 (lo = 0) or lo8 (lo = 1) operand, MMA k-step ks (32 e4m3 each).
__device__ __forceinline__ uint64_t f8_desc(uint32_t tile, bool mn, int lo, int ks) {
  return mn ? sdesc_sw128(tile + lo * 8192 + ks * 4096, 8192, 1024)   // 32 K-rows of 128 B
            : sdesc_sw128(tile + lo * 64 + ks * 32, 16, 1024);        // 32 B inside the 128 B row
}

template <class Cfg, class Epi>
__global__ void __launch_bounds__(256, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                     const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmB1,
                     const UmmaWork work, const Epi epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA0);
    if (Cfg::NA > 1) tma_prefetch_desc(&tmA1);
    tma_prefetch_desc(&tmB0);
    if (Cfg::NB > 1) tma_prefetch_desc(&tmB1);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int idx = blockIdx.x; idx < work.num_work; idx += gridDim.x) {
        int b, split, tm, tn, kt0, kt1;
        umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          load_operand_tile<Cfg::A_MN, Cfg::BM>(&tmA0, &full[stage], st, kt * 64, tm * Cfg::BM, b);
          if (Cfg::NA > 1)
            load_operand_tile<Cfg::A_MN, Cfg::BM>(&tmA1, &full[stage], st + Cfg::A_TILE, kt * 64, tm * Cfg::BM, b);
          uint8_t* sb = st + Cfg::NA * Cfg::A_TILE;
          load_operand_tile<Cfg::B_MN, Cfg::BN>(&tmB0, &full[stage], sb, kt * 64, tn * Cfg::BN, b);
          if (Cfg::NB > 1)
            load_operand_tile<Cfg::B_MN, Cfg::BN>(&tmB1, &full[stage], sb + Cfg::B_TILE, kt * 64, tn * Cfg::BN, b);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int idx = blockIdx.x; idx < work.num_work; idx += gridDim.x) {
        int b, split, tm, tn, kt0, kt1;
        umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * Cfg::BN);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = st + Cfg::NA * Cfg::A_TILE;
#pragma unroll
          for (int ks = 0; ks < Cfg::BK / 16; ++ks) {
#pragma unroll
            for (int t = 0; t < Cfg::NT; ++t) {
              const int ai = (Cfg::TERMS >> (2 * t)) & 1;
              const int bi = (Cfg::TERMS >> (2 * t + 1)) & 1;
              const uint64_t ad = operand_desc<Cfg::A_MN>(st + ai * Cfg::A_TILE, ks);
              const uint64_t bd = operand_desc<Cfg::B_MN>(sb + bi * Cfg::B_TILE, ks);
              umma_bf16(d_tmem, ad, bd, Cfg::IDESC, (kt > kt0 || ks > 0 || t > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[stage]);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int ew = warp - 4;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int idx = blockIdx.x; idx < work.num_work; idx += gridDim.x) {
      int b, split, tm, tn, kt0, kt1;
      umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = tm * Cfg::BM + ew * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * Cfg::BN);
#pragma unroll 1
      for (int c = 0; c < Cfg::BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(taddr + c * 32, r);
        tmem_wait_ld();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        epi(b, split, row, tn * Cfg::BN + c * 32, v);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// -------------------------------------------------------------------- host side
bool umma_make_kmajor_map(CUtensorMap* m, const void* base, int64_t rows, int64_t k, int64_t ld, int64_t batch,
                          int64_t bstride, int box_rows);
bool umma_make_mnmajor_map(CUtensorMap* m, const void* base, int64_t krows, int64_t mn, int64_t ld, int64_t batch,
                           int64_t bstride);
int device_sm_count();

inline UmmaWork umma_make_work(int M, int N, int K, int BN, int batch, bool syrk, int splits) {
  UmmaWork w;
  w.tiles_m = (M + 127) / 128;
  w.tiles_n = (N + BN - 1) / BN;
  w.syrk = syrk ? 1 : 0;
  w.k_tiles = (K + 63) / 64;
  w.splits = splits < 1 ? 1 : (splits > w.k_tiles ? w.k_tiles : splits);
  w.batch = batch;
  w.tiles_valid = syrk ? w.tiles_m * (w.tiles_m + 1) / 2 : w.tiles_m * w.tiles_n;
  w.num_work = w.tiles_valid * w.splits * batch;
  return w;
}

template <class Cfg, class Epi>
inline cudaError_t launch_umma(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
                               const CUtensorMap& b1, const UmmaWork& w, const Epi& epi, cudaStream_t stream) {
  static PerDeviceFlag configured;
  const int cfg_dev = PerDeviceFlag::current();
  if (!configured.test(cfg_dev)) {
    cudaError_t e = cudaFuncSetAttribute(umma_gemm_kernel<Cfg, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM);
    if (e != cudaSuccess) return e;
    configured.set(cfg_dev);
  }
  if (w.num_work <= 0) return cudaSuccess;
  const int sms = device_sm_count();
  const int grid = w.num_work < sms ? w.num_work : sms;
  umma_gemm_kernel<Cfg, Epi><<<grid, 256, Cfg::SMEM, stream>>>(a0, a1, b0, b1, w, epi);
  return cudaGetLastError();
}

}  // namespace unso
