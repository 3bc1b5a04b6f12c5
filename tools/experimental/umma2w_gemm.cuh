// EXPERIMENT (not used by default): 256 x 512 pair tiles for the single-term K-major GEMM (tall
// apply).  Each CTA stages 128 A rows and two 128-row B halves per k-block (48 KB) and issues two
// N = 256 MMAs per k-step into the two 256-column halves of one 512-column TMEM accumulator:
// 25 % fewer operand bytes per FLOP than the 256 x 256 tile.  The accumulator is single-buffered:
// the next tile's MMAs wait until the epilogue has drained it (the cost this prototype measures).
#pragma once
#include "umma2_gemm.cuh"

namespace unso {

constexpr int UW_STAGES = 4;
constexpr int UW_TILE = 128 * 64 * 2;            // 16 KB: 128 rows x 64 K of bf16
constexpr int UW_STAGE_BYTES = 3 * UW_TILE;      // A, B half 0, B half 1 (per CTA)
constexpr int UW_EPI_WARPS = 8;
constexpr int UW_THREADS = 128 + 32 * UW_EPI_WARPS;
constexpr int UW_STAGING = UW_EPI_WARPS * 32 * 32 * 4;  // one 4 KB 32 x 32 fp32 block per epilogue warp
constexpr int UW_SMEM = UW_STAGES * UW_STAGE_BYTES + 256 + UW_STAGING + 1024;
static_assert(UW_SMEM <= 227 * 1024, "smem budget");
static_assert(UW_EPI_WARPS == 8, "warps 4-7 drain column half 0, 8-11 half 1");

template <class E, class = void>
struct epi_has_split : std::false_type {};
template <class E>
struct epi_has_split<E, std::void_t<decltype(&E::split_ok)>> : std::true_type {};

template <class Epi>
__global__ void __launch_bounds__(UW_THREADS, 1)
    umma2w_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const UmmaWork work, const Epi epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + UW_STAGES * UW_STAGE_BYTES);
  uint64_t* empty = full + UW_STAGES;
  uint64_t* tfull = empty + UW_STAGES;   // [2]: column half h accumulated
  uint64_t* tempty = tfull + 2;          // [2]: column half h drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const uint32_t IDESC = idesc_bf16(256, 256, 0, 0);
  const int tiles_n = work.tiles_n;  // 512-wide column blocks
  const int per_mat = work.tiles_m * tiles_n;
  const int num_work = work.batch * per_mat;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < UW_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&tfull[h], 1);
      mbar_init(&tempty[h], 2 * (UW_EPI_WARPS / 2));  // the half's epilogue warps of both CTAs
    }
    fence_mbar_init();
  }
  cluster_sync_all();
  if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t lbar0 = leader_bar_addr(&full[0]);
      int stage = 0;
      uint32_t phase = 0;
      for (int idx = cluster; idx < num_work; idx += nclusters) {
        const int b = idx / per_mat;
        int tm, tn;
        umma_grouped_coords(idx - b * per_mat, work.tiles_m, tiles_n, tm, tn);
        const int arow = tm * 256 + static_cast<int>(rank) * 128;
        const int brow0 = tn * 512 + static_cast<int>(rank) * 128, brow1 = brow0 + 256;
        for (int kt = 0; kt < work.k_tiles; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * UW_STAGE_BYTES;
          const uint32_t lbar = lbar0 + stage * 8;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * UW_STAGE_BYTES);
          tma_load_3d_pair(&tmA, lbar, st, kt * 64, arow, b);
          tma_load_3d_pair(&tmB, lbar, st + UW_TILE, kt * 64, brow0, b);
          tma_load_3d_pair(&tmB, lbar, st + 2 * UW_TILE, kt * 64, brow1, b);
          if (++stage == UW_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // Half-by-half hand-off: the first KP k-blocks of a tile run their half-0 MMAs as soon as
      // half 0 is drained, and their half-1 MMAs (operands still in the stages) once half 1 is.
      int stage = 0;
      uint32_t phase = 0, tph = 0;
      const int K = work.k_tiles, KP = K < UW_STAGES ? K : UW_STAGES;
      auto mma_half = [&](int st_idx, int h, int kt) {
        const uint32_t st = smem_u32(smem + st_idx * UW_STAGE_BYTES);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_bf16_pair(tmem_base + 256 * h, operand_desc<false>(st, ks),
                         operand_desc<false>(st + (1 + h) * UW_TILE, ks), IDESC, (kt > 0 || ks > 0) ? 1u : 0u);
      };
      for (int idx = cluster; idx < num_work; idx += nclusters) {
        const int s0 = stage;
        const uint32_t p0 = phase;
        mbar_wait(&tempty[0], tph ^ 1);
        tc_fence_after();
        for (int kt = 0; kt < KP; ++kt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          mma_half(stage, 0, kt);
          if (++stage == UW_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (KP == K) umma_commit_pair(&tfull[0], 0x3);
        mbar_wait(&tempty[1], tph ^ 1);
        tc_fence_after();
        stage = s0;
        phase = p0;
        for (int kt = 0; kt < KP; ++kt) {
          mma_half(stage, 1, kt);
          umma_commit_pair(&empty[stage], 0x3);
          if (++stage == UW_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        for (int kt = KP; kt < K; ++kt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          mma_half(stage, 0, kt);
          if (kt == K - 1) umma_commit_pair(&tfull[0], 0x3);
          mma_half(stage, 1, kt);
          umma_commit_pair(&empty[stage], 0x3);
          if (++stage == UW_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull[1], 0x3);
        tph ^= 1;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // Epilogue: warps 4-7 drain column half 0, warps 8-11 half 1 (lane quarter = warp % 4); each
    // warp's 8 chunks are software-pipelined (TMEM load and X prefetch one chunk ahead).
    const int ew = warp - 4, q = warp & 3, h = ew / 4;
    uint32_t tph = 0;
    for (int idx = cluster; idx < num_work; idx += nclusters) {
      const int b = idx / per_mat;
      int tm, tn;
      umma_grouped_coords(idx - b * per_mat, work.tiles_m, tiles_n, tm, tn);
      mbar_wait(&tfull[h], tph);
      tph ^= 1;
      tc_fence_after();
      const int row = tm * 256 + static_cast<int>(rank) * 128 + q * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + 256 * h;
      const int colbase = tn * 512 + 256 * h;
      bool fast = false;
      if constexpr (epi_has_split<Epi>::value) fast = __all_sync(0xffffffffu, epi.split_ok(b, row, colbase));
      if (fast) {
        if constexpr (epi_has_split<Epi>::value) {
          float* stg = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256) + ew * 1024;
#pragma unroll 1
          for (int c = 0; c < 8; ++c) {
            uint32_t r[32];
            tmem_ld32(taddr + c * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<uint4*>(stg + lane * 32 + ((j ^ (lane & 7)) << 2)) =
                  make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
            __syncwarp();
            epi.rows4_wide(b, row - lane, colbase + c * 32, stg);
            __syncwarp();
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          uint32_t r[32];
          tmem_ld32(taddr + c * 32, r);
          tmem_wait_ld();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          epi(b, 0, row, colbase + c * 32, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[h], 0);
    }
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

template <class Epi>
inline cudaError_t launch_umma2w(const CUtensorMap& a, const CUtensorMap& b, const UmmaWork& w, const Epi& epi,
                                 cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(umma2w_gemm_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, UW_SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int num_work = w.batch * w.tiles_m * w.tiles_n;
  const int pairs = device_sm_count() / 2;
  const int nclusters = num_work < pairs ? num_work : pairs;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * nclusters));
  cfg.blockDim = dim3(UW_THREADS);
  cfg.dynamicSmemBytes = UW_SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, umma2w_gemm_kernel<Epi>, a, b, w, epi);
}

}  // namespace unso
