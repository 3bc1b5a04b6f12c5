// Two CTA pairs per cluster sharing the A operand through TMA multicast (non-SYRK GEMMs with
// K-major A, e.g. the tall apply Y = X R): pair p of a 4-CTA cluster computes the 256 x BN tile
// (tm, 2 j + p), so both pairs need the same 256 A rows per k-block.  CTA (p, r) loads the 64-row
// half p of its 128 A rows and multicasts it to CTAs r and r + 2; each CTA still loads its own B
// rows.  Per pair tile the L2 -> SM operand stream drops from A + B to A / 2 + B.
//
// Barriers: full[s] (pair leader, pair-local bytes: the multicast halves signal the leader of each
// destination pair through the cleared peer bit), empty[s] in every CTA counts the MMA commits of
// BOTH pairs (each issuer commits to all four CTAs), so a producer only overwrites a stage that
// both pairs have consumed.  Accumulator barriers stay pair-local.
// Same warp roles, epilogue interface and work filter as umma2_gemm.cuh.
#pragma once
#include "../../paper_2602_02500_b200/csrc/umma2_gemm.cuh"

namespace unso {

__device__ __forceinline__ void tma_load_3d_pair_mc(const CUtensorMap* m, uint32_t leader_bar, void* smem_dst, int c0,
                                                    int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

// Work item -> (b, tm, tile-column pair j); pair p computes tn = 2 j + p.
__device__ __forceinline__ void umma2mc_decode(const UmmaWork& w, int idx, int& b, int& tm, int& j) {
  const int tn2 = w.tiles_n >> 1;
  const int per = w.tiles_m * tn2;
  b = idx / per;
  const int t = idx - b * per;
  tm = t / tn2;
  j = t - tm * tn2;
}

// Cfg: Umma2Cfg with NA == NB == NT == 1, K-major A and B, no OPT.  tiles_n must be even.
template <class Cfg, class Epi>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    umma2mc_gemm_kernel(const __grid_constant__ CUtensorMap tmAhalf, const __grid_constant__ CUtensorMap tmB,
                        const UmmaWork work, const Epi epi) {
  static_assert(Cfg::NA == 1 && Cfg::NB == 1 && Cfg::NT == 1 && !Cfg::A_MN && !Cfg::B_MN && Cfg::OPT == 0,
                "multicast engine: single-term K-major GEMM");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();  // 0..3
  const int pair = static_cast<int>(crank >> 1);
  const uint32_t r = crank & 1u;
  const bool leader = r == 0;
  const uint32_t leader_rank = crank & ~1u;
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pair));
  const uint16_t a_mask = static_cast<uint16_t>((1u << r) | (1u << (r + 2)));
  const int cluster = blockIdx.x >> 2, nclusters = gridDim.x >> 2;
  const int num_work = work.batch * work.tiles_m * (work.tiles_n >> 1);
  if (work.mode_flag && work.mode_want >= 0) {  // all CTAs of the cluster see the same items
    bool any = false;                             // one flag read per matrix (items are batch-major)
    const int T = work.tiles_m * (work.tiles_n >> 1);
    const int blast = cluster < num_work ? (num_work - 1 - (num_work - 1 - cluster) % nclusters) / T : -1;
    for (int b = cluster < num_work ? cluster / T : 0; b <= blast && !any; ++b) {
      const int base = b * T;
      const int i0 = base + ((cluster - base) % nclusters + nclusters) % nclusters;
      if (i0 < base + T) any = !filtered_out(work, b);
    }
    if (!any) return;
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmAhalf);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);  // one commit from each pair
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * Cfg::EPI_WARPS);
    }
    fence_mbar_init();
  }
  cluster_sync_all();
  if (warp == 2) tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer (every CTA)
      const uint32_t lbar0 = leader_bar_addr(&full[0]);
      int stage = 0;
      uint32_t phase = 0;
      for (int idx = cluster; idx < num_work; idx += nclusters) {
        int b, tm, j;
        umma2mc_decode(work, idx, b, tm, j);
        if (filtered_out(work, b)) continue;
        const int tn = 2 * j + pair;
        const int arow = tm * Cfg::BM + static_cast<int>(r) * 128 + pair * 64;  // this CTA's A half
        const int brow = tn * Cfg::BN + static_cast<int>(r) * Cfg::HB;
        for (int kt = 0; kt < work.k_tiles; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          const uint32_t lbar = lbar0 + stage * 8;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
          tma_load_3d_pair_mc(&tmAhalf, lbar, st + pair * 8192, kt * 64, arow, b, a_mask);
          load_operand_tile_pair<false, Cfg::HB>(&tmB, lbar, st + Cfg::A_TILE, kt * 64, brow, b);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ------------------------------------------------------------ MMA issuer (pair leaders)
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int idx = cluster; idx < num_work; idx += nclusters) {
        int b, tm, j;
        umma2mc_decode(work, idx, b, tm, j);
        if (filtered_out(work, b)) continue;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * Cfg::BN);
        for (int kt = 0; kt < work.k_tiles; ++kt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * Cfg::STAGE_BYTES);
#pragma unroll
          for (int ks = 0; ks < Cfg::BK / 16; ++ks)
            umma_bf16_pair(d_tmem, operand_desc<false>(st, ks), operand_desc<false>(st + Cfg::A_TILE, ks), Cfg::IDESC,
                           (kt > 0 || ks > 0) ? 1u : 0u);
          umma_commit_pair(&empty[stage], 0xF);  // both pairs' producers wait on this stage
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull[acc], pair_mask);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue (every CTA)
    const int ew = warp - 4;
    const int q = warp & 3;
    constexpr int GROUPS = Cfg::EPI_WARPS / 4;
    constexpr int CPG = Cfg::BN / 32 / GROUPS;
    const int c0 = (ew / 4) * CPG;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int idx = cluster; idx < num_work; idx += nclusters) {
      int b, tm, j;
      umma2mc_decode(work, idx, b, tm, j);
      if (filtered_out(work, b)) continue;
      const int tn = 2 * j + pair;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = tm * Cfg::BM + static_cast<int>(r) * 128 + q * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * Cfg::BN);
#pragma unroll 1
      for (int c = c0; c < c0 + CPG; ++c) {
        uint32_t rr[32];
        tmem_ld32(taddr + c * 32, rr);
        tmem_wait_ld();
        float v[32];
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) v[jj] = __uint_as_float(rr[jj]);
        epi(b, 0, row, tn * Cfg::BN + c * 32, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[acc], leader_rank);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
  }
}

template <class Cfg, class Epi>
inline cudaError_t launch_umma2mc(const CUtensorMap& ahalf, const CUtensorMap& b, const UmmaWork& w, const Epi& epi,
                                  cudaStream_t stream) {
  static int max_clusters = -1;
  if (max_clusters < 0) {
    cudaError_t e = cudaFuncSetAttribute(umma2mc_gemm_kernel<Cfg, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(4 * 64);
    q.blockDim = dim3(Cfg::THREADS);
    q.dynamicSmemBytes = Cfg::SMEM;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = 4;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, umma2mc_gemm_kernel<Cfg, Epi>, &q);
    if (e != cudaSuccess || n < 1) return e != cudaSuccess ? e : cudaErrorInvalidConfiguration;
    max_clusters = n;
  }
  const int num_work = w.batch * w.tiles_m * (w.tiles_n >> 1);
  if (num_work <= 0) return cudaSuccess;
  const int nclusters = num_work < max_clusters ? num_work : max_clusters;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(4 * nclusters));
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 4;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, umma2mc_gemm_kernel<Cfg, Epi>, ahalf, b, w, epi);
}

}  // namespace unso
