// Reference contractions: the Gram densemat.matmul(a, transpose(a)) (ortho.py:156, 198) as a SYRK,
// the apply P.X (ortho.py:205) in the tall form Y = X P, and the NS products (ortho.py:215-230).
// CTA-pair (cta_group::2) tcgen05 engine: a cluster of 2 CTAs on one TPC computes a
// 256 x BN tile with M=256 MMAs issued by the leader CTA.  Each CTA stages its own
// 128 A-rows and BN/2 B-rows per k-block (TMA .cta_group::2, completion on the
// leader's mbarrier), so per-SM operand traffic per FLOP is half that of the 1-CTA
// 128 x 128 tile -- the lever against the ~60 B/clk/SM L2->SMEM ingest limit seen in
// ncu (profiles/round1_ncu_summary.md).  Accumulator: rows [128r, 128r+128) of the
// 256 x BN tile live in CTA r's TMEM (double-buffered, 2 x BN columns).
//
// Warp roles: 0 TMA producer (both CTAs), 1 MMA issuer (leader), 2 TMEM allocator,
// 3 idle, 4.. epilogue (EPI_WARPS warps: warp w reads TMEM lanes 32*(w%4).., the
// (w-4)/4-th column group of the tile), so the epilogue of one tile overlaps the
// mainloop of the next even when the tile's K-loop is short.
//
// Same term/operand conventions as umma_gemm.cuh; the epilogue functor receives
// (b, split, row, col0, v[32]) for the CTA's own rows.
#pragma once
#include <type_traits>

#include "umma_gemm.cuh"

namespace unso {

// OPT: 0 = all tiles always used; 1 = B tile 1 optional; 2 = A tile 1 optional (see UmmaWork::opt_skip).
template <int BN_, int NA_, int NB_, int NT_, int TERMS_, bool A_MN_, bool B_MN_, int STAGES_, int OPT_ = 0,
          int EPI_WARPS_ = 8>
struct Umma2Cfg {
  static constexpr int BM = 256, BN = BN_, BK = 64;       // pair tile
  static constexpr int HB = BN / 2;                        // B rows per CTA
  static constexpr int NA = NA_, NB = NB_, NT = NT_, TERMS = TERMS_, STAGES = STAGES_, OPT = OPT_;
  static constexpr int EPI_WARPS = EPI_WARPS_;
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr bool A_MN = A_MN_, B_MN = B_MN_;
  static constexpr int A_TILE = 128 * BK * 2;
  static constexpr int B_TILE = HB * BK * 2;
  static constexpr int STAGE_BYTES = NA * A_TILE + NB * B_TILE;  // per CTA
  static constexpr int SMEM = STAGES * STAGE_BYTES + 256 + 1024;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr uint32_t IDESC = idesc_bf16(256, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
  static_assert(BN == 128 || BN == 256, "BN");
  static_assert(EPI_WARPS == 4 || EPI_WARPS == 8, "epilogue warps");
  static_assert((BN / 32) % (EPI_WARPS / 4) == 0, "column groups");
  static_assert(SMEM <= 227 * 1024, "smem budget");
  static_assert(TMEM_COLS <= 512, "tmem budget");
};

template <bool MN, int ROWS>
__device__ __forceinline__ void load_operand_tile_pair(const CUtensorMap* map, uint32_t lbar, uint8_t* dst, int k0,
                                                       int r0, int b) {
  if constexpr (!MN) {
    tma_load_3d_pair(map, lbar, dst, k0, r0, b);
  } else {
#pragma unroll
    for (int c = 0; c < ROWS / 64; ++c) tma_load_3d_pair(map, lbar, dst + c * 8192, r0 + c * 64, k0, b);
  }
}

__device__ __forceinline__ bool opt_skipped(const UmmaWork& w, int b) {
  return w.opt_skip && w.opt_skip[static_cast<int64_t>(b) * w.opt_stride] != 0.0;
}
// Every role evaluates the same predicate on the same data, so all skip the same work items.
__device__ __forceinline__ bool filtered_out(const UmmaWork& w, int b) {
  if (!w.mode_flag || w.mode_want < 0) return false;
  return (w.mode_flag[static_cast<int64_t>(b) * w.opt_stride] != 0.0) != (w.mode_want == 1);
}

// Epilogues with a rows4(b, split, row0, col0, stage) member take the accumulator through shared memory.
template <class E, class = void>
struct epi_has_rows4 : std::false_type {};
template <class E>
struct epi_has_rows4<E, std::void_t<decltype(&E::rows4)>> : std::true_type {};

// lane = row: the lane's 32 accumulator columns go to the warp's 4 KB block, 16-byte chunk j at slot
// j ^ (row & 7) (conflict-free for these row-wise writes and for rows4's 4-rows-per-instruction
// reads), then the epilogue re-reads the block with lanes spread along the columns.
template <class Epi>
__device__ __forceinline__ void stage_block32(const Epi& epi, float* stage, int b, int split, int row0, int col0,
                                              const float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<float4*>(stage + lane * 32 + ((j ^ (lane & 7)) << 2)) =
        make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  __syncwarp();
  epi.rows4(b, split, row0, col0, stage);
  __syncwarp();
}

template <class Cfg, class Epi>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    umma2_gemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
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
  // diagonal SYRK tiles of a same-tensor product can share one operand copy when A and B tiles have
  // the same shape, major and count (each CTA's B half is then exactly its A half)
  constexpr bool kDiagShare = Cfg::OPT == 0 && Cfg::A_MN == Cfg::B_MN && Cfg::NA == Cfg::NB &&
                              Cfg::A_TILE == Cfg::B_TILE && Cfg::BM == Cfg::BN;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  if (work.mode_flag && work.mode_want >= 0) {
    // Both CTAs of the pair see the same items: if none passes the filter, leave before any
    // barrier / TMEM setup (the companion launch of the adaptive apply then costs ~a launch).
    // Items are batch-major (T per matrix): walk the matrices this cluster has items in, one flag
    // read per matrix (not per item: an all-filtered launch then costs ~a launch).
    bool any = false;
    const int T = work.num_work / work.batch;
    const int blast = (cluster < work.num_work) ? (work.num_work - 1 - (work.num_work - 1 - cluster) % nclusters) / T : -1;
    for (int b = (cluster < work.num_work ? cluster / T : 0); b <= blast && !any; ++b) {
      const int base = b * T;
      const int i0 = base + ((cluster - base) % nclusters + nclusters) % nclusters;
      if (i0 < base + T) any = !filtered_out(work, b);
    }
    if (!any) return;
  }

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
      mbar_init(&tempty[a], 2 * Cfg::EPI_WARPS);  // every epilogue warp of both CTAs
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
      // ------------------------------------------------------------ TMA producer (both CTAs)
      const uint32_t lbar0 = leader_bar_addr(&full[0]);
      int stage = 0;
      uint32_t phase = 0;
      for (int idx = cluster; idx < work.num_work; idx += nclusters) {
        int b, split, tm, tn, kt0, kt1;
        umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
        if (filtered_out(work, b)) continue;
        const int arow = tm * Cfg::BM + static_cast<int>(rank) * 128;
        const int brow = tn * Cfg::BN + static_cast<int>(rank) * Cfg::HB;
        const bool skip = Cfg::OPT != 0 && opt_skipped(work, b);
        const bool dshare = kDiagShare && work.diag_share && tm == tn;  // B rows = A rows: one copy
        const uint32_t bytes = dshare ? 2 * Cfg::NA * Cfg::A_TILE
                                      : 2 * (Cfg::STAGE_BYTES - (skip ? (Cfg::OPT == 1 ? Cfg::B_TILE : Cfg::A_TILE) : 0));
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          const uint32_t lbar = lbar0 + stage * 8;
          if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
          load_operand_tile_pair<Cfg::A_MN, 128>(&tmA0, lbar, st, kt * 64, arow, b);
          if (Cfg::NA > 1 && !(skip && Cfg::OPT == 2))
            load_operand_tile_pair<Cfg::A_MN, 128>(&tmA1, lbar, st + Cfg::A_TILE, kt * 64, arow, b);
          uint8_t* sb = st + Cfg::NA * Cfg::A_TILE;
          if (!dshare) {
            load_operand_tile_pair<Cfg::B_MN, Cfg::HB>(&tmB0, lbar, sb, kt * 64, brow, b);
            if (Cfg::NB > 1 && !(skip && Cfg::OPT == 1))
              load_operand_tile_pair<Cfg::B_MN, Cfg::HB>(&tmB1, lbar, sb + Cfg::B_TILE, kt * 64, brow, b);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (leader only): the whole
      // warp walks the loop, one elected lane issues (descriptors stay in uniform registers)
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int idx = cluster; idx < work.num_work; idx += nclusters) {
        int b, split, tm, tn, kt0, kt1;
        umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
        if (filtered_out(work, b)) continue;
        const bool skip = Cfg::OPT != 0 && opt_skipped(work, b);
        const bool dshare = kDiagShare && work.diag_share && tm == tn;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * Cfg::BN);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = dshare ? st : st + Cfg::NA * Cfg::A_TILE;
#pragma unroll
          for (int ks = 0; ks < Cfg::BK / 16; ++ks) {
#pragma unroll
            for (int t = 0; t < Cfg::NT; ++t) {
              const int ai = (Cfg::TERMS >> (2 * t)) & 1;
              const int bi = (Cfg::TERMS >> (2 * t + 1)) & 1;
              if (skip && ((Cfg::OPT == 1 && bi == 1) || (Cfg::OPT == 2 && ai == 1))) continue;
              const uint64_t ad = operand_desc<Cfg::A_MN>(st + ai * Cfg::A_TILE, ks);
              const uint64_t bd = operand_desc<Cfg::B_MN>(sb + bi * Cfg::B_TILE, ks);
              umma_bf16_pair_warp(d_tmem, ad, bd, Cfg::IDESC, (kt > kt0 || ks > 0 || t > 0) ? 1u : 0u);
            }
          }
          umma_commit_pair_warp(&empty[stage], 0x3);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair_warp(&tfull[acc], 0x3);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue (both CTAs)
    const int ew = warp - 4;
    const int q = warp & 3;                         // TMEM lane quarter this warp may access
    constexpr int GROUPS = Cfg::EPI_WARPS / 4;      // column groups
    constexpr int CPG = Cfg::BN / 32 / GROUPS;      // 32-column chunks per group
    const int c0 = (ew / 4) * CPG;
    float* stg = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256) + ew * 1024;
    (void)stg;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int idx = cluster; idx < work.num_work; idx += nclusters) {
      int b, split, tm, tn, kt0, kt1;
      umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
      if (filtered_out(work, b)) continue;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = tm * Cfg::BM + static_cast<int>(rank) * 128 + q * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * Cfg::BN);
#pragma unroll 1
      for (int c = c0; c < c0 + CPG; ++c) {
        uint32_t r[32];
        tmem_ld32(taddr + c * 32, r);
        tmem_wait_ld();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if constexpr (epi_has_rows4<Epi>::value)
          stage_block32(epi, stg, b, split, row - lane, tn * Cfg::BN + c * 32, v);
        else
          epi(b, split, row, tn * Cfg::BN + c * 32, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
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

inline UmmaWork umma2_make_work(int M, int N, int K, int BN, int batch, bool syrk, int splits) {
  UmmaWork w;
  w.tiles_m = (M + 255) / 256;
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
inline cudaError_t launch_umma2(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
                                const CUtensorMap& b1, const UmmaWork& w, const Epi& epi, cudaStream_t stream) {
  constexpr int smem = Cfg::SMEM + (epi_has_rows4<Epi>::value ? Cfg::EPI_WARPS * 4096 : 0);
  static_assert(smem <= 227 * 1024, "smem budget with the epilogue staging blocks");
  static PerDeviceFlag configured;
  const int cfg_dev = PerDeviceFlag::current();
  if (!configured.test(cfg_dev)) {
    cudaError_t e = cudaFuncSetAttribute(umma2_gemm_kernel<Cfg, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
    if (e != cudaSuccess) return e;
    configured.set(cfg_dev);
  }
  if (w.num_work <= 0) return cudaSuccess;
  const int pairs = device_sm_count() / 2;
  const int nclusters = w.num_work < pairs ? w.num_work : pairs;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * nclusters));
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, umma2_gemm_kernel<Cfg, Epi>, a0, a1, b0, b1, w, epi);
}

}  // namespace unso
