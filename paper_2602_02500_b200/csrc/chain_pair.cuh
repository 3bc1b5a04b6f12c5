// Reference: one iteration of unso()'s loop (ortho.py:201-203: P += a_k B_k; B <- B B) in the
// C-form C = I - B (identical in exact arithmetic), for every matrix of the batch.
// One C-form squaring step for large h (tiles > co-resident CTAs), on CTA pairs:
//   C_{k+1} = 2 C_k - C_k^2 (upper 256 x 256 pair tiles only), P -= c_{k+1} C_{k+1}
// with the bf16x3 split product hi*hi + hi*lo + lo*hi accumulated in TMEM.
//
// Only upper pair tiles of C are ever stored.  Row block I of C at k-slice kt is read
// directly (K-major TMA of stored tile (I, kt/4)) when kt/4 >= I and transposed
// (MN-major TMA of stored tile (kt/4, I)) otherwise; the tcgen05 instruction
// descriptor's A/B major bits follow per k-block.  Diagonal pair tiles are written in
// full (both triangles) because direct reads of a diagonal block touch both.
// Batch: one launch per step for every matrix of the batch (work = batch x upper tiles).
#pragma once
#include "umma2_gemm.cuh"

namespace unso {

struct SymMaps {
  CUtensorMap hiK, loK, hiMN, loMN;  // C_k hi/lo: K-major box {64,128}, MN-major box {64,64}
};

constexpr int SC_STAGES = 3;
constexpr int SC_TILE = 128 * 64 * 2;
constexpr int SC_STAGE_BYTES = 4 * SC_TILE;  // A hi, A lo, B hi, B lo (per CTA)
constexpr int SC_EPI_WARPS = 8;
constexpr int SC_THREADS = 128 + 32 * SC_EPI_WARPS;
constexpr int SC_STAGING = SC_EPI_WARPS * 32 * 32 * 4;  // one 4 KB 32 x 32 fp32 block per epilogue warp
constexpr int SC_SMEM = SC_STAGES * SC_STAGE_BYTES + 256 + SC_STAGING + 1024;


__device__ __forceinline__ void sc_load(const CUtensorMap* kmap, const CUtensorMap* mnmap, uint32_t lbar,
                                        uint8_t* dst, int blk256, int row0, int kt, int b) {
  if ((kt >> 2) >= blk256) {
    tma_load_3d_pair(kmap, lbar, dst, kt * 64, row0, b);
  } else {
    tma_load_3d_pair(mnmap, lbar, dst, row0, kt * 64, b);
    tma_load_3d_pair(mnmap, lbar, dst + 8192, row0 + 64, kt * 64, b);
  }
}

template <class Epi>
__global__ void __launch_bounds__(SC_THREADS, 1)
    chain_pair_kernel(const __grid_constant__ SymMaps maps, const UmmaWork work, const Epi epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SC_STAGES * SC_STAGE_BYTES);
  uint64_t* empty = full + SC_STAGES;
  uint64_t* tfull = empty + SC_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.hiK);
    tma_prefetch_desc(&maps.loK);
    tma_prefetch_desc(&maps.hiMN);
    tma_prefetch_desc(&maps.loMN);
    for (int s = 0; s < SC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * SC_EPI_WARPS);
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
      for (int idx = cluster; idx < work.num_work; idx += nclusters) {
        int b, split, tm, tn, kt0, kt1;
        umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
        const int arow = tm * 256 + static_cast<int>(rank) * 128;
        const int brow = tn * 256 + static_cast<int>(rank) * 128;
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * SC_STAGE_BYTES;
          const uint32_t lbar = lbar0 + stage * 8;
          // diagonal pair tiles: each CTA's B rows are its A rows, one copy serves both operands
          const uint32_t full_bytes = work.no_cross ? SC_STAGE_BYTES : 2 * SC_STAGE_BYTES;
          if (leader) mbar_arrive_expect_tx(&full[stage], tm == tn ? full_bytes / 2 : full_bytes);
          sc_load(&maps.hiK, &maps.hiMN, lbar, st, tm, arow, kt, b);
          if (!work.no_cross) sc_load(&maps.loK, &maps.loMN, lbar, st + SC_TILE, tm, arow, kt, b);
          if (tm != tn) {
            sc_load(&maps.hiK, &maps.hiMN, lbar, st + 2 * SC_TILE, tn, brow, kt, b);
            if (!work.no_cross) sc_load(&maps.loK, &maps.loMN, lbar, st + 3 * SC_TILE, tn, brow, kt, b);
          }
          if (++stage == SC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {  // whole warp walks the loop, one elected lane issues (uniform descriptors)
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int idx = cluster; idx < work.num_work; idx += nclusters) {
        int b, split, tm, tn, kt0, kt1;
        umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const bool a_mn = (kt >> 2) < tm, b_mn = (kt >> 2) < tn;
          const uint32_t idesc = idesc_bf16(256, 256, a_mn ? 1 : 0, b_mn ? 1 : 0);
          const uint32_t st = smem_u32(smem + stage * SC_STAGE_BYTES);
          const uint32_t sb = tm == tn ? st : st + 2 * SC_TILE;  // diagonal pair tile: B = A
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ah = a_mn ? operand_desc<true>(st, ks) : operand_desc<false>(st, ks);
            const uint64_t al = a_mn ? operand_desc<true>(st + SC_TILE, ks) : operand_desc<false>(st + SC_TILE, ks);
            const uint64_t bh = b_mn ? operand_desc<true>(sb, ks) : operand_desc<false>(sb, ks);
            const uint64_t bl = b_mn ? operand_desc<true>(sb + SC_TILE, ks) : operand_desc<false>(sb + SC_TILE, ks);
            umma_bf16_pair_warp(d_tmem, ah, bh, idesc, (kt > kt0 || ks > 0) ? 1u : 0u);
            if (!work.no_cross) {
              umma_bf16_pair_warp(d_tmem, ah, bl, idesc, 1u);
              umma_bf16_pair_warp(d_tmem, al, bh, idesc, 1u);
            }
          }
          umma_commit_pair_warp(&empty[stage], 0x3);
          if (++stage == SC_STAGES) {
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
    __syncwarp();
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = warp & 3;
    float* stg = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256) + ew * 1024;
    constexpr int CPG = 8 / (SC_EPI_WARPS / 4);
    const int c0 = (ew / 4) * CPG;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int idx = cluster; idx < work.num_work; idx += nclusters) {
      int b, split, tm, tn, kt0, kt1;
      umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = tm * 256 + static_cast<int>(rank) * 128 + q * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * 256);
#pragma unroll 1
      for (int c = c0; c < c0 + CPG; ++c) {
        uint32_t r[32];
        tmem_ld32(taddr + c * 32, r);
        tmem_wait_ld();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if constexpr (epi_has_rows4<Epi>::value)
          stage_block32(epi, stg, b, split, row - lane, tn * 256 + c * 32, v);
        else
          epi(b, split, row, tn * 256 + c * 32, v);
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
    tmem_dealloc_pair(tmem_base, 512);
  }
}

// Register-resident epilogue of one squaring step on the CTA's 128 rows of an upper pair tile.
struct EpiChainSym {
  const __nv_bfloat16* chi;
  const __nv_bfloat16* clo;
  __nv_bfloat16* nhi;
  __nv_bfloat16* nlo;
  float* P;
  int64_t ld, bs;
  int h;
  float coef;
  int write_next;
  __device__ __forceinline__ void operator()(int b, int, int row, int col0, const float (&v)[32]) const {
    if (row >= h) return;
    const int64_t o = static_cast<int64_t>(b) * bs + static_cast<int64_t>(row) * ld + col0;
    uint32_t hw[16], lw[16];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 a = *reinterpret_cast<const uint4*>(chi + o + 8 * j);
      const uint4 c = *reinterpret_cast<const uint4*>(clo + o + 8 * j);
      hw[4 * j] = a.x; hw[4 * j + 1] = a.y; hw[4 * j + 2] = a.z; hw[4 * j + 3] = a.w;
      lw[4 * j] = c.x; lw[4 * j + 1] = c.y; lw[4 * j + 2] = c.z; lw[4 * j + 3] = c.w;
    }
    float pv[32];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 t = *reinterpret_cast<const float4*>(P + o + 4 * j);
      pv[4 * j] = t.x; pv[4 * j + 1] = t.y; pv[4 * j + 2] = t.z; pv[4 * j + 3] = t.w;
    }
    uint32_t nh[16], nl[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float c0v = bf16_lo_to_f32(hw[j]) + bf16_lo_to_f32(lw[j]);
      const float c1v = bf16_hi_to_f32(hw[j]) + bf16_hi_to_f32(lw[j]);
      const float n0 = 2.0f * c0v - v[2 * j];
      const float n1 = 2.0f * c1v - v[2 * j + 1];
      pv[2 * j] -= coef * n0;
      pv[2 * j + 1] -= coef * n1;
      const uint32_t hh = pack_bf16x2(n0, n1);
      nh[j] = hh;
      nl[j] = pack_bf16x2(n0 - bf16_lo_to_f32(hh), n1 - bf16_hi_to_f32(hh));
    }
    if (write_next) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        *reinterpret_cast<uint4*>(nhi + o + 8 * j) = make_uint4(nh[4 * j], nh[4 * j + 1], nh[4 * j + 2], nh[4 * j + 3]);
        *reinterpret_cast<uint4*>(nlo + o + 8 * j) = make_uint4(nl[4 * j], nl[4 * j + 1], nl[4 * j + 2], nl[4 * j + 3]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<float4*>(P + o + 4 * j) = make_float4(pv[4 * j], pv[4 * j + 1], pv[4 * j + 2], pv[4 * j + 3]);
  }
};

// ------------------------------------------------------------------------------------------
// bf16 + fp8 variant: 2^24 C_k^2 ~= (2^12 hi)(2^12 hi) (bf16, K=16) + hi8*lo8 + lo8*hi8 (e4m3,
// K=32) with hi8 = e4m3(2^8 hi), lo8 = e4m3(2^16 (C - hi)).  The stored bf16 hi operand is
// pre-scaled by 2^12 (exact), so every product carries the same 2^24 and all three accumulate
// into ONE double-buffered TMEM accumulator; the kernel rescales by 2^-24 before the epilogue.
// The cross terms carry ~2^-9 of C^2, so e4m3's 2^-4 relative rounding costs ~2^-13 per step
// (tools/chain_precision_emulation.py: <= 2.7e-3 on cfg2/3/5-like spectra against 2e-2).
// e4m3 operands in 128-byte TMA rows (the per-SM TMA row rate, not bytes, bounds ingest):
//   K-major blocks: interleaved array, row r holds [hi8 k0..63 | lo8 k0..63] per 64-column block,
//                   one SWIZZLE_128B box {128 B, 128 rows} = both operands of the k-block;
//   MN-major (transposed) blocks: separate hi8 / lo8 planes, boxes {128 B (MN), 64 K-rows}.
struct SymMapsF8 {
  CUtensorMap hiK, hiMN;      // bf16 C_k hi (2^12-scaled), SWIZZLE_128B
  CUtensorMap f8K;            // e4m3 interleaved [hi8 | lo8] per 64-col block, box {128, 128}
  CUtensorMap h8MN, l8MN;     // e4m3 planes, box {128, 64}
};

constexpr int F8_TILE = 128 * 128;                           // 16 KB: both e4m3 operands of a k-block
constexpr int F8_STAGE_BYTES = 2 * (SC_TILE + F8_TILE);     // A: hi, f8; B: hi, f8
constexpr int F8_STAGES = 3;
constexpr int F8_SMEM = F8_STAGES * F8_STAGE_BYTES + 256 + SC_STAGING + 1024;
constexpr float F8_CROSS_SCALE = 5.9604644775390625e-08f;  // 2^-24

__device__ __forceinline__ void f8_load(const SymMapsF8& m, uint32_t lbar, uint8_t* dst, int blk256, int row0, int kt,
                                        int b) {
  if ((kt >> 2) >= blk256) {
    tma_load_3d_pair(&m.f8K, lbar, dst, kt * 128, row0, b);      // [128 rows][hi8 64 B | lo8 64 B]
  } else {
    tma_load_3d_pair(&m.h8MN, lbar, dst, row0, kt * 64, b);      // [64 K-rows][128 MN bytes] hi8
    tma_load_3d_pair(&m.l8MN, lbar, dst + 8192, row0, kt * 64, b);  // ... lo8
  }
}
template <class Epi>
__global__ void __launch_bounds__(SC_THREADS, 1)
    chain_pair_f8_kernel(const __grid_constant__ SymMapsF8 maps, const UmmaWork work, const Epi epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + F8_STAGES * F8_STAGE_BYTES);
  uint64_t* empty = full + F8_STAGES;
  uint64_t* tfull = empty + F8_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // stage layout (per CTA): [A hi 16K][B hi 16K][A f8 16K][B f8 16K]
  constexpr int OFF_BH = SC_TILE, OFF_A8 = 2 * SC_TILE, OFF_B8 = OFF_A8 + F8_TILE;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.hiK);
    tma_prefetch_desc(&maps.hiMN);
    tma_prefetch_desc(&maps.f8K);
    tma_prefetch_desc(&maps.h8MN);
    tma_prefetch_desc(&maps.l8MN);
    for (int s = 0; s < F8_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * SC_EPI_WARPS);
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
      for (int idx = cluster; idx < work.num_work; idx += nclusters) {
        int b, split, tm, tn, kt0, kt1;
        umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
        const int arow = tm * 256 + static_cast<int>(rank) * 128;
        const int brow = tn * 256 + static_cast<int>(rank) * 128;
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * F8_STAGE_BYTES;
          const uint32_t lbar = lbar0 + stage * 8;
          // diagonal pair tiles: each CTA's B rows are its A rows, one copy serves both operands
          const uint32_t full_bytes = work.no_cross ? 4 * SC_TILE : 2 * F8_STAGE_BYTES;
          if (leader) mbar_arrive_expect_tx(&full[stage], tm == tn ? full_bytes / 2 : full_bytes);
          sc_load(&maps.hiK, &maps.hiMN, lbar, st, tm, arow, kt, b);
          if (tm != tn) sc_load(&maps.hiK, &maps.hiMN, lbar, st + OFF_BH, tn, brow, kt, b);
          if (!work.no_cross) {
            f8_load(maps, lbar, st + OFF_A8, tm, arow, kt, b);
            if (tm != tn) f8_load(maps, lbar, st + OFF_B8, tn, brow, kt, b);
          }
          if (++stage == F8_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {  // whole warp walks the loop, one elected lane issues (uniform descriptors)
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int idx = cluster; idx < work.num_work; idx += nclusters) {
        int b, split, tm, tn, kt0, kt1;
        umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const bool a_mn = (kt >> 2) < tm, b_mn = (kt >> 2) < tn;
          const uint32_t id16 = idesc_bf16(256, 256, a_mn ? 1 : 0, b_mn ? 1 : 0);
          const uint32_t id8 = idesc_e4m3(256, 256, a_mn ? 1 : 0, b_mn ? 1 : 0);
          const uint32_t st = smem_u32(smem + stage * F8_STAGE_BYTES);
          const uint32_t off_bh = tm == tn ? 0 : OFF_BH, off_b8 = tm == tn ? OFF_A8 : OFF_B8;  // diagonal: B = A
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ah = a_mn ? operand_desc<true>(st, ks) : operand_desc<false>(st, ks);
            const uint64_t bh = b_mn ? operand_desc<true>(st + off_bh, ks) : operand_desc<false>(st + off_bh, ks);
            umma_bf16_pair_warp(d_tmem, ah, bh, id16, (kt > kt0 || ks > 0) ? 1u : 0u);
          }
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            if (work.no_cross) break;
            umma_f8_pair_warp(d_tmem, f8_desc(st + OFF_A8, a_mn, 0, ks), f8_desc(st + off_b8, b_mn, 1, ks), id8, 1u);
            umma_f8_pair_warp(d_tmem, f8_desc(st + OFF_A8, a_mn, 1, ks), f8_desc(st + off_b8, b_mn, 0, ks), id8, 1u);
          }
          umma_commit_pair_warp(&empty[stage], 0x3);
          if (++stage == F8_STAGES) {
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
    __syncwarp();
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = warp & 3;
    float* stg = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256) + ew * 1024;
    constexpr int CPG = 8 / (SC_EPI_WARPS / 4);
    const int c0 = (ew / 4) * CPG;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int idx = cluster; idx < work.num_work; idx += nclusters) {
      int b, split, tm, tn, kt0, kt1;
      umma_decode(work, idx, b, split, tm, tn, kt0, kt1);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = tm * 256 + static_cast<int>(rank) * 128 + q * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * 256);
#pragma unroll 1
      for (int c = c0; c < c0 + CPG; ++c) {
        uint32_t r0[32];
        tmem_ld32(taddr + c * 32, r0);
        tmem_wait_ld();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r0[j]) * F8_CROSS_SCALE;
        if constexpr (epi_has_rows4<Epi>::value)
          stage_block32(epi, stg, b, split, row - lane, tn * 256 + c * 32, v);
        else
          epi(b, split, row, tn * 256 + c * 32, v);
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
    tmem_dealloc_pair(tmem_base, 512);
  }
}

template <class Epi>
inline cudaError_t launch_chain_pair_f8(const SymMapsF8& maps, const UmmaWork& w, const Epi& epi,
                                        cudaStream_t stream) {
  static PerDeviceFlag configured;
  const int cfg_dev = PerDeviceFlag::current();
  if (!configured.test(cfg_dev)) {
    cudaError_t e =
        cudaFuncSetAttribute(chain_pair_f8_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, F8_SMEM);
    if (e != cudaSuccess) return e;
    configured.set(cfg_dev);
  }
  if (w.num_work <= 0) return cudaSuccess;
  const int pairs = device_sm_count() / 2;
  const int nclusters = w.num_work < pairs ? w.num_work : pairs;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * nclusters));
  cfg.blockDim = dim3(SC_THREADS);
  cfg.dynamicSmemBytes = F8_SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, chain_pair_f8_kernel<Epi>, maps, w, epi);
}

template <class Epi>
inline cudaError_t launch_chain_pair(const SymMaps& maps, const UmmaWork& w, const Epi& epi, cudaStream_t stream) {
  static PerDeviceFlag configured;
  const int cfg_dev = PerDeviceFlag::current();
  if (!configured.test(cfg_dev)) {
    cudaError_t e = cudaFuncSetAttribute(chain_pair_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, SC_SMEM);
    if (e != cudaSuccess) return e;
    configured.set(cfg_dev);
  }
  if (w.num_work <= 0) return cudaSuccess;
  const int pairs = device_sm_count() / 2;
  const int nclusters = w.num_work < pairs ? w.num_work : pairs;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * nclusters));
  cfg.blockDim = dim3(SC_THREADS);
  cfg.dynamicSmemBytes = SC_SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, chain_pair_kernel<Epi>, maps, w, epi);
}

}  // namespace unso
