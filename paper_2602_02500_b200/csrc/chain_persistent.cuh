// Fused persistent "scale + squaring chain" kernel (BF16 precision) over the 128x128 upper tiles
// of the h x h state(s), all tiles co-resident (cooperative launch, one or two tiles per CTA).
//
// Replaces, for the reference's ortho.py:156-167 + 197-204:
//   split-K finalize -> ||G||_F / trace -> s^2, status -> C_1 = G/s^2, P = alpha I - a_1 C_1
//   -> N-1 squarings C_{k+1} = 2 C_k - C_k^2 with P -= c_{k+1} C_{k+1} -> P/s split bf16 hi/lo.
// (C-form of B_{k+1} = B_k^2 with B = I - C; P = I + sum a_k B_k + b B_N = alpha I - sum c_k C_k.)
//
// Per CTA: up to two upper tiles (ti, tj), ti <= tj ("slots": tile ids blockIdx.x and blockIdx.x +
// gridDim.x of the launch, so a batch with up to 2 x #SM tiles runs in ONE co-resident launch).  The
// host sizes the grid to whole matrices, so slot s of every CTA belongs to matrix group s, and each
// group has its own barrier rounds: while group 0's tiles drain, publish, synchronise and fetch their
// first operands, the tensor pipe runs group 1's MMAs (and vice versa).  Per slot s:
//   TMEM  cols [256 s, 256 s + 128)        D: holds 2 C_k when step k starts; the MMAs run with the A
//                                          operand negated and accumulate into it (bf16x3: hi*hi + hi*lo +
//                                          lo*hi), so afterwards D = 2 C_k - C_k^2 = C_{k+1} in fp32
//         cols [256 s + 128, 256 s + 256)  P tile (fp32), resident for the whole chain
//   global: only the CTA's own upper tiles of C_{k+1} (bf16 hi/lo, ping-pong buffers) are
//   written per step.  Operand row-blocks are assembled from upper tiles: block (i, kb)
//   with kb < i is read through an MN-major (transposed) TMA map of tile (kb, i), and the
//   tcgen05 instruction descriptor's A/B major bits are switched per k-block.
//   A per-group grid barrier (gpu-scope release/acquire counter) separates the steps.
//
// Data-dependent truncation: each step also reduces ||I - C_{k+1}||_F^2 per tile.
// Before step k every role sums those partials (fixed order, so all CTAs agree) and, once every
// matrix of the launch has sum_{j>k} |c_j| (||I - C_k||_F^2)^(2^(j-k-1)) <= trunc_tau, stops: the
// remaining C_j (j > k) equal I up to ||B_k||_2^(2^(j-k)), so P -= tail[k] I replaces them
// (tail[k] = sum_{j>k} c_j; chain_tail_bound() below bounds the dropped terms).
#pragma once
#include "common.cuh"
#include "ptx_sm100.cuh"
#include "umma_gemm.cuh"

namespace unso {

constexpr int CHAIN_MAX_ORDER = 64;

#ifdef UNSO_EXP_TIMING  // timing experiment only: per-step event timestamps of three CTAs
__device__ unsigned long long g_chain_trace[3][CHAIN_MAX_ORDER][5];
__device__ __forceinline__ void chain_trace(int k, int ev) {
  const int c = blockIdx.x == 0 ? 0 : (blockIdx.x == gridDim.x / 2 ? 1 : (blockIdx.x == gridDim.x - 1 ? 2 : -1));
  if (c < 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_chain_trace[c][k][ev] = t;
}
#define CHAIN_TRACE(k, ev) chain_trace(k, ev)
// per-k-block timestamps of CTA 0, squaring 5: [0] MMA issuer saw the stage full, [1] producer found it empty
__device__ unsigned long long g_chain_kb[2][64];
__device__ __forceinline__ void chain_kb(int k, int which, int kt) {
  if (blockIdx.x != 0 || k != 5 || kt >= 64) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_chain_kb[which][kt] = t;
}
#define CHAIN_KB(k, which, kt) chain_kb(k, which, kt)
#else
#define CHAIN_KB(k, which, kt)
#define CHAIN_TRACE(k, ev)
#endif

struct ChainMaps {
  // [buffer][0 = hi, 1 = lo][0 = K-major box {64,128}, 1 = MN-major box {64,64}]
  CUtensorMap m[2][2][2];
};

struct ChainParams {
  const float* part;   // split-K Gram partials: part[(s * batch + b) * part_mat + r * part_ld + c]
  int64_t part_ld, part_mat;
  int splits;
  int h, nt, tiles_per_mat, batch;  // batch = TOTAL batch (split-K partial layout)
  int b0;                            // first matrix of this launch's chunk
  int nb;                            // matrices in this launch's chunk (persistent chain)
  int64_t ld, mat;     // padded leading dim / per-matrix elements of every h x h buffer
  __nv_bfloat16* chi[2];
  __nv_bfloat16* clo[2];
  __nv_bfloat16* phi;  // out: P/s, full symmetric
  __nv_bfloat16* plo;
  double* normbuf;     // [tiles][2]  phase-A norms
  double* pstat;       // [tiles][2]  final-P statistics (trace, weighted sum of squares)
  int adaptive;        // 1: decide per matrix whether the apply may drop the P_lo term
  double tau;          // bound threshold for that decision
  double* scal;        // [batch][SCAL_STRIDE]
  int32_t* status;     // [batch]
  unsigned long long* gbar;  // [CH_SLOTS][CHAIN_ROUNDS] per-group, per-round barrier words, zeroed before launch
  int order;
  int scal_mode;       // SM_GRAM / SM_PLAIN / SM_NONE
  double alpha;        // 1 + sum a + b
  float coef[CHAIN_MAX_ORDER];  // coef[k-1] multiplies C_k
  double trunc_tau;    // 0 disables truncation
  int hi_only;         // squarings k <= hi_only take the hi*hi product alone (lo tiles not loaded)
  float tail[CHAIN_MAX_ORDER];      // tail[k] = sum_{j > k} coef[j-1]
};

// Grid barrier, one 64-bit word per round r: every CTA adds (1 << 48) + a fixed-point (2^-33, clamped
// to [0, 1]) partial; the wait returns the exact, order-independent sum of the round's partials.
// Rounds: 0 = Gram norms, 1 = C_1 published, k + 1 = C_{k+1} published by step k, then the final P.
constexpr int CHAIN_ROUNDS = CHAIN_MAX_ORDER + 2;
constexpr double CHAIN_FIX = 8589934592.0;  // 2^33
__device__ __forceinline__ void grid_arrive(unsigned long long* gbar, int round, double partial = 0.0) {
  const double c = fmin(fmax(partial, 0.0), 1.0);
  // no __threadfence(): the release is cumulative over the CTA's writes ordered before it by bar.sync
  red_release_gpu_add_u64(gbar + round, (1ull << 48) + static_cast<uint64_t>(c * CHAIN_FIX));
}
__device__ __forceinline__ uint64_t grid_wait(const unsigned long long* gbar, int round, unsigned count = 0) {
  const long long t0 = clock64();
  const uint64_t T = count ? count : gridDim.x;
  uint64_t v;
  while (((v = ld_acquire_gpu_u64(gbar + round)) >> 48) < T) {
    __nanosleep(20);
    if (clock64() - t0 > UNSO_WATCHDOG_CYCLES) __trap();
  }
  return v & ((1ull << 48) - 1);
}
// Bound on the terms dropped by stopping before step k, from x = ||I - C_k||_F^2 = ||B_k||_F^2:
// ||B_j||_2 = ||B_k||_2^(2^(j-k)) <= x^(2^(j-k-1)), so || sum_{j>k} c_j B_j ||_2 <= sum_{j>k} |c_j| x^(2^(j-k-1))
// (coef[j-1] multiplies C_j).  Only the first term matters once x is small: one squaring fewer than
// the uniform bound (sum_{j>k} |c_j|) x on configs[3].
template <typename T>
__device__ __forceinline__ double chain_tail_bound(const T* coef, int order, int k, double x) {
  double s = 0.0, xp = x;
  for (int j = k + 1; j <= order; ++j) {
    s += fabs(static_cast<double>(coef[j - 1])) * xp;
    xp = xp < 1.0 ? xp * xp : xp;  // x >= 1 never passes; keep the sum finite
  }
  return s;
}
// After round k (C_k published, `sum` = that round's partials = sum over the launch's matrices of
// ||I - C_k||_F^2): every role takes the same decision whether the chain stops before step k.
__device__ __forceinline__ bool chain_truncate_before(const ChainParams& p, int k, uint64_t sum) {
  if (p.trunc_tau <= 0.0 || k < 2) return false;
  return chain_tail_bound(p.coef, p.order, k, static_cast<double>(sum) / CHAIN_FIX) <= p.trunc_tau;
}

// Sum of the launch-wide per-tile (x, y) partials of one matrix by all 256 threads of the CTA after the
// grid barrier: strided loads, fixed shuffle tree per warp, warps summed in order -- the same bits
// on every CTA of the matrix.  Result: sum of red[0][0..7] / red[1][0..7] after the trailing barrier.
__device__ __forceinline__ void sum_tile_partials(const double* buf, int first, int n, double (*red)[8]) {
  double a = 0.0, c = 0.0;
  for (int q = threadIdx.x; q < n; q += 256) {
    a += __ldcg(&buf[(first + q) * 2 + 0]);
    c += __ldcg(&buf[(first + q) * 2 + 1]);
  }
  a = warp_sum(a);
  c = warp_sum(c);
  __syncthreads();  // red[] free
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = a;
    red[1][threadIdx.x >> 5] = c;
  }
  __syncthreads();
}
__device__ __forceinline__ double sum8(const double* r) {
  return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

constexpr int CH_STAGES = 3;
constexpr int CH_TILE = 128 * 64 * 2;          // 16 KB operand tile
constexpr int CH_STAGE_BYTES = 4 * CH_TILE;    // A hi, A lo, B hi, B lo
constexpr int CH_SMEM = CH_STAGES * CH_STAGE_BYTES + 256 + 1024;
// TMEM columns of tile slot s: [256 s, 256 s + 128) the state D, [256 s + 128, 256 s + 256) P.
constexpr uint32_t CH_SLOT = 256, CH_D = 0, CH_P = 128;
constexpr int CH_SLOTS = 2;
constexpr int CH_GT_LD = 132;                    // phase A: row pitch (floats) of a staged 128 x 128 Gram tile
constexpr int CH_GT_FLOATS = 128 * CH_GT_LD;      // one staged tile per slot in the (still idle) pipeline stages
static_assert(CH_SLOTS * CH_GT_FLOATS * 4 <= CH_STAGES * CH_STAGE_BYTES, "staged Gram tiles must fit the stages");

__device__ __forceinline__ void ch_load_block(const ChainMaps& maps, int buf, int hl, uint64_t* bar, uint8_t* dst,
                                              int blk, int kt, int b) {
  const int kb = kt >> 1;  // 128-wide block index of this 64-wide k-slice
  if (blk <= kb) {
    tma_load_3d(&maps.m[buf][hl][0], bar, dst, kt * 64, blk * 128, b);      // rows of stored tile (blk, kb)
  } else {
    tma_load_3d(&maps.m[buf][hl][1], bar, dst, blk * 128, kt * 64, b);          // tile (kb, blk) read transposed
    tma_load_3d(&maps.m[buf][hl][1], bar, dst + 8192, blk * 128 + 64, kt * 64, b);
  }
}

// One CTA owns up to CH_SLOTS upper tiles of the launch (tile ids blockIdx.x and blockIdx.x + gridDim.x,
// possibly of different matrices).  The state of slot s lives in TMEM: D_s holds 2 C_k when step k's
// MMAs start; they run with the A operand negated and accumulate into it, D_s -= C_k C_k, so the
// accumulator IS C_{k+1} = 2 C_k - C_k^2 (no separate C copy), and the epilogue writes 2 C_{k+1} back.
// With two slots the epilogue of slot 0 runs under the MMAs of slot 1.
__global__ void __launch_bounds__(256, 1) chain_persistent_kernel(const __grid_constant__ ChainMaps maps,
                                                                  const __grid_constant__ ChainParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CH_STAGES * CH_STAGE_BYTES);
  uint64_t* empty = full + CH_STAGES;
  uint64_t* tfull = empty + CH_STAGES;   // [CH_SLOTS]
  uint64_t* tempty = tfull + CH_SLOTS;   // [CH_SLOTS]
  uint64_t* decbar = tempty + CH_SLOTS;  // [CH_SLOTS] the producer's per-step go / stop decision is posted
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(decbar + CH_SLOTS);
  // Only the producer polls the global barrier words; it posts each step's decision (0 = run step k,
  // 1 = the chain of this slot's group stops before step k) for the MMA and epilogue roles.
  __shared__ int s_dec[CH_SLOTS][2];
  __shared__ double red[2][8];
  __shared__ int s_steps[CH_SLOTS];
  __shared__ unsigned s_last_round[CH_SLOTS];
  __shared__ double s_scale[CH_SLOTS][2];  // per slot: inv_s2 (later the shift d), inv_s

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total_tiles = p.tiles_per_mat * p.nb;
  const int ns = (static_cast<int>(blockIdx.x + gridDim.x) < total_tiles) ? 2 : 1;
  // Slot s of every CTA belongs to matrix group s (the host sizes the grid to whole matrices), and each
  // group has its own barrier words: group 1's MMAs cover group 0's epilogue + barrier + first loads.
  const unsigned cnt0 = gridDim.x, cnt1 = static_cast<unsigned>(max(total_tiles - static_cast<int>(gridDim.x), 1));
  auto cnt = [&](int s) { return s ? cnt1 : cnt0; };
  // Slot coordinates, computed from blockIdx (warp-uniform values: the MMA issuer's descriptors and
  // instruction descriptor then stay in uniform registers) and selected per slot.
  int g_[CH_SLOTS], ti_[CH_SLOTS], tj_[CH_SLOTS];
#pragma unroll
  for (int s = 0; s < CH_SLOTS; ++s) {
    g_[s] = min(static_cast<int>(blockIdx.x + s * gridDim.x), total_tiles - 1);
    simt_tile_coords(g_[s] % p.tiles_per_mat, p.nt, p.nt, 1, ti_[s], tj_[s]);
  }
  const int g0 = g_[0], g1 = g_[1], ti0 = ti_[0], ti1 = ti_[1], tj0 = tj_[0], tj1 = tj_[1];
  auto s_g = [&](int s) { return s ? g1 : g0; };                                   // tile id in the launch
  auto s_lb = [&](int s) { return (s ? g1 : g0) / p.tiles_per_mat; };              // matrix within the chunk
  auto s_b = [&](int s) { return p.b0 + (s ? g1 : g0) / p.tiles_per_mat; };        // matrix in the batch
  auto s_t = [&](int s) { return (s ? g1 : g0) % p.tiles_per_mat; };               // tile within the matrix
  auto s_ti = [&](int s) { return s ? ti1 : ti0; };
  auto s_tj = [&](int s) { return s ? tj1 : tj0; };
  const int N = p.order;
  const int KT = (p.h + 63) / 64;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        for (int q = 0; q < 2; ++q) tma_prefetch_desc(&maps.m[i][j][q]);
    for (int s = 0; s < CH_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < CH_SLOTS; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
      mbar_init(&decbar[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;


  // ================================================================== phase A (all 8 warps)
  // G tile = sum of split-K partials -> shared memory; tile norms; scale; C_1, D = 2 C_1, P -> TMEM.
  // Warp w owns TMEM lanes 32 (w & 3) .. + 31 (row r of the tile per thread); warps 4-7 take the
  // column chunks 0-1 of every tile and warps 0-3 the chunks 2-3 (the producer / MMA roles start after C_1).
  const int ew = warp & 3;
  const int r = ew * 32 + lane;
  const int c0 = warp >= 4 ? 0 : 2;  // first of this warp's two 32-column chunks
  const uint32_t lane_base = tmem + (static_cast<uint32_t>(ew * 32) << 16);
  if (threadIdx.x == 128) CHAIN_TRACE(0, 0);
  // The split-K partials of a tile are read row by row, one 512-byte row per warp request (coalesced;
  // 16 rows x splits independent loads in flight per lane), summed, and staged in shared memory (the
  // pipeline stages are idle until C_1 is published) for the row-per-thread TMEM layout of the C_1 step.
  for (int s = 0; s < ns; ++s) {
    const int ti = s_ti(s), tj = s_tj(s), b = s_b(s);
    double tr = 0.0, fr = 0.0;
    const double wgt = (ti == tj) ? 1.0 : 2.0;
    float* gt = reinterpret_cast<float*>(smem) + s * CH_GT_FLOATS;
    float4 acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int sp = 0; sp < p.splits; ++sp) {
      const float* base = p.part + (static_cast<int64_t>(sp) * p.batch + b) * p.part_mat + tj * 128 + lane * 4;
      float4 v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int gr = ti * 128 + warp * 16 + q;
        // (a dense Gram read in place has part_ld = h, a multiple of 4: no read past the end of a row)
        v[q] = (gr < p.h && tj * 128 + lane * 4 < p.part_ld)
                   ? __ldcg(reinterpret_cast<const float4*>(base + static_cast<int64_t>(gr) * p.part_ld))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        acc[q].x += v[q].x;
        acc[q].y += v[q].y;
        acc[q].z += v[q].z;
        acc[q].w += v[q].w;
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = warp * 16 + q;
      const int gr = ti * 128 + i, gc = tj * 128 + lane * 4;
      const bool row_ok = gr < p.h;
      float e[4] = {acc[q].x, acc[q].y, acc[q].z, acc[q].w};
      float frc = 0.f;  // fp32 partial over this lane's 4 columns, accumulated in fp64 across rows
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool ok = row_ok && (gc + j) < p.h;
        e[j] = ok ? e[j] : 0.f;
        if (ok && gc + j == gr) tr += e[j];
        frc = fmaf(e[j], e[j], frc);
      }
      fr += wgt * static_cast<double>(frc);
      *reinterpret_cast<float4*>(gt + i * CH_GT_LD + lane * 4) = make_float4(e[0], e[1], e[2], e[3]);
    }
    tr = warp_sum(tr);
    fr = warp_sum(fr);
    __syncthreads();  // red[] free (slot 0's sums were consumed)
    if (lane == 0) {
      red[0][warp] = tr;
      red[1][warp] = fr;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      p.normbuf[s_g(s) * 2 + 0] = sum8(red[0]);
      p.normbuf[s_g(s) * 2 + 1] = sum8(red[1]);
    }
  }
  if (threadIdx.x == 0) {
    CHAIN_TRACE(0, 1);
    for (int s = 0; s < ns; ++s) grid_arrive(p.gbar + s * CHAIN_ROUNDS, 0);
    for (int s = 0; s < ns; ++s) grid_wait(p.gbar + s * CHAIN_ROUNDS, 0, cnt(s));
    CHAIN_TRACE(0, 2);
  }
  __syncthreads();  // every thread is past the grid barrier
  for (int s = 0; s < ns; ++s) {
    const int b = s_b(s);
    sum_tile_partials(p.normbuf, s_lb(s) * p.tiles_per_mat, p.tiles_per_mat, red);
    if (threadIdx.x == 0) {
      const double s0 = sum8(red[0]);
      const double s1 = sum8(red[1]);
      if (s == 0) CHAIN_TRACE(0, 4);
      double s2 = p.scal_mode == SM_PLAIN ? s0 : sqrt(s1);
      if (p.scal_mode == SM_NONE) s2 = 1.0;
      const double inv_s = 1.0 / sqrt(s2);
      const bool bad = p.scal_mode != SM_NONE &&
                       (!(s0 > 0.0) || !isfinite(s0) || !(s2 > 0.0) || !isfinite(s2) || !isfinite(inv_s));
      s_scale[s][0] = 1.0 / s2;
      s_scale[s][1] = inv_s;
      if (s_t(s) == 0) {
        double* o = p.scal + static_cast<int64_t>(b) * SCAL_STRIDE;
        o[S_TRACE] = s0;
        o[S_FRO2] = s1;
        o[S_S2] = s2;
        o[S_INV_S] = inv_s;
        if (p.status) p.status[b] = bad ? 2 : 0;
      }
    }
  }
  __syncthreads();
  {
    const float alpha_f = static_cast<float>(p.alpha);
    // ---- C_1 = G / s^2 (global buffer 0), D = 2 C_1, P = alpha I - coef_1 C_1 (TMEM)
    for (int s = 0; s < ns; ++s) {
      const int ti = s_ti(s), tj = s_tj(s);
      const int gr = ti * 128 + r;
      const bool row_ok = gr < p.h;
      const int64_t mbase = static_cast<int64_t>(s_b(s)) * p.mat;
      const float inv_s2 = static_cast<float>(s_scale[s][0]);
      const float* gt = reinterpret_cast<const float*>(smem) + s * CH_GT_FLOATS + r * CH_GT_LD;
      for (int c = c0; c < c0 + 2; ++c) {
        const int gc0 = tj * 128 + c * 32;
        uint32_t u[32], pu[32];
#pragma unroll
        for (int j = 0; j < 32; j += 4)  // row r of the staged tile: pitch 132 floats, conflict-free per quarter warp
          *reinterpret_cast<float4*>(&u[j]) = *reinterpret_cast<const float4*>(gt + c * 32 + j);
        __align__(16) __nv_bfloat16 hi[32];
        __align__(16) __nv_bfloat16 lo[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float cv = __uint_as_float(u[j]) * inv_s2;  // fp32 arithmetic: the state is fp32 anyway
          u[j] = __float_as_uint(2.0f * cv);
          const float pv = fmaf(-p.coef[0], cv, (gr == gc0 + j && row_ok) ? alpha_f : 0.f);
          pu[j] = __float_as_uint(pv);
          split_bf16(cv, hi[j], lo[j]);
        }
        tmem_st32(lane_base + s * CH_SLOT + CH_D + c * 32, u);
        tmem_st32(lane_base + s * CH_SLOT + CH_P + c * 32, pu);
        if (row_ok && N > 1) {
          const int64_t o = mbase + static_cast<int64_t>(gr) * p.ld + gc0;
#pragma unroll
          for (int j = 0; j < 32; j += 16) {  // 256-bit stores: whole sectors (ld % 256 == 0)
            st_global_v8(p.chi[0] + o + j, *reinterpret_cast<const uint32_t(*)[8]>(hi + j));
            st_global_v8(p.clo[0] + o + j, *reinterpret_cast<const uint32_t(*)[8]>(lo + j));
          }
        }
      }
    }
    tmem_wait_st();
    tc_fence_before();
    fence_proxy_async_global();
    fence_proxy_async_shared();  // the staged tiles (generic proxy) are done before TMA refills the stages
    __syncthreads();
    if (warp >= 4)
      for (int s = 0; s < ns; ++s) mbar_arrive(&tempty[s]);  // D_s = 2 C_1 is in place for step 1's MMAs
    if (threadIdx.x == 0) {
      CHAIN_TRACE(0, 3);
      for (int s = 0; s < ns; ++s) grid_arrive(p.gbar + s * CHAIN_ROUNDS, 1);  // group s: C_1 published
    }
  }

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- producer
      int stage = 0;
      uint32_t phase = 0;
      unsigned done = ns < 2 ? 2u : 0u;  // bit s: slot s's chain has stopped (truncated)
      for (int k = 1; k < N && done != 3u; ++k) {
        const int buf = (k - 1) & 1;
        const bool hi_only = k <= p.hi_only;
        for (int s = 0; s < CH_SLOTS; ++s) {
          if ((done >> s) & 1u) continue;
          const uint64_t e2 = grid_wait(p.gbar + s * CHAIN_ROUNDS, k, cnt(s));  // group s: C_k published (round k)
          const bool stop = chain_truncate_before(p, k, e2);
          *reinterpret_cast<volatile int*>(&s_dec[s][k & 1]) = stop ? 1 : 0;
          mbar_arrive(&decbar[s]);  // release: the decision is visible to whoever sees phase k - 1 complete
          if (stop) {
            done |= 1u << s;
            continue;
          }
          if (s == 0) CHAIN_TRACE(k, 0);
          fence_proxy_async_global();
          const int ti = s_ti(s), tj = s_tj(s), b = s_b(s);
          for (int kt = 0; kt < KT; ++kt) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (s == 0) CHAIN_KB(k, 1, kt);
            uint8_t* st = smem + stage * CH_STAGE_BYTES;
            // diagonal tiles: the B row block is the A row block (one copy in shared memory serves both)
            const int nblk = (ti == tj ? 1 : 2) * (hi_only ? 1 : 2);
            mbar_arrive_expect_tx(&full[stage], nblk * CH_TILE);
            ch_load_block(maps, buf, 0, &full[stage], st, ti, kt, b);
            if (!hi_only) ch_load_block(maps, buf, 1, &full[stage], st + CH_TILE, ti, kt, b);
            if (ti != tj) {
              ch_load_block(maps, buf, 0, &full[stage], st + 2 * CH_TILE, tj, kt, b);
              if (!hi_only) ch_load_block(maps, buf, 1, &full[stage], st + 3 * CH_TILE, tj, kt, b);
            }
            if (++stage == CH_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp, one
    // elected lane issues: warp-uniform control flow keeps the descriptors in uniform registers)
    int stage = 0;
    uint32_t phase = 0;
    uint32_t st_phase[CH_SLOTS] = {0, 0};
    unsigned done = ns < 2 ? 2u : 0u;
    for (int k = 1; k < N && done != 3u; ++k) {
#pragma unroll
      for (int s = 0; s < CH_SLOTS; ++s) {
        if ((done >> s) & 1u) continue;
        mbar_wait(&decbar[s], (k - 1) & 1);
        if (*reinterpret_cast<volatile int*>(&s_dec[s][k & 1])) {
          done |= 1u << s;
          continue;
        }
        const int ti = s_ti(s), tj = s_tj(s);
        mbar_wait(&tempty[s], st_phase[s]);  // D_s holds 2 C_k (phase A / the previous step's epilogue)
        st_phase[s] ^= 1;
        tc_fence_after();
        const uint32_t d_tmem = tmem + s * CH_SLOT + CH_D;
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(&full[stage], phase);
          if (s == 0) CHAIN_KB(k, 0, kt);
          if (kt == 0 && s == 0) CHAIN_TRACE(k, 1);
          tc_fence_after();
          const int kb = kt >> 1;
          const bool a_mn = kb < ti, b_mn = kb < tj;
          const uint32_t idesc = idesc_bf16(128, 128, a_mn ? 1 : 0, b_mn ? 1 : 0) | IDESC_NEGATE_A;
          const uint32_t st = smem_u32(smem + stage * CH_STAGE_BYTES);
          const uint32_t sb = ti == tj ? st : st + 2 * CH_TILE;  // diagonal tile: B = A
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ah = a_mn ? operand_desc<true>(st, ks) : operand_desc<false>(st, ks);
            const uint64_t al = a_mn ? operand_desc<true>(st + CH_TILE, ks) : operand_desc<false>(st + CH_TILE, ks);
            const uint64_t bh = b_mn ? operand_desc<true>(sb, ks) : operand_desc<false>(sb, ks);
            const uint64_t bl = b_mn ? operand_desc<true>(sb + CH_TILE, ks) : operand_desc<false>(sb + CH_TILE, ks);
            umma_bf16_warp(d_tmem, ah, bh, idesc, 1u);
            if (k > p.hi_only) {
              umma_bf16_warp(d_tmem, ah, bl, idesc, 1u);
              umma_bf16_warp(d_tmem, al, bh, idesc, 1u);
            }
          }
          umma_commit_warp(&empty[stage]);
          if (++stage == CH_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_warp(&tfull[s]);
        if (s == 0) CHAIN_TRACE(k, 2);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue warps
    const int tid = threadIdx.x - 128;
    // ---- phase B: squaring steps
    uint32_t acc_phase[CH_SLOTS] = {0, 0};
    int steps[CH_SLOTS] = {0, 0};
    unsigned last_round[CH_SLOTS] = {1, 1};  // rounds published so far: 0 (norms), 1 (C_1), then k+1 per step k
    unsigned done = ns < 2 ? 2u : 0u;        // bit s: slot s's chain has stopped (truncated)
    for (int k = 1; k < N && done != 3u; ++k) {
      const bool last = (k == N - 1);
      const float coef = p.coef[k];  // multiplies C_{k+1}
      const bool want_e2 = p.trunc_tau > 0.0 && !last;
#pragma unroll
      for (int s = 0; s < CH_SLOTS; ++s) {
        if ((done >> s) & 1u) continue;
        const int ti = s_ti(s), tj = s_tj(s);
        const int gr = ti * 128 + r;
        const bool row_ok = gr < p.h;
        {
          mbar_wait(&decbar[s], (k - 1) & 1);
          const int stop = *reinterpret_cast<volatile int*>(&s_dec[s][k & 1]);
          if (stop) {  // C_j = I for j > k: P -= tail[k] I on the diagonal; P stays in TMEM
            done |= 1u << s;
            if (ti == tj) {  // warp-uniform: only diagonal tiles hold diagonal entries
              const float tl = p.tail[k];
              for (int c = 0; c < 4; ++c) {
                const int gc0 = tj * 128 + c * 32;
                uint32_t up[32];
                tmem_ld32(lane_base + s * CH_SLOT + CH_P + c * 32, up);  // warp-collective: every lane
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (row_ok && gc0 + j == gr) up[j] = __float_as_uint(__uint_as_float(up[j]) - tl);
                tmem_st32(lane_base + s * CH_SLOT + CH_P + c * 32, up);
              }
              tmem_wait_st();
            }
            continue;
          }
        }
        ++steps[s];
        const int64_t mbase = static_cast<int64_t>(s_b(s)) * p.mat;
        mbar_wait(&tfull[s], acc_phase[s]);
        acc_phase[s] ^= 1;
        if (tid == 0 && s == 0) CHAIN_TRACE(k, 3);
        tc_fence_after();
        float e2 = 0.f;  // ||I - C_{k+1}||_F^2 over this thread's part of the tile (weighted below)
        // D_s = C_{k+1} (the MMAs subtracted C_k C_k from 2 C_k).  Per 32-column chunk: C_{k+1} to its
        // global bf16 hi/lo copies, 2 C_{k+1} back into D_s, P -= c_{k+1} C_{k+1} (one TMEM pass; a
        // separate P pass after the barrier arrival measured slower in both the one- and two-slot forms).
        for (int c = 0; c < 4; ++c) {
          const int gc0 = tj * 128 + c * 32;
          uint32_t ud[32], up[32];
          tmem_ld32(lane_base + s * CH_SLOT + CH_D + c * 32, ud);
          tmem_ld32(lane_base + s * CH_SLOT + CH_P + c * 32, up);
          tmem_wait_ld();
          __align__(16) __nv_bfloat16 hi[32];
          __align__(16) __nv_bfloat16 lo[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const bool ok = row_ok && gc0 + j < p.h;
            const float cn = ok ? __uint_as_float(ud[j]) : 0.f;
            ud[j] = __float_as_uint(2.0f * cn);
            up[j] = __float_as_uint(fmaf(-coef, cn, __uint_as_float(up[j])));
            split_bf16(cn, hi[j], lo[j]);
            if (want_e2) {
              const float dv = ok ? cn - (gc0 + j == gr ? 1.f : 0.f) : 0.f;
              e2 = fmaf(dv, dv, e2);
            }
          }
          if (!last) {
            if (row_ok) {
              const int nb = k & 1;
              const int64_t o = mbase + static_cast<int64_t>(gr) * p.ld + gc0;
#pragma unroll
              for (int j = 0; j < 32; j += 16) {  // 256-bit stores: whole sectors (ld % 256 == 0)
                st_global_v8(p.chi[nb] + o + j, *reinterpret_cast<const uint32_t(*)[8]>(hi + j));
                st_global_v8(p.clo[nb] + o + j, *reinterpret_cast<const uint32_t(*)[8]>(lo + j));
              }
            }
            tmem_st32(lane_base + s * CH_SLOT + CH_D + c * 32, ud);
          }
          tmem_st32(lane_base + s * CH_SLOT + CH_P + c * 32, up);  // the final P stays in TMEM for the shifted split
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&tempty[s]);
        if (!last) {
          if (want_e2) {
            const double e2w = warp_sum(((ti == tj) ? 1.0 : 2.0) * static_cast<double>(e2));
            if (lane == 0) red[0][ew] = e2w;
          }
          fence_proxy_async_global();
          named_bar_sync(1, 128);
          if (tid == 0) {
            if (s == 0) CHAIN_TRACE(k, 4);
            const double part = p.trunc_tau > 0.0 ? red[0][0] + red[0][1] + red[0][2] + red[0][3] : 0.0;
            // group s: C_{k+1} published, with its ||I - C||_F^2 partial
            grid_arrive(p.gbar + s * CHAIN_ROUNDS, k + 1, part);
          }
          last_round[s] = static_cast<unsigned>(k + 1);
          named_bar_sync(1, 128);  // red[] consumed before the next slot / step rewrites it
        }
      }
    }
    if (tid == 0) {
      for (int s = 0; s < CH_SLOTS; ++s) {
        s_steps[s] = steps[s];
        s_last_round[s] = last_round[s];
      }
    }
    tc_fence_before();
  }
  __syncthreads();  // every role is done: P is final in TMEM, the pipeline stages are idle
  tc_fence_after();
  // ================================================================== final P (all 8 warps, column
  // chunks split as in phase A): statistics -> identity shift d and the adaptive apply decision, then
  // R/s = (P - d I)/s split into bf16 hi/lo, written symmetric for the apply.
  {
    if (threadIdx.x == 128) CHAIN_TRACE(CHAIN_MAX_ORDER - 1, 0);
    for (int s = 0; s < ns; ++s) {
      const int ti = s_ti(s), tj = s_tj(s);
      const int gr = ti * 128 + r;
      const bool row_ok = gr < p.h;
      const double wgt = (ti == tj) ? 1.0 : 2.0;
      double trp = 0.0, sp2 = 0.0;
      for (int c = c0; c < c0 + 2; ++c) {
        const int gc0 = tj * 128 + c * 32;
        uint32_t up[32];
        tmem_ld32(lane_base + s * CH_SLOT + CH_P + c * 32, up);
        tmem_wait_ld();
        float s2c = 0.f;  // fp32 partial over 32 columns, fp64 across chunks
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const bool ok = row_ok && gc0 + j < p.h;
          const float v = ok ? __uint_as_float(up[j]) : 0.f;
          if (ok && gc0 + j == gr) trp += v;
          s2c = fmaf(v, v, s2c);
        }
        sp2 += wgt * static_cast<double>(s2c);
      }
      trp = warp_sum(trp);
      sp2 = warp_sum(sp2);
      __syncthreads();  // red[] free
      if (lane == 0) {
        red[0][warp] = trp;
        red[1][warp] = sp2;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        p.pstat[s_g(s) * 2 + 0] = sum8(red[0]);
        p.pstat[s_g(s) * 2 + 1] = sum8(red[1]);
      }
    }
    if (threadIdx.x == 0) {
      CHAIN_TRACE(CHAIN_MAX_ORDER - 1, 1);
      grid_arrive(p.gbar, static_cast<int>(s_last_round[0]) + 1);
      if (ns > 1) grid_arrive(p.gbar + CHAIN_ROUNDS, static_cast<int>(s_last_round[1]) + 1);
      grid_wait(p.gbar, static_cast<int>(s_last_round[0]) + 1, cnt(0));
      if (ns > 1) grid_wait(p.gbar + CHAIN_ROUNDS, static_cast<int>(s_last_round[1]) + 1, cnt(1));
      CHAIN_TRACE(CHAIN_MAX_ORDER - 1, 2);
    }
    __syncthreads();
    for (int s = 0; s < ns; ++s) {
      const int b = s_b(s);
      sum_tile_partials(p.pstat, s_lb(s) * p.tiles_per_mat, p.tiles_per_mat, red);
      if (threadIdx.x == 0) {
        const double tp = sum8(red[0]);
        const double s2p = sum8(red[1]);
        const double d = tp / p.h;
        const double r2 = fmax(s2p - tp * tp / p.h, 0.0);
        // ||X (R_hat - R)||_F <= ||X||_2 2^-9 ||R||_F with ||X||_2 <= 1 (gram/plain scaling), and
        // ||Y||_F >= min_sigma f(sigma)/sigma * ||X||_F = sqrt(tr C_1) (min f(s)/s = f(1) = 1).
        const double trc =
            fmax(s_scale[s][0] * __ldcg(&p.scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_TRACE]), 0.0);
        const double bound = ldexp(sqrt(r2), -9) / fmax(sqrt(trc), 1e-300);
        const bool single = p.adaptive && bound <= p.tau;
        s_scale[s][0] = d;
        if (s_t(s) == 0) {
          double* o = p.scal + static_cast<int64_t>(b) * SCAL_STRIDE;
          o[S_SHIFT] = static_cast<double>(static_cast<float>(d)) * s_scale[s][1];  // the shift R was formed with
          o[S_MODE] = single ? 1.0 : 0.0;
          o[S_BOUND] = bound;
          o[S_STEPS] = s_steps[s];
        }
      }
    }
    __syncthreads();
    for (int s = 0; s < ns; ++s) {
      const int ti = s_ti(s), tj = s_tj(s);
      const int gr = ti * 128 + r;
      const bool row_ok = gr < p.h;
      const int64_t mbase = static_cast<int64_t>(s_b(s)) * p.mat;
      const float d_f = static_cast<float>(s_scale[s][0]), inv_s_f = static_cast<float>(s_scale[s][1]);
      if ((p.h & 31) == 0) {
        // Whole 32 x 32 blocks: every lane stores its row segment with 16-byte vector stores, and
        // the mirror block goes through a per-warp shared-memory transpose (the pipeline stages
        // are idle now), so every global store is a run of whole sectors.
        uint32_t* tb = reinterpret_cast<uint32_t*>(smem) + warp * 32 * 33;
        const int gr0 = ti * 128 + ew * 32;
        for (int c = c0; c < c0 + 2; ++c) {
          const int gc0 = tj * 128 + c * 32;
          uint32_t up[32];
          tmem_ld32(lane_base + s * CH_SLOT + CH_P + c * 32, up);  // warp-collective: every lane
          tmem_wait_ld();
          const bool diag = ti == tj && c == ew;        // block straddling the diagonal
          if (gr0 >= p.h || gc0 >= p.h || (ti == tj && c < ew)) continue;  // warp-uniform
          uint32_t hl[32];                              // (hi << 16) | lo of row gr, columns gc0 + j
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float rv = __uint_as_float(up[j]) - (gc0 + j == gr ? d_f : 0.f);
            __nv_bfloat16 hi, lo;
            split_bf16(rv * inv_s_f, hi, lo);
            hl[j] = (static_cast<uint32_t>(__bfloat16_as_ushort(hi)) << 16) | __bfloat16_as_ushort(lo);
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) tb[lane * 33 + j] = hl[j];
          __syncwarp();
          if (diag) {  // lower half of the block from the transposed upper half: exact symmetry
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < lane) hl[j] = tb[j * 33 + lane];
          }
          const int64_t o = mbase + static_cast<int64_t>(gr) * p.ld + gc0;
#pragma unroll
          for (int j = 0; j < 32; j += 16) {  // 256-bit stores (one sector per lane and array)
            uint32_t vh[8], vl[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              vh[e] = (hl[j + 2 * e] >> 16) | (hl[j + 2 * e + 1] & 0xFFFF0000u);
              vl[e] = (hl[j + 2 * e] & 0xFFFFu) | (hl[j + 2 * e + 1] << 16);
            }
            st_global_v8(p.phi + o + j, vh);
            st_global_v8(p.plo + o + j, vl);
          }
          if (!diag) {  // mirror: lane writes row gc0 + lane, columns gr0 .. gr0 + 31
            const int64_t om = mbase + static_cast<int64_t>(gc0 + lane) * p.ld + gr0;
#pragma unroll
            for (int m = 0; m < 32; m += 16) {
              uint32_t w[16], vh[8], vl[8];
#pragma unroll
              for (int e = 0; e < 16; ++e) w[e] = tb[(m + e) * 33 + lane];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                vh[e] = (w[2 * e] >> 16) | (w[2 * e + 1] & 0xFFFF0000u);
                vl[e] = (w[2 * e] & 0xFFFFu) | (w[2 * e + 1] << 16);
              }
              st_global_v8(p.phi + om + m, vh);
              st_global_v8(p.plo + om + m, vl);
            }
          }
          __syncwarp();
        }
      } else {
        for (int c = c0; c < c0 + 2; ++c) {
          const int gc0 = tj * 128 + c * 32;
          uint32_t up[32];
          tmem_ld32(lane_base + s * CH_SLOT + CH_P + c * 32, up);  // warp-collective: every lane, row_ok or not
          tmem_wait_ld();
          if (row_ok) {
            for (int j = 0; j < 32; ++j) {
              const int gc = gc0 + j;
              if (gc >= p.h || (ti == tj && gc < gr)) continue;
              const float rv = __uint_as_float(up[j]) - (gc == gr ? d_f : 0.f);
              __nv_bfloat16 hi, lo;
              split_bf16(rv * inv_s_f, hi, lo);
              const int64_t o = mbase + static_cast<int64_t>(gr) * p.ld + gc;
              const int64_t om = mbase + static_cast<int64_t>(gc) * p.ld + gr;
              p.phi[o] = hi;
              p.plo[o] = lo;
              p.phi[om] = hi;
              p.plo[om] = lo;
            }
          }
        }
      }
    }
    if (threadIdx.x == 128) CHAIN_TRACE(CHAIN_MAX_ORDER - 1, 3);
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace unso
