// Fused persistent "scale + squaring chain" kernel (BF16 precision), one CTA per
// 128x128 upper tile of the h x h state, all tiles co-resident (cooperative launch).
//
// Replaces, for the reference's ortho.py:156-167 + 197-204:
//   split-K finalize -> ||G||_F / trace -> s^2, status -> C_1 = G/s^2, P = alpha I - a_1 C_1
//   -> N-1 squarings C_{k+1} = 2 C_k - C_k^2 with P -= c_{k+1} C_{k+1} -> P/s split bf16 hi/lo.
// (C-form of B_{k+1} = B_k^2 with B = I - C; P = I + sum a_k B_k + b B_N = alpha I - sum c_k C_k.)
//
// Per CTA (tile (ti, tj), ti <= tj):
//   TMEM  cols [0,128)   accumulator of C_k^2 for the tile (bf16x3: hi*hi + hi*lo + lo*hi)
//         cols [128,256) P tile (fp32), resident for the whole chain
//         cols [256,384) C_k tile (fp32), resident for the whole chain
//   global: only the CTA's own upper tile of C_{k+1} (bf16 hi/lo, ping-pong buffers) is
//   written per step.  Operand row-blocks are assembled from upper tiles: block (i, kb)
//   with kb < i is read through an MN-major (transposed) TMA map of tile (kb, i), and the
//   tcgen05 instruction descriptor's A/B major bits are switched per k-block.
//   A grid barrier (gpu-scope release/acquire counter) separates the steps.
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
  unsigned long long* gbar;  // [CHAIN_ROUNDS] per-round barrier words, zeroed before launch
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
  __threadfence();
  red_release_gpu_add_u64(gbar + round, (1ull << 48) + static_cast<uint64_t>(c * CHAIN_FIX));
}
__device__ __forceinline__ uint64_t grid_wait(const unsigned long long* gbar, int round) {
  const long long t0 = clock64();
  const uint64_t T = gridDim.x;
  uint64_t v;
  while (((v = ld_acquire_gpu_u64(gbar + round)) >> 48) < T) {
    __nanosleep(64);
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

// Sum of the launch-wide per-tile (x, y) partials of matrix `lb` by the 128 epilogue threads after the
// grid barrier: strided loads, fixed shuffle tree per warp, warps summed in order -- the same bits
// on every CTA of the matrix.  Result in red[0][0] / red[1][0] after the trailing barrier.
__device__ __forceinline__ void sum_tile_partials(const double* buf, int first, int n, int tid, double (*red)[4]) {
  double a = 0.0, c = 0.0;
  for (int q = tid; q < n; q += 128) {
    a += __ldcg(&buf[(first + q) * 2 + 0]);
    c += __ldcg(&buf[(first + q) * 2 + 1]);
  }
  a = warp_sum(a);
  c = warp_sum(c);
  named_bar_sync(1, 128);  // red[] free (its previous contents were consumed before the grid barrier)
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = a;
    red[1][tid >> 5] = c;
  }
  named_bar_sync(1, 128);
}

constexpr int CH_STAGES = 3;
constexpr int CH_TILE = 128 * 64 * 2;          // 16 KB operand tile
constexpr int CH_STAGE_BYTES = 4 * CH_TILE;    // A hi, A lo, B hi, B lo
constexpr int CH_SMEM = CH_STAGES * CH_STAGE_BYTES + 256 + 1024;
constexpr uint32_t CH_ACC = 0, CH_P = 128, CH_C = 256;

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

__global__ void __launch_bounds__(256, 1) chain_persistent_kernel(const __grid_constant__ ChainMaps maps,
                                                                  const __grid_constant__ ChainParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CH_STAGES * CH_STAGE_BYTES);
  uint64_t* empty = full + CH_STAGES;
  uint64_t* tfull = empty + CH_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  __shared__ double red[2][4];
  __shared__ double s_scale[2];  // inv_s2, inv_s

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lb = blockIdx.x / p.tiles_per_mat;  // matrix within this chunk
  const int b = p.b0 + lb;
  const int t = blockIdx.x % p.tiles_per_mat;
  int ti, tj;
  simt_tile_coords(t, p.nt, p.nt, 1, ti, tj);
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
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- producer
      int stage = 0;
      uint32_t phase = 0;
      for (int k = 1; k < N; ++k) {
        const uint64_t e2 = grid_wait(p.gbar, k);  // C_k published (round k)
        if (chain_truncate_before(p, k, e2)) break;
        CHAIN_TRACE(k, 0);
        fence_proxy_async_global();
        const int buf = (k - 1) & 1;
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          CHAIN_KB(k, 1, kt);
          uint8_t* st = smem + stage * CH_STAGE_BYTES;
          const bool hi_only = k <= p.hi_only;
          mbar_arrive_expect_tx(&full[stage], hi_only ? 2 * CH_TILE : CH_STAGE_BYTES);
          ch_load_block(maps, buf, 0, &full[stage], st, ti, kt, b);
          if (!hi_only) ch_load_block(maps, buf, 1, &full[stage], st + CH_TILE, ti, kt, b);
          ch_load_block(maps, buf, 0, &full[stage], st + 2 * CH_TILE, tj, kt, b);
          if (!hi_only) ch_load_block(maps, buf, 1, &full[stage], st + 3 * CH_TILE, tj, kt, b);
          if (++stage == CH_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp, one
    // elected lane issues: warp-uniform control flow keeps the descriptors in uniform registers)
    int stage = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int k = 1; k < N; ++k) {
      if (k >= 2 && p.trunc_tau > 0.0 && chain_truncate_before(p, k, grid_wait(p.gbar, k))) break;
      mbar_wait(tempty, acc_phase ^ 1);
      tc_fence_after();
      for (int kt = 0; kt < KT; ++kt) {
        mbar_wait(&full[stage], phase);
        CHAIN_KB(k, 0, kt);
        if (kt == 0) CHAIN_TRACE(k, 1);
        tc_fence_after();
        const int kb = kt >> 1;
        const bool a_mn = kb < ti, b_mn = kb < tj;
        const uint32_t idesc = idesc_bf16(128, 128, a_mn ? 1 : 0, b_mn ? 1 : 0);
        const uint32_t st = smem_u32(smem + stage * CH_STAGE_BYTES);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t ah = a_mn ? operand_desc<true>(st, ks) : operand_desc<false>(st, ks);
          const uint64_t al = a_mn ? operand_desc<true>(st + CH_TILE, ks) : operand_desc<false>(st + CH_TILE, ks);
          const uint64_t bh = b_mn ? operand_desc<true>(st + 2 * CH_TILE, ks)
                                   : operand_desc<false>(st + 2 * CH_TILE, ks);
          const uint64_t bl = b_mn ? operand_desc<true>(st + 3 * CH_TILE, ks)
                                   : operand_desc<false>(st + 3 * CH_TILE, ks);
          umma_bf16_warp(tmem + CH_ACC, ah, bh, idesc, (kt > 0 || ks > 0) ? 1u : 0u);
          if (k > p.hi_only) {
            umma_bf16_warp(tmem + CH_ACC, ah, bl, idesc, 1u);
            umma_bf16_warp(tmem + CH_ACC, al, bh, idesc, 1u);
          }
        }
        umma_commit_warp(&empty[stage]);
        if (++stage == CH_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit_warp(tfull);
      CHAIN_TRACE(k, 2);
      acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue warps
    const int ew = warp - 4;
    const int r = ew * 32 + lane;
    const int gr = ti * 128 + r;
    const bool row_ok = gr < p.h;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(ew * 32) << 16);
    const int64_t mbase = static_cast<int64_t>(b) * p.mat;
    const int tid = threadIdx.x - 128;

    // ---- phase A: G tile = sum of split-K partials -> TMEM C region; tile norms
    if (tid == 0) CHAIN_TRACE(0, 0);
    double tr = 0.0, fr = 0.0;
    const double wgt = (ti == tj) ? 1.0 : 2.0;
    // all four 32-column chunks of a split-K slice are loaded before any is summed: 32 independent
    // 16-byte loads in flight per thread (the phase was load-latency-bound chunk by chunk)
    float g4[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int j = 0; j < 32; ++j) g4[c][j] = 0.f;
    if (row_ok) {
      for (int sp = 0; sp < p.splits; ++sp) {
        const float* src = p.part + (static_cast<int64_t>(sp) * p.batch + b) * p.part_mat +
                           static_cast<int64_t>(gr) * p.part_ld + tj * 128;
        float4 v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = __ldcg(reinterpret_cast<const float4*>(src) + q);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          float* gq = &g4[q >> 3][(q & 7) * 4];
          gq[0] += v[q].x;
          gq[1] += v[q].y;
          gq[2] += v[q].z;
          gq[3] += v[q].w;
        }
      }
    }
    for (int c = 0; c < 4; ++c) {
      const int gc0 = tj * 128 + c * 32;
      float g[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) g[j] = g4[c][j];
      uint32_t u[32];
      float frc = 0.f;  // fp32 partial over the 32 columns, accumulated in fp64 across chunks
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool ok = row_ok && (gc0 + j) < p.h;
        const float v = ok ? g[j] : 0.f;
        if (ok && gc0 + j == gr) tr += v;
        frc = fmaf(v, v, frc);
        u[j] = __float_as_uint(v);
      }
      fr += wgt * static_cast<double>(frc);
      tmem_st32(lane_base + CH_C + c * 32, u);
    }
    tmem_wait_st();
    tr = warp_sum(tr);
    fr = warp_sum(fr);
    if (lane == 0) {
      red[0][ew] = tr;
      red[1][ew] = fr;
    }
    named_bar_sync(1, 128);
    if (tid == 0) {
      p.normbuf[blockIdx.x * 2 + 0] = red[0][0] + red[0][1] + red[0][2] + red[0][3];
      p.normbuf[blockIdx.x * 2 + 1] = red[1][0] + red[1][1] + red[1][2] + red[1][3];
      CHAIN_TRACE(0, 1);
      grid_arrive(p.gbar, 0);
      grid_wait(p.gbar, 0);
      CHAIN_TRACE(0, 2);
    }
    named_bar_sync(1, 128);  // every epilogue thread is past the grid barrier
    sum_tile_partials(p.normbuf, lb * p.tiles_per_mat, p.tiles_per_mat, tid, red);
    if (tid == 0) {
      const double s0 = red[0][0] + red[0][1] + red[0][2] + red[0][3];
      const double s1 = red[1][0] + red[1][1] + red[1][2] + red[1][3];
      CHAIN_TRACE(0, 4);
      double s2 = p.scal_mode == SM_PLAIN ? s0 : sqrt(s1);
      if (p.scal_mode == SM_NONE) s2 = 1.0;
      const double inv_s = 1.0 / sqrt(s2);
      const bool bad = p.scal_mode != SM_NONE &&
                       (!(s0 > 0.0) || !isfinite(s0) || !(s2 > 0.0) || !isfinite(s2) || !isfinite(inv_s));
      s_scale[0] = 1.0 / s2;
      s_scale[1] = inv_s;
      if (t == 0) {
        double* o = p.scal + static_cast<int64_t>(b) * SCAL_STRIDE;
        o[S_TRACE] = s0;
        o[S_FRO2] = s1;
        o[S_S2] = s2;
        o[S_INV_S] = inv_s;
        if (p.status) p.status[b] = bad ? 2 : 0;
      }
    }
    named_bar_sync(1, 128);
    const float inv_s2 = static_cast<float>(s_scale[0]);
    const float alpha_f = static_cast<float>(p.alpha);

    // ---- C_1 = G / s^2 (TMEM + global buffer 0), P = alpha I - coef_1 C_1 (TMEM)
    for (int c = 0; c < 4; ++c) {
      const int gc0 = tj * 128 + c * 32;
      uint32_t u[32], pu[32];
      tmem_ld32(lane_base + CH_C + c * 32, u);
      tmem_wait_ld();
      __align__(16) __nv_bfloat16 hi[32];
      __align__(16) __nv_bfloat16 lo[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float cv = __uint_as_float(u[j]) * inv_s2;  // fp32 arithmetic: the state is fp32 anyway
        u[j] = __float_as_uint(cv);
        const float pv = fmaf(-p.coef[0], cv, (gr == gc0 + j && row_ok) ? alpha_f : 0.f);
        pu[j] = __float_as_uint(pv);
        split_bf16(cv, hi[j], lo[j]);
      }
      tmem_st32(lane_base + CH_C + c * 32, u);
      tmem_st32(lane_base + CH_P + c * 32, pu);
      if (row_ok && N > 1) {
        const int64_t o = mbase + static_cast<int64_t>(gr) * p.ld + gc0;
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          *reinterpret_cast<uint4*>(p.chi[0] + o + j) = *reinterpret_cast<const uint4*>(hi + j);
          *reinterpret_cast<uint4*>(p.clo[0] + o + j) = *reinterpret_cast<const uint4*>(lo + j);
        }
      }
    }
    tmem_wait_st();
    fence_proxy_async_global();
    named_bar_sync(1, 128);
    if (tid == 0) {
      CHAIN_TRACE(0, 3);
      grid_arrive(p.gbar, 1);  // C_1 published
    }

    // ---- phase B: squaring steps
    __shared__ int s_stop;
    uint32_t acc_phase = 0;
    int steps = 0;
    unsigned last_round = 1;  // rounds published so far: 0 (norms), 1 (C_1), then k+1 per step k
    for (int k = 1; k < N; ++k) {
      if (k >= 2 && p.trunc_tau > 0.0) {
        if (tid == 0) s_stop = chain_truncate_before(p, k, grid_wait(p.gbar, k)) ? 1 : 0;
        named_bar_sync(1, 128);
        if (s_stop) {  // C_j = I for j > k: P -= tail[k] I on the diagonal; P stays in TMEM
          const float tl = p.tail[k];
          for (int c = 0; c < 4; ++c) {
            const int gc0 = tj * 128 + c * 32;
            uint32_t up[32];
            tmem_ld32(lane_base + CH_P + c * 32, up);  // warp-collective: every lane
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (row_ok && gc0 + j == gr) up[j] = __float_as_uint(__uint_as_float(up[j]) - tl);
            tmem_st32(lane_base + CH_P + c * 32, up);
          }
          tmem_wait_st();
          break;
        }
      }
      const bool last = (k == N - 1);
      const float coef = p.coef[k];  // multiplies C_{k+1}
      ++steps;
      mbar_wait(tfull, acc_phase);
      if (tid == 0) CHAIN_TRACE(k, 3);
      acc_phase ^= 1;
      tc_fence_after();
      const bool want_e2 = p.trunc_tau > 0.0 && !last;
      float e2 = 0.f;  // ||I - C_{k+1}||_F^2 over this thread's part of the tile (weighted below)
      if (!last) {
        // Critical path first: C_{k+1} to TMEM and to its global hi/lo copies, the barrier arrival;
        // the P update (not read by any other tile) follows while the next squaring's MMAs run.
        for (int c = 0; c < 4; ++c) {
          const int gc0 = tj * 128 + c * 32;
          uint32_t ua[32], uc[32];
          tmem_ld32(lane_base + CH_ACC + c * 32, ua);
          tmem_ld32(lane_base + CH_C + c * 32, uc);
          tmem_wait_ld();
          __align__(16) __nv_bfloat16 hi[32];
          __align__(16) __nv_bfloat16 lo[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const bool ok = row_ok && gc0 + j < p.h;
            const float cn = ok ? 2.0f * __uint_as_float(uc[j]) - __uint_as_float(ua[j]) : 0.f;
            uc[j] = __float_as_uint(cn);
            split_bf16(cn, hi[j], lo[j]);
            if (want_e2) {
              const float dv = ok ? cn - (gc0 + j == gr ? 1.f : 0.f) : 0.f;
              e2 = fmaf(dv, dv, e2);
            }
          }
          tmem_st32(lane_base + CH_C + c * 32, uc);
          if (row_ok) {
            const int nb = k & 1;
            const int64_t o = mbase + static_cast<int64_t>(gr) * p.ld + gc0;
#pragma unroll
            for (int j = 0; j < 32; j += 16) {  // 256-bit stores: whole sectors (ld % 256 == 0)
              st_global_v8(p.chi[nb] + o + j, *reinterpret_cast<const uint32_t(*)[8]>(hi + j));
              st_global_v8(p.clo[nb] + o + j, *reinterpret_cast<const uint32_t(*)[8]>(lo + j));
            }
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(tempty);
        if (want_e2) {
          const double e2w = warp_sum(wgt * static_cast<double>(e2));
          if (lane == 0) red[0][ew] = e2w;
        }
        fence_proxy_async_global();
        named_bar_sync(1, 128);
        if (tid == 0) {
          CHAIN_TRACE(k, 4);
          const double part = p.trunc_tau > 0.0 ? red[0][0] + red[0][1] + red[0][2] + red[0][3] : 0.0;
          grid_arrive(p.gbar, k + 1, part);  // C_{k+1} published, with its ||I - C||_F^2 partial
        }
        last_round = static_cast<unsigned>(k + 1);
        // P -= c_{k+1} C_{k+1}, off the critical path (the TMEM C region is not touched by the MMAs)
        for (int c = 0; c < 4; ++c) {
          uint32_t uc[32], up[32];
          tmem_ld32(lane_base + CH_C + c * 32, uc);
          tmem_ld32(lane_base + CH_P + c * 32, up);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) up[j] = __float_as_uint(__uint_as_float(up[j]) - coef * __uint_as_float(uc[j]));
          tmem_st32(lane_base + CH_P + c * 32, up);
        }
        tmem_wait_st();
        continue;
      }
      for (int c = 0; c < 4; ++c) {
        const int gc0 = tj * 128 + c * 32;
        uint32_t ua[32], uc[32], up[32];
        tmem_ld32(lane_base + CH_ACC + c * 32, ua);
        tmem_ld32(lane_base + CH_C + c * 32, uc);
        tmem_ld32(lane_base + CH_P + c * 32, up);
        tmem_wait_ld();
        __align__(16) __nv_bfloat16 hi[32];
        __align__(16) __nv_bfloat16 lo[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const bool ok = row_ok && gc0 + j < p.h;
          const float cn = ok ? 2.0f * __uint_as_float(uc[j]) - __uint_as_float(ua[j]) : 0.f;
          const float pv = __uint_as_float(up[j]) - coef * cn;
          uc[j] = __float_as_uint(cn);
          up[j] = __float_as_uint(pv);
          split_bf16(cn, hi[j], lo[j]);
          if (want_e2) {
            const float dv = ok ? cn - (gc0 + j == gr ? 1.f : 0.f) : 0.f;
            e2 = fmaf(dv, dv, e2);
          }
        }
        if (!last) {
          tmem_st32(lane_base + CH_C + c * 32, uc);
          tmem_st32(lane_base + CH_P + c * 32, up);
          if (row_ok) {
            const int nb = k & 1;
            const int64_t o = mbase + static_cast<int64_t>(gr) * p.ld + gc0;
#pragma unroll
            for (int j = 0; j < 32; j += 16) {  // 256-bit stores: whole sectors (ld % 256 == 0)
              st_global_v8(p.chi[nb] + o + j, *reinterpret_cast<const uint32_t(*)[8]>(hi + j));
              st_global_v8(p.clo[nb] + o + j, *reinterpret_cast<const uint32_t(*)[8]>(lo + j));
            }
          }
        } else {
          tmem_st32(lane_base + CH_P + c * 32, up);  // final P stays in TMEM for the shifted split
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(tempty);
      if (!last) {
        if (want_e2) {
          const double e2w = warp_sum(wgt * static_cast<double>(e2));
          if (lane == 0) red[0][ew] = e2w;
        }
        fence_proxy_async_global();
        named_bar_sync(1, 128);
        if (tid == 0) {
          CHAIN_TRACE(k, 4);
          const double part = p.trunc_tau > 0.0 ? red[0][0] + red[0][1] + red[0][2] + red[0][3] : 0.0;
          grid_arrive(p.gbar, k + 1, part);  // C_{k+1} published, with its ||I - C||_F^2 partial
        }
        last_round = static_cast<unsigned>(k + 1);
      }
    }
    // ---- final P: statistics -> identity shift d and the adaptive apply decision, then
    //      R/s = (P - d I)/s split into bf16 hi/lo, written symmetric for the apply.
    {
      if (tid == 0) CHAIN_TRACE(CHAIN_MAX_ORDER - 1, 0);
      double trp = 0.0, sp2 = 0.0;
      for (int c = 0; c < 4; ++c) {
        const int gc0 = tj * 128 + c * 32;
        uint32_t up[32];
        tmem_ld32(lane_base + CH_P + c * 32, up);
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
      if (lane == 0) {
        red[0][ew] = trp;
        red[1][ew] = sp2;
      }
      named_bar_sync(1, 128);
      if (tid == 0) {
        p.pstat[blockIdx.x * 2 + 0] = red[0][0] + red[0][1] + red[0][2] + red[0][3];
        p.pstat[blockIdx.x * 2 + 1] = red[1][0] + red[1][1] + red[1][2] + red[1][3];
        const int round = static_cast<int>(last_round) + 1;
        CHAIN_TRACE(CHAIN_MAX_ORDER - 1, 1);
        grid_arrive(p.gbar, round);
        grid_wait(p.gbar, round);
        CHAIN_TRACE(CHAIN_MAX_ORDER - 1, 2);
      }
      named_bar_sync(1, 128);
      sum_tile_partials(p.pstat, lb * p.tiles_per_mat, p.tiles_per_mat, tid, red);
      if (tid == 0) {
        const double tp = red[0][0] + red[0][1] + red[0][2] + red[0][3];
        const double s2p = red[1][0] + red[1][1] + red[1][2] + red[1][3];
        const double d = tp / p.h;
        const double r2 = fmax(s2p - tp * tp / p.h, 0.0);
        // ||X (R_hat - R)||_F <= ||X||_2 2^-9 ||R||_F with ||X||_2 <= 1 (gram/plain scaling), and
        // ||Y||_F >= min_sigma f(sigma)/sigma * ||X||_F = sqrt(tr C_1) (min f(s)/s = f(1) = 1).
        const double trc = fmax(s_scale[0] * __ldcg(&p.scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_TRACE]), 0.0);
        const double bound = ldexp(sqrt(r2), -9) / fmax(sqrt(trc), 1e-300);
        const bool single = p.adaptive && bound <= p.tau;
        s_scale[0] = d;
        if (t == 0) {
          double* o = p.scal + static_cast<int64_t>(b) * SCAL_STRIDE;
          o[S_SHIFT] = static_cast<double>(static_cast<float>(d)) * s_scale[1];  // the shift R was formed with
          o[S_MODE] = single ? 1.0 : 0.0;
          o[S_BOUND] = bound;
          o[S_STEPS] = steps;
        }
      }
      named_bar_sync(1, 128);
      const double d = s_scale[0];
      const float d_f = static_cast<float>(d), inv_s_f = static_cast<float>(s_scale[1]);
      if ((p.h & 31) == 0) {
        // Whole 32 x 32 blocks: every lane stores its row segment with 16-byte vector stores, and
        // the mirror block goes through a per-warp shared-memory transpose (the pipeline stages
        // are idle now), so every global store is a run of whole sectors.
        uint32_t* tb = reinterpret_cast<uint32_t*>(smem) + ew * 32 * 33;
        const int gr0 = ti * 128 + ew * 32;
        for (int c = 0; c < 4; ++c) {
          const int gc0 = tj * 128 + c * 32;
          uint32_t up[32];
          tmem_ld32(lane_base + CH_P + c * 32, up);  // warp-collective: every lane
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
          for (int j = 0; j < 32; j += 8) {
            uint4 vh, vl;
            vh.x = (hl[j] >> 16) | (hl[j + 1] & 0xFFFF0000u);
            vh.y = (hl[j + 2] >> 16) | (hl[j + 3] & 0xFFFF0000u);
            vh.z = (hl[j + 4] >> 16) | (hl[j + 5] & 0xFFFF0000u);
            vh.w = (hl[j + 6] >> 16) | (hl[j + 7] & 0xFFFF0000u);
            vl.x = (hl[j] & 0xFFFFu) | (hl[j + 1] << 16);
            vl.y = (hl[j + 2] & 0xFFFFu) | (hl[j + 3] << 16);
            vl.z = (hl[j + 4] & 0xFFFFu) | (hl[j + 5] << 16);
            vl.w = (hl[j + 6] & 0xFFFFu) | (hl[j + 7] << 16);
            *reinterpret_cast<uint4*>(p.phi + o + j) = vh;
            *reinterpret_cast<uint4*>(p.plo + o + j) = vl;
          }
          if (!diag) {  // mirror: lane writes row gc0 + lane, columns gr0 .. gr0 + 31
            const int64_t om = mbase + static_cast<int64_t>(gc0 + lane) * p.ld + gr0;
#pragma unroll
            for (int m = 0; m < 32; m += 8) {
              uint32_t w[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) w[e] = tb[(m + e) * 33 + lane];
              uint4 vh, vl;
              vh.x = (w[0] >> 16) | (w[1] & 0xFFFF0000u);
              vh.y = (w[2] >> 16) | (w[3] & 0xFFFF0000u);
              vh.z = (w[4] >> 16) | (w[5] & 0xFFFF0000u);
              vh.w = (w[6] >> 16) | (w[7] & 0xFFFF0000u);
              vl.x = (w[0] & 0xFFFFu) | (w[1] << 16);
              vl.y = (w[2] & 0xFFFFu) | (w[3] << 16);
              vl.z = (w[4] & 0xFFFFu) | (w[5] << 16);
              vl.w = (w[6] & 0xFFFFu) | (w[7] << 16);
              *reinterpret_cast<uint4*>(p.phi + om + m) = vh;
              *reinterpret_cast<uint4*>(p.plo + om + m) = vl;
            }
          }
          __syncwarp();
        }
      } else {
        for (int c = 0; c < 4; ++c) {
          const int gc0 = tj * 128 + c * 32;
          uint32_t up[32];
          tmem_ld32(lane_base + CH_P + c * 32, up);  // warp-collective: every lane, row_ok or not
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
      if (tid == 0) CHAIN_TRACE(CHAIN_MAX_ORDER - 1, 3);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace unso
