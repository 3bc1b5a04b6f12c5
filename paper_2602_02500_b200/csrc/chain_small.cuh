// Reference: preprocess's gram scale (ortho.py:153-157) + unso() (ortho.py:197-204) for h <= 128,
// with the Gram of the tall input (ortho.py:156/198) optionally fused.
// Single-CTA "scale + squaring chain" for h <= 128 (BF16 precision): one CTA per matrix, the
// whole C_k resident on chip for all N-1 squarings.
//
// chain_persistent.cuh spreads a chain over co-resident CTAs and pays, per step, a global
// write of C_{k+1}, a grid barrier and a TMA reload.  With h <= 128 the state is one 128 x 128
// tile, so here the epilogue writes the bf16 hi/lo operands of C_{k+1} straight into the
// shared-memory operand buffers (SWIZZLE_128B K-major, the layout the MMA descriptors read)
// and hands them to the MMA warp through an mbarrier: a step is 24 tcgen05.mma (bf16x3,
// K = 128) plus one TMEM round trip, with no global traffic and no inter-CTA sync.  Batches
// run one matrix per CTA (cfg1 and the small layers of a Muon step).
//
// Same arithmetic as chain_persistent (C-form, fp32 C and P resident in TMEM, bf16x3 products,
// the truncation test of SURVEY 8f-4 and the adaptive-apply decision), same outputs: scal[b],
// status[b], and the shifted symmetric P/s as bf16 hi/lo in the padded workspace layout.
//
// FUSED_GRAM: the CTA also computes G = X^T X itself (tall bf16 X, w rows): warp 0 streams 64-row
// MN-major tiles of X through the (still idle) operand buffers as a 4-stage TMA pipeline, the MMA
// warp accumulates G in TMEM, and phase A reads G from TMEM -- no Gram launch, no split-K partials.
#pragma once
#include "chain_persistent.cuh"

namespace unso {

constexpr uint32_t CH_ACC = 0, CH_C = 256;       // this kernel's TMEM columns: accumulator, C_k (P at CH_P = 128)
constexpr int CS_EPI_WARPS = 8;                  // two per TMEM lane quarter, each on two 32-column chunks
constexpr int CS_THREADS = 128 + 32 * CS_EPI_WARPS;  // warp 1 issues MMAs, warp 2 owns TMEM, warps 4.. epilogue
constexpr int CS_EPI = 32 * CS_EPI_WARPS;
constexpr int CS_CHUNK = 128 * 128;              // bytes of one 128-row x 64-column bf16 K-chunk
constexpr int CS_OPERAND = 2 * CS_CHUNK;         // 128 x 128 bf16, two K-chunks
constexpr int CS_SMEM = 2 * CS_OPERAND + 256 + 1024;

// byte offset of element (row r, column c) of a 128 x 128 bf16 operand in the SW128 K-major layout
__device__ __forceinline__ uint32_t cs_offset(int r, int c) {
  const int chunk = c >> 6, byte = (c & 63) * 2;
  return static_cast<uint32_t>(chunk * CS_CHUNK + r * 128 + ((((byte >> 4) ^ (r & 7))) << 4) + (byte & 15));
}

struct SmallGram {
  CUtensorMap x;  // MN-major bf16 map of the tall X (box {64, 64}), batch in the 3rd dimension
  int w;          // rows of X (the contraction length)
};

template <bool FUSED_GRAM>
__global__ void __launch_bounds__(CS_THREADS, 1) chain_small_kernel(const __grid_constant__ ChainParams p,
                                                                     const __grid_constant__ SmallGram sg) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* c_hi = smem;
  uint8_t* c_lo = smem + CS_OPERAND;
  uint64_t* ready = reinterpret_cast<uint64_t*>(smem + 2 * CS_OPERAND);  // operands of C_k written
  uint64_t* tfull = ready + 1;                                             // C_k^2 (or G) accumulated
  uint64_t* gfull = tfull + 1;                                             // [4] Gram stages loaded
  uint64_t* gempty = gfull + 4;                                            // [4] Gram stages consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gempty + 4);
  __shared__ double red[2][CS_EPI_WARPS];
  __shared__ double s_scale[2];
  __shared__ int s_stop;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = p.b0 + blockIdx.x;
  const int N = p.order;
  if (warp == 0 && lane == 0) {
    mbar_init(ready, CS_EPI);
    mbar_init(tfull, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&gfull[i], 1);
      mbar_init(&gempty[i], 1);
    }
    if (FUSED_GRAM) tma_prefetch_desc(&sg.x);
    fence_mbar_init();
    s_stop = 0;
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 128) CHAIN_TRACE(0, 0);

  const int gk = FUSED_GRAM ? (sg.w + 63) / 64 : 0;  // 64-row k-blocks of X
  if (FUSED_GRAM && warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ Gram producer (4 x 16 KB stages)
      for (int kt = 0; kt < gk; ++kt) {
        const int s = kt & 3;
        mbar_wait(&gempty[s], ((kt >> 2) & 1) ^ 1);
        mbar_arrive_expect_tx(&gfull[s], 16384);
        load_operand_tile<true, 128>(&sg.x, &gfull[s], smem + s * 16384, kt * 64, 0, b);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {
      // ---------------------------------------------------------------- MMA issuer (whole warp, one
      // elected lane issues: descriptors stay in uniform registers)
      const uint32_t idesc = idesc_bf16(128, 128, 0, 0);
      const uint32_t hi = smem_u32(c_hi), lo = smem_u32(c_lo);
      uint32_t phase = 0;
      if (FUSED_GRAM) {  // G = X^T X into the accumulator (A = B = the MN-major X tile)
        const uint32_t gdesc = idesc_bf16(128, 128, 1, 1);
        for (int kt = 0; kt < gk; ++kt) {
          const int s = kt & 3;
          mbar_wait(&gfull[s], (kt >> 2) & 1);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * 16384);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t d = operand_desc<true>(st, ks);
            umma_bf16_warp(tmem + CH_ACC, d, d, gdesc, (kt > 0 || ks > 0) ? 1u : 0u);
          }
          umma_commit_warp(&gempty[s]);
        }
        umma_commit_warp(tfull);
      }
      for (int k = 1; k < N; ++k) {
        mbar_wait(ready, phase);  // C_k's operands in shared memory (and the truncation verdict)
        phase ^= 1;
        if (s_stop) break;
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t off = (ks >> 2) * CS_CHUNK;
          const uint64_t dh = operand_desc<false>(hi + off, ks & 3);
          const uint64_t dl = operand_desc<false>(lo + off, ks & 3);
          umma_bf16_warp(tmem + CH_ACC, dh, dh, idesc, ks > 0 ? 1u : 0u);
          umma_bf16_warp(tmem + CH_ACC, dh, dl, idesc, 1u);
          umma_bf16_warp(tmem + CH_ACC, dl, dh, idesc, 1u);
        }
        umma_commit_warp(tfull);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue warps
    const int ew = warp - 4;
    const int q = warp & 3;                         // TMEM lane quarter
    const int c_begin = (ew >> 2) * 2, c_end = c_begin + 2;
    const int r = q * 32 + lane;  // tile row = TMEM lane
    const bool row_ok = r < p.h;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const int64_t mbase = static_cast<int64_t>(b) * p.mat;
    const int tid = threadIdx.x - 128;
    auto reduce2 = [&](double a0, double a1) {
      a0 = warp_sum(a0);
      a1 = warp_sum(a1);
      if (lane == 0) {
        red[0][ew] = a0;
        red[1][ew] = a1;
      }
      named_bar_sync(1, CS_EPI);
    };
    auto total = [&](int i) {
      double t = 0.0;
      for (int w = 0; w < CS_EPI_WARPS; ++w) t += red[i][w];
      return t;
    };
    // hi/lo of a 32-column chunk of row r into the operand buffers
    auto put_chunk = [&](int c0, const float (&v)[32]) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x0 = v[j + 2 * e], x1 = v[j + 2 * e + 1];
          const uint32_t hh = pack_bf16x2(x0, x1);
          hw[e] = hh;
          lw[e] = pack_bf16x2(x0 - bf16_lo_to_f32(hh), x1 - bf16_hi_to_f32(hh));
        }
        const uint32_t o = cs_offset(r, c0 + j);  // 8 columns = one 16-byte chunk
        *reinterpret_cast<uint4*>(c_hi + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(c_lo + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    };

    // ---- phase A: G = sum of split-K partials (or the dense reduced Gram) -> TMEM C; norms.
    // The sum is taken with lanes along the columns (whole lines per load) into a 64 KB fp32 tile
    // over the idle operand buffers, 16-byte chunks XOR-swizzled by row so the row-per-lane reads
    // below are conflict-free.
    float* gs = reinterpret_cast<float*>(c_hi);
    uint32_t acc_phase = 0;
    if (FUSED_GRAM) {
      mbar_wait(tfull, 0);
      acc_phase = 1;
      tc_fence_after();
    } else {
      constexpr int PER = 128 * 32 / CS_EPI;  // float4 positions per thread
      float4 acc[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      const int64_t sstride = static_cast<int64_t>(p.batch) * p.part_mat;
      const float* base = p.part + static_cast<int64_t>(b) * p.part_mat;
      for (int sp = 0; sp < p.splits; ++sp) {  // PER independent loads in flight per split
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          const int i = tid + q * CS_EPI, rr = i >> 5, c4 = i & 31;
          if (rr < p.h && c4 * 4 < p.h) {  // a dense G (h % 4 == 0) ends at column h
            const float4 v = *reinterpret_cast<const float4*>(base + sp * sstride + static_cast<int64_t>(rr) * p.part_ld +
                                                              c4 * 4);
            acc[q].x += v.x;
            acc[q].y += v.y;
            acc[q].z += v.z;
            acc[q].w += v.w;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int i = tid + q * CS_EPI, rr = i >> 5, c4 = i & 31;
        *reinterpret_cast<float4*>(gs + rr * 128 + ((c4 ^ (rr & 7)) << 2)) = acc[q];
      }
    }
    named_bar_sync(1, CS_EPI);
    double tr = 0.0, fr = 0.0;
    for (int c = c_begin; c < c_end; ++c) {
      float g[32];
      if (FUSED_GRAM) {
        uint32_t u[32];
        tmem_ld32(lane_base + CH_ACC + c * 32, u);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) g[j] = __uint_as_float(u[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 v = *reinterpret_cast<const float4*>(gs + r * 128 + (((c * 8 + j / 4) ^ (r & 7)) << 2));
          g[j] = v.x;
          g[j + 1] = v.y;
          g[j + 2] = v.z;
          g[j + 3] = v.w;
        }
      }
      uint32_t u[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool ok = row_ok && c * 32 + j < p.h;
        const float v = ok ? g[j] : 0.f;
        if (ok && c * 32 + j == r) tr += v;
        fr += static_cast<double>(v) * v;
        u[j] = __float_as_uint(v);
      }
      tmem_st32(lane_base + CH_C + c * 32, u);
    }
    tmem_wait_st();
    reduce2(tr, fr);
    if (tid == 0) {
      const double s0 = total(0), s1 = total(1);
      double s2 = p.scal_mode == SM_PLAIN ? s0 : sqrt(s1);
      if (p.scal_mode == SM_NONE) s2 = 1.0;
      const double inv_s = 1.0 / sqrt(s2);
      const bool bad = p.scal_mode != SM_NONE &&
                       (!(s0 > 0.0) || !isfinite(s0) || !(s2 > 0.0) || !isfinite(s2) || !isfinite(inv_s));
      s_scale[0] = 1.0 / s2;
      s_scale[1] = inv_s;
      double* o = p.scal + static_cast<int64_t>(b) * SCAL_STRIDE;
      o[S_TRACE] = s0;
      o[S_FRO2] = s1;
      o[S_S2] = s2;
      o[S_INV_S] = inv_s;
      if (p.status) p.status[b] = bad ? 2 : 0;
    }
    named_bar_sync(1, CS_EPI);

    // ---- C_1 = G / s^2 (TMEM + operands), P = alpha I - c_1 C_1 (TMEM)
    for (int c = c_begin; c < c_end; ++c) {
      uint32_t u[32], pu[32];
      tmem_ld32(lane_base + CH_C + c * 32, u);
      tmem_wait_ld();
      float cv[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        cv[j] = static_cast<float>(static_cast<double>(__uint_as_float(u[j])) * s_scale[0]);
        u[j] = __float_as_uint(cv[j]);
        pu[j] = __float_as_uint(static_cast<float>(((r == c * 32 + j && row_ok) ? p.alpha : 0.0) -
                                                   static_cast<double>(p.coef[0]) * cv[j]));
      }
      tmem_st32(lane_base + CH_C + c * 32, u);
      tmem_st32(lane_base + CH_P + c * 32, pu);
      put_chunk(c * 32, cv);
    }
    tmem_wait_st();
    fence_proxy_async_shared();
    tc_fence_before();
    mbar_arrive(ready);
    if (tid == 0) CHAIN_TRACE(0, 1);

    // ---- squarings
    int steps = 0;
    for (int k = 1; k < N; ++k) {
      const bool last = k == N - 1;
      const float coef = p.coef[k];
      mbar_wait(tfull, acc_phase);
      if (tid == 0) CHAIN_TRACE(k, 3);
      acc_phase ^= 1;
      tc_fence_after();
      ++steps;
      float e2 = 0.f;
      for (int c = c_begin; c < c_end; ++c) {
        uint32_t ua[32], uc[32], up[32];
        tmem_ld32(lane_base + CH_ACC + c * 32, ua);
        tmem_ld32(lane_base + CH_C + c * 32, uc);
        tmem_ld32(lane_base + CH_P + c * 32, up);
        tmem_wait_ld();
        float cn[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const bool ok = row_ok && c * 32 + j < p.h;
          cn[j] = ok ? 2.0f * __uint_as_float(uc[j]) - __uint_as_float(ua[j]) : 0.f;
          up[j] = __float_as_uint(__uint_as_float(up[j]) - coef * cn[j]);
          uc[j] = __float_as_uint(cn[j]);
          const float dv = ok ? cn[j] - (c * 32 + j == r ? 1.f : 0.f) : 0.f;
          e2 = fmaf(dv, dv, e2);
        }
        tmem_st32(lane_base + CH_P + c * 32, up);
        if (!last) {
          tmem_st32(lane_base + CH_C + c * 32, uc);
          put_chunk(c * 32, cn);
        }
      }
      tmem_wait_st();
      if (last) break;
      // truncation before step k+1, from ||I - C_{k+1}||_F^2 (block-reduced, every thread agrees)
      reduce2(static_cast<double>(e2), 0.0);
      const double e2s = total(0);
      const bool stop = p.trunc_tau > 0.0 && k + 1 >= 2 &&
                        chain_tail_bound(p.coef, p.order, k + 1, e2s) <= p.trunc_tau;
      if (tid == 0) s_stop = stop ? 1 : 0;
      fence_proxy_async_shared();
      tc_fence_before();
      named_bar_sync(1, CS_EPI);  // s_stop and every row's operands written; red[] free again
      mbar_arrive(ready);
      if (tid == 0) CHAIN_TRACE(k, 4);
      if (stop) {  // C_j = I for j > k+1: P -= tail[k+1] I
        const float tl = p.tail[k + 1];
        for (int c = c_begin; c < c_end; ++c) {
          uint32_t up[32];
          tmem_ld32(lane_base + CH_P + c * 32, up);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (row_ok && c * 32 + j == r) up[j] = __float_as_uint(__uint_as_float(up[j]) - tl);
          tmem_st32(lane_base + CH_P + c * 32, up);
        }
        tmem_wait_st();
        break;
      }
    }

    // ---- final P: trace / ||P||^2 -> shift d, adaptive decision; (P - d I)/s as bf16 hi/lo
    double trp = 0.0, sp2 = 0.0;
    for (int c = c_begin; c < c_end; ++c) {
      uint32_t up[32];
      tmem_ld32(lane_base + CH_P + c * 32, up);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool ok = row_ok && c * 32 + j < p.h;
        const double v = ok ? static_cast<double>(__uint_as_float(up[j])) : 0.0;
        if (ok && c * 32 + j == r) trp += v;
        sp2 += v * v;
      }
    }
    reduce2(trp, sp2);
    if (tid == 0) {
      const double tp = total(0), s2p = total(1);
      const double d = tp / p.h;
      const double r2 = fmax(s2p - tp * tp / p.h, 0.0);
      double* o = p.scal + static_cast<int64_t>(b) * SCAL_STRIDE;
      const double trc = fmax(s_scale[0] * o[S_TRACE], 0.0);  // tr C_1
      const double bound = ldexp(sqrt(r2), -9) / fmax(sqrt(trc), 1e-300);
      o[S_SHIFT] = d * s_scale[1];
      o[S_MODE] = (p.adaptive && bound <= p.tau) ? 1.0 : 0.0;
      o[S_BOUND] = bound;
      o[S_STEPS] = steps;
      s_scale[0] = d;
    }
    named_bar_sync(1, CS_EPI);
    // (P - d I)/s as bf16 hi/lo: rows into the idle operand buffers (row-major, 16-byte chunks
    // XOR-swizzled by row), then copied out with whole rows per warp instruction
    const double d = s_scale[0];
    const float inv_s = static_cast<float>(s_scale[1]);
    for (int c = c_begin; c < c_end; ++c) {
      uint32_t up[32];
      tmem_ld32(lane_base + CH_P + c * 32, up);  // warp-collective: every lane
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int gc = c * 32 + j + 2 * e;
          const float f0 = (row_ok && gc < p.h)
                               ? static_cast<float>((static_cast<double>(__uint_as_float(up[j + 2 * e])) -
                                                     (gc == r ? d : 0.0)) * s_scale[1])
                               : 0.f;
          const float f1 = (row_ok && gc + 1 < p.h)
                               ? static_cast<float>((static_cast<double>(__uint_as_float(up[j + 2 * e + 1])) -
                                                     (gc + 1 == r ? d : 0.0)) * s_scale[1])
                               : 0.f;
          hw[e] = pack_bf16x2(f0, f1);
          lw[e] = pack_bf16x2(f0 - bf16_lo_to_f32(hw[e]), f1 - bf16_hi_to_f32(hw[e]));
        }
        const int chunk = ((c * 32 + j) >> 3) ^ (r & 7);
        *reinterpret_cast<uint4*>(c_hi + r * 256 + chunk * 16) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(c_lo + r * 256 + chunk * 16) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    }
    (void)inv_s;
    named_bar_sync(1, CS_EPI);
    for (int rr = ew; rr < p.h && rr < 128; rr += CS_EPI_WARPS) {  // lane l: columns 4l .. 4l+3
      const int chunk = (lane >> 1) ^ (rr & 7);
      const int64_t o = mbase + static_cast<int64_t>(rr) * p.ld + 4 * lane;
      *reinterpret_cast<uint2*>(p.phi + o) = *reinterpret_cast<const uint2*>(c_hi + rr * 256 + chunk * 16 + (lane & 1) * 8);
      *reinterpret_cast<uint2*>(p.plo + o) = *reinterpret_cast<const uint2*>(c_lo + rr * 256 + chunk * 16 + (lane & 1) * 8);
    }
  }
  if (threadIdx.x == 128) CHAIN_TRACE(0, 2);
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace unso
