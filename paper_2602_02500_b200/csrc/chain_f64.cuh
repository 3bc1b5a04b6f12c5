// Reference: the squaring loop of unso() (ortho.py:197-204) in fp64 via the C-form restatement,
// with preprocess's Frobenius-gram scale (ortho.py:153-157) folded into phase A.
// Persistent fp64 squaring chain for the FP32 (fp64-grade) mode, h <= 256: every squaring of
// every matrix of a co-resident batch chunk in ONE cooperative launch (replacing N-1 launches of
// the DMMA engine, each of which is latency-bound at these sizes).
//
// One CTA per T x T upper tile (ti <= tj) of C, T = 16 (h <= 128) or 32.  Per step the CTA pulls row
// blocks ti and tj of
// C_k (full symmetric, f64, written by the previous step) into shared memory with one bulk copy
// per row (cp.async.bulk, completion on an mbarrier), the 4 warps each accumulate the WHOLE tile
// over a quarter of K on the fp64 tensor cores ((T/8)^2 independent m8n8k4 accumulators per warp),
// the quarters are summed through shared memory, and every thread updates its T^2/128 contiguous
// elements of C and P (resident in registers for the whole chain) and
// writes C_{k+1} (tile + mirror).  Steps are separated by the per-round 64-bit grid-barrier words
// of chain_persistent.cuh, which also carry the ||I - C_k||_F^2 partials of the truncation test
// (here in 2^-50 fixed point, partials clamped to 2^-15 so that up to CF_MAX_GRID CTAs cannot
// carry into the arrival count; fp32 mode stops only when the dropped terms are below 2^-30
// relative).
//
// Phase A (as chain_persistent.cuh): from the reduced Gram G (full symmetric f64) every CTA reduces
// its tile's trace / weighted ||G||^2 partials, all CTAs sum them in a fixed order after grid round
// 0 (deterministic), derive s^2 (gram / plain / none scaling), write scal[b] and status[b], and form
// C_1 = G/s^2 (written for step 1, round 1) and P = alpha I - c_1 C_1 (registers).
// Output: P (full symmetric) for finalize_p_kernel<0> + the apply; scal[b] incl. S_STEPS.
#pragma once
#include "chain_persistent.cuh"
#include "simt_gemm.cuh"

namespace unso {

constexpr int CF_MAX_H = 256;
constexpr double CF_FIX = 1125899906842624.0;  // 2^50
constexpr double CF_CLAMP = 1.0 / 32768.0;      // 2^-15: 2^35 units per CTA, <= 4096 CTAs stay below bit 48
constexpr int CF_MAX_GRID = 4096;
// tile edge: 16 for h <= 128 (more CTAs, shorter steps), 32 up to CF_MAX_H
__host__ __device__ inline int cf_tile(int h) { return h <= 128 ? 16 : 32; }
// dynamic shared memory: A and B row blocks [T][K16 + 4] doubles, 4 partial tiles [T][T+1], the mbarrier
__host__ __device__ inline int cf_smem_bytes(int h, int T) {
  const int k16 = (h + 15) & ~15;
  return 2 * T * (k16 + 4) * 8 + 4 * T * (T + 1) * 8 + 16;
}

struct ChainF64Params {
  const double* G;     // reduced Gram, full symmetric, [b][h][ld]
  double* C[2];        // C_k ping-pong, full symmetric, [b][h][ld]
  double* P;
  double* normbuf;     // [grid][2] phase-A partials
  int32_t* status;
  int scal_mode;       // SM_GRAM / SM_PLAIN / SM_NONE
  double alpha;        // 1 + sum of the coefficients
  int64_t ld, mat;
  int h, nt, tiles_per_mat, b0, order;
  unsigned long long* gbar;  // [CHAIN_ROUNDS], zeroed before launch
  double* scal;
  double trunc_tau;          // 0 disables truncation
  double coef[CHAIN_MAX_ORDER];
  double tail[CHAIN_MAX_ORDER];
};

__device__ __forceinline__ void cf_arrive(unsigned long long* gbar, int round, double partial) {
  const double c = fmin(fmax(partial, 0.0), CF_CLAMP);
  __threadfence();
  red_release_gpu_add_u64(gbar + round, (1ull << 48) + static_cast<uint64_t>(c * CF_FIX));
}

__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int T>
__global__ void __launch_bounds__(128, 1) chain_f64_kernel(const __grid_constant__ ChainF64Params p) {
  constexpr int FM = T / 8;                 // 8 x 8 DMMA fragments per tile edge
  constexpr int RED = T * (T + 1);          // one warp's partial tile (doubles, padded rows)
  constexpr int EPT = T * T / 128;          // tile elements per thread in the epilogue
  constexpr int TPR = T / EPT;              // threads per tile row
  extern __shared__ __align__(16) uint8_t dsm[];
  const int K16 = (p.h + 15) & ~15;
  const int S = K16 + 4;  // row stride (doubles): fragment loads conflict-free, 16-byte aligned rows
  double* As = reinterpret_cast<double*>(dsm);
  double* Bs = As + T * S;
  double* part = Bs + T * S;  // [4][T][T + 1]
  uint64_t* bar = reinterpret_cast<uint64_t*>(part + 4 * RED);
  __shared__ double red[4], red2[4];
  __shared__ double s_inv_s2;
  __shared__ int s_stop;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int lb = blockIdx.x / p.tiles_per_mat;
  const int b = p.b0 + lb;
  int ti, tj;
  simt_tile_coords(blockIdx.x % p.tiles_per_mat, p.nt, p.nt, 1, ti, tj);
  const int N = p.order;
  const int64_t mb = static_cast<int64_t>(b) * p.mat;
  const double wgt = ti == tj ? 1.0 : 2.0;
  const int arows = min(T, p.h - ti * T), brows = min(T, p.h - tj * T);
  const uint32_t row_bytes = static_cast<uint32_t>(p.h) * 8;

  // zero both row blocks once: columns >= h and rows past h are never written by the copies
  for (int i = threadIdx.x; i < 2 * T * S; i += 128) As[i] = 0.0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  // this thread's EPT contiguous tile elements: row tr, columns tc0 .. tc0+EPT-1
  const int tr = threadIdx.x / TPR, tc0 = (threadIdx.x % TPR) * EPT;
  const int gr = ti * T + tr;
  double cv[EPT], pv[EPT];
  // ---- phase A: norms of G -> s^2 (round 0), C_1 = G / s^2 (round 1), P = alpha I - c_1 C_1
  {
    double tr = 0.0, fr = 0.0;
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      const int gc = tj * T + tc0 + q;
      const bool ok = gr < p.h && gc < p.h;
      cv[q] = ok ? p.G[mb + static_cast<int64_t>(gr) * p.ld + gc] : 0.0;
      if (ok && gr == gc) tr += cv[q];
      fr += wgt * cv[q] * cv[q];
    }
    tr = warp_sum(tr);
    fr = warp_sum(fr);
    if (lane == 0) {
      red[warp] = tr;
      red2[warp] = fr;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      p.normbuf[blockIdx.x * 2 + 0] = red[0] + red[1] + red[2] + red[3];
      p.normbuf[blockIdx.x * 2 + 1] = red2[0] + red2[1] + red2[2] + red2[3];
      cf_arrive(p.gbar, 0, 0.0);
      grid_wait(p.gbar, 0);
      double s0 = 0.0, s1 = 0.0;
      const int first = lb * p.tiles_per_mat;
      for (int t = 0; t < p.tiles_per_mat; ++t) {  // fixed order: every CTA of the matrix agrees
        s0 += __ldcg(&p.normbuf[(first + t) * 2 + 0]);
        s1 += __ldcg(&p.normbuf[(first + t) * 2 + 1]);
      }
      double s2 = p.scal_mode == SM_PLAIN ? s0 : sqrt(s1);
      if (p.scal_mode == SM_NONE) s2 = 1.0;
      const double inv_s = 1.0 / sqrt(s2);
      const bool bad = p.scal_mode != SM_NONE &&
                       (!(s0 > 0.0) || !isfinite(s0) || !(s2 > 0.0) || !isfinite(s2) || !isfinite(inv_s));
      s_inv_s2 = 1.0 / s2;
      if (blockIdx.x % p.tiles_per_mat == 0) {
        double* o = p.scal + static_cast<int64_t>(b) * SCAL_STRIDE;
        o[S_TRACE] = s0;
        o[S_FRO2] = s1;
        o[S_S2] = s2;
        o[S_INV_S] = inv_s;
        o[S_DEV2] = 0.0;
        o[S_SHIFT] = 0.0;  // the fp64 apply uses P itself
        o[S_MODE] = 0.0;
        o[S_BOUND] = -1.0;
        if (p.status) p.status[b] = bad ? 2 : 0;
      }
    }
    __syncthreads();
    const double inv_s2 = s_inv_s2;
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      const int gc = tj * T + tc0 + q;
      const bool ok = gr < p.h && gc < p.h;
      cv[q] *= inv_s2;
      pv[q] = ok ? (gr == gc ? p.alpha : 0.0) - p.coef[0] * cv[q] : 0.0;
      if (ok && N > 1) {
        p.C[0][mb + static_cast<int64_t>(gr) * p.ld + gc] = cv[q];
        p.C[0][mb + static_cast<int64_t>(gc) * p.ld + gr] = cv[q];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) cf_arrive(p.gbar, 1, 0.0);  // C_1 published
  }

  int steps = 0;
  uint32_t phase = 0;
  for (int k = 1; k < N; ++k) {
    const double* cur = p.C[(k - 1) & 1];
    {
      if (threadIdx.x == 0) {
        const uint64_t sum = grid_wait(p.gbar, k);  // C_k published, with its ||I - C_k||_F^2 partials
        s_stop = p.trunc_tau > 0.0 && k >= 2 &&
                 chain_tail_bound(p.coef, p.order, k, static_cast<double>(sum) / CF_FIX) <= p.trunc_tau;
      }
      __syncthreads();
      if (s_stop) {  // C_j = I for j > k
#pragma unroll
        for (int q = 0; q < EPT; ++q)
          if (gr < p.h && gr == tj * T + tc0 + q) pv[q] -= p.tail[k];
        break;
      }
    }
    ++steps;
    if (threadIdx.x == 0) CHAIN_TRACE(k, 0);
    // row blocks ti (A) and tj (B) of C_k -> shared memory, one bulk copy per row
    if (warp == 0) {
      if (lane == 0) mbar_arrive_expect_tx(bar, (arows + brows) * row_bytes);
      __syncwarp();
      for (int r = lane; r < arows + brows; r += 32) {
        const bool isa = r < arows;
        const int row = isa ? r : r - arows;
        const int grow = (isa ? ti : tj) * T + row;
        bulk_copy_g2s((isa ? As : Bs) + row * S, cur + mb + static_cast<int64_t>(grow) * p.ld, row_bytes, bar);
      }
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    if (threadIdx.x == 0) CHAIN_TRACE(k, 1);
    // warp w: the whole T x T tile over k in [w K16/4, (w+1) K16/4)
    double acc[FM][FM][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FM; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int kq = K16 / 4;
    for (int ks = warp * kq; ks < (warp + 1) * kq; ks += 4) {
      const int kk = ks + tig;
      double a[FM], bv[FM];
#pragma unroll
      for (int i = 0; i < FM; ++i) a[i] = As[(i * 8 + gid) * S + kk];
#pragma unroll
      for (int j = 0; j < FM; ++j) bv[j] = Bs[(j * 8 + gid) * S + kk];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FM; ++j) dmma_884(acc[i][j], a[i], bv[j]);
    }
    double* mine = part + warp * RED;
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FM; ++j) {
        mine[(i * 8 + gid) * (T + 1) + j * 8 + 2 * tig] = acc[i][j][0];
        mine[(i * 8 + gid) * (T + 1) + j * 8 + 2 * tig + 1] = acc[i][j][1];
      }
    __syncthreads();  // partials complete; As/Bs free for the next step's copies
    if (threadIdx.x == 0) CHAIN_TRACE(k, 2);
    const bool last = k == N - 1;
    const double coef = p.coef[k];  // multiplies C_{k+1}
    double e2 = 0.0;
    double cn[EPT];
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      const int gc = tj * T + tc0 + q;
      const bool ok = gr < p.h && gc < p.h;
      const int o = tr * (T + 1) + tc0 + q;
      const double s2 = part[o] + part[RED + o] + part[2 * RED + o] + part[3 * RED + o];
      cn[q] = ok ? 2.0 * cv[q] - s2 : 0.0;
      pv[q] -= coef * cn[q];
      cv[q] = cn[q];
      const double dv = ok ? cn[q] - (gr == gc ? 1.0 : 0.0) : 0.0;
      e2 += wgt * dv * dv;
    }
    if (last) break;
    double* nxt = p.C[k & 1];
    if (gr < p.h) {
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int gc = tj * T + tc0 + q;
        if (gc < p.h) {
          nxt[mb + static_cast<int64_t>(gr) * p.ld + gc] = cn[q];
          nxt[mb + static_cast<int64_t>(gc) * p.ld + gr] = cn[q];
        }
      }
    }
    e2 = warp_sum(e2);
    if (lane == 0) red[warp] = e2;
    __syncthreads();  // red complete; every thread is done reading the partial tiles
    if (threadIdx.x == 0) {
      cf_arrive(p.gbar, k + 1, red[0] + red[1] + red[2] + red[3]);
      CHAIN_TRACE(k, 3);
    }
  }
  // final P (tile + mirror) for finalize_p_kernel<0>
  if (gr < p.h) {
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      const int gc = tj * T + tc0 + q;
      if (gc >= p.h) continue;
      p.P[mb + static_cast<int64_t>(gr) * p.ld + gc] = pv[q];
      p.P[mb + static_cast<int64_t>(gc) * p.ld + gr] = pv[q];
    }
  }
  if (threadIdx.x == 0 && blockIdx.x % p.tiles_per_mat == 0) p.scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_STEPS] = steps;
}

}  // namespace unso
