// Persistent fp64 squaring chain for the FP32 (fp64-grade) mode, h <= 256: every squaring of
// every matrix of a co-resident batch chunk in ONE cooperative launch (replacing N-1 launches of
// the DMMA engine, each of which is latency-bound at these sizes).
//
// One CTA per 32 x 32 upper tile (ti <= tj) of C; 4 warps of 16 x 16 (2 x 2 DMMA m8n8k4 fragments).
// The tile's C_k and P values stay in registers for the whole chain; per step the CTA streams
// row blocks ti and tj of C_k (full symmetric, f64, written by the previous step) into shared
// memory with cp.async, accumulates C_k^2 on the fp64 tensor cores, and writes C_{k+1} (tile +
// mirror) for the next step.  Steps are separated by the per-round 64-bit grid-barrier words of
// chain_persistent.cuh, which also carry the ||I - C_k||_F^2 partials of the truncation test
// (here in 2^-50 fixed point, partials clamped to 2^-15 so that up to CF_MAX_GRID CTAs cannot carry
// into the arrival count; fp32 mode stops only when the dropped terms are below 2^-30 relative).
//
// Inputs as the multi-launch fp32 path: C[0] = C_1 and P = alpha I - c_1 C_1 (prep_f64_kernel).
// Output: P (full symmetric) for finalize_p_kernel<0> + the apply; scal[b].S_STEPS.
#pragma once
#include "chain_persistent.cuh"
#include "simt_gemm.cuh"

namespace unso {

constexpr int CF_TILE = 32;
constexpr int CF_MAX_H = 256;
constexpr double CF_FIX = 1125899906842624.0;  // 2^50
constexpr double CF_CLAMP = 1.0 / 32768.0;  // 2^-15: 2^35 units per CTA, so <= 4096 CTAs stay below bit 48
constexpr int CF_MAX_GRID = 4096;

struct ChainF64Params {
  double* C[2];        // C_k ping-pong, full symmetric, [b][h][ld]
  double* P;
  int64_t ld, mat;
  int h, nt, tiles_per_mat, b0, order;
  unsigned long long* gbar;  // [CHAIN_ROUNDS], zeroed before launch
  double* scal;
  double trunc_tau;          // 0 disables truncation
  double coef[CHAIN_MAX_ORDER];
  double tail[CHAIN_MAX_ORDER];
  double tail_abs[CHAIN_MAX_ORDER];
};

__device__ __forceinline__ void cf_arrive(unsigned long long* gbar, int round, double partial) {
  const double c = fmin(fmax(partial, 0.0), CF_CLAMP);
  __threadfence();
  red_release_gpu_add_u64(gbar + round, (1ull << 48) + static_cast<uint64_t>(c * CF_FIX));
}

__global__ void __launch_bounds__(128, 1) chain_f64_kernel(const __grid_constant__ ChainF64Params p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int K16 = (p.h + 15) & ~15;
  const int S = K16 + 4;  // row stride (doubles): fragment loads conflict-free, 16-byte aligned rows
  double* As = reinterpret_cast<double*>(dsm);
  double* Bs = As + CF_TILE * S;
  __shared__ double red[4];
  __shared__ int s_stop;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1, gid = lane >> 2, tig = lane & 3;
  const int lb = blockIdx.x / p.tiles_per_mat;
  const int b = p.b0 + lb;
  int ti, tj;
  simt_tile_coords(blockIdx.x % p.tiles_per_mat, p.nt, p.nt, 1, ti, tj);
  const int N = p.order;
  const int64_t mb = static_cast<int64_t>(b) * p.mat;
  const double wgt = ti == tj ? 1.0 : 2.0;

  // this thread's 8 tile positions and their C_1 / P values
  int rr[8], cc[8];
  bool ok[8];
  double cv[8], pv[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = q >> 2, j = (q >> 1) & 1, e = q & 1;
    rr[q] = ti * CF_TILE + wm * 16 + i * 8 + gid;
    cc[q] = tj * CF_TILE + wn * 16 + j * 8 + 2 * tig + e;
    ok[q] = rr[q] < p.h && cc[q] < p.h;
    const int64_t o = mb + static_cast<int64_t>(rr[q]) * p.ld + cc[q];
    cv[q] = ok[q] ? p.C[0][o] : 0.0;
    pv[q] = ok[q] ? p.P[o] : 0.0;
  }

  int steps = 0;
  for (int k = 1; k < N; ++k) {
    const double* cur = p.C[(k - 1) & 1];
    if (k >= 2) {
      if (threadIdx.x == 0) {
        const uint64_t sum = grid_wait(p.gbar, k);  // C_k published, with its ||I - C_k||_F^2 partials
        s_stop = p.trunc_tau > 0.0 && p.tail_abs[k] * (static_cast<double>(sum) / CF_FIX) <= p.trunc_tau;
      }
      __syncthreads();
      if (s_stop) {  // C_j = I for j > k
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (ok[q] && rr[q] == cc[q]) pv[q] -= p.tail[k];
        break;
      }
    }
    ++steps;
    // row blocks ti (A) and tj (B) of C_k -> shared memory (columns >= h zero-filled)
    const int cpr = K16 / 2;  // 16-byte chunks per row
    for (int c = threadIdx.x; c < 2 * CF_TILE * cpr; c += 128) {
      const int which = c / (CF_TILE * cpr), rem = c % (CF_TILE * cpr);
      const int row = rem / cpr, col = (rem % cpr) * 2;
      const int grow = (which ? tj : ti) * CF_TILE + row;
      const int valid = (grow < p.h && col < p.h) ? min(2, p.h - col) : 0;
      const double* src = cur + mb + static_cast<int64_t>(valid ? grow : 0) * p.ld + (valid ? col : 0);
      cp_async16((which ? Bs : As) + row * S + col, src, valid * 8);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    double acc[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int ks = 0; ks < K16 / 4; ++ks) {
      const int kk = ks * 4 + tig;
      const double a0 = As[(wm * 16 + gid) * S + kk], a1 = As[(wm * 16 + 8 + gid) * S + kk];
      const double b0v = Bs[(wn * 16 + gid) * S + kk], b1v = Bs[(wn * 16 + 8 + gid) * S + kk];
      dmma_884(acc[0][0], a0, b0v);
      dmma_884(acc[0][1], a0, b1v);
      dmma_884(acc[1][0], a1, b0v);
      dmma_884(acc[1][1], a1, b1v);
    }
    const bool last = k == N - 1;
    const double coef = p.coef[k];  // multiplies C_{k+1}
    double e2 = 0.0;
    double* nxt = p.C[k & 1];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double cn = ok[q] ? 2.0 * cv[q] - acc[q >> 2][(q >> 1) & 1][q & 1] : 0.0;
      pv[q] -= coef * cn;
      cv[q] = cn;
      const double dv = ok[q] ? cn - (rr[q] == cc[q] ? 1.0 : 0.0) : 0.0;
      e2 += wgt * dv * dv;
      if (!last && ok[q]) {
        nxt[mb + static_cast<int64_t>(rr[q]) * p.ld + cc[q]] = cn;
        nxt[mb + static_cast<int64_t>(cc[q]) * p.ld + rr[q]] = cn;
      }
    }
    if (last) break;
    e2 = warp_sum(e2);
    if (lane == 0) red[warp] = e2;
    __syncthreads();  // also: every warp is done with As/Bs before the next step refills them
    if (threadIdx.x == 0) cf_arrive(p.gbar, k + 1, red[0] + red[1] + red[2] + red[3]);
  }
  // final P (tile + mirror) for finalize_p_kernel<0>
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (!ok[q]) continue;
    p.P[mb + static_cast<int64_t>(rr[q]) * p.ld + cc[q]] = pv[q];
    p.P[mb + static_cast<int64_t>(cc[q]) * p.ld + rr[q]] = pv[q];
  }
  if (threadIdx.x == 0 && blockIdx.x % p.tiles_per_mat == 0) p.scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_STEPS] = steps;
}

}  // namespace unso
