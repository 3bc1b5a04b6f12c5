// Reference: ortho.py:153-157 (scale), 197-204 (squarings, P) for large h.
// Glue-free multi-launch pipeline for large h (tiles > co-resident CTAs):
//   K1 gram epilogue -> G as bf16 hi/lo (upper pair tiles) + per-warp norm partials
//   scalars          -> s^2, 1/s, status               (fixed-order reduction, deterministic)
//   K2 step 1        -> C_1 = G/s^2 folded into the epilogue, P initialised (no P read)
//   K2 steps 2..N-1  -> C-form squarings, the last one emitting P statistics
//   decision         -> identity shift d, adaptive apply bound (as in chain_persistent.cuh)
//   finalize P       -> (P - d I)/s, bf16 hi/lo, symmetric
// Norm/statistics partials are written per (matrix, pair tile, 32-row group, 32-column chunk)
// by lane 0 after a warp reduction: no atomics, bitwise reproducible.
#pragma once
#include "common.cuh"
#include "elementwise.cuh"

namespace unso {

__device__ __forceinline__ int upper_tile_index(int tm, int tn, int nt) {
  return tm * nt - tm * (tm - 1) / 2 + (tn - tm);
}

// Slot of a (b, pair tile, row group, chunk) partial: row group = (row >> 5) & 7, chunk = (col0 >> 5) & 7.
__device__ __forceinline__ int64_t partial_slot(int b, int row, int col0, int nt) {
  const int tm = row >> 8, tn = col0 >> 8;
  const int T = nt * (nt + 1) / 2;
  return ((static_cast<int64_t>(b) * T + upper_tile_index(tm, tn, nt)) * 8 + ((row >> 5) & 7)) * 8 + ((col0 >> 5) & 7);
}

// Gram epilogue (CTA-pair engine, no split-K): G tile -> bf16 hi/lo + norm partials.
struct UEpiGramSplit {
  __nv_bfloat16* hi;
  __nv_bfloat16* lo;
  double* part;  // [slots][3]: trace, weighted ||.||^2, 0
  int64_t ld, bs;
  int h, nt;
  __device__ __forceinline__ void operator()(int b, int, int row, int col0, const float (&v)[32]) const {
    const bool rok = row < h;
    const double w = ((row >> 8) == (col0 >> 8)) ? 1.0 : 2.0;  // off-diagonal pair tiles stand for both triangles
    double tr = 0.0, fr = 0.0;
    uint32_t hw[16], lw[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = col0 + 2 * j;
      const bool ok0 = rok && c < h, ok1 = rok && c + 1 < h;
      const float x0 = ok0 ? v[2 * j] : 0.f, x1 = ok1 ? v[2 * j + 1] : 0.f;
      fr += w * (static_cast<double>(x0) * x0 + static_cast<double>(x1) * x1);
      if (c == row) tr += x0;
      if (c + 1 == row) tr += x1;
      const uint32_t hh = pack_bf16x2(x0, x1);
      hw[j] = hh;
      lw[j] = pack_bf16x2(x0 - bf16_lo_to_f32(hh), x1 - bf16_hi_to_f32(hh));
    }
    tr = warp_sum(tr);
    fr = warp_sum(fr);
    if ((threadIdx.x & 31) == 0) {
      double* o = part + partial_slot(b, row, col0, nt) * 3;
      o[0] = tr;
      o[1] = fr;
      o[2] = 0.0;
    }
    if (!rok) return;
    const int64_t o = static_cast<int64_t>(b) * bs + static_cast<int64_t>(row) * ld + col0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // 256-bit stores: whole sectors (ld % 256 == 0)
      st_global_v8(hi + o + 16 * j, *reinterpret_cast<const uint32_t(*)[8]>(hw + 8 * j));
      st_global_v8(lo + o + 16 * j, *reinterpret_cast<const uint32_t(*)[8]>(lw + 8 * j));
    }
  }
};

// Split-K finalize for the multi-launch path: sum partials -> bf16 hi/lo (both triangles)
// + one norm partial per 32x32 upper tile.
__global__ void finalize_split_kernel(const float* __restrict__ part, int splits, int batch, int h, int64_t ld,
                                      __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo,
                                      double* __restrict__ norms) {
  __shared__ float tile[32][33];
  __shared__ double scratch[32];
  const int nt = (h + 31) / 32;
  int ti, tj;
  sym_tile_coords(blockIdx.x, nt, ti, tj);
  const int b = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t mat = static_cast<int64_t>(h) * ld;
  double tr = 0.0, fr = 0.0;
  for (int r = ty; r < 32; r += 8) {
    const int gr = ti * 32 + r, gc = tj * 32 + tx;
    float s = 0.f;
    if (gr < h && gc < h) {
      for (int sp = 0; sp < splits; ++sp)
        s += part[(static_cast<int64_t>(sp) * batch + b) * mat + static_cast<int64_t>(gr) * ld + gc];
      if (gr == gc) tr += s;
      if (gr <= gc) fr += (gr == gc ? 1.0 : 2.0) * static_cast<double>(s) * s;
    }
    tile[r][tx] = s;
  }
  __syncthreads();
  const int64_t off = static_cast<int64_t>(b) * mat;
  for (int r = ty; r < 32; r += 8) {
    const int gr = ti * 32 + r, gc = tj * 32 + tx;
    if (gr < h && gc < h) split_bf16((ti == tj && r > tx) ? tile[tx][r] : tile[r][tx], hi[off + static_cast<int64_t>(gr) * ld + gc],
                                     lo[off + static_cast<int64_t>(gr) * ld + gc]);
    if (ti != tj) {
      const int mr = tj * 32 + r, mc = ti * 32 + tx;
      if (mr < h && mc < h) split_bf16(tile[tx][r], hi[off + static_cast<int64_t>(mr) * ld + mc], lo[off + static_cast<int64_t>(mr) * ld + mc]);
    }
  }
  tr = block_sum(tr, scratch);
  const double trs = tr;
  fr = block_sum(fr, scratch);
  if (threadIdx.x == 0) {
    double* o = norms + (static_cast<int64_t>(b) * gridDim.x + blockIdx.x) * 3;
    o[0] = trs;
    o[1] = fr;
    o[2] = 0.0;
  }
}

// Per matrix: reduce the final-P statistics (trace P, weighted ||P||^2) -> identity shift d,
// adaptive apply bound and mode (same rule as chain_persistent.cuh).
__global__ void apply_decision_kernel(const double* __restrict__ pstat, int nslots, double* __restrict__ scal, int h,
                                      int adaptive, double tau) {
  __shared__ double scratch[32];
  const int b = blockIdx.x;
  double t0 = 0.0, t1 = 0.0;
  for (int i = threadIdx.x; i < nslots; i += blockDim.x) {
    t0 += pstat[(static_cast<int64_t>(b) * nslots + i) * 2 + 0];
    t1 += pstat[(static_cast<int64_t>(b) * nslots + i) * 2 + 1];
  }
  t0 = block_sum(t0, scratch);
  const double tp = t0;
  t1 = block_sum(t1, scratch);
  if (threadIdx.x != 0) return;
  double* o = scal + static_cast<int64_t>(b) * SCAL_STRIDE;
  const double d = tp / h;
  const double r2 = fmax(t1 - tp * tp / h, 0.0);
  const double trc = fmax(o[S_TRACE] / o[S_S2], 0.0);
  const double bound = ldexp(sqrt(r2), -9) / fmax(sqrt(trc), 1e-300);
  o[S_SHIFT] = d * o[S_INV_S];
  o[S_MODE] = (adaptive && bound <= tau) ? 1.0 : 0.0;
  o[S_BOUND] = bound;
}

// One squaring step's epilogue on the CTA's rows of an upper pair tile (register resident).
//   first: the stored C is the unscaled Gram G; C_1 = G/s^2 and P = alpha I - a_1 C_1 - a_2 C_2.
//   pstat: on the last step, per-warp partials of trace(P) and weighted ||P||^2.
struct EpiChainStep {
  const __nv_bfloat16* chi;
  const __nv_bfloat16* clo;
  __nv_bfloat16* nhi;
  __nv_bfloat16* nlo;
  float* P;
  int64_t ld, bs;
  int h, nt;
  float coef;          // multiplies C_{k+1}
  int write_next;
  int first;
  float coef1;         // first step: multiplies C_1
  double alpha;        // first step: 1 + sum a + b
  const double* scal;  // first step: s^2
  double* pstat;       // last step: statistics partials (nullable)
  uint8_t* n8hi = nullptr;  // optional e4m3 operand copies of C_{k+1}: 2^8 hi, 2^16 (C - hi)
  uint8_t* n8lo = nullptr;
  float in_hi_scale = 1.f;   // stored hi of C_k is (2^12 hi) when produced for the fp8 kernel
  float out_hi_scale = 1.f;  // scale of the stored hi of C_{k+1} (2^12 when n8hi is set)
  uint8_t* n8i = nullptr;    // interleaved [hi8 | lo8] per 64-column block (row stride ld8i bytes)
  int64_t ld8i = 0;
  __device__ __forceinline__ void operator()(int b, int, int row, int col0, const float (&v)[32]) const {
    const bool rok = row < h;
    const int64_t o = static_cast<int64_t>(b) * bs + static_cast<int64_t>(row) * ld + col0;
    float cs = 1.f, as = 1.f;
    if (first) {
      const double is2 = 1.0 / scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_S2];
      cs = static_cast<float>(is2);
      as = static_cast<float>(is2 * is2);
    }
    uint32_t hw[16], lw[16];
    float pv[32];
    if (rok) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 a = *reinterpret_cast<const uint4*>(chi + o + 8 * j);
        const uint4 c = *reinterpret_cast<const uint4*>(clo + o + 8 * j);
        hw[4 * j] = a.x; hw[4 * j + 1] = a.y; hw[4 * j + 2] = a.z; hw[4 * j + 3] = a.w;
        lw[4 * j] = c.x; lw[4 * j + 1] = c.y; lw[4 * j + 2] = c.z; lw[4 * j + 3] = c.w;
      }
      if (!first) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 t = *reinterpret_cast<const float4*>(P + o + 4 * j);
          pv[4 * j] = t.x; pv[4 * j + 1] = t.y; pv[4 * j + 2] = t.z; pv[4 * j + 3] = t.w;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) hw[j] = lw[j] = 0u;
    }
    uint32_t nh[16], nl[16], q8h[16], q8l[16];
    double tr = 0.0, fr = 0.0;
    const double w = ((row >> 8) == (col0 >> 8)) ? 1.0 : 2.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      // Padding columns [h, ldc) hold bytes no epilogue owns (stale workspace): force them to zero
      // so the stored state is exactly zero-padded -- the interleaved e4m3 operand map spans the
      // padding (no TMA zero fill there) and stale NaN times a zero partner is still NaN.
      const bool cok0 = col0 + 2 * j < h, cok1 = col0 + 2 * j + 1 < h;
      const float c0v = cok0 ? fmaf(bf16_lo_to_f32(hw[j]), in_hi_scale, bf16_lo_to_f32(lw[j])) * cs : 0.f;
      const float c1v = cok1 ? fmaf(bf16_hi_to_f32(hw[j]), in_hi_scale, bf16_hi_to_f32(lw[j])) * cs : 0.f;
      const float n0 = cok0 ? 2.0f * c0v - v[2 * j] * as : 0.f;
      const float n1 = cok1 ? 2.0f * c1v - v[2 * j + 1] * as : 0.f;
      if (!first) {
        if (!cok0) pv[2 * j] = 0.f;
        if (!cok1) pv[2 * j + 1] = 0.f;
      }
      if (first) {
        const int c = col0 + 2 * j;
        pv[2 * j] = static_cast<float>((c == row ? alpha : 0.0) - static_cast<double>(coef1) * c0v);
        pv[2 * j + 1] = static_cast<float>((c + 1 == row ? alpha : 0.0) - static_cast<double>(coef1) * c1v);
      }
      pv[2 * j] -= coef * n0;
      pv[2 * j + 1] -= coef * n1;
      const uint32_t hh = pack_bf16x2(n0, n1);
      const float h0 = bf16_lo_to_f32(hh), h1 = bf16_hi_to_f32(hh);
      nh[j] = out_hi_scale == 1.f ? hh : pack_bf16x2(h0 * out_hi_scale, h1 * out_hi_scale);  // exact rescale
      nl[j] = pack_bf16x2(n0 - h0, n1 - h1);
      if (n8hi) {
        q8h[j] = pack_e4m3x2(h0 * 256.0f, h1 * 256.0f);
        q8l[j] = pack_e4m3x2((n0 - h0) * 65536.0f, (n1 - h1) * 65536.0f);
      }
      if (pstat) {
        const int c = col0 + 2 * j;
        const bool ok0 = rok && c < h, ok1 = rok && c + 1 < h;
        if (ok0) fr += w * static_cast<double>(pv[2 * j]) * pv[2 * j];
        if (ok1) fr += w * static_cast<double>(pv[2 * j + 1]) * pv[2 * j + 1];
        if (ok0 && c == row) tr += pv[2 * j];
        if (ok1 && c + 1 == row) tr += pv[2 * j + 1];
      }
    }
    if (pstat) {
      tr = warp_sum(tr);
      fr = warp_sum(fr);
      if ((threadIdx.x & 31) == 0) {
        double* s = pstat + partial_slot(b, row, col0, nt) * 2;
        s[0] = tr;
        s[1] = fr;
      }
    }
    if (!rok) return;
    if (write_next) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        *reinterpret_cast<uint4*>(nhi + o + 8 * j) = make_uint4(nh[4 * j], nh[4 * j + 1], nh[4 * j + 2], nh[4 * j + 3]);
        *reinterpret_cast<uint4*>(nlo + o + 8 * j) = make_uint4(nl[4 * j], nl[4 * j + 1], nl[4 * j + 2], nl[4 * j + 3]);
      }
      if (n8hi) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          *reinterpret_cast<uint4*>(n8hi + o + 16 * j) =
              make_uint4(q8h[8 * j] | (q8h[8 * j + 1] << 16), q8h[8 * j + 2] | (q8h[8 * j + 3] << 16),
                         q8h[8 * j + 4] | (q8h[8 * j + 5] << 16), q8h[8 * j + 6] | (q8h[8 * j + 7] << 16));
          *reinterpret_cast<uint4*>(n8lo + o + 16 * j) =
              make_uint4(q8l[8 * j] | (q8l[8 * j + 1] << 16), q8l[8 * j + 2] | (q8l[8 * j + 3] << 16),
                         q8l[8 * j + 4] | (q8l[8 * j + 5] << 16), q8l[8 * j + 6] | (q8l[8 * j + 7] << 16));
        }
        // interleaved copy: row r, 64-column block k: [hi8 (64 B) | lo8 (64 B)]
        uint8_t* ri = n8i + static_cast<int64_t>(b) * (bs / ld) * ld8i + static_cast<int64_t>(row) * ld8i +
                      (col0 >> 6) * 128 + (col0 & 63);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          *reinterpret_cast<uint4*>(ri + 16 * j) =
              make_uint4(q8h[8 * j] | (q8h[8 * j + 1] << 16), q8h[8 * j + 2] | (q8h[8 * j + 3] << 16),
                         q8h[8 * j + 4] | (q8h[8 * j + 5] << 16), q8h[8 * j + 6] | (q8h[8 * j + 7] << 16));
          *reinterpret_cast<uint4*>(ri + 64 + 16 * j) =
              make_uint4(q8l[8 * j] | (q8l[8 * j + 1] << 16), q8l[8 * j + 2] | (q8l[8 * j + 3] << 16),
                         q8l[8 * j + 4] | (q8l[8 * j + 5] << 16), q8l[8 * j + 6] | (q8l[8 * j + 7] << 16));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<float4*>(P + o + 4 * j) = make_float4(pv[4 * j], pv[4 * j + 1], pv[4 * j + 2], pv[4 * j + 3]);
  }

  // Row-coalesced form of the same step for a 32 x 32 block staged in shared memory (chain_pair.cuh
  // stage_block32): lane = (row sub-index, 4-column group), 4 rows per warp instruction, so every
  // global access is a run of whole 32-byte sectors instead of 32 scattered 16-byte pieces.
  // Extra knobs of this form: coefk (pending coefficient of C_k, added here when the previous step
  // skipped its P update) and write_p (0: leave P untouched, the coefficient stays pending).
  float coefk = 0.f;
  int write_p = 1;
  __device__ __forceinline__ void rows4(int b, int, int row0, int col0, const float* stage) const {
    const int lane = threadIdx.x & 31, cg = lane & 7, rs = lane >> 3;
    float cs = 1.f, as = 1.f;
    if (first) {
      const double is2 = 1.0 / scal[static_cast<int64_t>(b) * SCAL_STRIDE + S_S2];
      cs = static_cast<float>(is2);
      as = static_cast<float>(is2 * is2);
    }
    const int c = col0 + 4 * cg;
    const double w = ((row0 >> 8) == (col0 >> 8)) ? 1.0 : 2.0;
    double tr = 0.0, fr = 0.0;
    // all eight rows' loads first, so their latencies overlap
    uint2 hwv[8], lwv[8];
    float4 pvv[8];
    const bool load_p = !first && write_p;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int row = row0 + it * 4 + rs;
      const int64_t o = static_cast<int64_t>(b) * bs + static_cast<int64_t>(row) * ld + c;
      const bool ok = row < h;
      hwv[it] = ok ? *reinterpret_cast<const uint2*>(chi + o) : make_uint2(0u, 0u);
      lwv[it] = ok ? *reinterpret_cast<const uint2*>(clo + o) : make_uint2(0u, 0u);
      pvv[it] = (ok && load_p) ? *reinterpret_cast<const float4*>(P + o) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int r = it * 4 + rs, row = row0 + r;
      const float4 acc = *reinterpret_cast<const float4*>(stage + r * 32 + ((cg ^ (r & 7)) << 2));
      if (row >= h) continue;
      const int64_t o = static_cast<int64_t>(b) * bs + static_cast<int64_t>(row) * ld + c;
      const uint2 hw = hwv[it];
      const uint2 lw = lwv[it];
      float pv[4] = {pvv[it].x, pvv[it].y, pvv[it].z, pvv[it].w};
      float cv[4] = {fmaf(bf16_lo_to_f32(hw.x), in_hi_scale, bf16_lo_to_f32(lw.x)) * cs,
                     fmaf(bf16_hi_to_f32(hw.x), in_hi_scale, bf16_hi_to_f32(lw.x)) * cs,
                     fmaf(bf16_lo_to_f32(hw.y), in_hi_scale, bf16_lo_to_f32(lw.y)) * cs,
                     fmaf(bf16_hi_to_f32(hw.y), in_hi_scale, bf16_hi_to_f32(lw.y)) * cs};
      const float av[4] = {acc.x, acc.y, acc.z, acc.w};
      float nv[4], hv[4];
      uint32_t nh[2], nl[2], q8h = 0u, q8l = 0u;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (c + e >= h) {  // zero padding columns (see operator())
          cv[e] = 0.f;
          pv[e] = 0.f;
        }
        nv[e] = c + e < h ? 2.0f * cv[e] - av[e] * as : 0.f;
        if (first) pv[e] = static_cast<float>((c + e == row ? alpha : 0.0) - static_cast<double>(coef1) * cv[e]);
        else pv[e] -= coefk * cv[e];
        pv[e] -= coef * nv[e];
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t hh = pack_bf16x2(nv[2 * e], nv[2 * e + 1]);
        hv[2 * e] = bf16_lo_to_f32(hh);
        hv[2 * e + 1] = bf16_hi_to_f32(hh);
        nh[e] = out_hi_scale == 1.f ? hh : pack_bf16x2(hv[2 * e] * out_hi_scale, hv[2 * e + 1] * out_hi_scale);
        nl[e] = pack_bf16x2(nv[2 * e] - hv[2 * e], nv[2 * e + 1] - hv[2 * e + 1]);
      }
      if (n8hi) {
        q8h = pack_e4m3x2(hv[0] * 256.0f, hv[1] * 256.0f) | (pack_e4m3x2(hv[2] * 256.0f, hv[3] * 256.0f) << 16);
        q8l = pack_e4m3x2((nv[0] - hv[0]) * 65536.0f, (nv[1] - hv[1]) * 65536.0f) |
              (pack_e4m3x2((nv[2] - hv[2]) * 65536.0f, (nv[3] - hv[3]) * 65536.0f) << 16);
      }
      if (pstat) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (c + e < h) {
            fr += w * static_cast<double>(pv[e]) * pv[e];
            if (c + e == row) tr += pv[e];
          }
        }
      }
      if (write_next) {
        *reinterpret_cast<uint2*>(nhi + o) = make_uint2(nh[0], nh[1]);
        *reinterpret_cast<uint2*>(nlo + o) = make_uint2(nl[0], nl[1]);
        if (n8hi) {
          *reinterpret_cast<uint32_t*>(n8hi + o) = q8h;
          *reinterpret_cast<uint32_t*>(n8lo + o) = q8l;
          uint8_t* ri = n8i + static_cast<int64_t>(b) * (bs / ld) * ld8i + static_cast<int64_t>(row) * ld8i +
                        (c >> 6) * 128 + (c & 63);
          *reinterpret_cast<uint32_t*>(ri) = q8h;
          *reinterpret_cast<uint32_t*>(ri + 64) = q8l;
        }
      }
      if (first || write_p) *reinterpret_cast<float4*>(P + o) = make_float4(pv[0], pv[1], pv[2], pv[3]);
    }
    if (pstat) {
      tr = warp_sum(tr);
      fr = warp_sum(fr);
      if ((threadIdx.x & 31) == 0) {
        double* s = pstat + partial_slot(b, row0, col0, nt) * 2;
        s[0] = tr;
        s[1] = fr;
      }
    }
  }
};

}  // namespace unso
