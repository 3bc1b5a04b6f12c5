// Row-sharded Gram with the cross-rank sum done over NVLink peer memory, replacing
// unso_gram + ncclAllReduce for configs[3].  Three stream-ordered phases per rank:
//
//   1. push   : the CTA-pair Gram kernel's epilogue (UEpiPushF32) stores each 256 x 256 partial tile
//               (fp32, per split-K slice) straight into the slot buffer of the tile's OWNER rank
//               (owner = tile % world) with 256-bit stores to the peer-mapped address -- the
//               transfer overlaps the rest of the Gram; then one thread publishes "my partials are
//               in" to every rank's flag word (system-scope release).
//   2. reduce : each rank waits for every rank's phase-1 flag, sums the world x splits partials of
//               the tiles it owns in a fixed order (bit-identical on every rank), and writes the
//               reduced tile and its mirror into EVERY rank's dense G buffer; the last CTA
//               publishes phase-2 completion.
//   3. wait   : one thread waits for every rank's phase-2 flag; G is then complete locally and
//               unso_orthogonalize_from_gram continues as before.
//
// Flags are per-call epochs (monotonic), so nothing is reset between calls.  Splitting the phases
// lets one GPU emulate all ranks (run phase 1 for every rank, then phase 2, then 3) without any
// kernel ever spinning on work that has not been launched -- the multi-rank path is tested that
// way (tests/test_gpu_parity.py), and with world = 1 through real symmetric memory.
#pragma once
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace unso {

constexpr int GAR_MAX_WORLD = 8;
constexpr int GAR_TILE = 256;

// Slot of (source rank, split, owned tile j) in an owner's slot buffer, in floats.
__host__ __device__ inline int64_t gar_slot_offset(int src, int split, int j, int splits, int owned) {
  return ((static_cast<int64_t>(src) * splits + split) * owned + j) * (GAR_TILE * GAR_TILE);
}
__host__ __device__ inline int gar_tiles(int h) {
  const int nt = (h + GAR_TILE - 1) / GAR_TILE;
  return nt * (nt + 1) / 2;
}
__host__ __device__ inline int gar_owned_max(int h, int world) { return (gar_tiles(h) + world - 1) / world; }

struct GarPeers {
  float* slots[GAR_MAX_WORLD];     // every rank's slot buffer (peer-mapped)
  float* g[GAR_MAX_WORLD];         // every rank's dense h x h G buffer (peer-mapped)
  uint32_t* flags[GAR_MAX_WORLD];  // every rank's flag words [2][world] (peer-mapped)
};

// Phase 1 epilogue of the CTA-pair Gram: one lane = one row of 32 columns of a 256 x 256 pair tile.
struct UEpiPushF32 {
  GarPeers peers;
  int rank, world, splits, owned, h, nt;
  __device__ void operator()(int, int split, int row, int col0, const float* v) const {
    if (row >= h) return;
    const int tm = row / GAR_TILE, tn = col0 / GAR_TILE;
    const int t = tm * nt - tm * (tm - 1) / 2 + (tn - tm);  // upper pair-tile index
    const int owner = t % world, j = t / world;
    float* dst = peers.slots[owner] + gar_slot_offset(rank, split, j, splits, owned) +
                 static_cast<int64_t>(row % GAR_TILE) * GAR_TILE + (col0 % GAR_TILE);
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
      uint32_t w[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) w[e] = __float_as_uint(v[q + e]);
      st_global_v8(dst + q, w);
    }
  }
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void gar_wait_all(const uint32_t* flags, int world, uint32_t epoch) {
  const long long t0 = clock64();
  for (int r = 0; r < world; ++r) {
    while (static_cast<int32_t>(ld_acquire_sys(flags + r) - epoch) < 0) {
      __nanosleep(128);
      if (clock64() - t0 > UNSO_WATCHDOG_CYCLES) __trap();
    }
  }
}

// flag word `which` (0: partials pushed, 1: reduced tiles delivered) of every rank := epoch
__global__ void gar_signal_kernel(GarPeers peers, int rank, int world, int which, uint32_t epoch) {
  __threadfence_system();
  for (int q = 0; q < world; ++q) st_release_sys(peers.flags[q] + which * world + rank, epoch);
}

__global__ void gar_wait_kernel(const uint32_t* my_flags, int world, int which, uint32_t epoch) {
  gar_wait_all(my_flags + which * world, world, epoch);
  __threadfence();
}

// Phase 2: block (j, sub) reduces the 32 x 32 sub-block `sub` of owned tile j and delivers it (and
// its mirror) to every rank.  `done` counts finished blocks (zeroed before launch); the last one
// publishes phase-2 completion.
__global__ void __launch_bounds__(256) gar_reduce_kernel(GarPeers peers, int rank, int world, int splits, int owned,
                                                         int h, int nt, uint32_t epoch, unsigned* done) {
  __shared__ float tile[32][33];
  __shared__ bool last;
  if (threadIdx.x == 0) gar_wait_all(peers.flags[rank], world, epoch);
  __syncthreads();
  const int j = blockIdx.x, sub = blockIdx.y;
  const int t = j * world + rank;  // the tile this rank owns
  const int T = nt * (nt + 1) / 2;
  if (t < T) {
    int tm = 0, rem = t, len = nt;
    while (rem >= len) {
      rem -= len;
      ++tm;
      --len;
    }
    const int tn = tm + rem;
    const int sr = (sub / 8) * 32, sc = (sub % 8) * 32;  // sub-block origin inside the 256 x 256 tile
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const float* mine = peers.slots[rank];
    for (int r = ty; r < 32; r += 8) {
      float s = 0.f;
      for (int src = 0; src < world; ++src)  // fixed order: identical sums on every rank
        for (int sp = 0; sp < splits; ++sp)
          s += __ldcg(mine + gar_slot_offset(src, sp, j, splits, owned) + (sr + r) * GAR_TILE + sc + tx);
      tile[r][tx] = s;
    }
    __syncthreads();
    const int gr0 = tm * GAR_TILE + sr, gc0 = tn * GAR_TILE + sc;
    for (int q = 0; q < world; ++q) {
      float* g = peers.g[q];
      for (int r = ty; r < 32; r += 8) {
        const int gr = gr0 + r, gc = gc0 + tx;
        if (gr < h && gc < h) g[static_cast<int64_t>(gr) * h + gc] = tile[r][tx];
        if (tm != tn) {  // mirror: row gc0 + r of G takes column r of the sub-block
          const int mr = gc0 + r, mc = gr0 + tx;
          if (mr < h && mc < h) g[static_cast<int64_t>(mr) * h + mc] = tile[tx][r];
        }
      }
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < world; ++q) st_release_sys(peers.flags[q] + world + rank, epoch);
  }
}

}  // namespace unso
