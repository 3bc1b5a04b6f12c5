// Microbenchmark: dense tensor-core peak of tcgen05.mma on CTA pairs (M = 256, N = 256) for kind::f16
// (bf16, K = 16) and kind::i8 (s8, K = 32): back-to-back MMAs from shared memory into TMEM, no
// loads, 74 pairs.  Gives the measured int8 : bf16 ratio behind the fp32-mode roofline.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2602_02500_b200/csrc -o tc_peak tc_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx_sm100.cuh"
using namespace unso;

template <bool I8, bool NEG = false>
__global__ void __launch_bounds__(128, 1) peak_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  cluster_sync_all();
  if (warp == 0) tmem_alloc_pair(&tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  unsigned long long t0 = 0, t1 = 0;
  if (rank == 0 && warp == 1) {
    const uint32_t a = smem_u32(smem), b = a + 32768;
    const uint64_t da = sdesc_sw128(a, 16, 1024), db = sdesc_sw128(b, 16, 1024);
    const uint32_t idesc = I8 ? ((2u << 4) | (1u << 7) | (1u << 10) | (256u >> 3 << 17) | (256u >> 4 << 24))
                              : (idesc_bf16(256, 256, 0, 0) | (NEG ? IDESC_NEGATE_A : 0u));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t acc = (i > 0 || u > 0) ? 1u : 0u;
        if (I8)
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (u & 1) * 256),
                       "l"(da + 2 * u), "l"(db + 2 * u), "r"(idesc), "r"(acc)
                       : "memory");
        else
          umma_bf16_pair_warp(tmem + (u & 1) * 256, da + 2 * u, db + 2 * u, idesc, acc);
      }
    }
    umma_commit_pair_warp(&done, 0x3);
  }
  mbar_wait(&done, 0);
  if (rank == 0 && warp == 1 && (threadIdx.x & 31) == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[blockIdx.x >> 1] = t1 - t0;
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

template <bool I8, bool NEG = false>
void run(int sms) {
  const int pairs = sms / 2, iters = 20000;
  unsigned long long* d;
  cudaMalloc(&d, pairs * 8);
  cudaFuncSetAttribute(peak_kernel<I8, NEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 65536;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, peak_kernel<I8, NEG>, iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double k = I8 ? 32 : 16;
  const double ops = 2.0 * 256 * 256 * k * 8.0 * iters * pairs;
  printf("%s: %.3f ms, %.1f T%s/s dense (%d pairs, M=256 N=256 K=%d per instruction) err=%s\n",
         I8 ? "kind::i8 " : (NEG ? "kind::f16 negated A" : "kind::f16"), ms, ops / (ms * 1e-3) / 1e12, I8 ? "OP" : "FLOP", pairs, (int)k,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<false>(sms);
  run<false, true>(sms);
  run<true>(sms);
  run<false>(sms);
  run<true>(sms);
  return 0;
}
