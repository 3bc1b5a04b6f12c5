// Microbenchmark: per-SM throughput of the fp64 / conversion instructions the int8 digit engine's
// epilogue and split kernels use (B200).  The operands are loop-carried so the compiler cannot fold
// the conversions.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rates fp64_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void kern(double* out, int iters) {
  double d[4];
  long long q[4];
  float f[4];
  int k[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    d[u] = 1.0 + (threadIdx.x + u) * 1e-9;
    q[u] = 0x123456789ll + threadIdx.x * 7 + u;
    f[u] = 1.0f + threadIdx.x + u;
    k[u] = threadIdx.x + u;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (OP == 0) d[u] = fma(d[u], 1.0000001, 0.5);                            // DFMA
      if (OP == 1) { d[u] = __ll2double_rn(q[u]); q[u] = __double_as_longlong(d[u]) ^ i; }  // I2F.F64.S64
      if (OP == 2) { k[u] = __double2int_rn(d[u]); d[u] = __longlong_as_double(0x3FF0000000000000ll | (k[u] + i)); }  // F2I.S32.F64
      if (OP == 3) { f[u] = __double2float_rn(d[u]); d[u] = __longlong_as_double(0x3FF0000000000000ll | (__float_as_int(f[u]) + i)); }  // F2F.F32.F64
      if (OP == 4) f[u] = fmaf(f[u], 1.0000001f, 0.5f);                          // FFMA
      if (OP == 5) { d[u] = rint(d[u] * 1.5); }                                  // DMUL + FRND.F64
      if (OP == 6) { d[u] = __int2double_rn(k[u]); k[u] = static_cast<int>(__double_as_longlong(d[u]) >> 20) ^ i; }  // I2F.F64.S32
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) s += d[u] + f[u] + q[u] + k[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
float run(double* out, int sms, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    kern<OP><<<sms * 4, 512>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  return ms;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 4 * 512);
  const int iters = 2048;
  const char* names[] = {"DFMA", "I2F.F64.S64 (+LOP)", "F2I.S32.F64 (+LOP)", "F2F.F32.F64 (+LOP)", "FFMA",
                         "DMUL + FRND.F64", "I2F.F64.S32 (+LOP)"};
  float ms[7] = {run<0>(out, sms, iters), run<1>(out, sms, iters), run<2>(out, sms, iters), run<3>(out, sms, iters),
                 run<4>(out, sms, iters), run<5>(out, sms, iters), run<6>(out, sms, iters)};
  for (int op = 0; op < 7; ++op) {
    const double ops = double(sms) * 4 * 512 * iters * 4;
    printf("%-22s %8.3f ms  %7.1f per clk per SM (%d MHz nominal)\n", names[op], ms[op],
           ops / (ms[op] * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
