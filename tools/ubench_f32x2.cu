// Microbenchmark: issue throughput of paired fp32 (FFMA2/FADD2) vs scalar FFMA on sm_100a,
// alone and interleaved with integer ALU work.  Prints warp-instructions and fp32 ops per
// clock per SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench_f32x2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ unsigned long long f2(float a, float b) {
  return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}

template <int MODE>
__global__ void bench(float* out, float s, int iadd) {
  float x[8];
  unsigned long long p[4];
  int k[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { x[j] = threadIdx.x * 0.001f + j; k[j] = threadIdx.x + j; }
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j] = f2(x[2 * j], x[2 * j + 1]);
  const unsigned long long ss = f2(s, s), cc = f2(0.5f, 0.5f);
  for (int it = 0; it < ITERS; ++it) {
    if (MODE == 0 || MODE == 2) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = __fmaf_rn(x[j], s, 0.5f);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[j]) : "l"(ss), "l"(cc));
    }
    if (MODE >= 2) {
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("add.u32 %0, %0, %1;" : "+r"(k[j]) : "r"(iadd));
    }
  }
  float r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += x[j] + __uint_as_float((unsigned)(p[j / 2] >> (32 * (j & 1)))) + k[j];
  if (r == 12345.f) out[0] = r;
}

template <int MODE>
void run(const char* name, int sms, int clk_khz) {
  float* d;
  cudaMalloc(&d, 4);
  int blocks = sms * 4, threads = 512;
  bench<MODE><<<blocks, threads>>>(d, 1.0001f, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) bench<MODE><<<blocks, threads>>>(d, 1.0001f, 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double clocks = ms * 1e-3 * clk_khz * 1e3;
  double warps = 10.0 * blocks * threads / 32;
  double fpops = warps * 32 * ITERS * 8;                       // scalar-equivalent fp32 FMAs
  double inst = warps * ITERS * ((MODE == 0 || MODE == 2) ? 8 : 4) + (MODE >= 2 ? warps * ITERS * 8 : 0);
  printf("%-28s %.3f ms  fp32 FMA/clk/SM %.1f  warp-inst/clk/SM %.2f\n", name, ms,
         fpops / clocks / sms, inst / clocks / sms);
  cudaFree(d);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  run<0>("FFMA x8", sms, clk);
  run<1>("FFMA2 x4", sms, clk);
  run<2>("FFMA x8 + IADD x8", sms, clk);
  run<3>("FFMA2 x4 + IADD x8", sms, clk);
  return 0;
}
