// MUFU throughput probe: tanh.approx.f32 / tanh.approx.f16x2 / ex2.approx per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
#define OP(x)                                                                                 \
    if (MODE == 0) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x));                       \
    else if (MODE == 1) { uint32_t u = __float_as_uint(x); asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(u)); x = __uint_as_float(u); } \
    else asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));
    OP(a0) OP(a1) OP(a2) OP(a3) OP(a4) OP(a5) OP(a6) OP(a7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int mode = 0; mode < 3; ++mode) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, threads = 1024;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(o, iters);
      else if (mode == 1) k<1><<<blocks, threads>>>(o, iters);
      else k<2><<<blocks, threads>>>(o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 8;   // instructions x lanes
    printf("mode %d (%s): %.1f lane-ops/clk/SM at %d MHz nominal\n", mode, mode == 0 ? "tanh.f32" : mode == 1 ? "tanh.f16x2" : "ex2.f32",
           ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
  }
  return 0;
}
