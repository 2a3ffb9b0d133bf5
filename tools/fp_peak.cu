// Measured arithmetic peaks of the instructions the pass kernels use (no memory traffic):
//   FFMA2 (fma.rn.f32x2, 2 FP32 lane-ops each), FFMA (scalar fp32), DFMA (fp64), SHFL.
// Each thread runs 16 independent dependency chains; grid = SMs x 8 CTAs x 256 threads.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp tools/fp_peak.cu && /tmp/fp
#include <cuda_runtime.h>
#include <stdio.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

constexpr int ITERS = 4096;

__global__ void k_ffma2(u64* out, u64 c) {
  u64 x[16];
  for (int i = 0; i < 16; ++i) x[i] = c + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma2(x[i], c, c);
  u64 s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  if (s == 0x1234) out[0] = s;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
// MODE 0: FADD2 only, 1: FMUL2 only, 2: FFMA2 + FADD2 alternating (co-issue?)
template <int MODE>
__global__ void k_mix2(u64* out, u64 c) {
  u64 x[16];
  for (int i = 0; i < 16; ++i) x[i] = c + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = MODE == 0 ? add2(x[i], c) : MODE == 1 ? mul2(x[i], c) : ((i & 1) ? add2(x[i], c) : fma2(x[i], c, c));
  u64 s = 0;
  for (int i = 0; i < 16; ++i) s ^= x[i];
  if (s == 0x1234) out[0] = s;
}
__global__ void k_ffma(float* out, float c) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = c + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], c, c);
  float s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.f) out[0] = s;
}
__global__ void k_dfma(double* out, double c) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = c + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], c, c);
  double s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.0) out[0] = s;
}
__global__ void k_shfl(float* out, float c) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = c + threadIdx.x + i;
  for (int it = 0; it < ITERS / 4; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = __shfl_xor_sync(0xffffffffu, x[i], 1 + (i & 15));
  float s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.f) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void* buf;
  cudaMalloc(&buf, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  auto run = [&](const char* name, double ops_per_thread, auto f) {
    f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      f();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double ops = ops_per_thread * blocks * threads;
    printf("%-6s %8.3f ms  %8.2f T lane-ops/s  = %6.1f lane-ops/clk/SM at %d MHz\n", name, best, ops / best / 1e9,
           ops / (best * 1e-3) / sms / (clk * 1e3), clk / 1000);
  };
  run("FFMA2", 2.0 * ITERS * 16, [&] { k_ffma2<<<blocks, threads>>>((u64*)buf, 0x3f8000003f800000ull); });
  run("FADD2", 2.0 * ITERS * 16, [&] { k_mix2<0><<<blocks, threads>>>((u64*)buf, 0x3f8000003f800000ull); });
  run("FMUL2", 2.0 * ITERS * 16, [&] { k_mix2<1><<<blocks, threads>>>((u64*)buf, 0x3f8000003f800000ull); });
  run("MIX2", 2.0 * ITERS * 16, [&] { k_mix2<2><<<blocks, threads>>>((u64*)buf, 0x3f8000003f800000ull); });
  run("FFMA", 1.0 * ITERS * 16, [&] { k_ffma<<<blocks, threads>>>((float*)buf, 1.0001f); });
  run("DFMA", 1.0 * ITERS * 16, [&] { k_dfma<<<blocks, threads>>>((double*)buf, 1.0001); });
  run("SHFL", 1.0 * ITERS / 4 * 16, [&] { k_shfl<<<blocks, threads>>>((float*)buf, 1.0001f); });
  return 0;
}
