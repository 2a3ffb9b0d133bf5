// Achievable HBM bandwidth of the access patterns the pass kernels use (2 GiB state, in place):
//   copy      : b = a (torch-style copy, read + write different buffers)
//   rmw1      : a[i] = a[i] * s, grid-stride, one float4 per thread per trip
//   rmwU      : same, U float4 per thread per trip (loads first, then stores)
//   seg16     : 16 x 512 B segments per warp at a group stride (the pass kernels' unit shape)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/membench tools/membench.cu && /tmp/membench
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void rmw1_k(float4* __restrict__ a, size_t n, float s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(a + i);
    v.x *= s; v.y *= s; v.z *= s; v.w *= s;
    __stcs(a + i, v);
  }
}
template <int U>
__global__ void rmwU_k(float4* __restrict__ a, size_t n, float s) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * stride < n ? __ldcs(a + i + u * stride) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u].x *= s; v[u].y *= s; v[u].z *= s; v[u].w *= s;
      if (i + u * stride < n) __stcs(a + i + u * stride, v[u]);
    }
  }
}
// warp unit = 16 segments (512 B each) at segment stride 2^q (group slot), like a KHI=4 pass
template <int MINB>
__global__ void __launch_bounds__(256, MINB) seg16_k(float4* __restrict__ a, size_t n_units, int q, float s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (size_t ub = blockIdx.x; ub < n_units / 8; ub += gridDim.x) {
    size_t unit = ub * 8 + warp;
    size_t g = unit;
    // insert 4 zero bits at q, q+1, q+2, q+3 (one run of group bits)
    g = ((g >> q) << (q + 4)) | (g & ((1ull << q) - 1));
    float4 v[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] = __ldcs(a + ((g | ((size_t)c << q)) << 5) + lane);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      v[c].x *= s; v[c].y *= s; v[c].z *= s; v[c].w *= s;
      __stcs(a + ((g | ((size_t)c << q)) << 5) + lane, v[c]);
    }
  }
}

int main() {
  const size_t bytes = 2ull << 30, n = bytes / 16;
  float4 *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 0, bytes);
  cudaMemset(b, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto f) {
    f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      f();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); exit(1); }
    printf("%-28s %8.3f ms  %7.1f GB/s (read+write)\n", name, best, 2.0 * bytes / best / 1e6);
  };
  run("copy grid=4096x256", [&] { copy_k<<<4096, 256>>>(a, b, n); });
  run("copy grid=sms*8x256", [&] { copy_k<<<sms * 8, 256>>>(a, b, n); });
  run("rmw1 grid=sms*8x256", [&] { rmw1_k<<<sms * 8, 256>>>(a, n, 1.0f); });
  run("rmw1 grid=n/256", [&] { rmw1_k<<<(unsigned)(n / 256), 256>>>(a, n, 1.0f); });
  run("rmw4 grid=sms*4x256", [&] { rmwU_k<4><<<sms * 4, 256>>>(a, n, 1.0f); });
  run("rmw8 grid=sms*2x256", [&] { rmwU_k<8><<<sms * 2, 256>>>(a, n, 1.0f); });
  run("rmw16 grid=sms*2x256", [&] { rmwU_k<16><<<sms * 2, 256>>>(a, n, 1.0f); });
  const size_t units = n / 512;  // 16 segments x 32 float4
  for (int k : {1, 2, 4, 8, 16, 32}) {
    char nm[64];
    snprintf(nm, sizeof nm, "seg16 q=8 iters=%d", k);
    run(nm, [&] { seg16_k<2><<<(unsigned)(units / 8 / k), 256>>>(a, units, 8, 1.0f); });
  }
  for (int q : {0, 8, 14}) {
    char nm[64];
    snprintf(nm, sizeof nm, "seg16 q=%d 2cta", q);
    run(nm, [&] { seg16_k<2><<<sms * 2, 256>>>(a, units, q, 1.0f); });
    snprintf(nm, sizeof nm, "seg16 q=%d 1cta", q);
    run(nm, [&] { seg16_k<1><<<sms, 256>>>(a, units, q, 1.0f); });
    snprintf(nm, sizeof nm, "seg16 q=%d many", q);
    run(nm, [&] { seg16_k<2><<<(unsigned)(units / 8), 256>>>(a, units, q, 1.0f); });
  }
  return 0;
}
