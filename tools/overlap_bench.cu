// Overlap of HBM streaming with FP32 work, for the tile engine's execution scheme (2 GiB state,
// in place, 8192-amplitude tiles of 16 KB... 64 KB): time vs synthetic FFMA2 per amplitude.
//   np   : non-persistent grid, one tile per CTA (8 warps, 32 amps/thread), LDG -> FMA -> STG
//   tma  : persistent, 1 CTA/SM, tile k+1 bulk-copied (cp.async.bulk) into smem while tile k computes
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ob tools/overlap_bench.cu && /tmp/ob
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 r) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a; }
__device__ __forceinline__ float hi(u64 r) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return b; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

template <int K>
__device__ __forceinline__ void work(u64 (&x)[32], u64 c) {
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int p = 0; p < 32; ++p) x[p] = fma2(x[p], c, x[(p + 1) & 31]);
}

// tile = 16 segments x 8 warps? Here: tile of 8192 amps = 64 KB contiguous; warp w, lane l, reg p
// -> float4 index (w * 16 + p/2) * 32 + l (coalesced 512 B per warp instruction)
template <int K>
__global__ void __launch_bounds__(256, 2) np_k(float4* __restrict__ a, u64 c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4* t = a + (size_t)blockIdx.x * 4096;
  u64 x[32];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const float4 v = __ldcs(t + (warp * 16 + q) * 32 + lane);
    x[2 * q] = pk(v.x, v.y);
    x[2 * q + 1] = pk(v.z, v.w);
  }
  work<K>(x, c);
#pragma unroll
  for (int q = 0; q < 16; ++q)
    __stcs(t + (warp * 16 + q) * 32 + lane, make_float4(lo(x[2 * q]), hi(x[2 * q]), lo(x[2 * q + 1]), hi(x[2 * q + 1])));
}

// same tile, but the warp bits are segment slots t3..t5 (64 B sub-rows) and lane bits 2..4 are
// group bits: every warp instruction reads 8 chunks of 64 B (the 8 warps of the CTA together cover
// whole 512 B rows) -- lets phase changes keep the warp bits when slots 3..5 are untouched
template <int K>
__global__ void __launch_bounds__(256, 2) np64_k(float4* __restrict__ a, u64 c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4* t = a + (size_t)blockIdx.x * 4096;
  // tile float4 index: row r (16 rows of 32 float4 = 512 B), within row: (warp << 2) | (lane & 3)
  // rows: lane bits 2..4 (3 bits) + register bits (q: 1 bit... 16 loads: q bits 0..3 -> rows)
  u64 x[32];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int row = ((lane >> 2) + (q << 3)) & 127;  // 128 rows in the 64 KB tile
    const float4 v = __ldcs(t + row * 32 + (warp << 2) + (lane & 3));
    x[2 * q] = pk(v.x, v.y);
    x[2 * q + 1] = pk(v.z, v.w);
  }
  work<K>(x, c);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int row = ((lane >> 2) + (q << 3)) & 127;
    __stcs(t + row * 32 + (warp << 2) + (lane & 3), make_float4(lo(x[2 * q]), hi(x[2 * q]), lo(x[2 * q + 1]), hi(x[2 * q + 1])));
  }
}

__device__ __forceinline__ void mbar_init(unsigned a, unsigned n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned a, unsigned tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(tx) : "memory"); }
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned par) {
  unsigned done;
  do { asm volatile("{ .reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2; selp.b32 %0, 1, 0, P1; }" : "=r"(done) : "r"(a), "r"(par) : "memory"); } while (!done);
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}

// persistent, 1 CTA/SM, 2 smem stages of one tile (64 KB each); thread 0 issues 4 x 16 KB bulk copies
template <int K>
__global__ void __launch_bounds__(256, 1) tma_k(float4* __restrict__ a, u64 c, int ntiles) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long mb[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned sm_s = (unsigned)__cvta_generic_to_shared(sm), mb_s = (unsigned)__cvta_generic_to_shared(mb);
  if (threadIdx.x == 0) {
    mbar_init(mb_s, 1);
    mbar_init(mb_s + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int tile, int s) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(mb_s + 8 * s, 65536u);
      for (int j = 0; j < 4; ++j)
        bulk_g2s(sm_s + s * 65536 + j * 16384, (const char*)(a + (size_t)tile * 4096) + j * 16384, 16384u, mb_s + 8 * s);
    }
  };
  int k = 0;
  if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int s = k & 1;
    const int nxt = tile + gridDim.x;
    mbar_wait(mb_s + 8 * s, (k >> 1) & 1);
    const float4* st = reinterpret_cast<const float4*>(sm + s * 65536);
    u64 x[32];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const float4 v = st[(warp * 16 + q) * 32 + lane];
      x[2 * q] = pk(v.x, v.y);
      x[2 * q + 1] = pk(v.z, v.w);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // everyone done reading stage s^1's previous content? (stage s read done)
    if (nxt < ntiles) issue(nxt, s ^ 1);  // next tile into the other stage
    work<K>(x, c);
    float4* t = a + (size_t)tile * 4096;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      __stcs(t + (warp * 16 + q) * 32 + lane, make_float4(lo(x[2 * q]), hi(x[2 * q]), lo(x[2 * q + 1]), hi(x[2 * q + 1])));
  }
}

// np with T CTA-wide shared-memory transposes of the tile (write 16 B / amplitude pair, barrier,
// read back in another order, barrier), as the tile engine's phase changes do
template <int K, int T, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) npt_k(float4* __restrict__ a, u64 c) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4* t = a + (size_t)blockIdx.x * 4096;
  u64 x[32];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const float4 v = __ldcs(t + (warp * 16 + q) * 32 + lane);
    x[2 * q] = pk(v.x, v.y);
    x[2 * q + 1] = pk(v.z, v.w);
  }
  float4* s4 = reinterpret_cast<float4*>(sm);
#pragma unroll
  for (int r = 0; r < T; ++r) {
    work<K / (T + 1)>(x, c);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int u = (warp * 16 + q) * 32 + lane;
      s4[u] = make_float4(lo(x[2 * q]), hi(x[2 * q]), lo(x[2 * q + 1]), hi(x[2 * q + 1]));
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int u = (q * 8 + warp) * 32 + lane;  // rows exchanged across warps, lanes contiguous (conflict-free)
      const float4 v = s4[u];
      x[2 * q] = pk(v.x, v.y);
      x[2 * q + 1] = pk(v.z, v.w);
    }
    __syncthreads();
  }
  work<K - T * (K / (T + 1))>(x, c);
#pragma unroll
  for (int q = 0; q < 16; ++q)
    __stcs(t + (warp * 16 + q) * 32 + lane, make_float4(lo(x[2 * q]), hi(x[2 * q]), lo(x[2 * q + 1]), hi(x[2 * q + 1])));
}

template <int K, int T>
__global__ void __launch_bounds__(256, 1) tmat_k(float4* __restrict__ a, u64 c, int ntiles) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long mb[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned sm_s = (unsigned)__cvta_generic_to_shared(sm), mb_s = (unsigned)__cvta_generic_to_shared(mb);
  if (threadIdx.x == 0) {
    mbar_init(mb_s, 1);
    mbar_init(mb_s + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int tile, int s) {
    if (threadIdx.x == 0) mbar_expect_tx(mb_s + 8 * s, 65536u);
    __syncwarp();
    if (threadIdx.x < 32)  // 32 lanes x 2 KB
      bulk_g2s(sm_s + s * 65536 + threadIdx.x * 2048, (const char*)(a + (size_t)tile * 4096) + threadIdx.x * 2048, 2048u,
               mb_s + 8 * s);
  };
  int k = 0;
  if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int s = k & 1;
    const int nxt = tile + gridDim.x;
    if (nxt < ntiles) issue(nxt, s ^ 1);  // other buffer: freed by the barrier that ended tile k-1
    mbar_wait(mb_s + 8 * s, (k >> 1) & 1);
    float4* st = reinterpret_cast<float4*>(sm + s * 65536);
    u64 x[32];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const float4 v = st[(warp * 16 + q) * 32 + lane];
      x[2 * q] = pk(v.x, v.y);
      x[2 * q + 1] = pk(v.z, v.w);
    }
#pragma unroll
    for (int r = 0; r < T; ++r) {
      work<K / (T + 1)>(x, c);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int u = (warp * 16 + q) * 32 + lane;
        st[u] = make_float4(lo(x[2 * q]), hi(x[2 * q]), lo(x[2 * q + 1]), hi(x[2 * q + 1]));
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int u = (q * 8 + warp) * 32 + lane;
        const float4 v = st[u];
        x[2 * q] = pk(v.x, v.y);
        x[2 * q + 1] = pk(v.z, v.w);
      }
    }
    work<K - T * (K / (T + 1))>(x, c);
    float4* t = a + (size_t)tile * 4096;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      __stcs(t + (warp * 16 + q) * 32 + lane, make_float4(lo(x[2 * q]), hi(x[2 * q]), lo(x[2 * q + 1]), hi(x[2 * q + 1])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // buffer s free for the prefetch issued in iteration k + 1
  }
}

int main() {
  const size_t bytes = 2ull << 30, n4 = bytes / 16;
  const int ntiles = (int)(n4 / 4096);
  float4* a;
  cudaMalloc(&a, bytes);
  cudaMemset(a, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const u64 c = 0x3f8000003f800000ull;
  auto run = [&](const char* name, int K, auto f) {
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
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); exit(1); }
    const double fp_ms = (double)K * 2.0 * (bytes / 8) / (148.0 * 128 * 1.9e9) * 1e3;  // FFMA2 = 2 lane-ops
    printf("%-16s K=%3d FFMA2/amp  %7.3f ms  (%6.1f GB/s; FP-only floor %.3f ms)\n", name, K, best, 2.0 * bytes / best / 1e6, fp_ms);
  };
#define BOTH(K)                                                                                  \
  run("np", K, [&] { np_k<K><<<ntiles, 256>>>(a, c); });                                        \
  cudaFuncSetAttribute(tma_k<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);       \
  run("tma", K, [&] { tma_k<K><<<sms, 256, 2 * 65536>>>(a, c, ntiles); });
  // the tile engine's configuration: 2 CTAs/SM (75 KB shared each), carveout 67 % (L1 ~92 KB)
#define NPC(K)                                                                                    \
  cudaFuncSetAttribute(np_k<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 75 * 1024);          \
  cudaFuncSetAttribute(np_k<K>, cudaFuncAttributePreferredSharedMemoryCarveout, 67);              \
  run("np75/c67", K, [&] { np_k<K><<<ntiles, 256, 75 * 1024>>>(a, c); });

#define NP64(K)                                                                                   \
  cudaFuncSetAttribute(np64_k<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 75 * 1024);        \
  cudaFuncSetAttribute(np64_k<K>, cudaFuncAttributePreferredSharedMemoryCarveout, 67);            \
  run("np64B/c67", K, [&] { np64_k<K><<<ntiles, 256, 75 * 1024>>>(a, c); });

#define TR(K, T)                                                                                   \
  cudaFuncSetAttribute(npt_k<K, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4608 * 16);        \
  cudaFuncSetAttribute(npt_k<K, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 67);            \
  run("np+T" #T "/2cta", K, [&] { npt_k<K, T><<<ntiles, 256, 4608 * 16>>>(a, c); });
#define TR3(K, T)                                                                                  \
  cudaFuncSetAttribute(npt_k<K, T, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);         \
  cudaFuncSetAttribute(npt_k<K, T, 3>, cudaFuncAttributePreferredSharedMemoryCarveout, 86);         \
  { int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, npt_k<K, T, 3>, 256, 65536);      \
    printf("npt<3> occupancy %d\n", nb); }                                                           \
  run("np+T" #T "/3cta", K, [&] { npt_k<K, T, 3><<<ntiles, 256, 65536>>>(a, c); });
  TR(28, 1) TR3(28, 1) TR(48, 4) TR3(48, 4) TR(88, 4) TR3(88, 4) TR(28, 4) TR3(28, 4)
#define TT(K, T)                                                                                   \
  cudaFuncSetAttribute(tmat_k<K, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);       \
  run("tma+T" #T, K, [&] { tmat_k<K, T><<<sms, 256, 2 * 65536>>>(a, c, ntiles); });

  return 0;
}
