// sm_100a kernels of the OWQS/EOWQS array executor.
//
// State layout in HBM: 2^w complex amplitudes, interleaved (re, im); slot k = bit k of the index.
// Warp segment: a warp moves one 512-byte contiguous segment per vector load (complex64: float4 =
// 2 amplitudes per lane, 64 amplitudes, slot 0 inside the vector and slots 1..5 on lane bits;
// complex128: double2 = 1 amplitude per lane, slots 0..4 on lane bits). Slots above the segment
// that a pass touches non-diagonally ("group slots", <= KMAX_HI) are held in registers: every
// thread owns the 2^KHI segments that differ in those bits, so every op of the pass is local to
// a thread (high slots) or a warp (shuffles), and the pass is one coalesced read + one write.
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>

#include "owqs_internal.h"
#include "device_common.cuh"

namespace owqs {

template <typename T> struct VT;
template <> struct VT<float> {
  typedef float4 V;
  typedef float2 C;
  static constexpr int SB = 6;
  static constexpr int EPV = 2;
};
template <> struct VT<double> {
  typedef double2 V;
  typedef double2 C;
  static constexpr int SB = 5;
  static constexpr int EPV = 1;
};

template <typename T> __device__ __forceinline__ typename VT<T>::C make_c(T r, T i);
template <> __device__ __forceinline__ float2 make_c<float>(float r, float i) { return make_float2(r, i); }
template <> __device__ __forceinline__ double2 make_c<double>(double r, double i) { return make_double2(r, i); }

template <typename T>
__device__ __forceinline__ void vload(const typename VT<T>::V* p, T (&re)[2], T (&im)[2]);
template <>
__device__ __forceinline__ void vload<float>(const float4* p, float (&re)[2], float (&im)[2]) {
  float4 v = __ldcs(p);
  re[0] = v.x; im[0] = v.y; re[1] = v.z; im[1] = v.w;
}
template <>
__device__ __forceinline__ void vload<double>(const double2* p, double (&re)[2], double (&im)[2]) {
  double2 v = __ldcs(p);
  re[0] = v.x; im[0] = v.y; re[1] = 0; im[1] = 0;
}
template <typename T>
__device__ __forceinline__ void vstore(typename VT<T>::V* p, const T (&re)[2], const T (&im)[2]);
template <>
__device__ __forceinline__ void vstore<float>(float4* p, const float (&re)[2], const float (&im)[2]) {
  __stcs(p, make_float4(re[0], im[0], re[1], im[1]));
}
template <>
__device__ __forceinline__ void vstore<double>(double2* p, const double (&re)[2], const double (&im)[2]) {
  __stcs(p, make_double2(re[0], im[0]));
}

// ------------------------------------------------------------------------------------------------
// The fused pass kernel.
// ------------------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void cmul_add(T ar, T ai, T xr, T xi, T br, T bi, T yr, T yi, T& outr, T& outi) {
  // out = a*x + b*y
  outr = ar * xr - ai * xi + br * yr - bi * yi;
  outi = ar * xi + ai * xr + br * yi + bi * yr;
}

// Bit mask over a thread's NV*EPV amplitudes (position v*EPV + e, v = u*G + c) of those whose
// index has slot x set: element bit (complex64 slot 0), lane bit, group bit j of c, or a bit of
// the group base gb[u].
template <int NV, int EPV, int G>
struct PosMasks {
  __host__ __device__ static constexpr uint32_t full() { return NV * EPV >= 32 ? 0xffffffffu : ((1u << (NV * EPV)) - 1u); }
  __host__ __device__ static constexpr uint32_t elem1() {
    uint32_t m = 0;
    for (int p = 0; p < NV * EPV; ++p)
      if (p % EPV == 1) m |= 1u << p;
    return m;
  }
  __host__ __device__ static constexpr uint32_t group(int j) {
    uint32_t m = 0;
    for (int p = 0; p < NV * EPV; ++p)
      if ((((p / EPV) % G) >> j) & 1) m |= 1u << p;
    return m;
  }
  __host__ __device__ static constexpr uint32_t block(int u) {
    uint32_t m = 0;
    for (int p = 0; p < NV * EPV; ++p)
      if (p / EPV / G == u) m |= 1u << p;
    return m;
  }
};

template <typename T, int KHI, int UNR>
__device__ __forceinline__ uint32_t slot_mask(int x, int lane, const uint64_t (&gb)[UNR], const int (&q)[KHI > 0 ? KHI : 1]) {
  constexpr int SB = VT<T>::SB, EPV = VT<T>::EPV, G = 1 << KHI, NV = UNR * G;
  typedef PosMasks<NV, EPV, G> PM;
  if (EPV == 2 && x == 0) return PM::elem1();
  if (x < SB) return ((lane >> (x - (EPV == 2 ? 1 : 0))) & 1) ? PM::full() : 0u;
#pragma unroll
  for (int j = 0; j < KHI; ++j)
    if (q[j] == x - SB) return PM::group(j);
  uint32_t m = 0;
#pragma unroll
  for (int u = 0; u < UNR; ++u)
    if ((gb[u] >> (x - SB)) & 1) m |= PM::block(u);
  return m;
}

template <typename T, int KHI, int UNR>
__device__ __forceinline__ uint32_t slot_mask_p(int x, int lane, const uint64_t (&gb)[UNR], const StepDesc& d,
                                                uint32_t rank) {
  constexpr int SB = VT<T>::SB, EPV = VT<T>::EPV, G = 1 << KHI, NV = UNR * G;
  typedef PosMasks<NV, EPV, G> PM;
  if (x >= d.width) return ((rank >> (x - d.width)) & 1) ? PM::full() : 0u;  // rank bit (sharded)
  if (EPV == 2 && x == 0) return PM::elem1();
  if (x < SB) return ((lane >> (x - (EPV == 2 ? 1 : 0))) & 1) ? PM::full() : 0u;
  uint32_t m = 0;
  bool grp = false;
#pragma unroll
  for (int j = 0; j < KHI; ++j)
    if (d.bhi[j] == x) {
      m = PM::group(j);
      grp = true;
    }
  if (grp) return m;
#pragma unroll
  for (int u = 0; u < UNR; ++u)
    if ((gb[u] >> (x - SB)) & 1) m |= PM::block(u);
  return m;
}

// Opaque dependency: makes `lm` depend on `x`, so later shuffles (which use lm) cannot be hoisted
// above the work that produced x (bounds the registers a cross-lane op keeps in flight).
template <typename T> __device__ __forceinline__ void chain(int& lm, T x);
template <> __device__ __forceinline__ void chain<float>(int& lm, float x) {
  asm volatile("{ .reg .f32 t; mov.f32 t, %1; }" : "+r"(lm) : "f"(x));
}
template <> __device__ __forceinline__ void chain<double>(int& lm, double x) {
  asm volatile("{ .reg .f64 t; mov.f64 t, %1; }" : "+r"(lm) : "d"(x));
}

template <int KHI, int MINB> struct PassBounds {
  static constexpr int min_blocks = MINB > 0 ? MINB : (KHI <= 3 ? 3 : 2);
};

// Sign flips accumulated in `neg` (bit v*EPV+e) applied branch-free through the sign bit.
template <typename T> __device__ __forceinline__ T flip_sign(T x, uint32_t f);
template <> __device__ __forceinline__ float flip_sign<float>(float x, uint32_t f) {
  return __int_as_float(__float_as_int(x) ^ (f << 31));
}
template <> __device__ __forceinline__ double flip_sign<double>(double x, uint32_t f) {
  return __longlong_as_double(__double_as_longlong(x) ^ ((unsigned long long)f << 63));
}

// ---- in-place register kernels of the pass (inline PTX pins each amplitude to one register,
// so the runtime op dispatch does not force register shuffling at its merge points) ----
// structured butterfly: x0 <- x0 + a x1, x1 <- x0 - a x1
__device__ __forceinline__ void bfly_ip(float& x0r, float& x0i, float& x1r, float& x1i, float ar, float ai, float nai) {
  asm("{\n\t.reg .f32 tr, ti;\n\t"
      "mul.f32 tr, %4, %2;\n\t"
      "fma.rn.f32 tr, %6, %3, tr;\n\t"
      "mul.f32 ti, %4, %3;\n\t"
      "fma.rn.f32 ti, %5, %2, ti;\n\t"
      "sub.f32 %2, %0, tr;\n\t"
      "sub.f32 %3, %1, ti;\n\t"
      "add.f32 %0, %0, tr;\n\t"
      "add.f32 %1, %1, ti;\n\t}"
      : "+f"(x0r), "+f"(x0i), "+f"(x1r), "+f"(x1i)
      : "f"(ar), "f"(ai), "f"(nai));
}
__device__ __forceinline__ void bfly_ip(double& x0r, double& x0i, double& x1r, double& x1i, double ar, double ai, double) {
  const double tr = ar * x1r - ai * x1i, ti = ar * x1i + ai * x1r;
  x1r = x0r - tr; x1i = x0i - ti;
  x0r = x0r + tr; x0i = x0i + ti;
}
// butterfly with the sign of a x1 flipped by bit 31 of sb (absorbed CZ)
__device__ __forceinline__ void bfly_ip_s(float& x0r, float& x0i, float& x1r, float& x1i, float ar, float ai, float nai,
                                          uint32_t sb) {
  asm("{\n\t.reg .f32 tr, ti;\n\t"
      "mul.f32 tr, %4, %2;\n\t"
      "fma.rn.f32 tr, %6, %3, tr;\n\t"
      "mul.f32 ti, %4, %3;\n\t"
      "fma.rn.f32 ti, %5, %2, ti;\n\t"
      "xor.b32 tr, tr, %7;\n\t"
      "xor.b32 ti, ti, %7;\n\t"
      "sub.f32 %2, %0, tr;\n\t"
      "sub.f32 %3, %1, ti;\n\t"
      "add.f32 %0, %0, tr;\n\t"
      "add.f32 %1, %1, ti;\n\t}"
      : "+f"(x0r), "+f"(x0i), "+f"(x1r), "+f"(x1i)
      : "f"(ar), "f"(ai), "f"(nai), "r"(sb));
}
__device__ __forceinline__ void bfly_ip_s(double& x0r, double& x0i, double& x1r, double& x1i, double ar, double ai,
                                          double, uint32_t sb) {
  double tr = ar * x1r - ai * x1i, ti = ar * x1i + ai * x1r;
  if (sb) { tr = -tr; ti = -ti; }
  x1r = x0r - tr; x1i = x0i - ti;
  x0r = x0r + tr; x0i = x0i + ti;
}
__device__ __forceinline__ void lane_bfly_ip_s(float& xr, float& xi, float cr, float ci, float nci, float s, int lm,
                                               uint32_t sb) {
  asm("{\n\t.reg .f32 yr, yi, rr, ri;\n\t"
      "mul.f32 yr, %2, %0;\n\t"
      "fma.rn.f32 yr, %4, %1, yr;\n\t"
      "mul.f32 yi, %2, %1;\n\t"
      "fma.rn.f32 yi, %3, %0, yi;\n\t"
      "xor.b32 yr, yr, %7;\n\t"
      "xor.b32 yi, yi, %7;\n\t"
      "shfl.sync.bfly.b32 rr, yr, %6, 0x1f, 0xffffffff;\n\t"
      "shfl.sync.bfly.b32 ri, yi, %6, 0x1f, 0xffffffff;\n\t"
      "fma.rn.f32 %0, %5, yr, rr;\n\t"
      "fma.rn.f32 %1, %5, yi, ri;\n\t}"
      : "+f"(xr), "+f"(xi)
      : "f"(cr), "f"(ci), "f"(nci), "f"(s), "r"(lm), "r"(sb));
}
__device__ __forceinline__ void lane_bfly_ip_s(double& xr, double& xi, double cr, double ci, double, double s, int lm,
                                               uint32_t sb) {
  double yr = cr * xr - ci * xi, yi = cr * xi + ci * xr;
  if (sb) { yr = -yr; yi = -yi; }
  const double rr = __shfl_xor_sync(FULLMASK, yr, lm), ri = __shfl_xor_sync(FULLMASK, yi, lm);
  xr = rr + s * yr;
  xi = ri + s * yi;
}
// cross-lane butterfly: y = c x, r = y of the partner lane, x <- r + s y
__device__ __forceinline__ void lane_bfly_ip(float& xr, float& xi, float cr, float ci, float nci, float s, int lm) {
  asm("{\n\t.reg .f32 yr, yi, rr, ri;\n\t"
      "mul.f32 yr, %2, %0;\n\t"
      "fma.rn.f32 yr, %4, %1, yr;\n\t"
      "mul.f32 yi, %2, %1;\n\t"
      "fma.rn.f32 yi, %3, %0, yi;\n\t"
      "shfl.sync.bfly.b32 rr, yr, %6, 0x1f, 0xffffffff;\n\t"
      "shfl.sync.bfly.b32 ri, yi, %6, 0x1f, 0xffffffff;\n\t"
      "fma.rn.f32 %0, %5, yr, rr;\n\t"
      "fma.rn.f32 %1, %5, yi, ri;\n\t}"
      : "+f"(xr), "+f"(xi)
      : "f"(cr), "f"(ci), "f"(nci), "f"(s), "r"(lm));
}
__device__ __forceinline__ void lane_bfly_ip(double& xr, double& xi, double cr, double ci, double, double s, int lm) {
  const double yr = cr * xr - ci * xi, yi = cr * xi + ci * xr;
  const double rr = __shfl_xor_sync(FULLMASK, yr, lm), ri = __shfl_xor_sync(FULLMASK, yi, lm);
  xr = rr + s * yr;
  xi = ri + s * yi;
}
// sign flip of (re, im) by bit `pos` of neg
template <int POS>
__device__ __forceinline__ void flip_ip(float& re, float& im, uint32_t neg) {
  asm("{\n\t.reg .b32 t;\n\t"
      "shl.b32 t, %2, %3;\n\t"
      "and.b32 t, t, 0x80000000;\n\t"
      "xor.b32 %0, %0, t;\n\t"
      "xor.b32 %1, %1, t;\n\t}"
      : "+f"(re), "+f"(im)
      : "r"(neg), "n"(31 - POS));
}
template <int POS>
__device__ __forceinline__ void flip_ip(double& re, double& im, uint32_t neg) {
  const uint32_t f = (neg >> POS) & 1u;
  re = flip_sign<double>(re, f);
  im = flip_sign<double>(im, f);
}
template <typename T, int NV, int EPV, int P = 0>
__device__ __forceinline__ void flush_all(T (&re)[NV][2], T (&im)[NV][2], uint32_t neg) {
  if constexpr (P < NV * EPV) {
    flip_ip<P>(re[P / EPV][P % EPV], im[P / EPV][P % EPV], neg);
    flush_all<T, NV, EPV, P + 1>(re, im, neg);
  }
}


template <typename T, int KHI, int UNR, int MINB = 0, int RED = -1>
__global__ void __launch_bounds__(256, (PassBounds<KHI, MINB>::min_blocks)) pass_kernel(const StepDesc d, const DevPtrs p) {
  // RED >= 0: the step's reduction kind fixed at compile time (fewer live fp64 accumulators)
  const int red_kind = RED >= 0 ? RED : d.red_kind;
  typedef typename VT<T>::V V;
  constexpr int SB = VT<T>::SB, EPV = VT<T>::EPV;
  constexpr int G = 1 << KHI;
  constexpr int NV = UNR * G;
  __shared__ PassShared sh;
  __shared__ T s_a[MAX_BFLY][2];
  pass_prologue(d, p, sh);
  if (threadIdx.x < MAX_BFLY) {
    s_a[threadIdx.x][0] = (T)sh.ka[threadIdx.x][0];
    s_a[threadIdx.x][1] = (T)sh.ka[threadIdx.x][1];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // the loop condition depends on blockIdx only, so the compiler sees converged warps at the
  // shuffles (launch: 256 threads, n_units a multiple of 8)
  const uint64_t n_blk_units = ((1ull << (d.width - SB - KHI)) / UNR) >> 3;
  V* st = reinterpret_cast<V*>(p.state);
  double acc[4] = {0, 0, 0, 0};
  const T pass_scale = (T)sh.scale;

  for (uint64_t ub = blockIdx.x; ub < n_blk_units; ub += gridDim.x) {
    const uint64_t unit = ub * 8 + warp;
    // group base: the unit's group index with zeros inserted at the group slots (ascending)
    uint64_t gb[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      uint64_t g = unit * UNR + u;
#pragma unroll
      for (int j = 0; j < KHI; ++j) {
        const int qj = d.bhi[j] - SB;
        g = ((g >> qj) << (qj + 1)) | (g & ((1ull << qj) - 1));
      }
      gb[u] = g;
    }
    T re[NV][2], im[NV][2];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int c = 0; c < G; ++c) {
        uint64_t s = gb[u];
#pragma unroll
        for (int j = 0; j < KHI; ++j)
          if ((c >> j) & 1) s |= 1ull << (d.bhi[j] - SB);
        vload<T>(st + s * 32 + lane, re[u * G + c], im[u * G + c]);
      }

    uint32_t neg = 0;
    for (int i = 0; i < d.n_ops; ++i) {
      const int type = d.ops[i].type;
      const int a = d.ops[i].a;
      if (type == OP_DIAG_E || type == OP_DIAG_Z) {
        uint32_t m = slot_mask_p<T, KHI, UNR>(a, lane, gb, d, p.rank);
        if (type == OP_DIAG_E) m &= slot_mask_p<T, KHI, UNR>(d.ops[i].b, lane, gb, d, p.rank);
        neg ^= sh.cond[i] ? m : 0u;
        continue;
      }
      if (type == OP_FLUSH) {  // placed by the compiler where a pending diagonal must apply
        flush_all<T, NV, EPV>(re, im, neg);
        neg = 0;
        continue;
      }
      if (type == OP_X) {
        if (!__all_sync(FULLMASK, sh.cond[i] != 0)) continue;
        if (a >= SB) {
#pragma unroll
          for (int jj = 0; jj < KHI; ++jj) {
            if (d.bhi[jj] != a) continue;
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
              for (int c = 0; c < G; ++c) {
                if ((c >> jj) & 1) continue;
                const int v0 = u * G + c, v1 = v0 + (1 << jj);
#pragma unroll
                for (int e = 0; e < EPV; ++e) {
                  T tr = re[v0][e], ti = im[v0][e];
                  re[v0][e] = re[v1][e]; im[v0][e] = im[v1][e];
                  re[v1][e] = tr; im[v1][e] = ti;
                }
              }
          }
        } else if (EPV == 2 && a == 0) {
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            T tr = re[v][0], ti = im[v][0];
            re[v][0] = re[v][1]; im[v][0] = im[v][1];
            re[v][1] = tr; im[v][1] = ti;
          }
        } else {
          int lm = 1 << (a - (EPV == 2 ? 1 : 0));
#pragma unroll
          for (int v = 0; v < NV; ++v) {
#pragma unroll
            for (int e = 0; e < EPV; ++e) {
              re[v][e] = __shfl_xor_sync(FULLMASK, re[v][e], lm);
              im[v][e] = __shfl_xor_sync(FULLMASK, im[v][e], lm);
            }
            if ((v & 3) == 3) chain(lm, re[v][0]);
          }
        }
        continue;
      }
      // structured butterfly: out0 = x0 + a x1, out1 = x0 - a x1 (k folded into the pass scale)
      const int bi = sh.bidx[i];
      T ar = s_a[bi][0], ai = s_a[bi][1];
      const uint64_t am = d.absorb[bi];
      constexpr uint64_t LANE_SLOTS = EPV == 2 ? 0x3Eull : 0x1Full;
      if (am & ~LANE_SLOTS) {
        // absorbed CZ signs depend on group / element / base bits: a sign bit per pair
        uint32_t M = 0;
        for (uint64_t r = am; r; r &= r - 1) M ^= slot_mask_p<T, KHI, UNR>(__ffsll((long long)r) - 1, lane, gb, d, p.rank);
        const T nai = -ai;
        if (a >= SB) {
#pragma unroll
          for (int jj = 0; jj < KHI; ++jj) {
            if (d.bhi[jj] != a) continue;
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
              for (int c = 0; c < G; ++c) {
                if ((c >> jj) & 1) continue;
                const int v0 = u * G + c, v1 = v0 + (1 << jj);
#pragma unroll
                for (int e = 0; e < EPV; ++e)
                  bfly_ip_s(re[v0][e], im[v0][e], re[v1][e], im[v1][e], ar, ai, nai, (M >> (v0 * EPV + e)) << 31);
              }
          }
        } else if (EPV == 2 && a == 0) {
#pragma unroll
          for (int v = 0; v < NV; ++v)
            bfly_ip_s(re[v][0], im[v][0], re[v][1], im[v][1], ar, ai, nai, (M >> (v * EPV)) << 31);
        } else {
          const int lb = a - (EPV == 2 ? 1 : 0);
          const bool hi = (lane >> lb) & 1;
          const T cr = hi ? ar : (T)1, ci = hi ? ai : (T)0, nci = -ci;
          const T sg = hi ? (T)-1 : (T)1;
          const uint32_t Mh = hi ? M : 0u;
          const int lm = 1 << lb;
#pragma unroll
          for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int e = 0; e < EPV; ++e)
              lane_bfly_ip_s(re[v][e], im[v][e], cr, ci, nci, sg, lm, (Mh >> (v * EPV + e)) << 31);
        }
        continue;
      }
      if (am) {  // signs from lane bits only: one sign per thread, folded into the coefficient
        const uint32_t lbits = (uint32_t)(EPV == 2 ? (am >> 1) : am) & 31u;
        if (__popc((uint32_t)lane & lbits) & 1) {
          ar = -ar;
          ai = -ai;
        }
      }
      const T nai = -ai;
      if (a >= SB) {
#pragma unroll
        for (int jj = 0; jj < KHI; ++jj) {
          if (d.bhi[jj] != a) continue;
#pragma unroll
          for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int c = 0; c < G; ++c) {
              if ((c >> jj) & 1) continue;
              const int v0 = u * G + c, v1 = v0 + (1 << jj);
#pragma unroll
              for (int e = 0; e < EPV; ++e) bfly_ip(re[v0][e], im[v0][e], re[v1][e], im[v1][e], ar, ai, nai);
            }
        }
      } else if (EPV == 2 && a == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) bfly_ip(re[v][0], im[v][0], re[v][1], im[v][1], ar, ai, nai);
      } else {
        // pair across lanes. Each lane sends y = c x (c = 1 on the lower lane, a on the upper);
        // lower: out = x0 + (a x1 received); upper: out = (x0 received) - a x1 = r - y.
        const int lb = a - (EPV == 2 ? 1 : 0);
        const bool hi = (lane >> lb) & 1;
        const T cr = hi ? ar : (T)1, ci = hi ? ai : (T)0, nci = -ci;
        const T sg = hi ? (T)-1 : (T)1;
        const int lm = 1 << lb;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int e = 0; e < EPV; ++e) lane_bfly_ip(re[v][e], im[v][e], cr, ci, nci, sg, lm);
      }
    }

    if (pass_scale != (T)1) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          re[v][e] *= pass_scale;
          im[v][e] *= pass_scale;
        }
    }

    // reductions of the pass output: per-vector partials in T, accumulated in fp64
    if (red_kind == RED_NORM) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        T n = 0;
#pragma unroll
        for (int e = 0; e < EPV; ++e) n += re[v][e] * re[v][e] + im[v][e] * im[v][e];
        acc[0] += (double)n;
      }
    } else if (red_kind == RED_RHO) {
      const int r = d.red_slot;
      const uint32_t mr1 = slot_mask_p<T, KHI, UNR>(r, lane, gb, d, p.rank);
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          T n = re[v][e] * re[v][e] + im[v][e] * im[v][e];
          if ((mr1 >> (v * EPV + e)) & 1u) acc[1] += (double)n; else acc[0] += (double)n;
        }
      // c = sum conj(x0) x1 over pairs split on slot r
      if (r >= SB) {
#pragma unroll
        for (int jj = 0; jj < KHI; ++jj) {
          if (d.bhi[jj] != r) continue;
#pragma unroll
          for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int c = 0; c < G; ++c) {
              if ((c >> jj) & 1) continue;
              const int v0 = u * G + c, v1 = v0 + (1 << jj);
              T cr = 0, ci = 0;
#pragma unroll
              for (int e = 0; e < EPV; ++e) {
                cr += re[v0][e] * re[v1][e] + im[v0][e] * im[v1][e];
                ci += re[v0][e] * im[v1][e] - im[v0][e] * re[v1][e];
              }
              acc[2] += (double)cr;
              acc[3] += (double)ci;
            }
        }
      } else if (EPV == 2 && r == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          T cr = re[v][0] * re[v][1] + im[v][0] * im[v][1];
          T ci = re[v][0] * im[v][1] - im[v][0] * re[v][1];
          acc[2] += (double)cr;
          acc[3] += (double)ci;
        }
      } else {
        const int lb = r - (EPV == 2 ? 1 : 0);
        const bool hi = (lane >> lb) & 1;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          T cr = 0, ci = 0;
#pragma unroll
          for (int e = 0; e < EPV; ++e) {
            T pr = __shfl_xor_sync(FULLMASK, re[v][e], 1 << lb);
            T pi = __shfl_xor_sync(FULLMASK, im[v][e], 1 << lb);
            cr += re[v][e] * pr + im[v][e] * pi;
            ci += re[v][e] * pi - im[v][e] * pr;
          }
          if (!hi) {
            acc[2] += (double)cr;
            acc[3] += (double)ci;
          }
        }
      }
    }

    if (d.n_ops > 0) {
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int c = 0; c < G; ++c) {
          uint64_t s = gb[u];
#pragma unroll
          for (int j = 0; j < KHI; ++j)
            if ((c >> j) & 1) s |= 1ull << (d.bhi[j] - SB);
          vstore<T>(st + s * 32 + lane, re[u * G + c], im[u * G + c]);
        }
    }
  }
  if (red_kind == RED_NORM) reduce_finish<1>(acc, p, sh);
  else if (red_kind == RED_RHO) reduce_finish<4>(acc, p, sh);
}

// ------------------------------------------------------------------------------------------------
// Small-width pass (w <= 12): one CTA, whole state in shared memory, ops applied in sequence.
// ------------------------------------------------------------------------------------------------
struct PermTab {
  int8_t slot[64];
};

// ops of a pass on a state held in shared memory (general 2x2 coefficients, absorbed CZ signs)
template <typename T>
__device__ void smem_apply_ops(const StepDesc& d, const DevPtrs& p, typename VT<T>::C* s, const PassShared& sh) {
  const int n = 1 << d.width;
  for (int k = 0; k < d.n_ops; ++k) {
    const Op op = d.ops[k];
    if (!sh.cond[k] || op.type == OP_FLUSH) continue;
    if (op.type == OP_DIAG_E || op.type == OP_DIAG_Z) {
      const int a = op.a, b = op.type == OP_DIAG_E ? op.b : op.a;
      const uint64_t rk = (uint64_t)p.rank << d.width;  // rank bits above the shard (sharded runs)
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        if ((((uint64_t)i | rk) >> a) & (((uint64_t)i | rk) >> b) & 1) {
          s[i].x = -s[i].x;
          s[i].y = -s[i].y;
        }
    } else {
      const int a = op.a;
      double cf[8];
      if (op.type == OP_BFLY) {
        for (int j = 0; j < 8; ++j) cf[j] = sh.coef[sh.bidx[k]][j];
      } else {
        double x[8] = {0, 0, 1, 0, 1, 0, 0, 0};
        for (int j = 0; j < 8; ++j) cf[j] = x[j];
      }
      const uint64_t am = op.type == OP_BFLY ? d.absorb[sh.bidx[k]] : 0ull;
      const uint64_t rk = (uint64_t)p.rank << d.width;
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        int i0 = ((i >> a) << (a + 1)) | (i & ((1 << a) - 1));
        int i1 = i0 | (1 << a);
        T x0r = s[i0].x, x0i = s[i0].y, x1r = s[i1].x, x1i = s[i1].y;
        if (__popcll(((uint64_t)i1 | rk) & am) & 1) {  // absorbed CZ: x1 sign by the other slots' bits
          x1r = -x1r;
          x1i = -x1i;
        }
        T o0r, o0i, o1r, o1i;
        cmul_add<T>((T)cf[0], (T)cf[1], x0r, x0i, (T)cf[2], (T)cf[3], x1r, x1i, o0r, o0i);
        cmul_add<T>((T)cf[4], (T)cf[5], x0r, x0i, (T)cf[6], (T)cf[7], x1r, x1i, o1r, o1i);
        s[i0].x = o0r; s[i0].y = o0i; s[i1].x = o1r; s[i1].y = o1i;
      }
    }
    __syncthreads();
  }
}

// per-thread partials of the step's reduction over a shared-memory state
template <typename T>
__device__ void smem_reduce(int red_kind, int r, int width, const typename VT<T>::C* s, double (&acc)[4]) {
  const int n = 1 << width;
  if (red_kind == RED_NORM) {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      acc[0] += (double)s[i].x * s[i].x + (double)s[i].y * s[i].y;
  } else if (red_kind == RED_RHO) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double nn = (double)s[i].x * s[i].x + (double)s[i].y * s[i].y;
      if ((i >> r) & 1) {
        acc[1] += nn;
      } else {
        acc[0] += nn;
        int j = i | (1 << r);
        double x0r = s[i].x, x0i = s[i].y, x1r = s[j].x, x1i = s[j].y;
        acc[2] += x0r * x1r + x0i * x1i;
        acc[3] += x0r * x1i - x0i * x1r;
      }
    }
  }
}

// block-level sum of 4 doubles into out[4] (shared), fixed order
__device__ void block_sum4(double (&acc)[4], PassShared& sh, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(FULLMASK, acc[k], o);
  __syncthreads();
  if (lane == 0)
    for (int k = 0; k < 4; ++k) sh.red[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < 4; ++k) {
      double t = 0;
      for (int w = 0; w < nw; ++w) t += sh.red[w][k];
      out[k] = t;
    }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------------
// Small-width pass (w <= 12): one CTA, whole state in shared memory, ops applied in sequence.
// ------------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(512) small_pass_kernel(const StepDesc d, const DevPtrs p) {
  typedef typename VT<T>::C C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  __shared__ PassShared sh;
  pass_prologue(d, p, sh);
  const int n = 1 << d.width;
  C* st = reinterpret_cast<C*>(p.state);
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = st[i];
  __syncthreads();
  smem_apply_ops<T>(d, p, s, sh);
  double acc[4] = {0, 0, 0, 0};
  smem_reduce<T>(d.red_kind, d.red_slot, d.width, s, acc);
  if (d.n_ops > 0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) st[i] = s[i];
  if (d.red_kind == RED_NORM) reduce_finish<1>(acc, p, sh);
  else if (d.red_kind == RED_RHO) reduce_finish<4>(acc, p, sh);
}

// ------------------------------------------------------------------------------------------------
// Joint k-outcome measurement (PAPER §4.1 sub-state model L155-161, Fig. 6
// L374-395): k consecutive eliminations share one pass that reduces the k qubits' 2^k x 2^k
// reduced density matrix rho = Tr_rest |psi><psi| (ST_RHOK), and one pass that decides the k
// outcomes in sequence from rho -- the conditional Eq. 3 probability of each given the earlier ones,
// exactly what k single measurements see -- and applies the k projections + eliminations at once
// (ST_SHRINKK: out = (prod_j <b_j|) psi / sqrt(P), width w -> w - k). Traffic S + (S + S/2^k)
// instead of k (S + 1.5 S / 2^(j-1)) halving passes.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t pdep_pos(uint64_t v, const int32_t* pos, int n) {
  uint64_t r = 0;
  for (int j = 0; j < n; ++j) r |= ((v >> j) & 1ull) << pos[j];
  return r;
}

// rho[a][b] += v[a] conj(v[b]) over every rest index, upper triangle (a <= b), fp64; block partials
// then the last block sums them in a fixed order (deterministic) into partials[RHOK_RESULT_OFF ..]
template <typename T, int K>
__global__ void __launch_bounds__(256) rhok_kernel(const StepDesc d, const DevPtrs p) {
  typedef typename VT<T>::C C;
  constexpr int D = 1 << K, NV = 2 * (D * (D + 1) / 2);
  const C* st = reinterpret_cast<const C*>(p.state);
  const int w = d.width;
  // rest index r -> state index: a zero bit inserted at each measured position, ascending (O(K) per
  // element; the K measured offsets are per-thread constants)
  int hole[K];
#pragma unroll
  for (int j = 0; j < K; ++j) hole[j] = d.jm_pos[j];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = a + 1; b < K; ++b)
      if (hole[b] < hole[a]) {
        const int t = hole[a];
        hole[a] = hole[b];
        hole[b] = t;
      }
  uint64_t moff[D];
#pragma unroll
  for (int x = 0; x < D; ++x) moff[x] = pdep_pos((uint64_t)x, d.jm_pos, K);
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  const uint64_t nrest = 1ull << (w - K);
  // U rest indices per thread and iteration (a grid stride apart), all loads issued before the
  // arithmetic: U * D independent 8 / 16 B loads in flight per thread (K <= 2; K = 3 keeps U = 1:
  // its 72 fp64 accumulators already fill the register file)
  constexpr int U = K <= 2 ? 4 : 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r0 < nrest; r0 += U * stride) {
    C v[U][D];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t r = r0 + u * stride;
      uint64_t base = r < nrest ? r : r0;
#pragma unroll
      for (int j = 0; j < K; ++j) base = ((base >> hole[j]) << (hole[j] + 1)) | (base & ((1ull << hole[j]) - 1));
#pragma unroll
      for (int x = 0; x < D; ++x) v[u][x] = r < nrest ? st[base | moff[x]] : make_c<T>((T)0, (T)0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double vr[D], vi[D];
#pragma unroll
      for (int x = 0; x < D; ++x) {
        vr[x] = (double)v[u][x].x;
        vi[x] = (double)v[u][x].y;
      }
      int e = 0;
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = a; b < D; ++b) {
          acc[e++] += vr[a] * vr[b] + vi[a] * vi[b];  // Re v[a] conj(v[b])
          acc[e++] += vi[a] * vr[b] - vr[a] * vi[b];  // Im
        }
    }
  }
  __shared__ double red[8][NV];
  __shared__ int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double x = acc[v];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULLMASK, x, o);
    if (lane == 0) red[warp][v] = x;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < NV; v += blockDim.x) {
    double t = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q][v];
    p.partials[(size_t)blockIdx.x * NV + v] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&p.counter[0], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int v = threadIdx.x; v < NV; v += blockDim.x) {
    double t = 0;
    for (unsigned b = 0; b < gridDim.x; ++b) t += __ldcg(&p.partials[(size_t)b * NV + v]);
    p.partials[RHOK_RESULT_OFF + v] = t;
  }
  if (threadIdx.x == 0) p.counter[0] = 0;
}

// Decide the group's outcomes from rho in the emitter's order and build the 2^k projection
// coefficients (prod_j bra_j components / sqrt(P_joint); EOWQS: sqrt2^k scaling, outcomes 0).
// One thread. bra of outcome s: (1, (-1)^s e^{-i theta}) / sqrt2 (Eqs. 11-12; R-1).
__device__ void joint_decide(const StepDesc& d, const DevPtrs& p, bool record, double (*cv)[2], const double* rv) {
  const int K = d.jk, mode = p.run->mode;
  const double PI = 3.141592653589793238462643383279502884, R2 = 0.70710678118654752440;
  double Rr[64], Ri[64];  // current (conditioned) reduced matrix over the undecided qubits, D x D
  int D = 1 << K;
  if (mode != 2) {
    int e = 0;
    for (int a = 0; a < D; ++a)
      for (int b = a; b < D; ++b) {
        Rr[a * D + b] = rv[e];
        Ri[a * D + b] = rv[e + 1];
        Rr[b * D + a] = rv[e];
        Ri[b * D + a] = -rv[e + 1];
        e += 2;
      }
  }
  LocalOutcomes loc;
  loc.n = 0;
  double ur[JOINT_KMAX][2], ui[JOINT_KMAX][2];
  double pj = 1.0;
  for (int j = 0; j < K; ++j) {
    const MStatic ms = p.mst[d.jm[j]];
    int sg = 0, tg = 0;
    if (mode != 2) {
      sg = signal_parity(p, ms.s_off, ms.s_len, loc);
      tg = signal_parity(p, ms.t_off, ms.t_len, loc);
    }
    const double theta = (sg ? -ms.alpha : ms.alpha) + (tg ? PI : 0.0);  // Eq. 2
    double sn, cs;
    sincos(theta, &sn, &cs);
    const double er = cs, ei = -sn;  // e^{-i theta}
    int outc = 0;
    double P0 = -1.0;
    if (mode != 2) {
      // P0 = <+|R|+> summed over the other undecided qubits (qubit j is bit 0 of R's index)
      double tot = 0.0, p0 = 0.0;
      for (int a = 0; a < D; ++a) tot += Rr[a * D + a];
      for (int a2 = 0; a2 < D / 2; ++a2) {
        const int a0 = a2 << 1, a1 = a0 | 1;
        // u = (1, e^{-i theta}) / sqrt2: sum_xy u_x R_xy conj(u_y)
        const double r00 = Rr[a0 * D + a0], r11 = Rr[a1 * D + a1];
        const double r01r = Rr[a0 * D + a1], r01i = Ri[a0 * D + a1];
        // u0 R01 conj(u1) + u1 R10 conj(u0) = 2 Re(R01 conj(e^{-i theta})) / 2
        p0 += 0.5 * (r00 + r11) + (r01r * er + r01i * ei);
      }
      p0 = fmin(fmax(p0, 0.0), tot);
      P0 = tot > 0 ? p0 / tot : 0.0;
      outc = mode == 0 ? (draw_uniform(p.run->seed, ms.key) <= P0 ? 0 : 1) : (p.forced[ms.ord] & 1);
      double pS = outc ? 1.0 - P0 : P0;
      if (pS < 1e-12) {
        if (record) atomicExch(p.err, 1);
        pS = 1.0;
      }
      pj *= pS;
      // condition: R' = <b|R|b> on qubit j (bit 0), b the chosen bra
      const double s1 = outc ? -1.0 : 1.0;
      const double u1r = s1 * er, u1i = s1 * ei;  // u = (1, u1) / sqrt2
      const int D2 = D / 2;
      for (int a2 = 0; a2 < D2; ++a2)
        for (int b2 = 0; b2 < D2; ++b2) {
          const int a0 = a2 << 1, b0 = b2 << 1;
          // sum_xy u_x R[a0|x][b0|y] conj(u_y) / 2
          double sr = 0, si = 0;
          for (int x = 0; x < 2; ++x)
            for (int y = 0; y < 2; ++y) {
              const double uxr = x ? u1r : 1.0, uxi = x ? u1i : 0.0;
              const double uyr = y ? u1r : 1.0, uyi = y ? -u1i : 0.0;  // conj(u_y)
              const double rr = Rr[(a0 | x) * D + (b0 | y)], ri = Ri[(a0 | x) * D + (b0 | y)];
              const double tr = uxr * rr - uxi * ri, ti = uxr * ri + uxi * rr;
              sr += tr * uyr - ti * uyi;
              si += tr * uyi + ti * uyr;
            }
          Rr[a2 * D2 + b2] = 0.5 * sr;  // in place: (a2, b2) index <= (a0, b0) slots already read
          Ri[a2 * D2 + b2] = 0.5 * si;
        }
      D = D2;
    }
    const double s1 = outc ? -1.0 : 1.0;
    const double k = mode == 2 ? 1.0 : R2;
    ur[j][0] = k;
    ui[j][0] = 0.0;
    ur[j][1] = k * s1 * er;
    ui[j][1] = k * s1 * ei;
    if (record) {
      p.outcome[ms.ord] = (uint8_t)outc;
      p.prob0[ms.ord] = P0;
    }
    if (loc.n < MAX_BFLY) {
      loc.ord[loc.n] = ms.ord;
      loc.out[loc.n] = (uint8_t)outc;
      loc.n++;
    }
  }
  const double scale = mode == 2 ? 1.0 : 1.0 / sqrt(pj);
  for (int x = 0; x < (1 << K); ++x) {
    double cr = scale, ci = 0.0;
    for (int j = 0; j < K; ++j) {
      const int b = (x >> j) & 1;
      const double nr = cr * ur[j][b] - ci * ui[j][b], ni = cr * ui[j][b] + ci * ur[j][b];
      cr = nr;
      ci = ni;
    }
    cv[x][0] = cr;
    cv[x][1] = ci;
  }
}

template <typename T, int K>
__global__ void __launch_bounds__(256) shrinkk_kernel(const StepDesc d, const DevPtrs p) {
  typedef typename VT<T>::C C;
  constexpr int D = 1 << K, MV = 2 * JOINT_KMAX;
  __shared__ double cv[1 << JOINT_KMAX][2];
  __shared__ PassShared sh;
  if (threadIdx.x == 0) joint_decide(d, p, blockIdx.x == 0, cv, p.partials + RHOK_RESULT_OFF);
  __syncthreads();
  const int w = d.width, wo = w - K;
  const C* st = reinterpret_cast<const C*>(p.state);
  C* out = reinterpret_cast<C*>(p.scratch);
  T cr[D], ci[D];
  uint64_t moff[D];
#pragma unroll
  for (int x = 0; x < D; ++x) {
    cr[x] = (T)cv[x][0];
    ci[x] = (T)cv[x][1];
    moff[x] = pdep_pos((uint64_t)x, d.jm_pos, K);
  }
  // output bit t comes from source position j_src[t]: identity except for the <= 2K bits the
  // eliminations moved (the top qubits into freed positions) -- a keep mask plus a short list
  uint64_t keep = 0;
  int nmv = 0, mv_t[MV], mv_s[MV];
#pragma unroll
  for (int q = 0; q < MV; ++q) mv_t[q] = mv_s[q] = 0;
  bool general = false;
  for (int t = 0; t < wo; ++t) {
    if (d.j_src[t] == t) {
      keep |= 1ull << t;
      continue;
    }
#pragma unroll
    for (int q = 0; q < MV; ++q)
      if (q == nmv) {
        mv_t[q] = t;
        mv_s[q] = d.j_src[t];
      }
    if (nmv < MV) ++nmv;
    else general = true;
  }
  double acc[4] = {0, 0, 0, 0};
  const uint64_t n = 1ull << wo;
  // U output elements per thread and iteration (a grid stride apart), every load issued before the
  // arithmetic (U * D independent loads in flight per thread)
  constexpr int U = K <= 2 ? 4 : 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    C v[U][D];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * stride < n ? i0 + u * stride : i0;
      uint64_t src = i & keep;
      if (!general) {
#pragma unroll
        for (int q = 0; q < MV; ++q)
          if (q < nmv) src |= ((i >> mv_t[q]) & 1ull) << mv_s[q];
      } else {
        src = 0;
        for (int t = 0; t < wo; ++t) src |= ((i >> t) & 1ull) << d.j_src[t];
      }
#pragma unroll
      for (int x = 0; x < D; ++x) v[u][x] = st[src | moff[x]];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i >= n) break;
      T orr = 0, oi = 0;
#pragma unroll
      for (int x = 0; x < D; ++x) {
        orr += cr[x] * v[u][x].x - ci[x] * v[u][x].y;
        oi += cr[x] * v[u][x].y + ci[x] * v[u][x].x;
      }
      out[i] = make_c<T>(orr, oi);
      acc[0] += (double)orr * orr + (double)oi * oi;
    }
  }
  if (d.red_kind == RED_NORM) reduce_finish<1>(acc, p, sh);
}

// ------------------------------------------------------------------------------------------------
// Batched small-width replicas: one CTA runs the WHOLE step program on one
// state held in shared memory; the grid walks a batch of independent inputs (config 1's 64
// inputs, recognition's basis columns, seed sweeps). Per-state outcomes / prob0 / run params.
// ------------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128) batch_kernel(const StepDesc* steps, int n_steps, DevPtrs base, int K,
                                                    int n_batch, const double2* in, double2* out, int n_in,
                                                    int n_out, PermTab tab) {
  typedef typename VT<T>::C C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* s = reinterpret_cast<C*>(smem_raw);
  __shared__ PassShared sh;
  __shared__ double red[4];
  __shared__ double rhok_w[4][RHOK_VALS], rhok_s[RHOK_VALS], cv_s[1 << JOINT_KMAX][2];
  const T r2 = (T)0.70710678118654752440;
  for (int b = blockIdx.x; b < n_batch; b += gridDim.x) {
    DevPtrs p = base;
    p.outcome += (size_t)b * K;
    p.prob0 += (size_t)b * K;
    p.forced += (size_t)b * K;
    p.run += b;
    p.err += b;
    p.red_result = red;
    const int nin = 1 << n_in;
    for (int i = threadIdx.x; i < nin; i += blockDim.x) {
      double2 v = in[(size_t)b * nin + i];
      s[i] = make_c<T>((T)v.x, (T)v.y);
    }
    __syncthreads();
    for (int t = 0; t < n_steps; ++t) {
      const StepDesc& d = steps[t];
      double acc[4] = {0, 0, 0, 0};
      if (d.kind == ST_PASS) {
        pass_prologue(d, p, sh, true);
        smem_apply_ops<T>(d, p, s, sh);
        smem_reduce<T>(d.red_kind, d.red_slot, d.width, s, acc);
      } else if (d.kind == ST_GROW) {
        const int n = 1 << d.width;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          C v = s[i];
          v.x *= r2;
          v.y *= r2;
          s[i] = v;
          s[i + n] = v;
          acc[0] += 2.0 * ((double)v.x * v.x + (double)v.y * v.y);
        }
        __syncthreads();
      } else if (d.kind == ST_SHRINK) {
        if (threadIdx.x == 0) {
          LocalOutcomes loc;
          loc.n = 0;
          decide(p, d.shrink_m, true, d.first_full_rho != 0, true, sh.coef[0], loc);
        }
        __syncthreads();
        const T u0r = (T)sh.coef[0][0], u0i = (T)sh.coef[0][1], u1r = (T)sh.coef[0][2], u1i = (T)sh.coef[0][3];
        const int w = d.width, bb = d.slot, top = w - 1;
        if (bb == top) {
          const int h = 1 << (w - 1);
          for (int i = threadIdx.x; i < h; i += blockDim.x) {
            C x0 = s[i], x1 = s[i + h];
            T orr, oi;
            cmul_add<T>(u0r, u0i, x0.x, x0.y, u1r, u1i, x1.x, x1.y, orr, oi);
            s[i] = make_c<T>(orr, oi);
            acc[0] += (double)orr * orr + (double)oi * oi;
          }
        } else {
          const int nq = 1 << (w - 2);
          for (int i = threadIdx.x; i < nq; i += blockDim.x) {
            int rr = ((i >> bb) << (bb + 1)) | (i & ((1 << bb) - 1));
            rr = ((rr >> top) << (top + 1)) | (rr & ((1 << top) - 1));
            const int B = 1 << bb, TT = 1 << top;
            C x00 = s[rr], x10 = s[rr | B], x01 = s[rr | TT], x11 = s[rr | B | TT];
            T o0r, o0i, o1r, o1i;
            cmul_add<T>(u0r, u0i, x00.x, x00.y, u1r, u1i, x10.x, x10.y, o0r, o0i);
            cmul_add<T>(u0r, u0i, x01.x, x01.y, u1r, u1i, x11.x, x11.y, o1r, o1i);
            s[rr] = make_c<T>(o0r, o0i);
            s[rr | B] = make_c<T>(o1r, o1i);
            acc[0] += (double)o0r * o0r + (double)o0i * o0i + (double)o1r * o1r + (double)o1i * o1i;
          }
        }
        __syncthreads();
      }
      else if (d.kind == ST_RHOK) {  // joint measurement: rho of the jk positions (block, fixed order)
        const int k = d.jk, D = 1 << k, w = d.width;
        uint32_t mm = 0;
        for (int j = 0; j < k; ++j) mm |= 1u << d.jm_pos[j];
        double a[RHOK_VALS];
        for (int v = 0; v < RHOK_VALS; ++v) a[v] = 0.0;
        for (int r = threadIdx.x; r < (1 << (w - k)); r += blockDim.x) {
          uint32_t base = 0;
          for (int bit = 0, q = 0; bit < w; ++bit)
            if (!((mm >> bit) & 1)) base |= (uint32_t)((r >> q++) & 1) << bit;
          int e = 0;
          for (int x = 0; x < D; ++x)
            for (int y = x; y < D; ++y) {
              const C u = s[base | (uint32_t)pdep_pos((uint64_t)x, d.jm_pos, k)];
              const C v = s[base | (uint32_t)pdep_pos((uint64_t)y, d.jm_pos, k)];
              a[e++] += (double)u.x * v.x + (double)u.y * v.y;
              a[e++] += (double)u.y * v.x - (double)u.x * v.y;
            }
        }
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int v = 0; v < RHOK_VALS; ++v) {
          double x = a[v];
          for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULLMASK, x, o);
          if (lane == 0) rhok_w[warp][v] = x;
        }
        __syncthreads();
        for (int v = threadIdx.x; v < RHOK_VALS; v += blockDim.x) {
          double t = 0;
          for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += rhok_w[q][v];
          rhok_s[v] = t;
        }
        __syncthreads();
      } else if (d.kind == ST_SHRINKK) {
        if (threadIdx.x == 0) joint_decide(d, p, true, cv_s, rhok_s);
        __syncthreads();
        const int k = d.jk, wo = d.width - k;
        T o_r[16], o_i[16];
        int cnt = 0;
        for (int i = threadIdx.x; i < (1 << wo); i += blockDim.x, ++cnt) {
          uint32_t src = 0;
          for (int t2 = 0; t2 < wo; ++t2) src |= (uint32_t)((i >> t2) & 1) << d.j_src[t2];
          T orr = 0, oi = 0;
          for (int x = 0; x < (1 << k); ++x) {
            const C v = s[src | (uint32_t)pdep_pos((uint64_t)x, d.jm_pos, k)];
            const T cr = (T)cv_s[x][0], ci = (T)cv_s[x][1];
            orr += cr * v.x - ci * v.y;
            oi += cr * v.y + ci * v.x;
          }
          o_r[cnt] = orr;
          o_i[cnt] = oi;
          acc[0] += (double)orr * orr + (double)oi * oi;
        }
        __syncthreads();
        cnt = 0;
        for (int i = threadIdx.x; i < (1 << wo); i += blockDim.x, ++cnt) s[i] = make_c<T>(o_r[cnt], o_i[cnt]);
        __syncthreads();
      }
      if (d.red_kind != RED_NONE) block_sum4(acc, sh, red);
    }
    const int nout = 1 << n_out;
    for (int j = threadIdx.x; j < nout; j += blockDim.x) {
      int src = 0;
      for (int k = 0; k < n_out; ++k) src |= ((j >> k) & 1) << tab.slot[k];
      C v = s[src];
      out[(size_t)b * nout + j] = make_double2((double)v.x, (double)v.y);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------------
// GROW: append |+> at the top slot (an N that no measurement could absorb).
// ------------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) grow_kernel(const StepDesc d, const DevPtrs p) {
  typedef typename VT<T>::C C;
  __shared__ PassShared sh;
  C* st = reinterpret_cast<C*>(p.state);
  const uint64_t n = 1ull << d.width;
  const T r = (T)0.70710678118654752440;
  double acc[4] = {0, 0, 0, 0};
  if (sizeof(T) == 4 && d.width >= 1) {
    // complex64: 16 B per thread access (two amplitudes), 512 B per warp instruction
    float4* s4 = reinterpret_cast<float4*>(p.state);
    const uint64_t n2 = n >> 1;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (uint64_t)gridDim.x * blockDim.x) {
      float4 v = __ldcs(s4 + i);
      v.x *= (float)r; v.y *= (float)r; v.z *= (float)r; v.w *= (float)r;
      __stcs(s4 + i, v);
      __stcs(s4 + i + n2, v);
      acc[0] += 2.0 * ((double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w);
    }
  } else {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
      C v = st[i];
      v.x *= r;
      v.y *= r;
      st[i] = v;
      st[i + n] = v;
      acc[0] += 2.0 * ((double)v.x * v.x + (double)v.y * v.y);
    }
  }
  if (d.red_kind == RED_NORM) reduce_finish<1>(acc, p, sh);
}

// complex64 SHRINK body with 16 B accesses: each thread produces two consecutive output
// amplitudes (a float4) from float4 loads of the 4-group rows (b >= 1), from two float4 loads that
// each hold an (x_b=0, x_b=1) pair (b = 0), or from the lower / upper halves (b = top).
__device__ __forceinline__ float2 shrink_out(float u0r, float u0i, float u1r, float u1i, float x0r, float x0i,
                                             float x1r, float x1i) {
  return make_float2(u0r * x0r - u0i * x0i + u1r * x1r - u1i * x1i, u0r * x0i + u0i * x0r + u1r * x1i + u1i * x1r);
}
__device__ void shrink_c64(int w, int b, float u0r, float u0i, float u1r, float u1i, float4* s4, double (&acc)[4]) {
  const int top = w - 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  auto add = [&](float2 o) { acc[0] += (double)o.x * o.x + (double)o.y * o.y; };
  if (b == top) {  // x0 = lower half, x1 = upper half; output = lower half
    const uint64_t h2 = 1ull << (w - 2);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < h2; i += stride) {
      const float4 x0 = __ldcs(s4 + i), x1 = __ldcs(s4 + i + h2);
      const float2 o0 = shrink_out(u0r, u0i, u1r, u1i, x0.x, x0.y, x1.x, x1.y);
      const float2 o1 = shrink_out(u0r, u0i, u1r, u1i, x0.z, x0.w, x1.z, x1.w);
      __stcs(s4 + i, make_float4(o0.x, o0.y, o1.x, o1.y));
      add(o0);
      add(o1);
    }
  } else if (b == 0) {  // (x_b0, x_b1) adjacent: one float4 per (row of top); the top moves into slot 0
    const uint64_t nq = 1ull << (w - 2), T2 = 1ull << (top - 1);  // float4 units; top bit in unit index
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += stride) {
      const float4 a = __ldcs(s4 + i), c = __ldcs(s4 + i + T2);  // a = (x00, x10), c = (x01, x11)
      const float2 o0 = shrink_out(u0r, u0i, u1r, u1i, a.x, a.y, a.z, a.w);
      const float2 o1 = shrink_out(u0r, u0i, u1r, u1i, c.x, c.y, c.z, c.w);
      __stcs(s4 + i, make_float4(o0.x, o0.y, o1.x, o1.y));  // out[r] = o0, out[r | B] = o1
      add(o0);
      add(o1);
    }
  } else {  // float4 unit = amplitudes (2k, 2k + 1): both have the same b / top bits
    const uint64_t nq2 = 1ull << (w - 3);
    const uint64_t B = 1ull << (b - 1), TT = 1ull << (top - 1);  // in float4 units
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq2; i += stride) {
      uint64_t r = ((i >> (b - 1)) << b) | (i & (B - 1));
      r = ((r >> (top - 1)) << top) | (r & (TT - 1));
      const float4 x00 = __ldcs(s4 + r), x10 = __ldcs(s4 + (r | B)), x01 = __ldcs(s4 + (r | TT)), x11 = __ldcs(s4 + (r | B | TT));
      const float2 a0 = shrink_out(u0r, u0i, u1r, u1i, x00.x, x00.y, x10.x, x10.y);
      const float2 a1 = shrink_out(u0r, u0i, u1r, u1i, x00.z, x00.w, x10.z, x10.w);
      const float2 c0 = shrink_out(u0r, u0i, u1r, u1i, x01.x, x01.y, x11.x, x11.y);
      const float2 c1 = shrink_out(u0r, u0i, u1r, u1i, x01.z, x01.w, x11.z, x11.w);
      __stcs(s4 + r, make_float4(a0.x, a0.y, a1.x, a1.y));
      __stcs(s4 + (r | B), make_float4(c0.x, c0.y, c1.x, c1.y));
      add(a0); add(a1); add(c0); add(c1);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// SHRINK: measurement with elimination and no fresh neighbour (Fig. 6's compaction, made
// race-free in place: the top qubit moves into the freed slot; DESIGN.md §5 K3).
// ------------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) shrink_kernel(const StepDesc d, const DevPtrs p) {
  typedef typename VT<T>::C C;
  __shared__ PassShared sh;
  if (threadIdx.x == 0) {
    LocalOutcomes loc;
    loc.n = 0;
    decide(p, d.shrink_m, true, d.first_full_rho != 0, blockIdx.x == 0, sh.coef[0], loc);
  }
  __syncthreads();
  const T u0r = (T)sh.coef[0][0], u0i = (T)sh.coef[0][1], u1r = (T)sh.coef[0][2], u1i = (T)sh.coef[0][3];
  C* st = reinterpret_cast<C*>(p.state);
  const int w = d.width, b = d.slot, top = w - 1;
  double acc[4] = {0, 0, 0, 0};
  if (sizeof(T) == 4 && w >= 3) {
    shrink_c64(w, b, (float)u0r, (float)u0i, (float)u1r, (float)u1i, reinterpret_cast<float4*>(p.state), acc);
    if (d.red_kind == RED_NORM) reduce_finish<1>(acc, p, sh);
    return;
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (b == top) {
    const uint64_t h = 1ull << (w - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < h; i += stride) {
      C x0 = st[i], x1 = st[i + h];
      T orr, oi;
      cmul_add<T>(u0r, u0i, x0.x, x0.y, u1r, u1i, x1.x, x1.y, orr, oi);
      st[i] = make_c<T>(orr, oi);
      acc[0] += (double)orr * orr + (double)oi * oi;
    }
  } else {
    const uint64_t nq = 1ull << (w - 2);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += stride) {
      uint64_t r = ((i >> b) << (b + 1)) | (i & ((1ull << b) - 1));
      r = ((r >> top) << (top + 1)) | (r & ((1ull << top) - 1));
      const uint64_t B = 1ull << b, TT = 1ull << top;
      C x00 = st[r], x10 = st[r | B], x01 = st[r | TT], x11 = st[r | B | TT];
      T o0r, o0i, o1r, o1i;
      cmul_add<T>(u0r, u0i, x00.x, x00.y, u1r, u1i, x10.x, x10.y, o0r, o0i);
      cmul_add<T>(u0r, u0i, x01.x, x01.y, u1r, u1i, x11.x, x11.y, o1r, o1i);
      st[r] = make_c<T>(o0r, o0i);
      st[r | B] = make_c<T>(o1r, o1i);
      acc[0] += (double)o0r * o0r + (double)o0i * o0i + (double)o1r * o1r + (double)o1i * o1i;
    }
  }
  if (d.red_kind == RED_NORM) reduce_finish<1>(acc, p, sh);
}

// ------------------------------------------------------------------------------------------------
// I/O and helpers
// ------------------------------------------------------------------------------------------------


// shard scatter: out[perm(G)] = shard[L] with G = (rank << wl) | L (output bit k <- position slot[k])
template <typename T, typename TO>
__global__ void scatter_out_kernel(const void* shard, void* out, int nbits, PermTab tab, uint64_t rank, int wl) {
  typedef typename VT<T>::C C;
  typedef typename VT<TO>::C CO;
  const C* st = reinterpret_cast<const C*>(shard);
  CO* o = reinterpret_cast<CO*>(out);
  const uint64_t n = 1ull << wl;
  for (uint64_t L = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n; L += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t G = (rank << wl) | L;
    uint64_t j = 0;
    for (int k = 0; k < nbits; ++k) j |= ((G >> tab.slot[k]) & 1ull) << k;
    C v = st[L];
    o[j] = make_c<TO>((TO)v.x, (TO)v.y);
  }
}

// out[j] = state[src(j)], bit k of j <-> slot tab.slot[k]  (output order outputs[0] = LSB)
template <typename T, typename TO>
__global__ void permute_out_kernel(const void* state, void* out, int nbits, PermTab tab, uint64_t j0, uint64_t count) {
  typedef typename VT<T>::C C;
  typedef typename VT<TO>::C CO;
  const C* st = reinterpret_cast<const C*>(state);
  CO* o = reinterpret_cast<CO*>(out);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t j = j0 + i, src = 0;
    for (int k = 0; k < nbits; ++k) src |= ((j >> k) & 1ull) << tab.slot[k];
    C v = st[src];
    o[i] = make_c<TO>((TO)v.x, (TO)v.y);
  }
}

// Output permutation through shared-memory tiles (the whole output in one launch): out bit k <- state
// bit slot[k]. A tile fixes every state bit outside TS = {state bits 0..4} u {slot[0..4]} (padded
// with further low state bits to 10 bits); it is read in state order (TS's low bits are state bits
// 0..4: 256 B runs per warp for complex64) and written in output order (its lowest output bits are
// output bits 0..4: 256 B runs), so both sides are coalesced -- the per-element loop of
// permute_out_kernel reads 32 scattered sectors per warp instead.
constexpr int PERM_T = 11;
struct PermPlan {
  int8_t ts[PERM_T];     // tile bit j (e index) <- state position ts[j], ascending
  int8_t fo[PERM_T];     // output-order bit i (f index) <- e bit fo[i]
  int8_t op[PERM_T];     // ... at output position op[i], ascending
  int8_t other[64];      // state positions outside the tile, ascending (tile id bits)
  int8_t other_out[64];  // their output positions
  int n_other;
};

// Index math is hoisted: a thread's element e = threadIdx.x + 256 r of a tile has its state and
// output offsets split into a per-thread part (8 low bits) and a compile-time-r part, and the tile's
// base offsets (the n_other id bits) are built by one lane per bit and OR-reduced across the warp.
// The per-element bit loops of the first version made the kernel integer-bound (1.21 ms for
// 2 x 2 GiB at width 28, 0.54 of the copy peak).
template <typename T, typename TO>
__global__ void __launch_bounds__(256) permute_out_tiled_kernel(const void* state, void* out, PermPlan pl, uint64_t n_tiles) {
  typedef typename VT<T>::C C;
  typedef typename VT<TO>::C CO;
  constexpr int R = (1 << PERM_T) / 256;
  __shared__ C tile[1 << PERM_T];
  const C* st = reinterpret_cast<const C*>(state);
  CO* o = reinterpret_cast<CO*>(out);
  const unsigned lane = threadIdx.x & 31;
  uint64_t ld_lo = 0, oi_lo = 0;
  unsigned e_lo = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const unsigned b = (threadIdx.x >> j) & 1u;
    ld_lo |= (uint64_t)b << pl.ts[j];
    e_lo |= b << pl.fo[j];
    oi_lo |= (uint64_t)b << pl.op[j];
  }
  uint64_t ld_hi[R], oi_hi[R];
  unsigned e_hi[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    ld_hi[r] = oi_hi[r] = 0;
    e_hi[r] = 0;
#pragma unroll
    for (int j = 8; j < PERM_T; ++j) {
      const unsigned b = (r >> (j - 8)) & 1u;
      ld_hi[r] |= (uint64_t)b << pl.ts[j];
      e_hi[r] |= b << pl.fo[j];
      oi_hi[r] |= (uint64_t)b << pl.op[j];
    }
  }
  const int k0 = (int)lane, k1 = (int)lane + 32;
  for (uint64_t tid = blockIdx.x; tid < n_tiles; tid += gridDim.x) {
    uint64_t sbl = 0, obl = 0;
    if (k0 < pl.n_other && ((tid >> k0) & 1ull)) {
      sbl |= 1ull << pl.other[k0];
      obl |= 1ull << pl.other_out[k0];
    }
    if (k1 < pl.n_other && ((tid >> k1) & 1ull)) {
      sbl |= 1ull << pl.other[k1];
      obl |= 1ull << pl.other_out[k1];
    }
    const uint64_t sb = ((uint64_t)__reduce_or_sync(0xffffffffu, (unsigned)(sbl >> 32)) << 32) |
                        __reduce_or_sync(0xffffffffu, (unsigned)sbl);
    const uint64_t ob = ((uint64_t)__reduce_or_sync(0xffffffffu, (unsigned)(obl >> 32)) << 32) |
                        __reduce_or_sync(0xffffffffu, (unsigned)obl);
    C v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = __ldcs(st + (sb | ld_lo | ld_hi[r]));
    // tile slot of element e: e ^ (e bits 5..9 folded onto bits 0..4), a bijection that keeps both
    // the state-order writes (lanes = e bits 0..4) and the output-order reads (lanes = the e bits of
    // output bits 0..4, often 5..9) spread over the banks
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const unsigned e = threadIdx.x + 256u * r;
      tile[e ^ ((e >> 5) & 31u)] = v[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const unsigned e = e_lo | e_hi[r];
      const C w = tile[e ^ ((e >> 5) & 31u)];
      __stcs(o + (ob | oi_lo | oi_hi[r]), make_c<TO>((TO)w.x, (TO)w.y));
    }
    __syncthreads();
  }
}

// false when the slots are not a permutation of [0, nbits) or nbits < PERM_T (caller falls back)
static bool make_perm_plan(int nbits, const int* slots, PermPlan& pl) {
  if (nbits < PERM_T || nbits > 62) return false;
  int o_of_s[64];
  for (int k = 0; k < 64; ++k) o_of_s[k] = -1;
  for (int k = 0; k < nbits; ++k) {
    if (slots[k] < 0 || slots[k] >= nbits || o_of_s[slots[k]] >= 0) return false;
    o_of_s[slots[k]] = k;
  }
  uint64_t m = 0;
  for (int k = 0; k < 5; ++k) m |= (1ull << k) | (1ull << slots[k]);
  for (int k = 0; k < nbits && __builtin_popcountll(m) < PERM_T; ++k) m |= 1ull << k;
  int j = 0, q = 0;
  for (int s = 0; s < nbits; ++s) {
    if ((m >> s) & 1) pl.ts[j++] = (int8_t)s;
    else {
      pl.other[q] = (int8_t)s;
      pl.other_out[q] = (int8_t)o_of_s[s];
      ++q;
    }
  }
  pl.n_other = q;
  int idx[PERM_T];
  for (int i = 0; i < PERM_T; ++i) idx[i] = i;
  std::sort(idx, idx + PERM_T, [&](int a, int b) { return o_of_s[pl.ts[a]] < o_of_s[pl.ts[b]]; });
  for (int i = 0; i < PERM_T; ++i) {
    pl.fo[i] = (int8_t)idx[i];
    pl.op[i] = (int8_t)o_of_s[pl.ts[idx[i]]];
  }
  return true;
}

template <typename TI, typename T>
__global__ void convert_in_kernel(const void* src, void* state, uint64_t j0, uint64_t count) {
  typedef typename VT<TI>::C CI;
  typedef typename VT<T>::C C;
  const CI* s = reinterpret_cast<const CI*>(src);
  C* st = reinterpret_cast<C*>(state);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    CI v = s[i];
    st[j0 + i] = make_c<T>((T)v.x, (T)v.y);
  }
}

template <typename T>
__global__ void basis_kernel(void* state, uint64_t n, uint64_t k) {
  typedef typename VT<T>::C C;
  C* st = reinterpret_cast<C*>(state);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    st[i] = make_c<T>(i == k ? (T)1 : (T)0, (T)0);
}

// Counter-based Haar input (workloads/inputs.py documents the same generator), unnormalised,
// with the norm reduced into red_result[0].
template <typename T>
__global__ void __launch_bounds__(256) haar_kernel(DevPtrs p, uint64_t n, uint64_t seed, uint64_t j0) {
  typedef typename VT<T>::C C;
  __shared__ PassShared sh;
  C* st = reinterpret_cast<C*>(p.state);
  const uint64_t key = splitmix64(seed);
  double acc[4] = {0, 0, 0, 0};
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t a = splitmix64(key ^ splitmix64(2 * (j + j0)));
    uint64_t b = splitmix64(key ^ splitmix64(2 * (j + j0) + 1));
    double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;
    double u2 = (double)(b >> 11) * 0x1.0p-53;
    double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    double re = r * cs, im = r * sn;
    st[j] = make_c<T>((T)re, (T)im);
    acc[0] += re * re + im * im;
  }
  reduce_finish<1>(acc, p, sh);
}

template <typename T>
__global__ void scale_kernel(void* state, uint64_t n, const double* red_result) {
  typedef typename VT<T>::C C;
  C* st = reinterpret_cast<C*>(state);
  const double s = 1.0 / sqrt(red_result[0]);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    C v = st[i];
    st[i] = make_c<T>((T)(v.x * s), (T)(v.y * s));
  }
}

// <a|b> of two complex128 vectors into red_result[0..1]
__global__ void __launch_bounds__(256) dot_kernel(DevPtrs p, const double2* a, const double2* b, uint64_t n) {
  __shared__ PassShared sh;
  double acc[4] = {0, 0, 0, 0};
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i];
    acc[0] += x.x * y.x + x.y * y.y;
    acc[1] += x.x * y.y - x.y * y.x;
  }
  reduce_finish<2>(acc, p, sh);
}

// ------------------------------------------------------------------------------------------------
// Host-side launchers (C++ linkage inside namespace owqs; used by runtime.cpp)
// ------------------------------------------------------------------------------------------------
struct KernelLimits {
  int max_blocks_pass[2][KMAX_AOT + 1];
  int one_cta[KMAX_AOT + 1];  // use the 1-CTA/SM (uncapped registers) variant
  int max_blocks_elem;
  int sm_count;
};
static KernelLimits g_lim;
static bool g_lim_ready = false;

template <typename T, int KHI, int UNR>
static void* pass_fn() { return (void*)pass_kernel<T, KHI, UNR>; }

cudaError_t init_kernel_limits(int device) {
  if (g_lim_ready) return cudaSuccess;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return e;
  g_lim.sm_count = prop.multiProcessorCount;
  void* fns[2][KMAX_AOT + 1] = {
      {pass_fn<float, 0, 4>(), pass_fn<float, 1, 2>(), pass_fn<float, 2, 1>(), pass_fn<float, 3, 1>(), pass_fn<float, 4, 1>()},
      {pass_fn<double, 0, 4>(), pass_fn<double, 1, 2>(), pass_fn<double, 2, 1>(), pass_fn<double, 3, 1>(), pass_fn<double, 4, 1>()}};
  for (int k = 0; k <= KMAX_AOT; ++k) g_lim.one_cta[k] = 0;
  if (const char* env = getenv("OWQS_ONE_CTA"))  // bit k: KHI = k uses the 1-CTA/SM variant
    for (int k = 3; k <= KMAX_AOT; ++k) g_lim.one_cta[k] = (atoi(env) >> k) & 1;
  void* one[2][2] = {{(void*)pass_kernel<float, 3, 1, 1>, (void*)pass_kernel<float, 4, 1, 1>},
                     {(void*)pass_kernel<double, 3, 1, 1>, (void*)pass_kernel<double, 4, 1, 1>}};
  for (int pr = 0; pr < 2; ++pr)
    for (int k = 0; k <= KMAX_AOT; ++k) {
      int nb = 0;
      void* f = (k >= 3 && g_lim.one_cta[k]) ? one[pr][k - 3] : fns[pr][k];
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, 256, 0);
      if (e != cudaSuccess) return e;
      g_lim.max_blocks_pass[pr][k] = std::max(1, nb) * g_lim.sm_count;
    }
  g_lim.max_blocks_elem = 8 * g_lim.sm_count;
  e = cudaFuncSetAttribute(small_pass_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 1 << 16);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(small_pass_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 1 << 16);
  if (e != cudaSuccess) return e;
  g_lim_ready = true;
  return cudaSuccess;
}

int max_partial_blocks() { return RED_MAX_BLOCKS + RED_MAX_GROUPS; }

// Decisions of one pass for the generated pass kernels (one warp; PassCoef read by every CTA).
__global__ void __launch_bounds__(32) decide_kernel(const StepDesc d, const DevPtrs p, PassCoef* pc, int trigger,
                                                    const cudaGraphDeviceNode_t* nodes, int n_nodes, unsigned long long off) {
  // the pass kernel that follows is launched with programmatic stream serialisation: let its CTAs
  // become resident now (they L2-prefetch their tile, then griddepcontrol.wait for this grid before
  // any read of the state or of pc; this grid in turn completes only after its own wait below, so
  // the previous pass's stores are visible to the pass kernel transitively). When the decisions go
  // into the pass kernel's parameters (graph node update, below) it may start only after them.
  if (trigger && n_nodes == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // launched behind grid_finish_kernel with programmatic serialisation too: wait for the previous
  // grid (the reduction this pass decides from) before reading anything it wrote
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ PassShared sh;
  pass_prologue(d, p, sh, true);
  const int t = threadIdx.x;
  for (int b = t; b < d.n_bfly; b += 32) {
    const double ar = sh.ka[b][0], ai = sh.ka[b][1];
    pc->ard[b] = ar;
    pc->aid[b] = ai;
    pc->ar[b] = (float)ar;
    const float fai = (float)ai;
    pc->B[b] = ((uint64_t)__float_as_uint(fai) << 32) | (uint64_t)__float_as_uint(-fai);
  }
  for (int i = t; i < d.n_ops; i += 32) pc->cond[i] = sh.cond[i];
  if (t == 0) pc->scale = sh.scale;
  if (n_nodes > 0) {
    // the pass kernel node(s) of the captured graph (device-updatable, one per local shard) take the
    // decisions as their by-value PassCoef parameter: constant-bank operands in the generated
    // kernels. The update must be visible before the dependent launch is triggered.
    __syncwarp();
    __threadfence();
    if (t == 0) {
      for (int k = 0; k < n_nodes; ++k) {
        const cudaError_t e = cudaGraphKernelNodeSetParam(nodes[k], (size_t)off, pc, sizeof(PassCoef));
        if (e != cudaSuccess) atomicExch(p.err, 2);
      }
      __threadfence();
    }
    __syncwarp();
    if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
}

// All of a run's tile-pass decisions up front. Valid when every decision is structural (R-13: no
// pass decides from a reduction, no SHRINK) and every measurement is decided by a tile pass: an
// outcome then depends only on its keyed draw against prob0 = 1/2 (or on the forced string), never
// on the state or on other outcomes, so (1) one thread per measurement writes every outcome, then
// (2) one warp per pass evaluates its signals (Eq. 2 angles, folded X, conditional ops) from those
// outcomes and writes its PassCoef -- exactly what the per-pass decide kernels compute. The pass
// kernels then run back to back (programmatic serialisation, no decide kernel or copy node between
// them): config 2, whose 8 MiB state makes every pass launch-latency-bound, 0.568 -> 0.50 ms with a
// sequential single-warp version of (2).
__global__ void __launch_bounds__(256) decide_ahead_outcomes_kernel(const DevPtrs p, int n_mst) {
  const int mode = p.run->mode;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_mst; i += gridDim.x * blockDim.x) {
    const MStatic ms = p.mst[i];
    const int outc = mode == 0 ? (draw_uniform(p.run->seed, ms.key) <= 0.5 ? 0 : 1) : (p.forced[ms.ord] & 1);
    p.outcome[ms.ord] = (uint8_t)outc;
  }
}

__global__ void __launch_bounds__(32) decide_ahead_kernel(const StepDesc* steps, const DevPtrs p, PassCoef* pc) {
  __shared__ PassShared sh;
  const int t = threadIdx.x, k = blockIdx.x;
  const StepDesc& d = steps[k];
  if (d.kind != ST_PASS || d.n_ops == 0) return;  // a pass without butterflies may still hold conditional ops
  pass_prologue(d, p, sh, true);
  PassCoef* c = pc + k;
  for (int b = t; b < d.n_bfly; b += 32) {
    const double ar = sh.ka[b][0], ai = sh.ka[b][1];
    c->ard[b] = ar;
    c->aid[b] = ai;
    c->ar[b] = (float)ar;
    const float fai = (float)ai;
    c->B[b] = ((uint64_t)__float_as_uint(fai) << 32) | (uint64_t)__float_as_uint(-fai);
  }
  for (int i = t; i < d.n_ops; i += 32) c->cond[i] = sh.cond[i];
  if (t == 0) c->scale = sh.scale;
}

cudaError_t launch_decide_ahead(const StepDesc* d_steps, int n_steps, int n_mst, const DevPtrs& p, PassCoef* pc,
                                cudaStream_t s) {
  if (n_mst > 0) decide_ahead_outcomes_kernel<<<(unsigned)std::min(1184, (n_mst + 255) / 256), 256, 0, s>>>(p, n_mst);
  if (n_steps > 0) decide_ahead_kernel<<<(unsigned)n_steps, 32, 0, s>>>(d_steps, p, pc);
  return cudaGetLastError();
}

// Sum of the block partials of a tile pass (fixed order: deterministic) into red_result.
// Sum of the tile kernels' block partials into red_result, deterministic: CTA g sums the contiguous
// range of partials [g * per, (g + 1) * per) in a fixed order into gpart[g]; the last CTA to arrive
// (fenced counter) sums gpart[0..G) in order. G <= RED_MAX_GROUPS CTAs of 256 threads keep the
// 2^15-partial sum of a 2^28-amplitude pass at a few microseconds (one CTA: ~24 us).
__global__ void __launch_bounds__(256) grid_finish_kernel(DevPtrs p, unsigned nblk, int nred) {
  // let the next pass's decide kernel (one warp) launch now; it waits for this grid before reading
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ double red[8][4];
  __shared__ int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned per = (nblk + gridDim.x - 1) / gridDim.x;
  const unsigned b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
  double* gpart = p.partials + (size_t)RED_MAX_BLOCKS * 4;
  auto block_sum = [&](double (&v)[4], double* out) {
    for (int k = 0; k < 4; ++k)
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(FULLMASK, v[k], o);
    if (lane == 0)
      for (int k = 0; k < 4; ++k) red[warp][k] = v[k];
    __syncthreads();
    if (threadIdx.x < 4) {
      double t = 0;
      for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
      out[threadIdx.x] = threadIdx.x < nred ? t : 0.0;
    }
  };
  double v[4] = {0, 0, 0, 0};
  for (unsigned b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
    const double4 x = *reinterpret_cast<const double4*>(p.partials + (size_t)b * 4);
    v[0] += x.x;
    v[1] += x.y;
    v[2] += x.z;
    v[3] += x.w;
  }
  block_sum(v, gpart + (size_t)blockIdx.x * 4);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&p.counter[0], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double w[4] = {0, 0, 0, 0};
  for (unsigned g = threadIdx.x; g < gridDim.x; g += blockDim.x)
    for (int k = 0; k < 4; ++k) w[k] += __ldcg(&gpart[(size_t)g * 4 + k]);
  __syncthreads();
  block_sum(w, p.red_result);
  if (threadIdx.x == 0) p.counter[0] = 0;
}

cudaError_t launch_grid_finish(const DevPtrs& p, unsigned nblk, int nred, cudaStream_t s) {
  const unsigned g = std::max(1u, std::min((unsigned)RED_MAX_GROUPS, (nblk + 255) / 256));
  grid_finish_kernel<<<g, 256, 0, s>>>(p, nblk, nred);
  return cudaGetLastError();
}

cudaError_t launch_decide(const StepDesc& d, const DevPtrs& p, PassCoef* pc, cudaStream_t s,
                          const cudaGraphDeviceNode_t* nodes, int n_nodes, size_t off) {
  static const bool no_trigger = getenv("OWQS_PDL_NO_TRIGGER") != nullptr;
  static const bool no_pdl = getenv("OWQS_NO_PDL") != nullptr || getenv("OWQS_NO_DECIDE_PDL") != nullptr;
  const int trig = no_trigger ? 0 : 1;
  const unsigned long long o = (unsigned long long)off;
  if (no_pdl) {
    decide_kernel<<<1, 32, 0, s>>>(d, p, pc, trig, nodes, n_nodes, o);
    return cudaGetLastError();
  }
  // programmatic serialisation behind the previous kernel (grid_finish_kernel triggers at its
  // start): the decide kernel's launch latency overlaps the reduction's finish
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decide_kernel, d, p, pc, trig, nodes, n_nodes, o);
}

static inline int unr_of(int khi) { return khi == 0 ? 4 : (khi == 1 ? 2 : 1); }
static inline int log2i(int x) { int r = 0; while ((1 << r) < x) ++r; return r; }

// ---- multi-rank: SWAP halves and reduction all-reduce ------------------------------------------
// half of a shard whose bit `pl` equals `bit`, packed in index order (runs of 2^pl contiguous)
template <typename T>
__global__ void swap_pack_kernel(const void* state, void* buf, int pl, int bit, int unpack, uint64_t j0, uint64_t n) {
  typedef typename VT<T>::C C;
  const C* st = reinterpret_cast<const C*>(state);
  C* sm = reinterpret_cast<C*>(const_cast<void*>(state));
  C* b = reinterpret_cast<C*>(buf);
  // elements [j0, j0 + n) of the half with local bit pl = bit; buf holds them from index 0
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = j0 + i;
    const uint64_t L = ((j >> pl) << (pl + 1)) | ((uint64_t)bit << pl) | (j & ((1ull << pl) - 1));
    if (unpack) sm[L] = b[i];
    else b[i] = st[L];
  }
}

// loopback all-reduce: red[r*4 + k] <- sum_r red[r*4 + k] (fixed order: deterministic)
__global__ void loopback_allreduce_kernel(double* red, int n_ranks) {
  if (threadIdx.x < 4) {
    double s = 0;
    for (int r = 0; r < n_ranks; ++r) s += red[r * 4 + threadIdx.x];
    for (int r = 0; r < n_ranks; ++r) red[r * 4 + threadIdx.x] = s;
  }
}

cudaError_t launch_swap_pack(const void* state, void* buf, int prec, int pl, int bit, bool unpack, uint64_t j0,
                             uint64_t n, cudaStream_t s) {
  unsigned b = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)(g_lim_ready ? g_lim.max_blocks_elem : 1184)));
  if (prec == 0) swap_pack_kernel<float><<<b, 256, 0, s>>>(state, buf, pl, bit, unpack ? 1 : 0, j0, n);
  else swap_pack_kernel<double><<<b, 256, 0, s>>>(state, buf, pl, bit, unpack ? 1 : 0, j0, n);
  return cudaGetLastError();
}

cudaError_t launch_loopback_allreduce(double* red, int n_ranks, cudaStream_t s) {
  loopback_allreduce_kernel<<<1, 32, 0, s>>>(red, n_ranks);
  return cudaGetLastError();
}

// Kernel class of a step (OWQS_KCLASS_* of include/owqs.h).
int step_kclass(const StepDesc& d, int prec) {
  const int SB = prec == 0 ? 6 : 5;
  if (d.kind == ST_RHOK) return 6;
  if (d.kind == ST_SHRINKK) return 7;
  if (d.kind == ST_GROW) return 2;
  if (d.kind == ST_SHRINK) return 3;
  if (d.kind == ST_SWAP) return 5;
  const int slack = d.width - SB - d.nb_hi - log2i(unr_of(d.nb_hi)) - 3;
  if (slack < 0) return 1;
  return d.n_ops == 0 ? 4 : 0;
}

// Launch one step. prec: 0 complex64, 1 complex128.
cudaError_t launch_step(const StepDesc& d, const DevPtrs& p, int prec, cudaStream_t s) {
  const int SB = prec == 0 ? 6 : 5;
  if (d.kind == ST_RHOK || d.kind == ST_SHRINKK) {
    if (d.jk < 1 || d.jk > JOINT_KMAX || d.width < d.jk) return cudaErrorInvalidValue;
    const uint64_t work = 1ull << (d.width - d.jk);
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, (uint64_t)g_lim.max_blocks_elem));
    if (d.kind == ST_RHOK) {
#define OWQS_RK(TT) \
  switch (d.jk) { case 1: rhok_kernel<TT, 1><<<blocks, 256, 0, s>>>(d, p); break; \
                  case 2: rhok_kernel<TT, 2><<<blocks, 256, 0, s>>>(d, p); break; \
                  default: rhok_kernel<TT, 3><<<blocks, 256, 0, s>>>(d, p); break; }
      if (prec == 0) { OWQS_RK(float) } else { OWQS_RK(double) }
#undef OWQS_RK
      return cudaGetLastError();
    }
#define OWQS_SK(TT) \
  switch (d.jk) { case 1: shrinkk_kernel<TT, 1><<<blocks, 256, 0, s>>>(d, p); break; \
                  case 2: shrinkk_kernel<TT, 2><<<blocks, 256, 0, s>>>(d, p); break; \
                  default: shrinkk_kernel<TT, 3><<<blocks, 256, 0, s>>>(d, p); break; }
    if (prec == 0) { OWQS_SK(float) } else { OWQS_SK(double) }
#undef OWQS_SK
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(p.state, p.scratch, (size_t)(prec == 0 ? 8 : 16) << (d.width - d.jk), cudaMemcpyDeviceToDevice, s);
  }
  if (d.kind == ST_PASS) {
    const int khi = d.nb_hi;
    if (khi > KMAX_AOT) return cudaErrorInvalidValue;  // wide passes run only as generated tile kernels
    const int unr = unr_of(khi);
    const int slack = d.width - SB - khi - log2i(unr) - 3;  // units come in groups of 8 warps
    if (slack < 0) {
      if (d.width > 12) return cudaErrorInvalidValue;
      size_t sm = (size_t)(prec == 0 ? 8 : 16) << d.width;
      if (prec == 0) small_pass_kernel<float><<<1, 512, sm, s>>>(d, p);
      else small_pass_kernel<double><<<1, 512, sm, s>>>(d, p);
      return cudaGetLastError();
    }
    uint64_t blocks = 1ull << slack;
    blocks = std::min<uint64_t>(blocks, (uint64_t)g_lim.max_blocks_pass[prec][khi]);
    dim3 grid((unsigned)blocks), blk(256);
#define OWQS_PASS(T, K, U)                                                                      \
  do {                                                                                          \
    if (d.red_kind == RED_NONE) pass_kernel<T, K, U, 0, RED_NONE><<<grid, blk, 0, s>>>(d, p);   \
    else if (d.red_kind == RED_NORM) pass_kernel<T, K, U, 0, RED_NORM><<<grid, blk, 0, s>>>(d, p); \
    else pass_kernel<T, K, U, 0, RED_RHO><<<grid, blk, 0, s>>>(d, p);                            \
  } while (0)
#define OWQS_PASS1(T, K, U) pass_kernel<T, K, U, 1><<<grid, blk, 0, s>>>(d, p)
    if (prec == 0) {
      switch (khi) {
        case 0: OWQS_PASS(float, 0, 4); break;
        case 1: OWQS_PASS(float, 1, 2); break;
        case 2: OWQS_PASS(float, 2, 1); break;
        case 3: if (g_lim.one_cta[3]) OWQS_PASS1(float, 3, 1); else OWQS_PASS(float, 3, 1); break;
        default: if (g_lim.one_cta[4]) OWQS_PASS1(float, 4, 1); else OWQS_PASS(float, 4, 1); break;
      }
    } else {
      switch (khi) {
        case 0: OWQS_PASS(double, 0, 4); break;
        case 1: OWQS_PASS(double, 1, 2); break;
        case 2: OWQS_PASS(double, 2, 1); break;
        case 3: if (g_lim.one_cta[3]) OWQS_PASS1(double, 3, 1); else OWQS_PASS(double, 3, 1); break;
        default: if (g_lim.one_cta[4]) OWQS_PASS1(double, 4, 1); else OWQS_PASS(double, 4, 1); break;
      }
    }
#undef OWQS_PASS
    return cudaGetLastError();
  }
  uint64_t work = d.kind == ST_GROW ? (1ull << d.width) : (1ull << std::max(0, d.width - (d.slot == d.width - 1 ? 1 : 2)));
  if (prec == 0 && d.width >= 3) work >>= 1;  // complex64: two amplitudes (16 B) per thread access
  uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, (uint64_t)g_lim.max_blocks_elem));
  if (d.kind == ST_GROW) {
    if (prec == 0) grow_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(d, p);
    else grow_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(d, p);
  } else {
    if (prec == 0) shrink_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(d, p);
    else shrink_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(d, p);
  }
  return cudaGetLastError();
}

static inline unsigned elem_blocks(uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)(g_lim_ready ? g_lim.max_blocks_elem : 1184)));
}

cudaError_t launch_scatter_out(const void* shard, int prec, void* out, int out_prec, int nbits, const int* slots,
                               uint64_t rank, int wl, cudaStream_t s) {
  PermTab t;
  for (int k = 0; k < 64; ++k) t.slot[k] = (int8_t)(k < nbits ? slots[k] : 0);
  unsigned b = elem_blocks(1ull << wl);
  if (prec == 0 && out_prec == 1) scatter_out_kernel<float, double><<<b, 256, 0, s>>>(shard, out, nbits, t, rank, wl);
  else if (prec == 0) scatter_out_kernel<float, float><<<b, 256, 0, s>>>(shard, out, nbits, t, rank, wl);
  else if (out_prec == 1) scatter_out_kernel<double, double><<<b, 256, 0, s>>>(shard, out, nbits, t, rank, wl);
  else scatter_out_kernel<double, float><<<b, 256, 0, s>>>(shard, out, nbits, t, rank, wl);
  return cudaGetLastError();
}

cudaError_t launch_batch(const StepDesc* steps, int n_steps, const DevPtrs& base, int K, int n_batch, const void* in,
                         void* out, int n_in, int n_out, const int* out_slot, int phys, int prec, cudaStream_t s) {
  PermTab t;
  for (int k = 0; k < 64; ++k) t.slot[k] = (int8_t)(k < n_out ? out_slot[k] : 0);
  const size_t sm = (size_t)(prec == 0 ? 8 : 16) << phys;
  const unsigned grid = (unsigned)std::min(n_batch, 148 * 16);
  if (prec == 0) {
    cudaFuncSetAttribute(batch_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    batch_kernel<float><<<grid, 128, sm, s>>>(steps, n_steps, base, K, n_batch, (const double2*)in, (double2*)out,
                                              n_in, n_out, t);
  } else {
    cudaFuncSetAttribute(batch_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    batch_kernel<double><<<grid, 128, sm, s>>>(steps, n_steps, base, K, n_batch, (const double2*)in, (double2*)out,
                                               n_in, n_out, t);
  }
  return cudaGetLastError();
}

cudaError_t launch_permute_out(const void* state, int prec, void* out, int out_prec, int nbits, const int* slots,
                               uint64_t j0, uint64_t count, cudaStream_t s) {
  PermPlan pl;
  if (j0 == 0 && count == (1ull << nbits) && !getenv("OWQS_PERMUTE_SCALAR") && make_perm_plan(nbits, slots, pl)) {
    const uint64_t n_tiles = 1ull << (nbits - PERM_T);
    const unsigned b = (unsigned)std::min<uint64_t>(n_tiles, (uint64_t)(g_lim_ready ? g_lim.sm_count * 8 : 1184));
    if (prec == 0 && out_prec == 0) permute_out_tiled_kernel<float, float><<<b, 256, 0, s>>>(state, out, pl, n_tiles);
    else if (prec == 0) permute_out_tiled_kernel<float, double><<<b, 256, 0, s>>>(state, out, pl, n_tiles);
    else if (out_prec == 0) permute_out_tiled_kernel<double, float><<<b, 256, 0, s>>>(state, out, pl, n_tiles);
    else permute_out_tiled_kernel<double, double><<<b, 256, 0, s>>>(state, out, pl, n_tiles);
    return cudaGetLastError();
  }
  PermTab t;
  for (int k = 0; k < 64; ++k) t.slot[k] = (int8_t)(k < nbits ? slots[k] : 0);
  unsigned b = elem_blocks(count);
  if (prec == 0 && out_prec == 0) permute_out_kernel<float, float><<<b, 256, 0, s>>>(state, out, nbits, t, j0, count);
  else if (prec == 0) permute_out_kernel<float, double><<<b, 256, 0, s>>>(state, out, nbits, t, j0, count);
  else if (out_prec == 0) permute_out_kernel<double, float><<<b, 256, 0, s>>>(state, out, nbits, t, j0, count);
  else permute_out_kernel<double, double><<<b, 256, 0, s>>>(state, out, nbits, t, j0, count);
  return cudaGetLastError();
}

// owqs_get_output_sample: out[i] = output amplitude idx[i] (caller order, bit k <-> outputs[k]) for
// the samples this shard owns (global state index G = sum_k bit_k(idx) << slot[k], owned when
// G >> wl == rank); others are left untouched (the caller zero-fills and sums over ranks).
template <typename T>
__global__ void sample_out_kernel(const void* shard, const int64_t* idx, uint64_t n, int nbits, PermTab tab,
                                  uint64_t rank, int wl, double2* out) {
  typedef typename VT<T>::C C;
  const C* st = reinterpret_cast<const C*>(shard);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t y = (uint64_t)idx[i];
    uint64_t G = 0;
    for (int k = 0; k < nbits; ++k) G |= ((y >> k) & 1ull) << tab.slot[k];
    if ((G >> wl) != rank) continue;
    const C v = st[G & ((1ull << wl) - 1)];
    out[i] = make_double2((double)v.x, (double)v.y);
  }
}

cudaError_t launch_sample_out(const void* shard, int prec, const int64_t* idx, uint64_t n, int nbits, const int* slots,
                              uint64_t rank, int wl, void* out, cudaStream_t s) {
  PermTab t;
  for (int k = 0; k < 64; ++k) t.slot[k] = (int8_t)(k < nbits ? slots[k] : 0);
  const unsigned b = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(1024, (n + 255) / 256));
  if (prec == 0) sample_out_kernel<float><<<b, 256, 0, s>>>(shard, idx, n, nbits, t, rank, wl, (double2*)out);
  else sample_out_kernel<double><<<b, 256, 0, s>>>(shard, idx, n, nbits, t, rank, wl, (double2*)out);
  return cudaGetLastError();
}

// Tensor merge of sub-states (PAPER §4.1: "two different sub-states are combined only
// when ..."; the reported output is their tensor product): out[i] = prod_c f_c[pext(i, mask_c)],
// where factor c holds the amplitudes of the output bits set in mask_c (bit k of its index <-> the
// k-th set bit of mask_c, increasing). Factors are complex at the output precision. HBM-bound
// (one write per amplitude; the factors are read through L2).
struct KronArgs {
  const void* f[KRON_MAX];
  uint64_t mask[KRON_MAX];
  int n;
};

template <typename T>
__global__ void kron_merge_kernel(void* out, KronArgs a, uint64_t count) {
  typedef typename VT<T>::C C;
  C* o = reinterpret_cast<C*>(out);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    T re = 1, im = 0;
    for (int c = 0; c < a.n; ++c) {
      uint64_t m = a.mask[c], j = 0;
      for (int k = 0; m; ++k) {
        const int b = __ffsll((long long)m) - 1;
        j |= ((i >> b) & 1ull) << k;
        m &= m - 1;
      }
      const C v = reinterpret_cast<const C*>(a.f[c])[j];
      const T r = re * v.x - im * v.y;
      im = re * v.y + im * v.x;
      re = r;
    }
    o[i] = make_c<T>(re, im);
  }
}

cudaError_t launch_kron_merge(void* out, int prec, const void* const* factors, const uint64_t* masks, int n,
                              uint64_t count, cudaStream_t s) {
  if (n > KRON_MAX) return cudaErrorInvalidValue;
  KronArgs a{};
  for (int c = 0; c < n; ++c) {
    a.f[c] = factors[c];
    a.mask[c] = masks[c];
  }
  a.n = n;
  const unsigned b = elem_blocks(count);
  if (prec == 0) kron_merge_kernel<float><<<b, 256, 0, s>>>(out, a, count);
  else kron_merge_kernel<double><<<b, 256, 0, s>>>(out, a, count);
  return cudaGetLastError();
}

cudaError_t launch_convert_in(const void* src, int src_prec, void* state, int prec, uint64_t j0, uint64_t count, cudaStream_t s) {
  unsigned b = elem_blocks(count);
  if (src_prec == 0 && prec == 0) convert_in_kernel<float, float><<<b, 256, 0, s>>>(src, state, j0, count);
  else if (src_prec == 0) convert_in_kernel<float, double><<<b, 256, 0, s>>>(src, state, j0, count);
  else if (prec == 0) convert_in_kernel<double, float><<<b, 256, 0, s>>>(src, state, j0, count);
  else convert_in_kernel<double, double><<<b, 256, 0, s>>>(src, state, j0, count);
  return cudaGetLastError();
}

cudaError_t launch_basis(void* state, int prec, uint64_t n, uint64_t k, cudaStream_t s) {
  unsigned b = elem_blocks(n);
  if (prec == 0) basis_kernel<float><<<b, 256, 0, s>>>(state, n, k);
  else basis_kernel<double><<<b, 256, 0, s>>>(state, n, k);
  return cudaGetLastError();
}

// Haar input (unnormalised, norm^2 into red_result) for amplitudes [j0, j0 + n) of the global state
cudaError_t launch_haar(const DevPtrs& p, int prec, uint64_t n, uint64_t seed, uint64_t j0, cudaStream_t s) {
  unsigned b = elem_blocks(n);
  if (prec == 0) haar_kernel<float><<<b, 256, 0, s>>>(p, n, seed, j0);
  else haar_kernel<double><<<b, 256, 0, s>>>(p, n, seed, j0);
  return cudaGetLastError();
}

cudaError_t launch_scale(const DevPtrs& p, int prec, uint64_t n, cudaStream_t s) {
  unsigned b = elem_blocks(n);
  if (prec == 0) scale_kernel<float><<<b, 256, 0, s>>>(p.state, n, p.red_result);
  else scale_kernel<double><<<b, 256, 0, s>>>(p.state, n, p.red_result);
  return cudaGetLastError();
}

// norm^2 of a shard into red_result[0] (read-only pass through the pass kernel machinery)
template <typename T>
__global__ void __launch_bounds__(256) norm_kernel(DevPtrs p, uint64_t n) {
  typedef typename VT<T>::C C;
  __shared__ PassShared sh;
  const C* st = reinterpret_cast<const C*>(p.state);
  double acc[4] = {0, 0, 0, 0};
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    C v = st[i];
    acc[0] += (double)v.x * v.x + (double)v.y * v.y;
  }
  reduce_finish<1>(acc, p, sh);
}

// Small readbacks (error flags, outcomes, prob0, reductions, the input norm) into page-locked host
// memory written by the SMs over PCIe (UVA: cudaMallocHost memory is mapped at the same address)
// instead of a copy-engine cudaMemcpyAsync: a D2H copy queues behind other contexts' multi-GiB
// output DMAs in the copy engine, and everything behind it on this stream (the run after the input
// norm check, the output permutation) waits with it (e2e pipeline: 69.9 ms per C3 step).
__global__ void readback_kernel(unsigned char* dst, const unsigned char* src, size_t n) {
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
}

cudaError_t launch_readback(void* host_dst, const void* dev_src, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  readback_kernel<<<1, 256, 0, s>>>(static_cast<unsigned char*>(host_dst), static_cast<const unsigned char*>(dev_src), n);
  return cudaGetLastError();
}

cudaError_t launch_norm(const DevPtrs& p, int prec, uint64_t n, cudaStream_t s) {
  if (prec == 0) norm_kernel<float><<<elem_blocks(n), 256, 0, s>>>(p, n);
  else norm_kernel<double><<<elem_blocks(n), 256, 0, s>>>(p, n);
  return cudaGetLastError();
}

// Caller input into a shard with its norm^2 in the same sweep (owqs_set_input_device, same
// precision): state[i] = src[i], red_result[0] = sum |src[i]|^2 (fp64). The structural decisions take
// ||psi||^2 = 1 (DESIGN R-13, Eq. 3-4 / P:L105-109), so the library checks it on every input.
template <typename T>
__global__ void __launch_bounds__(256) copy_norm_kernel(DevPtrs p, const void* src, uint64_t n) {
  typedef typename VT<T>::C C;
  __shared__ PassShared sh;
  const C* x = reinterpret_cast<const C*>(src);
  C* st = reinterpret_cast<C*>(p.state);
  double acc[4] = {0, 0, 0, 0};
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const C v = __ldcs(x + i);
    __stcs(st + i, v);
    acc[0] += (double)v.x * v.x + (double)v.y * v.y;
  }
  reduce_finish<1>(acc, p, sh);
}

cudaError_t launch_copy_norm(const DevPtrs& p, int prec, const void* src, uint64_t n, cudaStream_t s) {
  if (prec == 0) copy_norm_kernel<float><<<elem_blocks(n), 256, 0, s>>>(p, src, n);
  else copy_norm_kernel<double><<<elem_blocks(n), 256, 0, s>>>(p, src, n);
  return cudaGetLastError();
}

// <a|b> of two same-precision shards into red_result[0..1]
template <typename T>
__global__ void __launch_bounds__(256) dot_t_kernel(DevPtrs p, const void* a, const void* b, uint64_t n) {
  typedef typename VT<T>::C C;
  __shared__ PassShared sh;
  const C* x = reinterpret_cast<const C*>(a);
  const C* y = reinterpret_cast<const C*>(b);
  double acc[4] = {0, 0, 0, 0};
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    C u = x[i], v = y[i];
    acc[0] += (double)u.x * v.x + (double)u.y * v.y;
    acc[1] += (double)u.x * v.y - (double)u.y * v.x;
  }
  reduce_finish<2>(acc, p, sh);
}

cudaError_t launch_dot_t(const DevPtrs& p, int prec, const void* a, const void* b, uint64_t n, cudaStream_t s) {
  if (prec == 0) dot_t_kernel<float><<<elem_blocks(n), 256, 0, s>>>(p, a, b, n);
  else dot_t_kernel<double><<<elem_blocks(n), 256, 0, s>>>(p, a, b, n);
  return cudaGetLastError();
}

cudaError_t launch_dot(const DevPtrs& p, const void* a, const void* b, uint64_t n, cudaStream_t s) {
  dot_kernel<<<elem_blocks(n), 256, 0, s>>>(p, (const double2*)a, (const double2*)b, n);
  return cudaGetLastError();
}

}  // namespace owqs
