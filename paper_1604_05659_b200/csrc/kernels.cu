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

#include <algorithm>

#include "owqs_internal.h"

namespace owqs {

#define FULLMASK 0xffffffffu

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Reading R-5: keyed uniform draw of the M with given-order ordinal `ord`.
__device__ __forceinline__ double draw_uniform(uint64_t seed, int ord) {
  return (double)(splitmix64(seed ^ splitmix64((uint64_t)(int64_t)ord)) >> 11) * 0x1.0p-53;
}

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
// Measurement decision (one thread). Eq. 2 angle, prob0 by Eq. 13 (structural or from rho),
// outcome by Fig. 6 "rand(0,1) <= prob" / forced / EOWQS 0, coefficients of Eqs. 11-12.
// ------------------------------------------------------------------------------------------------
struct LocalOutcomes {
  int n;
  int ord[MAX_BFLY];
  uint8_t out[MAX_BFLY];
};

__device__ int signal_parity(const DevPtrs& p, int off, int len, const LocalOutcomes& loc) {
  int s = 0;
  for (int i = 0; i < len; ++i) {
    int o = p.sig_pool[off + i];
    int v = -1;
    for (int j = 0; j < loc.n; ++j)
      if (loc.ord[j] == o) v = loc.out[j];
    if (v < 0) v = p.outcome[o];
    s ^= v;
  }
  return s & 1;
}

// Writes the 2x2 complex matrix (row-major re/im pairs) to coef[8]. For an elimination (reuse=0)
// only row 0 is used. red: NORM -> red[0] = ||psi||^2; RHO -> (n0, n1, Re c, Im c).
__device__ void decide(const DevPtrs& p, int m, bool use_red, bool full, bool record, double* coef,
                       LocalOutcomes& loc) {
  const MStatic ms = p.mst[m];
  const int mode = p.run->mode;
  int s = 0, t = 0;
  if (mode != 2) {
    s = signal_parity(p, ms.s_off, ms.s_len, loc);
    t = signal_parity(p, ms.t_off, ms.t_len, loc);
  }
  const double PI = 3.141592653589793238462643383279502884;
  double theta = (s ? -ms.alpha : ms.alpha) + (t ? PI : 0.0);  // Eq. 2
  double sn, cs;
  sincos(theta, &sn, &cs);
  const double er = cs, ei = -sn;  // e^{-i theta}
  int outc = 0;
  double pS = 0.5, P0 = -1.0;
  if (mode != 2) {
    double P1;
    if (full) {  // prob0 = 1/2 sum |x0 + e^{-i theta} x1|^2 = (n0 + n1)/2 + Re(e^{-i theta} c)
      const double* r = p.red_result;
      double tot = r[0] + r[1];
      P0 = 0.5 * tot + (er * r[2] - ei * r[3]);
      P0 = fmin(fmax(P0, 0.0), tot);
      P1 = tot - P0;
    } else {  // a fresh |+> neighbour dephases the qubit: prob0 = ||psi||^2 / 2 (R-13)
      double nrm = use_red ? p.red_result[0] : 1.0;
      P0 = 0.5 * nrm;
      P1 = 0.5 * nrm;
    }
    if (mode == 0) {
      outc = draw_uniform(p.run->seed, ms.ord) <= P0 ? 0 : 1;
    } else {
      outc = p.forced[ms.ord] & 1;
    }
    pS = outc ? P1 : P0;
    if (pS < 1e-12) {
      if (record) atomicExch(p.err, 1);
      pS = 1.0;
    }
  }
  const double sg = outc ? -1.0 : 1.0;
  if (ms.reuse) {
    // N_o E_io M_i: out[y] = (x0 + (-1)^{s+y} e^{-i theta} x1) / (2 sqrt(p_s)); EOWQS: sqrt2 * 1/2
    double k = (mode == 2) ? 0.70710678118654752440 : 0.5 / sqrt(pS);
    coef[0] = k; coef[1] = 0; coef[2] = k * sg * er; coef[3] = k * sg * ei;
    coef[4] = k; coef[5] = 0; coef[6] = -k * sg * er; coef[7] = -k * sg * ei;
  } else {
    // M_s of Eqs. 11-12: out = (x0 + (-1)^s e^{-i theta} x1) / (sqrt2 sqrt(p_s)); EOWQS: * sqrt2
    double k = (mode == 2) ? 1.0 : 1.0 / sqrt(2.0 * pS);
    coef[0] = k; coef[1] = 0; coef[2] = k * sg * er; coef[3] = k * sg * ei;
    coef[4] = 0; coef[5] = 0; coef[6] = 0; coef[7] = 0;
  }
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

// Prologue shared by the pass kernels: decisions of the pass's butterflies and op conditions.
struct PassShared {
  double coef[MAX_BFLY][8];
  uint8_t cond[MAX_OPS];
  uint8_t bidx[MAX_OPS];
  double red[32][4];
  int last;
};

__device__ void pass_prologue(const StepDesc& d, const DevPtrs& p, PassShared& sh) {
  if (threadIdx.x == 0) {
    LocalOutcomes loc;
    loc.n = 0;
    int bi = 0;
    const bool record = blockIdx.x == 0;
    for (int i = 0; i < d.n_ops; ++i) {
      const Op& op = d.ops[i];
      if (op.type == OP_BFLY) {
        decide(p, op.m, bi == 0 && d.first_uses_red, false, record, sh.coef[bi], loc);
        sh.bidx[i] = (uint8_t)bi++;
        sh.cond[i] = 1;
      } else {
        sh.cond[i] = op.cond ? (uint8_t)signal_parity(p, op.sig_off, op.sig_len, loc) : (uint8_t)1;
      }
    }
  }
  __syncthreads();
}

// Block reduction of up to 4 doubles; the last block to finish reduces all block partials in a
// fixed order (deterministic) into red_result and resets the counter.
template <int NRED>
__device__ void reduce_finish(double (&acc)[4], const DevPtrs& p, PassShared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NRED; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(FULLMASK, acc[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NRED; ++k) sh.red[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot[4] = {0, 0, 0, 0};
    for (int w = 0; w < nw; ++w)
      for (int k = 0; k < NRED; ++k) tot[k] += sh.red[w][k];
    for (int k = 0; k < NRED; ++k) p.partials[(size_t)blockIdx.x * 4 + k] = tot[k];
    __threadfence();
    unsigned t = atomicAdd(p.counter, 1u);
    sh.last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!sh.last) return;
  __threadfence();
  double s[4] = {0, 0, 0, 0};
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
    for (int k = 0; k < NRED; ++k) s[k] += __ldcg(&p.partials[(size_t)b * 4 + k]);
#pragma unroll
  for (int k = 0; k < NRED; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[k] += __shfl_xor_sync(FULLMASK, s[k], o);
  __syncthreads();
  if (lane == 0)
    for (int k = 0; k < NRED; ++k) sh.red[warp][k] = s[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot[4] = {0, 0, 0, 0};
    for (int w = 0; w < nw; ++w)
      for (int k = 0; k < NRED; ++k) tot[k] += sh.red[w][k];
    for (int k = 0; k < 4; ++k) p.red_result[k] = k < NRED ? tot[k] : 0.0;
    *p.counter = 0;
  }
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

template <typename T, int KHI, int UNR>
__global__ void __launch_bounds__(256) pass_kernel(const StepDesc d, const DevPtrs p) {
  typedef typename VT<T>::V V;
  constexpr int SB = VT<T>::SB, EPV = VT<T>::EPV;
  constexpr int G = 1 << KHI;
  constexpr int NV = UNR * G;
  __shared__ PassShared sh;
  pass_prologue(d, p, sh);

  const int lane = threadIdx.x & 31;
  const uint64_t warp_id = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t n_units = (1ull << (d.width - SB - KHI)) / UNR;
  int q[KHI > 0 ? KHI : 1];
#pragma unroll
  for (int j = 0; j < KHI; ++j) q[j] = d.bhi[j] - SB;
  V* st = reinterpret_cast<V*>(p.state);
  double acc[4] = {0, 0, 0, 0};
  const bool do_store = d.n_ops > 0;

  for (uint64_t unit = warp_id; unit < n_units; unit += n_warps) {
    uint64_t seg[NV];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      uint64_t g = unit * UNR + u;
#pragma unroll
      for (int j = 0; j < KHI; ++j) g = ((g >> q[j]) << (q[j] + 1)) | (g & ((1ull << q[j]) - 1));
#pragma unroll
      for (int c = 0; c < G; ++c) {
        uint64_t s = g;
#pragma unroll
        for (int j = 0; j < KHI; ++j)
          if ((c >> j) & 1) s |= 1ull << q[j];
        seg[u * G + c] = s;
      }
    }
    T re[NV][2], im[NV][2];
#pragma unroll
    for (int v = 0; v < NV; ++v) vload<T>(st + seg[v] * 32 + lane, re[v], im[v]);

    for (int i = 0; i < d.n_ops; ++i) {
      const Op op = d.ops[i];
      if (!sh.cond[i]) continue;
      if (op.type == OP_DIAG_E || op.type == OP_DIAG_Z) {
        const int a = op.a, b = op.type == OP_DIAG_E ? op.b : op.a;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int e = 0; e < EPV; ++e) {
            uint64_t idx = (seg[v] << SB) | (uint64_t)(lane * EPV + e);
            if ((idx >> a) & (idx >> b) & 1) {
              re[v][e] = -re[v][e];
              im[v][e] = -im[v][e];
            }
          }
      } else {
        // 2x2 on slot a: butterfly coefficients or X swap
        const int a = op.a;
        T c00r, c00i, c01r, c01i, c10r, c10i, c11r, c11i;
        if (op.type == OP_BFLY) {
          const double* cf = sh.coef[sh.bidx[i]];
          c00r = (T)cf[0]; c00i = (T)cf[1]; c01r = (T)cf[2]; c01i = (T)cf[3];
          c10r = (T)cf[4]; c10i = (T)cf[5]; c11r = (T)cf[6]; c11i = (T)cf[7];
        } else {
          c00r = 0; c00i = 0; c01r = 1; c01i = 0; c10r = 1; c10i = 0; c11r = 0; c11i = 0;
        }
        if (a >= SB) {
          const int qa = a - SB;
#pragma unroll
          for (int jj = 0; jj < KHI; ++jj) {
            if (q[jj] != qa) continue;
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
              for (int c = 0; c < G; ++c) {
                if ((c >> jj) & 1) continue;
                const int v0 = u * G + c, v1 = v0 + (1 << jj);
#pragma unroll
                for (int e = 0; e < EPV; ++e) {
                  T x0r = re[v0][e], x0i = im[v0][e], x1r = re[v1][e], x1i = im[v1][e];
                  cmul_add(c00r, c00i, x0r, x0i, c01r, c01i, x1r, x1i, re[v0][e], im[v0][e]);
                  cmul_add(c10r, c10i, x0r, x0i, c11r, c11i, x1r, x1i, re[v1][e], im[v1][e]);
                }
              }
          }
        } else if (EPV == 2 && a == 0) {
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            T x0r = re[v][0], x0i = im[v][0], x1r = re[v][1], x1i = im[v][1];
            cmul_add(c00r, c00i, x0r, x0i, c01r, c01i, x1r, x1i, re[v][0], im[v][0]);
            cmul_add(c10r, c10i, x0r, x0i, c11r, c11i, x1r, x1i, re[v][1], im[v][1]);
          }
        } else {
          const int lb = a - (EPV == 2 ? 1 : 0);
          const bool hi = (lane >> lb) & 1;
          // mine * cA + partner * cB
          const T aR = hi ? c11r : c00r, aI = hi ? c11i : c00i;
          const T bR = hi ? c10r : c01r, bI = hi ? c10i : c01i;
#pragma unroll
          for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int e = 0; e < EPV; ++e) {
              T pr = __shfl_xor_sync(FULLMASK, re[v][e], 1 << lb);
              T pi = __shfl_xor_sync(FULLMASK, im[v][e], 1 << lb);
              T mr = re[v][e], mi = im[v][e];
              cmul_add(aR, aI, mr, mi, bR, bI, pr, pi, re[v][e], im[v][e]);
            }
        }
      }
    }

    if (d.red_kind == RED_NORM) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < EPV; ++e)
          acc[0] += (double)re[v][e] * re[v][e] + (double)im[v][e] * im[v][e];
    } else if (d.red_kind == RED_RHO) {
      const int r = d.red_slot;
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < EPV; ++e) {
          uint64_t idx = (seg[v] << SB) | (uint64_t)(lane * EPV + e);
          double n = (double)re[v][e] * re[v][e] + (double)im[v][e] * im[v][e];
          if ((idx >> r) & 1) acc[1] += n; else acc[0] += n;
        }
      // c = sum conj(x0) x1 over pairs split on slot r
      if (r >= SB) {
        const int qr = r - SB;
#pragma unroll
        for (int jj = 0; jj < KHI; ++jj) {
          if (q[jj] != qr) continue;
#pragma unroll
          for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int c = 0; c < G; ++c) {
              if ((c >> jj) & 1) continue;
              const int v0 = u * G + c, v1 = v0 + (1 << jj);
#pragma unroll
              for (int e = 0; e < EPV; ++e) {
                double x0r = re[v0][e], x0i = im[v0][e], x1r = re[v1][e], x1i = im[v1][e];
                acc[2] += x0r * x1r + x0i * x1i;
                acc[3] += x0r * x1i - x0i * x1r;
              }
            }
        }
      } else if (EPV == 2 && r == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double x0r = re[v][0], x0i = im[v][0], x1r = re[v][1], x1i = im[v][1];
          acc[2] += x0r * x1r + x0i * x1i;
          acc[3] += x0r * x1i - x0i * x1r;
        }
      } else {
        const int lb = r - (EPV == 2 ? 1 : 0);
        const bool hi = (lane >> lb) & 1;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int e = 0; e < EPV; ++e) {
            T pr = __shfl_xor_sync(FULLMASK, re[v][e], 1 << lb);
            T pi = __shfl_xor_sync(FULLMASK, im[v][e], 1 << lb);
            if (!hi) {
              double x0r = re[v][e], x0i = im[v][e], x1r = pr, x1i = pi;
              acc[2] += x0r * x1r + x0i * x1i;
              acc[3] += x0r * x1i - x0i * x1r;
            }
          }
      }
    }

    if (do_store) {
#pragma unroll
      for (int v = 0; v < NV; ++v) vstore<T>(st + seg[v] * 32 + lane, re[v], im[v]);
    }
  }
  if (d.red_kind == RED_NORM) reduce_finish<1>(acc, p, sh);
  else if (d.red_kind == RED_RHO) reduce_finish<4>(acc, p, sh);
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
  for (int k = 0; k < d.n_ops; ++k) {
    const Op op = d.ops[k];
    if (!sh.cond[k]) continue;
    if (op.type == OP_DIAG_E || op.type == OP_DIAG_Z) {
      const int a = op.a, b = op.type == OP_DIAG_E ? op.b : op.a;
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        if ((i >> a) & (i >> b) & 1) {
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
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        int i0 = ((i >> a) << (a + 1)) | (i & ((1 << a) - 1));
        int i1 = i0 | (1 << a);
        T x0r = s[i0].x, x0i = s[i0].y, x1r = s[i1].x, x1i = s[i1].y;
        T o0r, o0i, o1r, o1i;
        cmul_add<T>((T)cf[0], (T)cf[1], x0r, x0i, (T)cf[2], (T)cf[3], x1r, x1i, o0r, o0i);
        cmul_add<T>((T)cf[4], (T)cf[5], x0r, x0i, (T)cf[6], (T)cf[7], x1r, x1i, o1r, o1i);
        s[i0].x = o0r; s[i0].y = o0i; s[i1].x = o1r; s[i1].y = o1i;
      }
    }
    __syncthreads();
  }
  double acc[4] = {0, 0, 0, 0};
  if (d.red_kind == RED_NORM) {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      acc[0] += (double)s[i].x * s[i].x + (double)s[i].y * s[i].y;
  } else if (d.red_kind == RED_RHO) {
    const int r = d.red_slot;
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
  if (d.n_ops > 0)
    for (int i = threadIdx.x; i < n; i += blockDim.x) st[i] = s[i];
  if (d.red_kind == RED_NORM) reduce_finish<1>(acc, p, sh);
  else if (d.red_kind == RED_RHO) reduce_finish<4>(acc, p, sh);
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
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    C v = st[i];
    v.x *= r;
    v.y *= r;
    st[i] = v;
    st[i + n] = v;
    acc[0] += 2.0 * ((double)v.x * v.x + (double)v.y * v.y);
  }
  if (d.red_kind == RED_NORM) reduce_finish<1>(acc, p, sh);
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

struct PermTab {
  int8_t slot[64];
};

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
__global__ void __launch_bounds__(256) haar_kernel(DevPtrs p, uint64_t n, uint64_t seed) {
  typedef typename VT<T>::C C;
  __shared__ PassShared sh;
  C* st = reinterpret_cast<C*>(p.state);
  const uint64_t key = splitmix64(seed);
  double acc[4] = {0, 0, 0, 0};
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t a = splitmix64(key ^ splitmix64(2 * j));
    uint64_t b = splitmix64(key ^ splitmix64(2 * j + 1));
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
  int max_blocks_pass[2][KMAX_HI + 1];
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
  void* fns[2][KMAX_HI + 1] = {
      {pass_fn<float, 0, 4>(), pass_fn<float, 1, 2>(), pass_fn<float, 2, 1>(), pass_fn<float, 3, 1>(), pass_fn<float, 4, 1>()},
      {pass_fn<double, 0, 4>(), pass_fn<double, 1, 2>(), pass_fn<double, 2, 1>(), pass_fn<double, 3, 1>(), pass_fn<double, 4, 1>()}};
  for (int pr = 0; pr < 2; ++pr)
    for (int k = 0; k <= KMAX_HI; ++k) {
      int nb = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fns[pr][k], 256, 0);
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

int max_partial_blocks() { return 16 * 148 * 2; }

static inline int unr_of(int khi) { return khi == 0 ? 4 : (khi == 1 ? 2 : 1); }
static inline int log2i(int x) { int r = 0; while ((1 << r) < x) ++r; return r; }

// Kernel class of a step (OWQS_KCLASS_* of include/owqs.h).
int step_kclass(const StepDesc& d, int prec) {
  const int SB = prec == 0 ? 6 : 5;
  if (d.kind == ST_GROW) return 2;
  if (d.kind == ST_SHRINK) return 3;
  const int slack = d.width - SB - d.nb_hi - log2i(unr_of(d.nb_hi));
  if (slack < 0) return 1;
  return d.n_ops == 0 ? 4 : 0;
}

// Launch one step. prec: 0 complex64, 1 complex128.
cudaError_t launch_step(const StepDesc& d, const DevPtrs& p, int prec, cudaStream_t s) {
  const int SB = prec == 0 ? 6 : 5;
  if (d.kind == ST_PASS) {
    const int khi = d.nb_hi;
    const int unr = unr_of(khi);
    const int slack = d.width - SB - khi - log2i(unr);
    if (slack < 0) {
      if (d.width > 12) return cudaErrorInvalidValue;
      size_t sm = (size_t)(prec == 0 ? 8 : 16) << d.width;
      if (prec == 0) small_pass_kernel<float><<<1, 512, sm, s>>>(d, p);
      else small_pass_kernel<double><<<1, 512, sm, s>>>(d, p);
      return cudaGetLastError();
    }
    const uint64_t units = 1ull << slack;
    uint64_t blocks = (units + 7) / 8;
    blocks = std::min<uint64_t>(blocks, (uint64_t)g_lim.max_blocks_pass[prec][khi]);
    dim3 grid((unsigned)blocks), blk(256);
#define OWQS_PASS(T, K, U) pass_kernel<T, K, U><<<grid, blk, 0, s>>>(d, p)
    if (prec == 0) {
      switch (khi) {
        case 0: OWQS_PASS(float, 0, 4); break;
        case 1: OWQS_PASS(float, 1, 2); break;
        case 2: OWQS_PASS(float, 2, 1); break;
        case 3: OWQS_PASS(float, 3, 1); break;
        default: OWQS_PASS(float, 4, 1); break;
      }
    } else {
      switch (khi) {
        case 0: OWQS_PASS(double, 0, 4); break;
        case 1: OWQS_PASS(double, 1, 2); break;
        case 2: OWQS_PASS(double, 2, 1); break;
        case 3: OWQS_PASS(double, 3, 1); break;
        default: OWQS_PASS(double, 4, 1); break;
      }
    }
#undef OWQS_PASS
    return cudaGetLastError();
  }
  uint64_t work = d.kind == ST_GROW ? (1ull << d.width) : (1ull << std::max(0, d.width - (d.slot == d.width - 1 ? 1 : 2)));
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

cudaError_t launch_permute_out(const void* state, int prec, void* out, int out_prec, int nbits, const int* slots,
                               uint64_t j0, uint64_t count, cudaStream_t s) {
  PermTab t;
  for (int k = 0; k < 64; ++k) t.slot[k] = (int8_t)(k < nbits ? slots[k] : 0);
  unsigned b = elem_blocks(count);
  if (prec == 0 && out_prec == 0) permute_out_kernel<float, float><<<b, 256, 0, s>>>(state, out, nbits, t, j0, count);
  else if (prec == 0) permute_out_kernel<float, double><<<b, 256, 0, s>>>(state, out, nbits, t, j0, count);
  else if (out_prec == 0) permute_out_kernel<double, float><<<b, 256, 0, s>>>(state, out, nbits, t, j0, count);
  else permute_out_kernel<double, double><<<b, 256, 0, s>>>(state, out, nbits, t, j0, count);
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

cudaError_t launch_haar(const DevPtrs& p, int prec, uint64_t n, uint64_t seed, cudaStream_t s) {
  unsigned b = elem_blocks(n);
  if (prec == 0) {
    haar_kernel<float><<<b, 256, 0, s>>>(p, n, seed);
    scale_kernel<float><<<b, 256, 0, s>>>(p.state, n, p.red_result);
  } else {
    haar_kernel<double><<<b, 256, 0, s>>>(p, n, seed);
    scale_kernel<double><<<b, 256, 0, s>>>(p.state, n, p.red_result);
  }
  return cudaGetLastError();
}

cudaError_t launch_dot(const DevPtrs& p, const void* a, const void* b, uint64_t n, cudaStream_t s) {
  dot_kernel<<<elem_blocks(n), 256, 0, s>>>(p, (const double2*)a, (const double2*)b, n);
  return cudaGetLastError();
}

}  // namespace owqs
