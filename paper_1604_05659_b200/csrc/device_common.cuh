// Device code shared by the ahead-of-time kernels (kernels.cu) and the pass kernels generated at
// load time (jit.cpp embeds this file verbatim in every NVRTC translation unit): the measurement
// decision of a pass (Eq. 2 angle, Eq. 13 prob0, Fig. 6 outcome, Eqs. 11-12 coefficients), the
// pass prologue and the deterministic grid reduction.
#pragma once
#ifndef __CUDACC_RTC__
#include <stdint.h>
#endif

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
      outc = draw_uniform(p.run->seed, ms.key) <= P0 ? 0 : 1;
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
  double ka[MAX_BFLY][2];  // structured butterfly U = k [[1, a], [1, -a]]: a (k folded into scale)
  double kk[MAX_BFLY];     // k of each butterfly
  double scale;            // product of the pass's butterfly k's
  uint8_t cond[MAX_OPS];
  uint8_t bidx[MAX_OPS];
  uint8_t bop[MAX_BFLY];   // op index of butterfly b
  int32_t lord[MAX_BFLY];  // given-order ordinal decided by butterfly b
  uint8_t lout[MAX_BFLY];  // its outcome
  double red[32][4];
  int last;
};

// parity of a signal domain: outcomes decided in this pass (lord / lout) or in earlier steps
__device__ __forceinline__ int signal_parity_sh(const DevPtrs& p, int off, int len, const PassShared& sh, int nb) {
  int s = 0;
  for (int i = 0; i < len; ++i) {
    const int o = p.sig_pool[off + i];
    int v = -1;
    for (int j = 0; j < nb; ++j)
      if (sh.lord[j] == o) v = sh.lout[j];
    if (v < 0) v = p.outcome[o];
    s ^= v;
  }
  return s & 1;
}

// Warp 0 decides every butterfly of the pass in parallel (lane b <-> butterfly b). Inside a pass
// every measurement has a fresh |+> neighbour, so prob0 = ||psi||^2 / 2 (reading R-13) does not
// depend on the angle: all outcomes are decided first (Fig. 6 "rand(0,1) <= prob", forced, or 0 in
// EOWQS), then the signal parities of Eq. 2 (which may reference outcomes of this same pass), then
// angles and the Eqs. 11-12 coefficients. Same values as the sequential decide() loop.
__device__ void pass_prologue(const StepDesc& d, const DevPtrs& p, PassShared& sh, bool record_all = false) {
  static_assert(MAX_BFLY <= 64, "two butterflies per lane");
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const bool record = record_all || blockIdx.x == 0;
    const int mode = p.run->mode;
    // butterfly numbering (ops order)
    int nb = 0;
    for (int base = 0; base < d.n_ops; base += 32) {
      const int i = base + lane;
      const bool isb = i < d.n_ops && d.ops[i].type == OP_BFLY;
      const unsigned bal = __ballot_sync(FULLMASK, isb);
      if (isb) {
        const int b = nb + __popc(bal & ((1u << lane) - 1u));
        sh.bidx[i] = (uint8_t)b;
        sh.bop[b] = (uint8_t)i;
      }
      nb += __popc(bal);
    }
    __syncwarp();
    // 1. outcomes (lane handles butterflies lane and lane + 32)
    double P0[2] = {-1.0, -1.0}, pS[2] = {0.5, 0.5};
    int outc[2] = {0, 0};
    MStatic ms[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int b = lane + 32 * h;
      if (b >= nb) continue;
      const Op& op = d.ops[sh.bop[b]];
      ms[h] = p.mst[op.m];
      if (mode != 2) {
        const double nrm = (b == 0 && d.first_uses_red) ? p.red_result[0] : 1.0;
        P0[h] = 0.5 * nrm;
        const double P1 = 0.5 * nrm;
        outc[h] = mode == 0 ? (draw_uniform(p.run->seed, ms[h].key) <= P0[h] ? 0 : 1) : (p.forced[ms[h].ord] & 1);
        pS[h] = outc[h] ? P1 : P0[h];
        if (pS[h] < 1e-12) {
          if (record) atomicExch(p.err, 1);
          pS[h] = 1.0;
        }
      }
      sh.lord[b] = ms[h].ord;
      sh.lout[b] = (uint8_t)outc[h];
    }
    __syncwarp();
    // 2. signals, angle, coefficients
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int b = lane + 32 * h;
      if (b >= nb) continue;
      const Op& op = d.ops[sh.bop[b]];
      int s = 0, t = 0;
      if (mode != 2) {
        s = signal_parity_sh(p, ms[h].s_off, ms[h].s_len, sh, nb);
        t = signal_parity_sh(p, ms[h].t_off, ms[h].t_len, sh, nb);
      }
      const double PI = 3.141592653589793238462643383279502884;
      const double theta = (s ? -ms[h].alpha : ms[h].alpha) + (t ? PI : 0.0);  // Eq. 2
      double sn, cs;
      sincos(theta, &sn, &cs);
      const double er = cs, ei = -sn;  // e^{-i theta}
      const double sg = outc[h] ? -1.0 : 1.0;
      double* cf = sh.coef[b];
      double k;
      if (ms[h].reuse) {  // N_o E_io M_i: out[y] = (x0 + (-1)^{s+y} e^{-i theta} x1) / (2 sqrt(p_s))
        k = (mode == 2) ? 0.70710678118654752440 : 0.5 / sqrt(pS[h]);
        cf[0] = k; cf[1] = 0; cf[2] = k * sg * er; cf[3] = k * sg * ei;
        cf[4] = k; cf[5] = 0; cf[6] = -k * sg * er; cf[7] = -k * sg * ei;
      } else {  // M_s of Eqs. 11-12
        k = (mode == 2) ? 1.0 : 1.0 / sqrt(2.0 * pS[h]);
        cf[0] = k; cf[1] = 0; cf[2] = k * sg * er; cf[3] = k * sg * ei;
        cf[4] = 0; cf[5] = 0; cf[6] = 0; cf[7] = 0;
      }
      // folded X_a^s of the butterfly: swap the output rows when the signal is 1
      if (op.cond && signal_parity_sh(p, op.sig_off, op.sig_len, sh, nb))
        for (int j = 0; j < 4; ++j) {
          const double tt = cf[j];
          cf[j] = cf[4 + j];
          cf[4 + j] = tt;
        }
      const double kk = cf[0];
      sh.ka[b][0] = kk != 0.0 ? cf[2] / kk : 0.0;
      sh.ka[b][1] = kk != 0.0 ? cf[3] / kk : 0.0;
      sh.kk[b] = kk;
      if (record) {
        p.outcome[ms[h].ord] = (uint8_t)outc[h];
        p.prob0[ms[h].ord] = P0[h];
      }
    }
    // 3. conditions of the other ops
    for (int i = lane; i < d.n_ops; i += 32) {
      const Op& op = d.ops[i];
      if (op.type == OP_BFLY)
        sh.cond[i] = 1;
      else
        sh.cond[i] = op.cond ? (uint8_t)signal_parity_sh(p, op.sig_off, op.sig_len, sh, nb) : (uint8_t)1;
    }
    __syncwarp();
    if (lane == 0) {
      double scale = 1.0;
      for (int b = 0; b < nb; ++b) scale *= sh.kk[b];
      sh.scale = scale;
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

// Block partial of up to 4 doubles into p.partials[blockIdx.x * 4 + k] (no fence, no atomics: the
// grid's partials are summed in a fixed order by grid_finish_kernel launched right after the pass,
// so a CTA retires without waiting for its own outstanding state stores to drain).
template <int NRED>
__device__ void block_partial(double (&acc)[4], const DevPtrs& p, double (*red)[4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NRED; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(FULLMASK, acc[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NRED; ++k) red[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < NRED) {
    double t = 0;
    for (int w = 0; w < nw; ++w) t += red[w][threadIdx.x];
    p.partials[(size_t)blockIdx.x * 4 + threadIdx.x] = t;
  }
}

// Deterministic two-level grid reduction of up to 4 doubles for grids of up to RED_MAX_BLOCKS
// blocks (the generated pass kernels launch one block per 8 warp units): block partials ->
// the last block of each group of RED_GROUP blocks sums its group in a fixed order -> the last
// group sums the group partials in a fixed order into red_result. Counters are reset by their
// last user. red: shared [32][4] scratch, flag: shared int.
template <int NRED>
__device__ void reduce_finish_grid(double (&acc)[4], const DevPtrs& p, double (*red)[4], int* flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned blk = blockIdx.x, nblk = gridDim.x;
  const unsigned g = blk / RED_GROUP, g0 = g * RED_GROUP;
  const unsigned gsz = min((unsigned)RED_GROUP, nblk - g0);
  const unsigned ngroups = (nblk + RED_GROUP - 1) / RED_GROUP;
  double* gpart = p.partials + (size_t)RED_MAX_BLOCKS * 4;
  auto block_sum = [&](double (&v)[4], double* out) {
#pragma unroll
    for (int k = 0; k < NRED; ++k)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(FULLMASK, v[k], o);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < NRED; ++k) red[warp][k] = v[k];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < NRED; ++k) {
        double t = 0;
        for (int w = 0; w < nw; ++w) t += red[w][k];
        out[k] = t;
      }
  };
  block_sum(acc, p.partials + (size_t)blk * 4);
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(&p.counter[1 + g], 1u);
    *flag = (t == gsz - 1);
  }
  __syncthreads();
  if (!*flag) return;
  __threadfence();
  double v[4] = {0, 0, 0, 0};
  for (unsigned b = threadIdx.x; b < gsz; b += blockDim.x)
    for (int k = 0; k < NRED; ++k) v[k] += __ldcg(&p.partials[(size_t)(g0 + b) * 4 + k]);
  __syncthreads();
  block_sum(v, gpart + (size_t)g * 4);
  if (threadIdx.x == 0) {
    p.counter[1 + g] = 0;
    __threadfence();
    const unsigned t = atomicAdd(&p.counter[0], 1u);
    *flag = (t == ngroups - 1);
  }
  __syncthreads();
  if (!*flag) return;
  __threadfence();
  double w[4] = {0, 0, 0, 0};
  for (unsigned b = threadIdx.x; b < ngroups; b += blockDim.x)
    for (int k = 0; k < NRED; ++k) w[k] += __ldcg(&gpart[(size_t)b * 4 + k]);
  __syncthreads();
  double tot[4];
  block_sum(w, tot);
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) p.red_result[k] = k < NRED ? tot[k] : 0.0;
    p.counter[0] = 0;
  }
}

}  // namespace owqs
