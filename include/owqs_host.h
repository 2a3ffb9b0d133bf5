/*
 * owqs_host.h — host-only introspection of the scheduler in libowqs.so (no CUDA calls; usable on
 * a machine without a GPU). It exposes what owqs_load_pattern computes before any device work:
 * the validated pattern (rules D0-D3), the PROA plan (Eq. 18, §4.3,
 * tuning L487) and the compiled device step program, so that tests can check
 * PROA against Table I / Eq. 23 / §4.6 and the slot-reuse compiler against the oracle on CPU.
 *
 * Ownership: owqs_host_compile allocates a handle that the caller releases with owqs_host_free.
 * All output buffers are caller-owned; sizes come from owqs_host_info. Errors: OWQS_E_ARG,
 * OWQS_E_PATTERN (message via owqs_host_error).
 */
#ifndef OWQS_HOST_H
#define OWQS_HOST_H

#include <stdint.h>

#include "owqs.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct owqs_host_plan owqs_host_plan; /* opaque */

typedef struct {
  int64_t n_steps;      /* device steps (kernel launches) of the compiled program          */
  int64_t n_measure;
  int64_t sig_len;      /* entries of the signal pool (given-order M ordinals)             */
  int32_t paper_m;      /* max MS of the plan                                               */
  int32_t phys_bits;    /* max physical width                                               */
  int32_t in_width, n_out;
  int32_t step_bytes;   /* sizeof(StepDesc), for layout checks                              */
  int32_t mstatic_bytes;/* sizeof(MStatic)                                                  */
  int32_t n_passes, n_grow, n_shrink, n_reduce;
  int32_t n_swaps;      /* global<->local qubit swaps (n_ranks > 1)                           */
  int32_t n_global;     /* log2(n_ranks): top slot positions that are rank bits               */
  double bytes_per_run; /* analytic HBM bytes of one run at `precision`, per rank             */
} owqs_host_info;

/* Validate + PROA + compile for `mode` (owqs_mode) at `precision` (64/128) with `flags`
 * (OWQS_FLAG_*). weights: NULL (paper defaults and tuning) or {alpha, beta, gamma, delta}.
 * n_ranks: power of two; > 1 compiles the sharded program (the top log2(n_ranks)
 * slot positions are rank bits; SWAP steps exchange a rank bit with a local bit). */
owqs_status owqs_host_compile(const int32_t* inputs, int32_t n_in, const int32_t* outputs, int32_t n_out,
                              const owqs_cmd* cmds, int64_t n_cmds, const int32_t* domain_pool, int64_t pool_len,
                              int32_t mode, int32_t precision, uint32_t flags, const double* weights,
                              int32_t n_ranks, owqs_host_plan** out);
owqs_status owqs_host_info_get(const owqs_host_plan* h, owqs_host_info* info);
/* Copy out the program. Any pointer may be NULL. steps: n_steps * step_bytes bytes; mst:
 * n_measure * mstatic_bytes bytes; sig: sig_len int32; out_slot: n_out int32 (slot of outputs[k]);
 * plan_qubits / plan_ms: n_measure int32 (measured qubit ids in plan order and their MS). */
owqs_status owqs_host_program(const owqs_host_plan* h, void* steps, void* mst, int32_t* sig, int32_t* out_slot,
                              int32_t* plan_qubits, int32_t* plan_ms);
/* gflow of the loaded pattern's open graph (see owqs_gflow in owqs.h): OWQS_OK or OWQS_E_NO_GFLOW;
 * layers[n_measure] by given-order ordinal (may be NULL), depth (may be NULL). */
owqs_status owqs_host_gflow(const owqs_host_plan* h, int32_t* layers, int32_t* depth);
/* Generated pass kernels: NVRTC-compile, for sm_100a, the kernel of every state pass
 * of the compiled program that runs as a generated kernel (no device needed). n_kernels receives
 * the number of distinct kernels, n_jit_steps the number of steps they cover, compile_ms the
 * compile time (0 when every kernel came from the process cache). Any output may be NULL.
 * OWQS_E_ARG with the NVRTC log in owqs_host_error on failure. */
owqs_status owqs_host_jit(owqs_host_plan* h, int64_t* n_kernels, int64_t* n_jit_steps, double* compile_ms);
/* Source of step `step`'s generated kernel (without the common prelude) into buf (capacity cap,
 * NUL-terminated, truncated if short); returns its length in *len, 0 if the step is not generated.
 * step = -1: the common prelude every generated translation unit starts with. */
owqs_status owqs_host_jit_source(const owqs_host_plan* h, int64_t step, char* buf, int64_t cap, int64_t* len);
/* Measurement-calculus standardisation: rewrite the pattern
 * given to owqs_host_compile into standard form N* E* M* C* (all N, then all E, then the M in their
 * given order with the absorbed corrections in their s/t domains, then the outputs' X then Z
 * corrections). Outcome labels and branch probabilities are unchanged; the output equals the
 * original's up to a branch-dependent global phase (reading R-18). signal_shift != 0 also
 * removes every t-domain (signal shifting): M_v's outcome label becomes s_v(new) = s_v(old) + |T_v|
 * with T_v returned in shift_pool. Two-call protocol: pass NULL buffers to get the sizes.
 * cmds/pool: output command list (qubit ids as in the input, domains as slices of pool);
 * shift_slices: 2 int32 (offset, length into shift_pool) per output command (length 0 unless a
 * shifted M); sizes[4] = {n_cmds, pool_len, shift_len, n_x_absorbed}. */
owqs_status owqs_host_standardize(const owqs_host_plan* h, int32_t signal_shift, owqs_cmd* cmds, int32_t* pool,
                                  int32_t* shift_slices, int32_t* shift_pool, int64_t* sizes);
/* Version of the NVRTC the pass-kernel generator compiles with (loaded by absolute path from the
 * CUDA toolkit the library was built against, in its own symbol scope, so a different
 * libnvrtc.so.12 already in the process -- e.g. torch's bundled copy -- is not used). Host only; no
 * GPU needed. Returns OWQS_E_CUDA (major = minor = 0) when NVRTC cannot be loaded. */
owqs_status owqs_host_nvrtc_version(int32_t* major, int32_t* minor);
/* Sub-states of the compiled pattern (PAPER §4.1; owqs_load_pattern): *n = the number of
 * components of its entanglement graph it runs as (1 when it stays one state vector: connected,
 * a signal crossing components, or more than 32 components). If n > 1 and the arrays are not NULL
 * (capacity cap >= n): masks[c] = the caller-order output bits sub-state c owns, phys_bits[c] =
 * the physical width of its compiled program (same mode, precision, flags as the plan). */
owqs_status owqs_host_substates(const owqs_host_plan* h, int32_t* n, uint64_t* masks, int32_t* phys_bits,
                                int32_t cap);
const char* owqs_host_error(const owqs_host_plan* h);
void owqs_host_free(owqs_host_plan* h);

#ifdef __cplusplus
}
#endif
#endif /* OWQS_HOST_H */
