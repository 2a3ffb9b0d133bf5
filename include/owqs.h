/*
 * owqs.h — C-ABI of the B200-native OWQS/EOWQS array executor (libowqs.so).
 *
 * What the library computes: the array (state-vector) execution of a one-way quantum computer
 * measurement pattern P = (V, I, O, A) (§2.2): commands N, E, M^alpha, X^s, Z^s
 * (L69-81), measurement angles adapted by Eq. 2 (L77), each measured qubit eliminated from the
 * state with the operators of Eqs. 11-12 (L193-195, §4.2), commands reordered by PROA (Eq. 18,
 * §4.3) and executed by fused sm_100a kernels (§4.4's implicit actions). "It takes a
 * pattern ... as well as the state of the input qubits ... the state of the output qubits is
 * reported" (L153, Fig. 1). EOWQS (L370-372): outcomes pre-selected to 0, no probabilities,
 * sqrt(2) renormalisation per measurement.
 *
 * Conventions:
 *  - Measurement basis: <+-a| = (<0| +- e^{-i a}<1|)/sqrt2 (reading R-1, Eqs. 9-12).
 *  - Amplitude index: bit k <-> inputs[k] (input state) / outputs[k] (output state); inputs[0]
 *    and outputs[0] are the least significant bit (Eq. 8 layout, L157-161).
 *  - Qubit ids are arbitrary non-negative int32. A non-input qubit used before an explicit N
 *    gets an implicit N at first use (reading R-11).
 *  - Sampled outcomes: u_M = (splitmix64(seed ^ splitmix64(ord)) >> 11) * 2^-53, ord = ordinal
 *    of the M command in the GIVEN list; outcome 0 iff u_M <= prob0 (Fig. 6, reading R-5).
 *  - Arrays indexed "per M" ([n_measure]) use that same given-order ordinal.
 *
 * Ownership and errors: every call returns owqs_status (0 = OK). The caller owns every buffer
 * it passes; the library copies what it needs during the call and never keeps caller pointers.
 * On error, owqs_last_error() describes the failure (string owned by the context, valid until
 * the next call on it). A context is single-writer (not thread-safe). Device memory is owned
 * by the context and released by owqs_destroy.
 */
#ifndef OWQS_H
#define OWQS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct owqs_ctx owqs_ctx; /* opaque */

typedef enum {
  OWQS_OK = 0,
  OWQS_E_ARG = 1,               /* bad argument (NULL, size mismatch, unknown enum)          */
  OWQS_E_PATTERN = 2,           /* rules D0-D3 (L83-91), duplicate E, E(u,u), second N, ...  */
  OWQS_E_NO_GFLOW = 3,          /* EOWQS on a pattern whose open graph has no gflow (L372)     */
  OWQS_E_BRANCH = 4,            /* forced outcome whose probability is < 1e-12               */
  OWQS_E_STATE = 5,             /* call order (run before set_input, output before run, ...)  */
  OWQS_E_NOMEM = 6,             /* state width exceeds device memory                          */
  OWQS_E_CUDA = 7,              /* CUDA runtime error                                         */
  OWQS_E_NCCL = 8,              /* NCCL error (multi-rank)                                    */
  OWQS_E_NOT_DETERMINISTIC = 9  /* EOWQS run whose final norm is not 1: some prob0 != 1/2     */
} owqs_status;

typedef enum { OWQS_CMD_N = 0, OWQS_CMD_E = 1, OWQS_CMD_M = 2, OWQS_CMD_X = 3, OWQS_CMD_Z = 4 } owqs_kind;

/* One command (L69-81). Layout fixed: 40 bytes.
 *  kind  : owqs_kind
 *  q0    : target qubit (u for E)           q1 : second qubit (E only, else ignored)
 *  s_off, s_len : s-signal domain = domain_pool[s_off .. s_off+s_len) (M, X, Z)
 *  t_off, t_len : t-signal domain (M only)
 *  angle : base angle alpha of Eq. 2, radians (M only) */
typedef struct {
  int32_t kind, q0, q1;
  int32_t s_off, s_len, t_off, t_len;
  int32_t reserved;
  double angle;
} owqs_cmd;

/* Context configuration.
 *  precision : 64 -> complex64 amplitudes (fp32 arithmetic, fp64 reductions);
 *              128 -> complex128 (fp64)
 *  n_ranks, rank : SPMD sharding of the top log2(n_ranks) slot bits (1 = single GPU)
 *  device    : CUDA device ordinal
 *  nccl_id   : pointer to a 128-byte ncclUniqueId shared by all ranks (n_ranks > 1), else NULL
 *  flags     : OWQS_FLAG_* bit set
 *  stream    : cudaStream_t to run on (NULL: the library creates a non-blocking stream) */
typedef struct {
  int32_t precision;
  int32_t n_ranks, rank, device;
  const void* nccl_id;
  uint32_t flags;
  int32_t reserved;
  void* stream;
} owqs_config;

#define OWQS_FLAG_NO_GRAPH    0x1u /* launch passes one by one instead of replaying a CUDA graph */
#define OWQS_FLAG_NO_FUSE     0x2u /* at most one measurement butterfly per state pass          */
#define OWQS_FLAG_GIVEN_ORDER 0x4u /* skip PROA: execute measurements in the given order         */
#define OWQS_FLAG_NO_TUNE     0x8u /* PROA with the initial weights only (no L487 tuning loop)   */
#define OWQS_FLAG_PROFILE     0x10u /* record a CUDA event after every kernel of owqs_run (event
                                       record nodes in the graph); see owqs_launch_profile       */
#define OWQS_FLAG_NO_GFLOW    0x40u /* EOWQS without the gflow pre-check of L372 (the final-norm
                                       check still reports OWQS_E_NOT_DETERMINISTIC)             */
#define OWQS_FLAG_NO_JIT      0x80u /* run every pass with the ahead-of-time (op-interpreting) pass
                                       kernel instead of the kernels generated for the pattern at
                                       owqs_load_pattern (NVRTC, sm_100a)          */
#define OWQS_FLAG_ONE_STATE   0x100u /* keep the whole pattern in one state vector even when its
                                        entanglement graph has several components (default: each
                                        component is its own sub-state, PAPER §4.1; see
                                        owqs_load_pattern)                                        */
#define OWQS_FLAG_MEASURED_NORM 0x200u /* structural decisions (a measurement whose partner is a
                                          fresh |+>: prob0 = 1/2 ||psi||^2, Eq. 13) from a ||psi||^2
                                          reduced by the previous pass instead of its exact value 1
                                          (DESIGN R-13): one extra reduction per pass; prob0_out then
                                          reports the device-measured value                       */
#define OWQS_FLAG_LOOPBACK    0x20u /* n_ranks > 1 on ONE device: the context holds every rank's
                                       shard and runs them one after the other (swaps and
                                       all-reduces by device copies); for testing the sharded path
                                       on one GPU. Without it, n_ranks > 1 means one process per GPU
                                       over NCCL (nccl_id from owqs_nccl_unique_id)              */

/* Kernel classes reported by owqs_launch_profile. */
#define OWQS_KCLASS_PASS   0 /* fused warp-segment pass kernel (read + write the state)          */
#define OWQS_KCLASS_SMALL  1 /* one-CTA shared-memory pass for widths <= 12                      */
#define OWQS_KCLASS_GROW   2 /* append |+> (N without a measurement to absorb it)                 */
#define OWQS_KCLASS_SHRINK 3 /* measurement with elimination (no fresh neighbour)                 */
#define OWQS_KCLASS_REDUCE 4 /* read-only pass: probability / norm reduction only                 */
#define OWQS_KCLASS_SWAP   5 /* multi-rank global<->local qubit swap (pack, exchange, unpack)       */

typedef enum { OWQS_SAMPLED = 0, OWQS_FORCED = 1, OWQS_EOWQS = 2 } owqs_mode;

/* Statistics (layout fixed). Valid after owqs_load_pattern; run fields after owqs_run. */
typedef struct {
  int64_t n_commands;        /* commands after implicit-N insertion                          */
  int64_t n_measure;         /* K = |V| - |O|                                                 */
  int32_t paper_m;           /* max PROA measurement state-space MS (append-then-measure m)   */
  int32_t phys_bits;         /* max physical width of the compiled program (slot reuse)      */
  int32_t n_passes;          /* full-state kernel passes in the compiled program (last mode) */
  int32_t n_grow, n_shrink, n_reduce;
  int32_t n_launches;        /* kernel launches per owqs_run (last mode)                      */
  int32_t n_swaps;           /* global<->local slot swaps (multi-rank)                        */
  double bytes_per_run;      /* analytic HBM bytes per owqs_run (all ranks' shards, this rank) */
  double last_run_ms;        /* device time of the last owqs_run (CUDA events)               */
  double schedule_ms;        /* host time spent in PROA + compile for the last mode          */
  double jit_ms;             /* host time generating + NVRTC-compiling the pass kernels of
                                both modes at load_pattern (0 when all came from the cache)    */
  double n_jit_steps;        /* steps of the last mode's program run by generated kernels    */
  double n_kernels;          /* kernel launches per owqs_run of the last mode (steps + the
                                decision kernels of tile-engine passes), per shard            */
  double n_substates;        /* sub-states (PAPER §4.1) the pattern runs as: 1, or the number
                                of components of its entanglement graph (owqs_load_pattern)   */
} owqs_stats_t;

/* Create / destroy a context on cfg->device.
 * Multi-rank: n_ranks = G (power of two) shards the state on its top log2(G) slot
 * positions (rank bits); every rank makes the same call sequence (SPMD). With NCCL, nccl_id points
 * to a 128-byte ncclUniqueId made by owqs_nccl_unique_id on one rank and broadcast by the caller;
 * the library owns the communicator. A sharded program must keep a constant physical width:
 * patterns whose compiled program has GROW or SHRINK steps (an N without a measurement to reuse
 * its slot, a measurement without a fresh neighbour) are refused at owqs_load_pattern with
 * OWQS_E_ARG -- the J/CZ circuit patterns and flow clusters of configs 2-5 are constant-width
 * after slot reuse; other patterns run on one rank (or as replicas).
 * Errors: OWQS_E_ARG, OWQS_E_CUDA, OWQS_E_NCCL. */
owqs_status owqs_create(const owqs_config* cfg, owqs_ctx** out);
/* Write a fresh 128-byte ncclUniqueId to out (call on one rank, broadcast to the others). */
owqs_status owqs_nccl_unique_id(void* out);
void owqs_destroy(owqs_ctx* ctx);

/* Load a pattern in its GIVEN (execution) order (L67; right-to-left notation already reversed).
 * Validates D0-D3 (L83-91), inserts implicit N, builds the dependency DAG of non-commuting
 * commands (Eqs. 14-16) and runs PROA (Eq. 18 with the tuning of L487). No device memory is
 * touched (device buffers are allocated at the first input / run).
 * inputs[n_in], outputs[n_out] : qubit ids; bit k of the input/output index is inputs[k]/outputs[k].
 * domain_pool[pool_len]        : qubit ids referenced by the cmds' signal domains.
 * Sub-states (§4.1): when the pattern's entanglement graph has several components (all
 * inputs count as one) and no signal domain crosses them, each component runs as its own state
 * vector (memory of the largest, not of their sum) and owqs_get_output returns their tensor
 * product; single rank only, disabled by OWQS_FLAG_ONE_STATE. Calls that need one state vector
 * (owqs_output_inner / _norm, owqs_recognize*, owqs_run_batch, owqs_submit_host, owqs_plan_order,
 * owqs_launch_profile) then return OWQS_E_STATE. owqs_stats().n_substates reports the split.
 * The pass kernels are generated and NVRTC-compiled here (kept in a process-wide cache).
 * Errors: OWQS_E_ARG, OWQS_E_PATTERN (message names the command index). */
owqs_status owqs_load_pattern(owqs_ctx* ctx, const int32_t* inputs, int32_t n_in,
                              const int32_t* outputs, int32_t n_out,
                              const owqs_cmd* cmds, int64_t n_cmds,
                              const int32_t* domain_pool, int64_t pool_len);

/* Input state of the input qubits (L153). amps: HOST array of n_amps = 2^n_in complex128 values,
 * interleaved (re, im). Copied to the device (converted to complex64 at precision 64).
 * Multi-rank: every rank passes the full array; each copies its shard.
 * CONTRACT (every owqs_set_input_* / owqs_submit_host / owqs_run_batch input): the state must be
 * normalised, |1 - ||psi||^2| <= 1e-9 (precision 128) / 1e-5 (precision 64). A measurement whose
 * partner qubit is a fresh |+> has prob0 = 1/2 ||psi||^2 exactly (Eq. 3 / Eq. 13; DESIGN
 * R-13); the executor takes ||psi||^2 = 1 there instead of reducing the state, and Eq. 4's
 * renormalisation keeps it 1 after every measurement that does reduce. The library
 * reduces ||psi||^2 on the device during the copy and refuses other inputs with OWQS_E_ARG (the
 * context then has no input); owqs_submit_host reports it from owqs_wait.
 * Errors: OWQS_E_ARG (size, norm), OWQS_E_STATE (no pattern), OWQS_E_NOMEM, OWQS_E_CUDA. */
owqs_status owqs_set_input(owqs_ctx* ctx, const double* amps, int64_t n_amps);

/* Same from a HOST buffer at `precision` (64: interleaved float pairs, 8 B per amplitude; 128:
 * double pairs). When it equals the context's precision the bytes go straight to the state
 * (page-locked buffers by DMA): complex64 end-to-end runs move half the PCIe bytes of
 * owqs_set_input. Errors as owqs_set_input, OWQS_E_ARG for another precision. */
owqs_status owqs_set_input_host(owqs_ctx* ctx, const void* amps, int32_t precision, int64_t n_amps);

/* Same from a DEVICE buffer on the context's device. precision 64: interleaved float pairs;
 * 128: interleaved double pairs. The buffer is read during the call only. NCCL multi-rank: the
 * buffer holds this rank's shard (n_amps = 2^n_in / n_ranks); loopback: the full state.
 * Same-precision input is copied and its norm^2 reduced in one sweep (norm contract above, the
 * all-ranks norm in the multi-rank case); the call synchronises the context's stream. */
owqs_status owqs_set_input_device(owqs_ctx* ctx, const void* dev_amps, int32_t precision, int64_t n_amps);

/* Device-generated Haar-random input (documented counter generator, workloads/inputs.py):
 * amp_j = sqrt(-2 ln u1) e^{2 pi i u2} from splitmix64 of (seed, j), then normalised (so it meets
 * the norm contract of owqs_set_input by construction). */
owqs_status owqs_set_input_random(owqs_ctx* ctx, uint64_t seed);

/* Execute the loaded pattern on the current input (consumes it: the state becomes the output).
 * mode OWQS_SAMPLED : outcomes drawn as in the conventions above from `seed`;
 *      (OWQS_EOWQS first checks the gflow: OWQS_E_NO_GFLOW, see owqs_gflow)
 *      OWQS_FORCED  : forced[n_measure] gives each outcome (given-order ordinal);
 *                     OWQS_E_BRANCH if a forced branch has probability < 1e-12;
 *      OWQS_EOWQS   : every outcome 0, no probability computation, sqrt2 per M (L372);
 *                     OWQS_E_NOT_DETERMINISTIC if the final norm^2 differs from 1 by more than
 *                     1e-8 (precision 128) / 1e-3 (precision 64).
 * outcomes_out[n_measure] (may be NULL): s_v per M (given-order ordinal).
 * prob0_out[n_measure] (may be NULL): <psi|P_0|psi> at that measurement (Eq. 3/13), -1 in EOWQS. */
owqs_status owqs_run(owqs_ctx* ctx, owqs_mode mode, uint64_t seed, const uint8_t* forced,
                     uint8_t* outcomes_out, double* prob0_out);

/* Asynchronous host-to-host run (serving path; the problem statement of L153 -- input state in,
 * output state out -- as one call that returns before the work is done). Enqueues on the
 * context's stream: the host->device copy of in_amps (2^n_in amplitudes at in_precision, caller
 * order), owqs_run(mode, seed, forced), and the device->host copy of the output (2^n_out amplitudes
 * at out_precision, bit k <-> outputs[k]) into out_amps; returns without waiting. Both host buffers
 * must be page-locked (cudaHostAlloc / cudaHostRegister: OWQS_E_ARG otherwise) and stay untouched
 * until owqs_wait. Two contexts on different streams pipeline: one run's PCIe copies overlap the
 * other's kernels. Single rank only (OWQS_E_ARG). Any other call on the context before owqs_wait
 * returns OWQS_E_STATE. Errors found while enqueueing are returned here; errors of the run itself
 * (OWQS_E_BRANCH, OWQS_E_NOT_DETERMINISTIC, CUDA faults) and an input that breaks the norm
 * contract of owqs_set_input (OWQS_E_ARG, output not valid) are returned by owqs_wait. */
owqs_status owqs_submit_host(owqs_ctx* ctx, owqs_mode mode, uint64_t seed, const uint8_t* forced,
                             const void* in_amps, int32_t in_precision, int64_t n_in, void* out_amps,
                             int32_t out_precision, int64_t n_out);
/* Wait for the submitted run; outcomes_out / prob0_out as for owqs_run (may be NULL). The output
 * buffer is complete when this returns OWQS_OK. OWQS_E_STATE if nothing is pending. */
owqs_status owqs_wait(owqs_ctx* ctx, uint8_t* outcomes_out, double* prob0_out);

/* Batched replicas: run the loaded pattern on n_batch independent inputs in
 * one launch (one CTA per state, the state in shared memory; single rank, physical width <= 12).
 * inputs  : HOST [n_batch][2^n_in] complex128 interleaved (input k of state b at b*2^n_in + k)
 * seeds   : [n_batch] sampled-mode seeds (NULL: all 0); forced: [n_batch][n_measure] (OWQS_FORCED)
 * outputs : HOST [n_batch][2^n_out] complex128; outcomes / prob0 (may be NULL): [n_batch][n_measure]
 * Semantics per state are those of owqs_set_input + owqs_run + owqs_get_output (OWQS_E_ARG for an
 * input off the norm contract, |1 - ||psi||^2| > 1e-9, checked on the host); EOWQS applies the
 * gflow gate, OWQS_E_BRANCH if any forced branch is impossible, OWQS_E_NOT_DETERMINISTIC if any
 * EOWQS output norm^2 is off by more than the owqs_run tolerance. Does not touch the context's
 * current input/output. */
owqs_status owqs_run_batch(owqs_ctx* ctx, owqs_mode mode, int64_t n_batch, const double* inputs,
                           const uint64_t* seeds, const uint8_t* forced, double* outputs,
                           uint8_t* outcomes, double* prob0);

/* Output state over O (L153, L419): HOST array of n_amps >= 2^n_out complex128, interleaved,
 * bit k <-> outputs[k]. Multi-rank (collective): gathered to rank 0, filled on rank 0 only
 * (amps may be NULL elsewhere); needs 2^n_out complex128 of free device memory on rank 0. */
owqs_status owqs_get_output(owqs_ctx* ctx, double* amps, int64_t n_amps);

/* Same into a HOST buffer at `precision` (64: float pairs, 128: double pairs); complex64 halves
 * the PCIe bytes of owqs_get_output. Single rank and loopback only (OWQS_E_ARG otherwise). */
owqs_status owqs_get_output_host(owqs_ctx* ctx, void* amps, int32_t precision, int64_t n_amps);

/* Output into a DEVICE buffer (precision 64: float pairs, 128: double pairs), n_amps >= 2^n_out
 * (single rank). */
owqs_status owqs_get_output_device(owqs_ctx* ctx, void* dev_amps, int32_t precision, int64_t n_amps);

/* Sampled output amplitudes ("the state of the output qubits is reported", for states too
 * large to copy out: SURVEY §8(a) a10 "device-side compare"): amps[i] = output amplitude idx[i],
 * caller order (bit k <-> outputs[k]), idx: HOST [n] in [0, 2^n_out), amps: HOST [n] complex128
 * interleaved, any state precision. Multi-rank: collective, every rank receives all n values.
 * Errors: OWQS_E_ARG (index range), OWQS_E_STATE (no output, sub-states), OWQS_E_NOMEM. */
owqs_status owqs_get_output_sample(owqs_ctx* ctx, const int64_t* idx, int64_t n, double* amps);

/* <a|b> of the output states of two contexts with the same output qubits, on the device.
 * Multi-rank: both contexts need the same sharding and final layout (collective call). */
owqs_status owqs_output_inner(owqs_ctx* a, owqs_ctx* b, double* re, double* im);

/* ||output||^2 on the device (all-reduced over ranks; collective call). */
owqs_status owqs_output_norm(owqs_ctx* ctx, double* norm2);

/* Recognition problem (L33): the unitary implemented by the loaded (deterministic) pattern.
 * Column k = EOWQS run on basis input |k> (all outcomes 0, sqrt2 per M: a linear map); the
 * 2^n_in columns run as one owqs_run_batch launch when the width allows.
 * U: HOST array of n = 2^n_out * 2^n_in complex128 (interleaved), column-major.
 * max_unitarity_err (may be NULL): max |(U^dag U - I)_ij|. Overwrites the current input. */
owqs_status owqs_recognize(owqs_ctx* ctx, double* U, int64_t n, double* max_unitarity_err);

/* Same result from ONE run on the Choi state: the loaded pattern is
 * extended by |I| reference qubits that no command touches (inputs I + R, outputs O + R) and run
 * (positive EOWQS branch) on sum_k |k>_I |k>_R / sqrt(2^|I|); the output, scaled by sqrt(2^|I|), is U
 * column-major. Runs at the pattern's width + |I| in a temporary context on the same device;
 * |I| + |O| <= 30. Same gflow check and errors as owqs_recognize. */
owqs_status owqs_recognize_choi(owqs_ctx* ctx, double* U, int64_t n, double* max_unitarity_err);

/* gflow of the pattern's open graph (L372, Mhalla-Perdrix [25]; all measurements in the XY plane):
 * OWQS_OK if one exists, else OWQS_E_NO_GFLOW ("the pattern is reported as an incorrect one").
 * layers[n_measure] (may be NULL): backward layer of each measured qubit (given-order ordinal;
 * outputs are layer 0); depth (may be NULL): number of layers. owqs_run(OWQS_EOWQS) and
 * owqs_recognize apply this check first (unless OWQS_FLAG_NO_GFLOW). Host only. */
owqs_status owqs_gflow(owqs_ctx* ctx, int32_t* layers, int32_t* depth);

/* Sizes after owqs_load_pattern (any pointer may be NULL). n_passes is for the sampled plan. */
owqs_status owqs_pattern_info(owqs_ctx* ctx, int64_t* n_measure, int32_t* paper_m, int32_t* phys_bits,
                              int32_t* n_passes);

/* PROA result for `mode`: measured qubit ids in plan order (qubits[n_measure]) and the MS of each
 * step (ms[n_measure], may be NULL). */
owqs_status owqs_plan_order(owqs_ctx* ctx, owqs_mode mode, int32_t* qubits, int32_t* ms, int64_t n);

/* Override the PROA weights (alpha, beta, gamma, delta of Eq. 18) for subsequent plans; tune != 0
 * re-enables the L487 loop that decrements alpha |O| times starting from these values. */
owqs_status owqs_set_proa_weights(owqs_ctx* ctx, double a, double b, double g, double d, int32_t tune);

owqs_status owqs_stats(owqs_ctx* ctx, owqs_stats_t* out);

/* Per-launch profile of the last owqs_run of a context created with OWQS_FLAG_PROFILE: for launch
 * i (i < n, n >= stats.n_launches) its kernel class (OWQS_KCLASS_*), its algorithmic HBM bytes
 * (read + write of the state it sweeps) and its device duration in ms measured by
 * CUDA events on the library's stream. Any pointer may be NULL. OWQS_E_STATE if not profiled. */
owqs_status owqs_launch_profile(owqs_ctx* ctx, int32_t* kclass, double* bytes, float* ms, int64_t n);
const char* owqs_last_error(const owqs_ctx* ctx);
const char* owqs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* OWQS_H */
