// Host-side scheduler: pattern validation, dependency DAG, PROA reordering (PAPER §4.3) and the
// slot-reuse compiler that turns a plan into the device pass program.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "owqs_internal.h"

namespace owqs {

enum HKind { H_N = 0, H_E = 1, H_M = 2, H_X = 3, H_Z = 4 };

struct HCmd {
  int kind = 0, q0 = -1, q1 = -1;  // dense qubit indices
  double angle = 0.0;
  std::vector<int> sdom, tdom;     // dense qubit indices
};

// A validated pattern with implicit N made explicit (reading R-11), qubits renumbered densely.
struct HostPattern {
  int nq = 0;
  std::vector<int32_t> ext_id;          // dense -> external id
  std::vector<int> inputs, outputs;     // dense
  std::vector<HCmd> cmds;               // given (execution) order, explicit N
  int n_measure = 0;
  std::vector<int> m_ord_of_cmd;        // given-order M ordinal of each cmd (-1 if not M)
  std::vector<int> m_ord_of_qubit;      // given-order M ordinal measuring each qubit (-1)
  std::vector<char> is_output, is_input;
  std::vector<int> draw_key;            // keyed-draw index per M ordinal (empty: the ordinal itself)
};

// Validate rules D0-D3 and normalise. Returns "" on success, else a message.
std::string validate_pattern(const int32_t* inputs, int n_in, const int32_t* outputs, int n_out,
                             const void* cmds /* owqs_cmd[] */, int64_t n_cmds,
                             const int32_t* pool, int64_t pool_len, HostPattern& out);

// PAPER §4.1 sub-states: the components of the E graph (all inputs in one), each as its own
// pattern over the same qubit ids and given-order M ordinals; masks[c] = its caller-order output
// bits. False (one state) when a signal domain crosses components or there are < 2 or > max_parts.
bool split_substates(const HostPattern& hp, std::vector<HostPattern>& parts, std::vector<uint64_t>& masks,
                     int max_parts);

struct ProaWeights {
  double a = -1, b = -1, g = 0.5, d = -1;  // alpha, beta, gamma, delta of Eq. 18 (-1: |O|)
  bool tune = true;                        // PAPER L487 loop
};

struct Plan {
  std::vector<int> order;   // command indices in execution order
  std::vector<int> m_cmds;  // M command indices in plan order
  std::vector<int> ms;      // MS(v) of each selected measurement (Eq. 18 first criterion)
  int paper_m = 0;          // max MS (append-then-measure width), at least |I|
};

// PROA (Eq. 18) over the DAG of non-commuting commands. eowqs: corrections and signal
// dependencies dropped ("there is no dependent list"). given_order: no reordering.
Plan make_plan(const HostPattern& hp, bool eowqs, bool given_order, const ProaWeights& w);

// Compiled device program.
struct Program {
  std::vector<StepDesc> steps;
  std::vector<MStatic> mst;        // plan order
  std::vector<int32_t> sig_pool;   // given-order M ordinals
  int phys_bits = 0;               // max width
  int in_width = 0;
  std::vector<int> out_slot;       // slot of outputs[k] at the end
  int n_passes = 0, n_grow = 0, n_shrink = 0, n_reduce = 0, n_swaps = 0;
  int n_global = 0;                // log2(ranks): top slot positions that are rank bits
  std::string error;               // non-empty: the program cannot be built (e.g. sharding)
  double bytes_per_run(int elem_bytes) const;  // per rank
};

// mode: 0 sampled / 1 forced (OWQS) or 2 EOWQS. seg_bits: 6 for complex64, 5 for complex128.
// kwide: group slots per pass for passes of width >= 13 (complex64 tile engine, up to KMAX_HI);
// narrower passes and the ahead-of-time kernels use KMAX_AOT.
// measured_norm (OWQS_FLAG_MEASURED_NORM): structural decisions reduce ||psi||^2 in the previous pass
// instead of taking its exact value 1 (reading R-13) -- a device-measured check of that reading.
Program compile_program(const HostPattern& hp, const Plan& plan, int mode, int seg_bits, bool fuse,
                        int n_global = 0, int kwide = KMAX_AOT, bool measured_norm = false);

// Plan + compile for a mode. For EOWQS two candidates are compiled — PROA without dependencies
// and the OWQS plan with its (identity) corrections dropped — and the one with the
// smaller physical width, then fewer passes, is kept.
void plan_and_compile(const HostPattern& hp, int mode, int seg_bits, bool fuse, bool given_order,
                      const ProaWeights& w, Plan& plan, Program& prog, int n_global = 0, int kwide = KMAX_AOT,
                      bool measured_norm = false);

// Standard form N* E* M* C* of a validated pattern (standardize.cpp); with
// signal_shift, t-domains are removed and returned per measured qubit in `shift` (new labels).
std::string standardize_pattern(const HostPattern& hp, bool signal_shift, std::vector<HCmd>& out,
                                std::vector<std::vector<int>>& shift, int* n_x_absorbed, int* n_signs);

// gflow of the pattern's open graph ([25]): "" if found, else the reason. layer[q] = 0
// for outputs, k >= 1 for the k-th backward layer; g[q] = correction set of measured q.
std::string find_gflow(const HostPattern& hp, std::vector<int>& layer, std::vector<std::vector<int>>& g);

}  // namespace owqs
