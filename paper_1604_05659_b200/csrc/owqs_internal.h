// Internal definitions shared by the host scheduler (C++) and the sm_100a kernels (CUDA).
// Plain-old-data only: the compiled pass program is uploaded / passed by value to kernels.
#pragma once
#ifdef __CUDACC_RTC__
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#else
#include <stdint.h>
#endif

namespace owqs {

// ---- device op encoding (16 bytes) ------------------------------------------------------------
enum OpType : uint8_t {
  OP_NONE = 0,
  OP_DIAG_E = 1,  // CZ sign flip on slots (a, b)               PAPER §4.4.1, Fig. 5 (E action)
  OP_DIAG_Z = 2,  // Z^s on slot a (sign on bit a = 1)
  OP_X = 3,       // X^s on slot a (swap pairs)
  OP_BFLY = 4,    // measurement butterfly on slot a, M record m (slot reuse: the new qubit takes
                  // slot a; Eqs. 11-12 with N_o E_io folded in)
  OP_FLUSH = 5,   // apply the sign flips accumulated by the preceding diagonal ops (placed by the
                  // compiler before the first 2x2 on a slot those diagonals touch)
};

struct Op {
  uint8_t type;
  uint8_t a;
  uint8_t b;
  uint8_t cond;     // 1: conditional on the XOR of outcomes sig_pool[sig_off .. sig_off+sig_len)
  int32_t sig_off;
  int32_t sig_len;
  int32_t m;        // M plan index (OP_BFLY)
};
static_assert(sizeof(Op) == 16, "Op layout");

constexpr int MAX_OPS = 128;     // ops per pass (incl. compiler-placed flushes)
constexpr int KMAX_HI = 8;       // group slots above the warp segment per pass (storage)
constexpr int KMAX_AOT = 4;      // ... in passes run by the ahead-of-time / direct-load kernels
constexpr int KTILE = 7;         // ... in passes run by the complex64 tile engine (13-bit CTA tile)
constexpr int MAX_BFLY = 64;     // butterflies per pass (fused mode)

enum StepKind : int32_t { ST_PASS = 0, ST_GROW = 1, ST_SHRINK = 2, ST_SWAP = 3, ST_RHOK = 4, ST_SHRINKK = 5 };
// joint k-outcome measurement: up to JOINT_KMAX consecutive eliminations share
// one reduced-density-matrix pass (ST_RHOK) and one projection + compaction pass (ST_SHRINKK)
constexpr int JOINT_KMAX = 3;
enum RedKind : int32_t { RED_NONE = 0, RED_NORM = 1, RED_RHO = 2 };

// One device step. Passed by value as a kernel parameter.
struct StepDesc {
  int32_t kind;        // StepKind
  int32_t width;       // state width (bits) when the step runs
  int32_t nb_hi;       // number of group slots >= segment bits
  int32_t bhi[KMAX_HI];
  int32_t n_ops;
  int32_t red_kind;    // reduction of the step's OUTPUT state (RedKind)
  int32_t red_slot;    // slot for RED_RHO
  int32_t slot;        // GROW: new top slot; SHRINK: measured slot
  int32_t shrink_m;    // SHRINK: M plan index
  int32_t n_bfly;      // number of OP_BFLY in ops
  int32_t first_uses_red;  // 1: the first butterfly (or the SHRINK) decides from red_result
  int32_t first_full_rho;  // 1: red_result holds (n0, n1, Re c, Im c) of the measured slot
  int32_t pad;
  Op ops[MAX_OPS];
  // absorb[bi]: slots whose bits flip the sign of butterfly bi's coefficient a — the CZ's
  // E(o, a) absorbed into the first following butterfly on slot a (U Z^{x_o} = k[[1,-+a],[1,+-a]])
  uint64_t absorb[MAX_BFLY];
  // ST_SWAP (multi-rank): exchange the qubit at global position swap_global (a rank bit) with the
  // one at local position swap_local; each rank trades half of its shard with rank ^ (1 << (g - wl))
  int32_t swap_local, swap_global;
  // ST_PASS on the tile engine: qubit remapping applied at the pass's store -- the amplitude bit at
  // physical position remap_a[k] is written to position remap_b[k] and vice versa (a segment slot
  // whose qubit has no further 2x2 op traded for a group slot of a still-active qubit)
  int32_t n_remap;
  int32_t remap_a[6], remap_b[6];
  // ST_RHOK / ST_SHRINKK: jk measured qubits in the emitter's (= the caller's plan) order; bit j of the
  // 2^jk joint index <-> physical position jm_pos[j] of the pre-group layout (width = the pre-group
  // width), jm[j] = its M plan index; ST_SHRINKK output bit t < width - jk comes from position
  // j_src[t] (the composition of jk SHRINK top moves, so the slot map is that of jk single SHRINKs)
  int32_t jk;
  int32_t jm_pos[4], jm[4];
  signed char j_src[64];
};

// Decisions of one pass, computed once by decide_kernel and read by every CTA of the generated pass
// kernel: the structured butterfly coefficient a = ar + i ai of each butterfly (k folded into
// scale), as fp32 (ar, packed (-ai, ai)) and fp64, and the condition of every op.
struct PassCoef {
  uint64_t B[MAX_BFLY];   // complex64: packed float pair (-ai, ai)
  double ard[MAX_BFLY];   // complex128
  double aid[MAX_BFLY];
  double scale;           // product of the pass's butterfly k's
  float ar[MAX_BFLY];     // complex64
  uint8_t cond[MAX_OPS];
};

// Grid-reduction scratch sizes (per shard): block partials and group partials (deterministic
// two-level reduction of the generated pass kernels).
constexpr int RED_MAX_BLOCKS = 1 << 22;  // one tile per CTA up to width 34 (complex64) / 33 (complex128)
constexpr int KRON_MAX = 32;  // sub-states merged by one kron_merge launch
constexpr int RED_GROUP = 256;
constexpr int RED_MAX_GROUPS = RED_MAX_BLOCKS / RED_GROUP;

// Static record of one measurement (plan order). Uploaded once per compiled plan.
struct MStatic {
  double alpha;       // base angle of Eq. 2
  int32_t ord;        // ordinal of the M in the GIVEN list (outcome / prob0 / draw index)
  int32_t s_off, s_len, t_off, t_len;  // domains as given-order ordinals in sig_pool
  int32_t reuse;      // 1: slot-reuse butterfly (fresh |+> neighbour folded), 0: elimination
  int32_t structural; // 1: prob0 = ||psi||^2 / 2 exactly (a fresh |+> neighbour dephases it)
  int32_t key;        // keyed sampling draw index (reading R-5): the caller's given-order ordinal
                      // (differs from ord only in a sub-state of a split pattern, PAPER §4.1)
};

// Run parameters in device memory (written by the host before each run).
struct RunParams {
  int32_t mode;       // owqs_mode
  int32_t pad;
  uint64_t seed;
};

// Device-side pointers, passed by value to kernels.
struct DevPtrs {
  void* state;                 // float2* (complex64) or double2* (complex128)
  const MStatic* mst;          // [n_measure] plan order
  double* coef;                // [n_measure][8]: resolved 2x2 (EOWQS precomputed on host)
  uint8_t* outcome;            // [n_measure] given-order ordinal
  double* prob0;               // [n_measure] given-order ordinal
  const uint8_t* forced;       // [n_measure] given-order ordinal
  const int32_t* sig_pool;     // domains as given-order ordinals
  const RunParams* run;
  double* partials;            // [max_blocks][4]
  unsigned int* counter;       // last-block-done counter
  double* red_result;          // [4]
  int32_t* err;                // device error flag (1 = forced branch with prob < 1e-12)
  uint32_t rank;               // multi-rank: this shard's rank = the global (top) index bits
  int32_t local_width;         // multi-rank: bits of the shard index (positions >= are rank bits)
  void* scratch;               // ST_SHRINKK output (2^(width - jk) amplitudes), copied back into state
};
// ST_RHOK result (the 2^k x 2^k reduced density matrix, upper triangle incl. diagonal, re / im
// interleaved) in the tail of the block-partials region of DevPtrs::partials
constexpr int RHOK_VALS = 2 * ((1 << JOINT_KMAX) * ((1 << JOINT_KMAX) + 1) / 2);  // 72
constexpr size_t RHOK_RESULT_OFF = (size_t)(1 << 20) * 4 - 128;

}  // namespace owqs
