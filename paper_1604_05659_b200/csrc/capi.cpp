// C-ABI implementation (include/owqs.h): context, device memory, CUDA-graph executor, sharding.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <cmath>
#include <string>
#include <vector>

#include "jit.h"
#include "owqs.h"
#include "scheduler.h"

namespace owqs {
cudaError_t init_kernel_limits(int device);
int max_partial_blocks();
cudaError_t launch_step(const StepDesc& d, const DevPtrs& p, int prec, cudaStream_t s);
cudaError_t launch_permute_out(const void* state, int prec, void* out, int out_prec, int nbits, const int* slots,
                               uint64_t j0, uint64_t count, cudaStream_t s);
cudaError_t launch_scatter_out(const void* shard, int prec, void* out, int out_prec, int nbits, const int* slots,
                               uint64_t rank, int wl, cudaStream_t s);
cudaError_t launch_convert_in(const void* src, int src_prec, void* state, int prec, uint64_t j0, uint64_t count,
                              cudaStream_t s);
cudaError_t launch_kron_merge(void* out, int prec, const void* const* factors, const uint64_t* masks, int n,
                              uint64_t count, cudaStream_t s);
cudaError_t launch_basis(void* state, int prec, uint64_t n, uint64_t k, cudaStream_t s);
cudaError_t launch_haar(const DevPtrs& p, int prec, uint64_t n, uint64_t seed, uint64_t j0, cudaStream_t s);
cudaError_t launch_scale(const DevPtrs& p, int prec, uint64_t n, cudaStream_t s);
cudaError_t launch_norm(const DevPtrs& p, int prec, uint64_t n, cudaStream_t s);
cudaError_t launch_readback(void* host_dst, const void* dev_src, size_t n, cudaStream_t s);
cudaError_t launch_sample_out(const void* shard, int prec, const int64_t* idx, uint64_t n, int nbits, const int* slots,
                              uint64_t rank, int wl, void* out, cudaStream_t s);
cudaError_t launch_copy_norm(const DevPtrs& p, int prec, const void* src, uint64_t n, cudaStream_t s);
cudaError_t launch_dot(const DevPtrs& p, const void* a, const void* b, uint64_t n, cudaStream_t s);
cudaError_t launch_dot_t(const DevPtrs& p, int prec, const void* a, const void* b, uint64_t n, cudaStream_t s);
cudaError_t launch_swap_pack(const void* state, void* buf, int prec, int pl, int bit, bool unpack, uint64_t j0,
                             uint64_t n, cudaStream_t s);
cudaError_t launch_loopback_allreduce(double* red, int n_ranks, cudaStream_t s);
int step_kclass(const StepDesc& d, int prec);
cudaError_t jit_launch(cudaKernel_t k, int max_blocks, const StepDesc& d, const DevPtrs& p, const PassCoef* pc, int prec,
                       cudaStream_t s, const PassCoef* cp_host, cudaGraphDeviceNode_t* dev_node, bool no_pdl);
cudaError_t launch_decide_ahead(const StepDesc* d_steps, int n_steps, int n_mst, const DevPtrs& p, PassCoef* pc,
                                cudaStream_t s);
cudaError_t launch_decide(const StepDesc& d, const DevPtrs& p, PassCoef* pc, cudaStream_t s,
                          const cudaGraphDeviceNode_t* nodes, int n_nodes, size_t off);
cudaError_t launch_grid_finish(const DevPtrs& p, unsigned nblk, int nred, cudaStream_t s);
cudaError_t launch_batch(const StepDesc* steps, int n_steps, const DevPtrs& base, int K, int n_batch, const void* in,
                         void* out, int n_in, int n_out, const int* out_slot, int phys, int prec, cudaStream_t s);
}  // namespace owqs

using namespace owqs;

namespace {
// NVTX range over a C-ABI call (SURVEY §5 tracing): host-side, shows load / input / run / output
// phases in an nsys or ncu --nvtx timeline; a no-op without an attached tool
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
struct CompiledMode {
  bool valid = false;
  Plan plan;
  Program prog;
  MStatic* d_mst = nullptr;
  int32_t* d_sig = nullptr;
  StepDesc* d_steps = nullptr;  // device copy of the program (batched replicas)
  cudaGraphExec_t gexec = nullptr;
  double schedule_ms = 0;
  // generated pass kernels (jit.h): per step kernel name ("" = ahead-of-time kernel), the cubins,
  // and once loaded on the device the kernel handles and their grid caps
  std::vector<std::string> jit_name;
  std::vector<JitModule> jit_mods;
  std::vector<cudaLibrary_t> jit_libs;
  std::vector<cudaKernel_t> jit_fn;
  std::vector<int> jit_blocks;
  int n_jit = 0;
  PassCoef* d_pc = nullptr;  // one decision block per step (engine-2 generated kernels)
  // coefp: the tile kernels take the decisions as their by-value PassCoef parameter (DESIGN.md
  // §5.1): in the captured graph decide_kernel writes it into the device-updatable kernel node(s)
  // of its pass (handles in d_devnodes[step * shards + r], parameter offset coef_off[step]); the
  // EOWQS mode's decisions are run-independent and set by the host at capture (static_cp)
  // COEF_CONST instead: decide_kernel's PassCoef is copied by a graph memcpy node into the kernel's
  // module __constant__ (cp_sym[step]); EOWQS's from d_static_cp (copied once when the kernel is
  // used by this step only, cp_once). Kernel nodes stay ordinary graph nodes (ncu-profilable).
  int coef_src = 0;  // jit.h COEF_*
  bool coefp = false;  // coef_src != COEF_POINTER
  cudaGraphDeviceNode_t* d_devnodes = nullptr;
  std::vector<size_t> coef_off;
  std::vector<PassCoef> static_cp;
  PassCoef* d_static_cp = nullptr;
  std::vector<void*> cp_sym;
  std::vector<char> cp_once;
  // EOWQS: every decision is run-independent (outcomes 0, no signals, no probabilities, static
  // scales), so d_pc written by the first EOWQS run is reused and later runs launch no decide kernel
  bool pc_static_ready = false;
};
// one rank's part of the state and its reduction scratch
struct Shard {
  void* d_state = nullptr;
  double* d_partials = nullptr;
  unsigned* d_counter = nullptr;
  int32_t* d_err = nullptr;
  double* d_red = nullptr;  // -> ctx->d_red_all + 4 * index
};
constexpr size_t kStagingBytes = 64ull << 20;
constexpr size_t kFullOutMaxBytes = 8ull << 30;
}  // namespace

struct owqs_ctx {
  owqs_config cfg{};
  int prec = 0;  // 0 complex64, 1 complex128
  int elem = 8;
  std::string err;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  HostPattern hp;
  bool loaded = false;
  CompiledMode cm[2];  // 0 OWQS (sampled / forced), 1 EOWQS
  ProaWeights weights;
  // sharding
  int n_ranks = 1, rank = 0, n_global = 0;
  bool loopback = false;
  ncclComm_t comm = nullptr;
  std::vector<Shard> shards;  // 1, or n_ranks in loopback mode
  double* d_red_all = nullptr;
  size_t shard_bytes = 0;
  void* d_swap = nullptr;  // one shard: the swap's chunk slots (2 send + 2 receive), or the gather buffer
  // NCCL swaps: the transfers run on comm_stream, pack / unpack on stream, chunk by chunk (events)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t sw_packed[2] = {}, sw_sent[2] = {}, sw_unpacked[2] = {};
  void* d_jscratch = nullptr;  // ST_SHRINKK output (joint k-outcome measurement), jscratch_bytes
  size_t jscratch_bytes = 0;
  // run state
  RunParams* d_run = nullptr;
  uint8_t* d_outcome = nullptr;
  double* d_prob0 = nullptr;
  uint8_t* d_forced = nullptr;
  size_t k_cap = 0;
  void* d_staging = nullptr;
  void* d_out_full = nullptr;  // owqs_submit_host: whole permuted output (<= kFullOutMaxBytes)
  size_t out_full_bytes = 0;
  void* h_staging = nullptr;  // pinned
  int32_t* h_err = nullptr;   // pinned, one per shard: device error flags copied in stream order
  double* h_innorm = nullptr;  // pinned: ||psi_in||^2 of the last input (R-13 precondition), stream-ordered
  bool has_input = false, has_output = false;
  int out_cm = -1;
  int pending = 0;  // owqs_submit_host: 1 + compiled mode of the enqueued run, until owqs_wait
  // PAPER §4.1 sub-states: one child context per component of the entanglement graph (subs[0]
  // holds the inputs when there are any); sub_mask[c] = the caller-order output bits it owns
  std::vector<owqs_ctx*> subs;
  std::vector<uint64_t> sub_mask;
  int pending_mode = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // decide-ahead graph capture: the copies of the decisions into the pass kernels' __constant__ fork
  // over kAux side streams (parallel graph branches) and join before the first pass
  static constexpr int kAux = 4;
  cudaStream_t aux[kAux] = {};
  cudaEvent_t fork_ev = nullptr, join_ev[kAux] = {};
  owqs_stats_t stats{};
  int last_cm = 0;
  std::vector<cudaEvent_t> prof_ev;  // OWQS_FLAG_PROFILE: event after every launch (+1 start)
  int prof_cm = -1;
  double jit_ms = 0;
  int gflow_state = 0;  // 0 unknown, 1 has a gflow, -1 none (L372 pre-check, cached per pattern)
  std::string gflow_msg;

  uint32_t shard_rank(int i) const { return loopback ? (uint32_t)i : (uint32_t)rank; }
};

namespace {

// decisions ahead for a sampled / forced run of m: constant-bank coefficients, one
// shard, every step a tile pass whose decisions are structural (no reduction feeds them, no SHRINK)
bool decide_ahead_ok(const owqs_ctx* ctx, const CompiledMode& m) {
  if (m.coef_src != COEF_CONST || m.jit_fn.empty() || m.cp_sym.empty() || ctx->shards.size() != 1) return false;
  if (getenv("OWQS_DECIDE_AHEAD") && atoi(getenv("OWQS_DECIDE_AHEAD")) == 0) return false;
  for (size_t i = 0; i < m.prog.steps.size(); ++i) {
    const StepDesc& s = m.prog.steps[i];
    if (s.kind != ST_PASS) return false;
    if (s.n_ops > 0 && (!m.jit_fn[i] || jit_engine(s, ctx->prec) != 2 || jit_tile_small(s, ctx->prec) ||
                        s.first_uses_red || !m.cp_sym[i]))
      return false;
  }
  return true;
}

// kernel launches of one run (per shard): every step, plus the decide kernel of each tile pass
// (or, with decisions ahead, the two decide-ahead kernels per run)
double kernels_per_run(const owqs_ctx* ctx, const CompiledMode& m) {
  if (&m == &ctx->cm[0] && !m.jit_fn.empty() && decide_ahead_ok(ctx, m)) {
    double n = 2;
    for (const StepDesc& s : m.prog.steps) n += 1 + (s.red_kind != RED_NONE ? 1 : 0);
    return n + 1.0 + ((ctx->hp.n_measure > 0 ? 2.0 : 0.0) + 1.0);
  }
  double n = 0;
  for (size_t i = 0; i < m.prog.steps.size(); ++i) {
    const StepDesc& s = m.prog.steps[i];
    n += 1;
    if (i < m.jit_name.size() && !m.jit_name[i].empty() && jit_engine(s, ctx->prec) == 2 &&
        !jit_tile_small(s, ctx->prec))  // decide (not in EOWQS runs after the first) + grid finish
      n += (m.pc_static_ready && !getenv("OWQS_EOWQS_DECIDE") ? 0 : 1) + (s.red_kind != RED_NONE ? 1 : 0);
  }
  // the run's readbacks (launch_readback: error flag per shard, outcomes + prob0, reduction)
  return n + 1.0 + ((ctx->hp.n_measure > 0 ? 2.0 : 0.0) + 1.0) / (double)std::max<size_t>(1, ctx->shards.size());
}

owqs_status fail(owqs_ctx* c, owqs_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? OWQS_E_NOMEM : OWQS_E_CUDA,      \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

#define NC(call)                                                                              \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) return fail(ctx, OWQS_E_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

DevPtrs dev_ptrs(owqs_ctx* ctx, const CompiledMode& m, int i) {
  DevPtrs p{};
  const Shard& s = ctx->shards[i];
  p.state = s.d_state;
  p.mst = m.d_mst;
  p.outcome = ctx->d_outcome;
  p.prob0 = ctx->d_prob0;
  p.forced = ctx->d_forced;
  p.sig_pool = m.d_sig;
  p.run = ctx->d_run;
  p.partials = s.d_partials;
  p.counter = s.d_counter;
  p.red_result = s.d_red;
  p.err = s.d_err;
  p.rank = ctx->shard_rank(i);
  p.local_width = m.prog.phys_bits - ctx->n_global;
  p.scratch = ctx->d_jscratch;
  return p;
}

void free_mode(CompiledMode& m) {
  if (m.gexec) cudaGraphExecDestroy(m.gexec);
  for (cudaLibrary_t l : m.jit_libs) cudaLibraryUnload(l);
  if (m.d_mst) cudaFree(m.d_mst);
  if (m.d_sig) cudaFree(m.d_sig);
  if (m.d_steps) cudaFree(m.d_steps);
  if (m.d_pc) cudaFree(m.d_pc);
  if (m.d_devnodes) cudaFree(m.d_devnodes);
  if (m.d_static_cp) cudaFree(m.d_static_cp);
  m = CompiledMode();
}

// EOWQS decisions of one tile pass (every outcome 0, no probabilities; reading R-15: the
// corrections are dropped, so every signal is 0 and Eq. 2 gives theta = alpha): what decide_kernel
// computes in mode 2 (device_common.cuh pass_prologue), fixed by the pattern alone -- the butterfly
// coefficient a = e^{-i alpha}, k = 1/sqrt2 per slot-reuse butterfly (1 for an elimination), the
// pass scale = prod k, conditional ops off. Set once as the graph nodes' PassCoef parameter.
void static_eowqs_coef(const StepDesc& d, const std::vector<MStatic>& mst, PassCoef& c) {
  c = PassCoef{};
  double scale = 1.0;
  int b = 0;
  for (int i = 0; i < d.n_ops; ++i) {
    const Op& op = d.ops[i];
    if (op.type != OP_BFLY) {
      c.cond[i] = op.cond ? 0 : 1;
      continue;
    }
    c.cond[i] = 1;
    const MStatic& ms = mst[op.m];
    const double ar = std::cos(ms.alpha), ai = -std::sin(ms.alpha);
    scale *= ms.reuse ? 0.70710678118654752440 : 1.0;
    c.ard[b] = ar;
    c.aid[b] = ai;
    c.ar[b] = (float)ar;
    const float fai = (float)ai, nfai = -fai;
    uint32_t uh, ul;
    memcpy(&uh, &fai, 4);
    memcpy(&ul, &nfai, 4);
    c.B[b] = ((uint64_t)uh << 32) | ul;
    ++b;
  }
  c.scale = scale;
}

// Where the tile kernels read their decisions (jit.h COEF_*): OWQS_FLAG_NO_GRAPH -> the pointer;
// else OWQS_COEF_SRC=ptr|param|const (default const)
int coef_source(uint32_t flags) {
  if (flags & OWQS_FLAG_NO_GRAPH) return COEF_POINTER;
  const char* e = getenv("OWQS_COEF_SRC");
  if (e && !strcmp(e, "ptr")) return COEF_POINTER;
  if (e && !strcmp(e, "param")) return COEF_PARAM;
  return COEF_CONST;
}

void drop_graphs(owqs_ctx* ctx) {
  for (int i = 0; i < 2; ++i)
    if (ctx->cm[i].gexec) {
      cudaGraphExecDestroy(ctx->cm[i].gexec);
      ctx->cm[i].gexec = nullptr;
    }
}

owqs_status compile_modes(owqs_ctx* ctx) {
  const int SB = ctx->prec == 0 ? 6 : 5;
  const bool fuse = !(ctx->cfg.flags & OWQS_FLAG_NO_FUSE);
  const bool given = (ctx->cfg.flags & OWQS_FLAG_GIVEN_ORDER) != 0;
  ProaWeights w = ctx->weights;
  if (ctx->cfg.flags & OWQS_FLAG_NO_TUNE) w.tune = false;
  for (int i = 0; i < 2; ++i) {
    free_mode(ctx->cm[i]);
    auto t0 = std::chrono::steady_clock::now();
    CompiledMode& m = ctx->cm[i];
    plan_and_compile(ctx->hp, i == 1 ? 2 : 0, SB, fuse, given, w, m.plan, m.prog, ctx->n_global,
                     jit_max_group(ctx->prec, (ctx->cfg.flags & OWQS_FLAG_NO_JIT) != 0),
                     (ctx->cfg.flags & OWQS_FLAG_MEASURED_NORM) != 0);
    if (!m.prog.error.empty()) return fail(ctx, OWQS_E_ARG, m.prog.error);
    m.schedule_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    m.valid = true;
  }
  // generated pass kernels of both modes, compiled together (one NVRTC batch, process cache)
  ctx->jit_ms = 0;
  if (!(ctx->cfg.flags & OWQS_FLAG_NO_JIT)) {
    std::vector<std::string> names, srcs;
    for (int i = 0; i < 2; ++i) {
      CompiledMode& m = ctx->cm[i];
      m.jit_name.assign(m.prog.steps.size(), std::string());
      for (size_t k = 0; k < m.prog.steps.size(); ++k) {
        if (!jit_eligible(m.prog.steps[k], ctx->prec)) continue;
        std::string nm;
        // graph launches (the default) take the decisions as kernel parameters; direct launches
        // (OWQS_FLAG_NO_GRAPH) read them from the PassCoef pointer
        m.coef_src = coef_source(ctx->cfg.flags);
        m.coefp = m.coef_src != COEF_POINTER;
        std::string src = jit_pass_source(m.prog.steps[k], ctx->prec, &nm, m.coef_src);
        if (src.empty()) return fail(ctx, OWQS_E_ARG, "pass kernel generation failed for step " + std::to_string(k));
        m.jit_name[k] = nm;
        ++m.n_jit;
        names.push_back(nm);
        srcs.push_back(src);
      }
    }
    std::vector<JitModule> mods;
    std::string e = jit_compile(names, srcs, mods, &ctx->jit_ms);
    if (!e.empty()) return fail(ctx, OWQS_E_ARG, "pass kernel compilation (NVRTC, sm_100a) failed: " + e);
    for (int i = 0; i < 2; ++i) ctx->cm[i].jit_mods = mods;  // each mode loads what it uses
  }
  if (ctx->n_global > 0 && ctx->cm[0].prog.phys_bits != ctx->cm[1].prog.phys_bits)
    return fail(ctx, OWQS_E_ARG, "multi-rank: OWQS and EOWQS programs differ in width");
  return OWQS_OK;
}

owqs_status ensure_device(owqs_ctx* ctx) {
  CU(cudaSetDevice(ctx->cfg.device));
  int phys = 0;
  for (int i = 0; i < 2; ++i) phys = std::max(phys, ctx->cm[i].prog.phys_bits);
  const int wl = phys - ctx->n_global;
  size_t need = std::max<size_t>((size_t)ctx->elem << wl, 64);
  if (ctx->shard_bytes < need) {
    drop_graphs(ctx);
    for (auto& s : ctx->shards) {
      cudaFree(s.d_state);
      s.d_state = nullptr;
    }
    cudaFree(ctx->d_swap);
    ctx->d_swap = nullptr;
    ctx->shard_bytes = 0;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t total_need = need * ctx->shards.size() + (ctx->n_global > 0 ? need : 0);
    if (total_need > free_b)
      return fail(ctx, OWQS_E_NOMEM, "state shard(s) of 2^" + std::to_string(wl) + " amplitudes (" +
                                         std::to_string(total_need >> 20) + " MiB) exceed free device memory");
    for (auto& s : ctx->shards) CU(cudaMalloc(&s.d_state, need));
    if (ctx->n_global > 0) CU(cudaMalloc(&ctx->d_swap, need));  // two halves: send | receive
    ctx->shard_bytes = need;
  }
  size_t jneed = 0;
  for (int i = 0; i < 2; ++i)
    for (const StepDesc& sd : ctx->cm[i].prog.steps)
      if (sd.kind == ST_SHRINKK) jneed = std::max(jneed, (size_t)ctx->elem << (sd.width - sd.jk));
  if (ctx->jscratch_bytes < jneed) {
    drop_graphs(ctx);
    cudaFree(ctx->d_jscratch);
    ctx->d_jscratch = nullptr;
    ctx->jscratch_bytes = 0;
    if (cudaMalloc(&ctx->d_jscratch, jneed) != cudaSuccess)
      return fail(ctx, OWQS_E_NOMEM, "joint-measurement scratch of " + std::to_string(jneed >> 20) + " MiB");
    ctx->jscratch_bytes = jneed;
  }
  size_t K = std::max<size_t>(1, (size_t)ctx->hp.n_measure);
  if (ctx->k_cap < K) {
    cudaFree(ctx->d_outcome);
    cudaFree(ctx->d_prob0);
    cudaFree(ctx->d_forced);
    CU(cudaMalloc(&ctx->d_outcome, K));
    CU(cudaMalloc(&ctx->d_prob0, K * sizeof(double)));
    CU(cudaMalloc(&ctx->d_forced, K));
    CU(cudaMemset(ctx->d_outcome, 0, K));
    ctx->k_cap = K;
    drop_graphs(ctx);
  }
  for (int i = 0; i < 2; ++i) {
    CompiledMode& m = ctx->cm[i];
    if (!m.d_mst && !m.prog.mst.empty()) {
      CU(cudaMalloc(&m.d_mst, m.prog.mst.size() * sizeof(MStatic)));
      CU(cudaMemcpy(m.d_mst, m.prog.mst.data(), m.prog.mst.size() * sizeof(MStatic), cudaMemcpyHostToDevice));
    }
    if (!m.d_sig && !m.prog.sig_pool.empty()) {
      CU(cudaMalloc(&m.d_sig, m.prog.sig_pool.size() * sizeof(int32_t)));
      CU(cudaMemcpy(m.d_sig, m.prog.sig_pool.data(), m.prog.sig_pool.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    if (m.n_jit > 0 && !m.d_pc) CU(cudaMalloc(&m.d_pc, m.prog.steps.size() * sizeof(PassCoef)));
    if (m.n_jit > 0 && m.coef_src == COEF_PARAM && !m.d_devnodes) {
      CU(cudaMalloc(&m.d_devnodes, m.prog.steps.size() * ctx->shards.size() * sizeof(cudaGraphDeviceNode_t)));
      CU(cudaMemset(m.d_devnodes, 0, m.prog.steps.size() * ctx->shards.size() * sizeof(cudaGraphDeviceNode_t)));
    }
    if (m.n_jit > 0 && m.jit_fn.empty()) {
      std::vector<cudaKernel_t> fn(m.prog.steps.size(), nullptr);
      std::vector<int> blocks(m.prog.steps.size(), 0);
      int sms = 0;
      CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->cfg.device));
      for (const JitModule& jm : m.jit_mods) {
        bool used = false;
        for (const std::string& n : jm.names)
          for (const std::string& want : m.jit_name) used = used || (n == want);
        if (!used) continue;
        cudaLibrary_t lib = nullptr;
        CU(cudaLibraryLoadData(&lib, jm.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
        m.jit_libs.push_back(lib);
        for (size_t k = 0; k < m.jit_name.size(); ++k) {
          if (m.jit_name[k].empty() || fn[k]) continue;
          if (std::find(jm.names.begin(), jm.names.end(), m.jit_name[k]) == jm.names.end()) continue;
          CU(cudaLibraryGetKernel(&fn[k], lib, m.jit_name[k].c_str()));
          if (m.coef_src == COEF_CONST && jit_engine(m.prog.steps[k], ctx->prec) == 2 &&
              !jit_tile_small(m.prog.steps[k], ctx->prec)) {
            if (m.cp_sym.empty()) m.cp_sym.assign(m.prog.steps.size(), nullptr);
            size_t bytes = 0;
            CU(cudaLibraryGetGlobal(&m.cp_sym[k], &bytes, lib, (m.jit_name[k] + "_cp").c_str()));
            if (bytes != sizeof(PassCoef)) return fail(ctx, OWQS_E_CUDA, "generated kernel " + m.jit_name[k] + ": bad _cp symbol");
          }
          const int eng = jit_engine(m.prog.steps[k], ctx->prec);
          const int dyn = jit_dyn_smem(eng, ctx->prec);
          if (dyn > 0) {
            CU(cudaFuncSetAttribute((const void*)fn[k], cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
            // shared-memory carveout just large enough for the CTAs the registers allow: the rest
            // stays L1, which stages the in-flight global loads (a max-shared carveout, L1 <= 32 KB,
            // costs 19 % of streaming bandwidth: profiles/r01b/overlap_bench.log)
            CU(cudaFuncSetAttribute((const void*)fn[k], cudaFuncAttributePreferredSharedMemoryCarveout,
                                    jit_smem_carveout(eng, ctx->prec)));
          }
          int nb = 0;
          CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)fn[k], jit_block_threads(eng, ctx->prec), dyn));
          blocks[k] = std::max(1, nb) * sms;
        }
      }
      for (size_t k = 0; k < m.jit_name.size(); ++k)
        if (!m.jit_name[k].empty() && !fn[k])
          return fail(ctx, OWQS_E_CUDA, "generated kernel " + m.jit_name[k] + " missing from its cubin");
      m.coef_off.assign(m.prog.steps.size(), (size_t)-1);
      m.static_cp.assign(i == 1 ? m.prog.steps.size() : 0, PassCoef{});
      for (size_t k = 0; k < m.jit_name.size(); ++k) {
        const StepDesc& sd = m.prog.steps[k];
        if (!fn[k] || jit_engine(sd, ctx->prec) != 2 || jit_tile_small(sd, ctx->prec)) continue;
        m.coef_off[k] = jit_coef_param_offset(fn[k]);
        if (m.coef_src == COEF_PARAM && m.coef_off[k] == (size_t)-1)
          return fail(ctx, OWQS_E_CUDA, "generated kernel " + m.jit_name[k] + ": no PassCoef parameter");
        if (i == 1) static_eowqs_coef(sd, m.prog.mst, m.static_cp[k]);
      }
      if (m.coef_src == COEF_CONST && i == 1 && !m.cp_sym.empty()) {
        // EOWQS: run-independent decisions; a kernel used by one step only gets them once here,
        // shared kernels get a memcpy node per run from d_static_cp
        CU(cudaMalloc(&m.d_static_cp, m.prog.steps.size() * sizeof(PassCoef)));
        CU(cudaMemcpy(m.d_static_cp, m.static_cp.data(), m.prog.steps.size() * sizeof(PassCoef), cudaMemcpyHostToDevice));
        m.cp_once.assign(m.prog.steps.size(), 0);
        for (size_t k = 0; k < m.cp_sym.size(); ++k) {
          if (!m.cp_sym[k]) continue;
          int uses = 0;
          for (size_t j = 0; j < m.cp_sym.size(); ++j) uses += m.cp_sym[j] == m.cp_sym[k];
          if (uses == 1) {
            CU(cudaMemcpy(m.cp_sym[k], &m.static_cp[k], sizeof(PassCoef), cudaMemcpyHostToDevice));
            m.cp_once[k] = 1;
          }
        }
      }
      m.jit_fn = fn;
      m.jit_blocks = blocks;
    }
  }
  return OWQS_OK;
}

// all-reduce of every shard's red_result (sum over ranks)
owqs_status allreduce_red(owqs_ctx* ctx) {
  if (ctx->n_ranks == 1) return OWQS_OK;
  if (ctx->loopback) {
    CU(launch_loopback_allreduce(ctx->d_red_all, ctx->n_ranks, ctx->stream));
  } else {
    NC(ncclAllReduce(ctx->d_red_all, ctx->d_red_all, 4, ncclDouble, ncclSum, ctx->comm, ctx->stream));
  }
  return OWQS_OK;
}

// ST_SWAP: every rank trades the half of its shard whose bit `pl` = 1 - (its rank bit) with rank ^ m
// swap chunk: a power of two of elements, ~256 MiB, at most 16 chunks per half-shard (OWQS_SWAP_CHUNK_MB)
uint64_t swap_chunk_elems(const owqs_ctx* ctx, uint64_t half_elems) {
  static const uint64_t mb = getenv("OWQS_SWAP_CHUNK_MB") ? (uint64_t)std::max(1, atoi(getenv("OWQS_SWAP_CHUNK_MB"))) : 256;
  uint64_t c = 1;
  while (c < half_elems && c * ctx->elem < (mb << 20)) c <<= 1;
  while (half_elems / c > 16) c <<= 1;
  return std::min(c, std::max<uint64_t>(1, half_elems / 2));  // >= 2 chunks: 4 slots fit in one shard
}

// ST_SWAP: every rank trades the half of its shard whose bit `pl` = 1 - (its rank bit) with
// rank ^ 2^g, in chunks of swap_chunk_elems: pack chunk c into send slot c % 2 (stream), transfer it
// (comm_stream: ncclSend of the slot, ncclRecv into receive slot c % 2), unpack it (stream) -- the
// transfer of chunk c overlaps the pack of chunk c + 1 and the unpack of chunk c - 1, and a slot is
// reused only after its transfer (send) or its unpack (receive) is done. The loopback backend runs
// the same chunk loop with device copies on one stream.
owqs_status do_swap(owqs_ctx* ctx, const StepDesc& d) {
  NvtxRange nvtx_("owqs: global<->local qubit swap");
  const int wl = d.width, pl = d.swap_local, gbit = d.swap_global - wl;
  const uint64_t half_elems = 1ull << (wl - 1);
  const uint64_t ce = swap_chunk_elems(ctx, half_elems), nch = half_elems / ce;
  const size_t cb = (size_t)ce * ctx->elem;
  char* base = (char*)ctx->d_swap;  // 4 slots of cb bytes: send 0, send 1, receive 0, receive 1 (4 cb <= one shard)
  char* send[2] = {base, base + cb};
  char* recv[2] = {base + 2 * cb, base + 3 * cb};
  if (ctx->loopback) {
    for (int r = 0; r < ctx->n_ranks; ++r) {
      const int p = r ^ (1 << gbit);
      if (p < r) continue;  // r has rank bit 0 (trades its bit-pl = 1 half), p has 1 (bit-pl = 0 half)
      for (uint64_t c = 0; c < nch; ++c) {
        const uint64_t j0 = c * ce;
        CU(launch_swap_pack(ctx->shards[r].d_state, send[c & 1], ctx->prec, pl, 1, false, j0, ce, ctx->stream));
        CU(launch_swap_pack(ctx->shards[p].d_state, recv[c & 1], ctx->prec, pl, 0, false, j0, ce, ctx->stream));
        CU(launch_swap_pack(ctx->shards[r].d_state, recv[c & 1], ctx->prec, pl, 1, true, j0, ce, ctx->stream));
        CU(launch_swap_pack(ctx->shards[p].d_state, send[c & 1], ctx->prec, pl, 0, true, j0, ce, ctx->stream));
      }
    }
    return OWQS_OK;
  }
  const int b = (ctx->rank >> gbit) & 1, partner = ctx->rank ^ (1 << gbit);
  for (uint64_t c = 0; c < nch; ++c) {
    const int k = (int)(c & 1);
    const uint64_t j0 = c * ce;
    if (c >= 2) CU(cudaStreamWaitEvent(ctx->stream, ctx->sw_sent[k], 0));  // send slot k free again
    CU(launch_swap_pack(ctx->shards[0].d_state, send[k], ctx->prec, pl, 1 - b, false, j0, ce, ctx->stream));
    CU(cudaEventRecord(ctx->sw_packed[k], ctx->stream));
    CU(cudaStreamWaitEvent(ctx->comm_stream, ctx->sw_packed[k], 0));
    if (c >= 2) CU(cudaStreamWaitEvent(ctx->comm_stream, ctx->sw_unpacked[k], 0));  // receive slot k free
    NC(ncclGroupStart());
    NC(ncclSend(send[k], cb, ncclChar, partner, ctx->comm, ctx->comm_stream));
    NC(ncclRecv(recv[k], cb, ncclChar, partner, ctx->comm, ctx->comm_stream));
    NC(ncclGroupEnd());
    CU(cudaEventRecord(ctx->sw_sent[k], ctx->comm_stream));
    CU(cudaStreamWaitEvent(ctx->stream, ctx->sw_sent[k], 0));
    CU(launch_swap_pack(ctx->shards[0].d_state, recv[k], ctx->prec, pl, 1 - b, true, j0, ce, ctx->stream));
    CU(cudaEventRecord(ctx->sw_unpacked[k], ctx->stream));
  }
  return OWQS_OK;
}

// Page-locked staging layout for one run: RunParams at 0, forced outcomes at 4096, then the run's
// readbacks (outcomes, prob0, the reduction result) copied in stream order right after the run.
struct RunStaging {
  size_t forced = 4096, outcomes, prob0, red, end;
  explicit RunStaging(int64_t K) {
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    outcomes = forced + up((size_t)std::max<int64_t>(K, 1));
    prob0 = outcomes + up((size_t)std::max<int64_t>(K, 1));
    red = prob0 + up((size_t)std::max<int64_t>(K, 1) * sizeof(double));
    end = red + 4 * sizeof(double);
  }
};

// Enqueue one run on ctx->stream without synchronising the host (run parameters and forced
// outcomes go through the page-locked staging buffer, so the copies are truly asynchronous; no
// earlier copy from it is pending because every call ends synchronised or with owqs_wait).
owqs_status run_enqueue(owqs_ctx* ctx, int cmi, int mode, uint64_t seed, const uint8_t* forced) {
  CompiledMode& m = ctx->cm[cmi];
  RunParams* rp = reinterpret_cast<RunParams*>(ctx->h_staging);
  *rp = RunParams{};
  rp->mode = mode;
  rp->seed = seed;
  CU(cudaMemcpyAsync(ctx->d_run, rp, sizeof(RunParams), cudaMemcpyHostToDevice, ctx->stream));
  const RunStaging rs(ctx->hp.n_measure);
  if (rs.end > kStagingBytes) return fail(ctx, OWQS_E_ARG, "too many measurements");
  if (mode == OWQS_FORCED && ctx->hp.n_measure > 0) {
    uint8_t* hf = static_cast<uint8_t*>(ctx->h_staging) + rs.forced;
    memcpy(hf, forced, ctx->hp.n_measure);
    CU(cudaMemcpyAsync(ctx->d_forced, hf, ctx->hp.n_measure, cudaMemcpyHostToDevice, ctx->stream));
  }
  for (auto& s : ctx->shards) CU(cudaMemsetAsync(s.d_err, 0, sizeof(int32_t), ctx->stream));
  // Decisions of the tile passes. coefp (graph launches): the sampled / forced graph's decide kernels
  // write them into the device-updatable pass-kernel nodes; EOWQS's are run-independent and set by
  // the host at capture, no decide kernel at all. Otherwise (OWQS_FLAG_NO_GRAPH) the kernels read
  // d_pc; EOWQS after its first run reuses it (CompiledMode::pc_static_ready) -- that first run
  // launches directly so that no captured graph contains the decide kernels.
  const bool eowqs_static = mode == OWQS_EOWQS && m.coefp;
  const bool static_pc = eowqs_static || (mode == OWQS_EOWQS && m.pc_static_ready && !getenv("OWQS_EOWQS_DECIDE"));
  const bool use_graph = !(ctx->cfg.flags & OWQS_FLAG_NO_GRAPH) && (mode != OWQS_EOWQS || static_pc);
  // decide ahead (sampled / forced, constant-bank coefficients): every step a tile pass whose
  // decisions are structural (no reduction feeds them, no SHRINK) -> one decide_ahead_kernel for
  // the whole run, the copies into the kernels' __constant__ up front, the pass kernels back to back
  // (OWQS_DECIDE_AHEAD=0: per-pass decide kernels)
  const bool ahead = mode != OWQS_EOWQS && decide_ahead_ok(ctx, m);
  if (ahead && !m.d_steps) {
    CU(cudaMalloc(&m.d_steps, std::max<size_t>(1, m.prog.steps.size()) * sizeof(StepDesc)));
    CU(cudaMemcpy(m.d_steps, m.prog.steps.data(), m.prog.steps.size() * sizeof(StepDesc), cudaMemcpyHostToDevice));
  }
  const bool dev_update = m.coef_src == COEF_PARAM && !eowqs_static;  // sampled / forced: device node updates
  const size_t NS = ctx->shards.size();
  std::vector<cudaGraphDeviceNode_t> hnodes(dev_update ? m.prog.steps.size() * NS : 0, nullptr);
  if (m.coefp && !use_graph) return fail(ctx, OWQS_E_STATE, "parameter-coefficient kernels need a CUDA graph");
  const bool prof = (ctx->cfg.flags & OWQS_FLAG_PROFILE) != 0;
  if (prof) {
    if (ctx->prof_cm != cmi && m.gexec) {  // event lists follow the compiled mode
      cudaGraphExecDestroy(m.gexec);
      m.gexec = nullptr;
    }
    while (ctx->prof_ev.size() < m.prog.steps.size() + 1) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      ctx->prof_ev.push_back(e);
    }
    ctx->prof_cm = cmi;
  }
  auto record = [&](int i, bool capturing) -> cudaError_t {
    return capturing ? cudaEventRecordWithFlags(ctx->prof_ev[i], ctx->stream, cudaEventRecordExternal)
                     : cudaEventRecord(ctx->prof_ev[i], ctx->stream);
  };
  // a kernel shared by several steps gets its constants copied right before each use
  auto shared_sym = [&](size_t i) {
    for (size_t j = 0; j < m.cp_sym.size(); ++j)
      if (j != i && m.cp_sym[j] == m.cp_sym[i]) return true;
    return false;
  };
  auto launch_all = [&](bool capturing) -> owqs_status {
    if (prof) CU(record(0, capturing));
    if (ahead) {
      CU(launch_decide_ahead(m.d_steps, (int)m.prog.steps.size(), (int)m.prog.mst.size(), dev_ptrs(ctx, m, 0), m.d_pc,
                             ctx->stream));
      std::vector<size_t> cp;
      for (size_t i = 0; i < m.prog.steps.size(); ++i)
        if (m.prog.steps[i].n_ops > 0 && !shared_sym(i)) cp.push_back(i);
      const int K = owqs_ctx::kAux;
      if (capturing && cp.size() > (size_t)K) {
        if (!ctx->fork_ev) {
          CU(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
          for (int a = 0; a < K; ++a) {
            CU(cudaStreamCreateWithFlags(&ctx->aux[a], cudaStreamNonBlocking));
            CU(cudaEventCreateWithFlags(&ctx->join_ev[a], cudaEventDisableTiming));
          }
        }
        CU(cudaEventRecord(ctx->fork_ev, ctx->stream));
        for (int a = 0; a < K; ++a) CU(cudaStreamWaitEvent(ctx->aux[a], ctx->fork_ev, 0));
        for (size_t k = 0; k < cp.size(); ++k)
          CU(cudaMemcpyAsync(m.cp_sym[cp[k]], m.d_pc + cp[k], sizeof(PassCoef), cudaMemcpyDeviceToDevice,
                             ctx->aux[k % K]));
        for (int a = 0; a < K; ++a) {
          CU(cudaEventRecord(ctx->join_ev[a], ctx->aux[a]));
          CU(cudaStreamWaitEvent(ctx->stream, ctx->join_ev[a], 0));
        }
      } else {
        for (size_t i : cp)
          CU(cudaMemcpyAsync(m.cp_sym[i], m.d_pc + i, sizeof(PassCoef), cudaMemcpyDeviceToDevice, ctx->stream));
      }
    }
    bool first_tile = true;  // decide ahead: the first pass kernel follows the copies (no PDL edge)
    for (size_t i = 0; i < m.prog.steps.size(); ++i) {
      const StepDesc& s = m.prog.steps[i];
      if (s.kind == ST_SWAP) {
        owqs_status st = do_swap(ctx, s);
        if (st != OWQS_OK) return st;
      } else {
        const bool jit = !m.jit_fn.empty() && m.jit_fn[i];
        const int eng = jit ? jit_engine(s, ctx->prec) : 0;
        const bool small = eng == 2 && jit_tile_small(s, ctx->prec);
        const bool upd = dev_update && eng == 2 && !small;
        if (eng == 2 && !small && !static_pc && !ahead)
          CU(launch_decide(s, dev_ptrs(ctx, m, 0), m.d_pc + i, ctx->stream, upd ? m.d_devnodes + i * NS : nullptr,
                           upd ? (int)NS : 0, upd ? m.coef_off[i] : 0));
        // COEF_CONST: the pass's decisions into its kernel's __constant__ (graph memcpy node)
        bool after_copy = false;
        if (m.coef_src == COEF_CONST && eng == 2 && !small && !m.cp_sym.empty() && m.cp_sym[i]) {
          const PassCoef* src = eowqs_static ? (m.cp_once.empty() || m.cp_once[i] ? nullptr : m.d_static_cp + i)
                                : (ahead && !shared_sym(i)) ? nullptr : m.d_pc + i;
          if (src) {
            CU(cudaMemcpyAsync(m.cp_sym[i], src, sizeof(PassCoef), cudaMemcpyDeviceToDevice, ctx->stream));
            after_copy = true;
          }
        }
        for (size_t r = 0; r < ctx->shards.size(); ++r) {
          if (jit)
            CU(jit_launch(m.jit_fn[i], m.jit_blocks[i], s, dev_ptrs(ctx, m, (int)r), m.d_pc + i, ctx->prec, ctx->stream,
                          (eowqs_static && eng == 2 && !small) ? &m.static_cp[i] : nullptr,
                          (upd && capturing) ? &hnodes[i * NS + r] : nullptr,
                          (after_copy || (ahead && first_tile)) && r == 0));
          else
            CU(launch_step(s, dev_ptrs(ctx, m, (int)r), ctx->prec, ctx->stream));
        }
        if (jit) first_tile = false;
        if (eng == 2 && !small && s.red_kind != RED_NONE)  // tile passes leave block partials
          for (size_t r = 0; r < ctx->shards.size(); ++r)
            CU(launch_grid_finish(dev_ptrs(ctx, m, (int)r), jit_tile_blocks(s, ctx->prec),
                                  s.red_kind == RED_NORM ? 1 : 4, ctx->stream));
        if (s.red_kind != RED_NONE) {
          owqs_status st = allreduce_red(ctx);
          if (st != OWQS_OK) return st;
        }
      }
      if (prof) CU(record((int)i + 1, capturing));
    }
    return OWQS_OK;
  };
  if (use_graph && !m.gexec) {
    cudaGraph_t g = nullptr;
    CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    owqs_status st = launch_all(true);
    if (st != OWQS_OK) {
      cudaStreamEndCapture(ctx->stream, &g);
      if (g) cudaGraphDestroy(g);
      return st;
    }
    CU(cudaStreamEndCapture(ctx->stream, &g));
    CU(cudaGraphInstantiate(&m.gexec, g, 0));
    cudaGraphDestroy(g);
    if (dev_update) {
      // handles of the device-updatable pass-kernel nodes for their decide kernels; a graph whose
      // nodes are updated from the device must be uploaded before it is launched
      CU(cudaMemcpyAsync(m.d_devnodes, hnodes.data(), hnodes.size() * sizeof(cudaGraphDeviceNode_t),
                         cudaMemcpyHostToDevice, ctx->stream));
      CU(cudaGraphUpload(m.gexec, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
    }
  }
  CU(cudaEventRecord(ctx->ev0, ctx->stream));
  if (use_graph) {
    CU(cudaGraphLaunch(m.gexec, ctx->stream));
  } else {
    owqs_status st = launch_all(false);
    if (st != OWQS_OK) return st;
  }
  CU(cudaEventRecord(ctx->ev1, ctx->stream));
  // error flags, outcomes, prob0 and the reduction to page-locked memory in stream order, written by
  // a one-CTA kernel (launch_readback): a copy-engine D2H would queue behind other contexts'
  // multi-GiB output transfers
  for (size_t r = 0; r < ctx->shards.size(); ++r)
    CU(launch_readback(ctx->h_err + r, ctx->shards[r].d_err, sizeof(int32_t), ctx->stream));
  {
    uint8_t* hs = static_cast<uint8_t*>(ctx->h_staging);
    const int64_t K = ctx->hp.n_measure;
    if (K > 0) {
      CU(launch_readback(hs + rs.outcomes, ctx->d_outcome, K, ctx->stream));
      CU(launch_readback(hs + rs.prob0, ctx->d_prob0, K * sizeof(double), ctx->stream));
    }
    CU(launch_readback(hs + rs.red, ctx->shards[0].d_red, 4 * sizeof(double), ctx->stream));
  }
  ctx->has_input = false;
  ctx->out_cm = cmi;
  return OWQS_OK;
}

// Wait for the enqueued run (and whatever follows it on the stream), then its time and error flag.
owqs_status run_complete(owqs_ctx* ctx, int cmi) {
  CU(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  ctx->stats.last_run_ms = ms;
  ctx->last_cm = cmi;
  int32_t herr = 0;
  for (size_t r = 0; r < ctx->shards.size(); ++r) herr |= ctx->h_err[r];
  ctx->has_output = true;
  if (herr & 2) return fail(ctx, OWQS_E_CUDA, "device-side update of a pass kernel's graph node failed");
  if (herr) return fail(ctx, OWQS_E_BRANCH, "forced outcome on a branch with probability < 1e-12");
  if (cmi == 1) ctx->cm[1].pc_static_ready = true;  // the EOWQS mode's decisions are in d_pc
  return OWQS_OK;
}

owqs_status run_internal(owqs_ctx* ctx, int cmi, int mode, uint64_t seed, const uint8_t* forced) {
  owqs_status s = run_enqueue(ctx, cmi, mode, seed, forced);
  if (s != OWQS_OK) return s;
  return run_complete(ctx, cmi);
}

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// output (complex128 when dst_prec = 1) in the caller's order into a device buffer of 2^n_out
owqs_status output_to_device_full(owqs_ctx* ctx, void* dst, int dst_prec) {
  const Program& pr = ctx->cm[ctx->out_cm].prog;
  const int nb = (int)pr.out_slot.size();
  const int wl = pr.phys_bits - ctx->n_global;
  if (ctx->n_ranks == 1) {
    CU(launch_permute_out(ctx->shards[0].d_state, ctx->prec, dst, dst_prec, nb, pr.out_slot.data(), 0, 1ull << nb,
                          ctx->stream));
    return OWQS_OK;
  }
  if (ctx->loopback) {
    for (int r = 0; r < ctx->n_ranks; ++r)
      CU(launch_scatter_out(ctx->shards[r].d_state, ctx->prec, dst, dst_prec, nb, pr.out_slot.data(), r, wl,
                            ctx->stream));
    return OWQS_OK;
  }
  // NCCL: shards travel to rank 0 (through the swap buffer), which scatters them into dst
  if (ctx->rank == 0) {
    CU(launch_scatter_out(ctx->shards[0].d_state, ctx->prec, dst, dst_prec, nb, pr.out_slot.data(), 0, wl,
                          ctx->stream));
    for (int r = 1; r < ctx->n_ranks; ++r) {
      NC(ncclRecv(ctx->d_swap, (size_t)ctx->elem << wl, ncclChar, r, ctx->comm, ctx->stream));
      CU(launch_scatter_out(ctx->d_swap, ctx->prec, dst, dst_prec, nb, pr.out_slot.data(), r, wl, ctx->stream));
    }
  } else {
    NC(ncclSend(ctx->shards[0].d_state, (size_t)ctx->elem << wl, ncclChar, 0, ctx->comm, ctx->stream));
  }
  return OWQS_OK;
}

owqs_status output_to_host_enqueue(owqs_ctx* ctx, void* amps, int out_prec, bool pinned, bool sync);

owqs_status output_to_host(owqs_ctx* ctx, void* amps, int out_prec) {
  const uint64_t n = 1ull << ctx->hp.outputs.size();
  const size_t oe = out_prec == 1 ? 16 : 8;
  if (ctx->n_ranks > 1) {
    void* d = nullptr;
    if (ctx->rank == 0 || ctx->loopback) CU(cudaMalloc(&d, n * oe));
    owqs_status s = output_to_device_full(ctx, d, out_prec);
    if (s == OWQS_OK && d) {
      cudaError_t e = cudaMemcpyAsync(amps, d, n * oe, cudaMemcpyDeviceToHost, ctx->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
      if (e != cudaSuccess) s = fail(ctx, OWQS_E_CUDA, cudaGetErrorString(e));
    } else if (s == OWQS_OK) {
      cudaError_t e = cudaStreamSynchronize(ctx->stream);
      if (e != cudaSuccess) s = fail(ctx, OWQS_E_CUDA, cudaGetErrorString(e));
    }
    cudaFree(d);
    return s;
  }
  return output_to_host_enqueue(ctx, amps, out_prec, is_pinned_host(amps), true);
}

// Single-rank output in the caller's order into host memory: permute into the device staging buffer
// chunk by chunk and DMA each chunk out. A page-locked destination is written directly (fully
// asynchronous when sync = false); a pageable one goes through the pinned host staging buffer.
owqs_status output_to_host_enqueue(owqs_ctx* ctx, void* amps, int out_prec, bool pinned, bool sync) {
  const uint64_t n = 1ull << ctx->hp.outputs.size();
  const size_t oe = out_prec == 1 ? 16 : 8;
  const Program& pr = ctx->cm[ctx->out_cm].prog;
  const uint64_t chunk = kStagingBytes / oe;
  char* dst = (char*)amps;
  if (pinned) {
    // outputs already in the caller's order at the state's precision: one DMA from the state
    bool ident = out_prec == ctx->prec && pr.out_slot.size() == ctx->hp.outputs.size();
    for (size_t k = 0; ident && k < pr.out_slot.size(); ++k) ident = pr.out_slot[k] == (int)k;
    if (ident) {
      CU(cudaMemcpyAsync(dst, ctx->shards[0].d_state, n * oe, cudaMemcpyDeviceToHost, ctx->stream));
      if (sync) CU(cudaStreamSynchronize(ctx->stream));
      return OWQS_OK;
    }
    // asynchronous (owqs_submit_host): one permute kernel into a full-size device buffer and one
    // DMA, instead of 64 MB chunks alternating kernel / copy -- each small permute kernel would wait
    // for SM slots behind other contexts' pass kernels and stall this context's copy stream
    if (!sync && n * oe <= kFullOutMaxBytes) {
      if (ctx->out_full_bytes < n * oe) {
        cudaFree(ctx->d_out_full);
        ctx->d_out_full = nullptr;
        ctx->out_full_bytes = 0;
        if (cudaMalloc(&ctx->d_out_full, n * oe) == cudaSuccess) ctx->out_full_bytes = n * oe;
        else cudaGetLastError();
      }
      if (ctx->d_out_full) {
        CU(launch_permute_out(ctx->shards[0].d_state, ctx->prec, ctx->d_out_full, out_prec, (int)pr.out_slot.size(),
                              pr.out_slot.data(), 0, n, ctx->stream));
        CU(cudaMemcpyAsync(dst, ctx->d_out_full, n * oe, cudaMemcpyDeviceToHost, ctx->stream));
        return OWQS_OK;
      }
    }
  }
  for (uint64_t j0 = 0; j0 < n; j0 += chunk) {
    uint64_t cnt = std::min(chunk, n - j0);
    CU(launch_permute_out(ctx->shards[0].d_state, ctx->prec, ctx->d_staging, out_prec, (int)pr.out_slot.size(),
                          pr.out_slot.data(), j0, cnt, ctx->stream));
    CU(cudaMemcpyAsync(pinned ? (void*)(dst + j0 * oe) : ctx->h_staging, ctx->d_staging, cnt * oe,
                       cudaMemcpyDeviceToHost, ctx->stream));
    if (!pinned) {
      CU(cudaStreamSynchronize(ctx->stream));
      memcpy(dst + j0 * oe, ctx->h_staging, cnt * oe);
    }
  }
  if (sync) CU(cudaStreamSynchronize(ctx->stream));
  return OWQS_OK;
}

constexpr int kBatchMaxBytes = 64 << 10;  // shared-memory state of one replica

owqs_status run_batch_internal(owqs_ctx* ctx, int mode, int64_t nb, const double* inputs, const uint64_t* seeds,
                               const uint8_t* forced, double* outputs, uint8_t* outcomes, double* prob0) {
  const int cmi = mode == OWQS_EOWQS ? 1 : 0;
  CompiledMode& m = ctx->cm[cmi];
  const Program& pr = m.prog;
  const int K = ctx->hp.n_measure, ni = (int)ctx->hp.inputs.size(), no = (int)ctx->hp.outputs.size();
  if (ctx->n_ranks > 1) return fail(ctx, OWQS_E_ARG, "batched replicas run on a single rank");
  if (((size_t)ctx->elem << pr.phys_bits) > (size_t)kBatchMaxBytes)
    return fail(ctx, OWQS_E_ARG, "batched replicas need a physical width <= 12 (complex128: 12, complex64: 13)");
  // R-13 precondition on every replica's input (small widths: checked on the host)
  for (int64_t b = 0; b < nb; ++b) {
    double n2 = 0.0;
    const double* x = inputs + (size_t)b * (2ull << ni);
    for (uint64_t i = 0; i < (2ull << ni); ++i) n2 += x[i] * x[i];
    if (!(std::fabs(n2 - 1.0) <= 1e-9))
      return fail(ctx, OWQS_E_ARG, "batch input " + std::to_string(b) + " not normalised: ||psi||^2 = " + std::to_string(n2));
  }
  owqs_status s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  if (!m.d_steps) {
    CU(cudaMalloc(&m.d_steps, std::max<size_t>(1, pr.steps.size()) * sizeof(StepDesc)));
    CU(cudaMemcpy(m.d_steps, pr.steps.data(), pr.steps.size() * sizeof(StepDesc), cudaMemcpyHostToDevice));
  }
  const size_t in_b = (size_t)nb * (16ull << ni), out_b = (size_t)nb * (16ull << no);
  const size_t Kb = std::max<size_t>(1, (size_t)K) * nb;
  char *d_in = nullptr, *d_out = nullptr, *d_runs = nullptr, *d_oc = nullptr, *d_p0 = nullptr, *d_f = nullptr,
       *d_err = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_in); cudaFree(d_out); cudaFree(d_runs); cudaFree(d_oc); cudaFree(d_p0); cudaFree(d_f); cudaFree(d_err);
  };
  cudaError_t e = cudaMalloc(&d_in, in_b);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, out_b);
  if (e == cudaSuccess) e = cudaMalloc(&d_runs, nb * sizeof(RunParams));
  if (e == cudaSuccess) e = cudaMalloc(&d_oc, Kb);
  if (e == cudaSuccess) e = cudaMalloc(&d_p0, Kb * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_f, Kb);
  if (e == cudaSuccess) e = cudaMalloc(&d_err, nb * sizeof(int32_t));
  if (e != cudaSuccess) {
    cleanup();
    return fail(ctx, OWQS_E_NOMEM, "batch buffers");
  }
  std::vector<RunParams> rp(nb);
  for (int64_t b = 0; b < nb; ++b) {
    rp[b].mode = mode;
    rp[b].seed = seeds ? seeds[b] : 0;
  }
  e = cudaMemcpyAsync(d_in, inputs, in_b, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_runs, rp.data(), nb * sizeof(RunParams), cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess && mode == OWQS_FORCED && K > 0)
    e = cudaMemcpyAsync(d_f, forced, (size_t)K * nb, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_err, 0, nb * sizeof(int32_t), ctx->stream);
  DevPtrs base = dev_ptrs(ctx, m, 0);
  base.outcome = (uint8_t*)d_oc;
  base.prob0 = (double*)d_p0;
  base.forced = (const uint8_t*)d_f;
  base.run = (const RunParams*)d_runs;
  base.err = (int32_t*)d_err;
  if (e == cudaSuccess)
    e = launch_batch(m.d_steps, (int)pr.steps.size(), base, K, (int)nb, d_in, d_out, ni, no, pr.out_slot.data(),
                     pr.phys_bits, ctx->prec, ctx->stream);
  std::vector<int32_t> herr(nb, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(outputs, d_out, out_b, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess && outcomes && K > 0 && mode != OWQS_EOWQS)
    e = cudaMemcpyAsync(outcomes, d_oc, (size_t)K * nb, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess && prob0 && K > 0 && mode != OWQS_EOWQS)
    e = cudaMemcpyAsync(prob0, d_p0, (size_t)K * nb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(herr.data(), d_err, nb * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cleanup();
  if (e != cudaSuccess) return fail(ctx, OWQS_E_CUDA, std::string("batch: ") + cudaGetErrorString(e));
  if (mode == OWQS_EOWQS && K > 0) {
    if (outcomes) memset(outcomes, 0, (size_t)K * nb);
    if (prob0)
      for (size_t i = 0; i < (size_t)K * nb; ++i) prob0[i] = -1.0;
  }
  for (int64_t b = 0; b < nb; ++b)
    if (herr[b]) return fail(ctx, OWQS_E_BRANCH, "forced outcome on a branch with probability < 1e-12 (batch item " +
                                                     std::to_string(b) + ")");
  if (mode == OWQS_EOWQS) {
    const double tol = ctx->prec == 1 ? 1e-8 : 1e-3;
    const uint64_t nout = 1ull << no;
    for (int64_t b = 0; b < nb; ++b) {
      double n2 = 0;
      for (uint64_t j = 0; j < 2 * nout; ++j) n2 += outputs[2 * nout * b + j] * outputs[2 * nout * b + j];
      if (!(std::fabs(n2 - 1.0) <= tol))
        return fail(ctx, OWQS_E_NOT_DETERMINISTIC, "EOWQS batch item " + std::to_string(b) + " norm^2 = " +
                                                       std::to_string(n2) + ": the pattern is not deterministic");
    }
  }
  return OWQS_OK;
}

// L372: EOWQS only for patterns with a gflow ("otherwise ... reported as an incorrect one")
owqs_status gflow_gate(owqs_ctx* ctx) {
  if (ctx->cfg.flags & OWQS_FLAG_NO_GFLOW) return OWQS_OK;
  if (ctx->gflow_state == 0) {
    std::vector<int> layer;
    std::vector<std::vector<int>> g;
    ctx->gflow_msg = find_gflow(ctx->hp, layer, g);
    ctx->gflow_state = ctx->gflow_msg.empty() ? 1 : -1;
  }
  if (ctx->gflow_state < 0) return fail(ctx, OWQS_E_NO_GFLOW, "EOWQS: " + ctx->gflow_msg);
  return OWQS_OK;
}

owqs_status norm_all(owqs_ctx* ctx, double* out) {
  const Program& pr = ctx->cm[ctx->out_cm >= 0 ? ctx->out_cm : 0].prog;
  const int nb = ctx->n_ranks > 1 ? pr.phys_bits - ctx->n_global : (int)ctx->hp.outputs.size();
  for (size_t r = 0; r < ctx->shards.size(); ++r)
    CU(launch_norm(dev_ptrs(ctx, ctx->cm[0], (int)r), ctx->prec, 1ull << nb, ctx->stream));
  owqs_status s = allreduce_red(ctx);
  if (s != OWQS_OK) return s;
  double red[4];
  CU(cudaMemcpyAsync(red, ctx->shards[0].d_red, sizeof(red), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *out = red[0];
  return OWQS_OK;
}

}  // namespace

extern "C" {

const char* owqs_version(void) { return "owqs-b200 0.2 (sm_100a)"; }

static thread_local std::string g_create_err;  // why the last owqs_create on this thread failed

const char* owqs_last_error(const owqs_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

owqs_status owqs_nccl_unique_id(void* out) {
  if (!out) return OWQS_E_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return OWQS_E_NCCL;
  memcpy(out, &id, sizeof(id));
  return OWQS_OK;
}

owqs_status owqs_create(const owqs_config* cfg, owqs_ctx** out) {
  if (!cfg || !out) return OWQS_E_ARG;
  *out = nullptr;
  if (cfg->precision != 64 && cfg->precision != 128) return OWQS_E_ARG;
  const int nr = cfg->n_ranks <= 0 ? 1 : cfg->n_ranks;
  if (nr & (nr - 1)) return OWQS_E_ARG;
  const bool loopback = nr > 1 && (cfg->flags & OWQS_FLAG_LOOPBACK);
  if (nr > 1 && !loopback && (!cfg->nccl_id || cfg->rank < 0 || cfg->rank >= nr)) return OWQS_E_ARG;
  owqs_ctx* ctx = new owqs_ctx();
  ctx->cfg = *cfg;
  ctx->n_ranks = nr;
  ctx->rank = loopback ? 0 : (nr > 1 ? cfg->rank : 0);
  ctx->loopback = loopback;
  while ((1 << ctx->n_global) < nr) ++ctx->n_global;
  ctx->prec = cfg->precision == 64 ? 0 : 1;
  ctx->elem = cfg->precision == 64 ? 8 : 16;
  g_create_err.clear();
  auto bail = [&](owqs_status s, const char* what = "") {
    const cudaError_t ce = cudaGetLastError();
    g_create_err = std::string("owqs_create: ") + what + (ce != cudaSuccess ? std::string(": ") + cudaGetErrorString(ce) : "");
    owqs_destroy(ctx);
    return s;
  };
  if (cudaSetDevice(cfg->device) != cudaSuccess) return bail(OWQS_E_CUDA, "cudaSetDevice");
  {
    const cudaError_t e = init_kernel_limits(cfg->device);
    if (e != cudaSuccess) {
      g_create_err = std::string("owqs_create: kernel limits: ") + cudaGetErrorString(e);
      owqs_destroy(ctx);
      return OWQS_E_CUDA;
    }
  }
  if (cfg->stream) {
    ctx->stream = (cudaStream_t)cfg->stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(OWQS_E_CUDA, "allocation/stream/event setup");
    ctx->own_stream = true;
  }
  if (cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) return bail(OWQS_E_CUDA, "allocation/stream/event setup");
  const int n_sh = loopback ? nr : 1;
  ctx->shards.resize(n_sh);
  if (cudaMalloc(&ctx->d_red_all, (size_t)n_sh * 4 * sizeof(double)) != cudaSuccess) return bail(OWQS_E_NOMEM, "allocation/stream/event setup");
  const int nb = max_partial_blocks();
  for (int i = 0; i < n_sh; ++i) {
    Shard& s = ctx->shards[i];
    s.d_red = ctx->d_red_all + 4 * i;
    if (cudaMalloc(&s.d_partials, (size_t)nb * 4 * sizeof(double)) != cudaSuccess) return bail(OWQS_E_NOMEM, "allocation/stream/event setup");
    if (cudaMalloc(&s.d_counter, (1 + RED_MAX_GROUPS) * sizeof(unsigned)) != cudaSuccess) return bail(OWQS_E_NOMEM, "allocation/stream/event setup");
    if (cudaMemset(s.d_counter, 0, (1 + RED_MAX_GROUPS) * sizeof(unsigned)) != cudaSuccess) return bail(OWQS_E_CUDA, "allocation/stream/event setup");
    if (cudaMalloc(&s.d_err, sizeof(int32_t)) != cudaSuccess) return bail(OWQS_E_NOMEM, "allocation/stream/event setup");
  }
  if (cudaMalloc(&ctx->d_run, sizeof(RunParams)) != cudaSuccess) return bail(OWQS_E_NOMEM, "allocation/stream/event setup");
  if (cudaMalloc(&ctx->d_staging, kStagingBytes) != cudaSuccess) return bail(OWQS_E_NOMEM, "allocation/stream/event setup");
  if (cudaMallocHost(&ctx->h_staging, kStagingBytes) != cudaSuccess) return bail(OWQS_E_NOMEM, "allocation/stream/event setup");
  if (cudaMallocHost(&ctx->h_innorm, sizeof(double)) != cudaSuccess) return bail(OWQS_E_NOMEM, "allocation/stream/event setup");
  if (cudaMallocHost(&ctx->h_err, std::max<size_t>(1, ctx->shards.size()) * sizeof(int32_t)) != cudaSuccess)
    return bail(OWQS_E_NOMEM, "allocation/stream/event setup");
  if (nr > 1 && !loopback) {
    if (cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(OWQS_E_CUDA, "allocation/stream/event setup");
    for (int k = 0; k < 2; ++k)
      if (cudaEventCreateWithFlags(&ctx->sw_packed[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx->sw_sent[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx->sw_unpacked[k], cudaEventDisableTiming) != cudaSuccess)
        return bail(OWQS_E_CUDA, "allocation/stream/event setup");
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_id, sizeof(id));
    if (ncclCommInitRank(&ctx->comm, nr, id, cfg->rank) != ncclSuccess) return bail(OWQS_E_NCCL, "allocation/stream/event setup");
  }
  *out = ctx;
  return OWQS_OK;
}

void owqs_destroy(owqs_ctx* ctx) {
  if (!ctx) return;
  for (owqs_ctx* c : ctx->subs) owqs_destroy(c);  // children use the parent's stream
  ctx->subs.clear();
  cudaSetDevice(ctx->cfg.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (int i = 0; i < 2; ++i) free_mode(ctx->cm[i]);
  for (auto& s : ctx->shards) {
    cudaFree(s.d_state);
    cudaFree(s.d_partials);
    cudaFree(s.d_counter);
    cudaFree(s.d_err);
  }
  cudaFree(ctx->d_red_all);
  cudaFree(ctx->d_swap);
  cudaFree(ctx->d_jscratch);
  cudaFree(ctx->d_run);
  cudaFree(ctx->d_outcome);
  cudaFree(ctx->d_prob0);
  cudaFree(ctx->d_forced);
  cudaFree(ctx->d_staging);
  cudaFree(ctx->d_out_full);
  if (ctx->h_staging) cudaFreeHost(ctx->h_staging);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->h_innorm) cudaFreeHost(ctx->h_innorm);
  for (cudaEvent_t e : ctx->prof_ev) cudaEventDestroy(e);
  for (int a = 0; a < owqs_ctx::kAux; ++a) {
    if (ctx->aux[a]) cudaStreamDestroy(ctx->aux[a]);
    if (ctx->join_ev[a]) cudaEventDestroy(ctx->join_ev[a]);
  }
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  for (int k = 0; k < 2; ++k) {
    if (ctx->sw_packed[k]) cudaEventDestroy(ctx->sw_packed[k]);
    if (ctx->sw_sent[k]) cudaEventDestroy(ctx->sw_sent[k]);
    if (ctx->sw_unpacked[k]) cudaEventDestroy(ctx->sw_unpacked[k]);
  }
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

owqs_status substates_unsupported(owqs_ctx* ctx, const char* what) {
  return fail(ctx, OWQS_E_STATE,
              std::string(what) + " is not available for a pattern run as " + std::to_string(ctx->subs.size()) +
                  " sub-states (disconnected entanglement graph); create the context with OWQS_FLAG_ONE_STATE");
}

owqs_status load_compiled(owqs_ctx* ctx);

// one child context per sub-state, on the parent's stream; the gflow pre-check of EOWQS stays with
// the parent (the whole pattern's graph), the children keep their final-norm check
owqs_status load_substates(owqs_ctx* ctx, std::vector<HostPattern>& parts) {
  owqs_config cc = ctx->cfg;
  cc.flags |= OWQS_FLAG_ONE_STATE | OWQS_FLAG_NO_GFLOW;
  cc.stream = ctx->stream;
  owqs_stats_t agg{};
  for (HostPattern& p : parts) {
    owqs_ctx* ch = nullptr;
    owqs_status s = owqs_create(&cc, &ch);
    if (s != OWQS_OK) return fail(ctx, s, "sub-state context: " + std::string(owqs_last_error(nullptr)));
    ctx->subs.push_back(ch);
    ch->weights = ctx->weights;
    ch->hp = std::move(p);
    s = load_compiled(ch);
    if (s != OWQS_OK) return fail(ctx, s, "sub-state: " + std::string(owqs_last_error(ch)));
    const owqs_stats_t& cs = ch->stats;
    agg.paper_m = std::max(agg.paper_m, cs.paper_m);
    agg.phys_bits = std::max(agg.phys_bits, cs.phys_bits);
    agg.n_passes += cs.n_passes;
    agg.n_grow += cs.n_grow;
    agg.n_shrink += cs.n_shrink;
    agg.n_reduce += cs.n_reduce;
    agg.n_launches += cs.n_launches;
    agg.bytes_per_run += cs.bytes_per_run;
    agg.schedule_ms += cs.schedule_ms;
    agg.jit_ms += cs.jit_ms;
    agg.n_jit_steps += cs.n_jit_steps;
    agg.n_kernels += cs.n_kernels;
  }
  agg.n_commands = (int64_t)ctx->hp.cmds.size();
  agg.n_measure = ctx->hp.n_measure;
  agg.n_substates = (double)ctx->subs.size();
  ctx->stats = agg;
  ctx->loaded = true;
  return OWQS_OK;
}

owqs_status owqs_load_pattern(owqs_ctx* ctx, const int32_t* inputs, int32_t n_in, const int32_t* outputs,
                              int32_t n_out, const owqs_cmd* cmds, int64_t n_cmds, const int32_t* domain_pool,
                              int64_t pool_len) {
  NvtxRange nvtx_("owqs_load_pattern");
  if (!ctx) return OWQS_E_ARG;
  if (ctx->pending) return fail(ctx, OWQS_E_STATE, "a submitted run is pending: owqs_wait first");
  ctx->loaded = false;
  ctx->has_input = ctx->has_output = false;
  ctx->gflow_state = 0;
  for (owqs_ctx* c : ctx->subs) owqs_destroy(c);
  ctx->subs.clear();
  ctx->sub_mask.clear();
  std::string e = validate_pattern(inputs, n_in, outputs, n_out, cmds, n_cmds, domain_pool, pool_len, ctx->hp);
  if (!e.empty()) return fail(ctx, OWQS_E_PATTERN, e);
  if (n_in > 40 || n_out > 40) return fail(ctx, OWQS_E_ARG, "more than 40 input/output qubits");
  std::vector<HostPattern> parts;
  if (!(ctx->cfg.flags & OWQS_FLAG_ONE_STATE) && ctx->n_ranks == 1 && split_substates(ctx->hp, parts, ctx->sub_mask, KRON_MAX))
    return load_substates(ctx, parts);
  return load_compiled(ctx);
}

// compile the context's validated pattern (both modes) and fill the load-time stats
owqs_status load_compiled(owqs_ctx* ctx) {
  owqs_status s = compile_modes(ctx);
  if (s != OWQS_OK) return s;
  const Program& pr = ctx->cm[0].prog;
  ctx->stats = owqs_stats_t{};
  ctx->stats.n_substates = 1;
  ctx->stats.n_commands = (int64_t)ctx->hp.cmds.size();
  ctx->stats.n_measure = ctx->hp.n_measure;
  ctx->stats.paper_m = ctx->cm[0].plan.paper_m;
  ctx->stats.phys_bits = pr.phys_bits;
  ctx->stats.n_passes = pr.n_passes;
  ctx->stats.n_grow = pr.n_grow;
  ctx->stats.n_shrink = pr.n_shrink;
  ctx->stats.n_reduce = pr.n_reduce;
  ctx->stats.n_swaps = pr.n_swaps;
  ctx->stats.n_launches = (int32_t)pr.steps.size();
  ctx->stats.bytes_per_run = pr.bytes_per_run(ctx->elem);
  ctx->stats.schedule_ms = ctx->cm[0].schedule_ms;
  ctx->stats.jit_ms = ctx->jit_ms;
  ctx->stats.n_jit_steps = ctx->cm[0].n_jit;
  ctx->stats.n_kernels = kernels_per_run(ctx, ctx->cm[0]);
  if (pr.phys_bits - ctx->n_global > 40) return fail(ctx, OWQS_E_NOMEM, "shard width above 40 bits");
  ctx->loaded = true;
  return OWQS_OK;
}

// R-13 precondition (Eq. 3-4): a measurement whose partner is a fresh |+>
// has prob0 = 1/2 ||psi||^2, and the structural decisions take ||psi||^2 = 1 without a reduction,
// so every caller input must be normalised (the oracle refuses the same inputs).
// input_norm_enqueue: ||psi_in||^2 of the state just written (the shards' red_result, unless the
// copy kernel already reduced it) all-reduced over the ranks and copied, in stream order, to
// page-locked memory; input_norm_check reads it after a synchronisation.
constexpr double kInNormTol64 = 1e-5, kInNormTol128 = 1e-9;

owqs_status input_norm_enqueue(owqs_ctx* ctx, bool reduced) {
  const uint64_t per = (1ull << ctx->hp.inputs.size()) >> ctx->n_global;
  if (!reduced)
    for (size_t r = 0; r < ctx->shards.size(); ++r)
      CU(launch_norm(dev_ptrs(ctx, ctx->cm[0], (int)r), ctx->prec, per, ctx->stream));
  owqs_status s = allreduce_red(ctx);
  if (s != OWQS_OK) return s;
  CU(launch_readback(ctx->h_innorm, ctx->shards[0].d_red, sizeof(double), ctx->stream));
  return OWQS_OK;
}

owqs_status input_norm_check(owqs_ctx* ctx) {
  const double n2 = *ctx->h_innorm, tol = ctx->prec == 1 ? kInNormTol128 : kInNormTol64;
  if (!(std::fabs(n2 - 1.0) <= tol)) {
    ctx->has_input = false;
    return fail(ctx, OWQS_E_ARG, "input state not normalised: ||psi||^2 = " + std::to_string(n2) +
                                     " (|1 - ||psi||^2| must be <= " + (ctx->prec == 1 ? "1e-9" : "1e-5") + ")");
  }
  return OWQS_OK;
}

owqs_status owqs_set_input(owqs_ctx* ctx, const double* amps, int64_t n_amps) {
  return owqs_set_input_host(ctx, amps, 128, n_amps);
}

owqs_status input_from_host_enqueue(owqs_ctx* ctx, const void* amps, int32_t precision);

owqs_status owqs_set_input_host(owqs_ctx* ctx, const void* amps, int32_t precision, int64_t n_amps) {
  NvtxRange nvtx_("owqs_set_input_host");
  if (!ctx) return OWQS_E_ARG;
  if (ctx->pending) return fail(ctx, OWQS_E_STATE, "a submitted run is pending: owqs_wait first");
  if (!ctx->subs.empty()) {  // the caller's input is the inputs' sub-state (PAPER §4.1)
    owqs_status st = owqs_set_input_host(ctx->subs[0], amps, precision, n_amps);
    if (st != OWQS_OK) return fail(ctx, st, owqs_last_error(ctx->subs[0]));
    ctx->has_input = true;
    ctx->has_output = false;
    return OWQS_OK;
  }
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "set_input before load_pattern");
  const uint64_t n = 1ull << ctx->hp.inputs.size();
  if (!amps || n_amps != (int64_t)n) return fail(ctx, OWQS_E_ARG, "input must hold 2^n_in amplitudes");
  if (precision != 64 && precision != 128) return fail(ctx, OWQS_E_ARG, "precision must be 64 or 128");
  owqs_status s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  s = input_from_host_enqueue(ctx, amps, precision);
  if (s != OWQS_OK) return s;
  s = input_norm_enqueue(ctx, false);
  if (s != OWQS_OK) return s;
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->has_output = false;
  s = input_norm_check(ctx);
  if (s != OWQS_OK) return s;
  ctx->has_input = true;
  return OWQS_OK;
}

// host input (caller order, either precision) into every local shard's state, on ctx->stream
owqs_status input_from_host_enqueue(owqs_ctx* ctx, const void* amps, int32_t precision) {
  const uint64_t n = 1ull << ctx->hp.inputs.size();
  const int sp = precision == 64 ? 0 : 1;
  const size_t se = precision == 64 ? 8 : 16;
  const uint64_t per = n >> ctx->n_global;  // amplitudes per shard
  const uint64_t chunk = kStagingBytes / se;
  for (size_t r = 0; r < ctx->shards.size(); ++r) {
    const uint64_t base = (uint64_t)ctx->shard_rank((int)r) * per;
    const char* src0 = (const char*)amps + base * se;
    if (sp == ctx->prec) {  // same precision: straight into the state (DMA when page-locked)
      CU(cudaMemcpyAsync(ctx->shards[r].d_state, src0, per * se, cudaMemcpyHostToDevice, ctx->stream));
      continue;
    }
    for (uint64_t j0 = 0; j0 < per; j0 += chunk) {
      const uint64_t cnt = std::min(chunk, per - j0);
      CU(cudaMemcpyAsync(ctx->d_staging, src0 + j0 * se, cnt * se, cudaMemcpyHostToDevice, ctx->stream));
      CU(launch_convert_in(ctx->d_staging, sp, ctx->shards[r].d_state, ctx->prec, j0, cnt, ctx->stream));
    }
  }
  return OWQS_OK;
}

owqs_status owqs_set_input_device(owqs_ctx* ctx, const void* dev_amps, int32_t precision, int64_t n_amps) {
  NvtxRange nvtx_("owqs_set_input_device");
  if (!ctx) return OWQS_E_ARG;
  if (ctx->pending) return fail(ctx, OWQS_E_STATE, "a submitted run is pending: owqs_wait first");
  if (!ctx->subs.empty()) {  // the caller's input is the inputs' sub-state (PAPER §4.1)
    owqs_status st = owqs_set_input_device(ctx->subs[0], dev_amps, precision, n_amps);
    if (st != OWQS_OK) return fail(ctx, st, owqs_last_error(ctx->subs[0]));
    ctx->has_input = true;
    ctx->has_output = false;
    return OWQS_OK;
  }
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "set_input before load_pattern");
  const uint64_t n = 1ull << ctx->hp.inputs.size();
  const uint64_t per = n >> ctx->n_global;
  const uint64_t expect = (ctx->n_ranks > 1 && !ctx->loopback) ? per : n;
  if (!dev_amps || n_amps != (int64_t)expect || (precision != 64 && precision != 128))
    return fail(ctx, OWQS_E_ARG, "input must hold the (shard's) amplitudes at precision 64 or 128");
  owqs_status s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  const int sp = precision == 64 ? 0 : 1;
  const size_t se = precision == 64 ? 8 : 16;
  for (size_t r = 0; r < ctx->shards.size(); ++r) {
    const char* src = (const char*)dev_amps + (ctx->loopback ? r * per * se : 0);
    if (sp == ctx->prec) {  // one sweep: copy + ||psi||^2
      CU(launch_copy_norm(dev_ptrs(ctx, ctx->cm[0], (int)r), ctx->prec, src, per, ctx->stream));
    } else {
      CU(launch_convert_in(src, sp, ctx->shards[r].d_state, ctx->prec, 0, per, ctx->stream));
    }
  }
  s = input_norm_enqueue(ctx, sp == ctx->prec);
  if (s != OWQS_OK) return s;
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->has_output = false;
  s = input_norm_check(ctx);
  if (s != OWQS_OK) return s;
  ctx->has_input = true;
  return OWQS_OK;
}

owqs_status owqs_set_input_random(owqs_ctx* ctx, uint64_t seed) {
  NvtxRange nvtx_("owqs_set_input_random");
  if (!ctx) return OWQS_E_ARG;
  if (ctx->pending) return fail(ctx, OWQS_E_STATE, "a submitted run is pending: owqs_wait first");
  if (!ctx->subs.empty()) {  // the caller's input is the inputs' sub-state (PAPER §4.1)
    owqs_status st = owqs_set_input_random(ctx->subs[0], seed);
    if (st != OWQS_OK) return fail(ctx, st, owqs_last_error(ctx->subs[0]));
    ctx->has_input = true;
    ctx->has_output = false;
    return OWQS_OK;
  }
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "set_input before load_pattern");
  owqs_status s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  const uint64_t per = (1ull << ctx->hp.inputs.size()) >> ctx->n_global;
  for (size_t r = 0; r < ctx->shards.size(); ++r)
    CU(launch_haar(dev_ptrs(ctx, ctx->cm[0], (int)r), ctx->prec, per, seed, (uint64_t)ctx->shard_rank((int)r) * per,
                   ctx->stream));
  s = allreduce_red(ctx);
  if (s != OWQS_OK) return s;
  for (size_t r = 0; r < ctx->shards.size(); ++r)
    CU(launch_scale(dev_ptrs(ctx, ctx->cm[0], (int)r), ctx->prec, per, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->has_input = true;
  ctx->has_output = false;
  return OWQS_OK;
}

owqs_status finish_run(owqs_ctx* ctx, int cmi, int mode, owqs_status s, uint8_t* outcomes_out, double* prob0_out);
owqs_status run_substates(owqs_ctx* ctx, owqs_mode mode, uint64_t seed, const uint8_t* forced, uint8_t* outcomes_out,
                          double* prob0_out);

owqs_status owqs_run(owqs_ctx* ctx, owqs_mode mode, uint64_t seed, const uint8_t* forced, uint8_t* outcomes_out,
                     double* prob0_out) {
  NvtxRange nvtx_("owqs_run");
  if (!ctx) return OWQS_E_ARG;
  if (ctx->pending) return fail(ctx, OWQS_E_STATE, "a submitted run is pending: owqs_wait first");
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "run before load_pattern");
  if (!ctx->has_input) return fail(ctx, OWQS_E_STATE, "run without a fresh input (set_input consumes per run)");
  if (mode != OWQS_SAMPLED && mode != OWQS_FORCED && mode != OWQS_EOWQS) return fail(ctx, OWQS_E_ARG, "bad mode");
  if (mode == OWQS_FORCED && ctx->hp.n_measure > 0 && !forced) return fail(ctx, OWQS_E_ARG, "forced outcomes missing");
  if (mode == OWQS_EOWQS) {
    owqs_status g = gflow_gate(ctx);
    if (g != OWQS_OK) return g;
  }
  if (!ctx->subs.empty()) return run_substates(ctx, mode, seed, forced, outcomes_out, prob0_out);
  const int cmi = mode == OWQS_EOWQS ? 1 : 0;
  owqs_status s = run_internal(ctx, cmi, mode, seed, forced);
  return finish_run(ctx, cmi, mode, s, outcomes_out, prob0_out);
}

// every sub-state in turn (independent: no signal crosses them); the others start from the
// 0-qubit state 1. Outcomes and prob0 gathered at the caller's ordinals.
owqs_status run_substates(owqs_ctx* ctx, owqs_mode mode, uint64_t seed, const uint8_t* forced, uint8_t* outcomes_out,
                          double* prob0_out) {
  const int64_t K = ctx->hp.n_measure;
  std::vector<uint8_t> oc(std::max<int64_t>(K, 1)), ao(std::max<int64_t>(K, 1));
  std::vector<double> p0(std::max<int64_t>(K, 1)), ap(std::max<int64_t>(K, 1));
  double ms = 0;
  ctx->has_input = false;
  owqs_status worst = OWQS_OK;
  std::vector<uint8_t> fc;
  for (size_t c = 0; c < ctx->subs.size(); ++c) {
    owqs_ctx* ch = ctx->subs[c];
    const std::vector<int>& key = ch->hp.draw_key;  // sub-state ordinal -> the caller's
    if (forced) {
      fc.assign(std::max<size_t>(key.size(), 1), 0);
      for (size_t k = 0; k < key.size(); ++k) fc[k] = forced[key[k]];
    }
    if (c > 0) {
      const double one[2] = {1.0, 0.0};
      owqs_status st = owqs_set_input_host(ch, one, 128, 1);
      if (st != OWQS_OK) return fail(ctx, st, owqs_last_error(ch));
    }
    owqs_status st = owqs_run(ch, mode, seed, forced ? fc.data() : nullptr, oc.data(), p0.data());
    if (st != OWQS_OK && st != OWQS_E_BRANCH) return fail(ctx, st, owqs_last_error(ch));
    if (st == OWQS_E_BRANCH) worst = st;
    for (size_t k = 0; k < key.size(); ++k) {
      ao[key[k]] = oc[k];
      ap[key[k]] = p0[k];
    }
    ms += ch->stats.last_run_ms;
  }
  if (K > 0 && outcomes_out) memcpy(outcomes_out, ao.data(), K);
  if (K > 0 && prob0_out) memcpy(prob0_out, ap.data(), K * sizeof(double));
  ctx->stats.last_run_ms = ms;
  if (worst != OWQS_OK) return fail(ctx, worst, "forced outcome on a branch with probability < 1e-12");
  ctx->has_output = true;
  return OWQS_OK;
}

// After a completed run: outcomes / prob0 to the caller, stats, the EOWQS norm check.
// (after run_complete: the run's readbacks are in the page-locked staging, RunStaging)
owqs_status finish_run(owqs_ctx* ctx, int cmi, int mode, owqs_status s, uint8_t* outcomes_out, double* prob0_out) {
  const int64_t K = ctx->hp.n_measure;
  const RunStaging rs(K);
  const uint8_t* hs = static_cast<const uint8_t*>(ctx->h_staging);
  if (K > 0 && (s == OWQS_OK || s == OWQS_E_BRANCH)) {
    if (outcomes_out) {
      if (mode == OWQS_EOWQS)
        memset(outcomes_out, 0, K);
      else
        memcpy(outcomes_out, hs + rs.outcomes, K);
    }
    if (prob0_out) {
      if (mode == OWQS_EOWQS)
        for (int64_t i = 0; i < K; ++i) prob0_out[i] = -1.0;
      else
        memcpy(prob0_out, hs + rs.prob0, K * sizeof(double));
    }
  }
  if (s != OWQS_OK) return s;
  const Program& pr = ctx->cm[cmi].prog;
  ctx->stats.n_passes = pr.n_passes;
  ctx->stats.n_grow = pr.n_grow;
  ctx->stats.n_shrink = pr.n_shrink;
  ctx->stats.n_reduce = pr.n_reduce;
  ctx->stats.n_swaps = pr.n_swaps;
  ctx->stats.n_launches = (int32_t)pr.steps.size();
  ctx->stats.bytes_per_run = pr.bytes_per_run(ctx->elem);
  ctx->stats.schedule_ms = ctx->cm[cmi].schedule_ms;
  ctx->stats.jit_ms = ctx->jit_ms;
  ctx->stats.n_jit_steps = ctx->cm[cmi].n_jit;
  ctx->stats.n_kernels = kernels_per_run(ctx, ctx->cm[cmi]);
  ctx->stats.phys_bits = pr.phys_bits;
  if (mode == OWQS_EOWQS) {
    double red[4];
    memcpy(red, hs + rs.red, sizeof(red));
    const double tol = ctx->prec == 1 ? 1e-8 : 1e-3;
    if (!(std::fabs(red[0] - 1.0) <= tol))
      return fail(ctx, OWQS_E_NOT_DETERMINISTIC,
                  "EOWQS output norm^2 = " + std::to_string(red[0]) + ": the pattern is not deterministic");
  }
  return OWQS_OK;
}

owqs_status owqs_submit_host(owqs_ctx* ctx, owqs_mode mode, uint64_t seed, const uint8_t* forced, const void* in_amps,
                             int32_t in_precision, int64_t n_in, void* out_amps, int32_t out_precision,
                             int64_t n_out) {
  NvtxRange nvtx_("owqs_submit_host");
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->subs.empty()) return substates_unsupported(ctx, "owqs_submit_host");
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "submit before load_pattern");
  if (ctx->pending) return fail(ctx, OWQS_E_STATE, "a submitted run is pending: owqs_wait first");
  if (ctx->n_ranks > 1) return fail(ctx, OWQS_E_ARG, "owqs_submit_host is single-rank");
  if (mode != OWQS_SAMPLED && mode != OWQS_FORCED && mode != OWQS_EOWQS) return fail(ctx, OWQS_E_ARG, "bad mode");
  if (mode == OWQS_FORCED && ctx->hp.n_measure > 0 && !forced) return fail(ctx, OWQS_E_ARG, "forced outcomes missing");
  if ((in_precision != 64 && in_precision != 128) || (out_precision != 64 && out_precision != 128))
    return fail(ctx, OWQS_E_ARG, "precision must be 64 or 128");
  if (!in_amps || n_in != (int64_t)(1ull << ctx->hp.inputs.size()))
    return fail(ctx, OWQS_E_ARG, "input must hold 2^n_in amplitudes");
  if (!out_amps || n_out < (int64_t)(1ull << ctx->hp.outputs.size()))
    return fail(ctx, OWQS_E_ARG, "output buffer smaller than 2^n_out");
  if (!is_pinned_host(in_amps) || !is_pinned_host(out_amps))
    return fail(ctx, OWQS_E_ARG, "owqs_submit_host needs page-locked host buffers (cudaHostAlloc)");
  if (mode == OWQS_EOWQS) {
    owqs_status g = gflow_gate(ctx);
    if (g != OWQS_OK) return g;
  }
  owqs_status s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  s = input_from_host_enqueue(ctx, in_amps, in_precision);
  if (s != OWQS_OK) return s;
  s = input_norm_enqueue(ctx, false);  // checked by owqs_wait (stream-ordered readback)
  if (s != OWQS_OK) return s;
  ctx->has_input = true;
  ctx->has_output = false;
  const int cmi = mode == OWQS_EOWQS ? 1 : 0;
  s = run_enqueue(ctx, cmi, mode, seed, forced);
  if (s != OWQS_OK) return s;
  s = output_to_host_enqueue(ctx, out_amps, out_precision == 64 ? 0 : 1, true, false);
  if (s != OWQS_OK) return s;
  ctx->pending = 1 + cmi;
  ctx->pending_mode = mode;
  return OWQS_OK;
}

owqs_status owqs_wait(owqs_ctx* ctx, uint8_t* outcomes_out, double* prob0_out) {
  NvtxRange nvtx_("owqs_wait");
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->pending) return fail(ctx, OWQS_E_STATE, "nothing submitted");
  const int cmi = ctx->pending - 1;
  ctx->pending = 0;
  owqs_status s = run_complete(ctx, cmi);
  if (s == OWQS_OK || s == OWQS_E_BRANCH) {  // the run completed: its input's norm is readable
    const owqs_status sn = input_norm_check(ctx);
    if (sn != OWQS_OK) {
      ctx->has_output = false;
      return sn;
    }
  }
  return finish_run(ctx, cmi, ctx->pending_mode, s, outcomes_out, prob0_out);
}

owqs_status owqs_run_batch(owqs_ctx* ctx, owqs_mode mode, int64_t n_batch, const double* inputs,
                           const uint64_t* seeds, const uint8_t* forced, double* outputs, uint8_t* outcomes,
                           double* prob0) {
  NvtxRange nvtx_("owqs_run_batch");
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->subs.empty()) return substates_unsupported(ctx, "owqs_run_batch");
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "run_batch before load_pattern");
  if (n_batch <= 0 || !inputs || !outputs) return fail(ctx, OWQS_E_ARG, "empty batch or NULL buffers");
  if (mode != OWQS_SAMPLED && mode != OWQS_FORCED && mode != OWQS_EOWQS) return fail(ctx, OWQS_E_ARG, "bad mode");
  if (mode == OWQS_FORCED && ctx->hp.n_measure > 0 && !forced) return fail(ctx, OWQS_E_ARG, "forced outcomes missing");
  if (mode == OWQS_EOWQS) {
    owqs_status g = gflow_gate(ctx);
    if (g != OWQS_OK) return g;
  }
  return run_batch_internal(ctx, mode, n_batch, inputs, seeds, forced, outputs, outcomes, prob0);
}

owqs_status owqs_get_output(owqs_ctx* ctx, double* amps, int64_t n_amps) {
  NvtxRange nvtx_("owqs_get_output");
  return owqs_get_output_host(ctx, amps, 128, n_amps);
}

// Output of a pattern run as sub-states: each sub-state's output (its outputs in caller order) into
// a device factor, then one kron_merge launch scatters their tensor product into the caller's
// output order (bit k <-> outputs[k]); into dst on the device, or through a device buffer to host.
owqs_status output_merged(owqs_ctx* ctx, void* dst, int out_prec, bool dst_device) {
  const size_t oe = out_prec == 1 ? 16 : 8;
  const int nc = (int)ctx->subs.size();
  std::vector<void*> f(nc, nullptr);
  void* tmp = nullptr;
  auto cleanup = [&]() {
    for (void* x : f) cudaFree(x);
    cudaFree(tmp);
  };
  for (int c = 0; c < nc; ++c) {
    const uint64_t nf = 1ull << ctx->subs[c]->hp.outputs.size();
    if (cudaMalloc(&f[c], nf * oe) != cudaSuccess) {
      cleanup();
      return fail(ctx, OWQS_E_NOMEM, "sub-state output factor");
    }
    owqs_status st = owqs_get_output_device(ctx->subs[c], f[c], out_prec == 1 ? 128 : 64, (int64_t)nf);
    if (st != OWQS_OK) {
      cleanup();
      return fail(ctx, st, owqs_last_error(ctx->subs[c]));
    }
  }
  const uint64_t n = 1ull << ctx->hp.outputs.size();
  void* d = dst;
  if (!dst_device && cudaMalloc(&tmp, n * oe) != cudaSuccess) {
    cleanup();
    return fail(ctx, OWQS_E_NOMEM, "merged output buffer");
  }
  if (!dst_device) d = tmp;
  cudaError_t e = launch_kron_merge(d, out_prec, f.data(), ctx->sub_mask.data(), nc, n, ctx->stream);
  if (e == cudaSuccess && !dst_device) e = cudaMemcpyAsync(dst, d, n * oe, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cleanup();
  if (e != cudaSuccess) return fail(ctx, OWQS_E_CUDA, cudaGetErrorString(e));
  return OWQS_OK;
}

owqs_status owqs_get_output_host(owqs_ctx* ctx, void* amps, int32_t precision, int64_t n_amps) {
  NvtxRange nvtx_("owqs_get_output_host");
  if (!ctx) return OWQS_E_ARG;
  if (ctx->pending) return fail(ctx, OWQS_E_STATE, "a submitted run is pending: owqs_wait first");
  if (!ctx->has_output) return fail(ctx, OWQS_E_STATE, "no output: run first");
  if (precision != 64 && precision != 128) return fail(ctx, OWQS_E_ARG, "precision must be 64 or 128");
  const uint64_t n = 1ull << ctx->hp.outputs.size();
  const bool root = ctx->n_ranks == 1 || ctx->loopback || ctx->rank == 0;
  if (root && (!amps || n_amps < (int64_t)n)) return fail(ctx, OWQS_E_ARG, "output buffer smaller than 2^n_out");
  if (!ctx->subs.empty()) return output_merged(ctx, amps, precision == 64 ? 0 : 1, false);
  return output_to_host(ctx, amps, precision == 64 ? 0 : 1);
}

owqs_status owqs_get_output_device(owqs_ctx* ctx, void* dev_amps, int32_t precision, int64_t n_amps) {
  NvtxRange nvtx_("owqs_get_output_device");
  if (!ctx) return OWQS_E_ARG;
  if (ctx->pending) return fail(ctx, OWQS_E_STATE, "a submitted run is pending: owqs_wait first");
  if (!ctx->has_output) return fail(ctx, OWQS_E_STATE, "no output: run first");
  const uint64_t n = 1ull << ctx->hp.outputs.size();
  const bool root = ctx->n_ranks == 1 || ctx->loopback || ctx->rank == 0;
  if ((root && (!dev_amps || n_amps < (int64_t)n)) || (precision != 64 && precision != 128))
    return fail(ctx, OWQS_E_ARG, "bad output buffer");
  if (!ctx->subs.empty()) return output_merged(ctx, dev_amps, precision == 64 ? 0 : 1, true);
  owqs_status s = output_to_device_full(ctx, dev_amps, precision == 64 ? 0 : 1);
  if (s != OWQS_OK) return s;
  CU(cudaStreamSynchronize(ctx->stream));
  return OWQS_OK;
}

owqs_status owqs_get_output_sample(owqs_ctx* ctx, const int64_t* idx, int64_t n, double* amps) {
  if (!ctx) return OWQS_E_ARG;
  if (ctx->pending) return fail(ctx, OWQS_E_STATE, "a submitted run is pending: owqs_wait first");
  if (!ctx->subs.empty()) return substates_unsupported(ctx, "owqs_get_output_sample");
  if (!ctx->has_output) return fail(ctx, OWQS_E_STATE, "no output: run first");
  if (n < 0 || (n > 0 && (!idx || !amps))) return fail(ctx, OWQS_E_ARG, "bad sample buffers");
  if (n == 0) return OWQS_OK;
  const int nbo = (int)ctx->hp.outputs.size();
  for (int64_t i = 0; i < n; ++i)
    if (idx[i] < 0 || (nbo < 63 && (uint64_t)idx[i] >= (1ull << nbo)))
      return fail(ctx, OWQS_E_ARG, "sample index " + std::to_string(i) + " outside [0, 2^n_out)");
  const Program& pr = ctx->cm[ctx->out_cm].prog;
  const int wl = pr.phys_bits - ctx->n_global;
  void* d = nullptr;
  const size_t ib = (size_t)n * sizeof(int64_t), ob = (size_t)n * 2 * sizeof(double);
  if (cudaMalloc(&d, ib + ob) != cudaSuccess) return fail(ctx, OWQS_E_NOMEM, "sample buffers");
  auto done = [&](owqs_status st) {
    cudaFree(d);
    return st;
  };
  int64_t* d_idx = (int64_t*)d;
  char* d_out = (char*)d + ib;
  cudaError_t e = cudaMemcpyAsync(d_idx, idx, ib, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_out, 0, ob, ctx->stream);
  for (size_t r = 0; e == cudaSuccess && r < ctx->shards.size(); ++r)
    e = launch_sample_out(ctx->shards[r].d_state, ctx->prec, d_idx, (uint64_t)n, nbo, pr.out_slot.data(),
                          (uint64_t)ctx->shard_rank((int)r), wl, d_out, ctx->stream);
  if (e != cudaSuccess) return done(fail(ctx, OWQS_E_CUDA, cudaGetErrorString(e)));
  if (ctx->n_ranks > 1 && !ctx->loopback &&
      ncclAllReduce(d_out, d_out, (size_t)n * 2, ncclDouble, ncclSum, ctx->comm, ctx->stream) != ncclSuccess)
    return done(fail(ctx, OWQS_E_NCCL, "all-reduce of the output samples"));
  e = cudaMemcpyAsync(amps, d_out, ob, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return done(fail(ctx, OWQS_E_CUDA, cudaGetErrorString(e)));
  return done(OWQS_OK);
}

owqs_status owqs_output_norm(owqs_ctx* ctx, double* norm2) {
  if (!ctx || !norm2) return OWQS_E_ARG;
  if (!ctx->subs.empty()) return substates_unsupported(ctx, "owqs_output_norm");
  if (!ctx->has_output) return fail(ctx, OWQS_E_STATE, "no output: run first");
  return norm_all(ctx, norm2);
}

owqs_status owqs_output_inner(owqs_ctx* a, owqs_ctx* b, double* re, double* im) {
  owqs_ctx* ctx = a;
  if (!a || !b || !re || !im) return OWQS_E_ARG;
  if (!a->subs.empty() || !b->subs.empty()) return substates_unsupported(a, "owqs_output_inner");
  if (!a->has_output || !b->has_output) return fail(a, OWQS_E_STATE, "no output: run first");
  if (a->hp.outputs.size() != b->hp.outputs.size()) return fail(a, OWQS_E_ARG, "output widths differ");
  if (a->n_ranks > 1 || b->n_ranks > 1) {
    const Program& pa = a->cm[a->out_cm].prog;
    const Program& pb = b->cm[b->out_cm].prog;
    if (a->n_ranks != b->n_ranks || a->loopback != b->loopback || a->prec != b->prec || pa.out_slot != pb.out_slot ||
        pa.phys_bits != pb.phys_bits)
      return fail(a, OWQS_E_ARG, "multi-rank inner product needs equal sharding, precision and final layout");
    const uint64_t per = 1ull << (pa.phys_bits - a->n_global);
    for (size_t r = 0; r < a->shards.size(); ++r)
      CU(launch_dot_t(dev_ptrs(a, a->cm[0], (int)r), a->prec, a->shards[r].d_state, b->shards[r].d_state, per,
                      a->stream));
    owqs_status s = allreduce_red(a);
    if (s != OWQS_OK) return s;
    double red[4];
    CU(cudaMemcpyAsync(red, a->shards[0].d_red, sizeof(red), cudaMemcpyDeviceToHost, a->stream));
    CU(cudaStreamSynchronize(a->stream));
    *re = red[0];
    *im = red[1];
    return OWQS_OK;
  }
  const uint64_t n = 1ull << a->hp.outputs.size();
  const Program& pa = a->cm[a->out_cm].prog;
  const Program& pb = b->cm[b->out_cm].prog;
  if (a->prec == b->prec && pa.out_slot == pb.out_slot && pa.phys_bits == pb.phys_bits &&
      pa.phys_bits == (int)a->hp.outputs.size()) {
    // same final layout: dot the states in place (no scratch; any size)
    CU(launch_dot_t(dev_ptrs(a, a->cm[0], 0), a->prec, a->shards[0].d_state, b->shards[0].d_state, n, a->stream));
    double red[4];
    CU(cudaMemcpyAsync(red, a->shards[0].d_red, sizeof(red), cudaMemcpyDeviceToHost, a->stream));
    CU(cudaStreamSynchronize(a->stream));
    *re = red[0];
    *im = red[1];
    return OWQS_OK;
  }
  // different layouts: permute both into the caller's output order chunk by chunk through the
  // staging buffer (two complex128 halves) and sum the chunk dots in a fixed order
  const uint64_t chunk = kStagingBytes / 32;
  char* ta = (char*)a->d_staging;
  char* tb = ta + chunk * 16;
  double sr = 0, si = 0;
  for (uint64_t j0 = 0; j0 < n; j0 += chunk) {
    const uint64_t cnt = std::min(chunk, n - j0);
    CU(launch_permute_out(a->shards[0].d_state, a->prec, ta, 1, (int)pa.out_slot.size(), pa.out_slot.data(), j0, cnt,
                          a->stream));
    CU(launch_permute_out(b->shards[0].d_state, b->prec, tb, 1, (int)pb.out_slot.size(), pb.out_slot.data(), j0, cnt,
                          a->stream));
    CU(launch_dot(dev_ptrs(a, a->cm[0], 0), ta, tb, cnt, a->stream));
    double red[4];
    CU(cudaMemcpyAsync(red, a->shards[0].d_red, sizeof(red), cudaMemcpyDeviceToHost, a->stream));
    CU(cudaStreamSynchronize(a->stream));
    sr += red[0];
    si += red[1];
  }
  *re = sr;
  *im = si;
  return OWQS_OK;
}

owqs_status owqs_recognize(owqs_ctx* ctx, double* U, int64_t n, double* max_unitarity_err) {
  NvtxRange nvtx_("owqs_recognize");
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->subs.empty()) return substates_unsupported(ctx, "owqs_recognize");
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "recognize before load_pattern");
  if (ctx->n_ranks > 1) return fail(ctx, OWQS_E_ARG, "recognize runs on a single rank");
  const int ni = (int)ctx->hp.inputs.size(), no = (int)ctx->hp.outputs.size();
  if (ni > 14 || no > 14) return fail(ctx, OWQS_E_ARG, "recognize is limited to 14 input/output qubits");
  const uint64_t rows = 1ull << no, cols = 1ull << ni;
  if (!U || n < (int64_t)(rows * cols)) return fail(ctx, OWQS_E_ARG, "U must hold 2^n_out * 2^n_in entries");
  owqs_status s = gflow_gate(ctx);
  if (s != OWQS_OK) return s;
  s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  if (((size_t)ctx->elem << ctx->cm[1].prog.phys_bits) <= (size_t)kBatchMaxBytes) {
    // all 2^n_in basis columns as one batched launch (U is column-major: column k = state k)
    std::vector<double> in(2 * cols * cols, 0.0);
    for (uint64_t k = 0; k < cols; ++k) in[2 * (k * cols + k)] = 1.0;
    s = run_batch_internal(ctx, OWQS_EOWQS, (int64_t)cols, in.data(), nullptr, nullptr, U, nullptr, nullptr);
    if (s != OWQS_OK) return s;
  } else {
    for (uint64_t k = 0; k < cols; ++k) {
      CU(launch_basis(ctx->shards[0].d_state, ctx->prec, cols, k, ctx->stream));
      ctx->has_input = true;
      s = run_internal(ctx, 1, OWQS_EOWQS, 0, nullptr);
      if (s != OWQS_OK) return s;
      s = output_to_host(ctx, U + 2 * k * rows, 1);
      if (s != OWQS_OK) return s;
    }
  }
  if (max_unitarity_err) {
    double worst = 0;
    for (uint64_t i = 0; i < cols; ++i)
      for (uint64_t j = 0; j < cols; ++j) {
        double sr = 0, si = 0;
        for (uint64_t r = 0; r < rows; ++r) {
          double ar = U[2 * (i * rows + r)], ai = U[2 * (i * rows + r) + 1];
          double br = U[2 * (j * rows + r)], bi = U[2 * (j * rows + r) + 1];
          sr += ar * br + ai * bi;
          si += ar * bi - ai * br;
        }
        if (i == j) sr -= 1.0;
        worst = std::max(worst, std::hypot(sr, si));
      }
    *max_unitarity_err = worst;
  }
  return OWQS_OK;
}

// Recognition from the Choi state: the pattern extended by |I|
// reference qubits that no command touches (inputs I + R, outputs O + R), run once on the maximally
// entangled input sum_k |k>_I |k>_R / sqrt(d) (positive EOWQS branch), gives sum_k (U |k>)_O |k>_R /
// sqrt(d): with outputs O in bits 0..|O|-1 and R above them, the output array IS U in column-major
// order up to the factor 1/sqrt(d). One run at width + |I| instead of 2^|I| runs.
owqs_status owqs_recognize_choi(owqs_ctx* ctx, double* U, int64_t n, double* max_unitarity_err) {
  NvtxRange nvtx_("owqs_recognize_choi");
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->subs.empty()) return substates_unsupported(ctx, "owqs_recognize_choi");
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "recognize before load_pattern");
  if (ctx->n_ranks > 1) return fail(ctx, OWQS_E_ARG, "recognize runs on a single rank");
  const HostPattern& hp = ctx->hp;
  const int ni = (int)hp.inputs.size(), no = (int)hp.outputs.size();
  if (ni + no > 30) return fail(ctx, OWQS_E_ARG, "Choi recognition is limited to |I| + |O| <= 30");
  const uint64_t rows = 1ull << no, cols = 1ull << ni;
  if (!U || n < (int64_t)(rows * cols)) return fail(ctx, OWQS_E_ARG, "U must hold 2^n_out * 2^n_in entries");
  owqs_status s = gflow_gate(ctx);
  if (s != OWQS_OK) return s;
  // the pattern's commands with external ids, plus |I| fresh reference ids
  std::vector<owqs_cmd> cmds;
  std::vector<int32_t> pool;
  int32_t maxid = 0;
  for (int32_t e : hp.ext_id) maxid = std::max(maxid, e);
  for (const HCmd& c : hp.cmds) {
    owqs_cmd o{};
    o.kind = c.kind;
    o.q0 = hp.ext_id[c.q0];
    o.q1 = c.kind == H_E ? hp.ext_id[c.q1] : 0;
    o.angle = c.angle;
    o.s_off = (int32_t)pool.size();
    o.s_len = (int32_t)c.sdom.size();
    for (int q : c.sdom) pool.push_back(hp.ext_id[q]);
    o.t_off = (int32_t)pool.size();
    o.t_len = (int32_t)c.tdom.size();
    for (int q : c.tdom) pool.push_back(hp.ext_id[q]);
    cmds.push_back(o);
  }
  std::vector<int32_t> ins, outs;
  for (int q : hp.inputs) ins.push_back(hp.ext_id[q]);
  for (int q : hp.outputs) outs.push_back(hp.ext_id[q]);
  for (int r = 0; r < ni; ++r) {
    ins.push_back(maxid + 1 + r);
    outs.push_back(maxid + 1 + r);
  }
  owqs_config cfg = ctx->cfg;
  cfg.flags |= OWQS_FLAG_NO_GFLOW;  // checked above on the same open graph
  cfg.stream = nullptr;
  owqs_ctx* sub = nullptr;
  if (owqs_create(&cfg, &sub) != OWQS_OK) return fail(ctx, OWQS_E_CUDA, "Choi recognition: context creation failed");
  auto done = [&](owqs_status st, const std::string& why) {
    if (st != OWQS_OK) ctx->err = "Choi recognition: " + why + ": " + owqs_last_error(sub);
    owqs_destroy(sub);
    return st;
  };
  s = owqs_load_pattern(sub, ins.data(), (int32_t)ins.size(), outs.data(), (int32_t)outs.size(), cmds.data(),
                        (int64_t)cmds.size(), pool.data(), (int64_t)pool.size());
  if (s != OWQS_OK) return done(s, "load");
  std::vector<double> in(2 * cols * cols, 0.0);
  const double amp = 1.0 / std::sqrt((double)cols);
  for (uint64_t k = 0; k < cols; ++k) in[2 * (k + (k << ni))] = amp;
  s = owqs_set_input_host(sub, in.data(), 128, (int64_t)(cols * cols));
  if (s != OWQS_OK) return done(s, "input");
  s = owqs_run(sub, OWQS_EOWQS, 0, nullptr, nullptr, nullptr);
  if (s != OWQS_OK) return done(s, "run");
  s = owqs_get_output_host(sub, U, 128, (int64_t)(rows * cols));
  if (s != OWQS_OK) return done(s, "output");
  const double sc = std::sqrt((double)cols);
  for (uint64_t i = 0; i < 2 * rows * cols; ++i) U[i] *= sc;
  done(OWQS_OK, "");
  if (max_unitarity_err) {
    double worst = 0;
    for (uint64_t i = 0; i < cols; ++i)
      for (uint64_t j = 0; j < cols; ++j) {
        double sr = 0, si = 0;
        for (uint64_t r = 0; r < rows; ++r) {
          double ar = U[2 * (i * rows + r)], ai = U[2 * (i * rows + r) + 1];
          double br = U[2 * (j * rows + r)], bi = U[2 * (j * rows + r) + 1];
          sr += ar * br + ai * bi;
          si += ar * bi - ai * br;
        }
        if (i == j) sr -= 1.0;
        worst = std::max(worst, std::hypot(sr, si));
      }
    *max_unitarity_err = worst;
  }
  return OWQS_OK;
}

owqs_status owqs_gflow(owqs_ctx* ctx, int32_t* layers, int32_t* depth) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "no pattern loaded");
  std::vector<int> layer;
  std::vector<std::vector<int>> g;
  std::string e = find_gflow(ctx->hp, layer, g);
  ctx->gflow_state = e.empty() ? 1 : -1;
  ctx->gflow_msg = e;
  int d = 0;
  for (int q = 0; q < ctx->hp.nq; ++q) {
    d = std::max(d, layer[q]);
    if (layers && ctx->hp.m_ord_of_qubit[q] >= 0) layers[ctx->hp.m_ord_of_qubit[q]] = layer[q];
  }
  if (depth) *depth = d;
  return e.empty() ? OWQS_OK : fail(ctx, OWQS_E_NO_GFLOW, e);
}

owqs_status owqs_pattern_info(owqs_ctx* ctx, int64_t* n_measure, int32_t* paper_m, int32_t* phys_bits,
                              int32_t* n_passes) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "no pattern loaded");
  if (n_measure) *n_measure = ctx->hp.n_measure;
  if (!ctx->subs.empty()) {  // largest sub-state (PAPER §4.1: memory O(2^m), m = largest), passes summed
    if (paper_m) *paper_m = ctx->stats.paper_m;
    if (phys_bits) *phys_bits = ctx->stats.phys_bits;
    if (n_passes) *n_passes = ctx->stats.n_passes;
    return OWQS_OK;
  }
  if (paper_m) *paper_m = ctx->cm[0].plan.paper_m;
  if (phys_bits) *phys_bits = ctx->cm[0].prog.phys_bits;
  if (n_passes) *n_passes = ctx->cm[0].prog.n_passes;
  return OWQS_OK;
}

owqs_status owqs_plan_order(owqs_ctx* ctx, owqs_mode mode, int32_t* qubits, int32_t* ms, int64_t n) {
  if (!ctx || !qubits) return OWQS_E_ARG;
  if (!ctx->subs.empty()) return substates_unsupported(ctx, "owqs_plan_order");
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "no pattern loaded");
  if (n < ctx->hp.n_measure) return fail(ctx, OWQS_E_ARG, "array smaller than n_measure");
  const CompiledMode& m = ctx->cm[mode == OWQS_EOWQS ? 1 : 0];
  for (size_t i = 0; i < m.plan.m_cmds.size(); ++i) {
    qubits[i] = ctx->hp.ext_id[ctx->hp.cmds[m.plan.m_cmds[i]].q0];
    if (ms) ms[i] = m.plan.ms[i];
  }
  return OWQS_OK;
}

owqs_status owqs_set_proa_weights(owqs_ctx* ctx, double a, double b, double g, double d, int32_t tune) {
  if (!ctx) return OWQS_E_ARG;
  if (!(a > 0 && b >= 0 && g >= 0 && d > 0)) return fail(ctx, OWQS_E_ARG, "weights must be positive");
  ctx->weights.a = a;
  ctx->weights.b = b;
  ctx->weights.g = g;
  ctx->weights.d = d;
  ctx->weights.tune = tune != 0;
  if (ctx->loaded && !ctx->subs.empty()) {  // recompile every sub-state
    for (owqs_ctx* c : ctx->subs) {
      c->weights = ctx->weights;
      owqs_status s = load_compiled(c);
      if (s != OWQS_OK) return fail(ctx, s, owqs_last_error(c));
      c->has_input = c->has_output = false;
    }
    ctx->has_input = ctx->has_output = false;
  } else if (ctx->loaded) {
    owqs_status s = compile_modes(ctx);
    if (s != OWQS_OK) return s;
    ctx->has_input = ctx->has_output = false;
  }
  return OWQS_OK;
}

owqs_status owqs_launch_profile(owqs_ctx* ctx, int32_t* kclass, double* bytes, float* ms, int64_t n) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->subs.empty()) return substates_unsupported(ctx, "owqs_launch_profile");
  if (!(ctx->cfg.flags & OWQS_FLAG_PROFILE) || ctx->prof_cm < 0 || !ctx->has_output)
    return fail(ctx, OWQS_E_STATE, "no profiled run (create the context with OWQS_FLAG_PROFILE)");
  const Program& pr = ctx->cm[ctx->prof_cm].prog;
  if (n < (int64_t)pr.steps.size()) return fail(ctx, OWQS_E_ARG, "arrays smaller than the launch count");
  for (size_t i = 0; i < pr.steps.size(); ++i) {
    const StepDesc& s = pr.steps[i];
    const double S = std::ldexp((double)ctx->elem, s.width) * (double)ctx->shards.size();
    int kc = step_kclass(s, ctx->prec);
    if (kclass) kclass[i] = kc;
    if (bytes)
      bytes[i] = s.kind == ST_GROW       ? 3 * S
                 : s.kind == ST_SHRINK   ? 1.5 * S
                 : s.kind == ST_SWAP     ? 2 * S
                 : s.kind == ST_RHOK     ? S
                 : s.kind == ST_SHRINKK  ? S + 3 * std::ldexp(S, -s.jk)
                                         : (s.n_ops > 0 ? 2 * S : S);
    if (ms) {
      float t = 0;
      CU(cudaEventElapsedTime(&t, ctx->prof_ev[i], ctx->prof_ev[i + 1]));
      ms[i] = t;
    }
  }
  return OWQS_OK;
}

owqs_status owqs_stats(owqs_ctx* ctx, owqs_stats_t* out) {
  if (!ctx || !out) return OWQS_E_ARG;
  *out = ctx->stats;
  return OWQS_OK;
}

}  // extern "C"
