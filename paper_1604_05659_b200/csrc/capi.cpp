// C-ABI implementation (include/owqs.h): context, device memory, CUDA-graph executor.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <string>
#include <vector>

#include "owqs.h"
#include "scheduler.h"

namespace owqs {
cudaError_t init_kernel_limits(int device);
int max_partial_blocks();
cudaError_t launch_step(const StepDesc& d, const DevPtrs& p, int prec, cudaStream_t s);
cudaError_t launch_permute_out(const void* state, int prec, void* out, int out_prec, int nbits, const int* slots,
                               uint64_t j0, uint64_t count, cudaStream_t s);
cudaError_t launch_convert_in(const void* src, int src_prec, void* state, int prec, uint64_t j0, uint64_t count,
                              cudaStream_t s);
cudaError_t launch_basis(void* state, int prec, uint64_t n, uint64_t k, cudaStream_t s);
cudaError_t launch_haar(const DevPtrs& p, int prec, uint64_t n, uint64_t seed, cudaStream_t s);
cudaError_t launch_dot(const DevPtrs& p, const void* a, const void* b, uint64_t n, cudaStream_t s);
int step_kclass(const StepDesc& d, int prec);
}  // namespace owqs

using namespace owqs;

namespace {
struct CompiledMode {
  bool valid = false;
  Plan plan;
  Program prog;
  MStatic* d_mst = nullptr;
  int32_t* d_sig = nullptr;
  cudaGraphExec_t gexec = nullptr;
  double schedule_ms = 0;
};
constexpr size_t kStagingBytes = 64ull << 20;
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
  void* d_state = nullptr;
  size_t state_bytes = 0;
  double* d_partials = nullptr;
  unsigned* d_counter = nullptr;
  double* d_red = nullptr;
  int32_t* d_err = nullptr;
  RunParams* d_run = nullptr;
  uint8_t* d_outcome = nullptr;
  double* d_prob0 = nullptr;
  uint8_t* d_forced = nullptr;
  size_t k_cap = 0;
  void* d_staging = nullptr;
  void* h_staging = nullptr;  // pinned
  bool has_input = false, has_output = false;
  int out_cm = -1;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  owqs_stats_t stats{};
  int last_cm = 0;
  std::vector<cudaEvent_t> prof_ev;  // OWQS_FLAG_PROFILE: event after every launch (+1 start)
  int prof_cm = -1;
};

namespace {

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

DevPtrs dev_ptrs(owqs_ctx* ctx, const CompiledMode& m) {
  DevPtrs p{};
  p.state = ctx->d_state;
  p.mst = m.d_mst;
  p.outcome = ctx->d_outcome;
  p.prob0 = ctx->d_prob0;
  p.forced = ctx->d_forced;
  p.sig_pool = m.d_sig;
  p.run = ctx->d_run;
  p.partials = ctx->d_partials;
  p.counter = ctx->d_counter;
  p.red_result = ctx->d_red;
  p.err = ctx->d_err;
  return p;
}

void free_mode(CompiledMode& m) {
  if (m.gexec) cudaGraphExecDestroy(m.gexec);
  if (m.d_mst) cudaFree(m.d_mst);
  if (m.d_sig) cudaFree(m.d_sig);
  m = CompiledMode();
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
    plan_and_compile(ctx->hp, i == 1 ? 2 : 0, SB, fuse, given, w, m.plan, m.prog);
    for (const auto& s : m.prog.steps)
      if (s.kind == ST_PASS && s.width > 12 && s.width - SB - s.nb_hi < 0)
        return fail(ctx, OWQS_E_PATTERN, "internal: pass grouping exceeds the register file");
    m.schedule_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    m.valid = true;
  }
  return OWQS_OK;
}

owqs_status ensure_device(owqs_ctx* ctx) {
  CU(cudaSetDevice(ctx->cfg.device));
  int phys = 0;
  for (int i = 0; i < 2; ++i) phys = std::max(phys, ctx->cm[i].prog.phys_bits);
  size_t need = (size_t)ctx->elem << phys;
  need = std::max<size_t>(need, 64);
  if (ctx->state_bytes < need) {
    if (ctx->d_state) cudaFree(ctx->d_state);
    ctx->d_state = nullptr;
    ctx->state_bytes = 0;
    for (int i = 0; i < 2; ++i)
      if (ctx->cm[i].gexec) {
        cudaGraphExecDestroy(ctx->cm[i].gexec);
        ctx->cm[i].gexec = nullptr;
      }
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (need > free_b)
      return fail(ctx, OWQS_E_NOMEM, "state of 2^" + std::to_string(phys) + " amplitudes (" +
                                         std::to_string(need >> 20) + " MiB) exceeds free device memory");
    CU(cudaMalloc(&ctx->d_state, need));
    ctx->state_bytes = need;
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
    for (int i = 0; i < 2; ++i)
      if (ctx->cm[i].gexec) {
        cudaGraphExecDestroy(ctx->cm[i].gexec);
        ctx->cm[i].gexec = nullptr;
      }
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
  }
  return OWQS_OK;
}

owqs_status run_internal(owqs_ctx* ctx, int cmi, int mode, uint64_t seed, const uint8_t* forced) {
  CompiledMode& m = ctx->cm[cmi];
  RunParams rp{};
  rp.mode = mode;
  rp.seed = seed;
  CU(cudaMemcpyAsync(ctx->d_run, &rp, sizeof(rp), cudaMemcpyHostToDevice, ctx->stream));
  if (mode == OWQS_FORCED && ctx->hp.n_measure > 0)
    CU(cudaMemcpyAsync(ctx->d_forced, forced, ctx->hp.n_measure, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemsetAsync(ctx->d_err, 0, sizeof(int32_t), ctx->stream));
  DevPtrs p = dev_ptrs(ctx, m);
  const bool use_graph = !(ctx->cfg.flags & OWQS_FLAG_NO_GRAPH);
  const bool prof = (ctx->cfg.flags & OWQS_FLAG_PROFILE) != 0;
  if (prof) {
    if (ctx->prof_cm != cmi) {
      // event lists are per compiled mode: rebuild (and drop this mode's graph) on a mode switch
      if (m.gexec) {
        cudaGraphExecDestroy(m.gexec);
        m.gexec = nullptr;
      }
    }
    while (ctx->prof_ev.size() < m.prog.steps.size() + 1) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      ctx->prof_ev.push_back(e);
    }
    ctx->prof_cm = cmi;
  }
  auto launch_all = [&](bool capturing) -> cudaError_t {
    cudaError_t e = cudaSuccess;
    if (prof) e = capturing ? cudaEventRecordWithFlags(ctx->prof_ev[0], ctx->stream, cudaEventRecordExternal)
                            : cudaEventRecord(ctx->prof_ev[0], ctx->stream);
    for (size_t i = 0; i < m.prog.steps.size() && e == cudaSuccess; ++i) {
      e = launch_step(m.prog.steps[i], p, ctx->prec, ctx->stream);
      if (e == cudaSuccess && prof)
        e = capturing ? cudaEventRecordWithFlags(ctx->prof_ev[i + 1], ctx->stream, cudaEventRecordExternal)
                      : cudaEventRecord(ctx->prof_ev[i + 1], ctx->stream);
    }
    return e;
  };
  if (use_graph && !m.gexec) {
    cudaGraph_t g = nullptr;
    CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = launch_all(true);
    if (e != cudaSuccess) {
      cudaStreamEndCapture(ctx->stream, &g);
      if (g) cudaGraphDestroy(g);
      return fail(ctx, OWQS_E_CUDA, std::string("launch during capture: ") + cudaGetErrorString(e));
    }
    CU(cudaStreamEndCapture(ctx->stream, &g));
    CU(cudaGraphInstantiate(&m.gexec, g, 0));
    cudaGraphDestroy(g);
  }
  CU(cudaEventRecord(ctx->ev0, ctx->stream));
  if (use_graph) {
    CU(cudaGraphLaunch(m.gexec, ctx->stream));
  } else {
    CU(launch_all(false));
  }
  CU(cudaEventRecord(ctx->ev1, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  ctx->stats.last_run_ms = ms;
  ctx->last_cm = cmi;
  int32_t herr = 0;
  CU(cudaMemcpy(&herr, ctx->d_err, sizeof(herr), cudaMemcpyDeviceToHost));
  ctx->has_input = false;
  ctx->has_output = true;
  ctx->out_cm = cmi;
  if (herr) return fail(ctx, OWQS_E_BRANCH, "forced outcome on a branch with probability < 1e-12");
  return OWQS_OK;
}

owqs_status output_to_device(owqs_ctx* ctx, void* dst, int dst_prec, uint64_t j0, uint64_t count) {
  const Program& pr = ctx->cm[ctx->out_cm].prog;
  CU(launch_permute_out(ctx->d_state, ctx->prec, dst, dst_prec, (int)pr.out_slot.size(), pr.out_slot.data(), j0,
                        count, ctx->stream));
  return OWQS_OK;
}

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

owqs_status output_to_host(owqs_ctx* ctx, double* amps) {
  const uint64_t n = 1ull << ctx->hp.outputs.size();
  const uint64_t chunk = kStagingBytes / 16;
  const bool pinned = is_pinned_host(amps);  // page-locked caller buffer: DMA straight into it
  for (uint64_t j0 = 0; j0 < n; j0 += chunk) {
    uint64_t cnt = std::min(chunk, n - j0);
    owqs_status s = output_to_device(ctx, ctx->d_staging, 1, j0, cnt);
    if (s != OWQS_OK) return s;
    CU(cudaMemcpyAsync(pinned ? (void*)(amps + 2 * j0) : ctx->h_staging, ctx->d_staging, cnt * 16,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (!pinned) memcpy(amps + 2 * j0, ctx->h_staging, cnt * 16);
  }
  return OWQS_OK;
}

}  // namespace

extern "C" {

const char* owqs_version(void) { return "owqs-b200 0.1 (sm_100a)"; }

const char* owqs_last_error(const owqs_ctx* ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }

owqs_status owqs_create(const owqs_config* cfg, owqs_ctx** out) {
  if (!cfg || !out) return OWQS_E_ARG;
  *out = nullptr;
  if (cfg->precision != 64 && cfg->precision != 128) return OWQS_E_ARG;
  if (cfg->n_ranks != 1 && cfg->n_ranks != 0) return OWQS_E_ARG;  // multi-rank: DESIGN.md §7
  owqs_ctx* ctx = new owqs_ctx();
  ctx->cfg = *cfg;
  ctx->cfg.n_ranks = 1;
  ctx->prec = cfg->precision == 64 ? 0 : 1;
  ctx->elem = cfg->precision == 64 ? 8 : 16;
  auto bail = [&](owqs_status s) {
    owqs_destroy(ctx);
    return s;
  };
  if (cudaSetDevice(cfg->device) != cudaSuccess) return bail(OWQS_E_CUDA);
  if (init_kernel_limits(cfg->device) != cudaSuccess) return bail(OWQS_E_CUDA);
  if (cfg->stream) {
    ctx->stream = (cudaStream_t)cfg->stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(OWQS_E_CUDA);
    ctx->own_stream = true;
  }
  if (cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) return bail(OWQS_E_CUDA);
  const int nb = max_partial_blocks();
  if (cudaMalloc(&ctx->d_partials, (size_t)nb * 4 * sizeof(double)) != cudaSuccess) return bail(OWQS_E_NOMEM);
  if (cudaMalloc(&ctx->d_counter, sizeof(unsigned)) != cudaSuccess) return bail(OWQS_E_NOMEM);
  if (cudaMemset(ctx->d_counter, 0, sizeof(unsigned)) != cudaSuccess) return bail(OWQS_E_CUDA);
  if (cudaMalloc(&ctx->d_red, 4 * sizeof(double)) != cudaSuccess) return bail(OWQS_E_NOMEM);
  if (cudaMalloc(&ctx->d_err, sizeof(int32_t)) != cudaSuccess) return bail(OWQS_E_NOMEM);
  if (cudaMalloc(&ctx->d_run, sizeof(RunParams)) != cudaSuccess) return bail(OWQS_E_NOMEM);
  if (cudaMalloc(&ctx->d_staging, kStagingBytes) != cudaSuccess) return bail(OWQS_E_NOMEM);
  if (cudaMallocHost(&ctx->h_staging, kStagingBytes) != cudaSuccess) return bail(OWQS_E_NOMEM);
  *out = ctx;
  return OWQS_OK;
}

void owqs_destroy(owqs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (int i = 0; i < 2; ++i) free_mode(ctx->cm[i]);
  cudaFree(ctx->d_state);
  cudaFree(ctx->d_partials);
  cudaFree(ctx->d_counter);
  cudaFree(ctx->d_red);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_run);
  cudaFree(ctx->d_outcome);
  cudaFree(ctx->d_prob0);
  cudaFree(ctx->d_forced);
  cudaFree(ctx->d_staging);
  if (ctx->h_staging) cudaFreeHost(ctx->h_staging);
  for (cudaEvent_t e : ctx->prof_ev) cudaEventDestroy(e);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

owqs_status owqs_load_pattern(owqs_ctx* ctx, const int32_t* inputs, int32_t n_in, const int32_t* outputs,
                              int32_t n_out, const owqs_cmd* cmds, int64_t n_cmds, const int32_t* domain_pool,
                              int64_t pool_len) {
  if (!ctx) return OWQS_E_ARG;
  ctx->loaded = false;
  ctx->has_input = ctx->has_output = false;
  std::string e = validate_pattern(inputs, n_in, outputs, n_out, cmds, n_cmds, domain_pool, pool_len, ctx->hp);
  if (!e.empty()) return fail(ctx, OWQS_E_PATTERN, e);
  if (n_in > 40 || n_out > 40) return fail(ctx, OWQS_E_ARG, "more than 40 input/output qubits");
  owqs_status s = compile_modes(ctx);
  if (s != OWQS_OK) return s;
  const Program& pr = ctx->cm[0].prog;
  ctx->stats = owqs_stats_t{};
  ctx->stats.n_commands = (int64_t)ctx->hp.cmds.size();
  ctx->stats.n_measure = ctx->hp.n_measure;
  ctx->stats.paper_m = ctx->cm[0].plan.paper_m;
  ctx->stats.phys_bits = pr.phys_bits;
  ctx->stats.n_passes = pr.n_passes;
  ctx->stats.n_grow = pr.n_grow;
  ctx->stats.n_shrink = pr.n_shrink;
  ctx->stats.n_reduce = pr.n_reduce;
  ctx->stats.n_launches = (int32_t)pr.steps.size();
  ctx->stats.bytes_per_run = pr.bytes_per_run(ctx->elem);
  ctx->stats.schedule_ms = ctx->cm[0].schedule_ms;
  if (pr.phys_bits > 40) return fail(ctx, OWQS_E_NOMEM, "physical width above 40 bits");
  ctx->loaded = true;
  return OWQS_OK;
}

owqs_status owqs_set_input(owqs_ctx* ctx, const double* amps, int64_t n_amps) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "set_input before load_pattern");
  const uint64_t n = 1ull << ctx->hp.inputs.size();
  if (!amps || n_amps != (int64_t)n) return fail(ctx, OWQS_E_ARG, "input must hold 2^n_in amplitudes");
  owqs_status s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  const uint64_t chunk = kStagingBytes / 16;
  for (uint64_t j0 = 0; j0 < n; j0 += chunk) {
    uint64_t cnt = std::min(chunk, n - j0);
    if (ctx->prec == 1) {
      CU(cudaMemcpyAsync((char*)ctx->d_state + j0 * 16, amps + 2 * j0, cnt * 16, cudaMemcpyHostToDevice, ctx->stream));
    } else {
      CU(cudaMemcpyAsync(ctx->d_staging, amps + 2 * j0, cnt * 16, cudaMemcpyHostToDevice, ctx->stream));
      CU(launch_convert_in(ctx->d_staging, 1, ctx->d_state, 0, j0, cnt, ctx->stream));
    }
  }
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->has_input = true;
  ctx->has_output = false;
  return OWQS_OK;
}

owqs_status owqs_set_input_device(owqs_ctx* ctx, const void* dev_amps, int32_t precision, int64_t n_amps) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "set_input before load_pattern");
  const uint64_t n = 1ull << ctx->hp.inputs.size();
  if (!dev_amps || n_amps != (int64_t)n || (precision != 64 && precision != 128))
    return fail(ctx, OWQS_E_ARG, "input must hold 2^n_in amplitudes of precision 64 or 128");
  owqs_status s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  const int sp = precision == 64 ? 0 : 1;
  if (sp == ctx->prec) {
    CU(cudaMemcpyAsync(ctx->d_state, dev_amps, n * ctx->elem, cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    CU(launch_convert_in(dev_amps, sp, ctx->d_state, ctx->prec, 0, n, ctx->stream));
  }
  ctx->has_input = true;
  ctx->has_output = false;
  return OWQS_OK;
}

owqs_status owqs_set_input_random(owqs_ctx* ctx, uint64_t seed) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "set_input before load_pattern");
  owqs_status s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  DevPtrs p = dev_ptrs(ctx, ctx->cm[0]);
  CU(launch_haar(p, ctx->prec, 1ull << ctx->hp.inputs.size(), seed, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->has_input = true;
  ctx->has_output = false;
  return OWQS_OK;
}

owqs_status owqs_run(owqs_ctx* ctx, owqs_mode mode, uint64_t seed, const uint8_t* forced, uint8_t* outcomes_out,
                     double* prob0_out) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "run before load_pattern");
  if (!ctx->has_input) return fail(ctx, OWQS_E_STATE, "run without a fresh input (set_input consumes per run)");
  if (mode != OWQS_SAMPLED && mode != OWQS_FORCED && mode != OWQS_EOWQS) return fail(ctx, OWQS_E_ARG, "bad mode");
  if (mode == OWQS_FORCED && ctx->hp.n_measure > 0 && !forced) return fail(ctx, OWQS_E_ARG, "forced outcomes missing");
  const int cmi = mode == OWQS_EOWQS ? 1 : 0;
  owqs_status s = run_internal(ctx, cmi, mode, seed, forced);
  const int64_t K = ctx->hp.n_measure;
  if (K > 0 && (s == OWQS_OK || s == OWQS_E_BRANCH)) {
    if (outcomes_out) {
      if (mode == OWQS_EOWQS)
        memset(outcomes_out, 0, K);
      else
        CU(cudaMemcpy(outcomes_out, ctx->d_outcome, K, cudaMemcpyDeviceToHost));
    }
    if (prob0_out) {
      if (mode == OWQS_EOWQS)
        for (int64_t i = 0; i < K; ++i) prob0_out[i] = -1.0;
      else
        CU(cudaMemcpy(prob0_out, ctx->d_prob0, K * sizeof(double), cudaMemcpyDeviceToHost));
    }
  }
  if (s != OWQS_OK) return s;
  const Program& pr = ctx->cm[cmi].prog;
  ctx->stats.n_passes = pr.n_passes;
  ctx->stats.n_grow = pr.n_grow;
  ctx->stats.n_shrink = pr.n_shrink;
  ctx->stats.n_reduce = pr.n_reduce;
  ctx->stats.n_launches = (int32_t)pr.steps.size();
  ctx->stats.bytes_per_run = pr.bytes_per_run(ctx->elem);
  ctx->stats.schedule_ms = ctx->cm[cmi].schedule_ms;
  ctx->stats.phys_bits = pr.phys_bits;
  if (mode == OWQS_EOWQS) {
    double red[4];
    CU(cudaMemcpy(red, ctx->d_red, sizeof(red), cudaMemcpyDeviceToHost));
    const double tol = ctx->prec == 1 ? 1e-8 : 1e-3;
    if (!(std::fabs(red[0] - 1.0) <= tol))
      return fail(ctx, OWQS_E_NOT_DETERMINISTIC,
                  "EOWQS output norm^2 = " + std::to_string(red[0]) + ": the pattern is not deterministic");
  }
  return OWQS_OK;
}

owqs_status owqs_get_output(owqs_ctx* ctx, double* amps, int64_t n_amps) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->has_output) return fail(ctx, OWQS_E_STATE, "no output: run first");
  const uint64_t n = 1ull << ctx->hp.outputs.size();
  if (!amps || n_amps < (int64_t)n) return fail(ctx, OWQS_E_ARG, "output buffer smaller than 2^n_out");
  return output_to_host(ctx, amps);
}

owqs_status owqs_get_output_device(owqs_ctx* ctx, void* dev_amps, int32_t precision, int64_t n_amps) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->has_output) return fail(ctx, OWQS_E_STATE, "no output: run first");
  const uint64_t n = 1ull << ctx->hp.outputs.size();
  if (!dev_amps || n_amps < (int64_t)n || (precision != 64 && precision != 128))
    return fail(ctx, OWQS_E_ARG, "bad output buffer");
  owqs_status s = output_to_device(ctx, dev_amps, precision == 64 ? 0 : 1, 0, n);
  if (s != OWQS_OK) return s;
  CU(cudaStreamSynchronize(ctx->stream));
  return OWQS_OK;
}

owqs_status owqs_output_inner(owqs_ctx* a, owqs_ctx* b, double* re, double* im) {
  owqs_ctx* ctx = a;
  if (!a || !b || !re || !im) return OWQS_E_ARG;
  if (!a->has_output || !b->has_output) return fail(a, OWQS_E_STATE, "no output: run first");
  if (a->hp.outputs.size() != b->hp.outputs.size()) return fail(a, OWQS_E_ARG, "output widths differ");
  const uint64_t n = 1ull << a->hp.outputs.size();
  void *ta = nullptr, *tb = nullptr;
  CU(cudaMalloc(&ta, n * 16));
  cudaError_t e2 = cudaMalloc(&tb, n * 16);
  if (e2 != cudaSuccess) {
    cudaFree(ta);
    return fail(a, OWQS_E_NOMEM, "inner product scratch");
  }
  owqs_status s = output_to_device(a, ta, 1, 0, n);
  if (s == OWQS_OK) {
    const Program& pb = b->cm[b->out_cm].prog;
    cudaError_t e = launch_permute_out(b->d_state, b->prec, tb, 1, (int)pb.out_slot.size(), pb.out_slot.data(), 0, n,
                                       a->stream);
    if (e == cudaSuccess) e = launch_dot(dev_ptrs(a, a->cm[0]), ta, tb, n, a->stream);
    double red[4] = {0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(red, a->d_red, sizeof(red), cudaMemcpyDeviceToHost, a->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(a->stream);
    if (e != cudaSuccess) s = fail(a, OWQS_E_CUDA, cudaGetErrorString(e));
    *re = red[0];
    *im = red[1];
  }
  cudaFree(ta);
  cudaFree(tb);
  return s;
}

owqs_status owqs_recognize(owqs_ctx* ctx, double* U, int64_t n, double* max_unitarity_err) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "recognize before load_pattern");
  const int ni = (int)ctx->hp.inputs.size(), no = (int)ctx->hp.outputs.size();
  if (ni > 14 || no > 14) return fail(ctx, OWQS_E_ARG, "recognize is limited to 14 input/output qubits");
  const uint64_t rows = 1ull << no, cols = 1ull << ni;
  if (!U || n < (int64_t)(rows * cols)) return fail(ctx, OWQS_E_ARG, "U must hold 2^n_out * 2^n_in entries");
  owqs_status s = ensure_device(ctx);
  if (s != OWQS_OK) return s;
  for (uint64_t k = 0; k < cols; ++k) {
    CU(launch_basis(ctx->d_state, ctx->prec, cols, k, ctx->stream));
    ctx->has_input = true;
    s = run_internal(ctx, 1, OWQS_EOWQS, 0, nullptr);
    if (s != OWQS_OK) return s;
    s = output_to_host(ctx, U + 2 * k * rows);
    if (s != OWQS_OK) return s;
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

owqs_status owqs_pattern_info(owqs_ctx* ctx, int64_t* n_measure, int32_t* paper_m, int32_t* phys_bits,
                              int32_t* n_passes) {
  if (!ctx) return OWQS_E_ARG;
  if (!ctx->loaded) return fail(ctx, OWQS_E_STATE, "no pattern loaded");
  if (n_measure) *n_measure = ctx->hp.n_measure;
  if (paper_m) *paper_m = ctx->cm[0].plan.paper_m;
  if (phys_bits) *phys_bits = ctx->cm[0].prog.phys_bits;
  if (n_passes) *n_passes = ctx->cm[0].prog.n_passes;
  return OWQS_OK;
}

owqs_status owqs_plan_order(owqs_ctx* ctx, owqs_mode mode, int32_t* qubits, int32_t* ms, int64_t n) {
  if (!ctx || !qubits) return OWQS_E_ARG;
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
  if (ctx->loaded) {
    owqs_status s = compile_modes(ctx);
    if (s != OWQS_OK) return s;
    ctx->has_input = ctx->has_output = false;
  }
  return OWQS_OK;
}

owqs_status owqs_launch_profile(owqs_ctx* ctx, int32_t* kclass, double* bytes, float* ms, int64_t n) {
  if (!ctx) return OWQS_E_ARG;
  if (!(ctx->cfg.flags & OWQS_FLAG_PROFILE) || ctx->prof_cm < 0 || !ctx->has_output)
    return fail(ctx, OWQS_E_STATE, "no profiled run (create the context with OWQS_FLAG_PROFILE)");
  const Program& pr = ctx->cm[ctx->prof_cm].prog;
  if (n < (int64_t)pr.steps.size()) return fail(ctx, OWQS_E_ARG, "arrays smaller than the launch count");
  for (size_t i = 0; i < pr.steps.size(); ++i) {
    const StepDesc& s = pr.steps[i];
    const double S = std::ldexp((double)ctx->elem, s.width);
    int kc = step_kclass(s, ctx->prec);
    if (kclass) kclass[i] = kc;
    if (bytes) bytes[i] = s.kind == ST_GROW ? 3 * S : s.kind == ST_SHRINK ? 1.5 * S : (s.n_ops > 0 ? 2 * S : S);
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
