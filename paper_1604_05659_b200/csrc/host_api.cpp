// Host-only introspection API (include/owqs_host.h): validation + PROA + compile, no CUDA calls.
#include <string.h>

#include <algorithm>
#include <string>

#include "owqs_host.h"
#include "jit.h"
#include "scheduler.h"

using namespace owqs;

struct owqs_host_plan {
  std::string err;
  HostPattern hp;
  Plan plan;
  Program prog;
  int elem = 16;
  int mode = 0, precision = 128;
  uint32_t flags = 0;
  ProaWeights w;
};

extern "C" {

owqs_status owqs_host_compile(const int32_t* inputs, int32_t n_in, const int32_t* outputs, int32_t n_out,
                              const owqs_cmd* cmds, int64_t n_cmds, const int32_t* domain_pool, int64_t pool_len,
                              int32_t mode, int32_t precision, uint32_t flags, const double* weights,
                              int32_t n_ranks, owqs_host_plan** out) {
  if (!out) return OWQS_E_ARG;
  *out = nullptr;
  if ((precision != 64 && precision != 128) || mode < 0 || mode > 2) return OWQS_E_ARG;
  if (n_ranks < 1 || (n_ranks & (n_ranks - 1))) return OWQS_E_ARG;
  int n_global = 0;
  while ((1 << n_global) < n_ranks) ++n_global;
  owqs_host_plan* h = new owqs_host_plan();
  *out = h;
  std::string e = validate_pattern(inputs, n_in, outputs, n_out, cmds, n_cmds, domain_pool, pool_len, h->hp);
  if (!e.empty()) {
    h->err = e;
    return OWQS_E_PATTERN;
  }
  ProaWeights w;
  if (weights) {
    w.a = weights[0];
    w.b = weights[1];
    w.g = weights[2];
    w.d = weights[3];
  }
  if (flags & OWQS_FLAG_NO_TUNE) w.tune = false;
  plan_and_compile(h->hp, mode, precision == 64 ? 6 : 5, !(flags & OWQS_FLAG_NO_FUSE),
                   (flags & OWQS_FLAG_GIVEN_ORDER) != 0, w, h->plan, h->prog, n_global,
                   jit_max_group(precision == 64 ? 0 : 1, (flags & OWQS_FLAG_NO_JIT) != 0),
                   (flags & OWQS_FLAG_MEASURED_NORM) != 0);
  h->elem = precision == 64 ? 8 : 16;
  h->mode = mode;
  h->precision = precision;
  h->flags = flags;
  h->w = w;
  if (!h->prog.error.empty()) {
    h->err = h->prog.error;
    return OWQS_E_ARG;
  }
  return OWQS_OK;
}

owqs_status owqs_host_substates(const owqs_host_plan* h, int32_t* n, uint64_t* masks, int32_t* phys_bits,
                                int32_t cap) {
  if (!h || !n) return OWQS_E_ARG;
  std::vector<HostPattern> parts;
  std::vector<uint64_t> mk;
  if (!split_substates(h->hp, parts, mk, KRON_MAX)) {
    *n = 1;
    return OWQS_OK;
  }
  *n = (int32_t)parts.size();
  if (!masks && !phys_bits) return OWQS_OK;
  if (cap < *n) return OWQS_E_ARG;
  for (size_t c = 0; c < parts.size(); ++c) {
    if (masks) masks[c] = mk[c];
    if (phys_bits) {
      Plan pl;
      Program pr;
      plan_and_compile(parts[c], h->mode, h->precision == 64 ? 6 : 5, !(h->flags & OWQS_FLAG_NO_FUSE),
                       (h->flags & OWQS_FLAG_GIVEN_ORDER) != 0, h->w, pl, pr, 0,
                       jit_max_group(h->precision == 64 ? 0 : 1, (h->flags & OWQS_FLAG_NO_JIT) != 0),
                       (h->flags & OWQS_FLAG_MEASURED_NORM) != 0);
      if (!pr.error.empty()) return OWQS_E_ARG;
      phys_bits[c] = pr.phys_bits;
    }
  }
  return OWQS_OK;
}

owqs_status owqs_host_info_get(const owqs_host_plan* h, owqs_host_info* info) {
  if (!h || !info) return OWQS_E_ARG;
  memset(info, 0, sizeof(*info));
  info->n_steps = (int64_t)h->prog.steps.size();
  info->n_measure = h->hp.n_measure;
  info->sig_len = (int64_t)h->prog.sig_pool.size();
  info->paper_m = h->plan.paper_m;
  info->phys_bits = h->prog.phys_bits;
  info->in_width = h->prog.in_width;
  info->n_out = (int32_t)h->hp.outputs.size();
  info->step_bytes = (int32_t)sizeof(StepDesc);
  info->mstatic_bytes = (int32_t)sizeof(MStatic);
  info->n_passes = h->prog.n_passes;
  info->n_grow = h->prog.n_grow;
  info->n_shrink = h->prog.n_shrink;
  info->n_reduce = h->prog.n_reduce;
  info->n_swaps = h->prog.n_swaps;
  info->n_global = h->prog.n_global;
  info->bytes_per_run = h->prog.bytes_per_run(h->elem);
  return OWQS_OK;
}

owqs_status owqs_host_program(const owqs_host_plan* h, void* steps, void* mst, int32_t* sig, int32_t* out_slot,
                              int32_t* plan_qubits, int32_t* plan_ms) {
  if (!h) return OWQS_E_ARG;
  if (steps && !h->prog.steps.empty()) memcpy(steps, h->prog.steps.data(), h->prog.steps.size() * sizeof(StepDesc));
  if (mst && !h->prog.mst.empty()) memcpy(mst, h->prog.mst.data(), h->prog.mst.size() * sizeof(MStatic));
  if (sig && !h->prog.sig_pool.empty()) memcpy(sig, h->prog.sig_pool.data(), h->prog.sig_pool.size() * sizeof(int32_t));
  if (out_slot)
    for (size_t k = 0; k < h->prog.out_slot.size(); ++k) out_slot[k] = h->prog.out_slot[k];
  for (size_t i = 0; i < h->plan.m_cmds.size(); ++i) {
    if (plan_qubits) plan_qubits[i] = h->hp.ext_id[h->hp.cmds[h->plan.m_cmds[i]].q0];
    if (plan_ms) plan_ms[i] = h->plan.ms[i];
  }
  return OWQS_OK;
}

owqs_status owqs_host_gflow(const owqs_host_plan* h, int32_t* layers, int32_t* depth) {
  if (!h) return OWQS_E_ARG;
  std::vector<int> layer;
  std::vector<std::vector<int>> g;
  std::string e = find_gflow(h->hp, layer, g);
  int d = 0;
  for (int q = 0; q < h->hp.nq; ++q) {
    d = std::max(d, layer[q]);
    if (layers && h->hp.m_ord_of_qubit[q] >= 0) layers[h->hp.m_ord_of_qubit[q]] = layer[q];
  }
  if (depth) *depth = d;
  return e.empty() ? OWQS_OK : OWQS_E_NO_GFLOW;
}

owqs_status owqs_host_jit(owqs_host_plan* h, int64_t* n_kernels, int64_t* n_jit_steps, double* compile_ms) {
  if (!h) return OWQS_E_ARG;
  const int prec = h->elem == 8 ? 0 : 1;
  std::vector<std::string> names, srcs;
  for (const StepDesc& d : h->prog.steps) {
    if (!jit_eligible(d, prec)) continue;
    std::string nm;
    std::string src = jit_pass_source(d, prec, &nm);
    if (src.empty()) {
      h->err = "pass kernel generation failed";
      return OWQS_E_ARG;
    }
    names.push_back(nm);
    srcs.push_back(src);
  }
  std::vector<JitModule> mods;
  double ms = 0;
  std::string e = jit_compile(names, srcs, mods, &ms);
  if (!e.empty()) {
    h->err = e;
    return OWQS_E_ARG;
  }
  int64_t nk = 0;
  for (auto& m : mods) nk += (int64_t)m.names.size();
  if (n_kernels) *n_kernels = nk;
  if (n_jit_steps) *n_jit_steps = (int64_t)names.size();
  if (compile_ms) *compile_ms = ms;
  return OWQS_OK;
}

owqs_status owqs_host_nvrtc_version(int32_t* major, int32_t* minor) {
  if (!major || !minor) return OWQS_E_ARG;
  int a = 0, b = 0;
  const std::string e = owqs::jit_nvrtc_version(&a, &b);
  *major = a;
  *minor = b;
  return e.empty() ? OWQS_OK : OWQS_E_CUDA;
}

owqs_status owqs_host_jit_source(const owqs_host_plan* h, int64_t step, char* buf, int64_t cap, int64_t* len) {
  if (!h || step < -1 || step >= (int64_t)h->prog.steps.size()) return OWQS_E_ARG;
  const int prec = h->elem == 8 ? 0 : 1;
  std::string src;
  if (step == -1)
    src = jit_prelude();
  else if (jit_eligible(h->prog.steps[step], prec)) src = jit_pass_source(h->prog.steps[step], prec, nullptr);
  if (len) *len = (int64_t)src.size();
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>((size_t)cap - 1, src.size());
    memcpy(buf, src.data(), n);
    buf[n] = 0;
  }
  return OWQS_OK;
}

owqs_status owqs_host_standardize(const owqs_host_plan* h, int32_t signal_shift, owqs_cmd* cmds, int32_t* pool,
                                  int32_t* shift_slices, int32_t* shift_pool, int64_t* sizes) {
  if (!h || !sizes) return OWQS_E_ARG;
  std::vector<HCmd> out;
  std::vector<std::vector<int>> shift;
  int nabs = 0, nsg = 0;
  std::string e = standardize_pattern(h->hp, signal_shift != 0, out, shift, &nabs, &nsg);
  if (!e.empty()) return OWQS_E_PATTERN;
  int64_t plen = 0, slen = 0;
  for (size_t k = 0; k < out.size(); ++k) {
    const HCmd& c = out[k];
    if (cmds) {
      owqs_cmd& o = cmds[k];
      memset(&o, 0, sizeof o);
      o.kind = c.kind;
      o.q0 = h->hp.ext_id[c.q0];
      o.q1 = c.kind == H_E ? h->hp.ext_id[c.q1] : 0;
      o.angle = c.angle;
      o.s_off = (int32_t)plen;
      o.s_len = (int32_t)c.sdom.size();
      if (pool)
        for (size_t j = 0; j < c.sdom.size(); ++j) pool[plen + j] = h->hp.ext_id[c.sdom[j]];
      o.t_off = (int32_t)(plen + c.sdom.size());
      o.t_len = (int32_t)c.tdom.size();
      if (pool)
        for (size_t j = 0; j < c.tdom.size(); ++j) pool[plen + c.sdom.size() + j] = h->hp.ext_id[c.tdom[j]];
      if (o.s_len == 0) o.s_off = 0;
      if (o.t_len == 0) o.t_off = 0;
    }
    plen += (int64_t)(c.sdom.size() + c.tdom.size());
    const std::vector<int>* sh = (c.kind == H_M && !shift.empty()) ? &shift[c.q0] : nullptr;
    if (shift_slices) {
      shift_slices[2 * k] = (int32_t)slen;
      shift_slices[2 * k + 1] = sh ? (int32_t)sh->size() : 0;
    }
    if (sh) {
      if (shift_pool)
        for (size_t j = 0; j < sh->size(); ++j) shift_pool[slen + j] = h->hp.ext_id[(*sh)[j]];
      slen += (int64_t)sh->size();
    }
  }
  sizes[0] = (int64_t)out.size();
  sizes[1] = plen;
  sizes[2] = slen;
  sizes[3] = nabs;
  return OWQS_OK;
}

const char* owqs_host_error(const owqs_host_plan* h) { return h ? h->err.c_str() : "NULL handle"; }

void owqs_host_free(owqs_host_plan* h) { delete h; }

}  // extern "C"
