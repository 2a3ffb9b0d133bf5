// Host scheduler: validation, dependency DAG (Eqs. 14-16), PROA (Eq. 18,
// tuning L487) and the slot-reuse compiler.
#include "scheduler.h"

#include <algorithm>
#include <functional>
#include <cmath>
#include <cstring>
#include <sstream>
#include <unordered_map>
#include <unordered_set>
#include <cstdio>
#include <cstdlib>

#include "owqs.h"

namespace owqs {

constexpr int MAX_OPS_HARD = MAX_OPS;

namespace {
std::string fmt_cmd(int64_t i) {
  std::ostringstream os;
  os << "command " << i;
  return os.str();
}
}  // namespace

// ------------------------------------------------------------------------------------------------
// Validation. States: 0 unprepared, 1 live, 2 measured. D0: signals only reference measured
// qubits. D1: no action on a measured qubit. D2: non-inputs are prepared before use (implicit N
// at first use, reading R-11). D3: measured iff not output.
// ------------------------------------------------------------------------------------------------
std::string validate_pattern(const int32_t* inputs, int n_in, const int32_t* outputs, int n_out,
                             const void* cmds_v, int64_t n_cmds, const int32_t* pool,
                             int64_t pool_len, HostPattern& hp) {
  const owqs_cmd* cmds = static_cast<const owqs_cmd*>(cmds_v);
  hp = HostPattern();
  std::unordered_map<int32_t, int> dense;
  auto idx = [&](int32_t ext) -> int {
    auto it = dense.find(ext);
    if (it != dense.end()) return it->second;
    int d = (int)hp.ext_id.size();
    dense.emplace(ext, d);
    hp.ext_id.push_back(ext);
    return d;
  };
  if (n_in < 0 || n_out < 0 || n_cmds < 0 || pool_len < 0) return "negative size";
  if ((n_in > 0 && !inputs) || (n_out > 0 && !outputs) || (n_cmds > 0 && !cmds)) return "NULL array";
  for (int i = 0; i < n_in; ++i) {
    if (inputs[i] < 0) return "negative qubit id in inputs";
    if (dense.count(inputs[i])) return "duplicate input qubit";
    hp.inputs.push_back(idx(inputs[i]));
  }
  std::unordered_set<int32_t> outset;
  for (int i = 0; i < n_out; ++i) {
    if (outputs[i] < 0) return "negative qubit id in outputs";
    if (!outset.insert(outputs[i]).second) return "duplicate output qubit";
  }
  // first pass: register ids in order of appearance
  for (int64_t c = 0; c < n_cmds; ++c) {
    const owqs_cmd& k = cmds[c];
    if (k.kind < 0 || k.kind > 4) return fmt_cmd(c) + ": unknown kind";
    if (k.q0 < 0) return fmt_cmd(c) + ": negative qubit id";
    idx(k.q0);
    if (k.kind == OWQS_CMD_E) {
      if (k.q1 < 0) return fmt_cmd(c) + ": negative qubit id";
      if (k.q1 == k.q0) return fmt_cmd(c) + ": E on a single qubit";
      idx(k.q1);
    }
    auto chk = [&](int32_t off, int32_t len) -> bool {
      return len == 0 || (off >= 0 && len > 0 && off + (int64_t)len <= pool_len && pool);
    };
    if (k.kind == OWQS_CMD_M || k.kind == OWQS_CMD_X || k.kind == OWQS_CMD_Z) {
      if (!chk(k.s_off, k.s_len)) return fmt_cmd(c) + ": s-domain out of domain_pool";
    }
    if (k.kind == OWQS_CMD_M && !chk(k.t_off, k.t_len)) return fmt_cmd(c) + ": t-domain out of domain_pool";
    if (k.kind == OWQS_CMD_M && !std::isfinite(k.angle)) return fmt_cmd(c) + ": non-finite angle";
  }
  for (int i = 0; i < n_out; ++i) hp.outputs.push_back(idx(outputs[i]));
  hp.nq = (int)hp.ext_id.size();
  hp.is_output.assign(hp.nq, 0);
  hp.is_input.assign(hp.nq, 0);
  for (int o : hp.outputs) hp.is_output[o] = 1;
  for (int i : hp.inputs) hp.is_input[i] = 1;

  std::vector<int> st(hp.nq, 0);
  for (int i : hp.inputs) st[i] = 1;
  std::unordered_set<uint64_t> epairs;
  hp.m_ord_of_qubit.assign(hp.nq, -1);
  auto need_live = [&](int q, int64_t c, std::string& err) {
    if (st[q] == 2) {
      err = fmt_cmd(c) + ": D1 violated (action on measured qubit " + std::to_string(hp.ext_id[q]) + ")";
      return;
    }
    if (st[q] == 0) {  // implicit N at first use (R-11)
      HCmd n;
      n.kind = H_N;
      n.q0 = q;
      hp.cmds.push_back(n);
      st[q] = 1;
    }
  };
  auto dom = [&](int32_t off, int32_t len, std::vector<int>& out, int64_t c, std::string& err) {
    for (int32_t j = 0; j < len; ++j) {
      int32_t e = pool[off + j];
      auto it = dense.find(e);
      if (it == dense.end() || st[it->second] != 2) {
        err = fmt_cmd(c) + ": D0 violated (signal on unmeasured qubit " + std::to_string(e) + ")";
        return;
      }
      out.push_back(it->second);
    }
  };
  for (int64_t c = 0; c < n_cmds; ++c) {
    const owqs_cmd& k = cmds[c];
    std::string err;
    HCmd h;
    h.kind = k.kind;
    h.q0 = dense[k.q0];
    if (k.kind == OWQS_CMD_N) {
      if (st[h.q0] != 0) return fmt_cmd(c) + ": N on a prepared, input or measured qubit";
      st[h.q0] = 1;
      hp.cmds.push_back(h);
      continue;
    }
    if (k.kind == OWQS_CMD_E) {
      h.q1 = dense[k.q1];
      need_live(h.q0, c, err);
      if (err.empty()) need_live(h.q1, c, err);
      if (!err.empty()) return err;
      uint64_t a = std::min(h.q0, h.q1), b = std::max(h.q0, h.q1);
      if (!epairs.insert((a << 32) | b).second) return fmt_cmd(c) + ": duplicate E on one qubit pair";
      hp.cmds.push_back(h);
      continue;
    }
    need_live(h.q0, c, err);
    if (!err.empty()) return err;
    dom(k.s_off, k.s_len, h.sdom, c, err);
    if (!err.empty()) return err;
    if (k.kind == OWQS_CMD_M) {
      dom(k.t_off, k.t_len, h.tdom, c, err);
      if (!err.empty()) return err;
      if (hp.is_output[h.q0]) return fmt_cmd(c) + ": D3 violated (output qubit measured)";
      h.angle = k.angle;
      hp.m_ord_of_qubit[h.q0] = hp.n_measure++;
      hp.cmds.push_back(h);
      st[h.q0] = 2;
      continue;
    }
    hp.cmds.push_back(h);  // X / Z
  }
  for (int q = 0; q < hp.nq; ++q) {
    if (!hp.is_output[q] && st[q] != 2)
      return "D3 violated: non-output qubit " + std::to_string(hp.ext_id[q]) + " is never measured";
    if (hp.is_output[q] && st[q] == 0) {  // output never touched: |+> (R-11)
      HCmd n;
      n.kind = H_N;
      n.q0 = q;
      hp.cmds.push_back(n);
      st[q] = 1;
    }
  }
  hp.m_ord_of_cmd.assign(hp.cmds.size(), -1);
  for (size_t c = 0; c < hp.cmds.size(); ++c)
    if (hp.cmds[c].kind == H_M) hp.m_ord_of_cmd[c] = hp.m_ord_of_qubit[hp.cmds[c].q0];
  return "";
}

// ------------------------------------------------------------------------------------------------
// DAG of non-commuting commands on a shared qubit (Eqs. 14-16 and the Pauli relations) plus
// signal edges M_v -> (command whose domain contains v) (D0, L79).
// ------------------------------------------------------------------------------------------------
namespace {

bool commute_on_shared(int ka, int kb) {
  if (ka == H_N || kb == H_N || ka == H_M || kb == H_M) return false;
  auto diag = [](int k) { return k == H_E || k == H_Z; };
  if (diag(ka) && diag(kb)) return true;     // E-E (Eq. 15), E-Z, Z-Z
  if (ka == H_X && kb == H_X) return true;   // X-X
  return false;                              // E-X, X-Z (anticommute: phase)
}

struct Dag {
  std::vector<std::vector<int>> pred;
  std::vector<char> active;  // command participates in this mode's plan
};

Dag build_dag(const HostPattern& hp, bool eowqs) {
  const int nc = (int)hp.cmds.size();
  Dag g;
  g.pred.assign(nc, {});
  g.active.assign(nc, 1);
  std::vector<std::vector<int>> on_qubit(hp.nq);
  std::vector<int> m_cmd_of_qubit(hp.nq, -1);
  for (int c = 0; c < nc; ++c) {
    const HCmd& h = hp.cmds[c];
    if (eowqs && (h.kind == H_X || h.kind == H_Z)) {  // signals are 0: corrections are identity
      g.active[c] = 0;
      continue;
    }
    int qs[2] = {h.q0, h.kind == H_E ? h.q1 : -1};
    for (int qi = 0; qi < 2; ++qi) {
      int q = qs[qi];
      if (q < 0) continue;
      for (int p : on_qubit[q])
        if (!commute_on_shared(hp.cmds[p].kind, h.kind)) g.pred[c].push_back(p);
      on_qubit[q].push_back(c);
    }
    if (!eowqs) {
      for (int v : h.sdom) g.pred[c].push_back(m_cmd_of_qubit[v]);
      for (int v : h.tdom) g.pred[c].push_back(m_cmd_of_qubit[v]);
    }
    if (h.kind == H_M) m_cmd_of_qubit[h.q0] = c;
    auto& P = g.pred[c];
    std::sort(P.begin(), P.end());
    P.erase(std::unique(P.begin(), P.end()), P.end());
  }
  return g;
}

struct ProaRun {
  Plan plan;
};

Plan proa_once(const HostPattern& hp, const Dag& g, bool eowqs, double A, double B, double G, double D) {
  const int nc = (int)hp.cmds.size();
  const int K = hp.n_measure;
  const int words = (K + 63) / 64;
  // M-ancestor bitsets (given order is a topological order)
  std::vector<uint64_t> anc((size_t)nc * std::max(words, 1), 0);
  for (int c = 0; c < nc; ++c) {
    if (!g.active[c]) continue;
    uint64_t* a = &anc[(size_t)c * words];
    for (int p : g.pred[c]) {
      const uint64_t* ap = &anc[(size_t)p * words];
      for (int w = 0; w < words; ++w) a[w] |= ap[w];
      int mo = hp.m_ord_of_cmd[p];
      if (mo >= 0) a[mo >> 6] |= 1ull << (mo & 63);
    }
  }
  std::vector<int> mcmd(K, -1);
  for (int c = 0; c < nc; ++c)
    if (hp.m_ord_of_cmd[c] >= 0) mcmd[hp.m_ord_of_cmd[c]] = c;
  std::vector<int> blocked(K, 0);
  std::vector<char> ready(K, 0), mdone(K, 0);
  for (int k = 0; k < K; ++k) {
    const uint64_t* a = &anc[(size_t)mcmd[k] * words];
    int cnt = 0;
    for (int w = 0; w < words; ++w) cnt += __builtin_popcountll(a[w]);
    blocked[k] = cnt;
    ready[k] = cnt == 0;
  }
  // incidence data for OS / flag / SS
  std::vector<std::vector<int>> e_of_qubit(hp.nq);
  std::vector<std::vector<int>> dependents(hp.nq);  // cmds whose domain contains the qubit
  for (int c = 0; c < nc; ++c) {
    if (!g.active[c]) continue;
    const HCmd& h = hp.cmds[c];
    if (h.kind == H_E) {
      e_of_qubit[h.q0].push_back(c);
      e_of_qubit[h.q1].push_back(c);
    }
    if (!eowqs) {
      for (int v : h.sdom) dependents[v].push_back(c);
      for (int v : h.tdom) dependents[v].push_back(c);
    }
  }
  std::vector<char> done(nc, 0), measured(hp.nq, 0);
  std::vector<int> visit_mark(nc, -1);
  int live = (int)hp.inputs.size();
  Plan plan;
  plan.paper_m = live;
  std::vector<int> stack, closure;
  auto collect = [&](int root, int tag) {
    closure.clear();
    stack.clear();
    stack.push_back(root);
    visit_mark[root] = tag;
    while (!stack.empty()) {
      int c = stack.back();
      stack.pop_back();
      closure.push_back(c);
      for (int p : g.pred[c])
        if (!done[p] && visit_mark[p] != tag) {
          visit_mark[p] = tag;
          stack.push_back(p);
        }
    }
  };
  int tag = 0;
  for (int step = 0; step < K; ++step) {
    int best = -1;
    double best_cost = 0;
    int best_ms = 0;
    for (int k = 0; k < K; ++k) {
      if (!ready[k] || mdone[k]) continue;
      collect(mcmd[k], ++tag);
      int n_new = 0;
      for (int c : closure)
        if (hp.cmds[c].kind == H_N) ++n_new;
      int v = hp.cmds[mcmd[k]].q0;
      int ms = live + n_new;  // MS(v): width of the state that measuring v creates
      int os = 0, flag = 0;
      for (int e : e_of_qubit[v]) {
        int w = hp.cmds[e].q0 == v ? hp.cmds[e].q1 : hp.cmds[e].q0;
        if (!done[e] && hp.is_output[w]) ++os;
        if (measured[w]) flag = 1;
      }
      std::unordered_set<int> ss;
      for (int c : dependents[v])
        if (!done[c]) ss.insert(hp.cmds[c].q0);
      double cost = flag ? A * ms + B * os - G * (double)ss.size()
                         : A * ((ms + 1) * D) + B * os - G * (double)ss.size();
      bool better = best < 0 || cost < best_cost - 1e-12 ||
                    (std::fabs(cost - best_cost) <= 1e-12 && hp.ext_id[v] < hp.ext_id[hp.cmds[mcmd[best]].q0]);
      if (better) {
        best = k;
        best_cost = cost;
        best_ms = ms;
      }
    }
    // execute the closure of the chosen M in given order, then the M
    collect(mcmd[best], ++tag);
    std::sort(closure.begin(), closure.end());
    for (int c : closure) {
      done[c] = 1;
      plan.order.push_back(c);
      if (hp.cmds[c].kind == H_N) ++live;
    }
    plan.paper_m = std::max(plan.paper_m, best_ms);
    plan.ms.push_back(best_ms);
    plan.m_cmds.push_back(mcmd[best]);
    measured[hp.cmds[mcmd[best]].q0] = 1;
    --live;
    mdone[best] = 1;
    for (int k = 0; k < K; ++k) {
      if (mdone[k] || ready[k]) continue;
      const uint64_t* a = &anc[(size_t)mcmd[k] * words];
      if (a[best >> 6] & (1ull << (best & 63))) {
        if (--blocked[k] == 0) ready[k] = 1;
      }
    }
  }
  for (int c = 0; c < nc; ++c)
    if (g.active[c] && !done[c]) {
      done[c] = 1;
      plan.order.push_back(c);
      if (hp.cmds[c].kind == H_N) ++live;
      plan.paper_m = std::max(plan.paper_m, live);
    }
  return plan;
}

}  // namespace

Plan make_plan(const HostPattern& hp, bool eowqs, bool given_order, const ProaWeights& w) {
  Dag g = build_dag(hp, eowqs);
  if (given_order) {
    Plan p;
    int live = (int)hp.inputs.size();
    p.paper_m = live;
    for (size_t c = 0; c < hp.cmds.size(); ++c) {
      if (!g.active[c]) continue;
      p.order.push_back((int)c);
      if (hp.cmds[c].kind == H_N) p.paper_m = std::max(p.paper_m, ++live);
      if (hp.cmds[c].kind == H_M) {
        p.m_cmds.push_back((int)c);
        p.ms.push_back(live);
        --live;
      }
    }
    return p;
  }
  const double O = (double)hp.outputs.size();
  double A0 = w.a >= 0 ? w.a : O, B0 = w.b >= 0 ? w.b : O, G0 = w.g, D0 = w.d >= 0 ? w.d : O;
  if (A0 <= 0) A0 = 1;
  if (D0 <= 0) D0 = 1;
  int iters = w.tune ? std::max(1, (int)O) : 1;
  Plan best;
  bool have = false;
  for (int it = 0; it < iters; ++it) {  // L487: alpha decreased by one |O| times, keep the best
    double A = A0 - it;
    if (A <= 0) break;
    Plan p = proa_once(hp, g, eowqs, A, B0, G0, D0);
    if (!have || p.paper_m < best.paper_m) {
      best = std::move(p);
      have = true;
    }
  }
  return best;
}

// ------------------------------------------------------------------------------------------------
// Compiler: plan -> logical op stream with slot reuse -> device steps.
// ------------------------------------------------------------------------------------------------
namespace {

struct LOp {
  int type;  // 1 DIAG_E, 2 DIAG_Z, 3 X, 4 BFLY, 10 GROW, 11 SHRINK
  int a = -1, b = -1, m = -1;
  std::vector<int> sig;  // given-order ordinals
};

struct Emitter {
  const HostPattern& hp;
  bool eowqs;
  std::vector<int> qs;        // 0 unprepared, 1 fresh (N done, not in the array), 2 live, 3 measured
  std::vector<int> slot_of;
  std::vector<int> qubit_at;  // slot -> qubit
  std::vector<std::vector<int>> pend;   // fresh q -> qubits with a pending E to q
  std::vector<std::vector<int>> pnb;    // any q -> fresh qubits that have a pending E to q
  std::vector<std::vector<std::vector<int>>> pendZ;  // fresh q -> pending Z signals
  int width = 0, max_width = 0;
  std::vector<LOp> ops;
  std::vector<MStatic> mst;
  std::vector<int32_t> pool;

  Emitter(const HostPattern& h, bool e) : hp(h), eowqs(e) {
    qs.assign(hp.nq, 0);
    slot_of.assign(hp.nq, -1);
    pend.assign(hp.nq, {});
    pnb.assign(hp.nq, {});
    pendZ.assign(hp.nq, {});
    for (size_t k = 0; k < hp.inputs.size(); ++k) {
      int q = hp.inputs[k];
      qs[q] = 2;
      slot_of[q] = (int)k;
      qubit_at.push_back(q);
    }
    width = max_width = (int)hp.inputs.size();
  }
  std::vector<int> sig_of(const std::vector<int>& dom) const {
    std::vector<int> s;
    for (int v : dom) s.push_back(hp.m_ord_of_qubit[v]);
    return s;
  }
  void diag_e(int u, int v) {
    LOp o;
    o.type = 1;
    o.a = slot_of[u];
    o.b = slot_of[v];
    ops.push_back(o);
  }
  void diag_z(int q, const std::vector<int>& sig) {
    LOp o;
    o.type = 2;
    o.a = slot_of[q];
    o.sig = sig;
    ops.push_back(o);
  }
  // apply a fresh qubit's deferred E's (to live qubits) and Z's after it got a slot
  void flush_pending(int q, int skip) {
    for (int w : pend[q]) {
      if (w == skip) continue;
      if (qs[w] == 2) diag_e(q, w);
      // a fresh w keeps the edge in pend[w]
    }
    pend[q].clear();
    for (auto& s : pendZ[q]) diag_z(q, s);
    pendZ[q].clear();
  }
  void materialize(int q) {  // N made real: append |+> at the top slot (GROW)
    LOp o;
    o.type = 10;
    o.a = width;
    ops.push_back(o);
    slot_of[q] = width;
    qubit_at.push_back(q);
    ++width;
    max_width = std::max(max_width, width);
    qs[q] = 2;
    flush_pending(q, -1);
  }
  std::vector<int> fresh_neighbours(int v) {
    std::vector<int> f;
    for (int u : pnb[v])
      if (qs[u] == 1 && std::find(pend[u].begin(), pend[u].end(), v) != pend[u].end() &&
          std::find(f.begin(), f.end(), u) == f.end())
        f.push_back(u);
    return f;
  }
  void add_pending_edge(int u, int v) {  // at least one of u, v is fresh
    if (qs[u] == 1) {
      pend[u].push_back(v);
      pnb[v].push_back(u);
    }
    if (qs[v] == 1) {
      pend[v].push_back(u);
      pnb[u].push_back(v);
    }
  }
  void measure(int v, const HCmd& h) {
    if (qs[v] == 1) materialize(v);
    std::vector<int> F = fresh_neighbours(v);
    MStatic ms{};
    ms.alpha = h.angle;
    ms.ord = hp.m_ord_of_qubit[v];
    ms.key = hp.draw_key.empty() ? ms.ord : hp.draw_key[ms.ord];
    std::vector<int> s = eowqs ? std::vector<int>() : sig_of(h.sdom);
    std::vector<int> t = eowqs ? std::vector<int>() : sig_of(h.tdom);
    ms.s_off = (int)pool.size();
    ms.s_len = (int)s.size();
    pool.insert(pool.end(), s.begin(), s.end());
    ms.t_off = (int)pool.size();
    ms.t_len = (int)t.size();
    pool.insert(pool.end(), t.begin(), t.end());
    int m = (int)mst.size();
    int b = slot_of[v];
    if (!F.empty()) {
      int o = F[0];
      for (size_t i = 1; i < F.size(); ++i) materialize(F[i]);
      ms.reuse = 1;
      ms.structural = 1;
      mst.push_back(ms);
      LOp op;
      op.type = 4;
      op.a = b;
      op.m = m;
      ops.push_back(op);
      qs[v] = 3;
      slot_of[v] = -1;
      qs[o] = 2;
      slot_of[o] = b;
      qubit_at[b] = o;
      flush_pending(o, v);
    } else {
      ms.reuse = 0;
      ms.structural = 0;
      mst.push_back(ms);
      LOp op;
      op.type = 11;
      op.a = b;
      op.m = m;
      ops.push_back(op);
      int top = width - 1;
      int tq = qubit_at[top];
      qubit_at[b] = tq;
      slot_of[tq] = b;
      qubit_at.pop_back();
      --width;
      qs[v] = 3;
      slot_of[v] = -1;
    }
  }
  void run(const Plan& plan) {
    for (int c : plan.order) {
      const HCmd& h = hp.cmds[c];
      switch (h.kind) {
        case H_N:
          qs[h.q0] = 1;
          break;
        case H_E:
          if (qs[h.q0] == 2 && qs[h.q1] == 2)
            diag_e(h.q0, h.q1);
          else
            add_pending_edge(h.q0, h.q1);
          break;
        case H_Z: {
          if (eowqs || h.sdom.empty()) break;
          auto s = sig_of(h.sdom);
          if (qs[h.q0] == 2)
            diag_z(h.q0, s);
          else
            pendZ[h.q0].push_back(s);
          break;
        }
        case H_X: {
          if (eowqs || h.sdom.empty()) break;
          auto s = sig_of(h.sdom);
          int q = h.q0;
          if (qs[q] == 1) {
            if (pend[q].empty() && pendZ[q].empty()) break;  // X|+> = |+>
            materialize(q);
          }
          // X_q E_uq = E_uq X_q Z_u: deferred E's with fresh u pick up a conditional Z_u
          for (int u : fresh_neighbours(q)) pendZ[u].push_back(s);
          LOp o;
          o.type = 3;
          o.a = slot_of[q];
          o.sig = s;
          ops.push_back(o);
          break;
        }
        case H_M:
          measure(h.q0, h);
          break;
      }
    }
    for (int o : hp.outputs)
      if (qs[o] == 1) materialize(o);
  }
};

}  // namespace

double Program::bytes_per_run(int eb) const {
  double b = 0;
  for (const auto& s : steps) {
    double S = std::ldexp((double)eb, s.width);
    if (s.kind == ST_PASS)
      b += s.n_ops > 0 ? 2 * S : S;
    else if (s.kind == ST_GROW)
      b += 3 * S;
    else if (s.kind == ST_SWAP)
      b += 2 * S;  // pack (read S/2, write S/2) + unpack (read S/2, write S/2)
    else if (s.kind == ST_RHOK)
      b += S;  // read-only
    else if (s.kind == ST_SHRINKK)
      b += S + 3 * std::ldexp(S, -s.jk);  // read S, write S / 2^k to scratch, copy back
    else
      b += 1.5 * S;
  }
  return b;
}

// Fusion-aware packing of the slot-level op stream into device steps.
//  * dependencies: on each slot, butterflies / X serialize with everything; diagonals (E, Z)
//    commute with each other; a decision waits for the ops that decide its signal domain;
//    GROW / SHRINK are barriers (they change the width and the slot map);
//  * X_a^s directly after the butterfly on slot a is folded into that butterfly (row swap);
//  * list scheduling: a pass owns the warp-segment slots (< SB) plus <= KMAX_HI group slots;
//    it greedily takes every ready op that fits, preferring ops on slots it already owns.
namespace {

struct Packer {
  const std::vector<LOp>& ops;
  std::vector<MStatic>& mst;
  Program& pr;
  const int SB;
  const bool eowqs;
  int max_bfly;
  int width;
  int kmax_hi = KMAX_AOT;       // group slots per pass (ahead-of-time / direct kernels)
  int kwide = KMAX_AOT;         // group slots per pass of width >= 13 run by the tile engine
  // butterflies per pass on warp-lane slots (cross-lane shuffles, ~4x the cost of a butterfly on a
  // register slot): capped for HBM-resident states so that no pass turns instruction-bound; the
  // deferred lane work lands in passes with idle issue slots (L2-resident states are launch-bound:
  // no cap, fewest passes)
  int max_lane_bfly = -1;
  bool measured_norm = false;  // OWQS_FLAG_MEASURED_NORM: structural decisions from a reduced ||psi||^2
  const int n_global;         // log2(ranks); positions >= width - n_global are rank bits
  std::vector<int> pos, at;   // virtual slot -> physical position, and back

  Packer(const std::vector<LOp>& o, Program& p, int sb, bool e, int mb, int ng)
      : ops(o), mst(p.mst), pr(p), SB(sb), eowqs(e), max_bfly(mb), width(p.in_width), n_global(ng) {
    if (const char* env = getenv("OWQS_KMAX_HI")) kmax_hi = std::max(0, std::min(KMAX_AOT, atoi(env)));
    if (const char* env = getenv("OWQS_MAX_LANE_BFLY")) max_lane_bfly = std::max(1, atoi(env));
    for (int v = 0; v < 64; ++v) {
      pos.push_back(v);
      at.push_back(v);
    }
  }
  int wl() const { return width - n_global; }
  // Qubit remapping (tile engine only, programs without GROW / SHRINK): the 6 segment slots are in
  // every pass's tile for free, so they should hold qubits that still have work. At the store of a
  // pass, a segment slot whose qubit has no remaining 2x2 op is traded for one of the pass's group
  // slots whose qubit has (the soonest-needed first): the next passes see up to 13 active qubits.
  bool remap = false;
  int remap_margin = 0;  // stream-order distance a swap must gain
  template <typename Nodes>
  void plan_remap(StepDesc& cur, const Nodes& nodes) {
    if (cur.n_ops == 0) return;  // a read-only pass has no store
    std::vector<int> next_use(64, 1 << 30);
    for (const auto& nd : nodes)
      if (!nd.done) {
        const LOp& l = ops[nd.op];
        if (l.type == 3 || l.type == 4) next_use[l.a] = std::min(next_use[l.a], nd.op);
      }
    // coldest segment slots (latest next 2x2 op, none = never) against the hottest group slots
    std::vector<int> seg, grp;
    for (int p = (SB == 6 ? 1 : 0); p < SB; ++p) seg.push_back(p);  // complex64 keeps slot 0 (float4 pairs)
    for (int j = 0; j < cur.nb_hi; ++j)
      if (next_use[at[cur.bhi[j]]] < (1 << 30)) grp.push_back(cur.bhi[j]);
    std::sort(seg.begin(), seg.end(), [&](int x, int y) { return next_use[at[x]] > next_use[at[y]]; });
    std::sort(grp.begin(), grp.end(), [&](int x, int y) { return next_use[at[x]] < next_use[at[y]]; });
    std::vector<int> dead, live;
    for (size_t k = 0; k < seg.size() && k < grp.size(); ++k) {
      if (next_use[at[seg[k]]] <= next_use[at[grp[k]]] + remap_margin) break;
      dead.push_back(seg[k]);
      live.push_back(grp[k]);
    }
    cur.n_remap = 0;
    for (size_t k = 0; k < dead.size() && k < live.size() && k < 6; ++k) {
      const int a = live[k], b = dead[k];
      cur.remap_a[cur.n_remap] = a;
      cur.remap_b[cur.n_remap] = b;
      ++cur.n_remap;
      const int va = at[a], vb = at[b];
      std::swap(pos[va], pos[vb]);
      at[pos[va]] = va;
      at[pos[vb]] = vb;
    }
  }

  // End of a pass with tile planning: choose the next pass's tile (plan_tile, limited to kmax qubits
  // outside this pass's tile), then remap -- segment positions whose qubit is not in the next tile
  // take next-tile qubits from this pass's group positions -- and return the next pass's group
  // positions (after the remap).
  template <typename PlanTile>
  void plan_next(StepDesc& cur, std::vector<char>& in_t, PlanTile& plan_tile, std::vector<int>& planned) {
    const int WL = wl();
    std::vector<char> prev(64, 0);
    for (int p = 0; p < SB && p < WL; ++p) prev[at[p]] = 1;
    for (int j = 0; j < cur.nb_hi; ++j) prev[at[cur.bhi[j]]] = 1;
    std::fill(in_t.begin(), in_t.end(), 0);
    const int p0 = SB == 6 ? 1 : 0;  // complex64 keeps slot 0 (float4 pairs): its qubit stays
    if (p0 == 1) in_t[at[0]] = 1;
    plan_tile(&prev);
    cur.n_remap = 0;
    if (cur.n_ops > 0) {  // a read-only pass has no store to remap
      std::vector<int> dead, live;
      for (int p = p0; p < SB && p < WL; ++p)
        if (!in_t[at[p]]) dead.push_back(p);
      for (int j = 0; j < cur.nb_hi; ++j)
        if (in_t[at[cur.bhi[j]]]) live.push_back(cur.bhi[j]);
      for (size_t k = 0; k < dead.size() && k < live.size() && k < 6; ++k) {
        const int a = live[k], b = dead[k];
        cur.remap_a[cur.n_remap] = a;
        cur.remap_b[cur.n_remap] = b;
        ++cur.n_remap;
        const int va = at[a], vb = at[b];
        std::swap(pos[va], pos[vb]);
        at[pos[va]] = va;
        at[pos[vb]] = vb;
      }
    }
    planned.clear();
    for (int p = SB; p < WL; ++p)
      if (in_t[at[p]]) planned.push_back(p);
  }

  // group slots allowed in a pass of (shard) width w
  int wide_at(int w) const { return (kwide > KMAX_AOT && w >= SB + kwide) ? kwide : kmax_hi; }
  // last step that computes something (a SWAP only permutes: it preserves the norm)
  StepDesc* last_compute() {
    for (int i = (int)pr.steps.size() - 1; i >= 0; --i)
      if (pr.steps[i].kind != ST_SWAP) return &pr.steps[i];
    return nullptr;
  }

  void emit(const StepDesc& s) {
    pr.steps.push_back(s);
    if (s.kind == ST_PASS) ++pr.n_passes;
    if (s.kind == ST_GROW) ++pr.n_grow;
    if (s.kind == ST_SHRINK) ++pr.n_shrink;
  }
  StepDesc blank(int kind) const {
    StepDesc d{};
    d.kind = kind;
    d.width = width - n_global;  // the shard's width
    d.red_slot = -1;
    d.slot = -1;
    d.shrink_m = -1;
    return d;
  }
  // the state produced by the last emitted step must carry its norm (first butterfly of a pass)
  // false: nothing computed yet -- the state is the caller's normalised input (set_input requires
  // ||psi||^2 = 1, the oracle checks it to 1e-9), so the first decision uses norm 1 and no
  // read-only norm pass is spent on it
  bool need_norm_before() {
    StepDesc* last = last_compute();
    if (!last) return false;
    if (last->red_kind == RED_NORM) return true;
    if (last->red_kind == RED_NONE) {
      last->red_kind = RED_NORM;
      return true;
    }
    StepDesc r = blank(ST_PASS);
    r.red_kind = RED_NORM;
    emit(r);
    return true;
  }
  void push_sig(Op& o, const std::vector<int>& sig) {
    o.cond = sig.empty() ? 0 : 1;
    o.sig_off = (int32_t)pr.sig_pool.size();
    o.sig_len = (int32_t)sig.size();
    pr.sig_pool.insert(pr.sig_pool.end(), sig.begin(), sig.end());
  }

  // Diagonal ops only XOR a sign mask in the kernel; a FLUSH applies it. A diagonal commutes with
  // a 2x2 on a slot it does not touch. An unconditional E(o, s) pending when the first butterfly
  // on s (or o) arrives is absorbed into that butterfly: U_s Z_s^{x_o} = butterfly with
  // coefficient (-1)^{x_o} a (absorb mask). Other pending diagonals touching the slot of a 2x2
  // are applied by a FLUSH placed right before it; leftovers are flushed at the end of the pass.
  void absorb_and_flush(StepDesc& cur) {
    Op out[MAX_OPS + MAX_OPS];
    uint64_t absorb[MAX_BFLY] = {0};
    int n = 0, bi = 0;
    struct Pend { int idx; int a, b; bool e; bool alive; };
    std::vector<Pend> pend;
    auto touches = [](const Pend& p, int s) { return p.a == s || p.b == s; };
    auto flush = [&]() {
      bool any = false;
      for (auto& p : pend) any |= p.alive;
      if (any) {
        Op f{};
        f.type = OP_FLUSH;
        out[n++] = f;
      }
      pend.clear();
    };
    for (int i = 0; i < cur.n_ops; ++i) {
      const Op& o = cur.ops[i];
      if (o.type == OP_DIAG_E || o.type == OP_DIAG_Z) {
        Pend p{n, o.a, o.type == OP_DIAG_E ? o.b : o.a, o.type == OP_DIAG_E && !o.cond, true};
        pend.push_back(p);
        out[n++] = o;
        continue;
      }
      const int s = o.a;
      bool conflict = false;  // a pending diagonal on s that cannot be absorbed
      for (auto& p : pend)
        if (p.alive && touches(p, s) && !(o.type == OP_BFLY && p.e)) conflict = true;
      if (conflict) {
        flush();
      } else if (o.type == OP_BFLY) {
        for (auto& p : pend)
          if (p.alive && touches(p, s)) {
            const int other = p.a == s ? p.b : p.a;
            absorb[bi] ^= 1ull << other;
            p.alive = false;
            out[p.idx].type = OP_NONE;  // removed below
          }
      }
      if (o.type == OP_BFLY) ++bi;
      out[n++] = o;
    }
    flush();
    int m = 0;
    for (int i = 0; i < n; ++i)
      if (out[i].type != OP_NONE) cur.ops[m++] = out[i];
    if (m > MAX_OPS_HARD) {
      fprintf(stderr, "owqs: internal op overflow\n");
      abort();
    }
    cur.n_ops = m;
    for (int k = 0; k < MAX_BFLY; ++k) cur.absorb[k] = absorb[k];
  }

  // schedule ops[lo, hi) (no barriers inside) into passes
  void segment(int lo, int hi) {
    // node list: X ops may be folded into a butterfly
    struct Node {
      int op;                   // index into ops
      std::vector<int> xsig;    // folded X signal (BFLY only)
      bool folded_x = false;
      std::vector<int> preds;
      int npred = 0;
      std::vector<int> succ;
      bool done = false;
      int lev = 0;  // butterflies / X on the longest dependency path to this node
    };
    std::vector<Node> nodes;
    std::vector<int> last_write(64, -1);
    std::vector<std::vector<int>> diags(64);
    std::unordered_map<int, int> decider;  // given-order ordinal -> node deciding it
    for (int i = lo; i < hi; ++i) {
      const LOp& l = ops[i];
      if (l.type == 3 && last_write[l.a] >= 0 && diags[l.a].empty()) {
        Node& w = nodes[last_write[l.a]];
        const LOp& wl = ops[w.op];
        bool ok = wl.type == 4 && !w.folded_x;
        if (ok)
          for (int o : l.sig) {
            auto it = decider.find(o);
            if (it != decider.end() && it->second > last_write[l.a]) ok = false;
          }
        if (ok) {
          w.folded_x = true;
          w.xsig = l.sig;
          for (int o : l.sig) {
            auto it = decider.find(o);
            if (it != decider.end() && it->second != last_write[l.a]) w.preds.push_back(it->second);
          }
          continue;
        }
      }
      Node n;
      n.op = i;
      const int id = (int)nodes.size();
      auto sigdeps = [&](const std::vector<int>& sig) {
        for (int o : sig) {
          auto it = decider.find(o);
          if (it != decider.end()) n.preds.push_back(it->second);
        }
      };
      if (l.type == 1 || l.type == 2) {
        const int b = l.type == 1 ? l.b : l.a;
        if (last_write[l.a] >= 0) n.preds.push_back(last_write[l.a]);
        if (last_write[b] >= 0) n.preds.push_back(last_write[b]);
        sigdeps(l.sig);
        diags[l.a].push_back(id);
        if (b != l.a) diags[b].push_back(id);
      } else {  // X or BFLY on slot a
        if (last_write[l.a] >= 0) n.preds.push_back(last_write[l.a]);
        for (int d : diags[l.a]) n.preds.push_back(d);
        diags[l.a].clear();
        last_write[l.a] = id;
        if (l.type == 3) sigdeps(l.sig);
        if (l.type == 4) {
          const MStatic& m = mst[l.m];
          for (int k = 0; k < m.s_len; ++k) {
            auto it = decider.find(pr.sig_pool[m.s_off + k]);
            if (it != decider.end()) n.preds.push_back(it->second);
          }
          for (int k = 0; k < m.t_len; ++k) {
            auto it = decider.find(pr.sig_pool[m.t_off + k]);
            if (it != decider.end()) n.preds.push_back(it->second);
          }
          decider[m.ord] = id;
        }
      }
      nodes.push_back(std::move(n));
    }
    const int N = (int)nodes.size();
    for (int i = 0; i < N; ++i) {
      auto& P = nodes[i].preds;
      std::sort(P.begin(), P.end());
      P.erase(std::unique(P.begin(), P.end()), P.end());
      nodes[i].npred = (int)P.size();
      for (int p : P) {
        nodes[p].succ.push_back(i);
        const int t = ops[nodes[p].op].type;
        nodes[i].lev = std::max(nodes[i].lev, nodes[p].lev + ((t == 3 || t == 4) ? 1 : 0));
      }
    }
    // Pick order inside a pass: dependency level first (a wavefront: fronts stay flat, so later
    // passes keep finding deep light cones), then stream order. Stream order alone (OWQS_LEVEL_PRIO=0)
    // follows PROA's measurement sweep, which on C3 builds a slope-1 staircase across all wires
    // that every later pass can only shift by two layers.
    static const bool level_prio = !(getenv("OWQS_LEVEL_PRIO") && atoi(getenv("OWQS_LEVEL_PRIO")) == 0);
    auto before = [&](int a, int b) {
      if (level_prio && nodes[a].lev != nodes[b].lev) return nodes[a].lev < nodes[b].lev;
      return nodes[a].op < nodes[b].op;
    };
    std::vector<int> ready;
    for (int i = 0; i < N; ++i)
      if (nodes[i].npred == 0) ready.push_back(i);
    int remaining = N;
    auto is_lane = [&](int a) { return a < SB && !(SB == 6 && a == 0); };
    // tile engine (width >= SB + 7): up to kwide group slots; lane slots reach registers
    // through shared-memory transposes, so no lane cap
    const bool wide = wide_at(wl()) > KMAX_AOT;
    const int kmax = wide_at(wl());
    const int lane_cap = max_lane_bfly > 0 ? max_lane_bfly : (!wide && wl() + (SB == 6 ? 3 : 4) >= 28 ? 4 : 64);
    // Tile planning (tile-engine passes; OWQS_SLOT_PICK=0: first-come slots + stream-order remap).
    // A pass's tile is the SB segment positions plus kmax group positions. The planner grows the
    // NEXT pass's tile qubit by qubit, each time adding the qubit that lets that pass run the most
    // butterflies (a dry run of the list scheduler restricted to the candidate tile; ties: the qubit
    // whose next 2x2 is earliest in the wavefront). It runs at the end of a pass, where the store's
    // remap can still move up to kmax of this pass's tile qubits into the segment, so the next tile
    // may hold at most kmax qubits from outside this pass's tile. First-come group slots plus a
    // stream-order remap made C3 a slope-1 staircase front (17 of 38 passes with 12-25 butterflies).
    static const bool slot_pick = !(getenv("OWQS_SLOT_PICK") && atoi(getenv("OWQS_SLOT_PICK")) == 0);
    std::vector<int> touched;
    std::vector<char> in_t(64, 0);  // dry-run tile, by virtual slot
    auto dry_run = [&](int* n_ops_out) {
      std::vector<int> rdy = ready;
      int n_ops = 0, n_bfly = 0;
      const int WL = wl();
      touched.clear();
      while (2 * n_ops + 2 <= MAX_OPS) {
        int best = -1;
        for (int k = 0; k < (int)rdy.size(); ++k) {
          const Node& n = nodes[rdy[k]];
          const LOp& l = ops[n.op];
          if (l.type == 4 && n_bfly >= max_bfly) continue;
          const bool diag = l.type == 1 || l.type == 2;
          if (!diag && (pos[l.a] >= WL || !in_t[l.a])) continue;
          if (best < 0 || before(rdy[k], rdy[best])) best = k;
        }
        if (best < 0) break;
        const int id = rdy[best];
        rdy[best] = rdy.back();
        rdy.pop_back();
        ++n_ops;
        if (ops[nodes[id].op].type == 4) ++n_bfly;
        for (int s : nodes[id].succ) {
          touched.push_back(s);
          if (--nodes[s].npred == 0) rdy.push_back(s);
        }
      }
      for (int s : touched) ++nodes[s].npred;
      if (n_ops_out) *n_ops_out = n_ops;
      return n_bfly;
    };
    // grow the tile in_t (already holding `fixed`) to SB + kmax qubits; prev: the qubits the previous
    // pass held (nullptr: no limit), at most kmax of the result may lie outside it
    // greedy tile growth from the qubits already in in_t (the seed), limited by prev (see above)
    auto grow_tile = [&](const std::vector<char>* prev) {
      const int WL = wl();
      std::vector<int> next_node(64, -1);  // first not-done 2x2 node per virtual slot
      for (int i = 0; i < (int)nodes.size(); ++i)
        if (!nodes[i].done) {
          const LOp& l = ops[nodes[i].op];
          if ((l.type == 3 || l.type == 4) && next_node[l.a] < 0) next_node[l.a] = i;
        }
      int n_in = 0, n_out = 0;
      for (int v = 0; v < 64; ++v)
        if (in_t[v]) {
          ++n_in;
          if (prev && !(*prev)[v]) ++n_out;
        }
      while (n_in < SB + kmax) {
        int best = -1, best_b = -1, best_o = -1;
        for (int p = 0; p < WL; ++p) {
          const int v = at[p];
          if (in_t[v] || next_node[v] < 0) continue;
          const bool out = prev && !(*prev)[v];
          if (out && n_out >= kmax) continue;
          in_t[v] = 1;
          int o = 0;
          const int b = dry_run(&o);
          in_t[v] = 0;
          if (best >= 0 && (b < best_b || (b == best_b && o < best_o))) continue;
          if (best >= 0 && b == best_b && o == best_o && !before(next_node[v], next_node[best])) continue;
          best = v;
          best_b = b;
          best_o = o;
        }
        if (best < 0) break;
        in_t[best] = 1;
        ++n_in;
        if (prev && !(*prev)[best]) ++n_out;
      }
      return next_node;
    };
    // run the pass of tile in_t for real on the node state (npred / done / ready), with an undo log
    struct Undo {
      std::vector<int> dec, done, ready;
    };
    auto commit_run = [&](Undo& u) {
      std::vector<int> rdy = ready;
      int n_ops = 0, n_bfly = 0;
      const int WL = wl();
      while (2 * n_ops + 2 <= MAX_OPS) {
        int best = -1;
        for (int k = 0; k < (int)rdy.size(); ++k) {
          const LOp& l = ops[nodes[rdy[k]].op];
          if (l.type == 4 && n_bfly >= max_bfly) continue;
          const bool diag = l.type == 1 || l.type == 2;
          if (!diag && (pos[l.a] >= WL || !in_t[l.a])) continue;
          if (best < 0 || before(rdy[k], rdy[best])) best = k;
        }
        if (best < 0) break;
        const int id = rdy[best];
        rdy[best] = rdy.back();
        rdy.pop_back();
        ++n_ops;
        if (ops[nodes[id].op].type == 4) ++n_bfly;
        nodes[id].done = true;
        u.done.push_back(id);
        for (int s2 : nodes[id].succ) {
          u.dec.push_back(s2);
          if (--nodes[s2].npred == 0) rdy.push_back(s2);
        }
      }
      u.ready = ready;
      ready = rdy;
      return n_bfly;
    };
    auto undo_run = [&](Undo& u) {
      for (int s2 : u.dec) ++nodes[s2].npred;
      for (int id : u.done) nodes[id].done = false;
      ready = u.ready;
    };
    // Two-pass look-ahead (OWQS_ENDGAME=B: only once at most B butterflies are left; 0: off): the
    // greedy tile maximises its own pass and can leave the remaining work spread over more qubits
    // than later tiles hold (C3's last 26 butterflies took passes of 16, 8 and 2). Every qubit with
    // work seeds its own greedy tile, and the tile maximising this pass plus the greedy next pass
    // wins. C3 30 -> 28 passes, C3W 31 -> 30, C4 21; about 1 s of host time per program.
    static const int endgame_bfly = getenv("OWQS_ENDGAME") ? atoi(getenv("OWQS_ENDGAME")) : (1 << 30);
    auto plan_tile = [&](const std::vector<char>* prev) {
      const std::vector<char> seed = in_t;
      int left = 0;
      for (int i = 0; i < (int)nodes.size(); ++i)
        if (!nodes[i].done && ops[nodes[i].op].type == 4) ++left;
      if (left > endgame_bfly) {
        grow_tile(prev);
        return;
      }
      const int WL = wl();
      std::vector<char> best_t;
      int best_sum = -1, best_b1 = -1;
      std::vector<int> seeds = {-1};
      {
        in_t = seed;
        const std::vector<int> nn = grow_tile(nullptr);  // only for next_node
        for (int p = 0; p < WL; ++p)
          if (nn[at[p]] >= 0 && !seed[at[p]]) seeds.push_back(at[p]);
      }
      for (int sv : seeds) {
        in_t = seed;
        if (sv >= 0) {
          if (prev && !(*prev)[sv] && kmax < 1) continue;
          in_t[sv] = 1;
        }
        grow_tile(prev);
        const std::vector<char> t1 = in_t;
        Undo u;
        const int b1 = commit_run(u);
        in_t.assign(64, 0);
        if (SB == 6) in_t[at[0]] = 1;
        grow_tile(&t1);
        const int b2 = dry_run(nullptr);
        undo_run(u);
        if (b1 + b2 > best_sum || (b1 + b2 == best_sum && b1 > best_b1)) {
          best_sum = b1 + b2;
          best_b1 = b1;
          best_t = t1;
        }
      }
      in_t = best_t;
    };
    std::vector<int> planned;  // group positions chosen for the next pass (valid when have_plan)
    bool have_plan = false;
    while (remaining > 0) {
      StepDesc cur = blank(ST_PASS);
      int n_lane = 0;
      const int WL = wl();
      auto has_slot = [&](int a) {
        if (a < SB) return true;
        for (int j = 0; j < cur.nb_hi; ++j)
          if (cur.bhi[j] == a) return true;
        return false;
      };
      if (wide && slot_pick) {
        if (!have_plan) {  // first pass of a segment: the segment qubits are given
          std::fill(in_t.begin(), in_t.end(), 0);
          for (int p = 0; p < SB && p < WL; ++p) in_t[at[p]] = 1;
          plan_tile(nullptr);
          planned.clear();
          for (int p = SB; p < WL; ++p)
            if (in_t[at[p]]) planned.push_back(p);
        }
        have_plan = false;
        for (int p : planned)
          if ((int)cur.nb_hi < kmax) cur.bhi[cur.nb_hi++] = p;
        std::sort(cur.bhi, cur.bhi + cur.nb_hi);
      }
      while (true) {
        if (2 * cur.n_ops + 2 > MAX_OPS) break;  // room for the FLUSH ops inserted afterwards
        // pick: (1) fits without a new slot, lowest stream index; (2) needs a new slot
        int best = -1, best_new = -1;
        for (int k = 0; k < (int)ready.size(); ++k) {
          const Node& n = nodes[ready[k]];
          const LOp& l = ops[n.op];
          if (l.type == 4 && cur.n_bfly >= max_bfly) continue;
          if (l.type == 4 && is_lane(pos[l.a]) && n_lane >= lane_cap) continue;
          const bool diag = l.type == 1 || l.type == 2;
          if (!diag && pos[l.a] >= WL) continue;  // 2x2 on a rank bit: needs a SWAP first
          bool fits = diag || has_slot(pos[l.a]);
          if (fits) {
            if (best < 0 || before(ready[k], ready[best])) best = k;
          } else if (cur.nb_hi < kmax) {
            if (best_new < 0 || before(ready[k], ready[best_new])) best_new = k;
          }
        }
        int pick = best >= 0 ? best : best_new;
        if (pick < 0) break;
        const int id = ready[pick];
        ready[pick] = ready.back();
        ready.pop_back();
        Node& n = nodes[id];
        const LOp& l = ops[n.op];
        if ((l.type == 3 || l.type == 4) && !has_slot(pos[l.a])) {
          cur.bhi[cur.nb_hi++] = pos[l.a];
          std::sort(cur.bhi, cur.bhi + cur.nb_hi);
        }
        Op o{};
        o.type = (uint8_t)l.type;
        o.a = (uint8_t)pos[std::max(l.a, 0)];
        o.b = (uint8_t)pos[std::max(l.b, 0)];
        o.m = l.m;
        if (l.type == 4) {
          push_sig(o, n.xsig);  // cond/sig of a butterfly = folded X_a^s
          if (cur.n_bfly == 0 && !eowqs) cur.first_uses_red = 1;
          ++cur.n_bfly;
          if (is_lane(pos[l.a])) ++n_lane;
        } else {
          push_sig(o, l.sig);
        }
        cur.ops[cur.n_ops++] = o;
        n.done = true;
        --remaining;
        for (int s : n.succ)
          if (--nodes[s].npred == 0) ready.push_back(s);
      }
      if (cur.n_ops == 0) {
        // every ready op is a 2x2 on a rank bit: bring its qubit into the shard, evicting the
        // local qubit whose next 2x2 is farthest away (Belady); light-cone skew falls out of the
        // list scheduler advancing everything local first
        int g = -1, gop = 1 << 30;
        for (int id : ready) {
          const LOp& l = ops[nodes[id].op];
          if ((l.type == 3 || l.type == 4) && pos[l.a] >= WL && nodes[id].op < gop) {
            gop = nodes[id].op;
            g = l.a;
          }
        }
        if (g < 0) break;  // cannot happen
        std::vector<int> next_use(64, 1 << 30);
        for (const Node& nd : nodes)
          if (!nd.done) {
            const LOp& l = ops[nd.op];
            if (l.type == 3 || l.type == 4) next_use[l.a] = std::min(next_use[l.a], nd.op);
          }
        int victim = -1;
        for (int p = WL - 1; p >= 0; --p) {
          const int v = at[p];
          if (victim < 0 || next_use[v] > next_use[victim]) victim = v;
        }
        StepDesc sw = blank(ST_SWAP);
        sw.swap_local = pos[victim];
        sw.swap_global = pos[g];
        emit(sw);
        ++pr.n_swaps;
        std::swap(pos[victim], pos[g]);
        at[pos[victim]] = victim;
        at[pos[g]] = g;
        continue;
      }
      // a structural first decision of a pass uses ||psi||^2 = 1, its exact value, instead of a norm
      // reduced by the previous pass (reading R-13): the input is normalised (enforced by every
      // owqs_set_input_*), a structural measurement's p_s = 1/2 ||psi||^2 = 1/2 and a SHRINK's
      // measured p_s both renormalise by 1/sqrt(p_s) (Eq. 4), so ||psi||^2 = 1 holds by induction.
      // C3 43.1 -> 41.8 ms, C2 0.72 -> 0.62 ms. The output's norm is still reduced by the last pass.
      // OWQS_FLAG_MEASURED_NORM keeps the reduction (tests check the reading with it at full width).
      if (cur.first_uses_red && (!measured_norm || !need_norm_before())) cur.first_uses_red = 0;
      absorb_and_flush(cur);
      if (remap && wide && slot_pick && remaining > 0) {
        plan_next(cur, in_t, plan_tile, planned);
        have_plan = true;
      } else if (remap && wide) {
        plan_remap(cur, nodes);
      }
      emit(cur);
    }
  }

  // joint k-outcome measurement of consecutive eliminations: ST_RHOK +
  // ST_SHRINKK for ops[i .. i + k). The physical bookkeeping is that of k single SHRINKs in a row
  // (same final slot map); j_src records where each output bit comes from.
  int joint_k = JOINT_KMAX;  // OWQS_JOINT_K (1 = off)
  void joint_shrink(int i, int k) {
    StepDesc r = blank(ST_RHOK), s = blank(ST_SHRINKK);
    r.jk = s.jk = k;
    int orig[64];
    for (int b = 0; b < 64; ++b) orig[b] = b;
    const int w0 = width;
    for (int j = 0; j < k; ++j) {
      const LOp& l = ops[i + j];
      const int vm = l.a, pm = pos[vm];
      r.jm_pos[j] = s.jm_pos[j] = orig[pm];
      r.jm[j] = s.jm[j] = l.m;
      const int vt = width - 1, pt = width - 1, u = at[pt], q = pos[vt];
      if (vm == vt) {
        if (pm != pt) {
          pos[u] = pm;
          at[pm] = u;
        }
      } else if (q == pt) {
        pos[vm] = pm;
        at[pm] = vm;
      } else {
        pos[vm] = q;
        at[q] = vm;
        pos[u] = pm;
        at[pm] = u;
      }
      pos[vt] = vt;
      at[pt] = vt;
      orig[pm] = orig[pt];  // the physical top qubit moves into the freed position
      --width;
    }
    for (int t = 0; t < w0 - k; ++t) s.j_src[t] = (int8_t)orig[t];
    r.width = s.width = w0 - n_global;
    if (!eowqs) emit(r);
    emit(s);
    pr.n_shrink += k;
  }

  void run() {
    int lo = 0;
    const int n = (int)ops.size();
    for (int i = 0; i <= n; ++i) {
      if (i < n && ops[i].type != 10 && ops[i].type != 11) continue;
      segment(lo, i);
      lo = i + 1;
      if (i == n) break;
      if (ops[i].type == 11 && joint_k > 1) {
        int k = 1;
        while (k < joint_k && i + k < n && ops[i + k].type == 11) ++k;
        if (k > 1) {
          joint_shrink(i, k);
          i += k - 1;
          lo = i + 1;
          continue;
        }
      }
      const LOp& l = ops[i];
      // GROW / SHRINK act on physical positions; with qubit remapping the emitter's virtual slots
      // map through pos[] (the kernels' conventions: GROW appends at the physical top, SHRINK moves
      // the physical top qubit into the freed position)
      if (l.type == 10) {  // the emitter appends its virtual top slot l.a = width
        StepDesc g = blank(ST_GROW);
        g.slot = width;
        pos[l.a] = width;
        at[width] = l.a;
        emit(g);
        ++width;
      } else {
        const int vm = l.a, pm = pos[vm];
        if (!eowqs) {  // rho of the measured slot from the last pass (or a read-only pass)
          StepDesc* last = pr.steps.empty() ? nullptr : &pr.steps.back();
          // the last pass reduces in its input layout: undo its store remap for vm's position
          int pl = pm;
          if (last && last->kind == ST_PASS)
            for (int k = 0; k < last->n_remap; ++k) {
              if (pm == last->remap_a[k]) pl = last->remap_b[k];
              if (pm == last->remap_b[k]) pl = last->remap_a[k];
            }
          bool room = last && last->kind == ST_PASS && last->red_kind == RED_NONE && last->width == width &&
                      (pl < SB || last->nb_hi < wide_at(last->width) ||
                       std::find(last->bhi, last->bhi + last->nb_hi, pl) != last->bhi + last->nb_hi);
          if (room) {
            if (pl >= SB && std::find(last->bhi, last->bhi + last->nb_hi, pl) == last->bhi + last->nb_hi) {
              last->bhi[last->nb_hi++] = pl;
              std::sort(last->bhi, last->bhi + last->nb_hi);
            }
            last->red_kind = RED_RHO;
            last->red_slot = pl;
          } else {
            StepDesc r = blank(ST_PASS);
            if (pm >= SB) r.bhi[r.nb_hi++] = pm;
            r.red_kind = RED_RHO;
            r.red_slot = pm;
            emit(r);
          }
        }
        StepDesc s = blank(ST_SHRINK);
        s.slot = pm;
        s.shrink_m = l.m;
        s.first_uses_red = eowqs ? 0 : 1;
        s.first_full_rho = eowqs ? 0 : 1;
        emit(s);
        // the emitter renames its virtual top vt into vm; physically the top qubit u moves into pm
        const int vt = width - 1, pt = width - 1, u = at[pt], q = pos[vt];
        if (vm == vt) {
          if (pm != pt) {
            pos[u] = pm;
            at[pm] = u;
          }
        } else if (q == pt) {
          pos[vm] = pm;
          at[pm] = vm;
        } else {
          pos[vm] = q;
          at[q] = vm;
          pos[u] = pm;
          at[pm] = u;
        }
        pos[vt] = vt;
        at[pt] = vt;
        --width;
      }
    }
    // final norm of the output state (EOWQS determinism check / drift report)
    StepDesc* lc = last_compute();
    if (lc && lc->red_kind == RED_NONE)
      lc->red_kind = RED_NORM;
    else if (!lc || lc->red_kind != RED_NORM || pr.steps.back().kind == ST_SWAP) {
      StepDesc r = blank(ST_PASS);
      r.red_kind = RED_NORM;
      emit(r);
    }
    for (const auto& s : pr.steps)
      if (s.red_kind != RED_NONE) ++pr.n_reduce;
  }
};

}  // namespace

Program compile_program(const HostPattern& hp, const Plan& plan, int mode, int SB, bool fuse, int n_global,
                        int kwide, bool measured_norm) {
  const bool eowqs = mode == 2;
  Emitter em(hp, eowqs);
  em.run(plan);
  Program pr;
  pr.mst = em.mst;
  pr.sig_pool = em.pool;
  pr.phys_bits = em.max_width;
  pr.in_width = (int)hp.inputs.size();
  pr.n_global = n_global;
  if (n_global > 0) {
    for (const LOp& l : em.ops)
      if (l.type == 10 || l.type == 11) {
        pr.error = "multi-rank execution needs a constant-width program (no GROW / SHRINK)";
        return pr;
      }
    if (pr.in_width - n_global < 2) {
      pr.error = "state too narrow for " + std::to_string(1 << n_global) + " ranks";
      return pr;
    }
  }
  Packer pk(em.ops, pr, SB, eowqs, fuse ? MAX_BFLY : 1, n_global);
  pk.measured_norm = measured_norm;
  if (const char* e = getenv("OWQS_JOINT_K")) pk.joint_k = std::max(1, std::min(JOINT_KMAX, atoi(e)));
  pk.kwide = std::max(KMAX_AOT, std::min(KTILE, kwide));
  if (const char* env = getenv("OWQS_MAX_BFLY")) pk.max_bfly = std::max(1, std::min(MAX_BFLY, atoi(env)));
  {
    bool resize = false;
    for (const LOp& l : em.ops) resize = resize || l.type == 10 || l.type == 11;
    const char* env = getenv("OWQS_REMAP");
    // default on (OWQS_REMAP=0 turns it off): C3 51 -> 35 passes, 51.0 -> 49.8 ms
    // (sharded programs too: a remap permutes local positions only; rank bits and the swap plan
    // follow the same pos / at maps)
    pk.remap = (!env || atoi(env) != 0) && (!resize || !getenv("OWQS_REMAP_NO_RESIZE")) && pk.kwide > KMAX_AOT;
    if (const char* m = getenv("OWQS_REMAP_MARGIN")) pk.remap_margin = atoi(m);
  }
  if (const char* env = getenv("OWQS_KWIDE")) pk.kwide = std::max(KMAX_AOT, std::min(KTILE, atoi(env)));
  pk.run();
  for (int o : hp.outputs) pr.out_slot.push_back(pk.pos[em.slot_of[o]]);
  return pr;
}

void plan_and_compile(const HostPattern& hp, int mode, int SB, bool fuse, bool given, const ProaWeights& w,
                      Plan& plan, Program& prog, int n_global, int kwide, bool measured_norm) {
  if (mode != 2) {
    plan = make_plan(hp, false, given, w);
    prog = compile_program(hp, plan, mode, SB, fuse, n_global, kwide, measured_norm);
    return;
  }
  plan = make_plan(hp, true, given, w);
  prog = compile_program(hp, plan, 2, SB, fuse, n_global, kwide, measured_norm);
  Plan alt = make_plan(hp, false, given, w);
  Plan filt;
  for (int c : alt.order)
    if (hp.cmds[c].kind != H_X && hp.cmds[c].kind != H_Z) filt.order.push_back(c);
  filt.m_cmds = alt.m_cmds;
  filt.ms = alt.ms;
  filt.paper_m = alt.paper_m;
  Program ap = compile_program(hp, filt, 2, SB, fuse, n_global, kwide, measured_norm);
  if (!prog.error.empty() ||
      (ap.error.empty() && (ap.phys_bits < prog.phys_bits ||
                            (ap.phys_bits == prog.phys_bits && ap.n_passes + ap.n_swaps < prog.n_passes + prog.n_swaps)))) {
    plan = std::move(filt);
    prog = std::move(ap);
  }
}

// PAPER §4.1 (L155): "Initially, all of the qubit states are separate (except the input qubits
// which can be entangled) ... Two different sub-states are combined only when the entanglement
// operation is applied". The sub-states that are never combined are the connected components of
// the pattern's E graph, with all inputs in one. Each component becomes its own pattern over the
// same dense qubit ids and the same given-order M ordinals (so keyed outcome draws, forced strings
// and the outcome / prob0 arrays keep the caller's indexing); it is split only when no signal
// domain crosses components (execution order between sub-states is then free) and there are at
// most KRON_MAX components. Returns false when the pattern stays one state.
bool split_substates(const HostPattern& hp, std::vector<HostPattern>& parts, std::vector<uint64_t>& masks,
                     int max_parts) {
  const int nq = hp.nq;
  std::vector<int> par(nq);
  for (int q = 0; q < nq; ++q) par[q] = q;
  std::function<int(int)> find = [&](int x) { return par[x] == x ? x : par[x] = find(par[x]); };
  auto unite = [&](int a, int b) { par[find(a)] = find(b); };
  for (size_t i = 1; i < hp.inputs.size(); ++i) unite(hp.inputs[0], hp.inputs[i]);
  for (const HCmd& c : hp.cmds)
    if (c.kind == H_E) unite(c.q0, c.q1);
  for (const HCmd& c : hp.cmds) {
    for (int q : c.sdom)
      if (find(q) != find(c.q0)) return false;
    for (int q : c.tdom)
      if (find(q) != find(c.q0)) return false;
  }
  std::vector<int> roots;
  auto add = [&](int q) {
    const int r = find(q);
    if (std::find(roots.begin(), roots.end(), r) == roots.end()) roots.push_back(r);
  };
  if (!hp.inputs.empty()) add(hp.inputs[0]);
  for (const HCmd& c : hp.cmds) add(c.q0);
  for (int q : hp.outputs) add(q);
  if (roots.size() < 2 || roots.size() > (size_t)max_parts || hp.outputs.size() > 63) return false;
  parts.clear();
  masks.clear();
  for (int r : roots) {
    HostPattern p;
    p.nq = nq;
    p.ext_id = hp.ext_id;
    p.n_measure = 0;  // dense ordinals per sub-state; draw_key keeps the caller's for sampling
    p.m_ord_of_qubit.assign(nq, -1);
    p.is_output.assign(nq, 0);
    p.is_input.assign(nq, 0);
    if (!hp.inputs.empty() && find(hp.inputs[0]) == r)
      for (int q : hp.inputs) {
        p.inputs.push_back(q);
        p.is_input[q] = 1;
      }
    uint64_t mask = 0;
    for (size_t k = 0; k < hp.outputs.size(); ++k)
      if (find(hp.outputs[k]) == r) {
        p.outputs.push_back(hp.outputs[k]);
        p.is_output[hp.outputs[k]] = 1;
        mask |= 1ull << k;
      }
    for (size_t i = 0; i < hp.cmds.size(); ++i)
      if (find(hp.cmds[i].q0) == r) {
        p.cmds.push_back(hp.cmds[i]);
        int o = -1;
        if (hp.m_ord_of_cmd[i] >= 0) {
          o = p.n_measure++;
          p.m_ord_of_qubit[hp.cmds[i].q0] = o;
          p.draw_key.push_back(hp.m_ord_of_cmd[i]);
        }
        p.m_ord_of_cmd.push_back(o);
      }
    parts.push_back(std::move(p));
    masks.push_back(mask);
  }
  return true;
}

}  // namespace owqs
