// Standardisation of measurement patterns: a wild pattern (the given
// execution order, corrections anywhere) is rewritten into the standard form the paper's problem
// statement assumes ("takes a pattern in the standard form"): N* E* M* C*, all preparations
// first, then all entanglings, then the measurements in their given order, then the corrections of
// the outputs (measurement calculus [Danos-Kashefi-Panangaden]). One left-to-right sweep keeps,
// per qubit, the corrections not yet applied (X^a Z^b in execution order, a and b signal domains):
//   * E_ij moves left past the pending corrections: E X_i^a = X_i^a Z_j^a E (exact), so j's pending
//     Z gains a (and i's gains j's pending X domain); Z commutes with E;
//   * X_i^d after pending X^a Z^b: X^a Z^b X^d = (-1)^{|b||d|} X^{a+d} Z^b (a sign, recorded);
//     Z_i^d: X^a Z^{b+d} (exact);
//   * M_i^{alpha, s, t} absorbs the pending X^a Z^b: <+-phi| Z^b = <+-(phi + b pi)| (exact) and
//     <+-phi| X = +-e^{-i phi} <+-(-phi)| (outcome-dependent global phase), i.e. the new domains are
//     s + a and t + b, the angle of Eq. 2 becomes (-1)^{s+a} alpha + (t+b) pi;
//   * the outputs' remaining pending corrections become the final X then Z commands.
// The standardised pattern has the same outcome labels and the same branch probabilities; its
// output equals the wild pattern's up to a global phase per branch (reading R-18).
// Signal shifting (optional): a t-domain T of M_i is removed and T added (XOR) to every later domain
// that references i: measuring at theta + pi is measuring at theta with the outcome label flipped
// (<+(theta+pi)| = <-theta|, exact), so s_i(old) = s_i(new) + |T|. The removed T of every M is
// returned so callers can map outcome strings.
#include <algorithm>
#include <string>
#include <vector>

#include "scheduler.h"

namespace owqs {

namespace {
// symmetric difference of sorted sets
std::vector<int> sym(const std::vector<int>& a, const std::vector<int>& b) {
  std::vector<int> r;
  std::set_symmetric_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(r));
  return r;
}
std::vector<int> sorted(std::vector<int> v) {
  std::sort(v.begin(), v.end());
  // a domain is an XOR: a repeated qubit cancels
  std::vector<int> r;
  for (size_t i = 0; i < v.size();) {
    size_t j = i;
    while (j < v.size() && v[j] == v[i]) ++j;
    if ((j - i) & 1) r.push_back(v[i]);
    i = j;
  }
  return r;
}
}  // namespace

std::string standardize_pattern(const HostPattern& hp, bool signal_shift, std::vector<HCmd>& out,
                                std::vector<std::vector<int>>& shift, int* n_x_absorbed, int* n_signs) {
  out.clear();
  shift.clear();
  std::vector<std::vector<int>> px(hp.nq), pz(hp.nq);
  std::vector<HCmd> ns, es, ms, cs;
  int nabs = 0, nsg = 0;
  for (const HCmd& c : hp.cmds) {
    switch (c.kind) {
      case H_N:
        ns.push_back(c);
        break;
      case H_E: {
        const int i = c.q0, j = c.q1;
        const std::vector<int> xi = px[i], xj = px[j];
        pz[j] = sym(pz[j], xi);
        pz[i] = sym(pz[i], xj);
        es.push_back(c);
        break;
      }
      case H_X: {
        const std::vector<int> d = sorted(c.sdom);
        if (!pz[c.q0].empty() && !d.empty()) ++nsg;  // (-1)^{|b||d|}: a branch-dependent sign
        px[c.q0] = sym(px[c.q0], d);
        break;
      }
      case H_Z:
        pz[c.q0] = sym(pz[c.q0], sorted(c.sdom));
        break;
      case H_M: {
        HCmd m = c;
        if (!px[c.q0].empty()) ++nabs;
        m.sdom = sym(sorted(c.sdom), px[c.q0]);
        m.tdom = sym(sorted(c.tdom), pz[c.q0]);
        px[c.q0].clear();
        pz[c.q0].clear();
        ms.push_back(m);
        break;
      }
      default:
        return "unknown command kind";
    }
  }
  for (int o : hp.outputs) {
    if (!px[o].empty()) {
      HCmd x;
      x.kind = H_X;
      x.q0 = o;
      x.sdom = px[o];
      cs.push_back(x);
    }
    if (!pz[o].empty()) {
      HCmd z;
      z.kind = H_Z;
      z.q0 = o;
      z.sdom = pz[o];
      cs.push_back(z);
    }
  }
  if (signal_shift) {
    // forward sweep over measurements then corrections: s_i(old) = s_i(new) + |T_i|
    std::vector<std::vector<int>> T(hp.nq);
    auto subst = [&](std::vector<int> d) {
      std::vector<int> r = d;
      for (int q : d)
        if (!T[q].empty()) r = sym(r, T[q]);
      return r;
    };
    for (HCmd& m : ms) {
      m.sdom = subst(m.sdom);
      m.tdom = subst(m.tdom);
      T[m.q0] = m.tdom;
      m.tdom.clear();
    }
    for (HCmd& c : cs) c.sdom = subst(c.sdom);
    shift.assign(hp.nq, {});
    for (const HCmd& m : ms) shift[m.q0] = T[m.q0];
  }
  out.insert(out.end(), ns.begin(), ns.end());
  out.insert(out.end(), es.begin(), es.end());
  out.insert(out.end(), ms.begin(), ms.end());
  out.insert(out.end(), cs.begin(), cs.end());
  if (n_x_absorbed) *n_x_absorbed = nabs;
  if (n_signs) *n_signs = nsg;
  return "";
}

}  // namespace owqs
