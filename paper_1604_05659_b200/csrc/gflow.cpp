// gflow finder for the EOWQS pre-check ("in [25] an algorithm is presented for finding
// a gflow in the patterns in polynomial time. If a pattern has a gflow, the probability of
// measurement results is 0.5; otherwise, the pattern is reported as an incorrect one").
//
// Open graph (G, I, O): vertices = qubits, edges = the pattern's E commands; every measurement is
// in the XY plane. A gflow (g, <) needs, for each measured u: g(u) in V \ I, u in Odd(g(u)), and
// every w in g(u) or Odd(g(u)) \ {u} later than u (Browne et al. [13]). Backward layering
// (Mhalla-Perdrix [25]): with `Out` = outputs, repeatedly find the unprocessed u for which some
// K in Out \ I has Odd(K) restricted to the unprocessed vertices = {u}; those u form the next
// layer (g(u) = K) and join Out. A gflow exists iff every vertex gets a layer. Each layer is one
// GF(2) elimination of the adjacency block (unprocessed x candidates) with a tracked row basis.
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "scheduler.h"

namespace owqs {

namespace {
struct BitRow {
  std::vector<uint64_t> w;
  explicit BitRow(int n = 0) : w((n + 63) / 64, 0) {}
  bool get(int i) const { return (w[i >> 6] >> (i & 63)) & 1; }
  void set(int i) { w[i >> 6] |= 1ull << (i & 63); }
  void flip(int i) { w[i >> 6] ^= 1ull << (i & 63); }
  void xor_with(const BitRow& o) {
    for (size_t k = 0; k < w.size(); ++k) w[k] ^= o.w[k];
  }
  bool any() const {
    for (uint64_t x : w)
      if (x) return true;
    return false;
  }
};
}  // namespace

std::string find_gflow(const HostPattern& hp, std::vector<int>& layer, std::vector<std::vector<int>>& g) {
  const int n = hp.nq;
  std::vector<std::vector<int>> adj(n);
  for (const HCmd& c : hp.cmds)
    if (c.kind == H_E) {
      adj[c.q0].push_back(c.q1);
      adj[c.q1].push_back(c.q0);
    }
  layer.assign(n, -1);
  g.assign(n, {});
  std::vector<char> out(n, 0);
  for (int o : hp.outputs) {
    out[o] = 1;
    layer[o] = 0;
  }
  int k = 1;
  while (true) {
    std::vector<int> rows, cols;  // unprocessed vertices, candidates Out \ I
    for (int v = 0; v < n; ++v)
      if (!out[v]) rows.push_back(v);
      else if (!hp.is_input[v]) cols.push_back(v);
    if (rows.empty()) return "";
    const int m = (int)rows.size(), c = (int)cols.size();
    std::vector<int> row_of(n, -1);
    for (int i = 0; i < m; ++i) row_of[rows[i]] = i;
    // A[i][j] = 1 iff rows[i] ~ cols[j]; we need x with A x = e_u (restricted odd neighbourhood).
    // Eliminate on the columns-as-equations form: augment each row with its identity (row basis).
    std::vector<BitRow> A(m, BitRow(c)), R(m, BitRow(m));
    for (int j = 0; j < c; ++j)
      for (int v : adj[cols[j]])
        if (row_of[v] >= 0) A[row_of[v]].set(j);
    for (int i = 0; i < m; ++i) R[i].set(i);
    // Gaussian elimination on rows (row ops recorded in R): reduced row echelon form
    std::vector<int> pivot_col_of_row(m, -1);
    int r = 0;
    for (int j = 0; j < c && r < m; ++j) {
      int p = -1;
      for (int i = r; i < m; ++i)
        if (A[i].get(j)) {
          p = i;
          break;
        }
      if (p < 0) continue;
      std::swap(A[p], A[r]);
      std::swap(R[p], R[r]);
      for (int i = 0; i < m; ++i)
        if (i != r && A[i].get(j)) {
          A[i].xor_with(A[r]);
          R[i].xor_with(R[r]);
        }
      pivot_col_of_row[r] = j;
      ++r;
    }
    // rows r..m-1 of A are zero: their R rows span the left null space {y : y^T A = 0}.
    // e_u is in the column space iff y_u = 0 for every such y.
    std::vector<char> blocked(m, 0);
    for (int i = r; i < m; ++i)
      for (int u = 0; u < m; ++u)
        if (R[i].get(u)) blocked[u] = 1;
    std::vector<int> found;
    for (int u = 0; u < m; ++u) {
      if (blocked[u]) continue;
      // solution: x = sum over pivot rows i with (R[i] . e_u) = 1 of e_{pivot col}: since
      // R A = E (echelon), A x = e_u  <=>  E x = R e_u on the pivot rows.
      std::vector<int> K;
      for (int i = 0; i < r; ++i)
        if (R[i].get(u)) K.push_back(cols[pivot_col_of_row[i]]);
      g[rows[u]] = K;
      found.push_back(rows[u]);
    }
    if (found.empty()) return "no gflow: " + std::to_string(m) + " measured qubits cannot be layered";
    for (int v : found) {
      out[v] = 1;
      layer[v] = k;
    }
    ++k;
  }
}

}  // namespace owqs
