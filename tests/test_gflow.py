"""gflow pre-check of EOWQS (refs [13], [25]) vs a brute-force search from the
definition on small open graphs, plus the paper's patterns. No GPU needed."""
import itertools

import numpy as np
import pytest

from paper_1604_05659_b200.host import host_gflow
from workloads import patterns as W


def brute_force_gflow(n, edges, I, O):
    """Exists (g, <) with, for every measured i: g(i) in V \\ I, i not in g(i), i in Odd(g(i)), and
    i < j for every j in g(i) or in Odd(g(i)) \\ {i} (XY-plane gflow, Browne et al. [13])?"""
    adj = [set() for _ in range(n)]
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    meas = [v for v in range(n) if v not in O]
    cand = [v for v in range(n) if v not in I]

    def odd(K):
        return {v for v in range(n) if len(adj[v] & K) % 2 == 1}

    choices = []
    for i in meas:
        opts = []
        for r in range(len(cand) + 1):
            for K in itertools.combinations([c for c in cand if c != i], r):
                K = set(K)
                if i in odd(K):
                    opts.append(K | (odd(K) - {i}))  # vertices that must come after i
            # (g(i) itself and Odd(g(i)) \ {i})
        if not opts:
            return False
        choices.append(opts)
    idx = {v: k for k, v in enumerate(meas)}
    for combo in itertools.product(*choices):
        # acyclicity of i -> j among measured vertices
        succ = {i: [j for j in after if j in idx] for i, after in zip(meas, combo)}
        color = {}

        def dfs(u):
            color[u] = 1
            for w in succ[u]:
                if color.get(w) == 1 or (w not in color and not dfs(w)):
                    return False
            color[u] = 2
            return True

        if all(color.get(u) == 2 or (u not in color and dfs(u)) for u in meas):
            return True
    return False


def open_graph_pattern(n, edges, I, O):
    cmds = [W.E(a, b) for a, b in edges] + [W.M(v, 0.3 + v) for v in range(n) if v not in O]
    return W.Pattern(list(I), list(O), cmds)


@pytest.mark.parametrize("seed", range(60))
def test_gflow_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 6))
    edges = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.uniform() < 0.55]
    I = sorted(int(x) for x in rng.choice(n, size=int(rng.integers(1, min(2, n) + 1)), replace=False))
    O = sorted(int(x) for x in rng.choice(n, size=int(rng.integers(1, min(3, n) + 1)), replace=False))
    has, layers, depth = host_gflow(open_graph_pattern(n, edges, I, O))
    assert has == brute_force_gflow(n, edges, I, O), (n, edges, I, O)


def test_gflow_known_patterns():
    assert host_gflow(W.cnot_pattern_eq22())[0]                      # Eq. 22 has a flow
    assert host_gflow(W.j_pattern(0.4))[0]                            # J(alpha)
    ok, layers, depth = host_gflow(W.linear_cluster_pattern(10, seed=1))
    assert ok and depth == 10 and sorted(layers) == list(range(1, 11))  # a chain: one layer per M
    for name in ("C1", "QFT:6", "BW:6x4", "CL:5x6"):
        assert host_gflow(W.config_pattern(name))[0], name
    ok, layers, depth = host_gflow(W.cluster_pattern(4, 5, seed=1))
    assert depth == 4  # one backward layer per measured column (§4.6 cluster)
    # two inputs funnelled into one output: no gflow (|O| < |I|)
    assert not host_gflow(W.Pattern([1, 2], [3], [W.E(1, 3), W.E(2, 3), W.M(1, 0.), W.M(2, 0.)]))[0]
    # an isolated measured qubit can never satisfy u in Odd(g(u))
    assert not host_gflow(W.Pattern([1], [2], [W.N(3), W.M(3, 0.1), W.N(2), W.E(1, 2), W.M(1, 0.2)]))[0]
