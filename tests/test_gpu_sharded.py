"""Sharded execution of the CUDA path on one B200 through the loopback backend:
G virtual ranks, each with its own shard, run one after the other on the device; SWAP steps trade
half-shards by device copies and reductions are all-reduced by a kernel. The per-rank kernels,
the rank-bit diagonals, the swap pack/unpack and the reduction all-reduce are the ones the NCCL
backend uses (only the transport differs). Checked against the oracle and against 1-rank runs."""
import numpy as np
import pytest

import oracle
from paper_1604_05659_b200 import FLAG_LOOPBACK, FLAG_MEASURED_NORM, Simulator
from parity_util import TOL, check, fidelity
from workloads import patterns as W
from workloads.inputs import haar_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("prec", [128, 64])
def test_loopback_vs_oracle(require_gpu, G, prec):
    s = Simulator(precision=prec, flags=FLAG_LOOPBACK, n_ranks=G)
    try:
        for name, seed in (("BW:14x6", 3), ("CL:13x4", 5), ("QFT:13", 1)):
            p = W.config_pattern(name, seed=seed)
            psi = haar_state(len(p.inputs), seed)
            check(s, p, psi, "sampled", seed=seed)
            check(s, p, psi, "forced", forced=np.random.default_rng(seed).integers(0, 2, p.n_measure))
            check(s, p, psi, "eowqs")
            assert s.stats()["n_swaps"] > 0 or name == "QFT:13"
    finally:
        s.close()


def test_loopback_c3_full_width_vs_single_rank(require_gpu):
    """Config 3 at full width sharded 8 ways (loopback) equals the 1-rank run: fidelity, norm and
    identical outcome strings (only the reduction order differs)."""
    p = W.config_pattern("C3", seed=1)
    a = Simulator(precision=64)
    b = Simulator(precision=64, flags=FLAG_LOOPBACK, n_ranks=8)
    try:
        a.load(p)
        b.load(p)
        assert b.stats()["n_swaps"] > 0
        a.set_input_random(11)
        b.set_input_random(11)
        oa, pa = a.run("sampled", seed=4)
        ob, pb = b.run("sampled", seed=4)
        assert list(oa) == list(ob)
        assert np.max(np.abs(pa - pb)) < 1e-6
        assert abs(b.norm2() - 1) < 1e-4
        xa, xb = a.get_output(), b.get_output()
        assert 1 - fidelity(xa, xb) < 1e-6
        assert np.max(np.abs(xa - xb)) < 1e-5
    finally:
        a.close()
        b.close()


def test_loopback_cluster_outcome_independence(require_gpu):
    """Config 5 family sharded (26 x 8 cluster, fp64, 8 virtual ranks): EOWQS equals random forced
    branches up to a global phase, every prob0 = 1/2, norm 1."""
    p = W.config_pattern("CL:26x8", seed=1)
    a = Simulator(precision=128, flags=FLAG_LOOPBACK | FLAG_MEASURED_NORM, n_ranks=8)
    try:
        a.load(p)
        a.set_input_random(3)
        a.run("eowqs")
        assert abs(a.norm2() - 1) < 1e-10
        ref = a.get_output()
        a.set_input_random(3)
        _, p0 = a.run("forced", forced=np.random.default_rng(2).integers(0, 2, p.n_measure))
        assert np.max(np.abs(p0 - 0.5)) < 1e-12
        out = a.get_output()
        assert abs(fidelity(out, ref) - 1) < 1e-10
    finally:
        a.close()
