"""owqs_submit_host / owqs_wait (include/owqs.h): the asynchronous host-to-host run (input state
in, output state out) against the oracle, two contexts pipelined on separate streams, and
the call contract (page-locked buffers, E_STATE while a run is pending)."""
import numpy as np
import pytest

import oracle
from paper_1604_05659_b200 import OwqsError, Simulator
from parity_util import TOL, fidelity
from workloads import patterns as W
from workloads.inputs import haar_state

pytestmark = pytest.mark.gpu


def pinned(n, prec):
    import torch
    return torch.empty(n, dtype=torch.complex64 if prec == 64 else torch.complex128, pin_memory=True)


@pytest.mark.parametrize("prec", [128, 64])
@pytest.mark.parametrize("shape", ["BW:14x4", "QFT:6"])
def test_submit_wait_matches_oracle(require_gpu, prec, shape):
    p = W.config_pattern(shape, seed=4)
    n = len(p.inputs)
    psi = haar_state(n, 21)
    s = Simulator(precision=prec)
    try:
        s.load(p)
        h_in, h_out = pinned(2 ** n, prec), pinned(2 ** len(p.outputs), prec)
        h_in.numpy()[:] = psi
        forced = np.random.default_rng(5).integers(0, 2, p.n_measure)
        s.submit_host(h_in.data_ptr(), prec, h_out.data_ptr(), prec, "forced", forced=forced)
        outc, p0 = s.wait(want=True)
        ref = oracle.run(p, psi, mode="forced", forced=forced)
        out = h_out.numpy().astype(np.complex128)
        assert list(outc) == list(forced)
        tol = TOL[prec]
        assert np.max(np.abs(out - ref.output)) <= tol["amp"]
        if prec == 64:
            assert 1 - fidelity(out, ref.output) <= tol["fid"]
        # sampled: the same outcomes and output as the synchronous calls on the same seed
        s.submit_host(h_in.data_ptr(), prec, h_out.data_ptr(), prec, "sampled", seed=9)
        a_outc, _ = s.wait(want=True)
        s.set_input(psi.astype(np.complex64) if prec == 64 else psi)
        b_outc, _ = s.run("sampled", seed=9)
        assert list(a_outc) == list(b_outc)
        np.testing.assert_allclose(h_out.numpy(), s.get_output().astype(h_out.numpy().dtype), atol=tol["amp"])
    finally:
        s.close()


def test_two_contexts_pipelined(require_gpu):
    """Two contexts on two streams, submits interleaved (each waits only for its own previous run):
    every output equals the oracle's for its own seed's branch."""
    import torch
    p = W.config_pattern("BW:16x3", seed=2)
    n = len(p.inputs)
    psi = haar_state(n, 3)
    sims = [Simulator(precision=128, stream=torch.cuda.Stream().cuda_stream) for _ in range(2)]
    try:
        h_in = pinned(2 ** n, 128)
        h_in.numpy()[:] = psi
        outs = [pinned(2 ** n, 128) for _ in range(2)]
        for x in sims:
            x.load(p)
        busy = [None, None]
        results = []
        for i in range(6):
            c = i % 2
            if busy[c] is not None:
                outc, _ = sims[c].wait(want=True)
                results.append((busy[c], outc, outs[c].numpy().copy()))
            sims[c].submit_host(h_in.data_ptr(), 128, outs[c].data_ptr(), 128, "sampled", seed=100 + i)
            busy[c] = 100 + i
        for c in range(2):
            outc, _ = sims[c].wait(want=True)
            results.append((busy[c], outc, outs[c].numpy().copy()))
        assert len(results) == 6
        for seed, outc, out in results:
            ref = oracle.run(p, psi, mode="forced", forced=outc)
            assert np.max(np.abs(out - ref.output)) <= TOL[128]["amp"]
            np.testing.assert_allclose(oracle.run(p, psi, mode="sampled", seed=seed).outcomes, outc)
    finally:
        for x in sims:
            x.close()


def test_submit_contract(require_gpu):
    p = W.config_pattern("BW:13x2", seed=1)
    n = len(p.inputs)
    s = Simulator(precision=64)
    try:
        s.load(p)
        h_in, h_out = pinned(2 ** n, 64), pinned(2 ** n, 64)
        h_in.numpy()[:] = haar_state(n, 1)
        with pytest.raises(OwqsError) as e:
            s.wait()
        assert e.value.status_name == "OWQS_E_STATE"
        pageable = np.zeros(2 ** n, dtype=np.complex64)
        with pytest.raises(OwqsError) as e:
            s.submit_host(pageable.ctypes.data, 64, h_out.data_ptr(), 64, "sampled")
        assert e.value.status_name == "OWQS_E_ARG"
        s.submit_host(h_in.data_ptr(), 64, h_out.data_ptr(), 64, "eowqs")
        for call in (lambda: s.set_input_random(1), lambda: s.run("eowqs"), lambda: s.get_output(),
                     lambda: s.submit_host(h_in.data_ptr(), 64, h_out.data_ptr(), 64, "eowqs")):
            with pytest.raises(OwqsError) as e:
                call()
            assert e.value.status_name == "OWQS_E_STATE"
        s.wait()
        assert abs(np.linalg.norm(h_out.numpy()) - 1.0) < 1e-3
    finally:
        s.close()
