"""Multi-rank (sharded) execution of the compiled program on CPU with the gloo backend.

Each process is one rank: it compiles the SAME pattern for n_ranks (include/owqs_host.h), runs its
shard through the test interpreter (tests/program_interp.py) — SWAP steps trade half-shards with the
partner rank over torch.distributed, reductions are all_reduced — and the gathered state is
compared with the oracle. This checks the host side of SURVEY §8(e) (placement, swap schedule,
rank-bit diagonals, reduction allreduce) without GPUs; the CUDA kernels of the same program are
checked on one B200 by the loopback backend (tests/test_gpu_sharded.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class GlooComm:
    def all_reduce_sum(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    def exchange(self, a, partner):
        me = dist.get_rank()
        send = torch.from_numpy(np.ascontiguousarray(np.stack([a.real, a.imag])))
        recv = torch.empty_like(send)
        if me < partner:
            dist.send(send, partner)
            dist.recv(recv, partner)
        else:
            dist.recv(recv, partner)
            dist.send(send, partner)
        r = recv.numpy()
        return r[0] + 1j * r[1]


def _worker(rank, world, port, cases, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, here)
        sys.path.insert(0, os.path.dirname(here))
        import oracle
        from paper_1604_05659_b200.host import compile_host
        from program_interp import Interp
        from workloads import patterns as W
        from workloads.inputs import haar_state
        comm = GlooComm()
        for name, seed, mode, prec in cases:
            p = W.config_pattern(name, seed=seed)
            prog = compile_host(p, mode, precision=prec, n_ranks=world)
            psi = haar_state(len(p.inputs), seed)
            forced = None
            if mode == "forced":
                forced = np.random.default_rng(seed).integers(0, 2, p.n_measure)
            it = Interp(prog, mode, seed=seed, forced=forced, rank=rank, world=world, comm=comm)
            shard = it.run(psi)
            gathered = [torch.empty(2, shard.size, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(np.stack([shard.real, shard.imag])))
            if rank == 0:
                full = np.concatenate([g[0].numpy() + 1j * g[1].numpy() for g in gathered])
                out = it.permute_out(full)
                if mode == "sampled":
                    ref = oracle.run(p, psi, mode="sampled", seed=seed)
                elif mode == "forced":
                    ref = oracle.run(p, psi, mode="forced", forced=forced)
                else:
                    ref = oracle.run(p, psi, mode="eowqs")
                err = float(np.max(np.abs(out - ref.output)))
                same = mode == "eowqs" or list(it.outcome) == list(ref.outcomes)
                out_q.put((name, mode, world, prog.info["n_swaps"], err, same))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_program_matches_oracle(world):
    # config 4's shape (brickwork, sampled) and config 5's (flow cluster, EOWQS and forced) scaled to
    # oracle size; world 8 = the 8-GPU split of SURVEY §8(e) (3 rank bits)
    cases = [("BW:14x6", 3, "sampled", 128), ("BW:15x4", 4, "eowqs", 64), ("CL:13x4", 5, "forced", 128),
             ("QFT:13", 1, "sampled", 128)]
    if world == 8:
        cases = [("BW:14x6", 3, "sampled", 128), ("CL:13x4", 5, "eowqs", 128), ("CL:13x4", 6, "forced", 128)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), cases, q), nprocs=world, join=True,
                       start_method="spawn")
    results = [q.get(timeout=60) for _ in cases]
    swaps = 0
    for name, mode, w, n_swaps, err, same in results:
        assert same, (name, mode, "outcome strings differ")
        assert err < 1e-10, (name, mode, err)
        swaps += n_swaps
    assert swaps > 0  # the cases do exercise global<->local swaps
