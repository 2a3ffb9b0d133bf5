"""Write tests/golden/c3_prefix_oracle.npz: the ORACLE's result on a full-width prefix of config 3.

Calls only oracle/ and workloads/ (the seeded pattern and input recipes); nothing from the CUDA path.
The GPU test (tests/test_gpu_fullwidth.py) runs the same prefix at the same width through the C-ABI
and compares outcome strings, prob0 and the sampled amplitudes stored here ("parity
runs a depth-k prefix at full width"; "outputs are verified ... random input states").

  python tools/make_golden_c3_prefix.py [layers=1] [wires=28]

Config 3 = 28-wire brickwork (BASELINE configs[2]); the prefix is its first `layers` layers (4
commands per J, 1 per CZ), input = the documented counter-Haar state (workloads/inputs.py, the same
recipe owqs_set_input_random implements on the device), sampled mode with seed 5. The oracle runs
at 2^(wires+1) complex128 amplitudes (~25 min and ~40 GB of host memory per layer at 28 wires).
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import patterns as W  # noqa: E402
from workloads.inputs import counter_haar_raw  # noqa: E402

IN_SEED, RUN_SEED, N_SAMPLE = 7, 5, 4096


def main():
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    wires = int(sys.argv[2]) if len(sys.argv) > 2 else 28
    base = W.config_pattern("C3", seed=1) if wires == 28 else W.config_pattern(f"BW:{wires}x40", seed=1)
    k = W.brickwork_layer_cmds(wires, layers)
    pre = W.prefix_pattern(base, k)
    n = 1 << wires
    psi = np.empty(n, dtype=np.complex128)
    step = 1 << 24
    for j0 in range(0, n, step):  # chunked: the generator's uint64 temporaries stay small
        psi[j0:j0 + step] = counter_haar_raw(IN_SEED, np.arange(j0, min(n, j0 + step), dtype=np.uint64))
    psi /= np.linalg.norm(psi)
    t0 = time.time()
    r = oracle.run(pre, psi, mode="sampled", seed=RUN_SEED)
    dt = time.time() - t0
    del psi
    rng = np.random.default_rng(12345)
    idx = np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, N_SAMPLE)])).astype(np.int64)
    out = os.path.join(ROOT, "tests", "golden", f"c3_prefix_l{layers}_w{wires}_oracle.npz")
    np.savez_compressed(out, idx=idx, amps=r.output[idx], outcomes=r.outcomes, prob0=r.prob0,
                        norm2=np.float64(np.vdot(r.output, r.output).real),
                        meta=np.array([wires, layers, k, IN_SEED, RUN_SEED, int(dt)]))
    print(f"{out}: {k} commands, {len(idx)} sampled amplitudes, oracle {dt:.0f} s")


if __name__ == "__main__":
    main()
