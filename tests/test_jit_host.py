"""CPU tests of the load-time generated pass kernels (csrc/jit.cpp): the generator's
output for representative programs NVRTC-compiles for sm_100a without a GPU, every state pass of a
wide complex64 program runs on the tile engine, and the phase plan keeps every butterfly, X and
reduction in registers (no cross-lane shuffles). GPU parity of the same kernels: test_gpu_parity.py."""
import re

import pytest

from paper_1604_05659_b200 import FLAG_NO_JIT
from paper_1604_05659_b200.host import compile_host, jit_host
from workloads import patterns as W


@pytest.mark.parametrize("shape,prec", [("BW:16x6", 64), ("BW:14x4", 128), ("QFT:13", 64)])
def test_generated_kernels_compile(shape, prec):
    p = W.config_pattern(shape, seed=3)
    r = jit_host(p, "sampled", prec, sources=True)
    hp = compile_host(p, "sampled", prec)
    passes = [k for k, s in enumerate(hp.steps) if s.kind == 0]
    assert r["n_jit_steps"] == sum(1 for k in passes if k in r["sources"])
    assert r["n_kernels"] >= 1
    for k, src in r["sources"].items():
        if k < 0:
            continue
        assert "extern \"C\" __global__" in src
        if hp.steps[k].width >= (13 if prec == 64 else 12):
            assert "tile engine" in src
            # every op of a tile-engine pass runs on register slots (the phase plan's guarantee)
            assert "(lane)" not in src and "shfl2(" not in src


def test_wide_passes_need_the_tile_engine():
    """Group slots per pass on the tile engine: 6 for complex64 (12-bit tiles, 4-warp CTAs; 7 with
    OWQS_TILE_G=7), 6 for complex128 (11-bit tiles); 4 otherwise (AOT / direct)."""
    p = W.config_pattern("C3")
    wide = compile_host(p, "sampled", 64)
    narrow = compile_host(p, "sampled", 64, flags=FLAG_NO_JIT)
    c128 = compile_host(p, "sampled", 128)
    assert max(s.nb_hi for s in wide.steps) == 6 and max(s.nb_hi for s in c128.steps) == 6
    assert max(s.nb_hi for s in narrow.steps) <= 4
    # wider tiles fuse more butterflies per state sweep: about half the passes (52 vs 100)
    assert wide.info["n_passes"] < 0.6 * narrow.info["n_passes"]


def test_tile_kernel_structure_c3():
    """Config 3's tile kernels: no lane butterflies, transposes only between phases, the pass scale
    folded into one butterfly, fence-free block partials for the deterministic grid finish."""
    r = jit_host(W.config_pattern("C3"), "sampled", 64, sources=True)
    srcs = [s for k, s in r["sources"].items() if k >= 0]
    assert srcs and all("tile engine" in s for s in srcs)
    for s in srcs:
        n_b = int(re.search(r"(\d+) butterflies", s).group(1))
        if n_b:
            assert s.count("scale folded") == 1
        phases = int(re.search(r"(\d+) phase\(s\)", s).group(1))
        trans = int(re.search(r"(\d+) transpose\(s\)", s).group(1))
        assert trans <= phases + 1
        # fence-free block partials (summed by grid_finish_kernel) exactly in the passes that reduce:
        # with R-13's ||psi||^2 = 1 only the last pass (the output's norm) does
        red = int(re.search(r"reduction (\d+)", s).group(1))
        assert ("block_partial" in s) == (red != 0)
    assert sum("block_partial" in s for s in srcs) >= 1


def test_generator_uses_toolkit_nvrtc_after_torch():
    """The generator compiles with the build toolkit's NVRTC (loaded by path, own symbol scope), not
    a libnvrtc.so.12 loaded earlier by another library: torch's bundled cu128 copy produces slower
    sm_100a code for the same source."""
    import subprocess
    import sys
    code = ("import torch; torch.zeros(1)\n"
            "from paper_1604_05659_b200.host import nvrtc_version, jit_host\n"
            "from workloads import patterns as W\n"
            "jit_host(W.config_pattern('BW:14x2', seed=1), 'sampled', 64)\n"
            "maps = [l.split()[-1] for l in open('/proc/self/maps') if 'libnvrtc.so' in l]\n"
            "print(nvrtc_version(), sorted(set(maps)))\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                         cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert out.returncode == 0, out.stderr[-2000:]
    maps = out.stdout
    from paper_1604_05659_b200.host import nvrtc_version
    major, minor = nvrtc_version()
    assert (major, minor) >= (12, 9)
    assert f"({major}, {minor})" in out.stdout
    assert "/usr/local/cuda" in maps or "cuda-12" in maps


@pytest.mark.parametrize("shape", ["BW:16x8", "BW:18x6"])
def test_tile_transposes_bank_conflict_free(shape):
    """Every shared-memory access of the generated tile kernels is quarter-warp conflict-free: the
    per-kernel bank classes give each layout's lane bits 0..2 independent bank-group bits
    (tools/bank_check.py)."""
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    from bank_check import conflicted_accesses
    src = jit_host(W.config_pattern(shape, seed=1), "sampled", 64, sources=True)["sources"]
    bad, tot = conflicted_accesses(src)
    assert tot > 0 and bad == 0, (bad, tot)


def test_t0_free_option_conflict_free_and_fewer_transposes(monkeypatch):
    """OWQS_T0_FREE (complex64 phases may leave t0 out of the registers; off by default, not faster
    on B200 -- profiles/r01c/README.md): still bank-conflict free, fewer transposes."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    from bank_check import conflicted_accesses

    def count(src):
        n = 0
        for k, s in src.items():
            m = re.search(r"(\d+) transpose\(s\)", s)
            n += int(m.group(1)) if m else 0
        return n

    p = W.config_pattern("BW:18x8", seed=2)
    base = jit_host(p, "sampled", 64, sources=True)["sources"]
    monkeypatch.setenv("OWQS_T0_FREE", "1")
    free = jit_host(p, "sampled", 64, sources=True)["sources"]
    bad, tot = conflicted_accesses(free)
    assert tot > 0 and bad == 0
    assert count(free) <= count(base)
    assert any("reinterpret_cast<float2*>" in s for s in free.values())


@pytest.mark.parametrize("g", ["5", "7"])
def test_other_tile_sizes_generate_conflict_free(g):
    """OWQS_TILE_G = 5 / 7 (2- / 8-warp complex64 CTAs) still generate conflict-free transposes
    (the setting is read once per process: checked in a subprocess)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(__file__))
    code = ("import sys; sys.path.insert(0, 'tools')\n"
            "from bank_check import conflicted_accesses\n"
            "from paper_1604_05659_b200.host import jit_host\n"
            "from workloads import patterns as W\n"
            "src = jit_host(W.config_pattern('BW:16x6', seed=1), 'sampled', 64, sources=True)['sources']\n"
            "bad, tot = conflicted_accesses(src)\n"
            "threads = {int(x) for x in __import__('re').findall(r'__launch_bounds__\\((\\d+),', ''.join(src.values()))}\n"
            "print(bad, tot, sorted(threads))\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, OWQS_TILE_G=g))
    assert out.returncode == 0, out.stderr[-2000:]
    bad, tot, threads = out.stdout.split(" ", 2)
    assert int(bad) == 0 and int(tot) > 0
    assert str(32 << (int(g) - 4)) in threads


@pytest.mark.parametrize("shape,prec", [("C3", 64), ("BW:16x6", 128)])
def test_tile_kernels_read_state_after_pdl_wait(shape, prec):
    """Tile kernels are launched with programmatic stream serialisation; PTX makes the prerequisite
    grid's stores visible only after griddepcontrol.wait, so no state load (or PassCoef read) may
    precede it -- only L2 bulk prefetches (L2 is the point of coherence)."""
    r = jit_host(W.config_pattern(shape, seed=3), "sampled", prec, sources=True)
    n = 0
    for k, s in r["sources"].items():
        if k < 0 or "tile engine" not in s:
            continue
        body = s[s.index("__global__"):]
        w = body.find("griddepcontrol.wait")
        assert w > 0
        assert "__ldcs(" not in body[:w] and "pc->" not in body[:w].split("// pc:")[-1].split("\n", 1)[-1]
        n += 1
    assert n > 0
