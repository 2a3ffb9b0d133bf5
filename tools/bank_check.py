"""Static bank-conflict check of generated tile kernels: for every layout's shared-memory base
`sb<l> = 16 * (XOR over lane/warp bits of coefficient)`, a quarter-warp (lanes 0..7) of 16 B
accesses is conflict-free iff the 16 B-unit coefficients of lane bits 0..2 have linearly independent
low 3 bits (bank groups). Counts conflicted layouts (weighted by their accesses) per kernel."""
import re
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1604_05659_b200.host import jit_host  # noqa: E402
from workloads.patterns import config_pattern  # noqa: E402


def rank_bits(vals, nbits):
    rows = list(vals)
    r = 0
    for b in reversed(range(nbits)):
        bit = 1 << b
        piv = next((i for i in range(r, len(rows)) if rows[i] & bit), None)
        if piv is None:
            continue
        rows[r], rows[piv] = rows[piv], rows[r]
        for i in range(len(rows)):
            if i != r and rows[i] & bit:
                rows[i] ^= rows[r]
        r += 1
    return r


def conflicted_accesses(sources):
    """(conflicted, total) shared-memory accesses over the generated kernel sources. Bases are byte
    offsets; a 16 B access (float4 / double2) is conflict-free when lane bits 0..2 give independent
    bank groups (bits 4..6 of the address), an 8 B access (float2) when lane bits 0..3 give
    independent 8 B slots of a 128 B wavefront (bits 3..6)."""
    tot = bad = 0
    for k, s in sorted(sources.items()):
        if k < 0:
            continue
        bases = {}
        for m in re.finditer(r"const int sb(\d+) = \((.*)\);", s):
            coef = {int(a): int(b) for a, b in re.findall(r"\(\(lane >> (\d)\) & 1\) \* (\d+)\)", m.group(2))}
            bases[m.group(1)] = coef
        for m in re.finditer(r"reinterpret_cast<(?:const )?(float4|double2|float2)\*>\(dsm \+ \(sb(\d+) \^", s):
            c = bases[m.group(2)]
            tot += 1
            if m.group(1) == "float2":
                ok = rank_bits([(c.get(j, 0) >> 3) & 15 for j in range(4)], 4) == 4
            else:
                ok = rank_bits([(c.get(j, 0) >> 4) & 7 for j in range(3)], 3) == 3
            bad += not ok
    return bad, tot


if __name__ == "__main__":
    wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
    src = jit_host(config_pattern(wl, seed=1), "sampled", 64, sources=True)["sources"]
    bad, tot = conflicted_accesses(src)
    print(f"{wl}: {bad} of {tot} shared-memory accesses from layouts with a conflicted quarter-warp")
