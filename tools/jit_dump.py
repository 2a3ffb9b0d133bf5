"""Dump the generated pass kernels of a config's program as one .cu file (prelude + kernels), for
offline SASS inspection: python tools/jit_dump.py C3 64 sampled out.cu  then
nvcc -gencode arch=compute_100a,code=sm_100a -cubin -Xptxas -v out.cu"""
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1604_05659_b200.host import jit_host  # noqa: E402
from workloads.patterns import config_pattern  # noqa: E402

name, prec, mode, out = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
steps = [int(s) for s in sys.argv[5].split(",")] if len(sys.argv) > 5 else None
r = jit_host(config_pattern(name), mode, prec, sources=True)
src = r["sources"]
with open(out, "w") as f:
    f.write(src.pop(-1))
    seen = set()
    for k in sorted(src):
        if steps is not None and k not in steps:
            continue
        body = src[k]
        nm = body.split("OWQS_KNAME")[0]
        if body in seen:
            continue
        seen.add(body)
        f.write(f"\n// ---- step {k}\n" + body)
print(out, len(seen), "kernels")
