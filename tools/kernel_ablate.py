"""Ablation harness for one generated tile kernel: builds a standalone .cu with the kernel's source
and variants (no reduction, no transposes, no butterflies, no PDL wait), times each on the state
size of the pass (nvcc + run on the GPU box). python tools/kernel_ablate.py C3 <step> out.cu"""
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_05659_b200.host import compile_host, jit_host  # noqa: E402
from workloads.patterns import config_pattern  # noqa: E402

name, step, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
pat = config_pattern(name)
r = jit_host(pat, "sampled", 64, sources=True)
hp = compile_host(pat, "sampled", 64)
prelude = r["sources"][-1]
src = r["sources"][step]
width = hp.steps[step].width


def variant(tag, body):
    return body.replace("OWQS_KNAME", "k_" + tag) if "OWQS_KNAME" in body else re.sub(
        r"(__global__ void __launch_bounds__\([^)]*\) )(\w+)", r"\1k_" + tag, body, count=1)


base = src
no_red = re.sub(r"  double acc\[4\] = \{acc0, acc1, acc2, acc3\};\n  reduce_finish_grid<\d>\(acc, p, red_s, &flag_s\);\n",
                "  if (acc0 == 12345.0) p.red_result[0] = acc0 + acc1 + acc2 + acc3;\n", base)
no_wait = base.replace('asm volatile("griddepcontrol.wait;" ::: "memory");', "")
# drop transposes: remove shared-memory store/load lines and the barriers between phases
lines = base.split("\n")
no_tr = "\n".join(l for l in lines if not ("dsm + sb" in l or l.strip() in ("__syncthreads();", "__syncwarp();")))
no_ops = "\n".join(l for l in lines if not (l.strip().startswith("{ const u64 y = ") or "shfl2(y" in l))
# block partial only (no fence, no atomics): a separate finish kernel sums the partials
red_part = re.sub(r"  double acc\[4\] = \{acc0, acc1, acc2, acc3\};\n  reduce_finish_grid<(\d)>\(acc, p, red_s, &flag_s\);\n",
                  r"  double acc[4] = {acc0, acc1, acc2, acc3};\n  block_partial<\1>(acc, p, red_s);\n", base)
# PDL wait just before the first PassCoef read after the loads
wl = base.replace('    asm volatile("griddepcontrol.wait;" ::: "memory");\n', "", 1)
i = wl.find("pc->", wl.find("__ldcs"))
j = wl.rfind("\n", 0, i)
wait_late = wl[:j + 1] + '    asm volatile("griddepcontrol.wait;" ::: "memory");\n' + wl[j + 1:]
both = red_part.replace('    asm volatile("griddepcontrol.wait;" ::: "memory");\n', "", 1)
i = both.find("pc->", both.find("__ldcs"))
j = both.rfind("\n", 0, i)
both = both[:j + 1] + '    asm volatile("griddepcontrol.wait;" ::: "memory");\n' + both[j + 1:]
vars_ = {"base": base, "red_part": red_part, "wait_late": wait_late, "both": both, "no_red": no_red, "no_wait": no_wait, "no_tr": no_tr, "no_ops": no_ops,
         "no_tr_red": re.sub(r"  double acc\[4\] = \{acc0, acc1, acc2, acc3\};\n  reduce_finish_grid<\d>\(acc, p, red_s, &flag_s\);\n",
                             "  if (acc0 == 12345.0) p.red_result[0] = acc0;\n", no_tr)}
with open(out, "w") as f:
    f.write("#include <cuda_runtime.h>\n#include <stdio.h>\n#include <string.h>\n" + prelude.replace("#ifdef __CUDACC_RTC__", "#if 0"))
    f.write("""
namespace owqs {
template <int NRED>
__device__ void block_partial(double (&acc)[4], const DevPtrs& p, double (*red)[4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < NRED; ++k)
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
  if (lane == 0) for (int k = 0; k < NRED; ++k) red[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < NRED) {
    double t = 0;
    for (int w = 0; w < nw; ++w) t += red[w][threadIdx.x];
    p.partials[(size_t)blockIdx.x * 4 + threadIdx.x] = t;
  }
}
}
""")
    for tag, body in vars_.items():
        m = re.search(r"__global__ void __launch_bounds__\([^)]*\) (\w+)\(", body)
        f.write("\n" + body.replace(m.group(1) + "(", "k_" + tag + "(", 1))
    f.write(f'''
int main() {{
  using namespace owqs;
  const int width = {width};
  const size_t n = 1ull << width;
  void* st; cudaMalloc(&st, n * 8); cudaMemset(st, 0, n * 8);
  double* part; cudaMalloc(&part, (RED_MAX_BLOCKS + RED_MAX_GROUPS) * 4 * sizeof(double));
  unsigned* cnt; cudaMalloc(&cnt, (1 + RED_MAX_GROUPS) * 4); cudaMemset(cnt, 0, (1 + RED_MAX_GROUPS) * 4);
  double* red; cudaMalloc(&red, 64);
  PassCoef h{{}}; h.scale = 0.7071;
  for (int b = 0; b < MAX_BFLY; ++b) {{ h.ar[b] = 0.6f; float ai = 0.8f; unsigned lo, hi; float nai = -ai;
    memcpy(&lo, &nai, 4); memcpy(&hi, &ai, 4); h.B[b] = ((unsigned long long)hi << 32) | lo; }}
  for (int i = 0; i < MAX_OPS; ++i) h.cond[i] = 1;
  PassCoef* pc; cudaMalloc(&pc, sizeof h); cudaMemcpy(pc, &h, sizeof h, cudaMemcpyHostToDevice);
  StepDesc d{{}}; DevPtrs p{{}}; p.state = st; p.partials = part; p.counter = cnt; p.red_result = red;
  const unsigned blocks = (unsigned)(n >> 13);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto time = [&](const char* tag, auto kern, int co) {{
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 74832);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, co);
    kern<<<blocks, 256, 74832>>>(d, p, pc); cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {{ cudaEventRecord(e0); kern<<<blocks, 256, 74832>>>(d, p, pc); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }}
    int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 256, 74832);
    printf("%-10s carveout %4d: %d CTAs/SM %.3f ms  %s\\n", tag, co, nb, best, cudaGetErrorString(cudaGetLastError()));
  }};
''')
    for tag in vars_:
        for co in (67,):
            f.write(f'  time("{tag}", k_{tag}, {co});\n')
    f.write("  return 0;\n}\n")
print(out, "width", width)
