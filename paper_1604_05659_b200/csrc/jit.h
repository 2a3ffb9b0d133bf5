// Load-time specialisation of the fused pass kernel (DESIGN.md §5 "generated pass kernels").
//
// Every state pass of a compiled program (StepDesc, ST_PASS) is turned into one straight-line
// sm_100a kernel: the pass's slots, op order, absorbed-CZ masks, folded X renamings, reduction kind
// and width are compile-time constants; only the measurement decisions (outcomes, Eq. 2 angles,
// Eqs. 11-12 coefficients, signal conditions) stay runtime values, computed by the shared prologue
// (device_common.cuh). NVRTC compiles the generated translation units for sm_100a at load_pattern
// time (host only, no device needed); the cubins are loaded on the device with the runtime's
// library API when the context first runs.
#pragma once

#include <stdint.h>

#include <cuda_runtime_api.h>

#include <string>
#include <vector>

#include "owqs_internal.h"

namespace owqs {

// SB = warp-segment bits (6 complex64, 5 complex128). Same UNR rule as the AOT kernel.
inline int jit_unr_of(int khi) { return khi == 0 ? 4 : (khi == 1 ? 2 : 1); }

// Engine of a step: 0 = not generated (ahead-of-time kernel), 1 = direct-load kernel (complex128,
// narrow complex64), 2 = TMA-pipelined complex64 kernel with shared-memory transposes (width >= 13).
int jit_engine(const StepDesc& d, int prec);
// Group slots per pass the packer may use for this precision (KTILE when the tile engine runs the
// wide passes, else KMAX_AOT).
int jit_max_group(int prec, bool no_jit);
// True when the step runs as a generated pass kernel.
bool jit_eligible(const StepDesc& d, int prec);
// Dynamic shared memory (bytes) and threads per block an engine's kernels are launched with.
int jit_dyn_smem(int engine, int prec);
int jit_block_threads(int engine, int prec);
// A tile-engine pass small enough (<= 2 waves) to decide and reduce inside its own kernel (no
// decide_kernel / grid_finish_kernel launches).
bool jit_tile_small(const StepDesc& d, int prec);
// Grid of a tile-engine pass (= its number of block partials for grid_finish_kernel).
unsigned jit_tile_blocks(const StepDesc& d, int prec);
// cudaFuncAttributePreferredSharedMemoryCarveout (percent) for an engine's kernels; -1 = default
int jit_smem_carveout(int engine, int prec);

// Kernel source of one pass (no prelude). *name receives the kernel's extern "C" name, which is
// a hash of the body (identical passes share one kernel). coef_src: where a tile kernel reads the
// pass's decisions (butterfly coefficients, scale, op conditions) --
//   0 COEF_POINTER: the PassCoef decide_kernel wrote to global memory (registers);
//   1 COEF_PARAM:   its by-value PassCoef parameter (constant bank 0: uniform operands), written into
//                   the device-updatable graph node by decide_kernel (host: run-independent EOWQS);
//   2 COEF_CONST:   the module's __constant__ <kernel>_cp (constant bank: uniform operands), filled by
//                   a graph memcpy node from decide_kernel's output (host: EOWQS). Unlike 1, the
//                   kernel nodes stay ordinary (profilable by ncu).
enum { COEF_POINTER = 0, COEF_PARAM = 1, COEF_CONST = 2 };
std::string jit_pass_source(const StepDesc& d, int prec, std::string* name, int coef_src = COEF_CONST);
// Byte offset of the by-value PassCoef parameter in a tile kernel's parameter buffer.
size_t jit_coef_param_offset(cudaKernel_t k);

// The common prelude every generated translation unit starts with.
const std::string& jit_prelude();

struct JitModule {
  std::vector<char> cubin;
  std::vector<std::string> names;  // kernels in this cubin
};

// Compile the given kernel sources (deduplicated by name) into cubins for sm_100a. Results are
// cached per process (keyed by the source text). Returns "" on success, else the NVRTC log.
std::string jit_compile(const std::vector<std::string>& names, const std::vector<std::string>& sources,
                        std::vector<JitModule>& out, double* compile_ms = nullptr);

// Version of the NVRTC jit_compile uses; "" on success, else why it cannot be loaded.
std::string jit_nvrtc_version(int* major, int* minor);

}  // namespace owqs
