// Probe: load a cubin with the runtime library API and report the error (diagnostics only).
#include <cuda_runtime.h>
#include <stdio.h>
int main(int argc, char** argv) {
  cudaLibrary_t lib;
  cudaError_t e = cudaLibraryLoadFromFile(&lib, argv[1], nullptr, nullptr, 0, nullptr, nullptr, 0);
  printf("load %s: %s\n", argv[1], cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  unsigned n = 0;
  cudaLibraryGetKernelCount(&n, lib);
  printf("kernels: %u\n", n);
  return 0;
}
