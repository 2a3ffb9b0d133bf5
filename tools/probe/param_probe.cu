// Probe: largest by-value kernel parameter block that loads/launches on this device.
#include <cuda_runtime.h>
#include <stdio.h>
template <int N> struct Blob { unsigned char b[N]; };
template <int N> __global__ void k(const Blob<N> x, int* out) { if (threadIdx.x == 0) *out = x.b[N - 1]; }
template <int N> void probe(int* d) {
  Blob<N> x{};
  x.b[N - 1] = 7;
  int nb = 0;
  cudaError_t e1 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k<N>, 256, 0);
  k<N><<<1, 32>>>(x, d);
  cudaError_t e2 = cudaDeviceSynchronize();
  int h = 0;
  cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("param %5d B: occupancy %s, launch %s, value %d\n", N, cudaGetErrorString(e1), cudaGetErrorString(e2), h);
  cudaGetLastError();
}
int main() {
  int* d;
  cudaMalloc(&d, 4);
  probe<1024>(d); probe<2048>(d); probe<2760>(d); probe<3200>(d); probe<4000>(d); probe<8000>(d);
  return 0;
}
