// Device-side kernel-node parameter update (CUDA 12.4+ device-updatable graph nodes), the mechanism
// that puts the tile kernels' runtime-decided coefficients into their parameter bank:
//   writer<<<1,32>>> (decide) -> reader<<<...>>> (pass kernel, PDL behind the writer)
// The writer reads a value the host changes before every graph launch and writes it into the
// reader node's by-value parameter struct with cudaGraphKernelNodeSetParam; the reader stores what
// it sees. Checks every launch over 2000 launches, with and without programmatic dependent launch.
// nvcc -rdc=true -gencode arch=compute_100a,code=sm_100a -o /tmp/du tools/devupdate_probe.cu -lcudadevrt && /tmp/du
#include <cuda_runtime.h>
#include <stdio.h>

struct Coef {
  float ar[64];
  unsigned long long B[64];
  double scale;
};

__global__ void writer(const int* src, cudaGraphDeviceNode_t* node, size_t off, int pdl) {
  __shared__ Coef c;
  const int v = *src;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    c.ar[i] = (float)(v + i);
    c.B[i] = (unsigned long long)(v * 3 + i);
  }
  if (threadIdx.x == 0) c.scale = v * 0.5;
  __syncthreads();
  if (threadIdx.x == 0) {
    cudaGraphKernelNodeSetParam(*node, off, &c, sizeof(Coef));
    __threadfence();
  }
  __syncthreads();
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void reader(int* out, const Coef c) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = (int)c.ar[5];
    out[1] = (int)c.B[63];
    out[2] = (int)(c.scale * 2);
  }
}

int main() {
  int *src, *out, *h;
  cudaMalloc(&src, 4);
  cudaMalloc(&out, 16);
  cudaMallocHost(&h, 16);
  cudaGraphDeviceNode_t* dnode;
  cudaMalloc(&dnode, sizeof(cudaGraphDeviceNode_t));
  size_t off = 0, sz = 0;
  cudaError_t e = cudaFuncGetParamInfo((const void*)reader, 1, &off, &sz);
  printf("param 1 offset %zu size %zu (%s)\n", off, sz, cudaGetErrorString(e));
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    writer<<<1, 32, 0, s>>>(src, dnode, off, pdl);
    Coef c0 = {};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(296);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeDeviceUpdatableKernelNode;
    at[0].val.deviceUpdatableKernelNode.deviceUpdatable = 1;
    at[0].val.deviceUpdatableKernelNode.devNode = nullptr;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, reader, out, c0);
    if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
    e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess) printf("capture: %s\n", cudaGetErrorString(e));
    cudaGraphDeviceNode_t hn = at[0].val.deviceUpdatableKernelNode.devNode;
    printf("pdl=%d devNode %p\n", pdl, (void*)hn);
    cudaMemcpy(dnode, &hn, sizeof(hn), cudaMemcpyHostToDevice);
    cudaGraphExec_t ge;
    e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) printf("instantiate: %s\n", cudaGetErrorString(e));
    e = cudaGraphUpload(ge, s);
    if (e != cudaSuccess) printf("upload: %s\n", cudaGetErrorString(e));
    int bad = 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int it = 0; it < 2000; ++it) {
      const int v = 1000 + 7 * it + pdl;
      cudaMemcpyAsync(src, &v, 4, cudaMemcpyHostToDevice, s);
      cudaGraphLaunch(ge, s);
      cudaMemcpyAsync(h, out, 12, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (h[0] != v + 5 || h[1] != v * 3 + 63 || h[2] != v) {
        if (bad < 5) printf("it %d: got %d %d %d want %d %d %d\n", it, h[0], h[1], h[2], v + 5, v * 3 + 63, v);
        ++bad;
      }
    }
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d: %d bad of 2000 (%s), %.1f us per launch incl. sync\n", pdl, bad,
           cudaGetErrorString(cudaGetLastError()), ms * 1e3 / 2000);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  return 0;
}
