// Can an instantiated graph's kernel node with a large parameter block be
// re-parameterised (cudaGraphExecKernelNodeSetParams)?  (tools/micro)
#include <cstdio>
#include <cuda_runtime.h>
template <int B> struct Blob { int v[B / 4]; };
template <int B> __global__ void k(const __grid_constant__ Blob<B> b, int *out) { if (threadIdx.x == 0) out[0] = b.v[B / 4 - 1]; }
template <int B> void probe(int *out) {
  Blob<B> b{};
  b.v[B / 4 - 1] = 1;
  void *args[2] = {&b, &out};
  cudaKernelNodeParams np{};
  np.func = (void *)k<B>;
  np.gridDim = dim3(1);
  np.blockDim = dim3(32);
  np.sharedMemBytes = 0;
  np.kernelParams = args;
  np.extra = nullptr;
  cudaGraph_t g; cudaGraphExec_t e; cudaGraphNode_t n;
  cudaGraphCreate(&g, 0);
  cudaError_t r1 = cudaGraphAddKernelNode(&n, g, nullptr, 0, &np);
  cudaError_t r2 = cudaGraphInstantiate(&e, g, 0);
  b.v[B / 4 - 1] = 2;
  cudaError_t r3 = cudaGraphExecKernelNodeSetParams(e, n, &np);
  cudaError_t r4 = cudaGraphLaunch(e, 0);
  cudaDeviceSynchronize();
  int h = 0;
  cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("%6d B: add %s inst %s set %s launch %s -> %d\n", B, cudaGetErrorString(r1), cudaGetErrorString(r2),
         cudaGetErrorString(r3), cudaGetErrorString(r4), h);
  cudaGetLastError();
}
int main() {
  int *out; cudaMalloc(&out, 4);
  probe<64>(out); probe<2048>(out); probe<4096>(out); probe<4100>(out); probe<8704>(out); probe<16384>(out);
  return 0;
}
