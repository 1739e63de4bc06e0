// Launch-overhead micro-benchmark (tools/micro): CUDA-event time of a trivial
// kernel vs parameter-block size, grid size and dynamic shared memory, direct
// and graph-replayed, with and without an L2 flush before each launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch launch.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int BYTES>
struct Blob {
  int v[BYTES / 4];
};

template <int BYTES>
__global__ void touch(const __grid_constant__ Blob<BYTES> b, int *out) {
  if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) out[0] = b.v[BYTES / 4 - 1];
}

__global__ void flush_k(unsigned char *p, size_t n, int v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 16; i += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<int4 *>(p)[i] = make_int4(v, v, v, v);
}

template <int BYTES>
float run(int grid, int threads, int smem, bool graph, bool flush, unsigned char *fl, size_t fn, int *out) {
  Blob<BYTES> b{};
  b.v[BYTES / 4 - 1] = 7;
  cudaFuncSetAttribute(touch<BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    touch<BYTES><<<grid, threads, smem, s>>>(b, out);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float tot = 0;
  const int iters = 50;
  for (int it = -5; it < iters; ++it) {
    if (flush) flush_k<<<592, 512, 0, s>>>(fl, fn, it);
    cudaEventRecord(e0, s);
    if (graph) cudaGraphLaunch(ge, s);
    else touch<BYTES><<<grid, threads, smem, s>>>(b, out);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 0) tot += ms;
  }
  cudaStreamDestroy(s);
  return tot / iters * 1000.0f;
}

int main() {
  int *out;
  cudaMalloc(&out, 64);
  size_t fn = 256u << 20;
  unsigned char *fl;
  cudaMalloc(&fl, fn);
  for (int flush = 0; flush < 2; ++flush)
    for (int graph = 0; graph < 2; ++graph) {
      printf("flush=%d graph=%d\n", flush, graph);
      printf("  1 CTA      64 B : %6.2f us\n", run<64>(1, 128, 0, graph, flush, fl, fn, out));
      printf("  1 CTA    8704 B : %6.2f us\n", run<8704>(1, 128, 0, graph, flush, fl, fn, out));
      printf("  1025 CTA   64 B : %6.2f us\n", run<64>(1025, 128, 6144, graph, flush, fl, fn, out));
      printf("  1025 CTA 4096 B : %6.2f us\n", run<4096>(1025, 128, 6144, graph, flush, fl, fn, out));
      printf("  1025 CTA 8704 B : %6.2f us\n", run<8704>(1025, 128, 6144, graph, flush, fl, fn, out));
      printf("  148 CTA  8704 B : %6.2f us\n", run<8704>(148, 128, 6144, graph, flush, fl, fn, out));
    }
  return 0;
}
