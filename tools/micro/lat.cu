// Latency micro-benchmarks on B200 (calibration for the SMPC merge chain).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ long long ck() { return clock64(); }

__global__ void chain(const int *next, int steps, long long *out, double *dout) {
  // pointer chase: dependent global loads
  int i = 0;
  long long c0 = ck();
  for (int s = 0; s < steps; ++s) i = __ldcg(next + i);
  long long c1 = ck();
  out[0] = (c1 - c0) / steps;
  out[1] = i;
  // exp double
  double x = dout[0];
  c0 = ck();
  for (int s = 0; s < 64; ++s) x = exp(-x / 0.05) + 0.5;
  c1 = ck();
  out[2] = (c1 - c0) / 64;
  dout[1] = x;
  // atomic round trip
  unsigned int *cnt = reinterpret_cast<unsigned int *>(dout + 8);
  c0 = ck();
  unsigned int a = 0;
  for (int s = 0; s < 16; ++s) a += atomicAdd(cnt, a & 1);
  c1 = ck();
  out[3] = (c1 - c0) / 16;
  // fence
  c0 = ck();
  for (int s = 0; s < 16; ++s) { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
  c1 = ck();
  out[4] = (c1 - c0) / 16;
  c0 = ck();
  for (int s = 0; s < 16; ++s) __threadfence();
  c1 = ck();
  out[5] = (c1 - c0) / 16;
  out[6] = a;
}

__global__ void bar_lat(long long *out) {
  long long c0 = ck();
  for (int s = 0; s < 64; ++s) __syncthreads();
  long long c1 = ck();
  if (threadIdx.x == 0) out[7] = (c1 - c0) / 64;
}

int main() {
  const int N = 1 << 22;  // 16 MB of indices: L2 resident
  int *h = new int[N];
  // random cycle with stride to defeat L1
  for (int i = 0; i < N; ++i) h[i] = (int)(((long long)i * 2654435761LL + 12345) % N);
  int *d; cudaMalloc(&d, N * 4); cudaMemcpy(d, h, N * 4, cudaMemcpyHostToDevice);
  long long *o; cudaMalloc(&o, 64 * 8); double *dd; cudaMalloc(&dd, 64 * 8); cudaMemset(dd, 0, 64 * 8);
  for (int rep = 0; rep < 3; ++rep) {
    chain<<<1, 1>>>(d, 256, o, dd);
    bar_lat<<<1, 128>>>(o);
    cudaDeviceSynchronize();
  }
  long long r[8]; cudaMemcpy(r, o, 64, cudaMemcpyDeviceToHost);
  printf("{\"dep_load_l2_cycles\": %lld, \"exp_f64_cycles\": %lld, \"atomic_rt_cycles\": %lld, \"fence_acq_rel_cycles\": %lld, \"threadfence_cycles\": %lld, \"syncthreads128_cycles\": %lld}\n",
         r[0], r[2], r[3], r[4], r[5], r[7]);
  return 0;
}
