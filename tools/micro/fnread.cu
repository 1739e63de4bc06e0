// Can a kernel read (and L2-prefetch) its own code through a function pointer?
#include <cstdio>
#include <cstdint>
__device__ __noinline__ float target_fn(float x) { return x * 3.0f + __sinf(x); }
__global__ void probe(unsigned long long *out, float x) {
  float (*fp)(float) = &target_fn;
  unsigned long long a;
  asm volatile("mov.b64 %0, %1;" : "=l"(a) : "l"((unsigned long long)fp));
  out[0] = a;
  asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
  const unsigned long long *p = reinterpret_cast<const unsigned long long *>(a);
  out[1] = p[0];
  out[2] = p[1];
  out[3] = __float_as_uint(fp(x));
}
int main() {
  unsigned long long *d, h[4] = {0, 0, 0, 0};
  cudaMalloc(&d, 32);
  probe<<<1, 1>>>(d, 1.0f);
  cudaError_t e = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(e));
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("addr %llx w0 %016llx w1 %016llx\n", h[0], h[1], h[2]);
  return 0;
}
