// Stand-alone timing of merge_block (tools/micro): 1024 partial rows.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
constexpr unsigned kFull = 0xffffffffu;
constexpr int kPartHead = 4;
__device__ __forceinline__ unsigned long long gtimer() { return (unsigned long long)clock64(); }
__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000ll); }
__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
  return x;
}
__device__ __forceinline__ double4 load_head(const double *row) {
  return make_double4(row[0], row[1], row[2], row[3]);
}

__device__ void merge_block(const double *src, int count, int hn, double lam, double *dst, double *scratch,
                            double *misc, unsigned long long *trace_head = nullptr) {
  // Merge `count` partial rows [m, Z, nonfinite, best, N (hn)] (row stride
  // kPartHead + hn) in row order.  Thread t owns rows [t r, t r + r):
  //   1. min and the first row attaining it (thread-local, warp shuffles,
  //      warps in order);
  //   2. scale_i = exp(-(m_i - min) / lam), Z = sum scale_i Z_i, non-finite
  //      count (thread-local in row order, then a fixed tree);
  //   3. rows with scale 0 (exp underflow: far above the minimum -- most of
  //      them at the planner's lam) are dropped by an order-preserving
  //      compaction, and N = sum scale_i N_i runs over the rest with all of a
  //      thread's row loads in flight.
  // scratch: >= 2 * max(count, 32) + 24 doubles; misc: >= 48 doubles.
  const int L = kPartHead + hn;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  if (trace_head && tid == 0) trace_head[3] = gtimer();
  const int r = (count + nt - 1) / nt;
  const int i0 = tid * r, i1 = min(count, i0 + r);
  // heads of this thread's rows, kR rows per batch with all loads in flight
  constexpr int kR = 8;
  const bool one_batch = r <= kR;
  double hm[kR], hz[kR], hf[kR];
  double mn = dinf();
  int bidx = 0x7fffffff;
  for (int b0 = i0; b0 < i1; b0 += kR) {
#pragma unroll
    for (int t = 0; t < kR; ++t) {
      const int i = b0 + t;
      const bool ok = i < i1;
      const double *row = src + (size_t)(ok ? i : 0) * L;  // row 0 always exists
      hm[t] = ok ? row[0] : dinf();
      hz[t] = ok ? row[1] : 0.0;
      hf[t] = ok ? row[2] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < kR; ++t)
      if (hm[t] < mn) {  // rows ascend: the first minimum wins
        mn = hm[t];
        bidx = b0 + t;
      }
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    const double ov = __shfl_xor_sync(kFull, mn, d);
    const int oi = __shfl_xor_sync(kFull, bidx, d);
    if (ov < mn || (ov == mn && oi < bidx)) {
      mn = ov;
      bidx = oi;
    }
  }
  if (lane == 0) {
    misc[warp] = mn;
    misc[16 + warp] = (double)bidx;
  }
  if (trace_head && tid == 0) trace_head[1] = gtimer();
  __syncthreads();
  if (tid == 0) {
    double m0 = dinf();
    int b0 = 0x7fffffff;
    for (int w = 0; w < nw; ++w) {
      const double v = misc[w];
      const int b = (int)misc[16 + w];
      if (v < m0 || (v == m0 && b < b0)) {
        m0 = v;
        b0 = b;
      }
    }
    misc[40] = m0;
    misc[41] = (double)b0;
  }
  __syncthreads();
  mn = misc[40];
  bidx = (int)misc[41];
  if (trace_head && tid == 0) trace_head[4] = gtimer();
  // scales, Z, non-finite count, per-thread nonzero count (row order)
  double z = 0.0, nf = 0.0;
  int nz = 0;
  double sc_r[kR];
#pragma unroll
  for (int t = 0; t < kR; ++t) sc_r[t] = 0.0;  // threads without rows keep zeros
  for (int b0 = i0; b0 < i1; b0 += kR) {
    if (!one_batch) {
#pragma unroll
      for (int t = 0; t < kR; ++t) {
        const int i = b0 + t;
        const bool ok = i < i1;
        const double *row = src + (size_t)(ok ? i : 0) * L;  // row 0 always exists
        hm[t] = ok ? row[0] : dinf();
        hz[t] = ok ? row[1] : 0.0;
        hf[t] = ok ? row[2] : 0.0;
      }
    }
#pragma unroll
    for (int t = 0; t < kR; ++t) {
      const double sc = (hm[t] < dinf()) ? exp(-(hm[t] - mn) / lam) : 0.0;
      sc_r[t] = sc;
      if (sc != 0.0) {
        z += sc * hz[t];
        ++nz;
      }
      nf += hf[t];
    }
  }
  if (trace_head && tid == 0) trace_head[5] = gtimer();
  // order-preserving compaction offsets: exclusive scan of nz over threads
  int inc = nz;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc += y;
  }
  const double zw = warp_sum_d(z), nfw = warp_sum_d(nf);
  if (lane == 31) misc[16 + warp] = (double)inc;  // warp totals (misc[16..32), free again)
  if (lane == 0) misc[32 + warp] = zw;
  __syncthreads();
  int woff = 0;
  for (int w = 0; w < warp; ++w) woff += (int)misc[16 + w];
  const int cmax = count > 32 ? count : 32;
  int *rows = reinterpret_cast<int *>(scratch + cmax);
  double *scale = scratch;
  int pos = woff + inc - nz;
  if (one_batch) {
#pragma unroll
    for (int t = 0; t < kR; ++t)
      if (i0 + t < i1 && sc_r[t] != 0.0) {
        rows[pos] = i0 + t;
        scale[pos] = sc_r[t];
        ++pos;
      }
  } else {
    for (int i = i0; i < i1; ++i) {
      const double v = src[(size_t)i * L];
      const double sc = (v < dinf()) ? exp(-(v - mn) / lam) : 0.0;
      if (sc != 0.0) {
        rows[pos] = i;
        scale[pos] = sc;
        ++pos;
      }
    }
  }
  if (trace_head && tid == 0) trace_head[2] = gtimer();
  // nonfinite: fixed tree via the same warp sums
  if (lane == 0) scratch[2 * cmax + 4 + warp] = nfw;
  __syncthreads();
  if (tid == 0) {
    double Z = 0.0, NF = 0.0;
    int nnz = 0;
    for (int w = 0; w < nw; ++w) {
      Z += misc[32 + w];
      NF += scratch[2 * cmax + 4 + w];
      nnz += (int)misc[16 + w];
    }
    dst[0] = mn;
    dst[1] = Z;
    dst[2] = NF;
    dst[3] = (bidx >= 0 && bidx < count) ? src[(size_t)bidx * L + 3] : -1.0;
    misc[42] = (double)nnz;
  }
  __syncthreads();
  if (trace_head && tid == 0) *trace_head = gtimer();
  const int nnz = (int)misc[42];
  for (int e = tid; e < hn; e += nt) {
    const double *col = src + kPartHead + e;
    double acc = 0.0;
    int i = 0;
    for (; i + 4 <= nnz; i += 4) {
      double a[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = col[(size_t)rows[i + t] * L];
#pragma unroll
      for (int t = 0; t < 4; ++t) acc += scale[i + t] * a[t];
    }
    for (; i < nnz; ++i) acc += scale[i] * col[(size_t)rows[i] * L];
    dst[kPartHead + e] = acc;
  }
  __syncthreads();
}


__global__ void k(const double *src, int count, int hn, double lam, double *dst, double *scratch, long long *cyc, unsigned long long *tr) {
  __shared__ double misc[48];
  long long c0 = clock64();
  merge_block(src, count, hn, lam, dst, scratch, misc, tr);
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}
int main() {
  const int count = 1024, hn = 224, L = kPartHead + hn;
  double *h = new double[(size_t)count * L];
  for (int i = 0; i < count; ++i) {
    h[(size_t)i * L + 0] = 1000.0 + 37.0 * ((i * 7919) % count);  // one clear minimum
    h[(size_t)i * L + 1] = 1.0; h[(size_t)i * L + 2] = 0.0; h[(size_t)i * L + 3] = i;
    for (int e = 0; e < hn; ++e) h[(size_t)i * L + 4 + e] = 0.001 * e;
  }
  double *d, *dst, *scr; long long *cyc; unsigned long long *tr;
  cudaMalloc(&d, (size_t)count * L * 8); cudaMemcpy(d, h, (size_t)count * L * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&dst, L * 8); cudaMalloc(&scr, (2 * count + 24) * 8); cudaMalloc(&cyc, 64); cudaMalloc(&tr, 64);
  for (int nt : {128, 256, 512}) {
    for (int rep = 0; rep < 4; ++rep) k<<<1, nt>>>(d, count, hn, 0.05, dst, scr, cyc, tr);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    unsigned long long t[6]; cudaMemcpy(t, tr, 48, cudaMemcpyDeviceToHost);
    printf("{\"threads\": %d, \"merge_cycles\": %lld, \"load+warp_argmin\": %lld, \"block_argmin\": %lld, \"scales\": %lld, \"compaction\": %lld, \"N\": %lld}\n", nt, c,
           (long long)(t[1] - t[3]), (long long)(t[4] - t[1]), (long long)(t[5] - t[4]), (long long)(t[2] - t[5]), (long long)(t[0] - t[2]));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
