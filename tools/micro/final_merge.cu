// Stand-alone timing of final_merge (tools/micro): 1024 CTA heads, one nonzero weight.
#include <cstdio>
#include <cmath>
#include <cstring>
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
template <typename ET> __device__ __forceinline__ double load_e(const ET *p) { return (double)__ldg(p); }
struct Shared { double *misc; };
struct SmpcIO { const void *eps; int64_t M; double lam; double *group_parts; double *rank_part; };
template <typename ET, int NWC>
__device__ void final_merge(const SmpcIO &io, const Shared &S, const double *heads, const double *costs, int ctas,
                            int hn, unsigned long long *trace_head) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double *misc = S.misc;
  double *wlist = io.group_parts;                                  // candidate weights (scratch)
  int *mlist = reinterpret_cast<int *>(io.group_parts + io.M + 64);  // candidate indices
  int *clist = reinterpret_cast<int *>(io.group_parts + io.M + 64) + io.M + 64;  // nonzero CTAs, per-warp slices
  const double inv_lam = 1.0 / io.lam;
  // 1. global minimum over the CTA heads (first CTA attaining it)
  constexpr int kHR = 8;  // heads kept in registers per lane (ctas <= nw * 32 * kHR)
  const int span = ((ctas + nw - 1) / nw + 31) & ~31;
  const int w0 = warp * span, w1 = min(ctas, w0 + span);
  const bool in_regs = span <= 32 * kHR;
  double hv[kHR];
  double mn = dinf();
  int bidx = 0x7fffffff;
  double nf = 0.0;
  if (in_regs) {
    double fv[kHR];
#pragma unroll
    for (int t = 0; t < kHR; ++t) {
      const int i = w0 + 32 * t + lane;
      hv[t] = i < w1 ? heads[i] : dinf();
      fv[t] = i < w1 ? heads[ctas + i] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < kHR; ++t) {
      nf += fv[t];
      if (hv[t] < mn) {
        mn = hv[t];
        bidx = w0 + 32 * t + lane;
      }
    }
  } else {
    for (int c = w0; c < w1; c += 32 * 4) {
      double v[4], f[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = c + 32 * t + lane;
        v[t] = i < w1 ? heads[i] : dinf();
        f[t] = i < w1 ? heads[ctas + i] : 0.0;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        nf += f[t];
        if (v[t] < mn) {
          mn = v[t];
          bidx = c + 32 * t + lane;
        }
      }
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
  nf = warp_sum_d(nf);
  if (lane == 0) {
    misc[warp] = mn;
    misc[16 + warp] = (double)bidx;
    misc[32 + warp] = nf;
  }
  __syncthreads();
  if (tid == 0) {
    double m0 = dinf(), NF = 0.0;
    int b0 = 0x7fffffff;
    for (int w = 0; w < nw; ++w) {
      const double v = misc[w];
      const int b = (int)misc[16 + w];
      NF += misc[32 + w];
      if (v < m0 || (v == m0 && b < b0)) {
        m0 = v;
        b0 = b;
      }
    }
    misc[40] = m0;
    misc[41] = (double)b0;
    misc[43] = NF;
  }
  __syncthreads();
  const double m0 = misc[40];
  // 2. (all warps) CTAs with a nonzero weight, compacted in order into this
  //    warp's slice of clist (cheap exponent pre-check; exp only near the min)
  int wn = 0;
  auto consider = [&](int i, double v) {
    const double x = (v - m0) * inv_lam;
    const bool nz = v < dinf() && x < 746.0 && exp(-x) != 0.0;
    const unsigned bal = __ballot_sync(kFull, nz);
    if (nz) clist[w0 + wn + __popc(bal & ((1u << lane) - 1u))] = i;
    wn += __popc(bal);
  };
  if (in_regs) {
#pragma unroll
    for (int t = 0; t < kHR; ++t) consider(w0 + 32 * t + lane, hv[t]);
  } else {
    for (int c = w0; c < w1; c += 32) {
      const int i = c + lane;
      consider(i, i < w1 ? heads[i] : dinf());
    }
  }
  if (lane == 0) misc[16 + warp] = (double)wn;
  __syncthreads();
  if (tid < 32) {
    // 3. (warp 0) the candidates of those CTAs, in order: weights and Z
    // candidates of the nonzero CTAs over the concatenated warp slices, 32
    // at a time: one load round trip per 32 candidates
    int off[16];
    int total = 0;
    for (int w = 0; w < nw; ++w) {
      off[w] = total;
      total += (int)misc[16 + w] * NWC;
    }
    int ncand = 0;
    double z = 0.0;
    for (int k0 = 0; k0 < total; k0 += 32) {
      const int k = k0 + lane;
      int m = -1;
      double wt = 0.0;
      if (k < total) {
        int w = 0;
        for (int u = 1; u < nw; ++u)
          if (k >= off[u]) w = u;
        const int r = k - off[w];
        m = clist[w * span + r / NWC] * NWC + (r % NWC);
        if (m < io.M) {
          const double c = costs[m];
          wt = c < dinf() ? exp(-(c - m0) * inv_lam) : 0.0;
        }
      }
      const unsigned bal = __ballot_sync(kFull, wt != 0.0);
      if (wt != 0.0) {
        const int p = ncand + __popc(bal & ((1u << lane) - 1u));
        mlist[p] = m;
        wlist[p] = wt;
      }
      z += wt;  // lane-strided partials in candidate order
      ncand += __popc(bal);
    }
    z = warp_sum_d(z);
    if (lane == 0) {
      const int b0 = (int)misc[41];
      double *dst = io.rank_part;
      dst[0] = m0;
      dst[1] = z;
      dst[2] = misc[43];
      dst[3] = (b0 >= 0 && b0 < ctas) ? heads[2 * (size_t)ctas + b0] : -1.0;
      misc[42] = (double)ncand;
      misc[45] = ncand == 1 ? (double)mlist[0] : -1.0;  // the only nonzero weight (U* = nominal + its eps)
    }
  }
  __syncthreads();
  if (trace_head && tid == 0) *trace_head = gtimer();
  // 3. N = sum_m w_m eps_m over the nonzero candidates, in candidate order
  const int ncand = (int)misc[42];
  const ET *eps = reinterpret_cast<const ET *>(io.eps);
  for (int e = tid; e < hn; e += nt) {
    double acc = 0.0;
    int k = 0;
    for (; k + 4 <= ncand; k += 4) {
      double a[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = load_e<ET>(eps + (size_t)mlist[k + t] * hn + e);
#pragma unroll
      for (int t = 0; t < 4; ++t) acc += wlist[k + t] * a[t];
    }
    for (; k < ncand; ++k) acc += wlist[k] * load_e<ET>(eps + (size_t)mlist[k] * hn + e);
    io.rank_part[kPartHead + e] = acc;
  }
  __syncthreads();
}


__global__ void k(SmpcIO io, const double *heads, const double *costs, int ctas, int hn, long long *cyc, unsigned long long *tr) {
  __shared__ double misc[48];
  Shared S{misc};
  long long c0 = clock64();
  final_merge<float, 4>(io, S, heads, costs, ctas, hn, tr);
  long long c1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = c1 - c0; cyc[1] = (long long)(tr[0]) - c0; }
}
int main() {
  const int ctas = 1024, M = 4096, hn = 224;
  double *hh = new double[3 * ctas], *hc = new double[M];
  for (int i = 0; i < ctas; ++i) { hh[i] = 3000.0 + 37.0 * ((i * 7919) % ctas); hh[ctas + i] = 0; hh[2 * ctas + i] = 4 * i; }
  for (int m = 0; m < M; ++m) hc[m] = hh[m / 4] + (m % 4);
  double *dh, *dc, *gp, *rp; float *eps; long long *cyc; unsigned long long *tr;
  cudaMalloc(&dh, 3 * ctas * 8); cudaMemcpy(dh, hh, 3 * ctas * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&dc, M * 8); cudaMemcpy(dc, hc, M * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&gp, (3 * M + 4096) * 8); cudaMalloc(&rp, (hn + 8) * 8); cudaMalloc(&eps, (size_t)M * hn * 4);
  cudaMemset(eps, 0, (size_t)M * hn * 4); cudaMalloc(&cyc, 64); cudaMalloc(&tr, 64);
  SmpcIO io{eps, M, 0.05, gp, rp};
  for (int rep = 0; rep < 5; ++rep) k<<<1, 128>>>(io, dh, dc, ctas, hn, cyc, tr);
  cudaDeviceSynchronize();
  long long c[2]; cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
  printf("{\"final_merge_cycles\": %lld, \"head_cycles\": %lld, \"err\": \"%s\"}\n", c[0], c[1], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
