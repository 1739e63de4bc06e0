// Softmin weights and the weighted-mean control update as standalone device
// reductions (sm_100a).  Replaces vp/planner.py:373-384 (soft_weights) and
// vp/planner.py:387-400 (update_controls); the SMPC step itself uses the fused
// per-CTA partials of rollout.cu.  All reductions run in a fixed order, so
// results are bitwise reproducible.
#include "vpb_common.cuh"

namespace vpb {

// Soft weights: w_m = exp(-(S_m - min)/lam) / Z with min/Z from a merged
// partial-style reduction over the raw costs.
__global__ void __launch_bounds__(256) cost_min_kernel(const double *__restrict__ costs, int64_t M,
                                                       int64_t chunk, double *__restrict__ out_min,
                                                       int *__restrict__ out_nonfinite) {
  __shared__ double red[256];
  __shared__ int nf[256];
  const int64_t b0 = (int64_t)blockIdx.x * chunk;
  const int64_t e0 = vmin64(b0 + chunk, M);
  double mn = __longlong_as_double(0x7ff0000000000000ll);
  int bad = 0;
  for (int64_t i = b0 + threadIdx.x; i < e0; i += blockDim.x) {
    const double c = costs[i];
    if (!isfinite(c)) ++bad;
    else mn = fmin(mn, c);
  }
  red[threadIdx.x] = mn;
  nf[threadIdx.x] = bad;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + s]);
      nf[threadIdx.x] += nf[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out_min[blockIdx.x] = red[0];
    out_nonfinite[blockIdx.x] = nf[0];
  }
}

__global__ void __launch_bounds__(256) soft_weights_kernel(const double *__restrict__ costs, int64_t M,
                                                           const double *__restrict__ block_min,
                                                           const int *__restrict__ block_nf, int64_t nblocks,
                                                           double lam, double *__restrict__ w,
                                                           double *__restrict__ block_sum) {
  __shared__ double red[256];
  __shared__ double mn_s;
  if (threadIdx.x == 0) {
    double mn = __longlong_as_double(0x7ff0000000000000ll);
    for (int64_t b = 0; b < nblocks; ++b) mn = fmin(mn, block_min[b]);
    mn_s = mn;
  }
  __syncthreads();
  const double mn = mn_s;
  const int64_t chunk = (M + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * chunk;
  const int64_t e0 = vmin64(b0 + chunk, M);
  double acc = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < e0; i += blockDim.x) {
    const double v = exp(-(costs[i] - mn) / lam);
    w[i] = v;
    acc += v;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) block_sum[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) normalize_kernel(double *__restrict__ w, int64_t M,
                                                        const double *__restrict__ block_sum, int64_t nblocks,
                                                        const double *__restrict__ block_min,
                                                        const int *__restrict__ block_nf, int64_t nmin,
                                                        double *__restrict__ stats) {
  __shared__ double Z_s;
  if (threadIdx.x == 0) {
    double Z = 0.0;
    for (int64_t b = 0; b < nblocks; ++b) Z += block_sum[b];
    Z_s = Z;
    if (blockIdx.x == 0 && stats) {
      double mn = __longlong_as_double(0x7ff0000000000000ll);
      int nf = 0;
      for (int64_t b = 0; b < nmin; ++b) {
        mn = fmin(mn, block_min[b]);
        nf += block_nf[b];
      }
      stats[0] = mn;
      stats[1] = Z;
      stats[2] = (double)nf;
    }
  }
  __syncthreads();
  const double Z = Z_s;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = w[i] / Z;
}

// update_controls: out[e] = nominal[e] + sum_m w_m eps[m][e]; fixed order
// over m inside fixed chunks, chunks summed in order by the second kernel.
template <typename ET>
__global__ void __launch_bounds__(256) wsum_partial_kernel(const ET *__restrict__ eps,
                                                           const double *__restrict__ w, int64_t M,
                                                           int64_t hn, int64_t chunk,
                                                           double *__restrict__ partial) {
  const int64_t c = blockIdx.y;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= hn) return;
  const int64_t m0 = c * chunk, m1 = vmin64(m0 + chunk, M);
  double acc = 0.0;
  for (int64_t m = m0; m < m1; ++m) acc += w[m] * (double)eps[m * hn + e];
  partial[c * hn + e] = acc;
}

__global__ void __launch_bounds__(256) wsum_final_kernel(const double *__restrict__ partial, int64_t nchunks,
                                                         const double *__restrict__ nominal, int64_t hn,
                                                         double *__restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= hn) return;
  double acc = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) acc += partial[c * hn + e];
  out[e] = nominal[e] + acc;
}

}  // namespace vpb

using namespace vpb;

extern "C" {

size_t vpb_soft_weights_workspace_bytes(int64_t M) {
  const int64_t nb = ceil_div(M > 0 ? M : 1, 4096) + 1;
  return align_up(nb * 8, 256) * 2 + align_up(nb * 4, 256) + 1024;
}

int vpb_soft_weights(const double *costs, int64_t M, double lam, double *weights, double *stats, void *workspace,
                     size_t workspace_bytes, void *stream) {
  VPB_REQUIRE(costs && weights && M >= 1, "bad arguments to vpb_soft_weights");
  VPB_REQUIRE(lam > 0.0, "temperature must be positive");
  VPB_REQUIRE(workspace && workspace_bytes >= vpb_soft_weights_workspace_bytes(M), "workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t chunk = 4096;
  const int64_t nb = ceil_div(M, chunk);
  char *ws = reinterpret_cast<char *>(workspace);
  double *bmin = reinterpret_cast<double *>(ws);
  double *bsum = reinterpret_cast<double *>(ws + align_up((nb + 1) * 8, 256));
  int *bnf = reinterpret_cast<int *>(ws + 2 * align_up((nb + 1) * 8, 256));
  cost_min_kernel<<<(unsigned)nb, 256, 0, s>>>(costs, M, chunk, bmin, bnf);
  int rc = check_launch("cost_min_kernel");
  if (rc) return rc;
  soft_weights_kernel<<<(unsigned)nb, 256, 0, s>>>(costs, M, bmin, bnf, nb, lam, weights, bsum);
  rc = check_launch("soft_weights_kernel");
  if (rc) return rc;
  normalize_kernel<<<(unsigned)vmin64(ceil_div(M, 256), 1184), 256, 0, s>>>(weights, M, bsum, nb, bmin, bnf,
                                                                                   nb, stats);
  return check_launch("normalize_kernel");
}

size_t vpb_update_controls_workspace_bytes(int64_t M, int64_t hn) {
  const int64_t chunks = ceil_div(M > 0 ? M : 1, 256);
  return align_up((size_t)chunks * hn * 8, 256);
}

int vpb_update_controls(const double *nominal, const void *eps, int dtype, const double *weights, int64_t M,
                        int64_t hn, double *out, void *workspace, size_t workspace_bytes, void *stream) {
  VPB_REQUIRE(nominal && eps && weights && out && M >= 1 && hn >= 1, "bad arguments to vpb_update_controls");
  VPB_REQUIRE(workspace && workspace_bytes >= vpb_update_controls_workspace_bytes(M, hn), "workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t chunk = 256, chunks = ceil_div(M, chunk);
  double *partial = reinterpret_cast<double *>(workspace);
  dim3 g((unsigned)ceil_div(hn, 256), (unsigned)chunks);
  if (dtype == VPB_DTYPE_F32)
    wsum_partial_kernel<float><<<g, 256, 0, s>>>(reinterpret_cast<const float *>(eps), weights, M, hn, chunk, partial);
  else
    wsum_partial_kernel<double><<<g, 256, 0, s>>>(reinterpret_cast<const double *>(eps), weights, M, hn, chunk,
                                                  partial);
  int rc = check_launch("wsum_partial_kernel");
  if (rc) return rc;
  wsum_final_kernel<<<(unsigned)ceil_div(hn, 256), 256, 0, s>>>(partial, chunks, nominal, hn, out);
  return check_launch("wsum_final_kernel");
}

}  // extern "C"
