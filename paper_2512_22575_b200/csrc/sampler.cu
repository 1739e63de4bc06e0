// On-device perturbation sampler (sm_100a).
// Replaces vp/planner.py:182-219 (smoothing_matrix, sample_perturbations) --
// SURVEY.md section 8f row 1.  One warp per (sample, 32-step chunk), lane =
// step, drawing exactly what the fused SMPC kernel draws in registers for the
// same candidate (noise.cuh), and writing it as an (M, H, n) buffer for the
// API paths that take perturbations (evaluate, the multi-device partial, the
// runtime-topology kernels).
#include "noise.cuh"

namespace vpb {

struct SamplerArgs {
  NoiseGen gen;
  int64_t M, H, n;
  void *out;
};

template <int NJ, int HALF, typename OT>
__global__ void __launch_bounds__(256) sampler_kernel(const __grid_constant__ SamplerArgs A) {
  const int lane = threadIdx.x & 31;
  const int H = (int)A.H, n = (int)A.n;
  const int nch = (H + 31) >> 5;
  const int64_t wg = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wg >= A.M * nch) return;  // warp-uniform
  const int64_t m = wg / nch;
  const int ch = (int)(wg - m * nch);
  float u[NJ];
  candidate_noise<NJ, HALF>(A.gen, m, H, ch, lane, u);
  const int k = 32 * ch + lane;
  if (k >= H) return;
  OT *o = reinterpret_cast<OT *>(A.out) + ((size_t)m * H + k) * n;
#pragma unroll
  for (int j = 0; j < NJ; ++j)
    if (j < n) o[j] = (OT)u[j];
}

template <int NJ, int HALF>
static void launch_sampler(const SamplerArgs &A, int dtype, unsigned grid, cudaStream_t s) {
  if (dtype == VPB_DTYPE_F32)
    sampler_kernel<NJ, HALF, float><<<grid, 256, 0, s>>>(A);
  else
    sampler_kernel<NJ, HALF, double><<<grid, 256, 0, s>>>(A);
}

}  // namespace vpb

using namespace vpb;

extern "C" int vpb_sample_perturbations(uint64_t seed, const uint64_t *seed_dev, int64_t m_offset, int64_t M,
                                        int64_t H, int64_t n, int64_t window, const double *sigma, int dtype,
                                        void *out, void *stream) {
  VPB_REQUIRE(out && sigma && M >= 0 && H >= 1 && n >= 1 && n <= VPB_MAX_JOINTS && m_offset >= 0,
              "bad arguments to vpb_sample_perturbations");
  VPB_REQUIRE(dtype == VPB_DTYPE_F32 || dtype == VPB_DTYPE_F64, "bad dtype");
  VPB_REQUIRE(window >= 1 && window <= 9, "noise window must be in [1, 9]");
  if (M == 0) return VPB_OK;
  SamplerArgs A;
  memset(&A, 0, sizeof(A));
  A.gen.seed = seed;
  A.gen.seed_dev = seed_dev;
  A.gen.m_offset = m_offset;
  A.gen.window = (int)window;
  for (int64_t j = 0; j < n; ++j) A.gen.sigma[j] = (float)sigma[j];
  A.M = M;
  A.H = H;
  A.n = n;
  A.out = out;
  const int64_t warps = M * ((H + 31) / 32);
  const unsigned grid = (unsigned)ceil_div(warps, 8);
  cudaStream_t s = as_stream(stream);
  const bool half2 = window <= 5;
  if (n == 7)
    half2 ? launch_sampler<7, 2>(A, dtype, grid, s) : launch_sampler<7, 4>(A, dtype, grid, s);
  else
    half2 ? launch_sampler<16, 2>(A, dtype, grid, s) : launch_sampler<16, 4>(A, dtype, grid, s);
  return check_launch("sampler_kernel");
}
