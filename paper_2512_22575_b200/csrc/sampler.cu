// On-device perturbation sampler (sm_100a).
// Replaces vp/planner.py:182-219 (smoothing_matrix, sample_perturbations) --
// SURVEY.md section 8f row 1.  Same structure: one counter-based stream per
// sample keyed by (seed, global sample index), standard normals, moving-
// average smoothing over the horizon with rows scaled to unit L2 norm, times
// the per-joint sigma, sample 0 reserved as the zero perturbation.  The
// generator is Philox4x32-10 + Box-Muller, so the draws are statistically
// (not bitwise) equivalent to numpy's Philox4x64 + ziggurat stream; the
// reference's own sampler tests are statistical (t/test_planner.py:52-90).
#include "vpb_common.cuh"

namespace vpb {

struct SamplerArgs {
  uint64_t seed;
  const uint64_t *seed_dev;  // optional: seed read from device memory (graph replays)
  int64_t m_offset, M, H, n, window;
  double sigma[VPB_MAX_JOINTS];
  void *out;
  int dtype;
};

__device__ __forceinline__ void philox_round(uint32_t &c0, uint32_t &c1, uint32_t &c2, uint32_t &c3, uint32_t k0,
                                             uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
  const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
  const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
  c0 = n0;
  c1 = n1;
  c2 = n2;
  c3 = n3;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint32_t k0, uint32_t k1) {
  uint32_t c0 = ctr.x, c1 = ctr.y, c2 = ctr.z, c3 = ctr.w;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c0, c1, c2, c3, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ void box_muller_f(uint32_t a, uint32_t b, float &z0, float &z1) {
  const float u1 = ((float)(a >> 8) + 0.5f) * 5.9604644775390625e-08f;  // (0,1), 24-bit
  const float u2 = ((float)(b >> 8) + 0.5f) * 5.9604644775390625e-08f;
  const float r = sqrtf(-2.0f * logf(u1));
  float s, c;
  sincospif(2.0f * u2, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, double &z0, double &z1) {
  const double u1 = ((double)a + 0.5) * 2.3283064365386963e-10;  // (0,1)
  const double u2 = ((double)b + 0.5) * 2.3283064365386963e-10;
  const double r = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// One warp per sample; raw normals staged in shared memory, then smoothed.
__global__ void __launch_bounds__(256) sampler_kernel(const __grid_constant__ SamplerArgs A) {
  extern __shared__ double raw[];  // [8][H*n]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t mloc = (int64_t)blockIdx.x * 8 + warp;
  const int64_t hn = A.H * A.n;
  double *r = raw + (size_t)warp * hn;
  if (mloc >= A.M) return;
  const int64_t mg = A.m_offset + mloc;
  const uint64_t seed = A.seed_dev ? *A.seed_dev : A.seed;
  const uint32_t k0 = (uint32_t)seed ^ (uint32_t)((uint64_t)mg * 0x9E3779B97F4A7C15ull);
  const uint32_t k1 = (uint32_t)(seed >> 32) ^ (uint32_t)((uint64_t)mg >> 32) ^ 0x85EBCA6Bu;
  const int64_t ncalls = (hn + 3) / 4;
  for (int64_t c = lane; c < ncalls; c += 32) {
    const uint4 x = philox4x32_10(make_uint4((uint32_t)c, (uint32_t)mg, (uint32_t)(mg >> 32), 0x5eedu), k0, k1);
    double z[4];
    if (A.dtype == VPB_DTYPE_F32) {
      float f[4];
      box_muller_f(x.x, x.y, f[0], f[1]);
      box_muller_f(x.z, x.w, f[2], f[3]);
#pragma unroll
      for (int t = 0; t < 4; ++t) z[t] = f[t];
    } else {
      box_muller(x.x, x.y, z[0], z[1]);
      box_muller(x.z, x.w, z[2], z[3]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (4 * c + t < hn) r[4 * c + t] = z[t];
  }
  __syncwarp();
  const int64_t back = (A.window - 1) / 2, fwd = A.window / 2;
  const bool smooth = A.window > 1;
  for (int64_t e = lane; e < hn; e += 32) {
    const int64_t h = e / A.n, j = e - h * A.n;
    double v;
    if (mg == 0) {
      v = 0.0;
    } else if (!smooth) {
      v = r[e];
    } else {
      const int64_t lo = h - back > 0 ? h - back : 0;
      const int64_t hi = h + fwd + 1 < A.H ? h + fwd + 1 : A.H;
      double acc = 0.0;
      for (int64_t k = lo; k < hi; ++k) acc += r[k * A.n + j];
      v = acc / sqrt((double)(hi - lo));
    }
    v *= A.sigma[j];
    const size_t o = (size_t)mloc * hn + e;
    if (A.dtype == VPB_DTYPE_F32)
      reinterpret_cast<float *>(A.out)[o] = (float)v;
    else
      reinterpret_cast<double *>(A.out)[o] = v;
  }
}

}  // namespace vpb

using namespace vpb;

extern "C" int vpb_sample_perturbations(uint64_t seed, const uint64_t *seed_dev, int64_t m_offset, int64_t M,
                                        int64_t H, int64_t n, int64_t window, const double *sigma, int dtype,
                                        void *out, void *stream) {
  VPB_REQUIRE(out && sigma && M >= 0 && H >= 1 && n >= 1 && n <= VPB_MAX_JOINTS && m_offset >= 0,
              "bad arguments to vpb_sample_perturbations");
  VPB_REQUIRE(dtype == VPB_DTYPE_F32 || dtype == VPB_DTYPE_F64, "bad dtype");
  if (M == 0) return VPB_OK;
  SamplerArgs A;
  memset(&A, 0, sizeof(A));
  A.seed = seed;
  A.seed_dev = seed_dev;
  A.m_offset = m_offset;
  A.M = M;
  A.H = H;
  A.n = n;
  A.window = window;
  for (int64_t j = 0; j < n; ++j) A.sigma[j] = sigma[j];
  A.out = out;
  A.dtype = dtype;
  const size_t smem = (size_t)8 * H * n * sizeof(double);
  VPB_REQUIRE(smem <= 200 * 1024, "horizon x dof too large for the sampler (max 3200)");
  if (smem > 48 * 1024)
    VPB_CUDA(cudaFuncSetAttribute(sampler_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  sampler_kernel<<<(unsigned)ceil_div(M, 8), 256, smem, as_stream(stream)>>>(A);
  return check_launch("sampler_kernel");
}
