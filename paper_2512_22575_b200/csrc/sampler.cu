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


// Thread = (sample m, 8-step chunk c, joint j), j fastest.  Column j of
// sample m is a Philox4x32-10 stream keyed by (seed, global m) with counter
// (4-step chunk, j, m): each thread draws the 16 normals of steps
// [8c - 4, 8c + 12) (neighbouring threads redraw the overlap bit-identically),
// applies the moving average of vp/planner.py:182-196 (window <= 9, rows
// scaled 1/sqrt(count)) and sigma_j, and writes its 8 outputs.  Everything
// stays in registers; no shared memory, no synchronisation.
constexpr int kChunk = 8;

template <typename OT>
__global__ void __launch_bounds__(256) sampler_kernel(const __grid_constant__ SamplerArgs A) {
  const int n = (int)A.n, H = (int)A.H;
  const unsigned C = (unsigned)(H + kChunk - 1) / kChunk;
  const unsigned gid = blockIdx.x * blockDim.x + threadIdx.x;  // < 2^31 (checked on the host)
  if (gid >= (unsigned)(A.M * (int64_t)C * n)) return;
  const unsigned mc = gid / (unsigned)n;
  const int j = (int)(gid - mc * (unsigned)n);
  const unsigned mq = mc / C;
  const int c = (int)(mc - mq * C);
  const int64_t mloc = mq;
  const int64_t mg = A.m_offset + mloc;
  const uint64_t seed = A.seed_dev ? *A.seed_dev : A.seed;
  const uint32_t k0 = (uint32_t)seed ^ (uint32_t)((uint64_t)mg * 0x9E3779B97F4A7C15ull);
  const uint32_t k1 = (uint32_t)(seed >> 32) ^ (uint32_t)((uint64_t)mg >> 32) ^ 0x85EBCA6Bu;
  const int h0 = c * kChunk;
  float z[16];  // steps h0 - 4 + i
  const int nq = (H + 3) >> 2;  // 4-step Philox chunks of the column
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int cq = 2 * c - 1 + q;  // 4-step chunk index
    if (cq >= 0 && cq < nq) {
      const uint4 x = philox4x32_10(make_uint4((uint32_t)cq, (uint32_t)j, (uint32_t)mg, 0x5eedu), k0, k1);
      box_muller_f(x.x, x.y, z[4 * q + 0], z[4 * q + 1]);
      box_muller_f(x.z, x.w, z[4 * q + 2], z[4 * q + 3]);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) z[4 * q + t] = 0.0f;
    }
  }
  const int back = (int)(A.window - 1) / 2, fwd = (int)A.window / 2;
  const bool zero = mg == 0;  // reserved nominal sample
  const float sig = (float)A.sigma[j];
  OT *out = reinterpret_cast<OT *>(A.out) + ((size_t)mloc * H) * n + j;
#pragma unroll
  for (int t = 0; t < kChunk; ++t) {
    const int h = h0 + t;
    if (h >= H) break;
    float v;
    if (A.window > 1) {
      float acc = 0.0f;
      int cnt = 0;
#pragma unroll
      for (int d = -4; d <= 4; ++d) {
        const bool in = d >= -back && d <= fwd && h + d >= 0 && h + d < H;
        acc += in ? z[t + 4 + d] : 0.0f;
        cnt += in ? 1 : 0;
      }
      v = acc * rsqrtf((float)cnt);
    } else {
      v = z[t + 4];
    }
    out[(size_t)h * n] = (OT)(zero ? 0.0f : v * sig);
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
  VPB_REQUIRE(window >= 1 && window <= 9, "noise window must be in [1, 9]");
  const int64_t C = (H + kChunk - 1) / kChunk;
  const int64_t total = M * C * n;
  VPB_REQUIRE(total < ((int64_t)1 << 31), "too many samples for one sampler launch");
  const unsigned grid = (unsigned)ceil_div(total, 256);
  cudaStream_t s = as_stream(stream);
  if (dtype == VPB_DTYPE_F32)
    sampler_kernel<float><<<grid, 256, 0, s>>>(A);
  else
    sampler_kernel<double><<<grid, 256, 0, s>>>(A);
  return check_launch("sampler_kernel");
}
