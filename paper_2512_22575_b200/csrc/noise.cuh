// Perturbation noise of one SMPC candidate on one warp (lane = horizon step).
//
// vp/planner.py:182-219 (smoothing_matrix, sample_perturbations): per sample m
// a counter-based stream keyed by (seed, global m); standard normals z[k][j];
// moving average over the window (rows scaled 1/sqrt(count)); times sigma_j;
// sample 0 is the zero perturbation.  Here the stream is Philox4x32-10 with
// counter (step k, joint quad, m) and Box-Muller normals, statistically (not
// bitwise) equivalent to numpy's Philox4x64 + ziggurat (the reference's own
// sampler tests are statistical, t/test_planner.py:52-90).
//
// The same function serves the stand-alone sampler kernel and the fused SMPC
// kernel, which draws each candidate's noise in registers instead of reading
// a precomputed buffer; both produce identical values.
#pragma once

#include "vpb_common.cuh"

namespace vpb {

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
  const float r = sqrtf(-2.0f * __logf(u1));  // MUFU.LG2; u1 in (0, 1) away from denormals
  // angle 2 pi (u2 - 1/2) in (-pi, pi), where MUFU.SIN/COS are accurate to
  // ~1e-6 absolute (the pair stays independent standard normal)
  float s, c;
  __sincosf(6.28318530717958647692f * (u2 - 0.5f), &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// Generator parameters (device-side seed for graph replays).
struct NoiseGen {
  uint64_t seed;
  const uint64_t *seed_dev;  // overrides `seed` when non-null
  int64_t m_offset;          // global index of local sample 0
  int window;                // 1..9
  float sigma[VPB_MAX_JOINTS];
};

__device__ __forceinline__ uint64_t noise_seed(const NoiseGen &G) { return G.seed_dev ? *G.seed_dev : G.seed; }

// The NJ raw normals of step k (k may lie outside [0, H): callers mask).
template <int NJ>
__device__ __forceinline__ void raw_normals(uint32_t k0, uint32_t k1, uint64_t mg, int k, float (&z)[NJ]) {
#pragma unroll
  for (int q = 0; q < (NJ + 3) / 4; ++q) {
    const uint4 x = philox4x32_10(make_uint4((uint32_t)k, (uint32_t)q, (uint32_t)mg, 0x5eedu), k0, k1);
    float a, b, c, d;
    box_muller_f(x.x, x.y, a, b);
    box_muller_f(x.z, x.w, c, d);
    if (4 * q + 0 < NJ) z[4 * q + 0] = a;
    if (4 * q + 1 < NJ) z[4 * q + 1] = b;
    if (4 * q + 2 < NJ) z[4 * q + 2] = c;
    if (4 * q + 3 < NJ) z[4 * q + 3] = d;
  }
}

// Noise of candidate `m_loc` at step k = 32 ch + lane (NJ joints): every lane
// of the warp must call it (shuffles).  Steps outside [0, H) get zeros.
template <int NJ, int HALF>
__device__ __forceinline__ void candidate_noise(const NoiseGen &G, int64_t m_loc, int H, int ch, int lane,
                                               float (&u)[NJ]) {
  static_assert(HALF == 2 || HALF == 4, "half window 2 (window <= 5) or 4 (window <= 9)");
  const uint64_t seed = noise_seed(G);
  const uint64_t mg = (uint64_t)(G.m_offset + m_loc);
  const uint32_t k0 = (uint32_t)seed ^ (uint32_t)(mg * 0x9E3779B97F4A7C15ull);
  const uint32_t k1 = (uint32_t)(seed >> 32) ^ (uint32_t)(mg >> 32) ^ 0x85EBCA6Bu;
  const int k = 32 * ch + lane;
  float zm[NJ];
  raw_normals<NJ>(k0, k1, mg, k, zm);
  const int back = (G.window - 1) >> 1, fwd = G.window >> 1;
  const bool multi = H > 32;  // halo steps from the neighbouring chunks
  float zh[NJ];
  if (multi) {
    // lanes 0..3: steps 32 ch - 4 .. 32 ch - 1; lanes 4..7: 32 ch + 32 .. + 35
    const int kh = lane < 4 ? 32 * ch - 4 + lane : 32 * ch + 28 + lane;
    raw_normals<NJ>(k0, k1, mg, kh, zh);
  }
  const int lo = max(0, k - back), hi = min(H, k + fwd + 1);
  const float scale = (mg == 0 || k >= H) ? 0.0f : rsqrtf((float)(hi - lo));
  // window offsets d in use at this step, computed once
  float dm[2 * HALF + 1];  // 1 / 0 per window offset
#pragma unroll
  for (int d = -HALF; d <= HALF; ++d)
    dm[d + HALF] = (d >= -back && d <= fwd && k + d >= 0 && k + d < H) ? 1.0f : 0.0f;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    float acc = 0.0f;
#pragma unroll
    for (int d = -HALF; d <= HALF; ++d) {
      const int src = lane + d;  // lane of step k + d within the chunk (may leave [0, 32))
      float v = __shfl_sync(kFull, zm[j], src & 31);
      if (multi) {  // warp-uniform
        const float vh = __shfl_sync(kFull, zh[j], src < 0 ? src + 4 : (src - 28) & 31);
        v = (src < 0 || src >= 32) ? vh : v;
      }
      acc = fmaf(dm[d + HALF], v, acc);  // == acc + (in window ? v : 0), v finite
    }
    u[j] = acc * scale * G.sigma[j];
  }
}

}  // namespace vpb
