// Compile-time-topology rollout step (sm_100a).
//
// The per-step work of vp/batch.py:240-314 for a robot whose topology (joint
// axes, offset structure, sphere -> link map, self pairs) is fixed at compile
// time.  Every loop over joints, spheres and pairs is unrolled into straight-
// line code: sphere centres live in registers, pair distances read them
// directly, every robot constant is an immediate constant-bank operand, and the
// eleven field gathers overlap the remaining forward kinematics.  The numeric
// values (offsets, radii, weights, limits) still come from the problem block,
// so one instantiation serves every robot with the same topology; other robots
// take the generic path in rollout.cu.
//
// Step shift: lane k of a warp evaluates FK at q_{k+1} (running pose cost for
// k+1 < H, terminal pose cost for k+1 == H, spheres for k+1 < H) while the
// limit / smoothness / null-space terms stay at (q_k, qd_k, u_k).  The
// q_0 terms are identical for every candidate and are computed once per CTA.
// The per-candidate sums are the reference's, reordered.
#pragma once

#include <type_traits>

#include "rollout.cuh"

namespace vpb {

template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F &&f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Axis codes: +-1 = x, +-2 = y, +-3 = z (sign = axis direction), 0 = general.
// Offset codes: 1 = identity rotation and translation (0, 0, z), 0 = general.
// Sphere codes: 1 = centre (0, 0, z) in its link frame, 0 = general.
struct TopoRobot7 {
  // vp/data/robot_7dof.yaml:11-77 (the reference's benchmark arm)
  static constexpr int NJ = 7, NS = 11, NP = 18;
  __host__ __device__ static constexpr int axis(int j) {
    constexpr int a[7] = {3, 2, 3, 2, 3, 2, 3};
    return a[j];
  }
  __host__ __device__ static constexpr int offset_kind(int) { return 1; }
  __host__ __device__ static constexpr int sphere_kind(int) { return 1; }
  __host__ __device__ static constexpr int link(int s) {
    constexpr int l[11] = {0, 1, 2, 2, 3, 3, 4, 4, 5, 6, 7};
    return l[s];
  }
  __host__ __device__ static constexpr int pair_i(int p) {
    constexpr int a[18] = {0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 3, 3, 3, 4, 4, 5};
    return a[p];
  }
  __host__ __device__ static constexpr int pair_j(int p) {
    constexpr int b[18] = {6, 7, 8, 9, 10, 6, 7, 9, 10, 6, 7, 10, 8, 9, 10, 9, 10, 10};
    return b[p];
  }
};

// Link li: R <- R * Rot(axis, q); t <- t + R_old * (0, 0, oz) for offset kind 1.
template <typename Topo, int J, typename T>
__device__ __forceinline__ void fixed_link(const Prob<T> &P, T q, T R[9], T t[3]) {
  if constexpr (Topo::offset_kind(J) == 1) {
    const T oz = P.off_t[3 * J + 2];
    t[0] = fma(R[2], oz, t[0]);
    t[1] = fma(R[5], oz, t[1]);
    t[2] = fma(R[8], oz, t[2]);
  } else {
    const T ox = P.off_t[3 * J], oy = P.off_t[3 * J + 1], oz = P.off_t[3 * J + 2];
#pragma unroll
    for (int a = 0; a < 3; ++a) t[a] = fma(R[3 * a], ox, fma(R[3 * a + 1], oy, fma(R[3 * a + 2], oz, t[a])));
    T M[9];
    const T *o = P.off_r + 9 * J;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      M[3 * a + 0] = fma(R[3 * a], o[0], fma(R[3 * a + 1], o[3], R[3 * a + 2] * o[6]));
      M[3 * a + 1] = fma(R[3 * a], o[1], fma(R[3 * a + 1], o[4], R[3 * a + 2] * o[7]));
      M[3 * a + 2] = fma(R[3 * a], o[2], fma(R[3 * a + 1], o[5], R[3 * a + 2] * o[8]));
    }
#pragma unroll
    for (int a = 0; a < 9; ++a) R[a] = M[a];
  }
  T s, c;
  tsincos<T>(q, &s, &c);
  constexpr int ax = Topo::axis(J);
  if constexpr (ax < 0) s = -s;
  if constexpr (ax == 3 || ax == -3) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T m0 = R[3 * a], m1 = R[3 * a + 1];
      R[3 * a + 0] = fma(m0, c, m1 * s);
      R[3 * a + 1] = fma(m1, c, -(m0 * s));
    }
  } else if constexpr (ax == 2 || ax == -2) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T m0 = R[3 * a], m2 = R[3 * a + 2];
      R[3 * a + 0] = fma(m0, c, -(m2 * s));
      R[3 * a + 2] = fma(m0, s, m2 * c);
    }
  } else if constexpr (ax == 1 || ax == -1) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T m1 = R[3 * a + 1], m2 = R[3 * a + 2];
      R[3 * a + 1] = fma(m1, c, m2 * s);
      R[3 * a + 2] = fma(m2, c, -(m1 * s));
    }
  } else {
    const T ux = P.axes[3 * J], uy = P.axes[3 * J + 1], uz = P.axes[3 * J + 2];
    const T *w = P.uu + 6 * J;
    const T ic = T(1) - c;
    const T j00 = fma(w[0], ic, c), j01 = fma(w[1], ic, -uz * s), j02 = fma(w[2], ic, uy * s);
    const T j10 = fma(w[1], ic, uz * s), j11 = fma(w[3], ic, c), j12 = fma(w[4], ic, -ux * s);
    const T j20 = fma(w[2], ic, -uy * s), j21 = fma(w[4], ic, ux * s), j22 = fma(w[5], ic, c);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T m0 = R[3 * a], m1 = R[3 * a + 1], m2 = R[3 * a + 2];
      R[3 * a + 0] = fma(m0, j00, fma(m1, j10, m2 * j20));
      R[3 * a + 1] = fma(m0, j01, fma(m1, j11, m2 * j21));
      R[3 * a + 2] = fma(m0, j02, fma(m1, j12, m2 * j22));
    }
  }
}

// Environment cost of one sphere centre (vp/mapping.py:616-685 inlined with
// the gap test of vp/batch.py:277-293).  The interpolation corner is clamped
// to n - 2 so the eight corners are base + {0, off0} + {0, off1} + {0, off2}
// (the reference's b = min(a + 1, n - 1) gives the same value: at the upper
// border its weight on b is 0 and ours puts weight 1 on the same voxel).
//
// fp32 (production): the containing cell floor(g) is loaded first.  The field
// holds exact squared distances between voxel centres (vpb_edt3d), so
// sqrt(field) is 1-Lipschitz and every interpolation corner -- the cell is one
// of them -- has sqrt(v) >= sqrt(cell) - sqrt(3); past C.far2 the interpolated
// distance is beyond d_act + r and the term is exactly 0.  Most spheres of
// most steps leave after that one load.
__device__ __forceinline__ float env_cost_f32(const Prob<float> &P, const FixedConsts<float> &C, const float *sq,
                                              int s, float px, float py, float pz) {
  const float g0 = (px - P.origin0) * P.inv_voxel - P.lo0;
  const float g1 = (py - P.origin1) * P.inv_voxel - P.lo1;
  const float g2 = (pz - P.origin2) * P.inv_voxel - P.lo2;
  if (!(g0 >= 0.0f && g0 < C.nf0 && g1 >= 0.0f && g1 < C.nf1 && g2 >= 0.0f && g2 < C.nf2)) return C.out_cost[s];
  const int k0 = (int)g0, k1 = (int)g1, k2 = (int)g2;  // floor (g >= 0)
  const float cell = __ldg(sq + ((k0 * P.n1 + k1) * P.n2 + k2));
  if (cell >= C.far2[s]) return 0.0f;
  if (cell == 0.0f) return C.zero_cost[s];  // containing cell occupied
  // c = g - 1/2 clamped to [0, n - 1] (vp/mapping.py:654-663)
  const float c0 = fminf(fmaxf(g0 - 0.5f, 0.0f), C.chi0);
  const float c1 = fminf(fmaxf(g1 - 0.5f, 0.0f), C.chi1);
  const float c2 = fminf(fmaxf(g2 - 0.5f, 0.0f), C.chi2);
  const float a0 = fminf(floorf(c0), C.amax0), a1 = fminf(floorf(c1), C.amax1), a2 = fminf(floorf(c2), C.amax2);
  const float f0 = c0 - a0, f1 = c1 - a1, f2 = c2 - a2;  // in [0, 1]
  const float *p = sq + (((int)a0 * P.n1 + (int)a1) * P.n2 + (int)a2);
  const float v0 = __ldg(p), v1 = __ldg(p + C.off2);
  const float *py_ = p + C.off1;
  const float v2 = __ldg(py_), v3 = __ldg(py_ + C.off2);
  const float *px_ = p + C.off0;
  const float v4 = __ldg(px_), v5 = __ldg(px_ + C.off2);
  const float *pxy = px_ + C.off1;
  const float v6 = __ldg(pxy), v7 = __ldg(pxy + C.off2);
  const float h0 = 1.0f - f0, h1 = 1.0f - f1, h2 = 1.0f - f2;
  const float c00 = fmaf(v4, f0, v0 * h0);
  const float c01 = fmaf(v5, f0, v1 * h0);
  const float c10 = fmaf(v6, f0, v2 * h0);
  const float c11 = fmaf(v7, f0, v3 * h0);
  const float c0v = fmaf(c10, f1, c00 * h1);
  const float c1v = fmaf(c11, f1, c01 * h1);
  const float value = fmaf(c1v, f2, c0v * h2);
  const float dist = P.voxel * (value * rsqrtf(fmaxf(value, 1e-30f)));
  const float gap = P.d_act - (dist - P.sph_r[s]);
  return gap > 0.0f ? P.w_env * gap * gap : 0.0f;
}

template <typename T>
__device__ __forceinline__ T env_cost(const Prob<T> &P, const FixedConsts<T> &C, const float *sq, int s, T px, T py,
                                      T pz) {
  if constexpr (sizeof(T) == 4) {
    return env_cost_f32(P, C, sq, s, px, py, pz);
  } else {
    const T g0 = (px - P.origin0) / P.voxel - P.lo0;
    const T g1 = (py - P.origin1) / P.voxel - P.lo1;
    const T g2 = (pz - P.origin2) / P.voxel - P.lo2;
    const bool inside = g0 >= T(0) && g0 < C.nf0 && g1 >= T(0) && g1 < C.nf1 && g2 >= T(0) && g2 < C.nf2;
    const T z0 = inside ? g0 : T(0), z1 = inside ? g1 : T(0), z2 = inside ? g2 : T(0);  // any in-range address
    // c = g - 1/2 clamped to [0, n - 1] (vp/mapping.py:654-663)
    T c0 = z0 - T(0.5), c1 = z1 - T(0.5), c2 = z2 - T(0.5);
    c0 = fmin(fmax(c0, T(0)), C.chi0);
    c1 = fmin(fmax(c1, T(0)), C.chi1);
    c2 = fmin(fmax(c2, T(0)), C.chi2);
    const T a0 = fmin(floor(c0), C.amax0), a1 = fmin(floor(c1), C.amax1), a2 = fmin(floor(c2), C.amax2);
    const T f0 = c0 - a0, f1 = c1 - a1, f2 = c2 - a2;  // in [0, 1]
    const float *p = sq + (((int)a0 * P.n1 + (int)a1) * P.n2 + (int)a2);
    const float v0 = __ldg(p), v1 = __ldg(p + C.off2);
    const float *py_ = p + C.off1;
    const float v2 = __ldg(py_), v3 = __ldg(py_ + C.off2);
    const float *px_ = p + C.off0;
    const float v4 = __ldg(px_), v5 = __ldg(px_ + C.off2);
    const float *pxy = px_ + C.off1;
    const float v6 = __ldg(pxy), v7 = __ldg(pxy + C.off2);
    // containing cell floor(g): the b corner on an axis iff g >= a + 1
    const bool sx = z0 >= a0 + T(1), sy = z1 >= a1 + T(1), sz = z2 >= a2 + T(1);
    const float e00 = sz ? v1 : v0, e01 = sz ? v3 : v2, e10 = sz ? v5 : v4, e11 = sz ? v7 : v6;
    const float e0 = sy ? e01 : e00, e1 = sy ? e11 : e10;
    const float cell = sx ? e1 : e0;
    const T h0 = T(1) - f0, h1 = T(1) - f1, h2 = T(1) - f2;
    const T c00 = fma((T)v4, f0, (T)v0 * h0);
    const T c01 = fma((T)v5, f0, (T)v1 * h0);
    const T c10 = fma((T)v6, f0, (T)v2 * h0);
    const T c11 = fma((T)v7, f0, (T)v3 * h0);
    const T c0v = fma(c10, f1, c00 * h1);
    const T c1v = fma(c11, f1, c01 * h1);
    const T value = fma(c1v, f2, c0v * h2);
    // branch-free selection (the all-inf field gives inf / NaN -> no cost)
    const T gap = P.d_act - (P.voxel * sqrt(value) - P.sph_r[s]);
    T env = gap > T(0) ? P.w_env * gap * gap : T(0);
    env = cell == 0.0f ? C.zero_cost[s] : env;
    return inside ? env : C.out_cost[s];
  }
}

// Which terms of a configuration one warp evaluates (warp-uniform): the
// environment queries of the spheres in `smask`, the self pairs in `pmask`,
// and the pose term when `pose`.  A candidate warp takes everything; the
// latency-critical single-configuration evaluations split the terms over the
// warps of a CTA (sphere centres are always computed: pairs need them).
struct Split {
  uint32_t smask;
  uint64_t pmask;
  bool pose;
};

template <typename Topo>
__device__ __forceinline__ Split make_split(int sub, int nsub) {
  static_assert(Topo::NS <= 32 && Topo::NP <= 64, "split masks hold 32 spheres / 64 pairs");
  if (nsub == 1) return Split{0xffffffffu, ~0ull, true};  // a candidate warp: everything
  Split w{0u, 0ull, sub == nsub - 1};
  for (int s = sub; s < Topo::NS; s += nsub) w.smask |= 1u << s;
  for (int p = sub; p < Topo::NP; p += nsub) w.pmask |= 1ull << p;
  return w;
}

// One configuration q: FK, pose cost (weights Wq or Wt), and -- when `spheres`
// -- the environment and self-collision terms, restricted to the warp's
// Split.  Returns false at the log-map singularity.
template <typename Topo, typename T>
__device__ __forceinline__ bool fixed_config(const Prob<T> &P, const FixedConsts<T> &C, const Dyn<T> &D,
                                             const T (&q)[Topo::NJ], bool spheres, bool terminal, const Split &W,
                                             T &pose, T &coll) {
  constexpr int NJ = Topo::NJ, NS = Topo::NS, NP = Topo::NP;
  T R[9], t[3];
#pragma unroll
  for (int a = 0; a < 9; ++a) R[a] = P.base_r[a];
  t[0] = P.base_t[0];
  t[1] = P.base_t[1];
  t[2] = P.base_t[2];
  T cx[NS], cy[NS], cz[NS];
  T env = T(0);
  static_for<0, NJ + 1>([&](auto lic) {
    constexpr int li = decltype(lic)::value;
    if constexpr (li > 0) fixed_link<Topo, li - 1, T>(P, q[li - 1], R, t);
    static_for<0, NS>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      if constexpr (Topo::link(s) == li) {
        if constexpr (Topo::sphere_kind(s) == 1) {
          const T lz = P.sph_loc[3 * s + 2];
          cx[s] = fma(R[2], lz, t[0]);
          cy[s] = fma(R[5], lz, t[1]);
          cz[s] = fma(R[8], lz, t[2]);
        } else {
          const T lx = P.sph_loc[3 * s], ly = P.sph_loc[3 * s + 1], lz = P.sph_loc[3 * s + 2];
          cx[s] = fma(R[0], lx, fma(R[1], ly, fma(R[2], lz, t[0])));
          cy[s] = fma(R[3], lx, fma(R[4], ly, fma(R[5], lz, t[1])));
          cz[s] = fma(R[6], lx, fma(R[7], ly, fma(R[8], lz, t[2])));
        }
        if (spheres && P.has_field && ((W.smask >> s) & 1u)) env += env_cost<T>(P, C, D.sq, s, cx[s], cy[s], cz[s]);
      }
    });
  });
  // pose error at the end effector (vp/batch.py:69-137)
  bool ok = true;
  pose = T(0);
  if (W.pose) {
    const T *G = D.goal_r;
    const T d00 = G[0] * R[0] + G[3] * R[3] + G[6] * R[6];
    const T d01 = G[0] * R[1] + G[3] * R[4] + G[6] * R[7];
    const T d02 = G[0] * R[2] + G[3] * R[5] + G[6] * R[8];
    const T d10 = G[1] * R[0] + G[4] * R[3] + G[7] * R[6];
    const T d11 = G[1] * R[1] + G[4] * R[4] + G[7] * R[7];
    const T d12 = G[1] * R[2] + G[4] * R[5] + G[7] * R[8];
    const T d20 = G[2] * R[0] + G[5] * R[3] + G[8] * R[6];
    const T d21 = G[2] * R[1] + G[5] * R[4] + G[8] * R[7];
    const T d22 = G[2] * R[2] + G[5] * R[5] + G[8] * R[8];
    const T rx = t[0] - D.goal_t[0], ry = t[1] - D.goal_t[1], rz = t[2] - D.goal_t[2];
    const T tx = G[0] * rx + G[3] * ry + G[6] * rz;
    const T ty = G[1] * rx + G[4] * ry + G[7] * rz;
    const T tz = G[2] * rx + G[5] * ry + G[8] * rz;
    T c = T(0.5) * (d00 + d11 + d22 - T(1));
    c = c > T(1) ? T(1) : (c < T(-1) ? T(-1) : c);
    const T sx = T(0.5) * (d21 - d12), sy = T(0.5) * (d02 - d20), sz = T(0.5) * (d10 - d01);
    T theta, scale;
    if constexpr (sizeof(T) == 8) {
      theta = acos(c);
      ok = theta < P.pi_limit;
      scale = theta < 1e-6 ? 1.0 + theta * theta / 6.0 : theta / sin(theta);
    } else {
      const float sn = sqrtf(sx * sx + sy * sy + sz * sz);
      theta = atan2f(sn, c);
      ok = theta < P.pi_limit;
      scale = theta < 1e-3f ? 1.0f + theta * theta * (1.0f / 6.0f) : theta / sn;
    }
    const T wx = scale * sx, wy = scale * sy, wz = scale * sz;
    T e;
    if (theta < T(0.1)) {
      const T t2 = theta * theta;
      e = T(1.0 / 12.0) + t2 / T(720.0) + t2 * t2 / T(30240.0);
    } else {
      T sth, cth;
      tsincos<T>(theta, &sth, &cth);
      e = (T(1) - T(0.5) * theta * sth / (T(1) - cth)) / (theta * theta);
    }
    const T wxx = wx * wx, wyy = wy * wy, wzz = wz * wz;
    const T m00 = T(1) + e * (-wzz - wyy), m01 = T(0.5) * wz + e * wx * wy, m02 = T(-0.5) * wy + e * wx * wz;
    const T m10 = T(-0.5) * wz + e * wx * wy, m11 = T(1) + e * (-wxx - wzz), m12 = T(0.5) * wx + e * wy * wz;
    const T m20 = T(0.5) * wy + e * wx * wz, m21 = T(-0.5) * wx + e * wy * wz, m22 = T(1) + e * (-wxx - wyy);
    T xi[6];
    xi[0] = m00 * tx + m01 * ty + m02 * tz;
    xi[1] = m10 * tx + m11 * ty + m12 * tz;
    xi[2] = m20 * tx + m21 * ty + m22 * tz;
    xi[3] = wx;
    xi[4] = wy;
    xi[5] = wz;
    const T *Wm = terminal ? C.Wt : C.Wq;
    T quad = T(0);
    if (C.w_diag) {
      quad = Wm[0] * xi[0] * xi[0] + Wm[6] * xi[1] * xi[1] + Wm[11] * xi[2] * xi[2] + Wm[15] * xi[3] * xi[3] +
             Wm[18] * xi[4] * xi[4] + Wm[20] * xi[5] * xi[5];
    } else {
      int idx = 0;
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        T row = T(0);
#pragma unroll
        for (int b = a; b < 6; ++b) row = fma(Wm[idx++], xi[b], row);
        quad = fma(xi[a], row, quad);
      }
    }
    pose = ok ? T(0.5) * quad : T(0);
  }
  // self pairs (vp/batch.py:294-302): squared pre-check, sqrt only on contact
  T self = T(0);
  if (spheres) {
    // fast pass: a pair can touch only if d^2 < rsum2 (a conservative bound
    // of (r_i + r_j)^2); the exact penalties are summed only on lanes where
    // some pair may touch (rare), in the same pair order as always
    bool touch = false;
    static_for<0, NP>([&](auto pc) {
      constexpr int p = decltype(pc)::value;
      constexpr int i = Topo::pair_i(p), j = Topo::pair_j(p);
      const T dx = cx[i] - cx[j], dy = cy[i] - cy[j], dz = cz[i] - cz[j];
      const T d2 = dx * dx + dy * dy + dz * dz;
      touch |= d2 < C.rsum2[p];  // (the split mask is applied in the exact pass)
    });
    if (touch) {
      static_for<0, NP>([&](auto pc) {
        constexpr int p = decltype(pc)::value;
        constexpr int i = Topo::pair_i(p), j = Topo::pair_j(p);
        const T dx = cx[i] - cx[j], dy = cy[i] - cy[j], dz = cz[i] - cz[j];
        const T d2 = dx * dx + dy * dy + dz * dz;
        T gap;
        if constexpr (sizeof(T) == 8) {
          gap = sqrt(d2) - C.rsum[p];
        } else {
          gap = d2 * rsqrtf(fmaxf(d2, 1e-30f)) - C.rsum[p];
        }
        const T pen = gap < T(0) ? P.w_self * gap * gap : T(0);
        self += ((W.pmask >> p) & 1ull) ? pen : T(0);
      });
    }
  }
  coll = env + self;
  return ok;
}

}  // namespace vpb
