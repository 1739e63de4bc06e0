// Device-side problem description and per-step math of the SMPC rollout.
// Restates vp/batch.py:25-158 (_fk_frames, _pose_error, _quad_form,
// _bound_violation) and vp/mapping.py:616-685 (_query_metric) in the compute
// precision T (float = production, double = parity mode).
#pragma once

#include "vpb_common.cuh"

namespace vpb {

constexpr int kMaxJ = VPB_MAX_JOINTS;
constexpr int kMaxS = VPB_MAX_SPHERES;
constexpr int kMaxP = VPB_MAX_PAIRS;

// Joint axis classes for the sparse Rodrigues fast paths (warp-uniform).
enum AxisKind : int8_t { kAxisGeneral = 0, kAxisX = 1, kAxisY = 2, kAxisZ = 3 };

// Per-sphere and per-pair derived constants (host-computed in T).
template <typename T>
struct FixedConsts {
  T dr[kMaxS];         // d_act + r_s
  T thr2[kMaxS];       // squared-voxel value above which the env term is certainly 0
  T far2[kMaxS];       // corner value above which every corner of the cell is beyond thr (see env_cost)
  T zero_cost[kMaxS];  // env cost when the containing cell is occupied (distance 0)
  T out_cost[kMaxS];   // env cost outside the field volume
  T rsum[kMaxP];       // r_i + r_j
  T rsum2[kMaxP];      // upper bound of (r_i + r_j)^2 (squared pre-check)
  T Wq[21], Wt[21];    // symmetric parts of Q and Q_H (upper triangle, row major)
  int w_diag;          // both weights diagonal
  int off0, off1, off2;  // corner strides along x / y / z (0 on a length-1 axis)
  T amax0, amax1, amax2;  // max(n - 2, 0): lower interpolation corner bound
  T nf0, nf1, nf2;        // n as T
  T chi0, chi1, chi2;     // n - 1
};

template <typename T>
struct Prob {
  int nj, ns, np, H;
  T dt;
  T lam;
  T base_r[9], base_t[3];
  T off_r[kMaxJ * 9], off_t[kMaxJ * 3];
  T axes[kMaxJ * 3];
  T uu[kMaxJ * 6];          // ux^2, ux uy, ux uz, uy^2, uy uz, uz^2
  T axis_sign[kMaxJ];       // +-1 for unit axes
  int8_t axis_kind[kMaxJ];
  int8_t off_identity[kMaxJ];
  int16_t sph_begin[kMaxJ + 2];  // spheres of link l: [sph_begin[l], sph_begin[l+1])
  int16_t sph_orig[kMaxS];
  int16_t pairs[kMaxP * 2];
  T sph_loc[kMaxS * 3], sph_r[kMaxS];
  T goal_r[9], goal_t[3];
  T Q[36], QH[36];
  T pos_lo[kMaxJ], pos_hi[kMaxJ], vel_lo[kMaxJ], vel_hi[kMaxJ], acc_lo[kMaxJ], acc_hi[kMaxJ];
  T q_ref[kMaxJ], q0[kMaxJ], qd0[kMaxJ];
  T w_env, w_self, w_q, w_qd, w_qdd, w_s, w_ns, d_act;
  // distance field (vp/mapping.py:556-583)
  const float *sq;
  const float *const *sq_dev;  // optional indirection (vpb_problem.field_sq_dev)
  int n0, n1, n2;
  int has_field;
  T lo0, lo1, lo2;
  T origin0, origin1, origin2;
  T voxel, inv_voxel, outside;
  T pi_limit;  // pi - _PI_MARGIN in T
  FixedConsts<T> fc;  // derived constants of the compile-time-topology path
};

// Per-call state (start state and goal).  Read from a device buffer when the
// caller provides one (graph replays update it with one tiny H2D copy), else
// from the launch parameters.  Device layout: [q0 (n), qd0 (n), goal_r (9),
// goal_t (3)] as f64.
template <typename T>
struct Dyn {
  T q0[kMaxJ], qd0[kMaxJ];
  T goal_r[9], goal_t[3];
  const float *sq;  // distance field of this launch (P.sq or *P.sq_dev)
};

template <typename T>
__device__ __forceinline__ T tsqrt(T x);
template <>
__device__ __forceinline__ float tsqrt<float>(float x) { return sqrtf(x); }
template <>
__device__ __forceinline__ double tsqrt<double>(double x) { return sqrt(x); }

template <typename T>
__device__ __forceinline__ void tsincos(T x, T *s, T *c);
// fp32 sin/cos without sincosf's Payne-Hanek slow path (a local-memory loop
// behind a branch for |x| >= 105615, which the unrolled FK would carry eight
// times per step): Cody-Waite reduction by pi/2 in three parts and the
// classic minimax polynomials on [-pi/4, pi/4] (about 1 ulp for the joint
// angles a rollout produces; accuracy only degrades, without branching, for
// |x| beyond ~1e5).
template <>
__device__ __forceinline__ void tsincos<float>(float x, float *s, float *c) {
  const float j = rintf(x * 0.636619772367581343f);
  const int q = (int)j;
  float r = fmaf(j, -1.57079625129699707031f, x);
  r = fmaf(j, -7.54978941586159635335e-08f, r);
  r = fmaf(j, -5.39030253145912640453e-15f, r);
  const float z = r * r;
  float ps = fmaf(-1.9515295891e-4f, z, 8.3321608736e-3f);
  ps = fmaf(ps, z, -1.6666654611e-1f);
  const float sn = fmaf(ps * z, r, r);
  float pc = fmaf(2.443315711809948e-5f, z, -1.388731625493765e-3f);
  pc = fmaf(pc, z, 4.166664568298827e-2f);
  const float cs = fmaf(pc * z, z, fmaf(-0.5f, z, 1.0f));
  const float s0 = (q & 1) ? cs : sn;
  const float c0 = (q & 1) ? sn : cs;
  *s = (q & 2) ? -s0 : s0;
  *c = ((q + 1) & 2) ? -c0 : c0;
}
template <>
__device__ __forceinline__ void tsincos<double>(double x, double *s, double *c) { sincos(x, s, c); }

// _query_metric, vp/mapping.py:616-685, split in two so a warp can issue the
// eight corner loads of several spheres before consuming any of them.  The
// reference first reads the containing cell (sq == 0 -> 0, inf -> inf); that
// cell is always one of the eight interpolation corners (cell index
// floor(g) is either floor(g - 1/2) or floor(g - 1/2) + 1, also at the clamped
// borders), so it is selected from the loaded corners instead of being a
// separate dependent load.
template <typename T>
struct Query {
  T f0, f1, f2;
  float v0, v1, v2, v3, v4, v5, v6, v7;  // corners (a/b along x, y, z)
  float cell;                            // value of the containing cell
  bool outside;
};

template <typename T>
__device__ __forceinline__ void query_issue(const Prob<T> &P, const float *sq, T px, T py, T pz, Query<T> &Q) {
  T g0, g1, g2;
  if constexpr (sizeof(T) == 8) {
    g0 = (px - P.origin0) / P.voxel - P.lo0;
    g1 = (py - P.origin1) / P.voxel - P.lo1;
    g2 = (pz - P.origin2) / P.voxel - P.lo2;
  } else {
    g0 = (px - P.origin0) * P.inv_voxel - P.lo0;
    g1 = (py - P.origin1) * P.inv_voxel - P.lo1;
    g2 = (pz - P.origin2) * P.inv_voxel - P.lo2;
  }
  const int n0 = P.n0, n1 = P.n1, n2 = P.n2;
  Q.outside = !(g0 >= T(0) && g0 < T(n0) && g1 >= T(0) && g1 < T(n1) && g2 >= T(0) && g2 < T(n2));
  if (Q.outside) {
    g0 = g1 = g2 = T(0);
  }
  const int i0 = (int)g0, i1 = (int)g1, i2 = (int)g2;
  T c0 = g0 - T(0.5), c1 = g1 - T(0.5), c2 = g2 - T(0.5);
  c0 = c0 < T(0) ? T(0) : (c0 > T(n0 - 1) ? T(n0 - 1) : c0);
  c1 = c1 < T(0) ? T(0) : (c1 > T(n1 - 1) ? T(n1 - 1) : c1);
  c2 = c2 < T(0) ? T(0) : (c2 > T(n2 - 1) ? T(n2 - 1) : c2);
  const int a0 = (int)c0, a1 = (int)c1, a2 = (int)c2;
  const int b0 = a0 + 1 < n0 ? a0 + 1 : a0;
  const int b1 = a1 + 1 < n1 ? a1 + 1 : a1;
  const int b2 = a2 + 1 < n2 ? a2 + 1 : a2;
  Q.f0 = c0 - T(a0);
  Q.f1 = c1 - T(a1);
  Q.f2 = c2 - T(a2);
  const size_t r00 = ((size_t)a0 * n1 + a1) * n2, r01 = ((size_t)a0 * n1 + b1) * n2;
  const size_t r10 = ((size_t)b0 * n1 + a1) * n2, r11 = ((size_t)b0 * n1 + b1) * n2;
  Q.v0 = __ldg(sq + r00 + a2);
  Q.v1 = __ldg(sq + r00 + b2);
  Q.v2 = __ldg(sq + r01 + a2);
  Q.v3 = __ldg(sq + r01 + b2);
  Q.v4 = __ldg(sq + r10 + a2);
  Q.v5 = __ldg(sq + r10 + b2);
  Q.v6 = __ldg(sq + r11 + a2);
  Q.v7 = __ldg(sq + r11 + b2);
  // containing cell = corner (i == a ? a : b) on every axis
  const bool sx = i0 != a0, sy = i1 != a1, sz = i2 != a2;
  const float e00 = sz ? Q.v1 : Q.v0, e01 = sz ? Q.v3 : Q.v2;
  const float e10 = sz ? Q.v5 : Q.v4, e11 = sz ? Q.v7 : Q.v6;
  const float e0 = sy ? e01 : e00, e1 = sy ? e11 : e10;
  Q.cell = sx ? e1 : e0;
}

template <typename T>
__device__ __forceinline__ T query_finish(const Prob<T> &P, const Query<T> &Q) {
  if (Q.outside) return P.outside;
  if (Q.cell == 0.0f) return T(0);
  if (isinf(Q.cell)) return (T)Q.cell;  // no source in the volume: all values inf
  const T e0 = T(1) - Q.f0, e1 = T(1) - Q.f1, e2 = T(1) - Q.f2;
  const T c00 = (T)Q.v0 * e0 + (T)Q.v4 * Q.f0;
  const T c01 = (T)Q.v1 * e0 + (T)Q.v5 * Q.f0;
  const T c10 = (T)Q.v2 * e0 + (T)Q.v6 * Q.f0;
  const T c11 = (T)Q.v3 * e0 + (T)Q.v7 * Q.f0;
  const T c0v = c00 * e1 + c10 * Q.f1;
  const T c1v = c01 * e1 + c11 * Q.f1;
  const T value = c0v * e2 + c1v * Q.f2;
  return P.voxel * tsqrt<T>(value);
}

// One chain link: R <- R * off_r[i] * Rot(axis_i, q); t <- t + R_old * off_t[i]
// (vp/batch.py:33-66).  Fast paths for identity offsets and unit axes are
// warp-uniform branches.
template <typename T>
__device__ __forceinline__ void fk_link(const Prob<T> &P, int i, T q, T R[9], T t[3]) {
  // translation uses the parent rotation
  const T ox = P.off_t[3 * i], oy = P.off_t[3 * i + 1], oz = P.off_t[3 * i + 2];
  t[0] = t[0] + R[0] * ox + R[1] * oy + R[2] * oz;
  t[1] = t[1] + R[3] * ox + R[4] * oy + R[5] * oz;
  t[2] = t[2] + R[6] * ox + R[7] * oy + R[8] * oz;
  T M[9];
  if (P.off_identity[i]) {
#pragma unroll
    for (int k = 0; k < 9; ++k) M[k] = R[k];
  } else {
    const T *o = P.off_r + 9 * i;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      M[3 * a + 0] = R[3 * a] * o[0] + R[3 * a + 1] * o[3] + R[3 * a + 2] * o[6];
      M[3 * a + 1] = R[3 * a] * o[1] + R[3 * a + 1] * o[4] + R[3 * a + 2] * o[7];
      M[3 * a + 2] = R[3 * a] * o[2] + R[3 * a + 1] * o[5] + R[3 * a + 2] * o[8];
    }
  }
  T s, c;
  tsincos<T>(q, &s, &c);
  const int kind = P.axis_kind[i];
  if (kind == kAxisZ) {
    s = s * P.axis_sign[i];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T m0 = M[3 * a], m1 = M[3 * a + 1];
      R[3 * a + 0] = m0 * c + m1 * s;
      R[3 * a + 1] = m1 * c - m0 * s;
      R[3 * a + 2] = M[3 * a + 2];
    }
  } else if (kind == kAxisY) {
    s = s * P.axis_sign[i];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T m0 = M[3 * a], m2 = M[3 * a + 2];
      R[3 * a + 0] = m0 * c - m2 * s;
      R[3 * a + 1] = M[3 * a + 1];
      R[3 * a + 2] = m0 * s + m2 * c;
    }
  } else if (kind == kAxisX) {
    s = s * P.axis_sign[i];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T m1 = M[3 * a + 1], m2 = M[3 * a + 2];
      R[3 * a + 0] = M[3 * a];
      R[3 * a + 1] = m1 * c + m2 * s;
      R[3 * a + 2] = m2 * c - m1 * s;
    }
  } else {
    const T ux = P.axes[3 * i], uy = P.axes[3 * i + 1], uz = P.axes[3 * i + 2];
    const T *w = P.uu + 6 * i;
    const T ic = T(1) - c;
    const T j00 = c + w[0] * ic, j01 = w[1] * ic - uz * s, j02 = w[2] * ic + uy * s;
    const T j10 = w[1] * ic + uz * s, j11 = c + w[3] * ic, j12 = w[4] * ic - ux * s;
    const T j20 = w[2] * ic - uy * s, j21 = w[4] * ic + ux * s, j22 = c + w[5] * ic;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T m0 = M[3 * a], m1 = M[3 * a + 1], m2 = M[3 * a + 2];
      R[3 * a + 0] = m0 * j00 + m1 * j10 + m2 * j20;
      R[3 * a + 1] = m0 * j01 + m1 * j11 + m2 * j21;
      R[3 * a + 2] = m0 * j02 + m1 * j12 + m2 * j22;
    }
  }
}

// _pose_error + _quad_form (vp/batch.py:69-148).  Returns false at the
// log-map singularity.  fp32 uses theta = atan2(|vee|, cos) (stable at small
// angles); fp64 follows the reference's acos exactly.
template <typename T>
__device__ __forceinline__ bool pose_quad(const Prob<T> &P, const Dyn<T> &D, const T R[9], const T t[3], const T *W,
                                          T *out) {
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
    if (theta >= P.pi_limit) return false;
    scale = theta < 1e-6 ? 1.0 + theta * theta / 6.0 : theta / sin(theta);
  } else {
    const float sn = sqrtf(sx * sx + sy * sy + sz * sz);
    theta = atan2f(sn, c);
    if (theta >= P.pi_limit) return false;
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
  T total = T(0);
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    T row = T(0);
#pragma unroll
    for (int b = 0; b < 6; ++b) row += W[6 * a + b] * xi[b];
    total += xi[a] * row;
  }
  *out = T(0.5) * total;
  return true;
}

template <typename T>
__device__ __forceinline__ T bound_violation(T x, T lo, T hi) {
  // x - clamp(x, lo, hi): x - hi above, x - lo below, exactly 0 inside (lo <
  // hi), the same FADD as the reference's branches (vp/batch.py:140-149)
  if constexpr (sizeof(T) == 4) return x - fminf(fmaxf(x, lo), hi);
  else return x - fmin(fmax(x, lo), hi);
}

}  // namespace vpb
