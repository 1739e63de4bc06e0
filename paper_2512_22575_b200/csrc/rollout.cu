// Fused SMPC rollout + cost kernel, softmin partials and the step finish
// (sm_100a).
//
// Replaces vp/batch.py:161-336 (evaluate_batch), vp/planner.py:373-400
// (soft_weights / update_controls) and the tail of vp/planner.py:594-630
// (smpc_step: U*, re-evaluation, clip, shift).
//
// Work mapping: one warp per candidate, lane = horizon
// step.  The semi-implicit double integrator qd_{k+1} = qd_k + u_k dt,
// q_{k+1} = q_k + qd_{k+1} dt becomes two warp prefix sums per joint, so every
// lane holds its own (q_k, qd_k) and evaluates FK, the SE(3) pose cost, the
// sphere/EDT collision cost, self pairs and the limit/smoothness/null-space
// terms for its step independently.  Horizons > 32 loop over 32-step chunks
// with a carried state.  Each CTA has NW candidate warps plus one terminal
// warp that evaluates the NW terminal costs (FK at q_H) while the candidate
// warps run their steps; q_H is handed over through shared memory and a
// named barrier as soon as the prefix sums are done.
//
// Softmin: each CTA reduces its own candidates to a partial
// (m_c, Z_c = sum exp(-(S - m_c)/lam), N_c = sum exp(...) eps) in fixed order;
// partials are merged in fixed index order by merge_partials_kernel, so the
// result is bitwise reproducible and identical across ranks.
#include <cfloat>

#include "rollout.cuh"

namespace vpb {

constexpr int NW = 8;                    // candidate warps per CTA
constexpr int kThreads = (NW + 1) * 32;  // + terminal warp
constexpr int kPartHead = 4;             // [m, Z, nonfinite, best_index]

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += y;
  }
  return x;
}

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
  return x;
}

template <typename ET>
__device__ __forceinline__ double load_e(const ET *p) {
  return (double)__ldg(p);
}

struct RolloutIO {
  const void *ctrl;        // M x H x n (ET)
  const double *nominal;   // H x n or null
  int64_t M;
  double *costs;           // M
  double *terms;           // M x 6 (may be null)
  uint8_t *flags;          // M
  double *traj_q, *traj_qd, *sph_out;  // optional
  double *parts;           // per-CTA softmin partials (kPartHead + H n) or null
  double lam;
  int64_t m_offset;        // global index of local sample 0 (best_index)
};

template <typename T, typename ET, int MAXJ>
__global__ void __launch_bounds__(kThreads, 2) rollout_kernel(const __grid_constant__ Prob<T> P,
                                                           const __grid_constant__ RolloutIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // shared layout
  T *centers = reinterpret_cast<T *>(smem_raw);  // [NW][ns*3][32]
  const int ns = P.ns;
  const size_t cen_bytes = (((size_t)NW * ns * 3 * 32 * sizeof(T)) + 15) & ~(size_t)15;
  double *sums_s = reinterpret_cast<double *>(smem_raw + cen_bytes);  // [NW][6]
  double *cost_s = sums_s + NW * 6;                                   // [NW]
  T *qH_s = reinterpret_cast<T *>(cost_s + NW);                       // [NW][MAXJ]
  int *fail_s = reinterpret_cast<int *>(qH_s + NW * MAXJ);            // [NW]
  int *tfail_s = fail_s + NW;                                         // [NW]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = P.H, nj = P.nj;
  const int64_t cta_m0 = (int64_t)blockIdx.x * NW;
  const ET *ctrl = reinterpret_cast<const ET *>(io.ctrl);

  if (warp < NW) {
    // ===================== candidate warp =====================
    const int64_t m = cta_m0 + warp;
    const bool valid = m < io.M;
    T *cen = centers + (size_t)warp * ns * 3 * 32 + lane;
    T qc[MAXJ], qdc[MAXJ];
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      qc[j] = j < nj ? P.q0[j] : T(0);
      qdc[j] = j < nj ? P.qd0[j] : T(0);
    }
    T s_pose = 0, s_coll = 0, s_lim = 0, s_smooth = 0, s_null = 0;
    bool fail = false;
    const int nchunks = (H + 31) >> 5;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int k = ch * 32 + lane;
      const bool act = valid && k < H;
      T u[MAXJ], q[MAXJ], qd[MAXJ];
      // load u_k = nominal_k + ctrl_k; prefix sums for the double integrator
#pragma unroll
      for (int j = 0; j < MAXJ; ++j) {
        T uj = T(0);
        if (j < nj && act) {
          const size_t off = ((size_t)m * H + k) * nj + j;
          double v = load_e<ET>(ctrl + off);
          if (io.nominal) v += io.nominal[(size_t)k * nj + j];
          uj = (T)v;
        }
        u[j] = uj;
        const T vdt = uj * P.dt;                         // u_k dt
        const T vin = warp_incl_scan<T>(vdt, lane);      // sum_{<=k}
        const T vex = vin - vdt;
        qd[j] = qdc[j] + vex;                            // qd_k
        const T qdn = act ? (qdc[j] + vin) : T(0);       // qd_{k+1}
        const T w = qdn * P.dt;
        const T win = warp_incl_scan<T>(w, lane);
        q[j] = qc[j] + (win - w);                        // q_k
        qdc[j] += __shfl_sync(kFull, vin, 31);
        qc[j] += __shfl_sync(kFull, win, 31);
      }
      if (ch == nchunks - 1) {
        // hand q_H to the terminal warp as early as possible
        if (lane == 0) {
#pragma unroll
          for (int j = 0; j < MAXJ; ++j) qH_s[warp * MAXJ + j] = qc[j];
          if (valid && io.traj_q) {
#pragma unroll
            for (int j = 0; j < MAXJ; ++j) {
              if (j < nj) {
                io.traj_q[((size_t)m * (H + 1) + H) * nj + j] = (double)qc[j];
                io.traj_qd[((size_t)m * (H + 1) + H) * nj + j] = (double)qdc[j];
              }
            }
          }
        }
        __syncwarp();
        named_bar_arrive(1, kThreads);
      }
      if (act) {
        if (io.traj_q) {
#pragma unroll
          for (int j = 0; j < MAXJ; ++j) {
            if (j < nj) {
              io.traj_q[((size_t)m * (H + 1) + k) * nj + j] = (double)q[j];
              io.traj_qd[((size_t)m * (H + 1) + k) * nj + j] = (double)qd[j];
            }
          }
        }
        // limits / smoothness / null space first (vp/batch.py:303-311) so u
        // and qd are dead before the FK
        T lim = 0, sm = 0, nu = 0;
#pragma unroll
        for (int j = 0; j < MAXJ; ++j) {
          if (j < nj) {
            const T vq = bound_violation<T>(q[j], P.pos_lo[j], P.pos_hi[j]);
            const T vv = bound_violation<T>(qd[j], P.vel_lo[j], P.vel_hi[j]);
            const T va = bound_violation<T>(u[j], P.acc_lo[j], P.acc_hi[j]);
            lim += P.w_q * vq * vq + P.w_qd * vv * vv + P.w_qdd * va * va;
            sm += P.w_s * u[j] * u[j];
            const T dq = q[j] - P.q_ref[j];
            nu += P.w_ns * dq * dq;
          }
        }
        s_lim += lim;
        s_smooth += sm;
        s_null += nu;
        // ---- FK; sphere centres emitted link by link into shared memory ----
        T R[9], t[3];
#pragma unroll
        for (int a = 0; a < 9; ++a) R[a] = P.base_r[a];
        t[0] = P.base_t[0];
        t[1] = P.base_t[1];
        t[2] = P.base_t[2];
#pragma unroll
        for (int li = 0; li <= MAXJ; ++li) {
          if (li > nj) break;
          if (li > 0) fk_link<T>(P, li - 1, q[li - 1], R, t);
          for (int s = P.sph_begin[li]; s < P.sph_begin[li + 1]; ++s) {
            const T lx = P.sph_loc[3 * s], ly = P.sph_loc[3 * s + 1], lz = P.sph_loc[3 * s + 2];
            const T px = R[0] * lx + R[1] * ly + R[2] * lz + t[0];
            const T py = R[3] * lx + R[4] * ly + R[5] * lz + t[1];
            const T pz = R[6] * lx + R[7] * ly + R[8] * lz + t[2];
            cen[(3 * s + 0) * 32] = px;
            cen[(3 * s + 1) * 32] = py;
            cen[(3 * s + 2) * 32] = pz;
            if (io.sph_out) {
              double *o = io.sph_out + (((size_t)m * H + k) * ns + P.sph_orig[s]) * 3;
              o[0] = (double)px;
              o[1] = (double)py;
              o[2] = (double)pz;
            }
          }
        }
        T pc;
        if (!pose_quad<T>(P, R, t, P.Q, &pc)) {
          fail = true;
          pc = T(0);
        }
        s_pose += pc;
        T coll = T(0);
        // environment term (vp/batch.py:250-293): two spheres per batch, all
        // sixteen corner loads in flight before any is consumed
        if (P.has_field) {
          for (int s0 = 0; s0 < ns; s0 += 2) {
            Query<T> Qa, Qb;
            const bool hb = s0 + 1 < ns;
            query_issue<T>(P, cen[(3 * s0) * 32], cen[(3 * s0 + 1) * 32], cen[(3 * s0 + 2) * 32], Qa);
            const int s1 = hb ? s0 + 1 : s0;
            query_issue<T>(P, cen[(3 * s1) * 32], cen[(3 * s1 + 1) * 32], cen[(3 * s1 + 2) * 32], Qb);
            const T da = query_finish<T>(P, Qa);
            const T ga = P.d_act - (da - P.sph_r[s0]);
            if (ga > T(0)) coll += P.w_env * ga * ga;
            if (hb) {
              const T db = query_finish<T>(P, Qb);
              const T gb = P.d_act - (db - P.sph_r[s1]);
              if (gb > T(0)) coll += P.w_env * gb * gb;
            }
          }
        }
        // self pairs (vp/batch.py:294-302)
        for (int p = 0; p < P.np; ++p) {
          const int i = P.pairs[2 * p], jj = P.pairs[2 * p + 1];
          const T dx = cen[(3 * i) * 32] - cen[(3 * jj) * 32];
          const T dy = cen[(3 * i + 1) * 32] - cen[(3 * jj + 1) * 32];
          const T dz = cen[(3 * i + 2) * 32] - cen[(3 * jj + 2) * 32];
          const T gap = tsqrt<T>(dx * dx + dy * dy + dz * dz) - (P.sph_r[i] + P.sph_r[jj]);
          if (gap < T(0)) coll += P.w_self * gap * gap;
        }
        s_coll += coll;
      }
    }
    // fixed-order warp reduction in fp64
    const double r_pose = warp_sum_d((double)s_pose);
    const double r_coll = warp_sum_d((double)s_coll);
    const double r_lim = warp_sum_d((double)s_lim);
    const double r_smooth = warp_sum_d((double)s_smooth);
    const double r_null = warp_sum_d((double)s_null);
    const bool any_fail = __any_sync(kFull, fail);
    if (lane == 0) {
      double *sm = sums_s + warp * 6;
      sm[0] = r_pose;
      sm[1] = r_coll;
      sm[2] = r_lim;
      sm[3] = r_smooth;
      sm[4] = r_null;
      fail_s[warp] = any_fail ? 1 : 0;
    }
  } else {
    // ===================== terminal warp =====================
    named_bar_sync(1, kThreads);
    const int64_t m = cta_m0 + lane;
    if (lane < NW && m < io.M) {
      T R[9], t[3];
#pragma unroll
      for (int a = 0; a < 9; ++a) R[a] = P.base_r[a];
      t[0] = P.base_t[0];
      t[1] = P.base_t[1];
      t[2] = P.base_t[2];
#pragma unroll
      for (int i = 0; i < MAXJ; ++i) {
        if (i < nj) fk_link<T>(P, i, qH_s[lane * MAXJ + i], R, t);
      }
      T tc;
      const bool ok = pose_quad<T>(P, R, t, P.QH, &tc);
      cost_s[lane] = ok ? (double)tc : 0.0;
      tfail_s[lane] = ok ? 0 : 1;
    }
  }
  __syncthreads();

  // ===================== finalize costs =====================
  if (threadIdx.x < NW) {
    const int w = threadIdx.x;
    const int64_t m = cta_m0 + w;
    if (m < io.M) {
      const double *sm = sums_s + w * 6;
      const bool failed = fail_s[w] != 0 || tfail_s[w] != 0;
      const double term = cost_s[w];
      const double total = sm[0] + sm[1] + sm[2] + sm[3] + sm[4] + term;
      io.flags[m] = failed ? 1 : 0;
      io.costs[m] = failed ? __longlong_as_double(0x7ff0000000000000ll) : total;
      if (io.terms) {
        double *tr = io.terms + (size_t)m * 6;
        if (failed) {
#pragma unroll
          for (int a = 0; a < 6; ++a) tr[a] = 0.0;
        } else {
          tr[0] = sm[0];
          tr[1] = sm[1];
          tr[2] = sm[2];
          tr[3] = sm[3];
          tr[4] = sm[4];
          tr[5] = term;
        }
      }
      sums_s[w * 6 + 5] = failed ? __longlong_as_double(0x7ff0000000000000ll) : total;
    } else {
      sums_s[w * 6 + 5] = __longlong_as_double(0x7ff0000000000000ll);
    }
  }
  if (io.parts == nullptr) return;
  __syncthreads();

  // ===================== softmin partial of this CTA =====================
  // fixed order over the NW candidates (vp/planner.py:373-400 restated as a
  // shift-invariant partial)
  const int hn = H * nj;
  double mn = __longlong_as_double(0x7ff0000000000000ll);
  int best = -1, nonfinite = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const double c = sums_s[w * 6 + 5];
    if (cta_m0 + w >= io.M) continue;
    if (!(c < __longlong_as_double(0x7ff0000000000000ll))) {
      ++nonfinite;
      continue;
    }
    if (c < mn) {
      mn = c;
      best = w;
    }
  }
  double wt[NW];
  double Z = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const double c = sums_s[w * 6 + 5];
    const bool ok = (cta_m0 + w < io.M) && (c < __longlong_as_double(0x7ff0000000000000ll));
    wt[w] = ok ? exp(-(c - mn) / io.lam) : 0.0;
    Z += wt[w];
  }
  double *part = io.parts + (size_t)blockIdx.x * (kPartHead + hn);
  if (threadIdx.x == 0) {
    part[0] = mn;
    part[1] = Z;
    part[2] = (double)nonfinite;
    part[3] = best >= 0 ? (double)(io.m_offset + cta_m0 + best) : -1.0;
  }
  for (int e = threadIdx.x; e < hn; e += blockDim.x) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      if (wt[w] != 0.0) acc += wt[w] * load_e<ET>(ctrl + (size_t)(cta_m0 + w) * hn + e);
    }
    part[kPartHead + e] = acc;
  }
}

// Merge consecutive groups of `group` partials (fixed order) into one each.
// parts: P x L, out: ceil(P/group) x L.  L = kPartHead + hn.
__global__ void __launch_bounds__(256) merge_partials_kernel(const double *__restrict__ parts, int64_t P,
                                                             int64_t group, int64_t hn, double lam,
                                                             double *__restrict__ out) {
  __shared__ double scale_s[1024];
  __shared__ double mn_s, bestidx_s;
  const int64_t L = kPartHead + hn;
  const int64_t g0 = (int64_t)blockIdx.x * group;
  const int64_t cnt = vmin64(group, P - g0);
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  if (threadIdx.x == 0) {
    double mn = INF, bi = -1.0;
    for (int64_t i = 0; i < cnt; ++i) {
      const double v = parts[(g0 + i) * L + 0];
      if (v < mn) {
        mn = v;
        bi = parts[(g0 + i) * L + 3];
      }
    }
    mn_s = mn;
    bestidx_s = bi;
  }
  __syncthreads();
  const double mn = mn_s;
  for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
    const double v = parts[(g0 + i) * L + 0];
    scale_s[i] = (v < INF) ? exp(-(v - mn) / lam) : 0.0;
  }
  __syncthreads();
  double *o = out + (int64_t)blockIdx.x * L;
  if (threadIdx.x == 0) {
    double Z = 0.0, nf = 0.0;
    for (int64_t i = 0; i < cnt; ++i) {
      if (scale_s[i] != 0.0) Z += scale_s[i] * parts[(g0 + i) * L + 1];
      nf += parts[(g0 + i) * L + 2];
    }
    o[0] = mn;
    o[1] = Z;
    o[2] = nf;
    o[3] = bestidx_s;
  }
  for (int64_t e = threadIdx.x; e < hn; e += blockDim.x) {
    double acc = 0.0;
    for (int64_t i = 0; i < cnt; ++i)
      if (scale_s[i] != 0.0) acc += scale_s[i] * parts[(g0 + i) * L + kPartHead + e];
    o[kPartHead + e] = acc;
  }
}

// U* = nominal + N / Z ; command = clip(U*[0]); next = [U*[1:], 0].
// out layout: [U* (hn), command (n), next (hn), wcost, terms6, best, Z, nonfinite, wflag]
struct AccLimit {
  double v[kMaxJ];
};

__global__ void finish_kernel(const double *__restrict__ part, const double *__restrict__ nominal, int64_t H,
                              int64_t n, const AccLimit acc, double *__restrict__ out) {
  const int64_t hn = H * n;
  const double Z = part[1];
  for (int64_t e = threadIdx.x; e < hn; e += blockDim.x) {
    const double u = nominal[e] + part[kPartHead + e] / Z;
    out[e] = u;
    if (e < n) {
      const double lim = acc.v[e];
      out[hn + e] = u < -lim ? -lim : (u > lim ? lim : u);
    }
    if (e >= n) out[hn + n + (e - n)] = u;
  }
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) out[hn + n + hn - n + e] = 0.0;
  if (threadIdx.x == 0) {
    const int64_t base = 2 * hn + n;
    out[base + 7] = part[0];  // best cost
    out[base + 8] = Z;
    out[base + 9] = part[2];  // nonfinite count
    out[base + 10] = part[3]; // index of the best sample
  }
}

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

// ---------------------------------------------------------------------------
// host-side helpers
// ---------------------------------------------------------------------------
template <typename T>
static int build_prob(const vpb_problem *p, const vpb_field *f, Prob<T> &P) {
  memset(&P, 0, sizeof(P));
  VPB_REQUIRE(p->n_joints >= 1 && p->n_joints <= kMaxJ, "n_joints %d outside [1, %d]", p->n_joints, kMaxJ);
  VPB_REQUIRE(p->n_spheres >= 0 && p->n_spheres <= kMaxS, "n_spheres %d outside [0, %d]", p->n_spheres, kMaxS);
  VPB_REQUIRE(p->n_pairs >= 0 && p->n_pairs <= kMaxP, "n_pairs %d outside [0, %d]", p->n_pairs, kMaxP);
  VPB_REQUIRE(p->horizon >= 1, "horizon must be >= 1");
  const int nj = p->n_joints, ns = p->n_spheres;
  P.nj = nj;
  P.ns = ns;
  P.np = p->n_pairs;
  P.H = p->horizon;
  P.dt = (T)p->dt;
  P.lam = (T)p->lam;
  for (int a = 0; a < 9; ++a) {
    P.base_r[a] = (T)p->base_r[a];
    P.goal_r[a] = (T)p->goal_r[a];
  }
  for (int a = 0; a < 3; ++a) {
    P.base_t[a] = (T)p->base_t[a];
    P.goal_t[a] = (T)p->goal_t[a];
  }
  for (int a = 0; a < 36; ++a) {
    P.Q[a] = (T)p->pose_weight[a];
    P.QH[a] = (T)p->terminal_weight[a];
  }
  for (int i = 0; i < nj; ++i) {
    bool ident = true;
    for (int a = 0; a < 9; ++a) {
      P.off_r[9 * i + a] = (T)p->off_r[9 * i + a];
      const double want = (a % 4 == 0) ? 1.0 : 0.0;
      if (p->off_r[9 * i + a] != want) ident = false;
    }
    P.off_identity[i] = ident ? 1 : 0;
    const double ux = p->axes[3 * i], uy = p->axes[3 * i + 1], uz = p->axes[3 * i + 2];
    for (int a = 0; a < 3; ++a) {
      P.off_t[3 * i + a] = (T)p->off_t[3 * i + a];
      P.axes[3 * i + a] = (T)p->axes[3 * i + a];
    }
    P.uu[6 * i + 0] = (T)(ux * ux);
    P.uu[6 * i + 1] = (T)(ux * uy);
    P.uu[6 * i + 2] = (T)(ux * uz);
    P.uu[6 * i + 3] = (T)(uy * uy);
    P.uu[6 * i + 4] = (T)(uy * uz);
    P.uu[6 * i + 5] = (T)(uz * uz);
    P.axis_kind[i] = kAxisGeneral;
    P.axis_sign[i] = (T)1;
    if (ux == 0.0 && uy == 0.0 && (uz == 1.0 || uz == -1.0)) {
      P.axis_kind[i] = kAxisZ;
      P.axis_sign[i] = (T)uz;
    } else if (ux == 0.0 && uz == 0.0 && (uy == 1.0 || uy == -1.0)) {
      P.axis_kind[i] = kAxisY;
      P.axis_sign[i] = (T)uy;
    } else if (uy == 0.0 && uz == 0.0 && (ux == 1.0 || ux == -1.0)) {
      P.axis_kind[i] = kAxisX;
      P.axis_sign[i] = (T)ux;
    }
    P.pos_lo[i] = (T)p->pos_lo[i];
    P.pos_hi[i] = (T)p->pos_hi[i];
    P.vel_lo[i] = (T)p->vel_lo[i];
    P.vel_hi[i] = (T)p->vel_hi[i];
    P.acc_lo[i] = (T)p->acc_lo[i];
    P.acc_hi[i] = (T)p->acc_hi[i];
    P.q_ref[i] = (T)p->q_ref[i];
    P.q0[i] = (T)p->q0[i];
    P.qd0[i] = (T)p->qd0[i];
  }
  // spheres sorted by link -> per-link ranges
  int prev = 0;
  for (int s = 0; s < ns; ++s) {
    const int l = p->sph_link[s];
    VPB_REQUIRE(l >= 0 && l <= nj, "sphere %d attached to link %d outside [0, %d]", s, l, nj);
    VPB_REQUIRE(l >= prev, "spheres must be sorted by link");
    prev = l;
    for (int a = 0; a < 3; ++a) P.sph_loc[3 * s + a] = (T)p->sph_loc[3 * s + a];
    P.sph_r[s] = (T)p->sph_r[s];
    P.sph_orig[s] = (int16_t)p->sph_orig[s];
  }
  for (int l = 0; l <= nj + 1; ++l) {
    int b = 0;
    while (b < ns && p->sph_link[b] < l) ++b;
    P.sph_begin[l] = (int16_t)b;
  }
  for (int q = 0; q < p->n_pairs; ++q) {
    const int i = p->pairs[2 * q], j = p->pairs[2 * q + 1];
    VPB_REQUIRE(i >= 0 && i < ns && j >= 0 && j < ns, "pair %d references an unknown sphere", q);
    P.pairs[2 * q] = (int16_t)i;
    P.pairs[2 * q + 1] = (int16_t)j;
  }
  P.w_env = (T)p->w_env;
  P.w_self = (T)p->w_self;
  P.w_q = (T)p->w_q;
  P.w_qd = (T)p->w_qd;
  P.w_qdd = (T)p->w_qdd;
  P.w_s = (T)p->w_s;
  P.w_ns = (T)p->w_ns;
  P.d_act = (T)p->d_act;
  P.pi_limit = (T)(3.141592653589793 - 1e-6);
  if (f && f->sq) {
    VPB_REQUIRE(f->n[0] >= 1 && f->n[1] >= 1 && f->n[2] >= 1, "empty field");
    VPB_REQUIRE(f->n[0] * f->n[1] * f->n[2] < ((int64_t)1 << 40), "field too large");
    P.sq = f->sq;
    P.has_field = 1;
    P.n0 = (int)f->n[0];
    P.n1 = (int)f->n[1];
    P.n2 = (int)f->n[2];
    P.lo0 = (T)f->lo[0];
    P.lo1 = (T)f->lo[1];
    P.lo2 = (T)f->lo[2];
    P.origin0 = (T)f->origin[0];
    P.origin1 = (T)f->origin[1];
    P.origin2 = (T)f->origin[2];
    P.voxel = (T)f->voxel;
    P.inv_voxel = (T)(1.0 / f->voxel);
    P.outside = (T)f->outside_default;
  }
  return VPB_OK;
}

static size_t rollout_smem(int ns, size_t tsize) {
  return align_up((size_t)NW * ns * 3 * 32 * tsize, 16) + NW * 6 * 8 + NW * 8 + NW * kMaxJ * tsize + 2 * NW * 4 + 64;
}

template <typename T, typename ET>
static int launch_rollout_t(const Prob<T> &P, const RolloutIO &io, cudaStream_t s) {
  const size_t smem = rollout_smem(P.ns, sizeof(T));
  const unsigned grid = (unsigned)ceil_div(io.M, NW);
  if (grid == 0) return VPB_OK;
  if (P.nj <= 8) {
    auto k = rollout_kernel<T, ET, 8>;
    if (smem > 48 * 1024) VPB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, kThreads, smem, s>>>(P, io);
  } else {
    auto k = rollout_kernel<T, ET, kMaxJ>;
    if (smem > 48 * 1024) VPB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, kThreads, smem, s>>>(P, io);
  }
  return check_launch("rollout_kernel");
}

static int launch_rollout(const vpb_problem *prob, const vpb_field *field, int precision, int dtype,
                          const RolloutIO &io, cudaStream_t s) {
  VPB_REQUIRE(dtype == VPB_DTYPE_F32 || dtype == VPB_DTYPE_F64, "bad dtype %d", dtype);
  if (precision == VPB_PREC_F64) {
    Prob<double> P;
    int rc = build_prob<double>(prob, field, P);
    if (rc) return rc;
    return dtype == VPB_DTYPE_F32 ? launch_rollout_t<double, float>(P, io, s)
                                  : launch_rollout_t<double, double>(P, io, s);
  }
  VPB_REQUIRE(precision == VPB_PREC_F32, "bad precision %d", precision);
  Prob<float> P;
  int rc = build_prob<float>(prob, field, P);
  if (rc) return rc;
  return dtype == VPB_DTYPE_F32 ? launch_rollout_t<float, float>(P, io, s) : launch_rollout_t<float, double>(P, io, s);
}

// Deterministic multi-level merge of `count` partials starting at `src` into
// a single partial at `dst`, using `tmp` (same capacity as src) as scratch.
static int merge_all(const double *src, int64_t count, int64_t hn, double lam, double *tmp_a, double *tmp_b,
                     double *dst, cudaStream_t s) {
  const int64_t L = kPartHead + hn;
  const int64_t group = 64;
  const double *cur = src;
  double *bufs[2] = {tmp_a, tmp_b};
  int which = 0;
  while (true) {
    const int64_t outn = ceil_div(count, group);
    double *target = outn == 1 ? dst : bufs[which];
    merge_partials_kernel<<<(unsigned)outn, 256, 0, s>>>(cur, count, group, hn, lam, target);
    int rc = check_launch("merge_partials_kernel");
    if (rc) return rc;
    if (outn == 1) break;
    cur = target;
    count = outn;
    which ^= 1;
  }
  (void)L;
  return VPB_OK;
}

}  // namespace vpb

using namespace vpb;

extern "C" {

int vpb_evaluate_batch(const vpb_problem *prob, const vpb_field *field, const void *controls, const void *nominal,
                       int dtype, int64_t M, int precision, double *costs, double *terms, uint8_t *flags,
                       double *traj_q, double *traj_qd, double *sphere_pos, void *stream) {
  VPB_REQUIRE(prob && controls && costs && flags, "null argument to vpb_evaluate_batch");
  VPB_REQUIRE(M >= 0, "M must be >= 0");
  VPB_REQUIRE((traj_q == nullptr) == (traj_qd == nullptr), "traj_q and traj_qd must both be given or both null");
  RolloutIO io;
  memset(&io, 0, sizeof(io));
  io.ctrl = controls;
  io.nominal = reinterpret_cast<const double *>(nominal);
  io.M = M;
  io.costs = costs;
  io.terms = terms;
  io.flags = flags;
  io.traj_q = traj_q;
  io.traj_qd = traj_qd;
  io.sph_out = sphere_pos;
  io.parts = nullptr;
  io.lam = prob->lam > 0 ? prob->lam : 1.0;
  return launch_rollout(prob, field, precision, dtype, io, as_stream(stream));
}

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

int64_t vpb_smpc_partial_len(int64_t H, int64_t n) { return kPartHead + H * n; }

size_t vpb_smpc_workspace_bytes(int64_t M, int64_t H, int64_t n) {
  const int64_t ctas = ceil_div(M > 0 ? M : 1, NW);
  const int64_t L = kPartHead + H * n;
  // per-CTA partials + two ping-pong merge buffers + M=1 rollout scratch
  return align_up((size_t)ctas * L * 8, 256) * 2 + align_up((size_t)(ctas / 64 + 2) * L * 8, 256) + 4096;
}

int vpb_smpc_partial(const vpb_problem *prob, const vpb_field *field, const void *eps, int dtype,
                     const double *nominal, int64_t M, int64_t m_offset, int precision, double *costs,
                     uint8_t *flags, double *part_out, void *workspace, size_t workspace_bytes, void *stream) {
  VPB_REQUIRE(prob && eps && nominal && costs && flags && part_out && M >= 1, "bad arguments to vpb_smpc_partial");
  VPB_REQUIRE(prob->lam > 0.0, "temperature must be positive");
  const int64_t H = prob->horizon, n = prob->n_joints;
  VPB_REQUIRE(workspace && workspace_bytes >= vpb_smpc_workspace_bytes(M, H, n), "workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t ctas = ceil_div(M, NW);
  const int64_t L = kPartHead + H * n;
  char *ws = reinterpret_cast<char *>(workspace);
  double *parts = reinterpret_cast<double *>(ws);
  double *tmp_a = reinterpret_cast<double *>(ws + align_up((size_t)ctas * L * 8, 256));
  double *tmp_b = reinterpret_cast<double *>(ws + 2 * align_up((size_t)ctas * L * 8, 256));
  RolloutIO io;
  memset(&io, 0, sizeof(io));
  io.ctrl = eps;
  io.nominal = nominal;
  io.M = M;
  io.costs = costs;
  io.terms = nullptr;
  io.flags = flags;
  io.parts = parts;
  io.lam = prob->lam;
  io.m_offset = m_offset;
  int rc = launch_rollout(prob, field, precision, dtype, io, s);
  if (rc) return rc;
  return merge_all(parts, ctas, H * n, prob->lam, tmp_a, tmp_b, part_out, s);
}

int64_t vpb_smpc_out_len(int64_t H, int64_t n) { return 2 * H * n + n + 11; }

size_t vpb_smpc_finish_workspace_bytes(int64_t n_parts, int64_t H, int64_t n) {
  const int64_t L = kPartHead + H * n;
  const int64_t g = ceil_div(n_parts > 0 ? n_parts : 1, 64);
  return align_up((size_t)L * 8, 256) + 2 * align_up((size_t)g * L * 8, 256) + 256;
}

int vpb_smpc_finish(const vpb_problem *prob, const vpb_field *field, const double *partials, int64_t n_parts,
                    const double *nominal, int precision, double *out, void *workspace, size_t workspace_bytes,
                    void *stream) {
  VPB_REQUIRE(prob && partials && nominal && out && n_parts >= 1, "bad arguments to vpb_smpc_finish");
  VPB_REQUIRE(prob->lam > 0.0, "temperature must be positive");
  const int64_t H = prob->horizon, n = prob->n_joints, hn = H * n;
  const int64_t L = kPartHead + hn;
  VPB_REQUIRE(n >= 1 && n <= kMaxJ, "bad joint count");
  VPB_REQUIRE(workspace && workspace_bytes >= vpb_smpc_finish_workspace_bytes(n_parts, H, n), "workspace too small");
  cudaStream_t s = as_stream(stream);
  char *ws = reinterpret_cast<char *>(workspace);
  const int64_t g = ceil_div(n_parts, 64);
  double *merged = reinterpret_cast<double *>(ws);
  double *tmp_a = reinterpret_cast<double *>(ws + align_up((size_t)L * 8, 256));
  double *tmp_b = reinterpret_cast<double *>(ws + align_up((size_t)L * 8, 256) + align_up((size_t)g * L * 8, 256));
  uint8_t *flag1 = reinterpret_cast<uint8_t *>(ws + align_up((size_t)L * 8, 256) + 2 * align_up((size_t)g * L * 8, 256));
  int rc = merge_all(partials, n_parts, hn, prob->lam, tmp_a, tmp_b, merged, s);
  if (rc) return rc;
  AccLimit acc;
  for (int j = 0; j < kMaxJ; ++j) acc.v[j] = j < n ? prob->acc_limit[j] : 0.0;
  finish_kernel<<<1, 256, 0, s>>>(merged, nominal, H, n, acc, out);
  rc = check_launch("finish_kernel");
  if (rc) return rc;
  // Re-evaluate U* (M = 1) for the diagnostics (vp/planner.py:616-617);
  // a flagged re-evaluation shows up as an infinite weighted cost.
  const int64_t base = 2 * hn + n;
  RolloutIO io;
  memset(&io, 0, sizeof(io));
  io.ctrl = out;  // U* (f64)
  io.nominal = nullptr;
  io.M = 1;
  io.costs = out + base;
  io.terms = out + base + 1;
  io.flags = flag1;
  io.lam = prob->lam;
  return launch_rollout(prob, field, precision, VPB_DTYPE_F64, io, s);
}

}  // extern "C"
