// Fused SMPC rollout + cost kernel and the fused SMPC step (sm_100a).
//
// Replaces vp/batch.py:161-336 (evaluate_batch) and vp/planner.py:594-630
// (smpc_step minus sampling: evaluate -> soft_weights -> update_controls ->
// re-evaluate U* -> clip -> shift).
//
// Work mapping: one warp per candidate, lane = horizon
// step.  The semi-implicit double integrator qd_{k+1} = qd_k + u_k dt,
// q_{k+1} = q_k + qd_{k+1} dt becomes two warp prefix sums per joint, so every
// lane holds its own (q_k, qd_k) and evaluates FK, the SE(3) pose cost, the
// sphere/EDT collision cost, self pairs and the limit/smoothness/null-space
// terms of its step independently.  Horizons > 32 loop over 32-step chunks
// with a carried state.  Each CTA has NW candidate warps plus one terminal
// warp that evaluates the NW terminal costs (FK at q_H) while the candidate
// warps run their steps; q_H is handed over through shared memory and a
// named barrier as soon as the prefix sums are done.
//
// SMPC step in one launch: every CTA reduces its candidates to a softmin
// partial (m_c, Z_c = sum exp(-(S - m_c)/lam), N_c = sum exp(...) eps); the
// last CTA of each group of kGroup CTAs merges the group, the last group
// merges the groups (fixed index order at both levels, so the result does
// not depend on which CTA finishes last), and on a single device that same
// CTA computes U* = nominal + N/Z, the clipped command, the shifted warm
// start and re-evaluates U* for the diagnostics.  Across devices the merged
// partial is what ranks all-gather; vpb_smpc_finish merges the
// rank partials in rank order and runs the same tail.
#include <cfloat>

#include "rollout.cuh"

namespace vpb {

constexpr int NW = 8;                    // candidate warps per CTA
constexpr int kThreads = (NW + 1) * 32;  // + terminal warp
constexpr int kPartHead = 4;             // [m, Z, nonfinite, best_index]
constexpr int kGroup = 32;               // CTAs merged by a group's last CTA

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

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000ll); }

template <typename ET>
__device__ __forceinline__ double load_e(const ET *p) {
  return (double)__ldg(p);
}

// ---------------------------------------------------------------------------
// shared memory layout (same computation on host and device)
// ---------------------------------------------------------------------------
struct SmemLayout {
  size_t centers, sums, cost, qH, fail, tfail, dyn, misc, scratch, total;
};

__host__ __device__ inline size_t al16(size_t v) { return (v + 15) & ~(size_t)15; }

__host__ __device__ inline SmemLayout smem_layout(int ns, size_t tsize, int scratch_doubles) {
  SmemLayout L;
  size_t o = 0;
  L.centers = o;
  o = al16(o + (size_t)NW * (ns > 0 ? ns : 1) * 3 * 32 * tsize);
  L.sums = o;
  o = al16(o + (size_t)NW * 6 * 8);
  L.cost = o;
  o = al16(o + (size_t)NW * 8);
  L.qH = o;
  o = al16(o + (size_t)NW * kMaxJ * tsize);
  L.fail = o;
  o = al16(o + (size_t)NW * 4);
  L.tfail = o;
  o = al16(o + (size_t)NW * 4);
  L.dyn = o;
  o = al16(o + (size_t)(2 * kMaxJ + 12) * tsize);
  L.misc = o;  // 32 doubles of reduction scratch + flags
  o = al16(o + 48 * 8);
  L.scratch = o;  // merge scales
  o = al16(o + (size_t)(scratch_doubles > 0 ? scratch_doubles : 1) * 8);
  L.total = o;
  return L;
}

template <typename T>
__device__ __forceinline__ void load_dyn(const Prob<T> &P, const double *dyn, Dyn<T> &D) {
  // called by one warp; the caller synchronises
  const int lane = threadIdx.x & 31;
  const int nj = P.nj;
  for (int i = lane; i < 2 * kMaxJ + 12; i += 32) {
    T v;
    if (i < kMaxJ) v = i < nj ? (dyn ? (T)dyn[i] : P.q0[i]) : T(0);
    else if (i < 2 * kMaxJ) v = (i - kMaxJ) < nj ? (dyn ? (T)dyn[nj + i - kMaxJ] : P.qd0[i - kMaxJ]) : T(0);
    else if (i < 2 * kMaxJ + 9) v = dyn ? (T)dyn[2 * nj + i - 2 * kMaxJ] : P.goal_r[i - 2 * kMaxJ];
    else v = dyn ? (T)dyn[2 * nj + 9 + i - 2 * kMaxJ - 9] : P.goal_t[i - 2 * kMaxJ - 9];
    if (i < kMaxJ) D.q0[i] = v;
    else if (i < 2 * kMaxJ) D.qd0[i - kMaxJ] = v;
    else if (i < 2 * kMaxJ + 9) D.goal_r[i - 2 * kMaxJ] = v;
    else D.goal_t[i - 2 * kMaxJ - 9] = v;
  }
}

struct CandOut {
  double *traj_q, *traj_qd, *sph_out;  // optional (null = not stored)
};

// ---------------------------------------------------------------------------
// One candidate on one warp (lane = step).  Writes the five running-cost sums
// (fp64, fixed-order warp reduction) and the failure flag to shared memory,
// publishes q_H and arrives on barrier `bar_id` (count `bar_count`) for the
// terminal warp.  u_k = nominal_k (optional, f64) + ctrl[k] (ET).
// ---------------------------------------------------------------------------
template <typename T, typename ET, int MAXJ>
__device__ __forceinline__ void candidate_warp(const Prob<T> &P, const Dyn<T> &D, const ET *ctrl,
                                               const double *nominal, int64_t m, bool valid, T *cen, T *qH_slot,
                                               double *sums_slot, int *fail_slot, const CandOut &co, int bar_id,
                                               int bar_count) {
  const int lane = threadIdx.x & 31;
  const int H = P.H, nj = P.nj, ns = P.ns;
  T qc[MAXJ], qdc[MAXJ];
#pragma unroll
  for (int j = 0; j < MAXJ; ++j) {
    qc[j] = j < nj ? D.q0[j] : T(0);
    qdc[j] = j < nj ? D.qd0[j] : T(0);
  }
  T s_pose = 0, s_coll = 0, s_lim = 0, s_smooth = 0, s_null = 0;
  bool fail = false;
  const int nchunks = (H + 31) >> 5;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int k = ch * 32 + lane;
    const bool act = valid && k < H;
    T u[MAXJ], q[MAXJ], qd[MAXJ];
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      T uj = T(0);
      if (j < nj && act) {
        double v = load_e<ET>(ctrl + (size_t)k * nj + j);
        if (nominal) v += nominal[(size_t)k * nj + j];
        uj = (T)v;
      }
      u[j] = uj;
      const T vdt = uj * P.dt;                     // u_k dt
      const T vin = warp_incl_scan<T>(vdt, lane);  // sum_{<=k}
      qd[j] = qdc[j] + (vin - vdt);                // qd_k
      const T qdn = act ? (qdc[j] + vin) : T(0);   // qd_{k+1}
      const T w = qdn * P.dt;
      const T win = warp_incl_scan<T>(w, lane);
      q[j] = qc[j] + (win - w);                    // q_k
      qdc[j] += __shfl_sync(kFull, vin, 31);
      qc[j] += __shfl_sync(kFull, win, 31);
    }
    if (ch == nchunks - 1) {
      // hand q_H to the terminal warp as early as possible
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < MAXJ; ++j) qH_slot[j] = qc[j];
        if (valid && co.traj_q) {
#pragma unroll
          for (int j = 0; j < MAXJ; ++j) {
            if (j < nj) {
              co.traj_q[((size_t)m * (H + 1) + H) * nj + j] = (double)qc[j];
              co.traj_qd[((size_t)m * (H + 1) + H) * nj + j] = (double)qdc[j];
            }
          }
        }
      }
      __syncwarp();
      if (bar_id >= 0) named_bar_arrive(bar_id, bar_count);
    }
    if (act) {
      if (co.traj_q) {
#pragma unroll
        for (int j = 0; j < MAXJ; ++j) {
          if (j < nj) {
            co.traj_q[((size_t)m * (H + 1) + k) * nj + j] = (double)q[j];
            co.traj_qd[((size_t)m * (H + 1) + k) * nj + j] = (double)qd[j];
          }
        }
      }
      // limits / smoothness / null space first (vp/batch.py:303-311) so u and
      // qd are dead before the FK
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
          if (co.sph_out) {
            double *o = co.sph_out + (((size_t)m * H + k) * ns + P.sph_orig[s]) * 3;
            o[0] = (double)px;
            o[1] = (double)py;
            o[2] = (double)pz;
          }
        }
      }
      T pc;
      if (!pose_quad<T>(P, D, R, t, P.Q, &pc)) {
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
    sums_slot[0] = r_pose;
    sums_slot[1] = r_coll;
    sums_slot[2] = r_lim;
    sums_slot[3] = r_smooth;
    sums_slot[4] = r_null;
    *fail_slot = any_fail ? 1 : 0;
  }
}

// Terminal cost at q_H (vp/batch.py:319-328).
template <typename T, int MAXJ>
__device__ __forceinline__ bool terminal_cost(const Prob<T> &P, const Dyn<T> &D, const T *qH, double *cost) {
  T R[9], t[3];
#pragma unroll
  for (int a = 0; a < 9; ++a) R[a] = P.base_r[a];
  t[0] = P.base_t[0];
  t[1] = P.base_t[1];
  t[2] = P.base_t[2];
#pragma unroll
  for (int i = 0; i < MAXJ; ++i) {
    if (i < P.nj) fk_link<T>(P, i, qH[i], R, t);
  }
  T tc;
  const bool ok = pose_quad<T>(P, D, R, t, P.QH, &tc);
  *cost = ok ? (double)tc : 0.0;
  return ok;
}

struct Shared {
  void *centers;
  double *sums, *cost;
  void *qH;
  int *fail, *tfail;
  void *dyn;
  double *misc, *scratch;
};

__device__ __forceinline__ Shared carve(unsigned char *base, const SmemLayout &L) {
  Shared S;
  S.centers = base + L.centers;
  S.sums = reinterpret_cast<double *>(base + L.sums);
  S.cost = reinterpret_cast<double *>(base + L.cost);
  S.qH = base + L.qH;
  S.fail = reinterpret_cast<int *>(base + L.fail);
  S.tfail = reinterpret_cast<int *>(base + L.tfail);
  S.dyn = base + L.dyn;
  S.misc = reinterpret_cast<double *>(base + L.misc);
  S.scratch = reinterpret_cast<double *>(base + L.scratch);
  return S;
}

// Evaluate NW candidates starting at cta_m0 (candidate warps + terminal warp),
// leaving per-warp sums in S.sums, terminal costs in S.cost and flags in
// S.fail / S.tfail.  Ends with __syncthreads().
template <typename T, typename ET, int MAXJ>
__device__ __forceinline__ void evaluate_cta(const Prob<T> &P, const Dyn<T> &D, const ET *ctrl, const double *nominal,
                                             int64_t M, int64_t cta_m0, const Shared &S, const CandOut &co) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ns = P.ns, H = P.H, nj = P.nj;
  T *centers = reinterpret_cast<T *>(S.centers);
  T *qH_s = reinterpret_cast<T *>(S.qH);
  if (warp < NW) {
    const int64_t m = cta_m0 + warp;
    const bool valid = m < M;
    T *cen = centers + (size_t)warp * (ns > 0 ? ns : 1) * 3 * 32 + lane;
    candidate_warp<T, ET, MAXJ>(P, D, ctrl + (valid ? (size_t)m * H * nj : 0), nominal, m, valid, cen,
                                qH_s + warp * kMaxJ, S.sums + warp * 6, S.fail + warp, co, 1, kThreads);
  } else {
    named_bar_sync(1, kThreads);
    const int64_t m = cta_m0 + lane;
    if (lane < NW && m < M) {
      double c;
      const bool ok = terminal_cost<T, MAXJ>(P, D, qH_s + lane * kMaxJ, &c);
      S.cost[lane] = c;
      S.tfail[lane] = ok ? 0 : 1;
    }
  }
  __syncthreads();
}

struct RolloutIO {
  const void *ctrl;       // M x H x n (ET)
  const double *nominal;  // H x n or null
  int64_t M;
  double *costs;   // M
  double *terms;   // M x 6 (may be null)
  uint8_t *flags;  // M
  double *traj_q, *traj_qd, *sph_out;  // optional
  const double *dyn;                   // per-call state or null
};

// evaluate_batch (vp/batch.py:161-336)
template <typename T, typename ET, int MAXJ>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? 2 : 1) rollout_kernel(const __grid_constant__ Prob<T> P,
                                                              const __grid_constant__ RolloutIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SmemLayout L = smem_layout(P.ns, sizeof(T), 0);
  const Shared S = carve(smem_raw, L);
  Dyn<T> &D = *reinterpret_cast<Dyn<T> *>(S.dyn);
  if (threadIdx.x < 32) load_dyn<T>(P, io.dyn, D);
  __syncthreads();
  const int64_t cta_m0 = (int64_t)blockIdx.x * NW;
  CandOut co{io.traj_q, io.traj_qd, io.sph_out};
  evaluate_cta<T, ET, MAXJ>(P, D, reinterpret_cast<const ET *>(io.ctrl), io.nominal, io.M, cta_m0, S, co);
  if (threadIdx.x < NW) {
    const int w = threadIdx.x;
    const int64_t m = cta_m0 + w;
    if (m < io.M) {
      const double *sm = S.sums + w * 6;
      const bool failed = S.fail[w] != 0 || S.tfail[w] != 0;
      const double term = S.cost[w];
      io.flags[m] = failed ? 1 : 0;
      io.costs[m] = failed ? dinf() : sm[0] + sm[1] + sm[2] + sm[3] + sm[4] + term;
      if (io.terms) {
        double *tr = io.terms + (size_t)m * 6;
        for (int a = 0; a < 5; ++a) tr[a] = failed ? 0.0 : sm[a];
        tr[5] = failed ? 0.0 : term;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// deterministic block-wide merge of `count` partials (fixed index order)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_sum_fixed(double v, double *misc) {
  // warp xor-tree (fixed pattern) then warps in order
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum_d(v);
  __syncthreads();
  if (lane == 0) misc[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += misc[w];
  __syncthreads();
  return t;
}

__device__ void merge_block(const double *src, int count, int hn, double lam, double *dst, double *scale,
                            double *misc) {
  const int L = kPartHead + hn;
  const int tid = threadIdx.x, nt = blockDim.x;
  // min (exact, order-free) with the smallest index among equal minima
  double mn = dinf();
  double bi = -1.0;
  int bidx = 0x7fffffff;
  for (int i = tid; i < count; i += nt) {
    const double v = src[(size_t)i * L];
    if (v < mn || (v == mn && i < bidx)) {
      mn = v;
      bidx = i;
    }
  }
  // warp argmin
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    const double ov = __shfl_xor_sync(kFull, mn, d);
    const int oi = __shfl_xor_sync(kFull, bidx, d);
    if (ov < mn || (ov == mn && oi < bidx)) {
      mn = ov;
      bidx = oi;
    }
  }
  __syncthreads();
  if ((tid & 31) == 0) {
    misc[tid >> 5] = mn;
    misc[16 + (tid >> 5)] = (double)bidx;
  }
  __syncthreads();
  if (tid == 0) {
    double m0 = dinf();
    int b0 = 0x7fffffff;
    for (int w = 0; w < (nt >> 5); ++w) {
      const double v = misc[w];
      const int b = (int)misc[16 + w];
      if (v < m0 || (v == m0 && b < b0)) {
        m0 = v;
        b0 = b;
      }
    }
    misc[40] = m0;
    misc[41] = (b0 >= 0 && b0 < count) ? src[(size_t)b0 * L + 3] : -1.0;
  }
  __syncthreads();
  mn = misc[40];
  bi = misc[41];
  for (int i = tid; i < count; i += nt) {
    const double v = src[(size_t)i * L];
    scale[i] = (v < dinf()) ? exp(-(v - mn) / lam) : 0.0;
  }
  __syncthreads();
  double zpart = 0.0, nfpart = 0.0;
  for (int i = tid; i < count; i += nt) {
    if (scale[i] != 0.0) zpart += scale[i] * src[(size_t)i * L + 1];
    nfpart += src[(size_t)i * L + 2];
  }
  const double Z = block_sum_fixed(zpart, misc);
  const double nf = block_sum_fixed(nfpart, misc);
  if (tid == 0) {
    dst[0] = mn;
    dst[1] = Z;
    dst[2] = nf;
    dst[3] = bi;
  }
  for (int e = tid; e < hn; e += nt) {
    double acc = 0.0;
    int i = 0;
    for (; i + 4 <= count; i += 4) {
      const double a0 = src[(size_t)i * L + kPartHead + e];
      const double a1 = src[(size_t)(i + 1) * L + kPartHead + e];
      const double a2 = src[(size_t)(i + 2) * L + kPartHead + e];
      const double a3 = src[(size_t)(i + 3) * L + kPartHead + e];
      if (scale[i] != 0.0) acc += scale[i] * a0;
      if (scale[i + 1] != 0.0) acc += scale[i + 1] * a1;
      if (scale[i + 2] != 0.0) acc += scale[i + 2] * a2;
      if (scale[i + 3] != 0.0) acc += scale[i + 3] * a3;
    }
    for (; i < count; ++i)
      if (scale[i] != 0.0) acc += scale[i] * src[(size_t)i * L + kPartHead + e];
    dst[kPartHead + e] = acc;
  }
  __syncthreads();
}

struct AccLimit {
  double v[kMaxJ];
};

struct SmpcIO {
  const void *eps;        // M x H x n (ET), perturbations of this shard
  const double *nominal;  // H x n
  int64_t M;
  int64_t m_offset;  // global index of local sample 0
  double lam;
  double *costs;     // M or null
  uint8_t *flags;    // M or null
  double *cta_parts;    // [ctas][L]
  double *group_parts;  // [groups][L]
  unsigned int *counters;  // [groups + 1], zero on entry
  double *rank_part;       // [L]
  int finish;              // 1: finish the step in this launch
  double *out;             // step output (see vpb_smpc_out_len)
  AccLimit acc;
  const double *dyn;
};

// U*, clip, shift, then the M = 1 re-evaluation of U* (vp/planner.py:614-629)
// on warps 0 and NW of the calling CTA.  `part` is the fully merged partial.
template <typename T, int MAXJ>
__device__ void smpc_tail(const Prob<T> &P, const Dyn<T> &D, const double *part, const double *nominal,
                          const AccLimit &acc, double *out, const Shared &S) {
  const int H = P.H, n = P.nj, hn = H * n;
  const double Z = part[1];
  for (int e = threadIdx.x; e < hn; e += blockDim.x) {
    const double u = nominal[e] + part[kPartHead + e] / Z;
    out[e] = u;
    if (e < n) {
      const double lim = acc.v[e];
      out[hn + e] = u < -lim ? -lim : (u > lim ? lim : u);
    } else {
      out[hn + n + (e - n)] = u;
    }
  }
  for (int e = threadIdx.x; e < n; e += blockDim.x) out[hn + n + hn - n + e] = 0.0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T *centers = reinterpret_cast<T *>(S.centers);
  T *qH_s = reinterpret_cast<T *>(S.qH);
  CandOut co{nullptr, nullptr, nullptr};
  if (warp == 0) {
    candidate_warp<T, double, MAXJ>(P, D, out, nullptr, 0, true, centers + lane, qH_s, S.sums, S.fail, co, 2, 64);
  } else if (warp == NW) {
    named_bar_sync(2, 64);
    if (lane == 0) {
      double c;
      const bool ok = terminal_cost<T, MAXJ>(P, D, qH_s, &c);
      S.cost[0] = c;
      S.tfail[0] = ok ? 0 : 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t base = 2 * hn + n;
    const bool failed = S.fail[0] != 0 || S.tfail[0] != 0;
    const double *sm = S.sums;
    out[base] = failed ? dinf() : sm[0] + sm[1] + sm[2] + sm[3] + sm[4] + S.cost[0];
    for (int a = 0; a < 5; ++a) out[base + 1 + a] = failed ? 0.0 : sm[a];
    out[base + 6] = failed ? 0.0 : S.cost[0];
    out[base + 7] = part[0];   // best cost
    out[base + 8] = Z;
    out[base + 9] = part[2];   // non-finite sample count
    out[base + 10] = part[3];  // best sample index
  }
}

// Fused SMPC step: rollout -> CTA partial -> group merge -> global merge
// [-> U*, clip, shift, re-evaluation].
template <typename T, typename ET, int MAXJ>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? 2 : 1) smpc_kernel(const __grid_constant__ Prob<T> P,
                                                           const __grid_constant__ SmpcIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ctas = gridDim.x;
  const int groups = (ctas + kGroup - 1) / kGroup;
  const SmemLayout L = smem_layout(P.ns, sizeof(T), groups > kGroup ? groups : kGroup);
  const Shared S = carve(smem_raw, L);
  Dyn<T> &D = *reinterpret_cast<Dyn<T> *>(S.dyn);
  if (threadIdx.x < 32) load_dyn<T>(P, io.dyn, D);
  __syncthreads();
  const int64_t cta_m0 = (int64_t)blockIdx.x * NW;
  const int hn = P.H * P.nj;
  const int Lp = kPartHead + hn;
  const ET *eps = reinterpret_cast<const ET *>(io.eps);
  CandOut co{nullptr, nullptr, nullptr};
  evaluate_cta<T, ET, MAXJ>(P, D, eps, io.nominal, io.M, cta_m0, S, co);

  // ---- per-candidate totals ----
  double *tot = S.misc + 24;  // NW doubles
  if (threadIdx.x < NW) {
    const int w = threadIdx.x;
    const int64_t m = cta_m0 + w;
    double c = dinf();
    bool failed = true;
    if (m < io.M) {
      const double *sm = S.sums + w * 6;
      failed = S.fail[w] != 0 || S.tfail[w] != 0;
      c = failed ? dinf() : sm[0] + sm[1] + sm[2] + sm[3] + sm[4] + S.cost[w];
      if (io.costs) io.costs[m] = c;
      if (io.flags) io.flags[m] = failed ? 1 : 0;
    }
    tot[w] = c;
  }
  __syncthreads();
  // ---- CTA partial (fixed order over the NW candidates) ----
  double *wt_s = S.misc + 32;  // NW weights
  if (threadIdx.x == 0) {
    double mn = dinf();
    int best = -1, nonfinite = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      if (cta_m0 + w >= io.M) continue;
      const double c = tot[w];
      if (!(c < dinf())) {
        ++nonfinite;
        continue;
      }
      if (c < mn) {
        mn = c;
        best = w;
      }
    }
    S.misc[45] = mn;
    S.misc[46] = (double)nonfinite;
    S.misc[47] = best >= 0 ? (double)(io.m_offset + cta_m0 + best) : -1.0;
  }
  __syncthreads();
  if (threadIdx.x < NW) {
    const int w = threadIdx.x;
    const double c = tot[w];
    const bool ok = (cta_m0 + w < io.M) && (c < dinf());
    wt_s[w] = ok ? exp(-(c - S.misc[45]) / io.lam) : 0.0;
  }
  __syncthreads();
  double *part = io.cta_parts + (size_t)blockIdx.x * Lp;
  if (threadIdx.x == 0) {
    double Zc = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) Zc += wt_s[w];
    part[0] = S.misc[45];
    part[1] = Zc;
    part[2] = S.misc[46];
    part[3] = S.misc[47];
  }
  {
    double wt[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) wt[w] = wt_s[w];
    for (int e = threadIdx.x; e < hn; e += blockDim.x) {
      double ev[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w)
        ev[w] = (cta_m0 + w < io.M) ? load_e<ET>(eps + (size_t)(cta_m0 + w) * hn + e) : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w)
        if (wt[w] != 0.0) acc += wt[w] * ev[w];
      part[kPartHead + e] = acc;
    }
  }
  // ---- group merge by the group's last CTA ----
  __threadfence();
  __syncthreads();
  unsigned int *flag = reinterpret_cast<unsigned int *>(S.misc + 44);
  const int g = blockIdx.x / kGroup;
  const int g0 = g * kGroup;
  const int gcount = min(kGroup, ctas - g0);
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(&io.counters[g], 1u);
    flag[0] = (prev == (unsigned int)(gcount - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (flag[0] == 0u) return;
  __threadfence();
  merge_block(io.cta_parts + (size_t)g0 * Lp, gcount, hn, io.lam, io.group_parts + (size_t)g * Lp, S.scratch,
              S.misc);
  if (threadIdx.x == 0) io.counters[g] = 0u;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(&io.counters[groups], 1u);
    flag[0] = (prev == (unsigned int)(groups - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (flag[0] == 0u) return;
  __threadfence();
  merge_block(io.group_parts, groups, hn, io.lam, io.rank_part, S.scratch, S.misc);
  if (threadIdx.x == 0) io.counters[groups] = 0u;
  if (!io.finish) return;
  __threadfence();
  __syncthreads();
  smpc_tail<T, MAXJ>(P, D, io.rank_part, io.nominal, io.acc, io.out, S);
}

// Multi-device finish: merge R rank partials in rank order, then the tail.
template <typename T, int MAXJ>
__global__ void __launch_bounds__(kThreads, 1) smpc_finish_kernel(const __grid_constant__ Prob<T> P,
                                                                   const double *parts, int n_parts, double lam,
                                                                   const double *nominal, const AccLimit acc,
                                                                   double *merged, double *out, const double *dyn) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SmemLayout L = smem_layout(P.ns, sizeof(T), n_parts);
  const Shared S = carve(smem_raw, L);
  Dyn<T> &D = *reinterpret_cast<Dyn<T> *>(S.dyn);
  if (threadIdx.x < 32) load_dyn<T>(P, dyn, D);
  __syncthreads();
  merge_block(parts, n_parts, P.H * P.nj, lam, merged, S.scratch, S.misc);
  __threadfence();
  __syncthreads();
  smpc_tail<T, MAXJ>(P, D, merged, nominal, acc, out, S);
}

// ---------------------------------------------------------------------------
// host side
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


template <typename T>
static size_t smem_bytes(const Prob<T> &P, int scratch) {
  return smem_layout(P.ns, sizeof(T), scratch).total;
}

template <typename K>
static int set_smem(K kern, size_t smem) {
  if (smem > 48 * 1024) VPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return VPB_OK;
}

template <typename T, typename ET>
static int launch_rollout_t(const Prob<T> &P, const RolloutIO &io, cudaStream_t s) {
  const size_t smem = smem_bytes(P, 0);
  const unsigned grid = (unsigned)ceil_div(io.M, NW);
  if (grid == 0) return VPB_OK;
  int rc;
  if (P.nj <= 8) {
    auto k = rollout_kernel<T, ET, 8>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<grid, kThreads, smem, s>>>(P, io);
  } else {
    auto k = rollout_kernel<T, ET, kMaxJ>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<grid, kThreads, smem, s>>>(P, io);
  }
  return check_launch("rollout_kernel");
}

template <typename T, typename ET>
static int launch_smpc_t(const Prob<T> &P, const SmpcIO &io, cudaStream_t s) {
  const int64_t ctas = ceil_div(io.M, NW);
  const int groups = (int)ceil_div(ctas, kGroup);
  const size_t smem = smem_bytes(P, groups > kGroup ? groups : kGroup);
  int rc;
  if (P.nj <= 8) {
    auto k = smpc_kernel<T, ET, 8>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<(unsigned)ctas, kThreads, smem, s>>>(P, io);
  } else {
    auto k = smpc_kernel<T, ET, kMaxJ>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<(unsigned)ctas, kThreads, smem, s>>>(P, io);
  }
  return check_launch("smpc_kernel");
}

template <typename T>
static int launch_finish_t(const Prob<T> &P, const double *parts, int n_parts, double lam, const double *nominal,
                           const AccLimit &acc, double *merged, double *out, const double *dyn, cudaStream_t s) {
  const size_t smem = smem_bytes(P, n_parts);
  int rc;
  if (P.nj <= 8) {
    auto k = smpc_finish_kernel<T, 8>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<1, kThreads, smem, s>>>(P, parts, n_parts, lam, nominal, acc, merged, out, dyn);
  } else {
    auto k = smpc_finish_kernel<T, kMaxJ>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<1, kThreads, smem, s>>>(P, parts, n_parts, lam, nominal, acc, merged, out, dyn);
  }
  return check_launch("smpc_finish_kernel");
}

static AccLimit acc_of(const vpb_problem *p) {
  AccLimit a;
  for (int j = 0; j < kMaxJ; ++j) a.v[j] = j < p->n_joints ? p->acc_limit[j] : 0.0;
  return a;
}

struct SmpcWs {
  double *cta_parts, *group_parts, *rank_part;
  unsigned int *counters;
  size_t bytes;
};

static SmpcWs smpc_ws(void *base, int64_t M, int64_t H, int64_t n) {
  const int64_t ctas = ceil_div(M > 0 ? M : 1, NW);
  const int64_t groups = ceil_div(ctas, kGroup);
  const int64_t L = kPartHead + H * n;
  SmpcWs w;
  char *b = reinterpret_cast<char *>(base);
  size_t o = 0;
  w.cta_parts = reinterpret_cast<double *>(b + o);
  o += align_up((size_t)ctas * L * 8, 256);
  w.group_parts = reinterpret_cast<double *>(b + o);
  o += align_up((size_t)groups * L * 8, 256);
  w.rank_part = reinterpret_cast<double *>(b + o);
  o += align_up((size_t)L * 8, 256);
  w.counters = reinterpret_cast<unsigned int *>(b + o);
  o += align_up((size_t)(groups + 1) * 4, 256);
  w.bytes = o;
  return w;
}

}  // namespace vpb

using namespace vpb;

static int prob_checks(const vpb_problem *prob, int precision, int dtype) {
  VPB_REQUIRE(prob, "null problem");
  VPB_REQUIRE(dtype == VPB_DTYPE_F32 || dtype == VPB_DTYPE_F64, "bad dtype %d", dtype);
  VPB_REQUIRE(precision == VPB_PREC_F32 || precision == VPB_PREC_F64, "bad precision %d", precision);
  return VPB_OK;
}

extern "C" {

int vpb_evaluate_batch(const vpb_problem *prob, const vpb_field *field, const void *controls, const void *nominal,
                       int dtype, int64_t M, int precision, double *costs, double *terms, uint8_t *flags,
                       double *traj_q, double *traj_qd, double *sphere_pos, void *stream) {
  int rc = prob_checks(prob, precision, dtype);
  if (rc) return rc;
  VPB_REQUIRE(controls && costs && flags, "null argument to vpb_evaluate_batch");
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
  io.dyn = prob->dyn_state;
  cudaStream_t s = as_stream(stream);
  if (precision == VPB_PREC_F64) {
    Prob<double> P;
    if ((rc = build_prob<double>(prob, field, P))) return rc;
    return dtype == VPB_DTYPE_F32 ? launch_rollout_t<double, float>(P, io, s) : launch_rollout_t<double, double>(P, io, s);
  }
  Prob<float> P;
  if ((rc = build_prob<float>(prob, field, P))) return rc;
  return dtype == VPB_DTYPE_F32 ? launch_rollout_t<float, float>(P, io, s) : launch_rollout_t<float, double>(P, io, s);
}

int64_t vpb_smpc_partial_len(int64_t H, int64_t n) { return kPartHead + H * n; }

size_t vpb_smpc_workspace_bytes(int64_t M, int64_t H, int64_t n) { return smpc_ws(nullptr, M, H, n).bytes + 256; }

int64_t vpb_smpc_out_len(int64_t H, int64_t n) { return 2 * H * n + n + 11; }

static int smpc_launch(const vpb_problem *prob, const vpb_field *field, const void *eps, int dtype,
                       const double *nominal, int64_t M, int64_t m_offset, int precision, double *costs,
                       uint8_t *flags, double *part_out, double *out, void *workspace, size_t workspace_bytes,
                       cudaStream_t s) {
  int rc = prob_checks(prob, precision, dtype);
  if (rc) return rc;
  VPB_REQUIRE(eps && nominal && M >= 1, "bad arguments to the SMPC step");
  VPB_REQUIRE(prob->lam > 0.0, "temperature must be positive");
  const int64_t H = prob->horizon, n = prob->n_joints;
  VPB_REQUIRE(M <= ((int64_t)1 << 31) * NW, "too many samples");
  const SmpcWs w = smpc_ws(workspace, M, H, n);
  VPB_REQUIRE(workspace && workspace_bytes >= w.bytes, "workspace too small");
  const int64_t ctas = ceil_div(M, NW);
  const int64_t groups = ceil_div(ctas, kGroup);
  VPB_CUDA(cudaMemsetAsync(w.counters, 0, (size_t)(groups + 1) * 4, s));
  SmpcIO io;
  memset(&io, 0, sizeof(io));
  io.eps = eps;
  io.nominal = nominal;
  io.M = M;
  io.m_offset = m_offset;
  io.lam = prob->lam;
  io.costs = costs;
  io.flags = flags;
  io.cta_parts = w.cta_parts;
  io.group_parts = w.group_parts;
  io.counters = w.counters;
  io.rank_part = part_out ? part_out : w.rank_part;
  io.finish = out != nullptr;
  io.out = out;
  io.acc = acc_of(prob);
  io.dyn = prob->dyn_state;
  if (precision == VPB_PREC_F64) {
    Prob<double> P;
    if ((rc = build_prob<double>(prob, field, P))) return rc;
    return dtype == VPB_DTYPE_F32 ? launch_smpc_t<double, float>(P, io, s) : launch_smpc_t<double, double>(P, io, s);
  }
  Prob<float> P;
  if ((rc = build_prob<float>(prob, field, P))) return rc;
  return dtype == VPB_DTYPE_F32 ? launch_smpc_t<float, float>(P, io, s) : launch_smpc_t<float, double>(P, io, s);
}

int vpb_smpc_partial(const vpb_problem *prob, const vpb_field *field, const void *eps, int dtype,
                     const double *nominal, int64_t M, int64_t m_offset, int precision, double *costs,
                     uint8_t *flags, double *part_out, void *workspace, size_t workspace_bytes, void *stream) {
  VPB_REQUIRE(part_out, "part_out is null");
  return smpc_launch(prob, field, eps, dtype, nominal, M, m_offset, precision, costs, flags, part_out, nullptr,
                     workspace, workspace_bytes, as_stream(stream));
}

int vpb_smpc_step(const vpb_problem *prob, const vpb_field *field, const void *eps, int dtype,
                  const double *nominal, int64_t M, int precision, double *costs, uint8_t *flags, double *out,
                  void *workspace, size_t workspace_bytes, void *stream) {
  VPB_REQUIRE(out, "out is null");
  return smpc_launch(prob, field, eps, dtype, nominal, M, 0, precision, costs, flags, nullptr, out, workspace,
                     workspace_bytes, as_stream(stream));
}

size_t vpb_smpc_finish_workspace_bytes(int64_t n_parts, int64_t H, int64_t n) {
  (void)n_parts;
  return align_up((size_t)(kPartHead + H * n) * 8, 256) + 256;
}

int vpb_smpc_finish(const vpb_problem *prob, const vpb_field *field, const double *partials, int64_t n_parts,
                    const double *nominal, int precision, double *out, void *workspace, size_t workspace_bytes,
                    void *stream) {
  int rc = prob_checks(prob, precision, VPB_DTYPE_F64);
  if (rc) return rc;
  VPB_REQUIRE(partials && nominal && out && n_parts >= 1 && n_parts <= 4096, "bad arguments to vpb_smpc_finish");
  VPB_REQUIRE(prob->lam > 0.0, "temperature must be positive");
  const int64_t H = prob->horizon, n = prob->n_joints;
  VPB_REQUIRE(workspace && workspace_bytes >= vpb_smpc_finish_workspace_bytes(n_parts, H, n), "workspace too small");
  double *merged = reinterpret_cast<double *>(workspace);
  cudaStream_t s = as_stream(stream);
  const AccLimit acc = acc_of(prob);
  if (precision == VPB_PREC_F64) {
    Prob<double> P;
    if ((rc = build_prob<double>(prob, field, P))) return rc;
    return launch_finish_t<double>(P, partials, (int)n_parts, prob->lam, nominal, acc, merged, out, prob->dyn_state,
                                   s);
  }
  Prob<float> P;
  if ((rc = build_prob<float>(prob, field, P))) return rc;
  return launch_finish_t<float>(P, partials, (int)n_parts, prob->lam, nominal, acc, merged, out, prob->dyn_state, s);
}

}  // extern "C"
