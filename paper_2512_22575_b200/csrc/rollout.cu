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
#include <cstdlib>

#include "noise.cuh"
#include "rollout_fixed.cuh"

namespace vpb {

// The fixed-topology SMPC kernel uses static shared memory so that ptxas may
// spill registers to shared memory (VPB_NO_SMEM_SPILL: the old dynamic layout)
#ifndef VPB_NO_SMEM_SPILL
#define VPB_SMEM_SPILL 1
#endif

constexpr int NW = 8;                    // candidate warps per CTA (generic path, rollout kernel)
constexpr int NWF = 4;                   // candidate warps per CTA of the fixed-topology SMPC kernel
constexpr int kThreads = (NW + 1) * 32;  // + terminal warp
// H n of the parameter-carried nominal (session path; larger H n take the
// staged-block session).  The launch cost grows with the parameter block
// (~0.4 us per KB on the C3 step): 256 covers C1/C3/C5 (H n = 140 / 224).
#define VPB_NOM_INLINE 256
constexpr int kPartHead = 4;             // [m, Z, nonfinite, best_index]
constexpr int kPartExt = 7;              // after N: [nonzero-weight count, the single candidate's 6 sums]
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

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// trace layout: [cta * 2 + 0] = start, [cta * 2 + 1] = candidates done,
// then at 2 * ctas: [group merge done, global merge done, tail done]
#define VPB_TRACE(io, idx)                                      \
  do {                                                          \
    if ((io).trace && threadIdx.x == 0) (io).trace[idx] = gtimer(); \
  } while (0)

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Inter-CTA waits of the merge protocol back off with __nanosleep and trap
// after 2 s: a broken invariant (e.g. counters not zeroed) becomes a CUDA
// error instead of a hung device.
struct SpinGuard {
  unsigned long long t0;
  __device__ SpinGuard() {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  }
  __device__ __forceinline__ void pause(unsigned ns) {
    __nanosleep(ns);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) __trap();
  }
};
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int *p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
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
  size_t centers, sums, cost, qH, fail, tfail, dyn, pro, misc, scratch, total;
};

__host__ __device__ constexpr size_t al16(size_t v) { return (v + 15) & ~(size_t)15; }

__host__ __device__ constexpr SmemLayout smem_layout(int ns, size_t tsize, int scratch_doubles) {
  SmemLayout L{};
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
  o = al16(o + (tsize == 8 ? sizeof(Dyn<double>) : sizeof(Dyn<float>)));
  L.pro = o;  // q_0 terms of the fixed-topology path (see pro_fail)
  o = al16(o + 8 * 8);
  L.misc = o;  // 32 doubles of reduction scratch + flags
  o = al16(o + 48 * 8);
  L.scratch = o;  // merge scales + compacted row indices (and the finish kernel's split sums)
  o = al16(o + (size_t)(2 * (scratch_doubles > 32 ? scratch_doubles : 32) + 24) * 8);
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
  if (lane == 0) D.sq = P.sq_dev ? *P.sq_dev : P.sq;
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
          query_issue<T>(P, D.sq, cen[(3 * s0) * 32], cen[(3 * s0 + 1) * 32], cen[(3 * s0 + 2) * 32], Qa);
          const int s1 = hb ? s0 + 1 : s0;
          query_issue<T>(P, D.sq, cen[(3 * s1) * 32], cen[(3 * s1 + 1) * 32], cen[(3 * s1 + 2) * 32], Qb);
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
  double *pro;
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
  S.pro = reinterpret_cast<double *>(base + L.pro);
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

// ---------------------------------------------------------------------------
// Fixed-topology candidate (rollout_fixed.cuh): lane k integrates to q_{k+1}
// and evaluates FK there; the limit terms use (q_k, qd_k, u_k).  Leaves the
// running sums (without the q_0 terms), the terminal cost and the flag.
// ---------------------------------------------------------------------------
struct TopoDyn {};  // marker: runtime topology (generic path)

template <typename Topo>
constexpr bool is_dyn_v = std::is_same_v<Topo, TopoDyn>;

// smpc_kernel shape: the generic path has a terminal warp per CTA; the fixed
// path has candidate warps only (its q_0 terms are added by the last CTA).
template <typename Topo>
constexpr int smpc_nw() {
  return is_dyn_v<Topo> ? NW : NWF;
}
template <typename Topo>
constexpr int smpc_threads() {
  return is_dyn_v<Topo> ? (NW + 1) * 32 : NWF * 32;
}
// fp32 fixed path: 7 CTAs of 4 warps per SM (<= 72 registers) so that a
// 4096-candidate step runs in a single wave on 148 SMs.
template <typename T, typename Topo>
constexpr int smpc_min_blocks() {
#ifndef VPB_SMPC_MINB
#define VPB_SMPC_MINB 7
#endif
  return sizeof(T) == 8 ? 1 : (is_dyn_v<Topo> ? 2 : VPB_SMPC_MINB);
}

// One fixed-topology evaluation per warp, lane = step.  The warp integrates
// u_k = ctrl[k] + nominal[k] (either may be null = 0) from (q0, qd0) and
// evaluates the configuration q_{k+shift}: shift 1 is a candidate (running
// pose + spheres for k+1 < H, terminal pose for k+1 == H); shift 0 with H = 1
// is the q_0 prologue (lane 0: pose + spheres at q_0; its limit terms are
// ignored).  Every caller goes through one call site per kernel so the
// unrolled step code exists once in the instruction stream.
template <typename T, typename ET, typename Topo>
__device__ __forceinline__ void fixed_candidate(const Prob<T> &P, const Dyn<T> &D, const ET *ctrl,
                                                const double *nominal, bool valid, int H, int shift, int sub,
                                                int nsub, double *sums_slot, double *term_slot, int *fail_slot,
                                                const NoiseGen *gen = nullptr, int64_t m_loc = 0,
                                                float *eps_out = nullptr) {
  constexpr int NJ = Topo::NJ;
  const int lane = threadIdx.x & 31;
  const Split W = make_split<Topo>(sub, nsub);
  const bool do_lim = sub == 0;
  T qc[NJ], qdc[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    qc[j] = D.q0[j];
    qdc[j] = D.qd0[j];
  }
  T s_pose = 0, s_coll = 0, s_lim = 0, s_smooth = 0, s_null = 0, term = 0;
  bool fail = false;
  const int nchunks = (H + 31) >> 5;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int k = ch * 32 + lane;
    const bool act = valid && k < H;
    T qe[NJ];
    T lim = 0, sm = 0, nu = 0;
    float gz[NJ];  // on-the-fly perturbation (noise.cuh), warp-uniform branch
    if (gen) {
      candidate_noise<NJ, 2>(*gen, m_loc, H, ch, lane, gz);
      if (act && eps_out) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) eps_out[((size_t)m_loc * H + k) * NJ + j] = gz[j];
      }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      double v = 0.0;
      if (act) {
        if (gen) v = (double)gz[j];
        else if (ctrl) v = load_e<ET>(ctrl + (size_t)k * NJ + j);
        if (nominal) v += nominal[(size_t)k * NJ + j];
      }
      const T uj = (T)v;
      const T vdt = uj * P.dt;
      const T vin = warp_incl_scan<T>(vdt, lane);
      const T qd = qdc[j] + (vin - vdt);          // qd_k
      const T qdn = act ? (qdc[j] + vin) : T(0);  // qd_{k+1}
      const T w = qdn * P.dt;
      const T win = warp_incl_scan<T>(w, lane);
      const T q = qc[j] + (win - w);              // q_k
      qe[j] = shift ? qc[j] + win : q;            // q_{k+shift}
      qdc[j] += __shfl_sync(kFull, vin, 31);
      qc[j] += __shfl_sync(kFull, win, 31);
      // limits / smoothness / null space at step k (vp/batch.py:303-311)
      const T vq = bound_violation<T>(q, P.pos_lo[j], P.pos_hi[j]);
      const T vv = bound_violation<T>(qd, P.vel_lo[j], P.vel_hi[j]);
      const T va = bound_violation<T>(uj, P.acc_lo[j], P.acc_hi[j]);
      lim += P.w_q * vq * vq + P.w_qd * vv * vv + P.w_qdd * va * va;
      sm += P.w_s * uj * uj;
      const T dq = q - P.q_ref[j];
      nu += P.w_ns * dq * dq;
    }
    if (act) {
      if (do_lim) {
        s_lim += lim;
        s_smooth += sm;
        s_null += nu;
      }
      const int idx = k + shift;
      const bool last = idx == H;
      T pose, coll;
      if (!fixed_config<Topo, T>(P, P.fc, D, qe, !last, last, W, pose, coll)) fail = true;
      if (last) term = pose;
      else s_pose += pose;
      s_coll += coll;
    }
  }
  const double r_pose = warp_sum_d((double)s_pose);
  const double r_coll = warp_sum_d((double)s_coll);
  const double r_lim = warp_sum_d((double)s_lim);
  const double r_smooth = warp_sum_d((double)s_smooth);
  const double r_null = warp_sum_d((double)s_null);
  const double r_term = warp_sum_d((double)term);  // one lane holds it
  const bool any_fail = __any_sync(kFull, fail);
  if (lane == 0) {
    sums_slot[0] = r_pose;
    sums_slot[1] = r_coll;
    sums_slot[2] = r_lim;
    sums_slot[3] = r_smooth;
    sums_slot[4] = r_null;
    *term_slot = r_term;
    *fail_slot = any_fail ? 1 : 0;
  }
}

// S.pro layout: [0..5] prologue sums (pose, collision, ...), [6] terminal
// (unused), int at [7] = failed.
__device__ __forceinline__ int *pro_fail(const Shared &S) { return reinterpret_cast<int *>(S.pro + 7); }

// Add the q_0 terms to candidate w's sums (after a __syncthreads).
__device__ __forceinline__ void fixed_add_prologue(const Shared &S, int w) {
  S.sums[w * 6 + 0] += S.pro[0];
  S.sums[w * 6 + 1] += S.pro[1];
  if (*pro_fail(S) != 0) S.fail[w] = 1;
  S.tfail[w] = 0;
}

// rollout_kernel, fixed path: warps < NW are candidates, warp NW the q_0
// prologue, through one call site.
template <typename T, typename ET, typename Topo>
__device__ __forceinline__ void evaluate_cta_fixed(const Prob<T> &P, const Dyn<T> &D, const ET *ctrl,
                                                   const double *nominal, int64_t M, int64_t cta_m0,
                                                   const Shared &S) {
  const int warp = threadIdx.x >> 5;
  const bool cand = warp < NW;
  const int64_t m = cta_m0 + warp;
  const bool valid = cand ? m < M : true;
  fixed_candidate<T, ET, Topo>(P, D, (cand && valid) ? ctrl + (size_t)m * P.H * Topo::NJ : nullptr,
                               cand ? nominal : nullptr, valid, cand ? P.H : 1, cand ? 1 : 0, 0, 1,
                               cand ? S.sums + warp * 6 : S.pro, cand ? S.cost + warp : S.pro + 6,
                               cand ? S.fail + warp : pro_fail(S));
  __syncthreads();
  if (threadIdx.x < NW) fixed_add_prologue(S, threadIdx.x);
  __syncthreads();
}

template <typename T, typename ET, int MAXJ, typename Topo>
__device__ __forceinline__ void evaluate_cta_any(const Prob<T> &P, const Dyn<T> &D, const ET *ctrl,
                                                 const double *nominal, int64_t M, int64_t cta_m0, const Shared &S,
                                                 const CandOut &co) {
  if constexpr (std::is_same_v<Topo, TopoDyn>) {
    evaluate_cta<T, ET, MAXJ>(P, D, ctrl, nominal, M, cta_m0, S, co);
  } else {
    evaluate_cta_fixed<T, ET, Topo>(P, D, ctrl, nominal, M, cta_m0, S);
  }
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
template <typename T, typename ET, int MAXJ, typename Topo>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? 2 : 1) rollout_kernel(const __grid_constant__ Prob<T> P,
                                                              const __grid_constant__ RolloutIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SmemLayout L = smem_layout(std::is_same_v<Topo, TopoDyn> ? P.ns : 0, sizeof(T), 0);
  const Shared S = carve(smem_raw, L);
  Dyn<T> &D = *reinterpret_cast<Dyn<T> *>(S.dyn);
  if (threadIdx.x < 32) load_dyn<T>(P, io.dyn, D);
  __syncthreads();
  const int64_t cta_m0 = (int64_t)blockIdx.x * NW;
  CandOut co{io.traj_q, io.traj_qd, io.sph_out};
  evaluate_cta_any<T, ET, MAXJ, Topo>(P, D, reinterpret_cast<const ET *>(io.ctrl), io.nominal, io.M, cta_m0, S, co);
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

// Partial rows to merge: head field f of row i at head[f * fstride + i *
// rstride] (fields m, Z, non-finite, best); N of row i at n[i * nstride].
// CTA partials are structure-of-arrays (fstride = rows, rstride = 1: a warp
// reads 32 consecutive heads with one coalesced load); rank records are the
// exchanged [m, Z, nf, best, N] rows (fstride = 1, rstride = nstride = L).
struct Rows {
  const double *head;
  const double *n;
  int64_t fstride, rstride, nstride;
  __device__ __forceinline__ double h(int f, int i) const { return head[f * fstride + (int64_t)i * rstride]; }
};

__device__ void merge_block(const Rows &R, int count, int hn, double lam, double *dst, double *scratch,
                            double *misc, unsigned long long *trace_head = nullptr) {
  // Merge `count` partial rows in row order.  Warp w owns the contiguous rows
  // [w span, (w + 1) span), lanes over consecutive rows (coalesced):
  //   1. min and the first row attaining it;
  //   2. scale_i = exp(-(m_i - min) / lam), Z = sum scale_i Z_i, non-finite
  //      count (lane-strided partial sums, then a fixed xor tree and the
  //      warps in order -- deterministic);
  //   3. rows with scale 0 (exp underflow: far above the minimum -- most of
  //      them at the planner's lam) are dropped by an order-preserving
  //      ballot compaction, and N = sum scale_i N_i runs over the rest.
  // scratch: >= 2 * (count + 512) + 24 doubles; misc: >= 48 doubles.
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int span = ((count + nw - 1) / nw + 31) & ~31;
  const int w0 = warp * span, w1 = min(count, w0 + span);
  double mn = dinf();
  int bidx = 0x7fffffff;
  for (int c = w0; c < w1; c += 32 * 4) {
    double v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = c + 32 * t + lane;
      v[t] = i < w1 ? R.h(0, i) : dinf();
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (v[t] < mn) {  // rows ascend per lane: the first minimum wins
        mn = v[t];
        bidx = c + 32 * t + lane;
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
  if (lane == 0) {
    misc[warp] = mn;
    misc[16 + warp] = (double)bidx;
  }
  if (trace_head && tid == 0) trace_head[1] = gtimer();
  __syncthreads();
  if (tid == 0) {
    double m0 = dinf();
    int b0 = 0x7fffffff;
    for (int w = 0; w < nw; ++w) {
      const double v = misc[w];
      const int b = (int)misc[16 + w];
      if (v < m0 || (v == m0 && b < b0)) {
        m0 = v;
        b0 = b;
      }
    }
    misc[40] = m0;
    misc[41] = (double)b0;
  }
  __syncthreads();
  mn = misc[40];
  bidx = (int)misc[41];
  // pass 2: scales, Z, non-finite count, and the order-preserving compaction
  // of this warp's nonzero rows into its own slice [w0, w0 + wnz) of the
  // row list (rows ascend within a warp; warps are concatenated in order)
  const int cap = count + 32 * nw;  // per-warp slices may overhang count
  double *scale = scratch;
  int *rows = reinterpret_cast<int *>(scratch + cap);
  double *nf_w = scratch + cap + cap / 2 + 2;
  const double inv_lam = 1.0 / lam;
  double z = 0.0, nf = 0.0;
  int wnz = 0;
  for (int c = w0; c < w1; c += 32 * 4) {
    double v[4], zi[4], fi[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = c + 32 * t + lane;
      const bool ok = i < w1;
      v[t] = ok ? R.h(0, i) : dinf();
      zi[t] = ok ? R.h(1, i) : 0.0;
      fi[t] = ok ? R.h(2, i) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const double sc = (v[t] < dinf()) ? exp(-(v[t] - mn) * inv_lam) : 0.0;
      if (sc != 0.0) z += sc * zi[t];
      nf += fi[t];
      const unsigned bal = __ballot_sync(kFull, sc != 0.0);
      if (sc != 0.0) {
        const int p = w0 + wnz + __popc(bal & ((1u << lane) - 1u));
        rows[p] = c + 32 * t + lane;
        scale[p] = sc;
      }
      wnz += __popc(bal);
    }
  }
  const double zw = warp_sum_d(z), nfw = warp_sum_d(nf);
  if (lane == 0) {
    misc[16 + warp] = (double)wnz;  // (misc[16..32) is free again)
    misc[32 + warp] = zw;
    nf_w[warp] = nfw;
  }
  if (trace_head && tid == 0) trace_head[2] = gtimer();
  __syncthreads();
  if (tid == 0) {
    double Z = 0.0, NF = 0.0;
    for (int w = 0; w < nw; ++w) {
      Z += misc[32 + w];
      NF += nf_w[w];
    }
    dst[0] = mn;
    dst[1] = Z;
    dst[2] = NF;
    dst[3] = (bidx >= 0 && bidx < count) ? R.h(3, bidx) : -1.0;
  }
  if (trace_head && tid == 0) *trace_head = gtimer();
  // N over the nonzero rows, warp slices in order
  for (int e = tid; e < hn; e += nt) {
    const double *col = R.n + e;
    double acc = 0.0;
    for (int w = 0; w < nw; ++w) {
      const int base = w * span, cnt = (int)misc[16 + w];
      int k = 0;
      for (; k + 4 <= cnt; k += 4) {
        double a[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) a[t] = col[(int64_t)rows[base + k + t] * R.nstride];
#pragma unroll
        for (int t = 0; t < 4; ++t) acc += scale[base + k + t] * a[t];
      }
      for (; k < cnt; ++k) acc += scale[base + k] * col[(int64_t)rows[base + k] * R.nstride];
    }
    dst[kPartHead + e] = acc;
  }
  __syncthreads();
}

// Rank records [m, Z, nf, best, N (hn)] as merge rows.
__device__ __forceinline__ Rows record_rows(const double *rec, int hn) {
  const int L = kPartHead + hn + kPartExt;
  return Rows{rec, rec + kPartHead, 1, L, L};
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
  unsigned long long *trace;  // optional per-phase %globaltimer stamps (tools/smpc_trace.py)
  double *pro;  // [NWF][4] q_0 terms per split warp (fixed path, prologue block 0)
  double *cand_costs;  // [M] candidate costs when io.costs is null (workspace)
  NoiseGen gen;    // on-the-fly perturbations (fixed path) when gen_on
  int gen_on;
  float *eps_out;  // where the drawn perturbations go (== eps for the merge)
  double *out_host;  // optional host-mapped copy of `out` (+ 1 slot: the done flag), written by the last CTA
  double *cand_terms;  // [M][6] per-candidate sums (fixed path): the re-evaluation shortcut
  int max_helpers;     // helper CTAs of the heavy merge (residency-capped, see merge_helpers)
  double *hparts;      // heavy merge: per-participant [Z, nonzero count, N (H n)] partials
  // session staging (fixed path): block 0 copies the host-mapped per-call
  // block into its device copy and raises the staging word; every other CTA
  // waits for it before reading its inputs
  const double *stage_src;
  double *stage_dst;
  int stage_len;
};

// Session (fused fixed path, smpc_kernel<..., INL = true>): the nominal
// inline in the launch parameters, copied into shared memory by every CTA.
// The other instantiations carry a one-element stub.
template <bool INL>
struct NomInline {
  double v[INL ? VPB_NOM_INLINE : 1];
  int n;
};

// U* = nominal + N / Z, the clipped command and the shifted warm start
// (vp/planner.py:614-619), written to `out` by all threads of the CTA.
__device__ __forceinline__ void tail_controls(const double *part, const double *nominal, const AccLimit &acc, int H,
                                              int n, double *out) {
  const int hn = H * n;
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
}

// Zero-copy completion: after every thread's host-mapped writes, one
// system-scope release (cumulative over the barrier) and the flag word the
// host spins on (vpb_smpc_session_step).
__device__ __forceinline__ void signal_host_done(double *flag_slot) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long *>(flag_slot) = 1ull;
  }
}

// Diagnostics of the step (thread 0): re-evaluated cost of U* from slot 0 of
// S (sums / cost / flags), best cost, Z, non-finite count, best index.
__device__ __forceinline__ void tail_output(const Shared &S, const double *part, int H, int n, double best,
                                            double nonfinite, double *out, double *out_host = nullptr) {
  const int64_t base = 2 * (int64_t)H * n + n;
  const int a = threadIdx.x;
  if (a >= 13) return;
  const bool failed = S.fail[0] != 0 || S.tfail[0] != 0;
  const double *sm = S.sums;
  // slot a of [cost(U*), 5 sums, terminal, best, Z, non-finite, best index, e_pos, e_ori (host)]
  double v;
  if (a == 0) v = failed ? dinf() : sm[0] + sm[1] + sm[2] + sm[3] + sm[4] + S.cost[0];
  else if (a < 6) v = failed ? 0.0 : sm[a - 1];
  else if (a == 6) v = failed ? 0.0 : S.cost[0];
  else if (a == 7) v = best;
  else if (a == 8) v = part[1];
  else if (a == 9) v = nonfinite;
  else if (a == 10) v = part[3];
  else v = __longlong_as_double(0x7ff8000000000000ll);
  out[base + a] = v;
  if (out_host) out_host[base + a] = v;
}

// Generic path tail: U*, then its M = 1 re-evaluation on warps 0 and NW.
template <typename T, int MAXJ>
__device__ void smpc_tail_dyn(const Prob<T> &P, const Dyn<T> &D, const double *part, const double *nominal,
                              const AccLimit &acc, double *out, const Shared &S) {
  tail_controls(part, nominal, acc, P.H, P.nj, out);
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
  tail_output(S, part, P.H, P.nj, part[0], part[2], out);
}

// Fixed path: add the q_0 terms (S.pro) to this shard's per-sample costs and,
// when `part` is given, to its merged partial's minimum (the softmin weights
// are shift invariant, so Z and N are unchanged).
__device__ __forceinline__ void fixed_shard_fixup(const Shared &S, int64_t M, double *costs, uint8_t *flags,
                                                  double *part) {
  const bool bad = *pro_fail(S) != 0;
  const double add = S.pro[0] + S.pro[1];
  // (kept rolled: this runs once per step on a cold instruction cache)
  if (costs || (flags && bad)) {
#pragma unroll 1
    for (int64_t m = threadIdx.x; m < M; m += blockDim.x) {
      if (costs) costs[m] = bad ? dinf() : costs[m] + add;
      if (flags && bad) flags[m] = 1;
    }
  }
  if (threadIdx.x == 0 && part) {
    part[0] = bad ? dinf() : part[0] + add;
    if (bad) part[2] = (double)M;
  }
}


// Many nonzero weights (a converged planner: costs within ~746 lam of the
// minimum) make the weights (one f64 exp each) and N = sum_k w_k eps_k an
// (ncand x H n) reduction -- too much for the merging CTA alone.  The CTAs
// that took the last kMergeHelpers tickets stay resident, spin on a
// per-launch flag and, when the merge asks for help, each takes a contiguous
// slice of the nonzero-CTA list: its candidates' weights, their Z and their
// N over all elements (heavy_part); the merger adds the partials in
// participant order (deterministic).  Words after the ticket
// (io.counters + groups + 2): epoch, flag = epoch << 2 | state, ncand, done;
// the epoch advances once per launch, so nothing has to be reset.
constexpr int kMergeHelpers = 127;
// merge words after the ticket and the prologue flag: the epoch shares their
// line (read once per CTA); the polled flag (+ count) and the done counter
// get lines of their own so the waiting helpers do not contend with them
constexpr int kHcFlag = 32, kHcCount = 33, kHcDone = 64, kHcDone2 = 65, kHcStage = 80, kHcWords = 96;
// heavy-merge parameters published with the verdict (on the flag's line):
// the minimum (f64 bits), the per-warp CTA-list lengths, their stride, the
// merger's warp count, the CTA-list length
constexpr int kHcM0 = 34, kHcWcount = 36, kHcSpan = 52, kHcNw = 53, kHcList = 54, kHcParts = 55;
constexpr int kLightMax = 32;  // up to this many nonzero weights the merging CTA computes N alone
// io.max_helpers (host: min(kMergeHelpers, resident CTA slots - 2)) keeps the
// spinning helpers from filling every slot while CTAs without a ticket still
// wait to be scheduled (small MIG / MPS partitions); 0 = the merger alone
__device__ __forceinline__ int merge_helpers(const SmpcIO &io, int ctas) {
  return ctas - 1 < io.max_helpers ? ctas - 1 : io.max_helpers;
}

// Heavy merge, one participant (a helper CTA or the merger): the weights of
// the candidates of its contiguous slice of the nonzero-CTA list (written to
// the candidate lists in list order), their Z and nonzero count (summed in
// list order) and their N = sum w eps over all H n elements (each thread its
// elements, candidates in list order) -> hparts[part].  The merger then adds
// the participants' partials in participant order: deterministic.
template <typename ET, int NWC>
__device__ void heavy_part(const SmpcIO &io, const Shared &S, const unsigned int *hc, int part, int P, int hn,
                           unsigned long long *ht = nullptr) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const ET *eps = reinterpret_cast<const ET *>(io.eps);
  const double *costs = io.costs ? io.costs : io.cand_costs;
  double *wlist = io.group_parts;
  int *mlist = reinterpret_cast<int *>(io.group_parts + io.M + 64);
  const int *clist = reinterpret_cast<const int *>(io.group_parts + io.M + 64) + io.M + 64;
  // the verdict words once per CTA instead of every thread of up to 128
  // participants loading them from the one L2 line (16k-candidate converged
  // step: -2..4 us)
  __shared__ unsigned int hcw[kHcParts - kHcM0];
  if (tid < kHcParts - kHcM0) hcw[tid] = __ldcg(hc + kHcM0 + tid);
  __syncthreads();
  const unsigned long long m0b = (unsigned long long)hcw[0] | ((unsigned long long)hcw[1] << 32);
  const double m0 = __longlong_as_double((long long)m0b);
  const double inv_lam = 1.0 / io.lam;
  const int span = (int)hcw[kHcSpan - kHcM0], nw = (int)hcw[kHcNw - kHcM0], list = (int)hcw[kHcList - kHcM0];
  int wc[16];
#pragma unroll
  for (int w = 0; w < 16; ++w) wc[w] = w < nw ? (int)hcw[kHcWcount - kHcM0 + w] : 0;
  const int per = (list + P - 1) / P;
  const int j0 = part * per, j1 = min(list, j0 + per);
  constexpr int kE = 2;  // N elements per thread and pass (passes over blocks of kE nt elements)
  double z = 0.0, nzc = 0.0;
  // [nt] weights and rows of the chunk, in the sphere-centre area (free after
  // the evaluation; the merge scratch still holds the record head)
  double *wbuf = reinterpret_cast<double *>(S.centers);
  int *mbuf = reinterpret_cast<int *>(wbuf + nt);
  for (int k0 = NWC * j0; k0 < NWC * j1; k0 += nt) {
    const int k = k0 + tid;
    double wt = 0.0;
    int mm = 0;
    if (k < NWC * j1) {
      const int j = k / NWC, r = k % NWC;
      int seg = 0, base = 0;
      while (seg < nw - 1 && j >= base + wc[seg]) {
        base += wc[seg];
        ++seg;
      }
      const int ci = __ldcg(clist + seg * span + (j - base));
      const int m = ci * NWC + r;
      if (m < io.M) {
        const double c = __ldcg(costs + m);
        wt = c < dinf() ? exp(-(c - m0) * inv_lam) : 0.0;
        mm = m;
      }
      mlist[k] = mm;  // (padding slot of the last CTA: weight 0, any valid row)
      wlist[k] = wt;
    }
    wbuf[tid] = wt;
    mbuf[tid] = mm;
    // Z and the count of the chunk: fixed-shape block reduction (warp xor
    // trees, then the warps in order), added to the running sums by thread 0
    const double zw = warp_sum_d(wt), cw = warp_sum_d(wt != 0.0 ? 1.0 : 0.0);
    double *wred = reinterpret_cast<double *>(mbuf + nt);  // [2][nw]
    if ((tid & 31) == 0) {
      wred[tid >> 5] = zw;
      wred[(nt >> 5) + (tid >> 5)] = cw;
    }
    __syncthreads();
    const int cnt = min(nt, NWC * j1 - k0);
    if (ht && tid == 0 && k0 == NWC * j0) ht[1] = gtimer();
    if (tid == 0) {
      for (int w = 0; w < (nt >> 5); ++w) {
        z += wred[w];
        nzc += wred[(nt >> 5) + w];
      }
    }
    // N: element blocks of kE nt; candidates in groups of kG with every row
    // load of the group in flight before the in-order accumulation (a zero
    // weight adds exactly 0); the block's partial sums go to hparts
    constexpr int kG = 8;
    double *dstn = io.hparts + (size_t)part * (2 + hn) + 2;
    for (int eb = 0; eb < hn; eb += kE * nt) {
      double nacc[kE];
#pragma unroll
      for (int q = 0; q < kE; ++q) nacc[q] = k0 == NWC * j0 ? 0.0 : dstn[eb + tid + q * nt < hn ? eb + tid + q * nt : 0];
      for (int i0 = 0; i0 < cnt; i0 += kG) {
        double wi[kG];
        double v[kG][kE];
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          const int i = i0 + g;
          wi[g] = i < cnt ? wbuf[i] : 0.0;
          const ET *row = eps + (size_t)(i < cnt ? mbuf[i] : 0) * hn;
#pragma unroll
          for (int q = 0; q < kE; ++q) {
            const int e = eb + tid + q * nt;
            v[g][q] = (e < hn && wi[g] != 0.0) ? load_e<ET>(row + e) : 0.0;
          }
        }
#pragma unroll
        for (int g = 0; g < kG; ++g)
#pragma unroll
          for (int q = 0; q < kE; ++q) nacc[q] += wi[g] * v[g][q];
      }
#pragma unroll
      for (int q = 0; q < kE; ++q) {
        const int e = eb + tid + q * nt;
        if (e < hn) dstn[e] = nacc[q];
      }
    }
    __syncthreads();
  }
  double *dst = io.hparts + (size_t)part * (2 + hn);
  if (tid == 0) {
    dst[0] = z;
    dst[1] = nzc;
  }
  if (j1 <= j0) {  // empty slice: zero N
    for (int e = tid; e < hn; e += nt) dst[2 + e] = 0.0;
  }
}

// Second stage of the heavy merge, by every participant: once all P
// partials are published (done == P), participant `part` adds, for its slice
// of the H n elements, the P partials in participant order (thread q holds
// participant q; fixed-shape block reduction) into N (rank_part), then
// counts itself in done2.  The merger waits for done2 == P.
__device__ void heavy_sum_slice(const SmpcIO &io, const Shared &S, unsigned int *hc, int part, int P, int hn) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  __syncthreads();
  if (tid == 0) {
    fence_acq_rel_gpu();  // this participant's partial before its count
    atomicAdd(hc + kHcDone, 1u);
    SpinGuard g;
    while (ld_acquire_gpu(hc + kHcDone) < (unsigned int)P) g.pause(32);
  }
  __syncthreads();
  const int Lp = 2 + hn;
  const int per = (hn + P - 1) / P;
  const int e0 = part * per, e1 = min(hn, e0 + per);
  (void)S;
  if (P <= 32) {
    // few partials (a long slice): each thread one element, the P partials
    // added in participant order, every element of the slice at once
    for (int e = e0 + tid; e < e1; e += nt) {
      const double *src = io.hparts + 2 + e;
      double acc = 0.0;
#pragma unroll 8
      for (int q = 0; q < P; ++q) acc += __ldcg(src + (size_t)q * Lp);
      io.rank_part[kPartHead + e] = acc;
    }
  } else {
    // many partials (a short slice): one warp per element, lane q adds
    // participants q, q + 32, ... in order, then a fixed xor tree
    for (int e = e0 + warp; e < e1; e += nw) {
      const double *src = io.hparts + 2 + e;
      double v = 0.0;
      for (int q = lane; q < P; q += 32) v += __ldcg(src + (size_t)q * Lp);
      const double ws = warp_sum_d(v);
      if (lane == 0) io.rank_part[kPartHead + e] = ws;
    }
  }
  __syncthreads();  // the slice is written before this participant counts itself
  if (tid == 0) {
    fence_acq_rel_gpu();
    atomicAdd(hc + kHcDone2, 1u);
  }
}

// A helper CTA (one of the last kMergeHelpers finishers): wait for the merge's
// verdict; on "help", compute slice `part` and report done.
template <typename ET, int NWC>
__device__ void merge_helper(const SmpcIO &io, const Shared &S, int ctas, int hn, int part, unsigned int ep) {
  unsigned int *c = io.counters + (ctas + kGroup - 1) / kGroup + 2;
  unsigned int *st = reinterpret_cast<unsigned int *>(S.misc + 47);
  if (threadIdx.x == 0) {
    unsigned int f;
    SpinGuard g;
    while (((f = ld_acquire_gpu(c + kHcFlag)) >> 2) != (ep & 0x3fffffffu) || (f & 3u) == 0u) g.pause(512);
    st[0] = f & 3u;
    st[1] = ld_acquire_gpu(c + kHcCount);
    st[2] = (f & 3u) == 2u ? __ldcg(c + kHcParts) : 0u;
  }
  __syncthreads();
  if (st[0] != 2u) return;
  const int P = (int)st[2];  // participants: helpers 0 .. P-2 and the merger
  if (part >= P - 1) return;
  // (tools/smpc_trace.py: per-helper stamps after the fixed slots)
  unsigned long long *ht = io.trace ? io.trace + 2 * ctas + 32 + 3 * part : nullptr;
  if (ht && threadIdx.x == 0) ht[0] = gtimer();
  heavy_part<ET, NWC>(io, S, c, part, P, hn, ht);  // ht[1]: weights of the first chunk done
  if (ht && threadIdx.x == 0) ht[2] = gtimer();
  heavy_sum_slice(io, S, c, part, P, hn);
}

// Shared-memory slots of the final merge and the fixed-path tail (S.scratch,
// kMergeScratch doubles): the merge keeps what the tail needs on chip so the
// last CTA's chain of dependent global round trips stays short.
constexpr int kMergeScratch = 64;  // smem_layout scratch argument of smpc_kernel (2 * 64 + 24 doubles)
constexpr int kFmW = 0;            // [32] weights of the first nonzero candidates
constexpr int kFmCT = 32;          // [6] sums of the minimum's candidate (speculative, for the shortcut)
constexpr int kFmRec = 40;         // [4] the shard record head: min, Z, non-finite, best index
constexpr int kFmBest = 44;        // local index of the minimum's candidate
constexpr int kFmCL = 48;          // ints: [nw][kFmCap] nonzero CTAs per warp
constexpr int kFmML = 120;         // ints: [32] indices of the first nonzero candidates
constexpr int kFmWN = 136;         // ints: [nw] nonzero CTA count per warp
constexpr int kFmCap = 16;

// Final merge of the single-device step, by the last CTA.  Inputs: the CTA
// heads (structure-of-arrays [3][ctas]: min cost, non-finite count, best
// global index) and every candidate's cost.  Output: the shard record
// [min, Z, non-finite, best, N (hn), ext] with weights
// w_m = exp(-(S_m - min)/lam) in candidate order (io.rank_part, and the head
// in smem at kFmRec).  A CTA whose own minimum is far above the global one
// (exp underflow) contributes exactly zero and is skipped before any of its
// candidates is touched; at the planner's lam almost all are.  Lists live in
// global scratch with their first entries mirrored in smem.  FIXED: while
// warp 0 expands the candidates, warp 1 fetches the minimum's sums (the
// single-weight shortcut) and warp 2 the q_0 prologue terms of block 0.
// `fused_u` (fixed path, finishing): U*, the clipped command and the shifted
// warm start are produced in the N pass itself (to out and out_host).
template <typename ET, int NWC, bool FIXED>
__device__ void final_merge(const SmpcIO &io, const Shared &S, const double *heads, const double *costs, int ctas,
                            int hn, int nj, bool fused_u, unsigned int ep, unsigned long long *trace_head,
                            const double *nominal) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double *misc = S.misc;
  double *sc = S.scratch;
  double *wlist = io.group_parts;                                  // candidate weights
  int *mlist = reinterpret_cast<int *>(io.group_parts + io.M + 64);  // candidate indices
  int *clist = reinterpret_cast<int *>(io.group_parts + io.M + 64) + io.M + 64;  // nonzero CTAs, per-warp slices
  int *sclist = reinterpret_cast<int *>(sc + kFmCL);
  int *smlist = reinterpret_cast<int *>(sc + kFmML);
  const double inv_lam = 1.0 / io.lam;
  if (fused_u) {  // the nominal is read by the U* pass at the end: start it towards L2 now
    if (__isGlobal(nominal))  // (the session's nominal lives in shared memory)
      for (int e = tid * 16; e < hn; e += nt * 16) asm volatile("prefetch.global.L2 [%0];" ::"l"(nominal + e));
  }
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
#pragma unroll 1
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
  if (trace_head && tid == 0) trace_head[1] = gtimer();
  if (lane == 0) {
    misc[warp] = mn;
    misc[16 + warp] = (double)bidx;
    misc[32 + warp] = nf;
  }
  __syncthreads();
  // every thread combines the warp results (fixed warp order)
  double m0 = dinf(), NF = 0.0;
  int b0 = 0x7fffffff;
#pragma unroll 1
  for (int w = 0; w < nw; ++w) {
    const double v = misc[w];
    const int b = (int)misc[16 + w];
    NF += misc[32 + w];
    if (v < m0 || (v == m0 && b < b0)) {
      m0 = v;
      b0 = b;
    }
  }
  if (trace_head && tid == 0) trace_head[2] = gtimer();
  // 2. (all warps) CTAs with a nonzero weight, compacted in order into this
  //    warp's slice of clist (+ its first kFmCap in smem); exp-free,
  //    conservative test (exp(-x) underflows to 0 for x > 745.14; the
  //    expansion below computes the exact weights)
  int wn = 0;
  auto consider = [&](int i, double v) {
    const bool nz = v < dinf() && (v - m0) * inv_lam < 746.0;
    const unsigned bal = __ballot_sync(kFull, nz);
    if (nz) {
      const int p = wn + __popc(bal & ((1u << lane) - 1u));
      clist[w0 + p] = i;
      if (p < kFmCap) sclist[warp * kFmCap + p] = i;
    }
    wn += __popc(bal);
  };
  if (in_regs) {
#pragma unroll
    for (int t = 0; t < kHR; ++t) consider(w0 + 32 * t + lane, hv[t]);
  } else {
#pragma unroll 1
    for (int c = w0; c < w1; c += 32) {
      const int i = c + lane;
      consider(i, i < w1 ? heads[i] : dinf());
    }
  }
  int *wcount = reinterpret_cast<int *>(sc + kFmWN);
  if (lane == 0) wcount[warp] = wn;
  __syncthreads();
  if (trace_head && tid == 0) trace_head[3] = gtimer();
  const int b0c = (b0 >= 0 && b0 < ctas) ? b0 : 0;
  if (warp == 1) {
    // the minimum's global index, and (fixed path) its candidate's sums: when
    // it is the only nonzero weight, they are the re-evaluation of U*
    const double bg = b0 < ctas ? heads[2 * (size_t)ctas + b0c] : -1.0;
    const double bd = bg - (double)io.m_offset;
    const int bl = (bg >= 0.0 && bd < (double)io.M) ? (int)bd : -1;
    if (FIXED && io.cand_terms && lane < 6 && bl >= 0) sc[kFmCT + lane] = __ldcg(io.cand_terms + 6 * (size_t)bl + lane);
    if (lane == 0) {
      sc[kFmRec + 3] = bg;
      sc[kFmBest] = (double)bl;
    }
    if (trace_head && lane == 0) trace_head[5] = gtimer();
  } else if (FIXED && warp == 2) {
    // block 0's q_0 prologue terms (normally long done), summed in split order
    unsigned int *pro_ready = io.counters + (ctas + kGroup - 1) / kGroup + 1;
    if (lane == 0) {
      SpinGuard g;
      while (ld_acquire_gpu(pro_ready) == 0u) g.pause(64);
      *pro_ready = 0u;  // counters return to zero for the next launch
    }
    __syncwarp();
    const bool has = lane < NWF;
    const double pw = has ? __ldcg(io.pro + 4 * lane + 0) : 0.0;
    const double cw = has ? __ldcg(io.pro + 4 * lane + 1) : 0.0;
    const unsigned badm = __ballot_sync(kFull, has && __ldcg(io.pro + 4 * lane + 2) != 0.0);
    const double pose0 = warp_sum_d(pw), coll0 = warp_sum_d(cw);
    if (lane == 0) {
      S.pro[0] = pose0;
      S.pro[1] = coll0;
      *pro_fail(S) = badm != 0u;
      if (trace_head) trace_head[6] = gtimer();
    }
  }
  // 3. (all threads) the candidates of those CTAs, in candidate order, NOT
  //    compacted (a zero weight stays in the list as (m, 0): it adds exactly
  //    nothing): weights, Z and the nonzero count.  Thread t takes list
  //    entries t, t + nt, ... (two dependent loads each, batched 8 deep).
  int total = 0;
  bool small = true;
  for (int w = 0; w < nw; ++w) {
    total += wcount[w] * NWC;
    small = small && wcount[w] <= kFmCap;
  }
  double z = 0.0;
  int nz = 0;
  if (total <= 32) {
    // the usual case (a handful of candidates near the minimum): warp 0,
    // one entry per lane, one round trip for the CTA index and one for the cost
    if (warp == 0 && lane < total) {
      int seg = 0, base = 0;
      while (seg < nw - 1 && lane >= base + wcount[seg] * NWC) {
        base += wcount[seg] * NWC;
        ++seg;
      }
      const int r = lane - base;
      const int ci = small ? sclist[seg * kFmCap + r / NWC] : clist[seg * span + r / NWC];
      const int m = ci * NWC + (r % NWC);
      double wt = 0.0;
      if (m < io.M) {
        const double c = costs[m];
        wt = c < dinf() ? exp(-(c - m0) * inv_lam) : 0.0;
      }
      const int mm = m < io.M ? m : 0;  // padding slot of the last CTA: weight 0, any valid row
      mlist[lane] = mm;
      wlist[lane] = wt;
      smlist[lane] = mm;
      sc[kFmW + lane] = wt;
      z = wt;
      nz = wt != 0.0 ? 1 : 0;
    }
  }
  // (more than kLightMax list entries: the heavy merge below expands them in
  // parallel over the helper CTAs)
  z = warp_sum_d(z);
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) nz += __shfl_xor_sync(kFull, nz, d);
  // the record head (warp 0 alone for a short list; after the participants'
  // partials for the heavy merge)
  auto write_head = [&](double Zs, double NZ) {
    double *dst = io.rank_part;
    dst[0] = m0;
    dst[1] = Zs;
    dst[2] = NF;
    sc[kFmRec + 0] = m0;
    sc[kFmRec + 1] = Zs;
    sc[kFmRec + 2] = NF;
    misc[41] = NZ;  // nonzero weights (the only one, if NZ == 1, is the minimum's: sc[kFmBest])
    if (trace_head) trace_head[4] = gtimer();
  };
  if (total <= 32 && tid == 0) write_head(z, (double)nz);
  __syncthreads();
  const int ncand = total;  // list length (zero weights included)
  const bool heavy = ncand > kLightMax;
  unsigned int *hc = io.counters + (ctas + kGroup - 1) / kGroup + 2;  // merge words (kHc*)
  const int ph = merge_helpers(io, ctas);
  if (tid == 0) {  // verdict to the waiting helper CTAs (the lists are published by the barrier + fence)
    // list length: read by the helpers (heavy) and by vpb_smpc_debug_weights
    hc[kHcCount] = (unsigned int)ncand;
    if (heavy) {  // what the participants need to expand their slices of the CTA list
      const unsigned long long mb = (unsigned long long)__double_as_longlong(m0);
      hc[kHcM0] = (unsigned int)mb;
      hc[kHcM0 + 1] = (unsigned int)(mb >> 32);
      for (int w = 0; w < nw; ++w) hc[kHcWcount + w] = (unsigned int)wcount[w];
      hc[kHcSpan] = (unsigned int)span;
      hc[kHcNw] = (unsigned int)nw;
      hc[kHcList] = (unsigned int)(ncand / NWC);
      // about nt / 8 candidates per participant: the slice's row loads take
      // two round trips; the partials are added per element in parallel
      // (heavy_sum_slice), so more participants cost little (r2: converged
      // C3 step 71.7 -> 59.6 us, converged M = 256 80.6 -> 55.3 us)
      const int want = (ncand + nt / 8 - 1) / (nt / 8);
      hc[kHcParts] = (unsigned int)(want < ph + 1 ? (want > 1 ? want : 1) : ph + 1);
      fence_acq_rel_gpu();  // helpers read the lists and these words after this release
    }
    *reinterpret_cast<volatile unsigned int *>(hc + kHcFlag) = ((ep & 0x3fffffffu) << 2) | (heavy ? 2u : 1u);
    hc[0] = ep + 1u;  // next launch's epoch (every CTA of this one has read it)
  }
  if (heavy) {
    // this CTA is the last participant; then the partials in participant order
    __syncthreads();  // (thread 0 published the participants' words above)
    if (trace_head && tid == 0) trace_head[7] = gtimer();
    const int P = (int)__ldcg(hc + kHcParts);
    heavy_part<ET, NWC>(io, S, hc, P - 1, P, hn);
    if (trace_head && tid == 0) trace_head[8] = gtimer();
    heavy_sum_slice(io, S, hc, P - 1, P, hn);
    if (tid == 0) {
      SpinGuard g;
      while (ld_acquire_gpu(hc + kHcDone2) != (unsigned int)P) g.pause(32);
      hc[kHcDone] = 0u;  // every participant is past both counters
      hc[kHcDone2] = 0u;
    }
    __syncthreads();
    if (trace_head && tid == 0) trace_head[9] = gtimer();
    // Z and the nonzero count: fixed-shape block reduction over the
    // participants (thread q holds participant q); N is in rank_part
    const int Lp = 2 + hn;
    const double zq = tid < P ? __ldcg(io.hparts + (size_t)tid * Lp) : 0.0;
    const double nq = tid < P ? __ldcg(io.hparts + (size_t)tid * Lp + 1) : 0.0;
    const double zw = warp_sum_d(zq), nw_ = warp_sum_d(nq);
    if (lane == 0) {
      misc[16 + warp] = zw;
      misc[32 + warp] = nw_;
    }
    __syncthreads();
    if (tid == 0) {
      double Zs = 0.0, NZ = 0.0;
      for (int w = 0; w < nw; ++w) {  // fixed warp order
        Zs += misc[16 + w];
        NZ += misc[32 + w];
      }
      write_head(Zs, NZ);
      if (trace_head) trace_head[10] = gtimer();
    }
    __syncthreads();
  }
  if (tid == 32) {
    // record tail: best index and the extension [nonzero count, the single
    // candidate's 6 sums] (lets a multi-device finish skip the re-evaluation)
    double *dst = io.rank_part;
    dst[3] = sc[kFmRec + 3];
    double *ext = dst + kPartHead + hn;
    const double nnz = misc[41];
    const bool one = nnz == 1.0 && io.cand_terms && sc[kFmBest] >= 0.0;
    ext[0] = (FIXED && io.cand_terms) ? nnz : -1.0;
    for (int a = 0; a < 6; ++a) ext[1 + a] = one ? sc[kFmCT + a] : 0.0;
  }
  // 4. N = sum_m w_m eps_m over the nonzero candidates, in candidate order
  //    (+ U* = nominal + N / Z, clipped command, shifted warm start)
  const ET *eps = reinterpret_cast<const ET *>(io.eps);
  const double Z = sc[kFmRec + 1];
#pragma unroll 1
  for (int e = tid; e < hn; e += nt) {
    double acc = 0.0;
    if (heavy) {
      acc = __ldcg(io.rank_part + kPartHead + e);  // (the participants' sums, acquired above)
    } else {  // <= kLightMax candidates: smem lists
      const int *ml = smlist;
      const double *wl = sc + kFmW;
      int k = 0;
#pragma unroll 1
      for (; k + 4 <= ncand; k += 4) {
        double a[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) a[t] = load_e<ET>(eps + (size_t)ml[k + t] * hn + e);
#pragma unroll
        for (int t = 0; t < 4; ++t) acc += wl[k + t] * a[t];
      }
#pragma unroll 1
      for (; k < ncand; ++k) acc += wl[k] * load_e<ET>(eps + (size_t)ml[k] * hn + e);
      io.rank_part[kPartHead + e] = acc;
    }
    if (fused_u) {  // tail_controls, element e
      const double u = nominal[e] + acc / Z;
      const int64_t o2 = (int64_t)hn + e;  // clipped command (e < nj) / shifted warm start
      double v2 = u;
      if (e < nj) {
        const double lim = io.acc.v[e];
        v2 = u < -lim ? -lim : (u > lim ? lim : u);
      }
      io.out[e] = u;
      io.out[o2] = v2;
      if (io.out_host) {
        io.out_host[e] = u;
        io.out_host[o2] = v2;
      }
    }
  }
  if (fused_u) {
    for (int e = tid; e < nj; e += nt) {
      io.out[2 * (int64_t)hn + e] = 0.0;
      if (io.out_host) io.out_host[2 * (int64_t)hn + e] = 0.0;
    }
  }
  __syncthreads();
}

// Per-CTA head (warp 0: min cost, non-finite count, best index of the CTA's
// candidates; costs to `costs`), publication, and -- on the last CTA -- the
// final merge.  Returns true on the CTA that merged.
template <typename ET, int NWC, bool FIXED>
__device__ bool cta_reduce_and_merge(const SmpcIO &io, const Shared &S, int64_t cta_m0, int hn, int nj, int cta,
                                     int ctas, const double *nominal) {
  const int groups = (ctas + kGroup - 1) / kGroup;
  double *heads = io.cta_parts;  // [3][ctas]
  double *costs = io.costs ? io.costs : io.cand_costs;
  unsigned int *flag = reinterpret_cast<unsigned int *>(S.misc + 44);
  if (threadIdx.x < 32) {
    // this launch's merge epoch (it advances only after the last ticket):
    // loaded first so its latency hides under the candidate writes below
    const unsigned int ep = threadIdx.x == 0 ? *reinterpret_cast<volatile unsigned int *>(io.counters + groups + 2) : 0u;
    const int w = threadIdx.x;
    const int64_t m = cta_m0 + w;
    double c = dinf();
    bool failed = false;
    if (w < NWC && m < io.M) {
      const double *sm = S.sums + w * 6;
      failed = S.fail[w] != 0 || S.tfail[w] != 0;
      c = failed ? dinf() : sm[0] + sm[1] + sm[2] + sm[3] + sm[4] + S.cost[w];
      costs[m] = c;
      if (io.flags) io.flags[m] = failed ? 1 : 0;
      if (io.cand_terms) {  // the five running sums + terminal (without the q_0 terms)
        double *ct = io.cand_terms + 6 * (size_t)m;
        for (int a = 0; a < 5; ++a) ct[a] = sm[a];
        ct[5] = S.cost[w];
      }
    }
    const bool real = w < NWC && m < io.M;
    // non-finite costs: the reference's flagged samples (DegenerateRotation,
    // vp/planner.py:540-546) counted apart from any other non-finite cost
    // (ValueError in soft_weights): count = flagged + 2^32 other
    const unsigned fmk = __ballot_sync(kFull, real && failed);
    const unsigned omk = __ballot_sync(kFull, real && !failed && !(c < dinf()));
    double mn = c;
    int bi = real ? w : 0x7fffffff;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      const double ov = __shfl_xor_sync(kFull, mn, d);
      const int oi = __shfl_xor_sync(kFull, bi, d);
      if (ov < mn || (ov == mn && oi < bi)) {
        mn = ov;
        bi = oi;
      }
    }
    // lanes 1.. wrote costs / flags / sums above: order them before lane 0's
    // release (__syncwarp orders memory among its threads; the fence is
    // cumulative only over writes lane 0 has observed)
    __syncwarp();
    if (w == 0) {
      heads[cta] = mn;
      heads[ctas + cta] = (double)__popc(fmk) + 4294967296.0 * (double)__popc(omk);
      heads[2 * (size_t)ctas + cta] = mn < dinf() ? (double)(io.m_offset + cta_m0 + bi) : -1.0;
      // publication: the ticket is an acquire-release atomic at gpu scope --
      // it releases this CTA's head (and, cumulatively, the lanes' writes
      // ordered by the __syncwarp above) and, for the CTA taking the last
      // ticket, acquires every other CTA's
#ifdef VPB_FENCED_TICKET
      fence_acq_rel_gpu();
      const unsigned int prev = atomicAdd(&io.counters[groups], 1u);
      const bool last = prev == (unsigned int)(ctas - 1);
      if (last) fence_acq_rel_gpu();
#else
      unsigned int prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&io.counters[groups]) : "memory");
      const bool last = prev == (unsigned int)(ctas - 1);
#endif
      const int ph = merge_helpers(io, ctas);
      const bool helper = !last && (int)prev >= ctas - 1 - ph;
      flag[0] = last ? 1u : (helper ? 3u : 0u);
      flag[1] = helper ? (unsigned int)((int)prev - (ctas - 1 - ph)) : 0u;
      reinterpret_cast<unsigned int *>(S.misc + 46)[0] = ep;
    }
  }
  __syncthreads();
  VPB_TRACE(io, 2 * ctas + 3 + (cta % 4));
  if (flag[0] == 0u) return false;
  const unsigned int ep = reinterpret_cast<const unsigned int *>(S.misc + 46)[0];
  if (flag[0] == 3u) {
    merge_helper<ET, NWC>(io, S, ctas, hn, (int)flag[1], ep);
    return false;
  }
  VPB_TRACE(io, 2 * ctas);
  final_merge<ET, NWC, FIXED>(io, S, heads, costs, ctas, hn, nj, FIXED && io.finish, ep,
                              io.trace ? io.trace + 2 * ctas + 13 : nullptr, nominal);
  if (threadIdx.x == 0) io.counters[groups] = 0u;
  VPB_TRACE(io, 2 * ctas + 1);
  return true;
}

// Session staging (see SmpcIO::stage_src).  The staging word holds
// epoch + 1 of the launch that filled the device copy; the epoch advances only
// after the merge, which no CTA of this launch can have passed yet.
__device__ __forceinline__ void stage_inputs(const SmpcIO &io, int ctas) {
  unsigned int *hc = io.counters + (ctas + kGroup - 1) / kGroup + 2;
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < io.stage_len; i += blockDim.x) io.stage_dst[i] = __ldcv(io.stage_src + i);
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int ep = *reinterpret_cast<volatile unsigned int *>(hc);
      fence_acq_rel_gpu();  // cumulative over the CTA's copies (ordered by the barrier)
      *reinterpret_cast<volatile unsigned int *>(hc + kHcStage) = ep + 1u;
    }
  } else {
    if (threadIdx.x == 0) {
      const unsigned int want = *reinterpret_cast<volatile unsigned int *>(hc) + 1u;
      SpinGuard g;
#ifndef VPB_STAGE_SLEEP_NS
#define VPB_STAGE_SLEEP_NS 20
#endif
      while (ld_acquire_gpu(hc + kHcStage) != want) g.pause(VPB_STAGE_SLEEP_NS);
    }
  }
  __syncthreads();
}

// Fused SMPC step: rollout -> CTA partial -> group merge -> global merge
// [-> U*, clip, shift, re-evaluation].
template <typename T, typename ET, int MAXJ, typename Topo, bool INL = false>
__global__ void __launch_bounds__(smpc_threads<Topo>(), smpc_min_blocks<T, Topo>())
    smpc_kernel(const __grid_constant__ Prob<T> P, const __grid_constant__ SmpcIO io,
                const __grid_constant__ NomInline<INL> nin) {
#ifdef VPB_SMEM_SPILL
  // the fixed path's layout is a compile-time constant: static shared memory,
  // and the register spills of the 72-register budget go to shared memory
  // instead of local memory (which 7 CTAs per SM push out of L1 into L2)
  unsigned char *smem_raw;
  if constexpr (!is_dyn_v<Topo>) {
    asm volatile(".pragma \"enable_smem_spilling\";");
    __shared__ __align__(16) unsigned char smem_fixed[smem_layout(0, sizeof(T), kMergeScratch).total];
    smem_raw = smem_fixed;
  } else {
    extern __shared__ __align__(16) unsigned char smem_dyn[];
    smem_raw = smem_dyn;
  }
#else
  extern __shared__ __align__(16) unsigned char smem_raw[];
#endif
  const SmemLayout L = smem_layout(is_dyn_v<Topo> ? P.ns : 0, sizeof(T), kMergeScratch);
  const Shared S = carve(smem_raw, L);
  Dyn<T> &D = *reinterpret_cast<Dyn<T> *>(S.dyn);
  const double *nominal = io.nominal;
  if constexpr (!is_dyn_v<Topo>) {
    if (io.stage_src) stage_inputs(io, (int)gridDim.x - 1);
    if constexpr (INL) {
      // session: the nominal rides in the launch parameters; each CTA copies
      // it to shared memory (ordered by the barrier below) and reads it there
      __shared__ double nom_s[VPB_NOM_INLINE];
      for (int i = threadIdx.x; i < nin.n; i += blockDim.x) nom_s[i] = nin.v[i];
      nominal = nom_s;
    }
  }
  if (threadIdx.x < 32) load_dyn<T>(P, io.dyn, D);
  __syncthreads();
  const int64_t cta_m0 = (int64_t)blockIdx.x * smpc_nw<Topo>();
  const int hn = P.H * P.nj;
  const ET *eps = reinterpret_cast<const ET *>(io.eps);
  if constexpr (is_dyn_v<Topo>) {
    VPB_TRACE(io, 2 * blockIdx.x);
    CandOut co{nullptr, nullptr, nullptr};
    evaluate_cta<T, ET, MAXJ>(P, D, eps, io.nominal, io.M, cta_m0, S, co);
    if (!cta_reduce_and_merge<ET, smpc_nw<Topo>(), false>(io, S, cta_m0, hn, P.nj, blockIdx.x, gridDim.x,
                                                         io.nominal))
      return;
    if (io.finish) {
      smpc_tail_dyn<T, MAXJ>(P, D, io.rank_part, io.nominal, io.acc, io.out, S);
      if (io.out_host) {
        __syncthreads();
        const int len = 2 * P.H * P.nj + P.nj + 13;
        for (int e = threadIdx.x; e < len; e += blockDim.x) io.out_host[e] = io.out[e];
        signal_host_done(io.out_host + len);
      }
    }
  } else {
    if (blockIdx.x > 0) VPB_TRACE(io, 2 * (blockIdx.x - 1));
    // One call site, three uses: state 0 -- block 0 computes the q_0
    // prologue split over its warps into io.pro and raises the ready flag
    // (it is an extra block: it runs beside the candidates, off the critical
    // path); state 1 -- every warp of blocks 1.. scores its candidate;
    // state 2 (last candidate CTA) -- U* re-evaluated, split over the warps.
    const int warp = threadIdx.x >> 5;
    const int cta = (int)blockIdx.x - 1, ncta = (int)gridDim.x - 1;
    const int64_t cm0 = (int64_t)cta * smpc_nw<Topo>();
    unsigned int *pro_ready = io.counters + (ncta + kGroup - 1) / kGroup + 1;
    int state = blockIdx.x == 0 ? 0 : 1;
#pragma unroll 1
    for (;;) {
      const int64_t m = cm0 + warp;
      const bool cand = state == 1;
      const ET *ctrl = (cand && m < io.M) ? eps + (size_t)m * hn : nullptr;
      const double *nom = state == 1 ? nominal : (state == 2 ? io.out : nullptr);
      fixed_candidate<T, ET, Topo>(P, D, io.gen_on ? nullptr : ctrl, nom, cand ? m < io.M : true,
                                   state == 0 ? 1 : P.H, state == 0 ? 0 : 1, cand ? 0 : warp, cand ? 1 : NWF,
                                   S.sums + warp * 6, S.cost + warp, S.fail + warp,
                                   (cand && io.gen_on) ? &io.gen : nullptr, m, io.eps_out);
      __syncthreads();
      if (state == 0) {
        if (threadIdx.x < NWF) {
          const int w = threadIdx.x;
          io.pro[4 * w + 0] = S.sums[w * 6 + 0];
          io.pro[4 * w + 1] = S.sums[w * 6 + 1];
          io.pro[4 * w + 2] = (double)S.fail[w];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          fence_acq_rel_gpu();
          atomicExch(pro_ready, 1u);
        }
        return;
      }
      if (state == 2) break;
      S.tfail[warp] = 0;
      __syncthreads();
      VPB_TRACE(io, 2 * cta + 1);
      // (the final merge also fetched the q_0 terms into S.pro and, when
      // finishing, wrote U*, the command and the warm start)
      if (!cta_reduce_and_merge<ET, smpc_nw<Topo>(), true>(io, S, cm0, hn, P.nj, cta, ncta, nominal)) return;
      if (!io.finish) {
        fixed_shard_fixup(S, io.M, io.costs, io.flags, io.rank_part);
        return;
      }
      VPB_TRACE(io, 2 * ncta + 11);
      // One nonzero weight (the usual case at small lam): w = exp(0) = 1 and
      // Z = 1, so U* = nominal + eps_best exactly and its re-evaluation is the
      // best candidate's own evaluation -- reuse its sums (fetched by the
      // merge when that candidate is the minimum's, as it must be).
      // the only nonzero weight is the minimum's (w = exp(0) = 1): U* = nominal + its eps
      const int single = S.misc[41] == 1.0 ? (int)S.scratch[kFmBest] : -1;
      if (single >= 0 && S.scratch[kFmRec + 1] == 1.0) {
        if (threadIdx.x < NWF) {
          const bool spec = (int)S.scratch[kFmBest] == single;
          const double *ct = io.cand_terms + 6 * (size_t)single;
          const int w = threadIdx.x;
          for (int a = 0; a < 5; ++a) S.sums[w * 6 + a] = w == 0 ? (spec ? S.scratch[kFmCT + a] : __ldcg(ct + a)) : 0.0;
          S.cost[w] = w == 0 ? (spec ? S.scratch[kFmCT + 5] : __ldcg(ct + 5)) : 0.0;
          S.fail[w] = 0;
        }
        __syncthreads();
        break;
      }
      state = 2;
    }
    VPB_TRACE(io, 2 * ncta + 12);
    // combine the split re-evaluation (fixed warp order) + the q_0 terms
    if (threadIdx.x == 0) {
      for (int a = 0; a < 5; ++a) {
        double v = 0.0;
        for (int w = 0; w < NWF; ++w) v += S.sums[w * 6 + a];
        S.sums[a] = v;
      }
      double c = 0.0;
      int f = 0;
      for (int w = 0; w < NWF; ++w) {
        c += S.cost[w];
        f |= S.fail[w];
      }
      S.cost[0] = c;
      S.fail[0] = f;
      fixed_add_prologue(S, 0);
    }
    __syncthreads();
    const bool bad = *pro_fail(S) != 0;
    const double *rec = S.scratch + kFmRec;
    const double best = bad ? dinf() : rec[0] + S.pro[0] + S.pro[1];
    // (out_host: zero-copy result, posted PCIe writes visible after the kernel completes)
    tail_output(S, rec, P.H, P.nj, best, bad ? (double)io.M : rec[2], io.out, io.out_host);
    fixed_shard_fixup(S, io.M, io.costs, io.flags, nullptr);
    if (io.out_host) signal_host_done(io.out_host + 2 * P.H * P.nj + P.nj + 13);
    VPB_TRACE(io, 2 * ncta + 2);
  }
}

// Multi-device finish: merge R rank partials in rank order (their minima
// already include the q_0 terms), then the tail.
template <typename T, int MAXJ, typename Topo>
__global__ void __launch_bounds__(smpc_threads<Topo>(), 1)
    smpc_finish_kernel(const __grid_constant__ Prob<T> P, const double *parts, int n_parts, double lam,
                       const double *nominal, const AccLimit acc, double *merged, double *out, const double *dyn) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SmemLayout L = smem_layout(is_dyn_v<Topo> ? P.ns : 0, sizeof(T), n_parts + 512);
  const Shared S = carve(smem_raw, L);
  Dyn<T> &D = *reinterpret_cast<Dyn<T> *>(S.dyn);
  if (threadIdx.x < 32) load_dyn<T>(P, dyn, D);
  __syncthreads();
  merge_block(record_rows(parts, P.H * P.nj), n_parts, P.H * P.nj, lam, merged, S.scratch, S.misc);
  if constexpr (is_dyn_v<Topo>) {
    smpc_tail_dyn<T, MAXJ>(P, D, merged, nominal, acc, out, S);
  } else {
    tail_controls(merged, nominal, acc, P.H, P.nj, out);
    // one nonzero weight over all ranks (merged Z == 1, the minimum's rank has
    // a single nonzero candidate): U* = nominal + eps_best, reuse its sums
    const int hn = P.H * P.nj, Lr = kPartHead + hn + kPartExt;
    int *short_row = reinterpret_cast<int *>(S.misc + 46);
    if (threadIdx.x == 0) {
      int r0 = -1, nz = 0;
      for (int r = 0; r < n_parts; ++r) {
        const double mr = parts[(size_t)r * Lr], zr = parts[(size_t)r * Lr + 1];
        if (!(mr < dinf()) || zr * exp(-(mr - merged[0]) / lam) == 0.0) continue;
        ++nz;
        if (parts[(size_t)r * Lr + kPartHead + hn] == 1.0) r0 = r;
      }
      *short_row = (nz == 1 && merged[1] == 1.0) ? r0 : -1;
    }
    __syncthreads();
    const int srow = *short_row;
    const int warp = threadIdx.x >> 5;
    // pass 0: U* split over the warps (skipped by the shortcut); pass 1: the q_0 prologue, split
#pragma unroll 1
    for (int pass = srow >= 0 ? 1 : 0; pass < 2; ++pass) {
      double *base = pass == 0 ? S.sums : S.scratch;
      fixed_candidate<T, double, Topo>(P, D, nullptr, pass == 0 ? out : nullptr, true, pass == 0 ? P.H : 1,
                                       pass == 0 ? 1 : 0, warp, NWF, base + warp * 6,
                                       (pass == 0 ? S.cost : S.scratch + 6 * NWF) + warp,
                                       pass == 0 ? S.fail + warp : S.tfail + warp);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      for (int a = 0; a < 5; ++a) {
        double v = 0.0;
        for (int w = 0; w < NWF; ++w) v += S.sums[w * 6 + a];
        S.sums[a] = v;
      }
      double c = 0.0, pose0 = 0.0, coll0 = 0.0;
      int f = 0, bad = 0;
      for (int w = 0; w < NWF; ++w) {
        c += S.cost[w];
        f |= S.fail[w];
        pose0 += S.scratch[w * 6 + 0];
        coll0 += S.scratch[w * 6 + 1];
        bad |= S.tfail[w];
      }
      S.cost[0] = c;
      S.fail[0] = f;
      if (srow >= 0) {
        const double *ext = parts + (size_t)srow * Lr + kPartHead + hn + 1;
        for (int a = 0; a < 5; ++a) S.sums[a] = ext[a];
        S.cost[0] = ext[5];
        S.fail[0] = 0;
      }
      S.pro[0] = pose0;
      S.pro[1] = coll0;
      *pro_fail(S) = bad;
      fixed_add_prologue(S, 0);
    }
    __syncthreads();
    tail_output(S, merged, P.H, P.nj, merged[0], merged[2], out);
  }
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
    P.sq_dev = p->field_sq_dev;
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
  // derived constants of the fixed-topology path
  FixedConsts<T> &C = P.fc;
  const double vox = (f && f->sq) ? f->voxel : 1.0;
  const double outside = (f && f->sq) ? f->outside_default : 0.0;
  for (int s = 0; s < ns; ++s) {
    const double r = p->sph_r[s];
    const double dr = p->d_act + r;
    C.dr[s] = (T)dr;
    const double t = dr / vox;
    C.thr2[s] = (T)(t * t * (1.0 + 1e-4) + 1e-12);
    const double tf = t + 1.7320508075688772 + 0.01;  // + the cell diagonal + rounding margin (voxels)
    C.far2[s] = (T)(tf * tf);
    C.zero_cost[s] = (T)(p->w_env * (p->d_act - (0.0 - r)) * (p->d_act - (0.0 - r)));
    const double go = p->d_act - (outside - r);
    C.out_cost[s] = (T)(go > 0.0 ? p->w_env * go * go : 0.0);
  }
  for (int q = 0; q < p->n_pairs; ++q) {
    const double rs = p->sph_r[p->pairs[2 * q]] + p->sph_r[p->pairs[2 * q + 1]];
    C.rsum[q] = (T)rs;
    C.rsum2[q] = (T)(rs * rs * (1.0 + 1e-4) + 1e-12);
  }
  bool diag = true;
  int idx = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b, ++idx) {
      const double wq = a == b ? p->pose_weight[6 * a + a] : p->pose_weight[6 * a + b] + p->pose_weight[6 * b + a];
      const double wt =
          a == b ? p->terminal_weight[6 * a + a] : p->terminal_weight[6 * a + b] + p->terminal_weight[6 * b + a];
      C.Wq[idx] = (T)wq;
      C.Wt[idx] = (T)wt;
      if (a != b && (wq != 0.0 || wt != 0.0)) diag = false;
    }
  C.w_diag = diag ? 1 : 0;
  const int fn0 = P.has_field ? P.n0 : 1, fn1 = P.has_field ? P.n1 : 1, fn2 = P.has_field ? P.n2 : 1;
  C.off2 = fn2 >= 2 ? 1 : 0;
  C.off1 = fn1 >= 2 ? fn2 : 0;
  C.off0 = fn0 >= 2 ? fn1 * fn2 : 0;
  C.amax0 = (T)(fn0 >= 2 ? fn0 - 2 : 0);
  C.amax1 = (T)(fn1 >= 2 ? fn1 - 2 : 0);
  C.amax2 = (T)(fn2 >= 2 ? fn2 - 2 : 0);
  C.nf0 = (T)fn0;
  C.nf1 = (T)fn1;
  C.nf2 = (T)fn2;
  C.chi0 = (T)(fn0 - 1);
  C.chi1 = (T)(fn1 - 1);
  C.chi2 = (T)(fn2 - 1);
  return VPB_OK;
}

// VPB_GENERIC_ROLLOUT=1 forces the runtime-topology kernels (A/B parity tests).
static bool fixed_topology_disabled() {
  const char *e = getenv("VPB_GENERIC_ROLLOUT");
  return e && e[0] == '1';
}

// Does the packed problem have exactly the compile-time topology `Topo`?
static int axis_code(const double *u) {
  if (u[1] == 0.0 && u[2] == 0.0 && (u[0] == 1.0 || u[0] == -1.0)) return u[0] > 0 ? 1 : -1;
  if (u[0] == 0.0 && u[2] == 0.0 && (u[1] == 1.0 || u[1] == -1.0)) return u[1] > 0 ? 2 : -2;
  if (u[0] == 0.0 && u[1] == 0.0 && (u[2] == 1.0 || u[2] == -1.0)) return u[2] > 0 ? 3 : -3;
  return 0;
}

template <typename Topo>
static bool topo_matches(const vpb_problem *p) {
  if (p->n_joints != Topo::NJ || p->n_spheres != Topo::NS || p->n_pairs != Topo::NP) return false;
  for (int j = 0; j < Topo::NJ; ++j) {
    if (Topo::axis(j) != 0 && axis_code(p->axes + 3 * j) != Topo::axis(j)) return false;
    if (Topo::offset_kind(j) == 1) {
      for (int a = 0; a < 9; ++a)
        if (p->off_r[9 * j + a] != ((a % 4 == 0) ? 1.0 : 0.0)) return false;
      if (p->off_t[3 * j] != 0.0 || p->off_t[3 * j + 1] != 0.0) return false;
    }
  }
  for (int s = 0; s < Topo::NS; ++s) {
    if (p->sph_link[s] != Topo::link(s)) return false;
    if (Topo::sphere_kind(s) == 1 && (p->sph_loc[3 * s] != 0.0 || p->sph_loc[3 * s + 1] != 0.0)) return false;
  }
  for (int q = 0; q < Topo::NP; ++q)
    if (p->pairs[2 * q] != Topo::pair_i(q) || p->pairs[2 * q + 1] != Topo::pair_j(q)) return false;
  return true;
}

// 0 = generic (runtime topology), 1 = TopoRobot7
static int topo_id(const vpb_problem *p) { return topo_matches<TopoRobot7>(p) ? 1 : 0; }


template <typename T>
static size_t smem_bytes(const Prob<T> &P, int scratch, int topo) {
  return smem_layout(topo ? 0 : P.ns, sizeof(T), scratch).total;
}

template <typename K>
static int set_smem(K kern, size_t smem) {
  if (smem > 48 * 1024) VPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return VPB_OK;
}

template <typename T, typename ET>
static int launch_rollout_t(const Prob<T> &P, const RolloutIO &io, int topo, cudaStream_t s) {
#ifdef VPB_QUICK  // SASS-inspection builds (tools/quick_sass.sh): the production smpc kernel only
  return VPB_ERR_ARG;
#endif
  const size_t smem = smem_bytes(P, 0, topo);
  const unsigned grid = (unsigned)ceil_div(io.M, NW);
  if (grid == 0) return VPB_OK;
  int rc;
  if (topo == 1) {
    auto k = rollout_kernel<T, ET, 8, TopoRobot7>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<grid, kThreads, smem, s>>>(P, io);
  } else if (P.nj <= 8) {
    auto k = rollout_kernel<T, ET, 8, TopoDyn>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<grid, kThreads, smem, s>>>(P, io);
  } else {
    auto k = rollout_kernel<T, ET, kMaxJ, TopoDyn>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<grid, kThreads, smem, s>>>(P, io);
  }
  return check_launch("rollout_kernel");
}

// Resident CTA slots of kernel k on the current device (occupancy x SMs),
// cached per (kernel, device, smem): the helper cap of the merge protocol.
template <typename K>
static int resident_slots(K k, int threads, size_t smem) {
  static thread_local const void *c_k = nullptr;
  static thread_local int c_dev = -1, c_slots = 0;
  static thread_local size_t c_smem = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (c_k == (const void *)k && c_dev == dev && c_smem == smem) return c_slots;
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  c_k = (const void *)k;
  c_dev = dev;
  c_smem = smem;
  c_slots = per_sm * sms;
  return c_slots;
}

template <typename T, typename ET>
static int launch_smpc_t(const Prob<T> &P, const SmpcIO &io, int topo, cudaStream_t s) {
  const int64_t ctas = ceil_div(io.M, topo ? NWF : NW) + (topo ? 1 : 0);  // fixed path: + prologue block
  const size_t smem = smem_bytes(P, kMergeScratch, topo);
  int rc;
  auto go = [&](auto k, int threads) {
    SmpcIO io2 = io;
    const int slots = resident_slots(k, threads, smem);
    io2.max_helpers = slots - 2 < kMergeHelpers ? (slots - 2 > 0 ? slots - 2 : 0) : kMergeHelpers;
#ifdef VPB_SMEM_SPILL
    const size_t dsm = topo == 1 ? 0 : smem;
#else
    const size_t dsm = smem;
#endif
    k<<<(unsigned)ctas, threads, dsm, s>>>(P, io2, NomInline<false>{});
  };
#ifdef VPB_QUICK
  if constexpr (!std::is_same_v<T, float> || !std::is_same_v<ET, float>) return VPB_ERR_ARG;
  else {
    auto k = smpc_kernel<T, ET, 8, TopoRobot7>;
    if ((rc = set_smem(k, smem))) return rc;
    go(k, smpc_threads<TopoRobot7>());
    return check_launch("smpc_kernel");
  }
#endif
  if (topo == 1) {
    auto k = smpc_kernel<T, ET, 8, TopoRobot7>;
    if ((rc = set_smem(k, smem))) return rc;
    go(k, smpc_threads<TopoRobot7>());
  } else if (P.nj <= 8) {
    auto k = smpc_kernel<T, ET, 8, TopoDyn>;
    if ((rc = set_smem(k, smem))) return rc;
    go(k, kThreads);
  } else {
    auto k = smpc_kernel<T, ET, kMaxJ, TopoDyn>;
    if ((rc = set_smem(k, smem))) return rc;
    go(k, kThreads);
  }
  return check_launch("smpc_kernel");
}

template <typename T>
static int launch_finish_t(const Prob<T> &P, const double *parts, int n_parts, double lam, const double *nominal,
                           const AccLimit &acc, double *merged, double *out, const double *dyn, int topo,
                           cudaStream_t s) {
#ifdef VPB_QUICK
  return VPB_ERR_ARG;
#endif
  const size_t smem = smem_bytes(P, n_parts + 512, topo);
  int rc;
  if (topo == 1) {
    auto k = smpc_finish_kernel<T, 8, TopoRobot7>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<1, smpc_threads<TopoRobot7>(), smem, s>>>(P, parts, n_parts, lam, nominal, acc, merged, out, dyn);
  } else if (P.nj <= 8) {
    auto k = smpc_finish_kernel<T, 8, TopoDyn>;
    if ((rc = set_smem(k, smem))) return rc;
    k<<<1, kThreads, smem, s>>>(P, parts, n_parts, lam, nominal, acc, merged, out, dyn);
  } else {
    auto k = smpc_finish_kernel<T, kMaxJ, TopoDyn>;
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
  double *cta_parts, *group_parts, *rank_part, *pro, *cand_costs, *cand_terms, *hparts;
  unsigned int *counters;
  size_t bytes;
};

static SmpcWs smpc_ws(void *base, int64_t M, int64_t H, int64_t n) {
  const int64_t ctas = ceil_div(M > 0 ? M : 1, NWF);  // the larger CTA count of the two paths
  const int64_t groups = ceil_div(ctas, kGroup);
  const int64_t L = kPartHead + H * n + kPartExt;
  SmpcWs w;
  char *b = reinterpret_cast<char *>(base);
  size_t o = 0;
  w.cta_parts = reinterpret_cast<double *>(b + o);  // CTA heads [3][ctas]
  o += align_up((size_t)ctas * 3 * 8, 256);
  w.group_parts = reinterpret_cast<double *>(b + o);  // merge scratch: weights, candidate and CTA lists
  o += align_up((size_t)(2 * (M + 64) + ctas + 600) * 8, 256);
  w.cand_costs = reinterpret_cast<double *>(b + o);
  o += align_up((size_t)(M > 0 ? M : 1) * 8, 256);
  w.cand_terms = reinterpret_cast<double *>(b + o);
  o += align_up((size_t)(M > 0 ? M : 1) * 6 * 8, 256);
  w.rank_part = reinterpret_cast<double *>(b + o);
  o += align_up((size_t)L * 8, 256);
  w.pro = reinterpret_cast<double *>(b + o);
  o += align_up((size_t)NWF * 4 * 8, 256);
  w.counters = reinterpret_cast<unsigned int *>(b + o);
  o += align_up((size_t)(groups + 2 + kHcWords) * 4, 256);  // group counters, ticket, prologue flag, merge words
  w.hparts = reinterpret_cast<double *>(b + o);  // heavy-merge partials of up to kMergeHelpers + 1 participants
  o += align_up((size_t)(kMergeHelpers + 1) * (2 + H * n) * 8, 256);
  w.bytes = o;
  return w;
}

}  // namespace vpb

using namespace vpb;

static unsigned long long *g_smpc_trace = nullptr;

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
  // the fixed-topology kernels do not emit per-step trajectories / spheres
  const int topo = (traj_q || sphere_pos || fixed_topology_disabled()) ? 0 : topo_id(prob);
  if (precision == VPB_PREC_F64) {
    Prob<double> P;
    if ((rc = build_prob<double>(prob, field, P))) return rc;
    return dtype == VPB_DTYPE_F32 ? launch_rollout_t<double, float>(P, io, topo, s)
                                  : launch_rollout_t<double, double>(P, io, topo, s);
  }
  Prob<float> P;
  if ((rc = build_prob<float>(prob, field, P))) return rc;
  return dtype == VPB_DTYPE_F32 ? launch_rollout_t<float, float>(P, io, topo, s)
                                : launch_rollout_t<float, double>(P, io, topo, s);
}

int64_t vpb_smpc_partial_len(int64_t H, int64_t n) { return kPartHead + H * n + kPartExt; }

void vpb_debug_smpc_trace(unsigned long long *dev_buffer) { g_smpc_trace = dev_buffer; }

size_t vpb_smpc_workspace_bytes(int64_t M, int64_t H, int64_t n) { return smpc_ws(nullptr, M, H, n).bytes + 256; }

int64_t vpb_smpc_out_len(int64_t H, int64_t n) { return 2 * H * n + n + 13; }

static int smpc_launch(const vpb_problem *prob, const vpb_field *field, const void *eps, int dtype,
                       const double *nominal, int64_t M, int64_t m_offset, int precision, double *costs,
                       uint8_t *flags, double *part_out, double *out, void *workspace, size_t workspace_bytes,
                       cudaStream_t s, const NoiseGen *gen = nullptr, bool counters_zeroed = false,
                       double *out_host = nullptr, const double *stage_src = nullptr,
                       double *stage_dst = nullptr, int64_t stage_len = 0) {
  int rc = prob_checks(prob, precision, dtype);
  if (rc) return rc;
  VPB_REQUIRE(eps && nominal && M >= 1, "bad arguments to the SMPC step");
  VPB_REQUIRE(prob->lam > 0.0, "temperature must be positive");
  const int64_t H = prob->horizon, n = prob->n_joints;
  VPB_REQUIRE(M <= ((int64_t)1 << 31) * NWF, "too many samples");
  const SmpcWs w = smpc_ws(workspace, M, H, n);
  VPB_REQUIRE(workspace && workspace_bytes >= w.bytes, "workspace too small");
  const int64_t ctas = ceil_div(M, NWF);
  const int64_t groups = ceil_div(ctas, kGroup);
  if (!counters_zeroed) VPB_CUDA(cudaMemsetAsync(w.counters, 0, (size_t)(groups + 2 + kHcWords) * 4, s));
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
  io.pro = w.pro;
  io.cand_costs = w.cand_costs;
  io.cand_terms = w.cand_terms;
  io.hparts = w.hparts;
  io.finish = out != nullptr;
  io.out = out;
  io.acc = acc_of(prob);
  io.dyn = prob->dyn_state;
  io.trace = g_smpc_trace;
  io.out_host = out_host;
  io.stage_src = stage_src;
  io.stage_dst = stage_dst;
  io.stage_len = (int)stage_len;
  const int topo = fixed_topology_disabled() ? 0 : topo_id(prob);
  if (gen) {  // fused draw (eps is the output buffer of the draws)
    io.gen = *gen;
    io.gen_on = 1;
    io.eps_out = reinterpret_cast<float *>(const_cast<void *>(eps));
  }
  if (precision == VPB_PREC_F64) {
    Prob<double> P;
    if ((rc = build_prob<double>(prob, field, P))) return rc;
    return dtype == VPB_DTYPE_F32 ? launch_smpc_t<double, float>(P, io, topo, s)
                                  : launch_smpc_t<double, double>(P, io, topo, s);
  }
  Prob<float> P;
  if ((rc = build_prob<float>(prob, field, P))) return rc;
  return dtype == VPB_DTYPE_F32 ? launch_smpc_t<float, float>(P, io, topo, s)
                                : launch_smpc_t<float, double>(P, io, topo, s);
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

int vpb_smpc_generate(const vpb_problem *prob, const vpb_field *field, uint64_t seed, const uint64_t *seed_dev,
                      int64_t m_offset, int64_t window, const double *sigma, const double *nominal, int64_t M,
                      int precision, double *costs, uint8_t *flags, void *eps_out, double *part_out, double *out,
                      void *workspace, size_t workspace_bytes, void *stream) {
  VPB_REQUIRE(prob && sigma && eps_out, "null argument to vpb_smpc_generate");
  VPB_REQUIRE((part_out == nullptr) != (out == nullptr), "exactly one of part_out / out");
  VPB_REQUIRE(window >= 1 && window <= 9, "noise window must be in [1, 9]");
  cudaStream_t s = as_stream(stream);
  const int64_t H = prob->horizon, n = prob->n_joints;
  const int dtype = precision == VPB_PREC_F32 ? VPB_DTYPE_F32 : VPB_DTYPE_F64;
  const bool fused = precision == VPB_PREC_F32 && window <= 5 && !fixed_topology_disabled() && topo_id(prob) == 1;
  if (fused) {
    NoiseGen g;
    memset(&g, 0, sizeof(g));
    g.seed = seed;
    g.seed_dev = seed_dev;
    g.m_offset = m_offset;
    g.window = (int)window;
    for (int64_t j = 0; j < n; ++j) g.sigma[j] = (float)sigma[j];
    return smpc_launch(prob, field, eps_out, VPB_DTYPE_F32, nominal, M, m_offset, precision, costs, flags, part_out,
                       out, workspace, workspace_bytes, s, &g);
  }
  // runtime topology / fp64 / wide windows: the stand-alone sampler (same draws), then the step
  int rc = vpb_sample_perturbations(seed, seed_dev, m_offset, M, H, n, window, sigma, dtype, eps_out, stream);
  if (rc) return rc;
  return smpc_launch(prob, field, eps_out, dtype, nominal, M, m_offset, precision, costs, flags, part_out, out,
                     workspace, workspace_bytes, s);
}

}  // extern "C"

namespace vpb {
// Debug export of the fused step's softmin weights: the final merge leaves
// its weight list (w_k = exp(-(S_k - min)/lam), uncompacted, zero weights
// included) and candidate indices in the workspace and the list length in
// the merge words; w_m / Z is scattered to weights[m].
__global__ void debug_weights_kernel(const double *wlist, const int *mlist, const unsigned int *ncand_p,
                                     const double *rank_part, double *weights) {
  const int ncand = (int)*ncand_p;
  const double Z = rank_part[1];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ncand; k += gridDim.x * blockDim.x) {
    const double w = wlist[k];
    if (w != 0.0) weights[mlist[k]] = w / Z;  // zero-weight padding slots may alias sample 0
  }
}
}  // namespace vpb

extern "C" {
int vpb_smpc_debug_weights(const vpb_problem *prob, int64_t M, const void *workspace, size_t workspace_bytes,
                           double *weights, void *stream) {
  VPB_REQUIRE(prob && workspace && weights && M >= 1, "bad arguments to vpb_smpc_debug_weights");
  const SmpcWs w = smpc_ws(const_cast<void *>(workspace), M, prob->horizon, prob->n_joints);
  VPB_REQUIRE(workspace_bytes >= w.bytes, "workspace too small");
  const int topo = fixed_topology_disabled() ? 0 : topo_id(prob);
  const int64_t ctas = ceil_div(M, topo ? NWF : NW);
  const int64_t groups = ceil_div(ctas, kGroup);
  const unsigned int *hc = w.counters + groups + 2;
  cudaStream_t s = as_stream(stream);
  VPB_CUDA(cudaMemsetAsync(weights, 0, (size_t)M * 8, s));
  debug_weights_kernel<<<(unsigned)(ceil_div(M, 256) < 1024 ? ceil_div(M, 256) : 1024), 256, 0, s>>>(
      w.group_parts, reinterpret_cast<const int *>(w.group_parts + M + 64), hc + kHcCount, w.rank_part, weights);
  return check_launch("debug_weights_kernel");
}
}  // extern "C"

namespace vpb {
// Session variant of vpb_smpc_generate (single-device step): the workspace's
// counters are zero on entry (zeroed once at session creation; every launch
// returns them to zero), and the result is also written to a host-mapped
// buffer by the kernel itself -- no memset and no D2H copy node.
int smpc_generate_session(const vpb_problem *prob, const vpb_field *field, const uint64_t *seed_dev, int64_t window,
                          const double *sigma, const double *nominal, int64_t M, int precision, void *eps_out,
                          double *out, double *out_host, void *workspace, size_t workspace_bytes,
                          cudaStream_t s, const double *stage_src, double *stage_dst, int64_t stage_len) {
  const int64_t n = prob->n_joints;
  const bool fused = precision == VPB_PREC_F32 && window <= 5 && !fixed_topology_disabled() && topo_id(prob) == 1;
  const bool in_kernel_stage = fused && getenv("VPB_SESSION_COPY_NODE") == nullptr;
  if (stage_src && !in_kernel_stage)
    VPB_CUDA(cudaMemcpyAsync(stage_dst, stage_src, (size_t)stage_len * 8, cudaMemcpyHostToDevice, s));
  if (fused) {
    NoiseGen g;
    memset(&g, 0, sizeof(g));
    g.seed_dev = seed_dev;
    g.window = (int)window;
    for (int64_t j = 0; j < n; ++j) g.sigma[j] = (float)sigma[j];
    return smpc_launch(prob, field, eps_out, VPB_DTYPE_F32, nominal, M, 0, precision, nullptr, nullptr, nullptr, out,
                       workspace, workspace_bytes, s, &g, true, out_host, in_kernel_stage ? stage_src : nullptr,
                       stage_dst, stage_len);
  }
  const int dtype = precision == VPB_PREC_F32 ? VPB_DTYPE_F32 : VPB_DTYPE_F64;
  int rc = vpb_sample_perturbations(0, seed_dev, 0, M, prob->horizon, n, window, sigma, dtype, eps_out, s);
  if (rc) return rc;
  return smpc_launch(prob, field, eps_out, dtype, nominal, M, 0, precision, nullptr, nullptr, nullptr, out, workspace,
                     workspace_bytes, s, nullptr, true, out_host);
}

// Session launch of the fused fp32 fixed-topology step with the per-call
// state in the launch parameters: q0, qd0, goal in Prob, the seed in the
// noise generator, the field pointer in Prob, the nominal inline in SmpcIO.
// Built once per session, patched every step (smpc_session_node_patch).
struct SmpcNode {
  Prob<float> P;
  SmpcIO io;
  NomInline<true> nin;
  void *args[3];
  cudaKernelNodeParams np;
  int nj, hn;
};

int smpc_session_node(const vpb_problem *prob, const vpb_field *field, int64_t window, const double *sigma,
                      int64_t M, int precision, void *eps_out, double *out, double *out_host, void *workspace,
                      size_t workspace_bytes, SmpcNode **res) {
  *res = nullptr;
  const bool fused = precision == VPB_PREC_F32 && window <= 5 && !fixed_topology_disabled() && topo_id(prob) == 1 &&
                     (int64_t)prob->horizon * prob->n_joints <= VPB_NOM_INLINE;
  if (!fused || getenv("VPB_SESSION_STAGE")) return VPB_OK;  // the caller stages the per-call block instead
  int rc = prob_checks(prob, precision, VPB_DTYPE_F32);
  if (rc) return rc;
  VPB_REQUIRE(prob->lam > 0.0, "temperature must be positive");
  const int64_t H = prob->horizon, n = prob->n_joints;
  VPB_REQUIRE(M >= 1 && M <= ((int64_t)1 << 31) * NWF, "bad sample count");
  const SmpcWs w = smpc_ws(workspace, M, H, n);
  VPB_REQUIRE(workspace && workspace_bytes >= w.bytes, "workspace too small");
  vpb_problem pb = *prob;
  pb.dyn_state = nullptr;  // the per-call state travels in the launch parameters
  pb.field_sq_dev = nullptr;
  auto *nd = new SmpcNode();
  memset(nd, 0, sizeof(*nd));
  if ((rc = build_prob<float>(&pb, field, nd->P))) {
    delete nd;
    return rc;
  }
  SmpcIO &io = nd->io;
  io.eps = eps_out;
  io.nominal = nullptr;  // (the INL kernel reads nin instead)
  io.M = M;
  io.lam = prob->lam;
  io.cta_parts = w.cta_parts;
  io.group_parts = w.group_parts;
  io.counters = w.counters;
  io.rank_part = w.rank_part;
  io.pro = w.pro;
  io.cand_costs = w.cand_costs;
  io.cand_terms = w.cand_terms;
  io.hparts = w.hparts;
  io.finish = 1;
  io.out = out;
  io.acc = acc_of(prob);
  io.trace = g_smpc_trace;
  io.out_host = out_host;
  nd->nin.n = (int)(H * n);
  io.gen.window = (int)window;
  for (int64_t j = 0; j < n; ++j) io.gen.sigma[j] = (float)sigma[j];
  io.gen_on = 1;
  io.eps_out = reinterpret_cast<float *>(eps_out);
  auto k = smpc_kernel<float, float, 8, TopoRobot7, true>;
  const size_t smem = smem_bytes(nd->P, kMergeScratch, 1);
  if ((rc = set_smem(k, smem))) {
    delete nd;
    return rc;
  }
  const int threads = smpc_threads<TopoRobot7>();
  const int slots = resident_slots(k, threads, smem);
  io.max_helpers = slots - 2 < kMergeHelpers ? (slots - 2 > 0 ? slots - 2 : 0) : kMergeHelpers;
#ifdef VPB_SMEM_SPILL
  const size_t dsm = 0;
#else
  const size_t dsm = smem;
#endif
  nd->args[0] = &nd->P;
  nd->args[1] = &nd->io;
  nd->args[2] = &nd->nin;
  nd->np.func = reinterpret_cast<void *>(k);
  nd->np.gridDim = dim3((unsigned)(ceil_div(M, NWF) + 1));
  nd->np.blockDim = dim3((unsigned)threads);
  nd->np.sharedMemBytes = (unsigned)dsm;
  nd->np.kernelParams = nd->args;
  nd->np.extra = nullptr;
  nd->nj = (int)n;
  nd->hn = (int)(H * n);
  *res = nd;
  return VPB_OK;
}

void smpc_session_node_patch(SmpcNode *nd, const double *q0, const double *qd0, const double *goal_r,
                             const double *goal_t, const double *nominal, uint64_t seed, const float *sq) {
  for (int j = 0; j < nd->nj; ++j) {
    nd->P.q0[j] = (float)q0[j];
    nd->P.qd0[j] = (float)qd0[j];
  }
  for (int a = 0; a < 9; ++a) nd->P.goal_r[a] = (float)goal_r[a];
  for (int a = 0; a < 3; ++a) nd->P.goal_t[a] = (float)goal_t[a];
  if (nd->P.has_field && sq) nd->P.sq = sq;
  if (nominal) memcpy(nd->nin.v, nominal, (size_t)nd->hn * 8);
  else memset(nd->nin.v, 0, (size_t)nd->hn * 8);
  nd->io.gen.seed = seed;
}

const cudaKernelNodeParams *smpc_session_node_params(const SmpcNode *nd) { return &nd->np; }

void smpc_session_node_free(SmpcNode *nd) { delete nd; }

}  // namespace vpb

extern "C" {

size_t vpb_smpc_finish_workspace_bytes(int64_t n_parts, int64_t H, int64_t n) {
  (void)n_parts;
  return align_up((size_t)(kPartHead + H * n + kPartExt) * 8, 256) + 256;
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
  const int topo = fixed_topology_disabled() ? 0 : topo_id(prob);
  if (precision == VPB_PREC_F64) {
    Prob<double> P;
    if ((rc = build_prob<double>(prob, field, P))) return rc;
    return launch_finish_t<double>(P, partials, (int)n_parts, prob->lam, nominal, acc, merged, out, prob->dyn_state,
                                   topo, s);
  }
  Prob<float> P;
  if ((rc = build_prob<float>(prob, field, P))) return rc;
  return launch_finish_t<float>(P, partials, (int)n_parts, prob->lam, nominal, acc, merged, out, prob->dyn_state,
                                topo, s);
}

}  // extern "C"
