// Robot-masked voxel-projection occupancy fusion (sm_100a).
//
// Replaces vp/mapping.py:266-354 (_fuse_voxels), vp/mapping.py:357-380
// (_masked_pixels) and the occupancy threshold of vp/mapping.py:113-114.
//
// Parity: log_odds / observed are bitwise equal to the reference.  Every
// floating-point operation is an explicit round-to-nearest intrinsic
// (__dmul_rn / __dadd_rn / __ddiv_rn) in the reference's left-to-right order,
// so no FMA can be contracted regardless of compiler flags.
//
// Layout: one thread per voxel, a warp covers 32 consecutive z of one (x, y)
// line aligned to a 32-voxel word of the packed occupancy mask, so log_odds /
// observed accesses are coalesced and the occupancy word is rebuilt with one
// ballot.  Voxels outside the robot's bounding box skip the sphere test;
// voxels whose projection misses the image touch no memory at all.
#include <climits>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "vpb_common.cuh"

namespace vpb {

struct FusionArgs {
  double *log_odds;
  uint8_t *observed;
  uint32_t *occ_bits;  // may be null
  int64_t gy, gz, words_z;
  int64_t lo0, lo1, lo2, n0, n1, n2;
  int64_t wz_begin, wz_count;  // z-words covering the box
  double origin0, origin1, origin2, voxel;
  double r[9], t[3];
  double fx, fy, cx, cy, d_min, d_max;
  int64_t width, height;
  const double *depth;
  const uint8_t *pixel_masked;
  const float *pixf;  // optional (vpb_update_occupancy): usable return depth in fp32, NaN if not usable
  double tau, l_hit, l_miss, l_min, l_max, l_thr;
  int n_mask;
  double aabb_lo[3], aabb_hi[3];
  // fp32 prefilter constants
  float of0, of1, of2, oabs, azmax, voxf, rf[9], tf[3], tabs, fxf, fyf, cxh, cyh, ku, kv, au, av, wf, hf;
  int usable;  // pixel_masked carries bit1 = usable return (vpb_update_occupancy)
  const int *bbox;  // optional bounding rectangle of usable pixels (chunk early-out)
  float tauf;
  float inv_fx, inv_fy, inv_vox;  // reciprocals for the (margin-padded) frustum footprint
  float bb_lo[3], bb_hi[3];
  // frustum culling (fp32, conservative): camera centre and camera->world
  // rotation, voxel-index box of the mask spheres (empty if none)
  float camc[3], c2w[9];
  int mask_i_lo[3], mask_i_hi[3];
  vpb_journal journal;  // undo records of the modified words (journal.idx == null: off)
  double mc[VPB_MAX_MASK_SPHERES * 3];
  double mr2[VPB_MAX_MASK_SPHERES];
  // fp32 mask-sphere classification: centre, and squared radii below which a
  // voxel centre is certainly inside / above which certainly outside (the
  // reference's strict fp64 test decides only the thin shell in between)
  float mcf[VPB_MAX_MASK_SPHERES * 3];
  float mr2_in[VPB_MAX_MASK_SPHERES], mr2_out[VPB_MAX_MASK_SPHERES];
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// Exact fp64 restatement of one voxel's update (vp/mapping.py:300-354), the
// reference's operations in its order.  Returns true if the voxel is
// touched (observed becomes 1); *newval receives its new log-odds (the caller
// writes both).  Kept out of line so the fp32 prefilter loop stays small.
__device__ __noinline__ bool exact_voxel(const FusionArgs &A, int64_t x, int64_t y, int64_t z, int64_t g,
                                         double *newval) {
  const double px = dadd(A.origin0, dmul(dadd((double)x, 0.5), A.voxel));
  const double py = dadd(A.origin1, dmul(dadd((double)y, 0.5), A.voxel));
  const double pz = dadd(A.origin2, dmul(dadd((double)z, 0.5), A.voxel));
  // Robot mask (vp/mapping.py:310-325), exact strict-< test.
  if (A.n_mask > 0 && px >= A.aabb_lo[0] && px <= A.aabb_hi[0] && py >= A.aabb_lo[1] && py <= A.aabb_hi[1] &&
      pz >= A.aabb_lo[2] && pz <= A.aabb_hi[2]) {
    for (int s = 0; s < A.n_mask; ++s) {
      const double dx = dsub(px, A.mc[3 * s + 0]);
      const double dy = dsub(py, A.mc[3 * s + 1]);
      const double dz = dsub(pz, A.mc[3 * s + 2]);
      const double d2 = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
      if (d2 < A.mr2[s]) {
        const double old = A.log_odds[g];
        *newval = old > 0.0 ? 0.0 : old;
        return true;
      }
    }
  }
  // Camera transform (vp/mapping.py:327-329): ((r0 px + r1 py) + r2 pz) + t
  const double qx = dadd(dadd(dadd(dmul(A.r[0], px), dmul(A.r[1], py)), dmul(A.r[2], pz)), A.t[0]);
  const double qy = dadd(dadd(dadd(dmul(A.r[3], px), dmul(A.r[4], py)), dmul(A.r[5], pz)), A.t[1]);
  const double qz = dadd(dadd(dadd(dmul(A.r[6], px), dmul(A.r[7], py)), dmul(A.r[8], pz)), A.t[2]);
  if (!(qz > 0.0)) return false;
  // u = fx * qx / qz + cx ; nearest pixel floor(u + 0.5) (:332-335)
  const double u = dadd(__ddiv_rn(dmul(A.fx, qx), qz), A.cx);
  const double v = dadd(__ddiv_rn(dmul(A.fy, qy), qz), A.cy);
  const double uf = floor(dadd(u, 0.5));
  const double vf = floor(dadd(v, 0.5));
  if (!(uf >= 0.0 && uf < (double)A.width && vf >= 0.0 && vf < (double)A.height)) return false;
  const int64_t pix = (int64_t)vf * A.width + (int64_t)uf;
  const double measured = __ldg(A.depth + pix);
  if (!(measured >= A.d_min && measured <= A.d_max) || (__ldg(A.pixel_masked + pix) & 1)) return false;
  int cls = 0;
  if (fabs(dsub(qz, measured)) <= A.tau) cls = 1;       // hit
  else if (qz < dsub(measured, A.tau)) cls = 2;          // miss
  if (!cls) return false;                                // occluded
  double value = dadd(A.log_odds[g], cls == 1 ? A.l_hit : A.l_miss);
  if (value < A.l_min) value = A.l_min;
  else if (value > A.l_max) value = A.l_max;
  *newval = value;
  return true;
}

// The voxels the reference can touch in one update are (a) those inside the
// pyramid from the camera centre through the rectangle of usable pixels, out
// to the farthest usable return + tau, and (b) those inside a mask sphere.
// Per CTA: the voxel-index box of (a) from the apex and the 4 far corners,
// and of (b) from the mask AABB.  Per (x, y) line of that footprint: the
// z-interval of (a), solved analytically from the 6 linear constraints
// (in front of / before the far plane / inside the 4 side planes, each
// a + b z >= 0 in camera space), widened by 2 pixels and 2 voxels, united
// with the mask interval.  Only those voxels run the per-voxel prefilter
// below, which makes the exact decision (the culling is conservative: it may
// include voxels the reference skips, never the reverse).
struct Interval {
  int lo, hi;  // inclusive, empty if lo > hi
};

__device__ __forceinline__ void clip_lin(float a, float b, float &zlo, float &zhi) {
  // keep z with a + b z >= 0
  // (__fdividef: <= 2 ulp, next to the intervals' 2-voxel widening)
  if (b > 0.0f) zlo = fmaxf(zlo, __fdividef(-a, b));
  else if (b < 0.0f) zhi = fminf(zhi, __fdividef(-a, b));
  else if (a < 0.0f) zhi = -1e30f;
}

struct Frustum {
  int ok;                // usable pixels exist
  float ulo, uhi, vlo, vhi, dfar;
  int xlo, xhi, ylo, yhi;  // footprint lines (box-clipped voxel indices)
};

__device__ void frustum_setup(const FusionArgs &A, Frustum &F) {
  int u0 = 0, u1 = -1, v0 = 0, v1 = -1;
  float dmax = 0.0f;
  if (A.bbox) {  // zero-identity max encoding (masked_pixels_kernel)
    u0 = (int)A.width - __ldcg(A.bbox + 0);
    u1 = __ldcg(A.bbox + 1) - 1;
    v0 = (int)A.height - __ldcg(A.bbox + 2);
    v1 = __ldcg(A.bbox + 3) - 1;
    dmax = __int_as_float(__ldcg(A.bbox + 4));
  }
  float lo[3] = {1e30f, 1e30f, 1e30f}, hi[3] = {-1e30f, -1e30f, -1e30f};
  F.ok = A.bbox == nullptr || u1 >= u0;
  if (F.ok) {
    // pixel index floor(u + 1/2) in [u0, u1] <=> u in [u0 - 1/2, u1 + 1/2);
    // 2 pixels and 2 voxels of margin
    F.ulo = (float)u0 - 2.5f;
    F.uhi = (float)u1 + 2.5f;
    F.vlo = (float)v0 - 2.5f;
    F.vhi = (float)v1 + 2.5f;
    F.dfar = A.bbox ? dmax + A.tauf + 2.0f * A.voxf : 3.0e30f;
    if (!A.bbox) {  // no rectangle (vpb_fuse_voxels): the whole image, any depth
      F.ulo = -2.5f;
      F.uhi = (float)A.width + 1.5f;
      F.vlo = -2.5f;
      F.vhi = (float)A.height + 1.5f;
    }
    if (A.bbox) {
      for (int k = 0; k < 3; ++k) lo[k] = hi[k] = A.camc[k];
      for (int c = 0; c < 4; ++c) {
        const float u = c & 1 ? F.uhi : F.ulo, v = c & 2 ? F.vhi : F.vlo;
        const float dc[3] = {(u - (float)A.cx) * A.inv_fx * F.dfar, (v - (float)A.cy) * A.inv_fy * F.dfar, F.dfar};
        for (int k = 0; k < 3; ++k) {
          const float w = A.camc[k] + A.c2w[3 * k + 0] * dc[0] + A.c2w[3 * k + 1] * dc[1] + A.c2w[3 * k + 2] * dc[2];
          lo[k] = fminf(lo[k], w);
          hi[k] = fmaxf(hi[k], w);
        }
      }
    } else {
      for (int k = 0; k < 3; ++k) {
        lo[k] = -3.0e30f;
        hi[k] = 3.0e30f;
      }
    }
  }
  // voxel-index footprint: frustum box U mask box, clipped to the update box
  int ilo[2], ihi[2];
  const float org[2] = {A.of0, A.of1};
  const int64_t blo[2] = {A.lo0, A.lo1}, bn[2] = {A.n0, A.n1};
  for (int k = 0; k < 2; ++k) {
    int a = INT_MAX, b = INT_MIN;
    if (F.ok) {
      // (reciprocal products: a few ulp next to the 2-pixel / 2-voxel margins)
      const float fa = fmaxf(fminf((lo[k] - org[k]) * A.inv_vox - 0.5f, 2.0e9f), -2.0e9f);
      const float fb = fmaxf(fminf((hi[k] - org[k]) * A.inv_vox - 0.5f, 2.0e9f), -2.0e9f);
      a = (int)floorf(fa) - 2;
      b = (int)ceilf(fb) + 2;
    }
    if (A.n_mask > 0) {
      a = min(a, A.mask_i_lo[k]);
      b = max(b, A.mask_i_hi[k]);
    }
    ilo[k] = max(a, (int)blo[k]);
    ihi[k] = min(b, (int)(blo[k] + bn[k] - 1));
  }
  F.xlo = ilo[0], F.xhi = ihi[0], F.ylo = ilo[1], F.yhi = ihi[1];
}

// z-interval (voxel indices, box-clipped) of line (x, y) that may be touched
__device__ __forceinline__ void line_intervals(const FusionArgs &A, const Frustum &F, int64_t x, int64_t y,
                                               Interval &a, Interval &m) {
  const int zb0 = (int)A.lo2, zb1 = (int)(A.lo2 + A.n2 - 1);
  a.lo = 1, a.hi = 0;
  m.lo = 1, m.hi = 0;
  const float px = A.of0 + ((float)x + 0.5f) * A.voxf, py = A.of1 + ((float)y + 0.5f) * A.voxf;
  if (F.ok) {
    // camera coordinates along the line: q(z) = qa + z qb
    const float pz0 = A.of2 + 0.5f * A.voxf;
    float qa[3], qb[3];
    for (int k = 0; k < 3; ++k) {
      qa[k] = A.rf[3 * k + 0] * px + A.rf[3 * k + 1] * py + A.rf[3 * k + 2] * pz0 + A.tf[k];
      qb[k] = A.rf[3 * k + 2] * A.voxf;
    }
    float zlo = (float)zb0 - 2.0f, zhi = (float)zb1 + 2.0f;
    const float eps = 2e-3f;  // depth slab around the camera plane kept whole (see below)
    clip_lin(qa[2] + eps, qb[2], zlo, zhi);        // qz >= -eps
    clip_lin(F.dfar - qa[2], -qb[2], zlo, zhi);    // qz <= dfar
    float flo = zlo, fhi = zhi;
    const float fx = A.fxf, fy = A.fyf, cx = (float)A.cx, cy = (float)A.cy;
    // u >= ulo: fx qx - (ulo - cx) qz >= 0 ; u <= uhi: (uhi - cx) qz - fx qx >= 0 (for qz > 0)
    clip_lin(fx * qa[0] - (F.ulo - cx) * qa[2], fx * qb[0] - (F.ulo - cx) * qb[2], flo, fhi);
    clip_lin((F.uhi - cx) * qa[2] - fx * qa[0], (F.uhi - cx) * qb[2] - fx * qb[0], flo, fhi);
    clip_lin(fy * qa[1] - (F.vlo - cy) * qa[2], fy * qb[1] - (F.vlo - cy) * qb[2], flo, fhi);
    clip_lin((F.vhi - cy) * qa[2] - fy * qa[1], (F.vhi - cy) * qb[2] - fy * qb[1], flo, fhi);
    if (flo <= fhi) {
      a.lo = max(zb0, (int)floorf(flo) - 2);
      a.hi = min(zb1, (int)ceilf(fhi) + 2);
    }
    // Within eps of the camera plane the side-plane test loses its margin to
    // fp32 rounding: if the line passes within 2 voxels of the camera centre,
    // the voxels there with -eps <= qz <= eps are kept as well.
    const float dx = px - A.camc[0], dy = py - A.camc[1];
    if (dx * dx + dy * dy <= 4.0f * A.voxf * A.voxf + 1e-6f && qb[2] != 0.0f) {
      float nlo = (float)zb0, nhi = (float)zb1;
      clip_lin(qa[2] + eps, qb[2], nlo, nhi);
      clip_lin(eps - qa[2], -qb[2], nlo, nhi);
      if (nlo <= nhi) {
        const int l = max(zb0, (int)floorf(nlo) - 2), h = min(zb1, (int)ceilf(nhi) + 2);
        if (a.lo > a.hi) {
          a.lo = l;
          a.hi = h;
        } else {
          a.lo = min(a.lo, l);
          a.hi = max(a.hi, h);
        }
      }
    }
  }
  if (A.n_mask > 0 && x >= A.mask_i_lo[0] && x <= A.mask_i_hi[0] && y >= A.mask_i_lo[1] && y <= A.mask_i_hi[1]) {
    m.lo = max(zb0, A.mask_i_lo[2]);
    m.hi = min(zb1, A.mask_i_hi[2]);
  }
}

// Voxels the fp32 prefilter cannot decide take the exact fp64 path.  They are
// a few per cent of the footprint but scattered: run in place, almost every
// 32-voxel word would carry one and drag its whole warp through the fp64
// path.  Instead each warp queues them (x, y, z in shared memory) and runs
// them 32 at a time, one per lane; a queued voxel's word was journaled when it
// was queued, and its occupancy bit is set or cleared atomically.
constexpr int kFuseQueue = 64;  // per warp: a word adds <= 32 entries, a flush takes 32

__device__ __forceinline__ void flush_exact(const FusionArgs &A, int4 *q, int &qn, int lane, bool all) {
  while (qn >= 32 || (all && qn > 0)) {
    const int take = qn < 32 ? qn : 32;
    const int base = qn - take;
    bool touched = false;
    double newval = 0.0;
    int64_t g = 0, x = 0, y = 0, z = 0;
    if (lane < take) {
      const int4 e = q[base + lane];
      x = e.x, y = e.y, z = e.z;
      g = (x * A.gy + y) * A.gz + z;
      touched = exact_voxel(A, x, y, z, g, &newval);
      if (touched) {
        A.log_odds[g] = newval;
        A.observed[g] = 1;
        if (A.occ_bits != nullptr) {
          uint32_t *ow = A.occ_bits + (x * A.gy + y) * A.words_z + (z >> 5);
          const uint32_t bit = 1u << (z & 31);
          if (newval >= A.l_thr) atomicOr(ow, bit);
          else atomicAnd(ow, ~bit);
        }
      }
    }
    qn = base;
    __syncwarp();
  }
}

// Persistent: each warp takes (x, y) lines of the footprint; per line the
// 32-voxel words overlapping its intervals run the per-voxel prefilter.
#ifdef VPB_FUSE_MINB
#define VPB_FUSE_BOUNDS __launch_bounds__(256, VPB_FUSE_MINB)
#else
#define VPB_FUSE_BOUNDS __launch_bounds__(256)
#endif
__global__ void VPB_FUSE_BOUNDS fuse_kernel(const __grid_constant__ FusionArgs A) {
  __shared__ Frustum Fs;
  __shared__ int4 queue[8][kFuseQueue];
  pdl_release();
  pdl_wait();  // the pixel codes and the usable rectangle come from masked_pixels_kernel
  if (threadIdx.x == 0) frustum_setup(A, Fs);
  __syncthreads();
  const Frustum F = Fs;
  const int lane = threadIdx.x & 31;
  const int nx = F.xhi - F.xlo + 1, ny = F.yhi - F.ylo + 1;
  if (nx <= 0 || ny <= 0) return;
  const int64_t lines = (int64_t)nx * ny;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  int4 *q = queue[threadIdx.x >> 5];
  int qn = 0;  // warp-uniform queue length
  // Rounds of blockDim lines per CTA, interleaved over the CTAs (line
  // r0 + blockIdx + t * gridDim for thread t): every thread solves one line's
  // z-intervals (the analytic frustum clip, SIMT-parallel instead of 32 lanes
  // repeating it), the non-empty lines are compacted in thread order, then
  // the warps take them round robin.
  __shared__ int s_line[256];
  __shared__ int4 s_iv[256];
  __shared__ int s_wcnt[8];
  const int warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  (void)warps;
  for (int64_t r0 = 0; r0 < lines; r0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t myli = r0 + blockIdx.x + (int64_t)threadIdx.x * gridDim.x;
    Interval mia{1, 0}, mim{1, 0};
    if (myli < lines) line_intervals(A, F, F.xlo + myli / ny, F.ylo + myli % ny, mia, mim);
    const bool nonempty = mia.lo <= mia.hi || mim.lo <= mim.hi;
    const unsigned bal = __ballot_sync(kFull, nonempty);
    if (lane == 0) s_wcnt[warp] = __popc(bal);
    __syncthreads();
    int base = 0, total = 0;
    for (int w = 0; w < nwarp; ++w) {
      base += w < warp ? s_wcnt[w] : 0;
      total += s_wcnt[w];
    }
    if (nonempty) {
      const int pos = base + __popc(bal & ((1u << lane) - 1u));
      s_line[pos] = (int)myli;
      s_iv[pos] = make_int4(mia.lo, mia.hi, mim.lo, mim.hi);
    }
    __syncthreads();
  for (int le = warp; le < total; le += nwarp) {
    const int64_t li = s_line[le];
    const int4 iv = s_iv[le];
    const int64_t x = F.xlo + li / ny, y = F.ylo + li % ny;
    Interval ia{iv.x, iv.y}, im{iv.z, iv.w};
    // ---- line constants of the conservative fp32 prefilter ----
    // Decides, with explicit error bounds, the voxels whose reference result
    // is certainly "skip" (behind the camera, outside the image, or landing
    // on a pixel without a usable return).  Everything else -- robot-mask
    // candidates, pixel-boundary ambiguities, voxels that fuse -- takes the
    // exact fp64 path, so the result is bitwise the reference's.
    const float axf = ((float)x + 0.5f) * A.voxf, ayf = ((float)y + 0.5f) * A.voxf;
    const float pxf = A.of0 + axf, pyf = A.of1 + ayf;
    const float qx0 = fmaf(A.rf[0], pxf, fmaf(A.rf[1], pyf, A.tf[0]));
    const float qy0 = fmaf(A.rf[3], pxf, fmaf(A.rf[4], pyf, A.tf[1]));
    const float qz0 = fmaf(A.rf[6], pxf, fmaf(A.rf[7], pyf, A.tf[2]));
    // |q_f - q| <= dq: each centre coordinate is off by <= 2e-7 (|origin| +
    // |(i + 1/2) voxel|), rotation entries are <= 1 and the three FMAs add
    // <= 2e-7 of the row magnitude: 4e-7 in total, taken with a 2.5x margin.
    const float dq = 1e-6f * (A.oabs + fabsf(axf) + fabsf(ayf) + A.azmax + A.tabs) + 1e-12f;
    const bool line_mask = A.n_mask > 0 && pxf >= A.bb_lo[0] && pxf <= A.bb_hi[0] && pyf >= A.bb_lo[1] &&
                           pyf <= A.bb_hi[1];
    const int64_t gline = (x * A.gy + y) * A.gz;
    // words overlapping the union of the two intervals (hull when they overlap)
    const int zlo = ia.lo <= ia.hi ? (im.lo <= im.hi ? min(ia.lo, im.lo) : ia.lo) : im.lo;
    const int zhi = ia.lo <= ia.hi ? (im.lo <= im.hi ? max(ia.hi, im.hi) : ia.hi) : im.hi;
    const bool gap = ia.lo <= ia.hi && im.lo <= im.hi && (ia.hi < im.lo - 32 || im.hi < ia.lo - 32);
    for (int64_t wz = zlo >> 5; wz <= (zhi >> 5); ++wz) {
      if (gap) {  // two separate intervals: skip the words between them
        const int w0 = (int)wz * 32, w1 = w0 + 31;
        const bool in_a = !(w1 < ia.lo || w0 > ia.hi), in_m = !(w1 < im.lo || w0 > im.hi);
        if (!in_a && !in_m) continue;
      }
      const int64_t z = wz * 32 + lane;
      const bool in_box = (z >= A.lo2) && (z < A.lo2 + A.n2);
      const int64_t g = gline + z;
      // the old log-odds, loaded before the classification needs it (one
      // coalesced 256 B read per word, overlapping the pixel load instead of
      // following it)
      const double old = in_box ? A.log_odds[g] : 0.0;
      bool exact = false;
      int fast = 0;  // 1 = certain hit, 2 = certain miss (fp32 classification)
      if (in_box) {
        const float pzf = A.of2 + ((float)z + 0.5f) * A.voxf;
        int mcls = 0;  // robot mask (vp/mapping.py:310-325): 0 outside all, 1 certainly inside one, 2 unsure
        if (line_mask && pzf >= A.bb_lo[2] && pzf <= A.bb_hi[2]) {
          for (int sm = 0; sm < A.n_mask; ++sm) {
            const float dx = pxf - A.mcf[3 * sm + 0], dy = pyf - A.mcf[3 * sm + 1], dz = pzf - A.mcf[3 * sm + 2];
            const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            if (d2 <= A.mr2_in[sm]) {
              mcls = 1;
              break;
            }
            if (d2 < A.mr2_out[sm]) mcls = 2;
          }
        }
        if (mcls == 1) {
          fast = 3;  // masked: new value min(old, 0), observed
        } else if (mcls == 2) {
          exact = true;  // within fp32 error of a sphere surface
        } else {
          const float qzf = fmaf(A.rf[8], pzf, qz0);
          if (qzf < -dq) {
            // qz <= 0 for sure: the reference skips this voxel
          } else if (qzf <= 2.0f * dq + 1e-30f) {
            exact = true;
          } else {
            const float qxf = fmaf(A.rf[2], pzf, qx0);
            const float qyf = fmaf(A.rf[5], pzf, qy0);
            const float iz = __fdividef(1.0f, qzf);  // <= 2 ulp, inside the margins below
            const float ue = fmaf(A.fxf * qxf, iz, A.cxh);  // u + 1/2
            const float ve = fmaf(A.fyf * qyf, iz, A.cyh);
            // |d u / d q| <= fx (|qx| + qz) / (qz (qz - dq)) <= 8 fx (|qx_f| + qz_f + dq) / qz_f^2
            // for qz_f > 2 dq; 10 fx taken.  Relative fp32 error of the
            // projection itself <= 4 ulp: 1e-6 |u| + 1e-6 |c| + 4e-5.
            const float iz2 = iz * iz;
            const float du = A.ku * dq * (fabsf(qxf) + qzf + dq) * iz2 + 1e-6f * fabsf(ue) + A.au;
            const float dv = A.kv * dq * (fabsf(qyf) + qzf + dq) * iz2 + 1e-6f * fabsf(ve) + A.av;
            if (!(ue < -du || ue >= A.wf + du || ve < -dv || ve >= A.hf + dv)) {
              const float fu = floorf(ue), fv = floorf(ve);
              if ((ue - fu <= du) || (fu + 1.0f - ue <= du) || (ve - fv <= dv) || (fv + 1.0f - ve <= dv) ||
                  fu < 0.0f || fu >= A.wf || fv < 0.0f || fv >= A.hf) {
                exact = true;  // pixel index not certain
              } else {
                const int pix = (int)fv * (int)A.width + (int)fu;
                bool usable;
                float mf;
                if (A.pixf) {  // one 4-byte load: usable <=> not NaN
                  mf = __ldg(A.pixf + pix);
                  usable = mf == mf;
                } else if (A.usable) {
                  usable = __ldg(A.pixel_masked + pix) == 2;
                  mf = usable ? (float)__ldg(A.depth + pix) : 0.0f;
                } else {
                  const double m = __ldg(A.depth + pix);
                  usable = (__ldg(A.pixel_masked + pix) & 1) == 0 && m >= A.d_min && m <= A.d_max;
                  mf = (float)m;
                }
                if (usable) {
                  // classification |qz - D| <= tau (hit) / qz < D - tau (miss) /
                  // occluded, decided in fp32 when clear of both boundaries
                  const float dd = qzf - mf;
                  const float e = dq + 2e-7f * (fabsf(mf) + A.tauf) + 1e-6f;
                  if (fabsf(dd) <= A.tauf - e) fast = 1;
                  else if (dd < -A.tauf - e) fast = 2;
                  else if (!(dd > A.tauf + e)) exact = true;  // near a class boundary
                  // else: certainly occluded -> skip
                }
              }
            }
            // else: certainly outside the image -> skip
          }
        }
      }
      bool touched = false;
      double newval = 0.0;
      if (fast == 3) {
        newval = old > 0.0 ? 0.0 : old;
        touched = true;
      } else if (fast) {
        // certain hit / miss: the reference's fp64 update, bit for bit
        double value = dadd(old, fast == 1 ? A.l_hit : A.l_miss);
        if (value < A.l_min) value = A.l_min;
        else if (value > A.l_max) value = A.l_max;
        newval = value;
        touched = true;
      }
      const unsigned touched_mask = __ballot_sync(kFull, touched);
      const unsigned exact_mask = __ballot_sync(kFull, exact);
      if ((touched_mask | exact_mask) == 0u) continue;
      uint32_t *ow = A.occ_bits != nullptr ? A.occ_bits + (x * A.gy + y) * A.words_z + wz : nullptr;
      if (A.journal.idx != nullptr) {
        // undo record of this word before its first write (snapshot journal):
        // the old log-odds / observed of all 32 z and the old occupancy word
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(A.journal.count, 1ull);
        slot = __shfl_sync(kFull, slot, 0);
        if (slot < A.journal.capacity) {
          const bool inz = z < A.gz;
          A.journal.lo[slot * 32 + lane] = inz ? (in_box ? old : A.log_odds[g]) : 0.0;
          A.journal.ob[slot * 32 + lane] = inz ? A.observed[g] : 0;
          if (lane == 0) {
            A.journal.idx[slot] = (x * A.gy + y) * A.words_z + wz;  // word index of the grid
            A.journal.occ[slot] = ow ? *ow : 0u;
          }
        } else if (lane == 0) {
          atomicOr(A.journal.overflow, 1u);  // (the host sizes the journal so this cannot happen)
        }
        __syncwarp();
      }
      if (touched) {
        A.log_odds[g] = newval;
        A.observed[g] = 1;
      }
      if (ow != nullptr && touched_mask != 0u) {
        const unsigned occ_mask = __ballot_sync(kFull, touched && newval >= A.l_thr);
        if (lane == 0) *ow = (*ow & ~touched_mask) | (occ_mask & touched_mask);
      }
      if (exact_mask != 0u) {
        __syncwarp();  // (the word's plain occupancy update above precedes the queued voxels' atomics)
        if (exact) q[qn + __popc(exact_mask & ((1u << lane) - 1u))] = make_int4((int)x, (int)y, (int)z, 0);
        qn += __popc(exact_mask);
        __syncwarp();
        flush_exact(A, q, qn, lane, false);
      }
    }
  }
    __syncthreads();  // the round's line list is reused by the next round
  }
  __syncwarp();
  flush_exact(A, q, qn, lane, true);
}

struct MaskPixArgs {
  const double *depth;
  uint8_t *out;
  float *out_f;  // optional: (float)depth where usable, NaN elsewhere (the fusion's one-load pixel test)
  int64_t width, height;
  double fx, fy, cx, cy, d_min, d_max;
  double r[9], t[3];
  int n_mask;
  int encode_usable;  // out = 1 masked, 2 usable return, 0 otherwise
  // optional: the usable pixels' rectangle and farthest return, reduced by
  // atomicMax into bbox as [W - umin, umax + 1, H - vmin, vmax + 1, dmax bits]
  // (zero = empty, so a zeroed slot is the identity); bbox_next is the other
  // slot of the pair, consumed by the previous call's fusion: zeroed here for
  // the next call (no ticket, no last-CTA pass, no memset)
  unsigned *bbox;
  unsigned *bbox_next;
  // journal segment bookkeeping (vpb_journal.starts / seg / reset), before fusion's first record
  unsigned long long *j_count;
  int64_t *j_starts;
  int j_seg, j_reset;
  double pad;
  double mc[VPB_MAX_MASK_SPHERES * 3];
  double mr[VPB_MAX_MASK_SPHERES];
};

// vp/mapping.py:357-380, one thread per pixel.
__global__ void __launch_bounds__(256) masked_pixels_kernel(const __grid_constant__ MaskPixArgs A) {
  pdl_release();
  pdl_wait();
  if (A.j_count != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    if (A.j_reset) *A.j_count = 0ull;
    if (A.j_starts != nullptr) A.j_starts[A.j_seg] = (int64_t)*A.j_count;
  }
  const int64_t idx0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool px = idx0 < A.width * A.height;  // (threads past the image join the CTA reduction)
  const int64_t idx = px ? idx0 : 0;
  const int64_t vv = idx / A.width, uu = idx - vv * A.width;
  const double d = px ? A.depth[idx] : -1.0;
  uint8_t inside = 0;
  const bool valid = d >= A.d_min && d <= A.d_max;
  if (A.n_mask > 0 && valid) {
    const double z = d;
    const double xx = dmul(__ddiv_rn(dsub((double)uu, A.cx), A.fx), z);
    const double yy = dmul(__ddiv_rn(dsub((double)vv, A.cy), A.fy), z);
    double p[3];
#pragma unroll
    for (int j = 0; j < 3; ++j)
      p[j] = dadd(dadd(dadd(dmul(xx, A.r[3 * j + 0]), dmul(yy, A.r[3 * j + 1])), dmul(z, A.r[3 * j + 2])), A.t[j]);
    for (int s = 0; s < A.n_mask; ++s) {
      const double dx = dsub(p[0], A.mc[3 * s + 0]);
      const double dy = dsub(p[1], A.mc[3 * s + 1]);
      const double dz = dsub(p[2], A.mc[3 * s + 2]);
      const double r = dadd(A.mr[s], A.pad);
      if (dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)) < dmul(r, r)) inside = 1;
    }
  }
  const uint8_t code = px ? (inside ? 1 : (valid ? 2 : 0)) : 0;
  if (px) A.out[idx] = A.encode_usable ? code : inside;
  if (px && A.out_f) A.out_f[idx] = code == 2 ? (float)d : __int_as_float(0x7fc00000);
  if (A.bbox) {
    __shared__ unsigned red[5][8];
    if (blockIdx.x == 0 && threadIdx.x < 5) A.bbox_next[threadIdx.x] = 0u;
    const bool use = code == 2;
    // (float bits of a non-negative depth rounded up order like the depths)
    const unsigned r0 = __reduce_max_sync(kFull, use ? (unsigned)(A.width - uu) : 0u);
    const unsigned r1 = __reduce_max_sync(kFull, use ? (unsigned)(uu + 1) : 0u);
    const unsigned r2 = __reduce_max_sync(kFull, use ? (unsigned)(A.height - vv) : 0u);
    const unsigned r3 = __reduce_max_sync(kFull, use ? (unsigned)(vv + 1) : 0u);
    const unsigned r4 = __reduce_max_sync(kFull, use ? __float_as_uint(fmaxf(__double2float_ru(d), 0.0f)) : 0u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
      red[0][warp] = r0;
      red[1][warp] = r1;
      red[2][warp] = r2;
      red[3][warp] = r3;
      red[4][warp] = r4;
    }
    __syncthreads();
    if (threadIdx.x < 5) {
      unsigned m = 0u;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = max(m, red[threadIdx.x][w]);
      if (m != 0u) atomicMax(A.bbox + threadIdx.x, m);
    }
  }
}

// occupancy bits from log_odds: one warp per 32-voxel word.
__global__ void __launch_bounds__(256) occ_bits_kernel(const double *__restrict__ log_odds,
                                                       uint32_t *__restrict__ bits, int64_t lines,
                                                       int64_t gz, int64_t words_z, double thr) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= lines * words_z) return;
  const int64_t line = w / words_z, wz = w - line * words_z;
  const int64_t z = wz * 32 + lane;
  const bool occ = z < gz && log_odds[line * gz + z] >= thr;
  const unsigned m = __ballot_sync(kFull, occ);
  if (lane == 0) bits[w] = m;
}

// One warp per undo record: the word's 32 old log-odds / observed and its
// old occupancy word back into the clone.
__global__ void __launch_bounds__(256) journal_restore_kernel(double *__restrict__ log_odds,
                                                              uint8_t *__restrict__ observed,
                                                              uint32_t *__restrict__ occ_bits, int64_t gz,
                                                              int64_t words_z, const int64_t *__restrict__ idx,
                                                              const double *__restrict__ jlo,
                                                              const uint8_t *__restrict__ job,
                                                              const uint32_t *__restrict__ jocc, int64_t first,
                                                              int64_t last) {
  const int lane = threadIdx.x & 31;
  const int64_t r = first + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= last) return;
  const int64_t w = idx[r];
  const int64_t line = w / words_z, wz = w - line * words_z;
  const int64_t z = wz * 32 + lane;
  if (z < gz) {
    log_odds[line * gz + z] = jlo[r * 32 + lane];
    observed[line * gz + z] = job[r * 32 + lane];
  }
  if (lane == 0 && occ_bits) occ_bits[w] = jocc[r];
}

}  // namespace vpb

using namespace vpb;

static int fill_mask(const double *centers, const double *radii, int64_t n_mask, double *mc,
                     double *aabb_lo, double *aabb_hi) {
  VPB_REQUIRE(n_mask >= 0 && n_mask <= VPB_MAX_MASK_SPHERES, "mask sphere count %lld outside [0, %d]",
              (long long)n_mask, VPB_MAX_MASK_SPHERES);
  VPB_REQUIRE(n_mask == 0 || (centers && radii), "mask centers/radii are null");
  for (int k = 0; k < 3; ++k) {
    aabb_lo[k] = 1e300;
    aabb_hi[k] = -1e300;
  }
  for (int64_t s = 0; s < n_mask; ++s) {
    for (int k = 0; k < 3; ++k) {
      mc[3 * s + k] = centers[3 * s + k];
      const double r = fabs(radii[s]);
      aabb_lo[k] = fmin(aabb_lo[k], centers[3 * s + k] - r - 1e-9 - 1e-12 * fabs(centers[3 * s + k]));
      aabb_hi[k] = fmax(aabb_hi[k], centers[3 * s + k] + r + 1e-9 + 1e-12 * fabs(centers[3 * s + k]));
    }
  }
  return VPB_OK;
}

extern "C" {

int64_t vpb_occ_words(const int64_t dims[3]) { return dims[0] * dims[1] * ceil_div(dims[2], 32); }

int vpb_occ_bits_from_log_odds(const vpb_grid *grid, double thr, void *stream) {
  VPB_REQUIRE(grid && grid->log_odds && grid->occ_bits, "grid/log_odds/occ_bits is null");
  const int64_t lines = grid->dims[0] * grid->dims[1];
  const int64_t wz = ceil_div(grid->dims[2], 32);
  const int64_t warps = lines * wz;
  if (warps == 0) return VPB_OK;
  occ_bits_kernel<<<(unsigned)ceil_div(warps, 8), 256, 0, as_stream(stream)>>>(
      grid->log_odds, grid->occ_bits, lines, grid->dims[2], wz, thr);
  return check_launch("occ_bits_kernel");
}

static int masked_pixels_impl(const double *depth, const vpb_camera *cam, const double *centers,
                              const double *radii, int64_t n_mask, double pad, uint8_t *out, int encode,
                              int *bbox, void *stream, const vpb_journal *journal = nullptr,
                              float *pixf = nullptr, int *bbox_pair = nullptr) {
  VPB_REQUIRE(depth && cam && out, "null argument to vpb_masked_pixels");
  MaskPixArgs A;
  memset(&A, 0, sizeof(A));
  double lo[3], hi[3];
  int rc = fill_mask(centers, radii, n_mask, A.mc, lo, hi);
  if (rc) return rc;
  for (int64_t s = 0; s < n_mask; ++s) A.mr[s] = radii[s];
  A.depth = depth;
  A.out = out;
  A.out_f = pixf;
  A.width = cam->width;
  A.height = cam->height;
  A.fx = cam->fx; A.fy = cam->fy; A.cx = cam->cx; A.cy = cam->cy;
  A.d_min = cam->d_min; A.d_max = cam->d_max;
  memcpy(A.r, cam->pose_r, sizeof(A.r));
  memcpy(A.t, cam->pose_t, sizeof(A.t));
  A.n_mask = (int)n_mask;
  A.encode_usable = encode;
  if (bbox) {  // slot pair [8 ints][8 ints]: this call's and the next call's
    A.bbox = reinterpret_cast<unsigned *>(bbox);
    A.bbox_next = reinterpret_cast<unsigned *>(bbox == bbox_pair ? bbox_pair + 8 : bbox_pair);
  }
  A.pad = pad;
  if (journal != nullptr && journal->count != nullptr) {
    A.j_count = journal->count;
    A.j_starts = journal->starts;
    A.j_seg = journal->seg;
    A.j_reset = journal->reset;
  }
  const int64_t npx = cam->width * cam->height;
  if (npx == 0) {
    if (A.j_count != nullptr) {  // (no launch to carry the journal bookkeeping)
      cudaStream_t st = as_stream(stream);
      if (A.j_reset) VPB_CUDA(cudaMemsetAsync(A.j_count, 0, sizeof(unsigned long long), st));
      if (A.j_starts) VPB_CUDA(cudaMemcpyAsync(A.j_starts + A.j_seg, A.j_count, 8, cudaMemcpyDeviceToDevice, st));
    }
    return VPB_OK;
  }
  VPB_CUDA(launch_pdl(masked_pixels_kernel, dim3((unsigned)ceil_div(npx, 256)), dim3(256), 0, as_stream(stream), A));
  return check_launch("masked_pixels_kernel");
}

static int fuse_impl(const vpb_grid *grid, const int64_t lo[3], const int64_t n[3], const vpb_camera *cam,
                     const double *depth, const uint8_t *pixel_masked, const double *centers,
                     const double *radii, int64_t n_mask, const vpb_map_params *p, int usable, const int *bbox,
                     void *stream, const vpb_journal *journal = nullptr, const float *pixf = nullptr) {
  VPB_REQUIRE(grid && grid->log_odds && grid->observed && cam && depth && pixel_masked && p,
              "null argument to vpb_fuse_voxels");
  for (int k = 0; k < 3; ++k)
    VPB_REQUIRE(lo[k] >= 0 && n[k] >= 1 && lo[k] + n[k] <= grid->dims[k], "box outside grid on axis %d", k);
  FusionArgs A;
  memset(&A, 0, sizeof(A));
  int rc = fill_mask(centers, radii, n_mask, A.mc, A.aabb_lo, A.aabb_hi);
  if (rc) return rc;
  for (int64_t s = 0; s < n_mask; ++s) A.mr2[s] = radii[s] * radii[s];
  {
    // fp32 sphere test bounds.  A voxel centre's fp32 coordinates are off by
    // <= 2^-23 (|origin| + |(i + 1/2) voxel|) per rounding (two roundings), a
    // centre's by 2^-24 |c|; dx = p_f - c_f adds one more rounding.  delta
    // bounds |dx_f - dx| per axis (4x margin); the squared distance then
    // carries <= 2 sqrt(3) delta d + 3 delta^2 from the coordinates and
    // < 1e-6 d^2 from its own three roundings.
    double cmax = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double o = k == 0 ? grid->origin[0] : (k == 1 ? grid->origin[1] : grid->origin[2]);
      const double far = fabs(o) + (double)(grid->dims[k] + 1) * grid->voxel;
      cmax = fmax(cmax, far);
    }
    for (int64_t s = 0; s < n_mask; ++s)
      for (int k = 0; k < 3; ++k) cmax = fmax(cmax, fabs(centers[3 * s + k]) + fabs(radii[s]));
    const double delta = 4.0 * (3.0 * 1.2e-7 * cmax) + 1e-12;
    for (int64_t s = 0; s < n_mask; ++s) {
      for (int k = 0; k < 3; ++k) A.mcf[3 * s + k] = (float)centers[3 * s + k];
      const double r = fabs(radii[s]);
      const double err = 2.0 * 1.7320508075688772 * delta * (r + 4.0 * delta) + 3.0 * delta * delta;
      const double in2 = r * r * (1.0 - 4e-6) - err;
      const double out2 = r * r * (1.0 + 4e-6) + err;
      // rounded towards the safe side
      A.mr2_in[s] = in2 > 0.0 ? nextafterf((float)in2, 0.0f) : -1.0f;
      A.mr2_out[s] = nextafterf((float)out2, 3.0e38f);
    }
  }
  A.log_odds = grid->log_odds;
  A.observed = grid->observed;
  A.occ_bits = grid->occ_bits;
  if (journal) {
    VPB_REQUIRE(journal->idx && journal->lo && journal->ob && journal->occ && journal->count && journal->overflow,
                "incomplete snapshot journal");
    A.journal = *journal;
  }
  A.gy = grid->dims[1];
  A.gz = grid->dims[2];
  A.words_z = ceil_div(grid->dims[2], 32);
  A.lo0 = lo[0]; A.lo1 = lo[1]; A.lo2 = lo[2];
  A.n0 = n[0]; A.n1 = n[1]; A.n2 = n[2];
  A.wz_begin = lo[2] / 32;
  A.wz_count = (lo[2] + n[2] - 1) / 32 - A.wz_begin + 1;
  A.origin0 = grid->origin[0]; A.origin1 = grid->origin[1]; A.origin2 = grid->origin[2];
  A.voxel = grid->voxel;
  memcpy(A.r, cam->w2c_r, sizeof(A.r));
  memcpy(A.t, cam->w2c_t, sizeof(A.t));
  A.fx = cam->fx; A.fy = cam->fy; A.cx = cam->cx; A.cy = cam->cy;
  A.d_min = cam->d_min; A.d_max = cam->d_max;
  A.width = cam->width; A.height = cam->height;
  A.depth = depth;
  A.pixel_masked = pixel_masked;
  A.pixf = pixf;
  A.tau = p->tau; A.l_hit = p->l_hit; A.l_miss = p->l_miss;
  A.l_min = p->l_min; A.l_max = p->l_max; A.l_thr = p->l_occ_threshold;
  A.n_mask = (int)n_mask;
  A.usable = usable;
  A.bbox = bbox;
  A.tauf = (float)A.tau;
  A.of0 = (float)A.origin0;
  A.of1 = (float)A.origin1;
  A.of2 = (float)A.origin2;
  A.voxf = (float)A.voxel;
  A.oabs = fabsf(A.of0) + fabsf(A.of1) + fabsf(A.of2);
  A.tabs = 0.0f;
  for (int k = 0; k < 9; ++k) A.rf[k] = (float)A.r[k];
  for (int k = 0; k < 3; ++k) {
    A.tf[k] = (float)A.t[k];
    A.tabs += fabsf(A.tf[k]);
    // fp32 AABB of the mask spheres with a generous pad (fp32 centre error)
    const double pad = 1e-4 + 1e-5 * (fabs(A.aabb_lo[k]) + fabs(A.aabb_hi[k]));
    A.bb_lo[k] = (float)(A.aabb_lo[k] - pad);
    A.bb_hi[k] = (float)(A.aabb_hi[k] + pad);
  }
  A.fxf = (float)A.fx;
  A.fyf = (float)A.fy;
  A.inv_fx = (float)(1.0 / A.fx);
  A.inv_fy = (float)(1.0 / A.fy);
  A.inv_vox = (float)(1.0 / A.voxel);
  A.cxh = (float)(A.cx + 0.5);
  A.cyh = (float)(A.cy + 0.5);
  A.ku = 10.0f * fabsf(A.fxf);
  A.kv = 10.0f * fabsf(A.fyf);
  A.au = 1e-6f * fabsf(A.cxh) + 4e-5f;
  A.av = 1e-6f * fabsf(A.cyh) + 4e-5f;
  A.azmax = fmaxf(fabsf((float)((double)lo[2] + 0.5) * A.voxf), fabsf((float)((double)(lo[2] + n[2]) + 0.5) * A.voxf));
  A.wf = (float)A.width;
  A.hf = (float)A.height;
  // the fp32 prefilter assumes an orthonormal world->camera rotation and a
  // scene within float range; anything else simply takes the exact path
  for (int k = 0; k < 3; ++k) A.camc[k] = (float)cam->pose_t[k];
  for (int k = 0; k < 9; ++k) A.c2w[k] = (float)cam->pose_r[k];
  for (int k = 0; k < 3; ++k) {
    // voxel indices whose fp32 centre can fall in the padded mask box (+1)
    const double o = k == 0 ? A.origin0 : (k == 1 ? A.origin1 : A.origin2);
    if (n_mask > 0) {
      A.mask_i_lo[k] = (int)fmax(-2.0e9, floor(((double)A.bb_lo[k] - o) / A.voxel - 0.5) - 1.0);
      A.mask_i_hi[k] = (int)fmin(2.0e9, ceil(((double)A.bb_hi[k] - o) / A.voxel - 0.5) + 1.0);
    } else {
      A.mask_i_lo[k] = 1;
      A.mask_i_hi[k] = 0;
    }
  }
  // persistent: warps stride over the footprint lines each CTA derives; one
  // resident wave (every CTA pays the frustum setup once)
  static int occ = 0;
  if (occ == 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fuse_kernel, 256, 0) != cudaSuccess) {
    cudaGetLastError();
    occ = 4;
  }
  const int64_t max_ctas = ceil_div(A.n0 * A.n1, 8);
  static const int per_sm_env = getenv("VPB_FUSE_CTAS_PER_SM") ? atoi(getenv("VPB_FUSE_CTAS_PER_SM")) : 0;
  const int64_t slots = (int64_t)sm_count() * (per_sm_env > 0 ? per_sm_env : (occ > 0 ? occ : 4));
  const int64_t ctas = max_ctas < slots ? max_ctas : slots;
  VPB_CUDA(launch_pdl(fuse_kernel, dim3((unsigned)ctas), dim3(256), 0, as_stream(stream), A));
  return check_launch("fuse_kernel");
}

int vpb_masked_pixels(const double *depth, const vpb_camera *cam, const double *centers, const double *radii,
                      int64_t n_mask, double pad, uint8_t *out, void *stream) {
  return masked_pixels_impl(depth, cam, centers, radii, n_mask, pad, out, 0, nullptr, stream);
}

int vpb_fuse_voxels(const vpb_grid *grid, const int64_t lo[3], const int64_t n[3], const vpb_camera *cam,
                    const double *depth, const uint8_t *pixel_masked, const double *centers, const double *radii,
                    int64_t n_mask, const vpb_map_params *p, void *stream) {
  return fuse_impl(grid, lo, n, cam, depth, pixel_masked, centers, radii, n_mask, p, 0, nullptr, stream);
}

// pixel scratch: [class byte per pixel | 2 rectangle slots of 8 ints (+ spare) | fp32 depth per pixel]
// (the slot size term is the old per-CTA partial area, kept so the layout of
// the scratch the callers allocate does not move)
static size_t pixf_offset(int64_t npx) {
  return align_up(align_up((size_t)npx, 16) + 32 + 32 * (size_t)ceil_div(npx > 0 ? npx : 1, 256) + 64, 16);
}

int64_t vpb_pixel_scratch_bytes(int64_t width, int64_t height) {
  const int64_t npx = width * height;
  return (int64_t)pixf_offset(npx) + 4 * npx;
}

int vpb_update_occupancy(const vpb_grid *grid, const int64_t lo[3], const int64_t n[3], const vpb_camera *cam,
                         const double *depth, const double *centers, const double *radii, int64_t n_mask,
                         double mask_pad, const vpb_map_params *params, uint8_t *pixel_scratch, void *stream) {
  return vpb_update_occupancy_journaled(grid, lo, n, cam, depth, centers, radii, n_mask, mask_pad, params,
                                        pixel_scratch, nullptr, stream);
}

int vpb_update_occupancy_journaled(const vpb_grid *grid, const int64_t lo[3], const int64_t n[3],
                                   const vpb_camera *cam, const double *depth, const double *centers,
                                   const double *radii, int64_t n_mask, double mask_pad,
                                   const vpb_map_params *params, uint8_t *pixel_scratch, const vpb_journal *journal,
                                   void *stream) {
  VPB_REQUIRE(pixel_scratch, "pixel scratch is null");
  // pixel classes in one byte: 1 = return on the robot body, 2 = usable
  // return; followed by the bounding rectangle of the usable pixels
  const int64_t npx = cam->width * cam->height;
  int *pair = reinterpret_cast<int *>(pixel_scratch + align_up((size_t)npx, 16));
  // the slot of this call alternates per scratch buffer (stream-ordered calls)
  unsigned parity;
  {
    static std::mutex mu;
    static std::unordered_map<const void *, unsigned> calls;
    std::lock_guard<std::mutex> lk(mu);
    parity = calls[pair]++ & 1u;
  }
  int *bbox = pair + 8 * parity;
  float *pixf = reinterpret_cast<float *>(pixel_scratch + pixf_offset(npx));
  int rc = masked_pixels_impl(depth, cam, centers, radii, n_mask, mask_pad, pixel_scratch, 1, bbox, stream, journal,
                              pixf, pair);
  if (rc) return rc;
  return fuse_impl(grid, lo, n, cam, depth, pixel_scratch, centers, radii, n_mask, params, 1, bbox, stream, journal,
                   pixf);
}

int vpb_journal_restore(const vpb_grid *grid, const vpb_journal *j, int64_t first, int64_t last, void *stream) {
  VPB_REQUIRE(grid && grid->log_odds && grid->observed && j && j->idx && j->lo && j->ob && j->occ,
              "null argument to vpb_journal_restore");
  VPB_REQUIRE(first >= 0 && first <= last && (uint64_t)last <= j->capacity, "journal range outside capacity");
  if (last == first) return VPB_OK;
  journal_restore_kernel<<<(unsigned)ceil_div(last - first, 8), 256, 0, as_stream(stream)>>>(
      grid->log_odds, grid->observed, grid->occ_bits, grid->dims[2], ceil_div(grid->dims[2], 32), j->idx, j->lo,
      j->ob, j->occ, first, last);
  return check_launch("journal_restore_kernel");
}

}  // extern "C"
