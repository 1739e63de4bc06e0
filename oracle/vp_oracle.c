/*
 * vp_oracle.c -- CPU restatement of the ParaMaP reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * (paper_2512_22575_b200) never links or calls it.
 *
 * Every function restates one reference function op for op, in float64, in
 * the reference's evaluation order, compiled with -ffp-contract=off so no FMA
 * is formed (numba emits none for these kernels).
 * Parity of this restatement is pinned against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py -> tests/golden/*.npz).
 *
 * Reference = /root/reference/pkg/src/voxplan (abbreviated vp/).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define VPO_INF_SENTINEL 1e20 /* vp/mapping.py:32 */

int vpo_version(void) { return 1; }

/* Worker count for the parallel loops (the reference's prange loops run on
 * numba's OpenMP pool, vp/parallel.py:13-65).  Static contiguous chunking,
 * every item writes only its own outputs, so results are independent of the
 * worker count -- the same contract as the reference. */
static int g_threads = 0;

int vpo_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

void vpo_set_threads(int n) { g_threads = n > 0 ? n : 0; }

int vpo_get_threads(void) { return g_threads > 0 ? g_threads : vpo_max_threads(); }

typedef void (*vpo_body_fn)(void *ctx, int64_t begin, int64_t end);
typedef struct {
  vpo_body_fn fn;
  void *ctx;
  int64_t begin, end;
} vpo_chunk;

static void *vpo_chunk_main(void *arg) {
  vpo_chunk *c = (vpo_chunk *)arg;
  if (c->begin < c->end) c->fn(c->ctx, c->begin, c->end);
  return NULL;
}

static void vpo_parallel_for(int64_t count, vpo_body_fn fn, void *ctx) {
  int t = vpo_get_threads();
  if (t > 256) t = 256;
  if (count < t) t = (int)(count > 0 ? count : 1);
  if (t <= 1) {
    if (count > 0) fn(ctx, 0, count);
    return;
  }
  pthread_t tid[256];
  vpo_chunk ch[256];
  for (int i = 0; i < t; ++i) {
    ch[i].fn = fn;
    ch[i].ctx = ctx;
    ch[i].begin = count * i / t;
    ch[i].end = count * (i + 1) / t;
  }
  for (int i = 1; i < t; ++i) pthread_create(&tid[i], NULL, vpo_chunk_main, &ch[i]);
  vpo_chunk_main(&ch[0]);
  for (int i = 1; i < t; ++i) pthread_join(tid[i], NULL);
}

/* ------------------------------------------------------------------------ */
/* Masked pixels: vp/mapping.py:357-380 (_masked_pixels).                    */
/* pose_r/pose_t = camera->world pose (cam.pose), row-major 3x3.             */
/* ------------------------------------------------------------------------ */
void vpo_masked_pixels(const double *depth, int64_t height, int64_t width,
                       double fx, double fy, double cx, double cy,
                       double d_min, double d_max, const double *pose_r,
                       const double *pose_t, const double *centers,
                       const double *radii, int64_t n_mask, double pad,
                       uint8_t *out) {
  for (int64_t v = 0; v < height; ++v) {
    for (int64_t u = 0; u < width; ++u) {
      int64_t idx = v * width + u;
      double d = depth[idx];
      out[idx] = 0;
      if (n_mask == 0) continue;
      if (!(d >= d_min && d <= d_max)) continue;
      double z = d;
      /* x = (us - cx) / fx * z  (left to right) */
      double x = ((double)u - cx) / fx * z;
      double y = ((double)v - cy) / fy * z;
      /* pts = [x,y,z] @ R^T + t : p_j = x*R[j,0] + y*R[j,1] + z*R[j,2] + t_j */
      double p[3];
      for (int j = 0; j < 3; ++j)
        p[j] = ((x * pose_r[3 * j + 0] + y * pose_r[3 * j + 1]) +
                z * pose_r[3 * j + 2]) + pose_t[j];
      int inside = 0;
      for (int64_t s = 0; s < n_mask; ++s) {
        double dx = p[0] - centers[3 * s + 0];
        double dy = p[1] - centers[3 * s + 1];
        double dz = p[2] - centers[3 * s + 2];
        double r = radii[s] + pad;
        if ((dx * dx + dy * dy) + dz * dz < r * r) inside = 1;
      }
      out[idx] = (uint8_t)inside;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Voxel-projection fusion: vp/mapping.py:266-354 (_fuse_voxels).            */
/* Serial, like the reference (njit without parallel=True).                  */
/* Grid arrays are full (gx, gy, gz) C-order; box = lo + [0, n).             */
/* ------------------------------------------------------------------------ */
void vpo_fuse_voxels(double *log_odds, uint8_t *observed, int64_t gx,
                     int64_t gy, int64_t gz, int64_t lo0, int64_t lo1,
                     int64_t lo2, int64_t n0, int64_t n1, int64_t n2,
                     const double *origin, double voxel, const double *cam_r,
                     const double *cam_t, double fx, double fy, double cx,
                     double cy, int64_t width, int64_t height, double d_min,
                     double d_max, const double *depth,
                     const uint8_t *pixel_masked, const double *mask_centers,
                     const double *mask_radii, int64_t n_mask, double tau,
                     double l_hit, double l_miss, double l_min, double l_max) {
  (void)gx;
  int64_t total = n0 * n1 * n2;
  for (int64_t flat = 0; flat < total; ++flat) {
    int64_t i0 = flat / (n1 * n2);
    int64_t rem = flat % (n1 * n2);
    int64_t i1 = rem / n2;
    int64_t i2 = rem % n2;
    int64_t x = lo0 + i0, y = lo1 + i1, z = lo2 + i2;
    int64_t g = (x * gy + y) * gz + z;
    double px = origin[0] + ((double)x + 0.5) * voxel;
    double py = origin[1] + ((double)y + 0.5) * voxel;
    double pz = origin[2] + ((double)z + 0.5) * voxel;
    int masked = 0;
    for (int64_t s = 0; s < n_mask; ++s) {
      double dx = px - mask_centers[3 * s + 0];
      double dy = py - mask_centers[3 * s + 1];
      double dz = pz - mask_centers[3 * s + 2];
      if ((dx * dx + dy * dy) + dz * dz < mask_radii[s] * mask_radii[s]) {
        masked = 1;
        break;
      }
    }
    if (masked) {
      if (log_odds[g] > 0.0) log_odds[g] = 0.0;
      observed[g] = 1;
      continue;
    }
    double qx = ((cam_r[0] * px + cam_r[1] * py) + cam_r[2] * pz) + cam_t[0];
    double qy = ((cam_r[3] * px + cam_r[4] * py) + cam_r[5] * pz) + cam_t[1];
    double qz = ((cam_r[6] * px + cam_r[7] * py) + cam_r[8] * pz) + cam_t[2];
    if (qz <= 0.0) continue;
    double u = fx * qx / qz + cx;
    double v = fy * qy / qz + cy;
    int64_t ui = (int64_t)floor(u + 0.5);
    int64_t vi = (int64_t)floor(v + 0.5);
    if (ui < 0 || ui >= width || vi < 0 || vi >= height) continue;
    double measured = depth[vi * width + ui];
    if (!(measured >= d_min && measured <= d_max)) continue;
    if (pixel_masked[vi * width + ui]) continue;
    double value;
    if (fabs(qz - measured) <= tau)
      value = log_odds[g] + l_hit;
    else if (qz < measured - tau)
      value = log_odds[g] + l_miss;
    else
      continue;
    if (value < l_min)
      value = l_min;
    else if (value > l_max)
      value = l_max;
    log_odds[g] = value;
    observed[g] = 1;
  }
}

/* ------------------------------------------------------------------------ */
/* FH lower envelope: vp/mapping.py:458-483 (_fh_envelope).                  */
/* ------------------------------------------------------------------------ */
static void fh_envelope(const double *f, double *d, int64_t *v, double *zz,
                        int64_t n) {
  int64_t k = 0;
  v[0] = 0;
  zz[0] = -VPO_INF_SENTINEL;
  zz[1] = VPO_INF_SENTINEL;
  for (int64_t q = 1; q < n; ++q) {
    double fq = f[q] + (double)(q * q);
    double s;
    for (;;) {
      int64_t p = v[k];
      s = (fq - (f[p] + (double)(p * p))) / (2.0 * (double)(q - p));
      if (s <= zz[k])
        k -= 1;
      else
        break;
    }
    k += 1;
    v[k] = q;
    zz[k] = s;
    zz[k + 1] = VPO_INF_SENTINEL;
  }
  k = 0;
  for (int64_t q = 0; q < n; ++q) {
    while (zz[k + 1] < (double)q) k += 1;
    int64_t p = v[k];
    d[q] = (double)((q - p) * (q - p)) + f[p];
  }
}

/* fh_1d (vp/mapping.py:486-499): line with +inf as "no source". */
void vpo_fh_1d(const double *line, double *out, int64_t n) {
  double *f = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int64_t *v = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  double *zz = (double *)malloc(sizeof(double) * (size_t)(n + 1));
  for (int64_t i = 0; i < n; ++i) f[i] = isfinite(line[i]) ? line[i] : VPO_INF_SENTINEL;
  if (n > 0) fh_envelope(f, out, v, zz, n);
  for (int64_t i = 0; i < n; ++i)
    if (out[i] >= VPO_INF_SENTINEL / 2.0) out[i] = INFINITY;
  free(f);
  free(v);
  free(zz);
}

/* One axis pass over a C-contiguous (nx, ny, nz) array, in place:
 * vp/mapping.py:502-550 (_edt_pass_x/_y/_z), parallel over lines. */
typedef struct {
  double *vals;
  int64_t ny, nz, len, stride;
  int axis;
} edt_pass_ctx;

static void edt_pass_body(void *vctx, int64_t begin, int64_t end) {
  edt_pass_ctx *c = (edt_pass_ctx *)vctx;
  int64_t len = c->len, stride = c->stride;
  double *f = (double *)malloc(sizeof(double) * (size_t)len);
  double *d = (double *)malloc(sizeof(double) * (size_t)len);
  int64_t *v = (int64_t *)malloc(sizeof(int64_t) * (size_t)len);
  double *zz = (double *)malloc(sizeof(double) * (size_t)(len + 1));
  for (int64_t idx = begin; idx < end; ++idx) {
    int64_t base;
    if (c->axis == 0) {
      base = idx; /* (y, z) = divmod(idx, nz): base = y*nz + z = idx */
    } else if (c->axis == 1) {
      int64_t x = idx / c->nz, z = idx % c->nz;
      base = x * c->ny * c->nz + z;
    } else {
      base = idx * c->nz;
    }
    for (int64_t i = 0; i < len; ++i) f[i] = c->vals[base + i * stride];
    fh_envelope(f, d, v, zz, len);
    for (int64_t i = 0; i < len; ++i) c->vals[base + i * stride] = d[i];
  }
  free(f);
  free(d);
  free(v);
  free(zz);
}

static void edt_pass(double *vals, int64_t nx, int64_t ny, int64_t nz, int axis) {
  edt_pass_ctx c;
  c.vals = vals;
  c.ny = ny;
  c.nz = nz;
  c.axis = axis;
  c.len = axis == 0 ? nx : (axis == 1 ? ny : nz);
  c.stride = axis == 0 ? ny * nz : (axis == 1 ? nz : 1);
  int64_t lines = axis == 0 ? ny * nz : (axis == 1 ? nx * nz : nx * ny);
  vpo_parallel_for(lines, edt_pass_body, &c);
}

/* edt_3d body (vp/mapping.py:586-613): occupancy threshold on log_odds over
 * the box, init 0 / 1e20, passes in `order` (0=x,1=y,2=z), >= 5e19 -> inf.
 * out: (n0, n1, n2) float64. */
void vpo_edt3d(const double *log_odds, int64_t gx, int64_t gy, int64_t gz,
               int64_t lo0, int64_t lo1, int64_t lo2, int64_t n0, int64_t n1,
               int64_t n2, double threshold, const int32_t *order,
               double *out) {
  (void)gx;
  for (int64_t a = 0; a < n0; ++a)
    for (int64_t b = 0; b < n1; ++b)
      for (int64_t c = 0; c < n2; ++c) {
        double lv = log_odds[((lo0 + a) * gy + (lo1 + b)) * gz + (lo2 + c)];
        out[(a * n1 + b) * n2 + c] = (lv >= threshold) ? 0.0 : VPO_INF_SENTINEL;
      }
  for (int i = 0; i < 3; ++i) edt_pass(out, n0, n1, n2, order[i]);
  int64_t total = n0 * n1 * n2;
  for (int64_t i = 0; i < total; ++i)
    if (out[i] >= VPO_INF_SENTINEL / 2.0) out[i] = INFINITY;
}

/* ------------------------------------------------------------------------ */
/* Distance query: vp/mapping.py:616-685 (_query_metric).                    */
/* ------------------------------------------------------------------------ */
double vpo_query_metric(const double *sq, int64_t n0, int64_t n1, int64_t n2,
                        int64_t lo0, int64_t lo1, int64_t lo2, double origin0,
                        double origin1, double origin2, double voxel,
                        double outside_default, double px, double py,
                        double pz) {
  double g0 = (px - origin0) / voxel - (double)lo0;
  double g1 = (py - origin1) / voxel - (double)lo1;
  double g2 = (pz - origin2) / voxel - (double)lo2;
  if (g0 < 0.0 || g0 >= (double)n0 || g1 < 0.0 || g1 >= (double)n1 ||
      g2 < 0.0 || g2 >= (double)n2)
    return outside_default;
  int64_t i0 = (int64_t)g0, i1 = (int64_t)g1, i2 = (int64_t)g2;
  double cell = sq[(i0 * n1 + i1) * n2 + i2];
  if (cell == 0.0) return 0.0;
  if (cell == INFINITY) return INFINITY;
  double c0 = g0 - 0.5, c1 = g1 - 0.5, c2 = g2 - 0.5;
  if (c0 < 0.0) c0 = 0.0; else if (c0 > (double)n0 - 1.0) c0 = (double)n0 - 1.0;
  if (c1 < 0.0) c1 = 0.0; else if (c1 > (double)n1 - 1.0) c1 = (double)n1 - 1.0;
  if (c2 < 0.0) c2 = 0.0; else if (c2 > (double)n2 - 1.0) c2 = (double)n2 - 1.0;
  int64_t a0 = (int64_t)c0, a1 = (int64_t)c1, a2 = (int64_t)c2;
  int64_t b0 = a0 + 1 < n0 ? a0 + 1 : a0;
  int64_t b1 = a1 + 1 < n1 ? a1 + 1 : a1;
  int64_t b2 = a2 + 1 < n2 ? a2 + 1 : a2;
  double f0 = c0 - (double)a0, f1 = c1 - (double)a1, f2 = c2 - (double)a2;
#define SQ(i, j, k) sq[((i)*n1 + (j)) * n2 + (k)]
  double v000 = SQ(a0, a1, a2), v001 = SQ(a0, a1, b2);
  double v010 = SQ(a0, b1, a2), v011 = SQ(a0, b1, b2);
  double v100 = SQ(b0, a1, a2), v101 = SQ(b0, a1, b2);
  double v110 = SQ(b0, b1, a2), v111 = SQ(b0, b1, b2);
#undef SQ
  double c00 = v000 * (1.0 - f0) + v100 * f0;
  double c01 = v001 * (1.0 - f0) + v101 * f0;
  double c10 = v010 * (1.0 - f0) + v110 * f0;
  double c11 = v011 * (1.0 - f0) + v111 * f0;
  double c0v = c00 * (1.0 - f1) + c10 * f1;
  double c1v = c01 * (1.0 - f1) + c11 * f1;
  double value = c0v * (1.0 - f2) + c1v * f2;
  return voxel * sqrt(value);
}

/* ------------------------------------------------------------------------ */
/* Rollout evaluator: vp/batch.py:25-336.                                    */
/* ------------------------------------------------------------------------ */
#define VPO_SMALL_ANGLE 1e-6      /* vp/batch.py:20 */
#define VPO_PI_MARGIN 1e-6        /* vp/batch.py:21 */
#define VPO_V_INV_SERIES_ANGLE 0.1 /* vp/batch.py:22 */

/* _fk_frames, vp/batch.py:25-66. frames_r (n+1)*9, frames_t (n+1)*3. */
static void fk_frames(const double *base_r, const double *base_t,
                      const double *off_r, const double *off_t,
                      const double *axes, const double *q, int64_t n,
                      double *fr, double *ft) {
  for (int a = 0; a < 3; ++a) {
    ft[a] = base_t[a];
    for (int b = 0; b < 3; ++b) fr[3 * a + b] = base_r[3 * a + b];
  }
  for (int64_t i = 0; i < n; ++i) {
    double ux = axes[3 * i + 0], uy = axes[3 * i + 1], uz = axes[3 * i + 2];
    double c = cos(q[i]), s = sin(q[i]);
    double ic = 1.0 - c;
    double j00 = c + ux * ux * ic;
    double j01 = ux * uy * ic - uz * s;
    double j02 = ux * uz * ic + uy * s;
    double j10 = uy * ux * ic + uz * s;
    double j11 = c + uy * uy * ic;
    double j12 = uy * uz * ic - ux * s;
    double j20 = uz * ux * ic - uy * s;
    double j21 = uz * uy * ic + ux * s;
    double j22 = c + uz * uz * ic;
    const double *o = off_r + 9 * i;
    const double *pr = fr + 9 * i;
    double *nr = fr + 9 * (i + 1);
    for (int a = 0; a < 3; ++a) {
      double pr0 = pr[3 * a + 0], pr1 = pr[3 * a + 1], pr2 = pr[3 * a + 2];
      double m0 = pr0 * o[0] + pr1 * o[3] + pr2 * o[6];
      double m1 = pr0 * o[1] + pr1 * o[4] + pr2 * o[7];
      double m2 = pr0 * o[2] + pr1 * o[5] + pr2 * o[8];
      nr[3 * a + 0] = m0 * j00 + m1 * j10 + m2 * j20;
      nr[3 * a + 1] = m0 * j01 + m1 * j11 + m2 * j21;
      nr[3 * a + 2] = m0 * j02 + m1 * j12 + m2 * j22;
      ft[3 * (i + 1) + a] = ft[3 * i + a] + pr0 * off_t[3 * i + 0] +
                            pr1 * off_t[3 * i + 1] + pr2 * off_t[3 * i + 2];
    }
  }
}

/* _pose_error, vp/batch.py:69-137. Returns 0 on the log singularity. */
static int pose_error(const double *er, const double *et, const double *gr,
                      const double *gt, double *xi) {
#define G(a, b) gr[3 * (a) + (b)]
#define E(a, b) er[3 * (a) + (b)]
  double d00 = G(0, 0) * E(0, 0) + G(1, 0) * E(1, 0) + G(2, 0) * E(2, 0);
  double d01 = G(0, 0) * E(0, 1) + G(1, 0) * E(1, 1) + G(2, 0) * E(2, 1);
  double d02 = G(0, 0) * E(0, 2) + G(1, 0) * E(1, 2) + G(2, 0) * E(2, 2);
  double d10 = G(0, 1) * E(0, 0) + G(1, 1) * E(1, 0) + G(2, 1) * E(2, 0);
  double d11 = G(0, 1) * E(0, 1) + G(1, 1) * E(1, 1) + G(2, 1) * E(2, 1);
  double d12 = G(0, 1) * E(0, 2) + G(1, 1) * E(1, 2) + G(2, 1) * E(2, 2);
  double d20 = G(0, 2) * E(0, 0) + G(1, 2) * E(1, 0) + G(2, 2) * E(2, 0);
  double d21 = G(0, 2) * E(0, 1) + G(1, 2) * E(1, 1) + G(2, 2) * E(2, 1);
  double d22 = G(0, 2) * E(0, 2) + G(1, 2) * E(1, 2) + G(2, 2) * E(2, 2);
  double rx = et[0] - gt[0], ry = et[1] - gt[1], rz = et[2] - gt[2];
  double tx = G(0, 0) * rx + G(1, 0) * ry + G(2, 0) * rz;
  double ty = G(0, 1) * rx + G(1, 1) * ry + G(2, 1) * rz;
  double tz = G(0, 2) * rx + G(1, 2) * ry + G(2, 2) * rz;
#undef G
#undef E
  double c = 0.5 * (d00 + d11 + d22 - 1.0);
  if (c > 1.0) c = 1.0; else if (c < -1.0) c = -1.0;
  double theta = acos(c);
  if (theta >= M_PI - VPO_PI_MARGIN) return 0;
  double sx = 0.5 * (d21 - d12), sy = 0.5 * (d02 - d20), sz = 0.5 * (d10 - d01);
  double scale = theta < VPO_SMALL_ANGLE ? 1.0 + theta * theta / 6.0
                                         : theta / sin(theta);
  double wx = scale * sx, wy = scale * sy, wz = scale * sz;
  double e;
  if (theta < VPO_V_INV_SERIES_ANGLE) {
    double t2 = theta * theta;
    e = 1.0 / 12.0 + t2 / 720.0 + t2 * t2 / 30240.0;
  } else {
    e = (1.0 - 0.5 * theta * sin(theta) / (1.0 - cos(theta))) / (theta * theta);
  }
  double wxx = wx * wx, wyy = wy * wy, wzz = wz * wz;
  double m00 = 1.0 + e * (-wzz - wyy);
  double m01 = 0.5 * wz + e * wx * wy;
  double m02 = -0.5 * wy + e * wx * wz;
  double m10 = -0.5 * wz + e * wx * wy;
  double m11 = 1.0 + e * (-wxx - wzz);
  double m12 = 0.5 * wx + e * wy * wz;
  double m20 = 0.5 * wy + e * wx * wz;
  double m21 = -0.5 * wx + e * wy * wz;
  double m22 = 1.0 + e * (-wxx - wyy);
  xi[0] = m00 * tx + m01 * ty + m02 * tz;
  xi[1] = m10 * tx + m11 * ty + m12 * tz;
  xi[2] = m20 * tx + m21 * ty + m22 * tz;
  xi[3] = wx;
  xi[4] = wy;
  xi[5] = wz;
  return 1;
}

/* _quad_form, vp/batch.py:140-148. */
static double quad_form(const double *w, const double *xi) {
  double total = 0.0;
  for (int a = 0; a < 6; ++a) {
    double row = 0.0;
    for (int b = 0; b < 6; ++b) row += w[6 * a + b] * xi[b];
    total += xi[a] * row;
  }
  return 0.5 * total;
}

/* _bound_violation, vp/batch.py:151-158. */
static double bound_violation(double x, double lo, double hi) {
  double v = 0.0;
  if (x > hi) v = x - hi;
  else if (x < lo) v = x - lo;
  return v;
}

/* Flat argument block mirroring evaluate_batch's 49 positional arguments
 * (vp/batch.py:162-212).  Layout must match oracle/__init__.py. */
typedef struct {
  int64_t n;          /* dof */
  int64_t n_spheres;
  int64_t n_pairs;
  double dt;
  const double *q0, *qd0;
  const double *base_r, *base_t, *off_r, *off_t, *axes;
  const int64_t *sph_link;
  const double *sph_loc, *sph_r;
  const int64_t *pairs;
  const double *goal_r, *goal_t, *pose_weight, *terminal_weight;
  const double *pos_lo, *pos_hi, *vel_lo, *vel_hi, *acc_lo, *acc_hi;
  double w_env, w_self, w_q, w_qd, w_qdd, w_s, w_ns, d_act;
  const double *q_ref;
  const double *field_sq;
  int64_t field_n0, field_n1, field_n2;
  int64_t field_lo0, field_lo1, field_lo2;
  double field_origin0, field_origin1, field_origin2, field_voxel, field_outside;
} vpo_rollout_args;

/* evaluate_batch per-sample body, vp/batch.py:161-336 (prange m). */
typedef struct {
  const vpo_rollout_args *A;
  const double *controls;
  int64_t horizon;
  double *costs, *terms;
  uint8_t *flags;
  double *traj_q, *traj_qd, *sphere_pos;
} rollout_ctx;

static void rollout_body(void *vctx, int64_t begin, int64_t end) {
  rollout_ctx *C = (rollout_ctx *)vctx;
  const vpo_rollout_args *A = C->A;
  const double *controls = C->controls;
  const int64_t horizon = C->horizon;
  double *costs = C->costs, *terms = C->terms;
  uint8_t *flags = C->flags;
  double *traj_q = C->traj_q, *traj_qd = C->traj_qd, *sphere_pos = C->sphere_pos;
  const int64_t n = A->n, ns = A->n_spheres, np_ = A->n_pairs;
  {
    double *q = (double *)malloc(sizeof(double) * (size_t)n);
    double *qd = (double *)malloc(sizeof(double) * (size_t)n);
    double *fr = (double *)malloc(sizeof(double) * (size_t)(9 * (n + 1)));
    double *ft = (double *)malloc(sizeof(double) * (size_t)(3 * (n + 1)));
    double *centers = (double *)malloc(sizeof(double) * (size_t)(3 * (ns > 0 ? ns : 1)));
    double xi[6];
    for (int64_t m = begin; m < end; ++m) {
      for (int64_t i = 0; i < n; ++i) {
        q[i] = A->q0[i];
        qd[i] = A->qd0[i];
      }
      double pose_sum = 0.0, coll_sum = 0.0, lim_sum = 0.0, smooth_sum = 0.0,
             null_sum = 0.0;
      int failed = 0;
      const double *um = controls + m * horizon * n;
      for (int64_t k = 0; k < horizon; ++k) {
        if (traj_q) {
          for (int64_t i = 0; i < n; ++i) {
            traj_q[(m * (horizon + 1) + k) * n + i] = q[i];
            traj_qd[(m * (horizon + 1) + k) * n + i] = qd[i];
          }
        }
        fk_frames(A->base_r, A->base_t, A->off_r, A->off_t, A->axes, q, n, fr, ft);
        if (!pose_error(fr + 9 * n, ft + 3 * n, A->goal_r, A->goal_t, xi)) {
          failed = 1;
          break;
        }
        pose_sum += quad_form(A->pose_weight, xi);
        for (int64_t s = 0; s < ns; ++s) {
          int64_t li = A->sph_link[s];
          const double *R = fr + 9 * li, *T = ft + 3 * li, *L = A->sph_loc + 3 * s;
          double px = R[0] * L[0] + R[1] * L[1] + R[2] * L[2] + T[0];
          double py = R[3] * L[0] + R[4] * L[1] + R[5] * L[2] + T[1];
          double pz = R[6] * L[0] + R[7] * L[1] + R[8] * L[2] + T[2];
          centers[3 * s + 0] = px;
          centers[3 * s + 1] = py;
          centers[3 * s + 2] = pz;
          if (sphere_pos) {
            double *sp = sphere_pos + ((m * horizon + k) * ns + s) * 3;
            sp[0] = px;
            sp[1] = py;
            sp[2] = pz;
          }
          double dist = vpo_query_metric(
              A->field_sq, A->field_n0, A->field_n1, A->field_n2, A->field_lo0,
              A->field_lo1, A->field_lo2, A->field_origin0, A->field_origin1,
              A->field_origin2, A->field_voxel, A->field_outside, px, py, pz);
          double gap = A->d_act - (dist - A->sph_r[s]);
          if (gap > 0.0) coll_sum += A->w_env * gap * gap;
        }
        for (int64_t p = 0; p < np_; ++p) {
          int64_t i = A->pairs[2 * p], j = A->pairs[2 * p + 1];
          double dx = centers[3 * i] - centers[3 * j];
          double dy = centers[3 * i + 1] - centers[3 * j + 1];
          double dz = centers[3 * i + 2] - centers[3 * j + 2];
          double gap = sqrt(dx * dx + dy * dy + dz * dz) - (A->sph_r[i] + A->sph_r[j]);
          if (gap < 0.0) coll_sum += A->w_self * gap * gap;
        }
        for (int64_t i = 0; i < n; ++i) {
          double u = um[k * n + i];
          double vq = bound_violation(q[i], A->pos_lo[i], A->pos_hi[i]);
          double vv = bound_violation(qd[i], A->vel_lo[i], A->vel_hi[i]);
          double va = bound_violation(u, A->acc_lo[i], A->acc_hi[i]);
          lim_sum += A->w_q * vq * vq + A->w_qd * vv * vv + A->w_qdd * va * va;
          smooth_sum += A->w_s * u * u;
          double dq = q[i] - A->q_ref[i];
          null_sum += A->w_ns * dq * dq;
        }
        for (int64_t i = 0; i < n; ++i) {
          qd[i] = qd[i] + um[k * n + i] * A->dt;
          q[i] = q[i] + qd[i] * A->dt;
        }
      }
      if (failed) {
        flags[m] = 1;
        costs[m] = INFINITY;
        continue;
      }
      if (traj_q) {
        for (int64_t i = 0; i < n; ++i) {
          traj_q[(m * (horizon + 1) + horizon) * n + i] = q[i];
          traj_qd[(m * (horizon + 1) + horizon) * n + i] = qd[i];
        }
      }
      fk_frames(A->base_r, A->base_t, A->off_r, A->off_t, A->axes, q, n, fr, ft);
      if (!pose_error(fr + 9 * n, ft + 3 * n, A->goal_r, A->goal_t, xi)) {
        flags[m] = 1;
        costs[m] = INFINITY;
        continue;
      }
      double term_sum = quad_form(A->terminal_weight, xi);
      double *t = terms + 6 * m;
      t[0] = pose_sum;
      t[1] = coll_sum;
      t[2] = lim_sum;
      t[3] = smooth_sum;
      t[4] = null_sum;
      t[5] = term_sum;
      costs[m] = pose_sum + coll_sum + lim_sum + smooth_sum + null_sum + term_sum;
      flags[m] = 0;
    }
    free(q);
    free(qd);
    free(fr);
    free(ft);
    free(centers);
  }
}

/* evaluate_batch entry: parallel over samples like the reference's prange. */
void vpo_evaluate_batch(const vpo_rollout_args *A, const double *controls,
                        int64_t n_samples, int64_t horizon, double *costs,
                        double *terms, uint8_t *flags, double *traj_q,
                        double *traj_qd, double *sphere_pos) {
  rollout_ctx C;
  C.A = A;
  C.controls = controls;
  C.horizon = horizon;
  C.costs = costs;
  C.terms = terms;
  C.flags = flags;
  C.traj_q = traj_q;
  C.traj_qd = traj_qd;
  C.sphere_pos = sphere_pos;
  vpo_parallel_for(n_samples, rollout_body, &C);
}

/* ------------------------------------------------------------------------ */
/* soft_weights (vp/planner.py:373-384) and update_controls (:387-400).     */
/* Validation lives in the Python wrapper (raises like the reference).       */
/* ------------------------------------------------------------------------ */
void vpo_soft_weights(const double *costs, int64_t m, double lam, double *w) {
  double mn = costs[0];
  for (int64_t i = 1; i < m; ++i)
    if (costs[i] < mn) mn = costs[i];
  double total = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    w[i] = exp(-(costs[i] - mn) / lam);
    total += w[i];
  }
  for (int64_t i = 0; i < m; ++i) w[i] = w[i] / total;
}

void vpo_update_controls(const double *nominal, const double *eps,
                         const double *w, int64_t m, int64_t hn, double *out) {
  for (int64_t j = 0; j < hn; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < m; ++i) acc += w[i] * eps[i * hn + j];
    out[j] = nominal[j] + acc;
  }
}
