// Batched distance-field query in fp64 (sm_100a).
// Replaces vp/mapping.py:616-710 (_query_metric / query_distance), evaluated
// op for op in float64 on the f32-stored exact squared distances.
#include "vpb_common.cuh"

namespace vpb {

struct QueryArgs {
  const float *sq;
  int64_t n0, n1, n2, lo0, lo1, lo2;
  double origin0, origin1, origin2, voxel, outside;
  const double *pts;
  double *out;
  int64_t count;
};

__global__ void __launch_bounds__(256) query_kernel(const __grid_constant__ QueryArgs A) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.count) return;
  const double px = A.pts[3 * i], py = A.pts[3 * i + 1], pz = A.pts[3 * i + 2];
  double r;
  if (A.sq == nullptr) {
    r = __longlong_as_double(0x7ff0000000000000ll);
  } else {
    const double g0 = __dsub_rn(__ddiv_rn(__dsub_rn(px, A.origin0), A.voxel), (double)A.lo0);
    const double g1 = __dsub_rn(__ddiv_rn(__dsub_rn(py, A.origin1), A.voxel), (double)A.lo1);
    const double g2 = __dsub_rn(__ddiv_rn(__dsub_rn(pz, A.origin2), A.voxel), (double)A.lo2);
    if (g0 < 0.0 || g0 >= (double)A.n0 || g1 < 0.0 || g1 >= (double)A.n1 || g2 < 0.0 || g2 >= (double)A.n2 ||
        isnan(g0) || isnan(g1) || isnan(g2)) {
      r = A.outside;
    } else {
      const int64_t i0 = (int64_t)g0, i1 = (int64_t)g1, i2 = (int64_t)g2;
      const double cell = (double)A.sq[(i0 * A.n1 + i1) * A.n2 + i2];
      if (cell == 0.0) {
        r = 0.0;
      } else if (isinf(cell)) {
        r = cell;
      } else {
        double c0 = __dsub_rn(g0, 0.5), c1 = __dsub_rn(g1, 0.5), c2 = __dsub_rn(g2, 0.5);
        const double m0 = (double)A.n0 - 1.0, m1 = (double)A.n1 - 1.0, m2 = (double)A.n2 - 1.0;
        c0 = c0 < 0.0 ? 0.0 : (c0 > m0 ? m0 : c0);
        c1 = c1 < 0.0 ? 0.0 : (c1 > m1 ? m1 : c1);
        c2 = c2 < 0.0 ? 0.0 : (c2 > m2 ? m2 : c2);
        const int64_t a0 = (int64_t)c0, a1 = (int64_t)c1, a2 = (int64_t)c2;
        const int64_t b0 = a0 + 1 < A.n0 ? a0 + 1 : a0;
        const int64_t b1 = a1 + 1 < A.n1 ? a1 + 1 : a1;
        const int64_t b2 = a2 + 1 < A.n2 ? a2 + 1 : a2;
        const double f0 = __dsub_rn(c0, (double)a0), f1 = __dsub_rn(c1, (double)a1), f2 = __dsub_rn(c2, (double)a2);
#define SQ(x, y, z) ((double)A.sq[((x) * A.n1 + (y)) * A.n2 + (z)])
        const double v000 = SQ(a0, a1, a2), v001 = SQ(a0, a1, b2), v010 = SQ(a0, b1, a2), v011 = SQ(a0, b1, b2);
        const double v100 = SQ(b0, a1, a2), v101 = SQ(b0, a1, b2), v110 = SQ(b0, b1, a2), v111 = SQ(b0, b1, b2);
#undef SQ
        const double e0 = __dsub_rn(1.0, f0), e1 = __dsub_rn(1.0, f1), e2 = __dsub_rn(1.0, f2);
        const double c00 = __dadd_rn(__dmul_rn(v000, e0), __dmul_rn(v100, f0));
        const double c01 = __dadd_rn(__dmul_rn(v001, e0), __dmul_rn(v101, f0));
        const double c10 = __dadd_rn(__dmul_rn(v010, e0), __dmul_rn(v110, f0));
        const double c11 = __dadd_rn(__dmul_rn(v011, e0), __dmul_rn(v111, f0));
        const double c0v = __dadd_rn(__dmul_rn(c00, e1), __dmul_rn(c10, f1));
        const double c1v = __dadd_rn(__dmul_rn(c01, e1), __dmul_rn(c11, f1));
        const double value = __dadd_rn(__dmul_rn(c0v, e2), __dmul_rn(c1v, f2));
        r = __dmul_rn(A.voxel, __dsqrt_rn(value));
      }
    }
  }
  A.out[i] = r;
}

}  // namespace vpb

using namespace vpb;

extern "C" int vpb_query_distance(const vpb_field *field, const double *points, int64_t count, double *out,
                                  void *stream) {
  VPB_REQUIRE(field && points && out && count >= 0, "bad arguments to vpb_query_distance");
  if (count == 0) return VPB_OK;
  QueryArgs A;
  memset(&A, 0, sizeof(A));
  A.sq = field->sq;
  A.n0 = field->n[0];
  A.n1 = field->n[1];
  A.n2 = field->n[2];
  A.lo0 = field->lo[0];
  A.lo1 = field->lo[1];
  A.lo2 = field->lo[2];
  A.origin0 = field->origin[0];
  A.origin1 = field->origin[1];
  A.origin2 = field->origin[2];
  A.voxel = field->voxel;
  A.outside = field->outside_default;
  A.pts = points;
  A.out = out;
  A.count = count;
  query_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, as_stream(stream)>>>(A);
  return check_launch("query_kernel");
}
