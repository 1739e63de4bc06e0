// Exact separable squared Euclidean distance transform (sm_100a).
//
// Replaces the body of vp/mapping.py:586-613 (edt_3d): the occupancy
// threshold, the three _edt_pass_{x,y,z} passes of the Felzenszwalb-
// Huttenlocher lower envelope (vp/mapping.py:458-550) and the inf mapping.
//
// The result is the exact squared distance, so any exact algorithm yields
// the reference's values bit for bit.  This implementation:
//   pass Z  (from the packed occupancy mask, 1 bit / voxel): nearest source
//           along z by bit scans -> u16 distance (0xFFFF = none on the line);
//   pass Y  FH lower envelope along y of f = dz^2 -> i32 (INT_MAX = none);
//   pass X  FH along x -> f32 output, +inf where no source exists.
// Lines are processed one per thread with lanes over the contiguous z axis,
// so every global access of every pass is coalesced.  FH comparisons are
// integer cross-multiplications of the parabola intersections (exact; no
// division), with only finite sources ever entering the envelope.
#include <climits>
#include <cstdlib>

#include <cuda.h>

#include "vpb_common.cuh"

namespace vpb {

constexpr uint16_t kNoSrc16 = 0xFFFFu;
constexpr int32_t kNoSrc32 = INT_MAX;

// ---------------------------------------------------------------------------
// Pass Z: bits -> u16 nearest-source distance along z.
// One warp per (x, y) line of the box; lanes walk z in chunks of 32.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t load_bits_window(const uint32_t *__restrict__ w, int64_t z0,
                                                     int64_t words_z = INT64_MAX) {
  // 32 bits of the line starting at global z0 (z0 may be unaligned); bits
  // past the line's last word read as 0.
  const int64_t wi = z0 >> 5;
  const int sh = (int)(z0 & 31);
  const uint32_t a = wi < words_z ? __ldg(w + wi) : 0u;
  if (sh == 0) return a;
  const uint32_t b = wi + 1 < words_z ? __ldg(w + wi + 1) : 0u;
  return __funnelshift_r(a, b, sh);
}

__global__ void __launch_bounds__(256) edt_pass_z_bits(const uint32_t *__restrict__ bits, int64_t gy,
                                                       int64_t words_z, int64_t lo0, int64_t lo1,
                                                       int64_t lo2, int64_t n0, int64_t n1, int64_t n2,
                                                       uint16_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t line = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (line >= n0 * n1) return;
  const int64_t i0 = line / n1, i1 = line - i0 * n1;
  const uint32_t *w = bits + ((lo0 + i0) * gy + (lo1 + i1)) * words_z;
  const int64_t nchunks = (n2 + 31) >> 5;
  // last/next source index (box-local z) carried across chunks by a
  // forward sweep (left) and a backward sweep (right).
  // Forward: for every z, nearest source at <= z.
  int64_t carry_left = -1;  // box-local index of last source before chunk
  uint16_t *o = out + line * n2;
  // We store left distances first, then fix up with right distances.
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t zb = c * 32;
    uint32_t m = load_bits_window(w, lo2 + zb);
    const int valid = (int)vmin64(32, n2 - zb);
    if (valid < 32) m &= (1u << valid) - 1u;
    // sources at positions <= lane within this chunk
    const uint32_t le = m & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
    int64_t left = le ? zb + (31 - __clz(le)) : carry_left;
    if (lane < valid) {
      const int64_t zz = zb + lane;
      o[zz] = left < 0 ? kNoSrc16 : (uint16_t)vmin64(zz - left, 0xFFFE);
    }
    if (m) carry_left = zb + (31 - __clz(m));
  }
  __syncwarp();
  int64_t carry_right = -1;
  for (int64_t c = nchunks - 1; c >= 0; --c) {
    const int64_t zb = c * 32;
    uint32_t m = load_bits_window(w, lo2 + zb);
    const int valid = (int)vmin64(32, n2 - zb);
    if (valid < 32) m &= (1u << valid) - 1u;
    const uint32_t ge = m & (0xffffffffu << lane);
    int64_t right = ge ? zb + (__ffs(ge) - 1) : carry_right;
    if (lane < valid && right >= 0) {
      const int64_t zz = zb + lane;
      const uint16_t d = (uint16_t)vmin64(right - zz, 0xFFFE);
      const uint16_t cur = o[zz];
      if (d < cur) o[zz] = d;
    }
    if (m) carry_right = zb + (__ffs(m) - 1);
  }
}

// Same pass reading the log-odds threshold directly (no packed mask).
__global__ void __launch_bounds__(256) edt_pass_z_logodds(const double *__restrict__ log_odds, int64_t gy,
                                                          int64_t gz, int64_t lo0, int64_t lo1, int64_t lo2,
                                                          int64_t n0, int64_t n1, int64_t n2, double thr,
                                                          uint16_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t line = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (line >= n0 * n1) return;
  const int64_t i0 = line / n1, i1 = line - i0 * n1;
  const double *src = log_odds + ((lo0 + i0) * gy + (lo1 + i1)) * gz + lo2;
  const int64_t nchunks = (n2 + 31) >> 5;
  uint16_t *o = out + line * n2;
  int64_t carry_left = -1;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t zb = c * 32;
    const bool occ = (zb + lane < n2) && (src[zb + lane] >= thr);
    const uint32_t m = __ballot_sync(kFull, occ);
    const uint32_t le = m & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
    int64_t left = le ? zb + (31 - __clz(le)) : carry_left;
    if (zb + lane < n2) {
      const int64_t zz = zb + lane;
      o[zz] = left < 0 ? kNoSrc16 : (uint16_t)vmin64(zz - left, 0xFFFE);
    }
    if (m) carry_left = zb + (31 - __clz(m));
  }
  __syncwarp();
  int64_t carry_right = -1;
  for (int64_t c = nchunks - 1; c >= 0; --c) {
    const int64_t zb = c * 32;
    const bool occ = (zb + lane < n2) && (src[zb + lane] >= thr);
    const uint32_t m = __ballot_sync(kFull, occ);
    const uint32_t ge = m & (0xffffffffu << lane);
    int64_t right = ge ? zb + (__ffs(ge) - 1) : carry_right;
    if (zb + lane < n2 && right >= 0) {
      const int64_t zz = zb + lane;
      const uint16_t d = (uint16_t)vmin64(right - zz, 0xFFFE);
      if (d < o[zz]) o[zz] = d;
    }
    if (m) carry_right = zb + (__ffs(m) - 1);
  }
}

// ---------------------------------------------------------------------------
// FH pass along a strided axis with lanes over z.
// TIn: uint16_t (distance, squared on load) or int32_t (squared distance).
// TOut: int32_t (intermediate) or float (final, +inf for no source).
// Acc: int32 when 3(N-1)^3 < 2^31, else int64.
// ---------------------------------------------------------------------------
template <typename TIn>
__device__ __forceinline__ int64_t load_f(const TIn *p);
template <>
__device__ __forceinline__ int64_t load_f<uint16_t>(const uint16_t *p) {
  const uint16_t d = *p;
  return d == kNoSrc16 ? -1 : (int64_t)d * (int64_t)d;
}
template <>
__device__ __forceinline__ int64_t load_f<int32_t>(const int32_t *p) {
  const int32_t v = *p;
  return v == kNoSrc32 ? -1 : (int64_t)v;
}

template <typename TOut>
__device__ __forceinline__ void store_out(TOut *p, int64_t v);
template <>
__device__ __forceinline__ void store_out<int32_t>(int32_t *p, int64_t v) {
  *p = v < 0 ? kNoSrc32 : (int32_t)v;
}
template <>
__device__ __forceinline__ void store_out<float>(float *p, int64_t v) {
  *p = v < 0 ? __int_as_float(0x7f800000) : (float)v;
}

// Lines: for line index L = (a, z) with a in [0, n_outer), z in [0, n2):
//   element p of the line lives at base(a, z) + p * stride,
//   base(a, z) = a * outer_stride + z.
// Block = 2 warps; stack of each thread in shared memory, interleaved.
template <typename TIn, typename TOut, typename Acc>
__global__ void __launch_bounds__(64) edt_pass_fh(const TIn *__restrict__ in, TOut *__restrict__ out,
                                                  int64_t n_outer, int64_t outer_stride, int64_t n2,
                                                  int64_t len, int64_t stride) {
  extern __shared__ uint16_t stack[];  // [len][64]
  const int tid = threadIdx.x;
  const int64_t zchunks = (n2 + 31) >> 5;
  const int64_t warp = (int64_t)blockIdx.x * 2 + (tid >> 5);
  if (warp >= n_outer * zchunks) return;
  const int64_t a = warp / zchunks;
  const int64_t z = (warp - a * zchunks) * 32 + (tid & 31);
  if (z >= n2) return;
  const int64_t base = a * outer_stride + z;
  const TIn *src = in + base;
  TOut *dst = out + base;
#define STK(k) stack[(int64_t)(k) * 64 + tid]

  // Forward sweep: lower envelope of the finite parabolas.
  int k = -1;           // top index
  Acc vt = 0, Ft = 0;   // top
  Acc vp = 0, Fp = 0;   // below top
  for (int64_t q = 0; q < len; ++q) {
    const int64_t f = load_f<TIn>(src + q * stride);
    if (f < 0) continue;
    const Acc qa = (Acc)q;
    const Acc Fq = (Acc)f + qa * qa;
    while (k >= 1) {
      // pop top if s(vt, q) <= s(vp, vt)
      if ((Fq - Ft) * (vt - vp) <= (Ft - Fp) * (qa - vt)) {
        --k;
        vt = vp;
        Ft = Fp;
        if (k >= 1) {
          vp = (Acc)STK(k - 1);
          Fp = (Acc)load_f<TIn>(src + (int64_t)vp * stride) + vp * vp;
        }
      } else {
        break;
      }
    }
    ++k;
    STK(k) = (uint16_t)q;
    vp = vt;
    Fp = Ft;
    vt = qa;
    Ft = Fq;
  }
  if (k < 0) {
    for (int64_t q = 0; q < len; ++q) store_out<TOut>(dst + q * stride, -1);
    return;
  }
  // Output sweep: advance through the envelope while the next parabola's
  // intersection lies strictly left of q (vp/mapping.py:478-483).
  int j = 0;
  Acc vj = (Acc)STK(0);
  Acc fj = (Acc)load_f<TIn>(src + (int64_t)vj * stride);
  Acc Fj = fj + vj * vj;
  Acc vn = 0, Fn = 0, fn = 0;
  if (k >= 1) {
    vn = (Acc)STK(1);
    fn = (Acc)load_f<TIn>(src + (int64_t)vn * stride);
    Fn = fn + vn * vn;
  }
  for (int64_t q = 0; q < len; ++q) {
    const Acc qa = (Acc)q;
    // s(vj, vn) < q  <=>  Fn - Fj < 2 q (vn - vj)
    while (j < k && (Fn - Fj) < 2 * qa * (vn - vj)) {
      ++j;
      vj = vn;
      fj = fn;
      Fj = Fn;
      if (j < k) {
        vn = (Acc)STK(j + 1);
        fn = (Acc)load_f<TIn>(src + (int64_t)vn * stride);
        Fn = fn + vn * vn;
      }
    }
    const Acc dq = qa - vj;
    store_out<TOut>(dst + q * stride, (int64_t)(dq * dq + fj));
  }
#undef STK
}

// ---------------------------------------------------------------------------
// Shared-memory FH pass.  A 32-thread CTA owns 32 lines (lanes over the
// contiguous z axis), stages them as a [len][32] u32 tile (coalesced loads,
// conflict-free column access), runs the lower-envelope sweep per lane and
// keeps its stack IN PLACE: stack entry k (packed (f << 10) | v) overwrites
// tile slot k, whose input has always been consumed already (k <= q).  The
// output sweep reads the stack and writes the line back coalesced.
// len <= 1024 and f < 2^22 (3 (len-1)^2) so an entry fits 32 bits.
// ---------------------------------------------------------------------------
constexpr uint32_t kTileInf = 0xFFFFFFFFu;

template <typename TIn>
__device__ __forceinline__ uint32_t tile_in(TIn v);
template <>
__device__ __forceinline__ uint32_t tile_in<uint16_t>(uint16_t d) {
  return d == kNoSrc16 ? kTileInf : (uint32_t)d * (uint32_t)d;
}
template <>
__device__ __forceinline__ uint32_t tile_in<int32_t>(int32_t v) {
  return v == kNoSrc32 ? kTileInf : (uint32_t)v;
}

template <typename TOut>
__device__ __forceinline__ void store_tile_out(TOut *p, uint32_t v);
template <>
__device__ __forceinline__ void store_tile_out<int32_t>(int32_t *p, uint32_t v) {
  *p = v == kTileInf ? kNoSrc32 : (int32_t)v;
}
template <>
__device__ __forceinline__ void store_tile_out<float>(float *p, uint32_t v) {
  *p = v == kTileInf ? __int_as_float(0x7f800000) : (float)v;
}

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(32) edt_pass_fh_smem(const TIn *__restrict__ in, TOut *__restrict__ out,
                                                       int64_t n_outer, int64_t outer_stride, int n2, int len,
                                                       int64_t stride) {
  extern __shared__ uint32_t tile[];  // [len][32]
  const int lane = threadIdx.x;
  // grid: (zchunks, n_outer)
  const int64_t a = blockIdx.y;
  const int z = (int)blockIdx.x * 32 + lane;
  const bool act = z < n2;
  const int64_t base = a * outer_stride + (act ? z : 0);
  const TIn *src = in + base;
  // ---- stage the 32 lines (8 independent loads in flight per thread) ----
  int q = 0;
  for (; q + 8 <= len; q += 8) {
    TIn v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = act ? src[(int64_t)(q + t) * stride] : (TIn)0;
#pragma unroll
    for (int t = 0; t < 8; ++t) tile[(q + t) * 32 + lane] = act ? tile_in<TIn>(v[t]) : kTileInf;
  }
  for (; q < len; ++q) tile[q * 32 + lane] = act ? tile_in<TIn>(src[(int64_t)q * stride]) : kTileInf;
  if (!act) return;
  // ---- forward sweep: lower envelope, stack in place ----
  int k = -1;
  int vt = 0, vp = 0;
  int Ft = 0, Fp = 0;
  for (int qq = 0; qq < len; ++qq) {
    const uint32_t e = tile[qq * 32 + lane];
    if (e == kTileInf) continue;
    const int fq = (int)e;
    const int Fq = fq + qq * qq;
    while (k >= 1) {
      // pop the top if s(vt, q) <= s(vp, vt)
      if ((long long)(Fq - Ft) * (vt - vp) <= (long long)(Ft - Fp) * (qq - vt)) {
        --k;
        vt = vp;
        Ft = Fp;
        if (k >= 1) {
          const uint32_t se = tile[(k - 1) * 32 + lane];
          vp = (int)(se & 1023u);
          Fp = (int)(se >> 10) + vp * vp;
        }
      } else {
        break;
      }
    }
    ++k;
    tile[k * 32 + lane] = ((uint32_t)fq << 10) | (uint32_t)qq;
    vp = vt;
    Fp = Ft;
    vt = qq;
    Ft = Fq;
  }
  TOut *dst = out + base;
  if (k < 0) {
    for (int qq = 0; qq < len; ++qq) store_tile_out<TOut>(dst + (int64_t)qq * stride, kTileInf);
    return;
  }
  // ---- output sweep ----
  int j = 0;
  uint32_t se = tile[lane];
  int vj = (int)(se & 1023u), fj = (int)(se >> 10);
  int Fj = fj + vj * vj;
  int vn = 0, fn = 0, Fn = 0;
  if (k >= 1) {
    se = tile[32 + lane];
    vn = (int)(se & 1023u);
    fn = (int)(se >> 10);
    Fn = fn + vn * vn;
  }
  for (int qq = 0; qq < len; ++qq) {
    while (j < k && (Fn - Fj) < 2 * qq * (vn - vj)) {
      ++j;
      vj = vn;
      fj = fn;
      Fj = Fn;
      if (j < k) {
        se = tile[(j + 1) * 32 + lane];
        vn = (int)(se & 1023u);
        fn = (int)(se >> 10);
        Fn = fn + vn * vn;
      }
    }
    const int dq = qq - vj;
    store_tile_out<TOut>(dst + (int64_t)qq * stride, (uint32_t)(dq * dq + fj));
  }
}

template <typename TIn, typename TOut>
static int launch_fh_smem(const TIn *in, TOut *out, int64_t n_outer, int64_t outer_stride, int64_t n2, int64_t len,
                          int64_t stride, cudaStream_t s) {
  if (n_outer == 0) return VPB_OK;
  VPB_REQUIRE(n_outer <= 65535, "EDT box side too long for the grid y dimension");
  const size_t smem = (size_t)len * 32 * sizeof(uint32_t);
  auto kern = edt_pass_fh_smem<TIn, TOut>;
  if (smem > 48 * 1024) VPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<dim3((unsigned)((n2 + 31) >> 5), (unsigned)n_outer), 32, smem, s>>>(in, out, n_outer, outer_stride, (int)n2,
                                                                              (int)len, stride);
  return check_launch("edt_pass_fh_smem");
}

// ---------------------------------------------------------------------------
// Segmented FH line kernels (the production path for lines <= 1024).
//
// A 128-thread CTA owns 32 lines (lane = line, over the contiguous z axis)
// staged as a [len][32] u32 tile in shared memory (row q = element q of the
// 32 lines; a warp reads one 128 B row, conflict-free).  Each line is split
// into KSEG = 4 segments, segment = warp: every thread builds the lower
// envelope of its segment IN PLACE (stack entry k overwrites tile row
// q0 + k, whose input is already consumed; entry = (F << 10) | v with
// F = f + v^2 < 2^22), the runs are merged pairwise (the envelope of two runs
// is a prefix of the left run plus a suffix of the right one: drop boundary
// parabolas dominated by their neighbours), then every thread locates the
// parabola covering its first output by binary search and sweeps its
// segment run-length: the envelope switches from c to n at the integer
// q_sw = floor((F_n - F_c) / 2 (v_n - v_c)) + 1, computed with one
// approximate fp32 division and an exact integer correction (no 64-bit
// division), so a run of outputs costs one multiply-add and one store each.
// Every comparison is exact integer arithmetic, so the result equals the
// reference's f64 FH (vp/mapping.py:458-483) bit for bit.
// ---------------------------------------------------------------------------
// KS segments per line (KS warps per CTA); SegLine<KS> holds the run bounds.
template <int KS>
struct SegLine {
  int lo[KS], hi[KS];
};

struct Elem {
  int v, F;  // F = f + v^2
};

// Shared-memory accesses by explicit 32-bit shared-window address (the
// generic-pointer form made the compiler re-derive the window base from
// SR_CgaCtaId on every access inside the envelope loops).
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}

__device__ __forceinline__ Elem unpack_entry(uint32_t e) {
  Elem r;
  r.v = (int)(e & 1023u);
  r.F = (int)(e >> 10);
  return r;
}

// column address of (row r) for this thread: col + r * 128
__device__ __forceinline__ Elem elem_at(uint32_t col, int B, int seg, int idx) {
  return unpack_entry(lds_u32(col + (uint32_t)(seg * B + idx) * 128u));
}

// s(a, b) < q  <=>  F_b - F_a < 2 q (v_b - v_a).  WIDE: 64-bit products
// (lines longer than 512, where 3 (n-1)^3 can exceed 2^31).
template <bool WIDE>
__device__ __forceinline__ bool boundary_lt(const Elem &a, const Elem &b, int q) {
  if constexpr (WIDE) return (long long)(b.F - a.F) < 2ll * q * (b.v - a.v);
  else return (b.F - a.F) < 2 * q * (b.v - a.v);
}

// dominated(l, p, r): s(l, p) >= s(p, r)
template <bool WIDE>
__device__ __forceinline__ bool dominated(const Elem &l, const Elem &p, const Elem &r) {
  if constexpr (WIDE) return (long long)(p.F - l.F) * (r.v - p.v) >= (long long)(r.F - p.F) * (p.v - l.v);
  else return (p.F - l.F) * (r.v - p.v) >= (r.F - p.F) * (p.v - l.v);
}

// previous / next non-empty element in segment order
template <class SL>
__device__ __forceinline__ bool prev_elem(const SL &S, int seg, int idx, int first_seg, int &ps, int &pi) {
  if (idx > S.lo[seg]) {
    ps = seg;
    pi = idx - 1;
    return true;
  }
  for (int t = seg - 1; t >= first_seg; --t)
    if (S.hi[t] > S.lo[t]) {
      ps = t;
      pi = S.hi[t] - 1;
      return true;
    }
  return false;
}

template <class SL>
__device__ __forceinline__ bool next_elem(const SL &S, int seg, int idx, int last_seg, int &ns, int &ni) {
  if (idx + 1 < S.hi[seg]) {
    ns = seg;
    ni = idx + 1;
    return true;
  }
  for (int t = seg + 1; t <= last_seg; ++t)
    if (S.hi[t] > S.lo[t]) {
      ns = t;
      ni = S.lo[t];
      return true;
    }
  return false;
}

// Merge left run (segments a..b) with right run (b+1..c) of one line.
template <bool WIDE, class SL>
__device__ void merge_runs(uint32_t col, int B, SL &S, int a, int b, int c) {
  int ls = -1, li = 0, rs = -1, ri = 0;
  for (int t = b; t >= a; --t)
    if (S.hi[t] > S.lo[t]) {
      ls = t;
      li = S.hi[t] - 1;
      break;
    }
  for (int t = b + 1; t <= c; ++t)
    if (S.hi[t] > S.lo[t]) {
      rs = t;
      ri = S.lo[t];
      break;
    }
  if (ls < 0 || rs < 0) return;
  while (true) {
    bool changed = false;
    const Elem L1 = elem_at(col, B, ls, li);
    const Elem R1 = elem_at(col, B, rs, ri);
    int ps, pi;
    if (prev_elem(S, ls, li, a, ps, pi)) {
      const Elem L2 = elem_at(col, B, ps, pi);
      if (dominated<WIDE>(L2, L1, R1)) {
        S.hi[ls] = li;  // drop the left run's last element
        ls = ps;
        li = pi;
        changed = true;
      }
    }
    if (!changed) {
      int ns, ni;
      if (next_elem(S, rs, ri, c, ns, ni)) {
        const Elem R2 = elem_at(col, B, ns, ni);
        if (dominated<WIDE>(L1, R1, R2)) {
          S.lo[rs] = ri + 1;  // drop the right run's first element
          rs = ns;
          ri = ni;
          changed = true;
        }
      }
    }
    if (!changed) break;
  }
}

template <typename TOut>
__device__ __forceinline__ void store_dist(TOut *p, int v);
template <>
__device__ __forceinline__ void store_dist<int32_t>(int32_t *p, int v) {
  *p = v;  // -1 = no source: the X pass stages it raw (== kTileInf)
}
template <>
__device__ __forceinline__ void store_dist<float>(float *p, int v) {
  *p = v < 0 ? __int_as_float(0x7f800000) : (float)v;
}
// a finite value (>= 0)
template <typename TOut>
__device__ __forceinline__ void store_val(TOut *p, int v) {
  *p = (TOut)v;
}

// Forward sweep of one thread's segment [q0, q1): lower envelope of the finite
// parabolas, stack IN PLACE at column rows q0 + k (entry (F << 10) | v).
// `State` carries the top two entries in registers.
struct FwdState {
  int k, vt, vp, Ft, Fp;
};

template <bool WIDE>
__device__ __forceinline__ void fwd_step(FwdState &S, uint32_t stk, int q, uint32_t e) {
  if (e == kTileInf) return;
  const int Fq = (int)e + q * q;
  while (S.k >= 1) {
    const bool pop = WIDE ? ((long long)(Fq - S.Ft) * (S.vt - S.vp) <= (long long)(S.Ft - S.Fp) * (q - S.vt))
                          : ((Fq - S.Ft) * (S.vt - S.vp) <= (S.Ft - S.Fp) * (q - S.vt));
    if (!pop) break;
    --S.k;
    S.vt = S.vp;
    S.Ft = S.Fp;
    if (S.k >= 1) {
      const Elem p = unpack_entry(lds_u32(stk + 128u * (uint32_t)(S.k - 1)));
      S.vp = p.v;
      S.Fp = p.F;
    }
  }
  ++S.k;
  sts_u32(stk + 128u * (uint32_t)S.k, ((uint32_t)Fq << 10) | (uint32_t)q);
  S.vp = S.vt;
  S.Fp = S.Ft;
  S.vt = q;
  S.Ft = Fq;
}

// Merges of the 4 segment runs + output sweep (all ETHREADS threads; no early
// return, so it can sit inside a persistent loop).  `k` = this thread's stack
// top from the forward sweep.  dst_base[line + q * stride] receives output q.
template <typename TOut, bool WIDE, int KSEG>
__device__ __forceinline__ void fh_merge_output(uint32_t tile_s, SegLine<KSEG> *segs, int len, bool act, int k,
                                                TOut *__restrict__ dst_base, uint32_t stride) {
  const int tid = threadIdx.x;
  const int s = tid >> 5;     // segment = warp index
  const int line = tid & 31;  // z lane
  const int B = (len + KSEG - 1) / KSEG;
  const int q0 = s * B, q1 = min(len, q0 + B);
  const uint32_t col = tile_s + 4u * (uint32_t)line;
  segs[line].lo[s] = 0;
  segs[line].hi[s] = k + 1;
  __syncthreads();
  // ---- pairwise merges up a binary tree: (0,1) (2,3) ..., then (01,23) ... ----
#pragma unroll
  for (int w = 1; w < KSEG; w <<= 1) {
    if (act && (s & (2 * w - 1)) == 0) merge_runs<WIDE>(col, B, segs[line], s, s + w - 1, s + 2 * w - 1);
    __syncthreads();
  }
  if (act && q0 < q1) {
    // segment bounds of the merged envelope in registers (indexed only
    // through unrolled selects: no local memory)
    int lo_[KSEG], hi_[KSEG];
#pragma unroll
    for (int t = 0; t < KSEG; ++t) {
      lo_[t] = segs[line].lo[t];
      hi_[t] = segs[line].hi[t];
    }
    int total = 0;
#pragma unroll
    for (int t = 0; t < KSEG; ++t) total += hi_[t] - lo_[t];
    TOut *dst = dst_base + line + (size_t)q0 * stride;
    if (total == 0) {
      for (int q = q0; q < q1; ++q, dst += stride) store_dist<TOut>(dst, -1);
    } else {
      auto rank_to = [&](int r, int &sg, int &ix) {
        sg = KSEG - 1;
        ix = hi_[KSEG - 1] - 1;
        bool found = false;
#pragma unroll
        for (int t = 0; t < KSEG; ++t) {
          const int sz = hi_[t] - lo_[t];
          if (!found && r < sz) {
            sg = t;
            ix = lo_[t] + r;
            found = true;
          }
          if (!found) r -= sz;
        }
      };
      auto elem = [&](int sg, int ix) { return elem_at(col, B, sg, ix); };
      // largest r with r == 0 or s(e_{r-1}, e_r) < q0
      int lo = 0, hi = total - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        int sa, ia, sb, ib;
        rank_to(mid - 1, sa, ia);
        rank_to(mid, sb, ib);
        if (boundary_lt<WIDE>(elem(sa, ia), elem(sb, ib), q0))
          lo = mid;
        else
          hi = mid - 1;
      }
      int cs, ci;
      rank_to(lo, cs, ci);
      int left = total - 1 - lo;  // parabolas after cur
      Elem cur = elem(cs, ci);
      // the envelope in rank order: (ns, ni) walks the merged runs, with the
      // current run's end cached in `hend`
      auto sel = [&](const int(&a)[KSEG], int t) {
        int v = a[0];
#pragma unroll
        for (int u = 1; u < KSEG; ++u) v = t == u ? a[u] : v;
        return v;
      };
      int ns = cs, ni = ci, hend = sel(hi_, cs);
      auto advance = [&]() {
        if (++ni >= hend) {
          int t2 = ns;
#pragma unroll
          for (int t = KSEG - 1; t >= 1; --t)
            if (t > ns && hi_[t] > lo_[t]) t2 = t;
          ns = t2;
          ni = sel(lo_, t2);
          hend = sel(hi_, t2);
        }
      };
      // advance to the next parabola at the first q with thr < q * den2
      // (thr = F_n - F_c, den2 = 2 (v_n - v_c); |both| < 2^22, so 32-bit is
      // exact for every line length on this path); none left: never.
      int thr = 0x7fffffff, den2 = 0;
      Elem nxt = cur;
      if (left > 0) {
        advance();
        nxt = elem(ns, ni);
        thr = nxt.F - cur.F;
        den2 = 2 * (nxt.v - cur.v);
      }
      // Output sweep (vp/mapping.py:478-483): advance while the next
      // parabola's intersection lies strictly left of q; d(q) = (q - v)^2 + f
      // (f >= 0: only finite parabolas are in the envelope).
      int v = cur.v, f = cur.F - cur.v * cur.v;
      for (int q = q0; q < q1; ++q, dst += stride) {
        while (thr < q * den2) {
          cur = nxt;
          v = cur.v;
          f = cur.F - v * v;
          thr = 0x7fffffff;
          den2 = 0;
          if (--left > 0) {
            advance();
            nxt = elem(ns, ni);
            thr = nxt.F - cur.F;
            den2 = 2 * (nxt.v - v);
          }
        }
        const int d = q - v;
        store_val<TOut>(dst, d * d + f);
      }
    }
  }
}

// "No source on this side" markers of the z scan: far enough that
// min(z - L, R - z) >= 0x8000 flags a line without sources.
constexpr int kNoneLo = -0x10000;
constexpr int kNoneHi = 0x20000;

// Pass Z+Y fused, persistent: work item = (z chunk, x).  Warp w owns the
// rows of segment w.  For 32 of its rows at a time (one row per lane, all of
// the line's occupancy words in flight at once) it resolves the chunk's own
// 32-bit word and the nearest source on each side of the chunk; the rows are
// then broadcast lane to lane (shuffles), every lane computes dz^2 for its z
// and feeds it straight into the forward envelope sweep along y (no tile
// fill pass).  Output: int32 g(x, y, z) = min over y' of (y - y')^2 + dz^2
// (-1 = no source in the (x) plane).
template <bool WIDE, int KSEG>
__global__ void __launch_bounds__(32 * KSEG) edt_zy_kernel(const uint32_t *__restrict__ bits, int64_t gy,
                                                          int64_t words_z, int64_t lo0, int64_t lo1, int lo2, int n0,
                                                          int n1, int n2, int zc_base, int gz,
                                                          int32_t *__restrict__ out) {
  extern __shared__ __align__(128) uint32_t smem[];
  const uint32_t tile_s = (uint32_t)__cvta_generic_to_shared(smem);    // [n1][32]
  SegLine<KSEG> *segs = reinterpret_cast<SegLine<KSEG> *>(smem + (size_t)n1 * 32);  // [32]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = (n2 + 31) >> 5;
  const uint32_t le_mask = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
  const uint32_t ge_mask = 0xffffffffu << lane;
  const int B = (n1 + KSEG - 1) / KSEG;
  const bool aligned = (lo2 & 31) == 0;
  const int y0 = warp * B, y1 = min(n1, y0 + B);
  const uint32_t stk = tile_s + 4u * (uint32_t)lane + 128u * (uint32_t)y0;
  pdl_release();
  pdl_wait();  // the occupancy bits come from the fusion; the g tile buffer may still be read by the last X pass
  const int items = gz * n0;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int zc = zc_base + item % gz;
    const int64_t x = item / gz;
    const int zb = 32 * zc;
    const int nlines = min(32, n2 - zb);
    const bool act = lane < nlines;
    const int z = zb + lane;
    const uint32_t *wbase = bits + ((lo0 + x) * gy + lo1) * words_z + (lo2 >> 5);
    FwdState S{-1, 0, 0, 0, 0};
    for (int yb = y0; yb < y1; yb += 32) {
      // lane = row yb + lane: the chunk word and the nearest source on each side
      const int yr = yb + lane;
      uint32_t cw = 0;
      int L = kNoneLo, R = kNoneHi;
      if (yr < y1) {
        const uint32_t *w = wbase + (int64_t)yr * words_z;
        for (int c0 = 0; c0 < nw; c0 += 4) {
          uint32_t m[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int c = c0 + t;
            uint32_t v = 0u;
            if (c < nw) {
              v = aligned ? __ldg(w + c) : load_bits_window(w - (lo2 >> 5), lo2 + 32 * c, words_z);
              const int valid = n2 - 32 * c;
              if (valid < 32) v &= (1u << valid) - 1u;
            }
            m[t] = v;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int c = c0 + t;
            if (m[t] && c < zc) L = 32 * c + 31 - __clz(m[t]);
            if (c == zc) cw = m[t];
            if (m[t] && c > zc && R == kNoneHi) R = 32 * c + __ffs(m[t]) - 1;
          }
        }
      }
      // rows whose (x, y) line holds no source give +inf at every z: skip them
      // (warp-uniform: the row data is shared by all 32 lanes)
      uint32_t live = __ballot_sync(kFull, yr < y1 && (cw != 0u || L != kNoneLo || R != kNoneHi));
      while (live) {
        const int t = __ffs(live) - 1;
        live &= live - 1u;
        const uint32_t word = __shfl_sync(kFull, cw, t);
        const int Lw = __shfl_sync(kFull, L, t), Rw = __shfl_sync(kFull, R, t);
        const uint32_t le = word & le_mask, ge = word & ge_mask;
        const int left = le ? zb + 31 - __clz(le) : Lw;
        const int rgt = ge ? zb + __ffs(ge) - 1 : Rw;
        const int d = min(z - left, rgt - z);
        if (act) fwd_step<WIDE>(S, stk, yb + t, d < 0x8000 ? (uint32_t)(d * d) : kTileInf);
      }
    }
    fh_merge_output<int32_t, WIDE, KSEG>(tile_s, segs, n1, act, S.k, out + (x * n1) * (int64_t)n2 + zb, (uint32_t)n2);
    __syncthreads();  // the tile is reused by the next item
  }
}

// --- TMA helpers (cp.async.bulk.tensor + mbarrier) ---------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(a),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(d),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(b)
      : "memory");
}

constexpr int kTmaRows = 256;  // TMA box rows per copy (the box-dimension limit)

// Pass X, persistent: work item = (z chunk, y).  The [n0][32] tile of
// g(:, y, zchunk) is staged by TMA (ceil(n0 / 256) box copies of 256 rows x
// 128 B on one mbarrier; g holds -1 == kTileInf for "no source", so the copy
// is raw; out-of-range z lanes arrive zero-filled and stay inactive), then the
// segmented FH runs along x and writes the f32 field.
template <bool WIDE, int KSEG>
__global__ void __launch_bounds__(32 * KSEG) edt_x_kernel(const __grid_constant__ CUtensorMap gmap, int n0, int n1,
                                                         int n2, int zc_base, int gz, float *__restrict__ out) {
  extern __shared__ __align__(128) uint32_t smem[];
  const int ncopies = (n0 + kTmaRows - 1) / kTmaRows;
  const int rows = ncopies == 1 ? n0 : ncopies * kTmaRows;
  uint32_t *tile = smem;                                                  // [rows][32]
  SegLine<KSEG> *segs = reinterpret_cast<SegLine<KSEG> *>(smem + (size_t)rows * 32);  // [32]
  uint64_t *bar = reinterpret_cast<uint64_t *>(segs + 32);
  const uint32_t tile_s = (uint32_t)__cvta_generic_to_shared(tile);
  const int tid = threadIdx.x, lane = tid & 31, s = tid >> 5;
  const int B = (n0 + KSEG - 1) / KSEG;
  const int q0 = s * B, q1 = min(n0, q0 + B);
  const uint32_t col = tile_s + 4u * (uint32_t)lane;
  const uint32_t stk = col + 128u * (uint32_t)q0;
  const int box = ncopies == 1 ? n0 : kTmaRows;
  pdl_release();
  pdl_wait();  // g comes from edt_zy_kernel
  if (tid == 0) mbar_init(bar, 1);
  __syncthreads();
  const int items = gz * n1;
  unsigned phase = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x, phase ^= 1u) {
    const int zc = zc_base + item % gz;
    const int y = item / gz;
    const int nlines = min(32, n2 - zc * 32);
    const bool act = lane < nlines;
    if (tid == 0) {
      // order this CTA's earlier generic-proxy smem accesses before the async-proxy writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, (unsigned)(ncopies * box * 128));
      for (int c = 0; c < ncopies; ++c)
        tma_load_3d(tile + (size_t)c * kTmaRows * 32, &gmap, zc * 32, y, c * kTmaRows, bar);
    }
    mbar_wait(bar, phase);
    FwdState S{-1, 0, 0, 0, 0};
    if (act && q0 < q1) {
      uint32_t e_next = lds_u32(stk);
      for (int q = q0; q < q1; ++q) {
        const uint32_t e = e_next;
        if (q + 1 < q1) e_next = lds_u32(col + 128u * (uint32_t)(q + 1));
        fwd_step<WIDE>(S, stk, q, e);
      }
    }
    fh_merge_output<float, WIDE, KSEG>(tile_s, segs, n0, act, S.k, out + (int64_t)y * n2 + zc * 32, (uint32_t)(n1 * n2));
    __syncthreads();  // every thread is done with the tile before the next copy lands
  }
}

// Tensor map of g (int32, dims (n2, n1, n0), z innermost) with a
// (32, 1, min(n0, 256)) box, built with the driver's cuTensorMapEncodeTiled
// (resolved once through the runtime: no -lcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int make_g_map(CUtensorMap *map, const int32_t *g, int64_t n0, int64_t n1, int64_t n2) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    VPB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    VPB_REQUIRE(p && q == cudaDriverEntryPointSuccess, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)n0};
  const cuuint64_t strides[2] = {(cuuint64_t)n2 * 4, (cuuint64_t)n1 * n2 * 4};
  const cuuint32_t box[3] = {32, 1, (cuuint32_t)(n0 < kTmaRows ? n0 : kTmaRows)};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, const_cast<int32_t *>(g), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  VPB_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return VPB_OK;
}

static size_t x_tile_rows(int64_t n0) {
  const int64_t c = (n0 + kTmaRows - 1) / kTmaRows;
  return (size_t)(c == 1 ? n0 : c * kTmaRows);
}

template <typename TIn, typename TOut>
static int launch_fh(const TIn *in, TOut *out, int64_t n_outer, int64_t outer_stride, int64_t n2, int64_t len,
                     int64_t stride, int64_t max_dim, cudaStream_t s) {
  const int64_t warps = n_outer * ((n2 + 31) >> 5);
  const size_t smem = (size_t)len * 64 * sizeof(uint16_t);
  const unsigned grid = (unsigned)ceil_div(warps, 2);
  if (grid == 0) return VPB_OK;
  // 3 (N-1)^3 must fit the accumulator.
  const double worst = 3.0 * (double)(max_dim) * (double)(max_dim) * (double)(max_dim);
  if (worst < 2.0e9) {
    auto kern = edt_pass_fh<TIn, TOut, int32_t>;
    if (smem > 48 * 1024) VPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, 64, smem, s>>>(in, out, n_outer, outer_stride, n2, len, stride);
  } else {
    auto kern = edt_pass_fh<TIn, TOut, long long>;
    if (smem > 48 * 1024) VPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, 64, smem, s>>>(in, out, n_outer, outer_stride, n2, len, stride);
  }
  return check_launch("edt_pass_fh");
}

// The production path (lines <= 1024, z % 4 == 0): pass Z+Y fused from the
// occupancy words, then pass X (TMA-staged), both persistent.  The z chunks
// run in groups sized so one group's int32 g stays in L2 between the two
// launches (VPB_EDT_L2_MB, default 128 MB: at 512^3 four 32 MB chunks per group
// measured best, 1.14 -> 0.89 ms for the bench scene; the 126 MB L2 keeps most of it).
template <bool WIDE, int KS>
static int edt_tiled(const vpb_grid *grid, const int64_t lo[3], const int64_t n[3], int32_t *g2, float *out_sq,
                     cudaStream_t s) {
  const size_t smem_zy = (size_t)n[1] * 32 * 4 + sizeof(SegLine<KS>) * 32;
  const size_t smem_x = x_tile_rows(n[0]) * 32 * 4 + sizeof(SegLine<KS>) * 32 + 16;
  auto kzy = edt_zy_kernel<WIDE, KS>;
  auto kx = edt_x_kernel<WIDE, KS>;
  // host-side setup cached per (device, shape, g buffer): attributes, the
  // tensor map and the occupancy queries cost ~10 us of host time per call
  struct Setup {
    int dev = -1;
    int64_t n0 = 0, n1 = 0, n2 = 0;
    const int32_t *g = nullptr;
    CUtensorMap gmap;
    int occ_zy = 0, occ_x = 0;
  };
  static thread_local Setup cache;
  int dev = 0;
  VPB_CUDA(cudaGetDevice(&dev));
  int rc = VPB_OK;
  if (cache.dev != dev || cache.n0 != n[0] || cache.n1 != n[1] || cache.n2 != n[2] || cache.g != g2) {
    VPB_CUDA(cudaFuncSetAttribute(kzy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_zy));
    VPB_CUDA(cudaFuncSetAttribute(kx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_x));
    if ((rc = make_g_map(&cache.gmap, g2, n[0], n[1], n[2]))) return rc;
    VPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cache.occ_zy, kzy, 32 * KS, smem_zy));
    VPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cache.occ_x, kx, 32 * KS, smem_x));
    cache.dev = dev;
    cache.n0 = n[0], cache.n1 = n[1], cache.n2 = n[2];
    cache.g = g2;
  }
  const CUtensorMap gmap = cache.gmap;
  const int zch = (int)((n[2] + 31) / 32);
  static const double l2_mb = getenv("VPB_EDT_L2_MB") ? atof(getenv("VPB_EDT_L2_MB")) : 128.0;
  const double chunk_mb = (double)n[0] * (double)n[1] * 32.0 * 4.0 / 1048576.0;
  int group = (int)(l2_mb / chunk_mb);
  group = group < 1 ? 1 : (group > zch ? zch : group);
  // persistent grids: every SM filled with as many CTAs as smem / registers allow
  const int occ_zy = cache.occ_zy, occ_x = cache.occ_x;
  const int64_t slots_zy = (int64_t)sm_count() * (occ_zy > 0 ? occ_zy : 1);
  const int64_t slots_x = (int64_t)sm_count() * (occ_x > 0 ? occ_x : 1);
  // VPB_EDT_PDL: 0 none (default), 1 the Z+Y pass launched under the fusion's tail, 2 also X under
  // Z+Y.  Measured on the replan: 1 costs 1-2 us and 2 costs 11 us (the early-resident waiting CTAs
  // slow the running grid more than the hidden launch saves); the fusion pair gains 2 us.
  static const int pdl_mode = getenv("VPB_EDT_PDL") ? atoi(getenv("VPB_EDT_PDL")) : 0;
  const bool pdl_zy = pdl_enabled() && pdl_mode >= 1, pdl_x = pdl_enabled() && pdl_mode >= 2;
  for (int z0 = 0; z0 < zch; z0 += group) {
    const int gz = z0 + group <= zch ? group : zch - z0;
    const int64_t it_zy = (int64_t)gz * n[0], it_x = (int64_t)gz * n[1];
    VPB_CUDA(launch_ex(pdl_zy, kzy, dim3((unsigned)(it_zy < slots_zy ? it_zy : slots_zy)), dim3(32 * KS), smem_zy, s,
                        grid->occ_bits, grid->dims[1], ceil_div(grid->dims[2], 32), lo[0], lo[1], (int)lo[2],
                        (int)n[0], (int)n[1], (int)n[2], z0, gz, g2));
    rc = check_launch("edt_zy_kernel");
    if (rc) return rc;
    VPB_CUDA(launch_ex(pdl_x, kx, dim3((unsigned)(it_x < slots_x ? it_x : slots_x)), dim3(32 * KS), smem_x, s, gmap,
                        (int)n[0], (int)n[1], (int)n[2], z0, gz, out_sq));
    rc = check_launch("edt_x_kernel");
    if (rc) return rc;
  }
  return VPB_OK;
}

}  // namespace vpb

using namespace vpb;

extern "C" {

size_t vpb_edt3d_workspace_bytes(const int64_t n[3]) {
  const size_t vox = (size_t)n[0] * (size_t)n[1] * (size_t)n[2];
  // u16 z distances or the per-word left/right table (n0 n1 ceil(n2/32) u32), then int32 g
  const size_t lrb = (size_t)n[0] * (size_t)n[1] * (size_t)((n[2] + 31) / 32) * 4;
  return align_up(vox * sizeof(uint16_t) > lrb ? vox * sizeof(uint16_t) : lrb, 256) +
         align_up(vox * sizeof(int32_t), 256);
}

int vpb_edt3d(const vpb_grid *grid, const int64_t lo[3], const int64_t n[3], double thr, int use_bits,
              float *out_sq, void *workspace, size_t workspace_bytes, void *stream) {
  VPB_REQUIRE(grid && out_sq, "null argument to vpb_edt3d");
  for (int k = 0; k < 3; ++k)
    VPB_REQUIRE(lo[k] >= 0 && n[k] >= 1 && lo[k] + n[k] <= grid->dims[k], "box outside grid on axis %d", k);
  VPB_REQUIRE(n[0] <= 65535 && n[1] <= 65535 && n[2] <= 65535, "box side too long (max 65535)");
  VPB_REQUIRE(workspace && workspace_bytes >= vpb_edt3d_workspace_bytes(n), "EDT workspace too small");
  // FH stack of a line lives in shared memory: 64 threads x len x 2 B.
  VPB_REQUIRE((n[0] > n[1] ? n[0] : n[1]) * 64 * 2 <= 220 * 1024, "box side too long for the FH stack (max 1760)");
  cudaStream_t s = as_stream(stream);
  const size_t vox = (size_t)n[0] * (size_t)n[1] * (size_t)n[2];
  uint16_t *dz = reinterpret_cast<uint16_t *>(workspace);
  const size_t lrb = (size_t)n[0] * (size_t)n[1] * (size_t)((n[2] + 31) / 32) * 4;
  int32_t *g2 = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(workspace) + align_up(vox * 2 > lrb ? vox * 2 : lrb, 256));
  const int64_t lines_z = n[0] * n[1];
  const int64_t maxd = n[0] > n[1] ? (n[0] > n[2] ? n[0] : n[2]) : (n[1] > n[2] ? n[1] : n[2]);
  int rc = VPB_OK;
  if (maxd <= 1024 && use_bits && n[0] <= 65535 && n[1] <= 65535 && n[2] % 4 == 0) {  // 16 B-aligned g rows
    VPB_REQUIRE(grid->occ_bits, "use_bits set but grid->occ_bits is null");
    // 4 segments per line up to ~384 (6 CTAs x 4 warps per SM at 256), 8 for
    // longer lines (the tile halves the CTAs per SM; 8 warps keep 24 resident)
    static const int kseg_env = getenv("VPB_EDT_KSEG") ? atoi(getenv("VPB_EDT_KSEG")) : 0;
    const int kseg = kseg_env ? kseg_env : ((n[0] > 384 || n[1] > 384) ? 8 : 4);
    const bool wide = maxd > 512;
    if (kseg == 8)
      return wide ? edt_tiled<true, 8>(grid, lo, n, g2, out_sq, s) : edt_tiled<false, 8>(grid, lo, n, g2, out_sq, s);
    return wide ? edt_tiled<true, 4>(grid, lo, n, g2, out_sq, s) : edt_tiled<false, 4>(grid, lo, n, g2, out_sq, s);
  }
  if (use_bits) {
    VPB_REQUIRE(grid->occ_bits, "use_bits set but grid->occ_bits is null");
    edt_pass_z_bits<<<(unsigned)ceil_div(lines_z, 8), 256, 0, s>>>(
        grid->occ_bits, grid->dims[1], ceil_div(grid->dims[2], 32), lo[0], lo[1], lo[2], n[0], n[1], n[2], dz);
  } else {
    VPB_REQUIRE(grid->log_odds, "log_odds is null");
    edt_pass_z_logodds<<<(unsigned)ceil_div(lines_z, 8), 256, 0, s>>>(
        grid->log_odds, grid->dims[1], grid->dims[2], lo[0], lo[1], lo[2], n[0], n[1], n[2], thr, dz);
  }
  rc = check_launch("edt_pass_z");
  if (rc) return rc;
  if (maxd <= 1024) {
    rc = launch_fh_smem<uint16_t, int32_t>(dz, g2, n[0], n[1] * n[2], n[2], n[1], n[2], s);
    if (rc) return rc;
    return launch_fh_smem<int32_t, float>(g2, out_sq, n[1], n[2], n[2], n[0], n[1] * n[2], s);
  }
  rc = launch_fh<uint16_t, int32_t>(dz, g2, n[0], n[1] * n[2], n[2], n[1], n[2], maxd, s);
  if (rc) return rc;
  return launch_fh<int32_t, float>(g2, out_sq, n[1], n[2], n[2], n[0], n[1] * n[2], maxd, s);
}

}  // extern "C"
