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
// Fast z pass (box z-length <= 1024): one warp per (x, y) line.  Lane i holds
// the i-th 32-bit word of the line's occupancy; a warp max-scan / min-scan
// over the words gives every word the last source before it and the first
// source after it, so each output needs one word and two shuffled carries.
// Writes u16 nearest-source distances (0xFFFF = no source on the line).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) edt_pass_z_scan(const uint32_t *__restrict__ bits, int64_t gy,
                                                       int64_t words_z, int64_t lo0, int64_t lo1, int lo2,
                                                       int64_t n0, int64_t n1, int n2, uint16_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  // grid: (ceil(n1 / 8), n0)
  const int64_t i1 = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i1 >= n1) return;
  const int64_t i0 = blockIdx.y;
  const int64_t line = i0 * n1 + i1;
  const uint32_t *w = bits + ((lo0 + i0) * gy + (lo1 + i1)) * words_z;
  const int nw = (n2 + 31) >> 5;
  uint32_t word = 0;
  if (lane < nw) {
    const int zb = lo2 + 32 * lane;  // global z of bit 0 of this window
    const int wi = zb >> 5, sh = zb & 31;
    const uint32_t a = __ldg(w + wi);
    const uint32_t b = (sh != 0 && wi + 1 < words_z) ? __ldg(w + wi + 1) : 0u;
    word = sh ? __funnelshift_r(a, b, sh) : a;
    const int valid = n2 - 32 * lane;
    if (valid < 32) word &= (1u << valid) - 1u;
  }
  // last source at or before each word / first source at or after it
  int last = word ? 32 * lane + 31 - __clz(word) : -1;
  int first = word ? 32 * lane + __ffs(word) - 1 : 0x7fffffff;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int l = __shfl_up_sync(kFull, last, d);
    if (lane >= d) last = max(last, l);
    const int f = __shfl_down_sync(kFull, first, d);
    if (lane + d < 32) first = min(first, f);
  }
  // exclusive versions: before word i / after word i
  int last_ex = __shfl_up_sync(kFull, last, 1);
  if (lane == 0) last_ex = -1;
  int first_ex = __shfl_down_sync(kFull, first, 1);
  if (lane == 31) first_ex = 0x7fffffff;
  uint16_t *o = out + line * n2;
  const uint32_t le_mask = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
  const uint32_t ge_mask = 0xffffffffu << lane;
  for (int c = 0; c < nw; ++c) {
    const uint32_t wc = __shfl_sync(kFull, word, c);
    const int lx = __shfl_sync(kFull, last_ex, c);
    const int fx = __shfl_sync(kFull, first_ex, c);
    const int z = 32 * c + lane;
    const uint32_t le = wc & le_mask, ge = wc & ge_mask;
    const int left = le ? 32 * c + 31 - __clz(le) : lx;
    const int right = ge ? 32 * c + __ffs(ge) - 1 : fx;
    int d = 0x7fffffff;
    if (left >= 0) d = z - left;
    if (right != 0x7fffffff) d = min(d, right - z);
    if (z < n2) o[z] = d == 0x7fffffff ? kNoSrc16 : (uint16_t)min(d, 0xFFFE);
  }
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
// A 128-thread CTA owns 32 lines (lanes over the contiguous z axis) staged as
// a [len][32] u32 tile in shared memory.  Each line is split into KSEG = 4
// segments handled by 4 threads: each builds the lower envelope of its
// segment in place (stack entry (f << 10) | v over consumed input slots),
// the envelopes are merged pairwise (the merged envelope of two runs is a
// prefix of the left run plus a suffix of the right one, found by dropping
// boundary parabolas that are dominated by their neighbours), and every
// thread then locates the parabola covering its first output by binary
// search and sweeps its segment.  Tile columns are rotated by 8 per segment
// so the 4 threads of a line hit different banks.
// ---------------------------------------------------------------------------
constexpr int KSEG = 4;
constexpr int LINES = 32;
constexpr int ETHREADS = LINES * KSEG;

struct SegLine {
  int lo[KSEG], hi[KSEG];
};

__device__ __forceinline__ int tslot(int line, int seg, int row) { return row * 32 + ((line + 8 * seg) & 31); }

struct Elem {
  int v, f, F;
};

__device__ __forceinline__ Elem elem_at(const uint32_t *tile, int line, int B, int seg, int idx) {
  const uint32_t e = tile[tslot(line, seg, seg * B + idx)];
  Elem r;
  r.v = (int)(e & 1023u);
  r.f = (int)(e >> 10);
  r.F = r.f + r.v * r.v;
  return r;
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
__device__ __forceinline__ bool prev_elem(const SegLine &S, int seg, int idx, int first_seg, int &ps, int &pi) {
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

__device__ __forceinline__ bool next_elem(const SegLine &S, int seg, int idx, int last_seg, int &ns, int &ni) {
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
template <bool WIDE>
__device__ void merge_runs(const uint32_t *tile, int line, int B, SegLine &S, int a, int b, int c) {
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
    const Elem L1 = elem_at(tile, line, B, ls, li);
    const Elem R1 = elem_at(tile, line, B, rs, ri);
    int ps, pi;
    if (prev_elem(S, ls, li, a, ps, pi)) {
      const Elem L2 = elem_at(tile, line, B, ps, pi);
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
        const Elem R2 = elem_at(tile, line, B, ns, ni);
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
  *p = v < 0 ? -1 : v;  // -1 = no source: the X pass copies it raw (== kTileInf)
}
template <>
__device__ __forceinline__ void store_dist<float>(float *p, int v) {
  *p = v < 0 ? __int_as_float(0x7f800000) : (float)v;
}

// Envelope + output for the tile (called by all ETHREADS threads after the
// tile is filled and synchronised).  dst_base + line + q * stride receives
// output q of `line`.
template <typename TOut, bool WIDE>
__device__ void segmented_fh(uint32_t *tile, SegLine *segs, int len, int nlines_active, TOut *dst_base,
                             int64_t stride) {
  const int tid = threadIdx.x;
  const int s = tid >> 5;     // segment = warp index
  const int line = tid & 31;  // z lane
  const int B = (len + KSEG - 1) / KSEG;
  const int q0 = s * B, q1 = min(len, q0 + B);
  const bool act = line < nlines_active;
  uint32_t *col = tile + ((line + 8 * s) & 31);  // this thread's column; row r at col[r * 32]
  // ---- forward sweep on this segment (stack in place) ----
  int k = -1;
  if (act) {
    int vt = 0, vp = 0, Ft = 0, Fp = 0;
    const uint32_t *src = col + q0 * 32;
    for (int q = q0; q < q1; ++q, src += 32) {
      const uint32_t e = *src;
      if (e == kTileInf) continue;
      const int fq = (int)e;
      const int Fq = fq + q * q;
      while (k >= 1) {
        const bool pop = WIDE ? ((long long)(Fq - Ft) * (vt - vp) <= (long long)(Ft - Fp) * (q - vt))
                              : ((Fq - Ft) * (vt - vp) <= (Ft - Fp) * (q - vt));
        if (!pop) break;
        --k;
        vt = vp;
        Ft = Fp;
        if (k >= 1) {
          const uint32_t se = col[(q0 + k - 1) * 32];
          vp = (int)(se & 1023u);
          Fp = (int)(se >> 10) + vp * vp;
        }
      }
      ++k;
      col[(q0 + k) * 32] = ((uint32_t)fq << 10) | (uint32_t)q;
      vp = vt;
      Fp = Ft;
      vt = q;
      Ft = Fq;
    }
  }
  segs[line].lo[s] = 0;
  segs[line].hi[s] = k + 1;
  __syncthreads();
  // ---- merges: (0,1) and (2,3), then (01, 23) ----
  if (act && (s == 0 || s == 2)) merge_runs<WIDE>(tile, line, B, segs[line], s, s, s + 1);
  __syncthreads();
  if (act && s == 0) merge_runs<WIDE>(tile, line, B, segs[line], 0, 1, 3);
  __syncthreads();
  if (!act || q0 >= q1) return;
  // segment bounds of the merged envelope in registers (indexed only through
  // unrolled selects: no local memory)
  int lo_[KSEG], hi_[KSEG];
#pragma unroll
  for (int t = 0; t < KSEG; ++t) {
    lo_[t] = segs[line].lo[t];
    hi_[t] = segs[line].hi[t];
  }
  auto sel = [&](const int (&a)[KSEG], int t) {
    int v = a[0];
#pragma unroll
    for (int u = 1; u < KSEG; ++u) v = t == u ? a[u] : v;
    return v;
  };
  int total = 0;
#pragma unroll
  for (int t = 0; t < KSEG; ++t) total += hi_[t] - lo_[t];
  TOut *dst = dst_base + line + (int64_t)q0 * stride;
  if (total == 0) {
    for (int q = q0; q < q1; ++q, dst += stride) store_dist<TOut>(dst, -1);
    return;
  }
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
  auto elem = [&](int sg, int ix) { return elem_at(tile, line, B, sg, ix); };
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
  int rk = lo;  // rank of cur
  Elem cur = elem(cs, ci);
  // next element: same segment, else the next non-empty one
  auto step = [&](int &sg, int &ix) {
    if (ix + 1 < sel(hi_, sg)) {
      ++ix;
      return;
    }
    int ns = sg, ni = ix;
#pragma unroll
    for (int t = KSEG - 1; t >= 1; --t)
      if (t > sg && hi_[t] > lo_[t]) {
        ns = t;
        ni = lo_[t];
      }
    sg = ns;
    ix = ni;
  };
  int ns = cs, ni = ci;
  bool has_next = rk + 1 < total;
  Elem nxt = cur;
  if (has_next) {
    step(ns, ni);
    nxt = elem(ns, ni);
  }
  // The envelope changes to `nxt` at the first q with F_n - F_c < 2 q (v_n - v_c)
  // (v_n > v_c): q_sw = floor((F_n - F_c) / (2 (v_n - v_c))) + 1.  Between
  // switches the outputs are a run of (q - v)^2 + f.
  auto q_switch = [&](const Elem &c, const Elem &nx) -> int {
    const long long num = (long long)nx.F - c.F, den = 2ll * (nx.v - c.v);
    long long fl = num / den;
    if ((num % den != 0) && (num < 0)) --fl;  // floor for a negative numerator
    return (int)(fl + 1);
  };
  int qs = has_next ? q_switch(cur, nxt) : 0x7fffffff;
  int q = q0;
  while (q < q1) {
    while (q >= qs) {  // advance (possibly over several parabolas)
      cur = nxt;
      ++rk;
      has_next = rk + 1 < total;
      if (has_next) {
        step(ns, ni);
        nxt = elem(ns, ni);
        qs = q_switch(cur, nxt);
      } else {
        qs = 0x7fffffff;
      }
    }
    const int qe = qs < q1 ? qs : q1;
    const int v = cur.v, f = cur.f;
    for (; q < qe; ++q, dst += stride) {
      const int d = q - v;
      store_dist<TOut>(dst, d * d + f);
    }
  }
}

// Per (x, y) line of the box, per 32-z word w of the box line: the nearest
// source strictly left of the word (box-local z + 1, 0 = none) in the low 16
// bits and the nearest strictly right (0xFFFF = none) in the high 16 bits.
// One thread per line; 2 MB of bits in, n0 n1 ceil(n2 / 32) words out.
__global__ void __launch_bounds__(256) edt_line_lr_kernel(const uint32_t *__restrict__ bits, int64_t gy,
                                                          int64_t words_z, int64_t lo0, int64_t lo1, int lo2,
                                                          int n0, int n1, int n2, uint32_t *__restrict__ lr) {
  const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= (int64_t)n0 * n1) return;
  const int64_t i0 = line / n1, i1 = line - i0 * n1;
  const uint32_t *w = bits + ((lo0 + i0) * gy + (lo1 + i1)) * words_z;
  const int nw = (n2 + 31) >> 5;
  uint32_t *o = lr + line * nw;
  // all of the line's words in flight at once (nw <= 32 on this path)
  uint32_t m[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    uint32_t v = 0u;
    if (c < nw) {
      v = load_bits_window(w, lo2 + 32 * c, words_z);
      const int valid = n2 - 32 * c;
      if (valid < 32) v &= (1u << valid) - 1u;
    }
    m[c] = v;
  }
  uint32_t left[32];
  int last = -1;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    left[c] = (uint32_t)(last + 1);
    if (m[c]) last = 32 * c + 31 - __clz(m[c]);
  }
  int first = 0xFFFF;
#pragma unroll
  for (int c = 31; c >= 0; --c) {
    if (c < nw) o[c] = left[c] | ((uint32_t)first << 16);
    if (m[c]) first = 32 * c + __ffs(m[c]) - 1;
  }
}

// Pass Z+Y fused: CTA = (z chunk, x).  The tile row y holds dz(x, y, z)^2 for
// the 32 z of the chunk, computed from the packed occupancy words of line
// (x, y): the word of the chunk gives the in-chunk neighbours, a ballot over
// the line's non-empty words gives the nearest non-empty word on each side
// (no z-pass intermediate).  The FH then runs along y.
// Output: int32 g(x, y, z) = min over y' of (y - y')^2 + dz^2 (INT_MAX = none).
template <bool WIDE>
__global__ void __launch_bounds__(ETHREADS) edt_zy_kernel(const uint32_t *__restrict__ bits, int64_t gy,
                                                          int64_t words_z, int64_t lo0, int64_t lo1, int lo2,
                                                          int n1, int n2, const uint32_t *__restrict__ lr,
                                                          int32_t *__restrict__ out) {
  extern __shared__ uint32_t smem[];
  uint32_t *tile = smem;                                                // [n1][32]
  SegLine *segs = reinterpret_cast<SegLine *>(smem + (size_t)n1 * 32);  // [32]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int zc = blockIdx.x;
  const int64_t x = blockIdx.y;
  const int nw = (n2 + 31) >> 5;
  const int nlines = min(32, n2 - zc * 32);
  const uint32_t le_mask = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
  const uint32_t ge_mask = 0xffffffffu << lane;
  const int B = (n1 + KSEG - 1) / KSEG;
  const int z = 32 * zc + lane;
  const int valid = n2 - 32 * zc;
  const uint32_t vmask = valid < 32 ? (1u << valid) - 1u : 0xffffffffu;
  const uint32_t *wbase = bits + ((lo0 + x) * gy + lo1) * words_z;
  const uint32_t *lrbase = lr + (x * n1) * (int64_t)nw + zc;
  uint32_t *dcol = tile + ((lane + 8 * warp) & 31);
  // warp w fills the rows of segment w (its rotated column is warp-uniform):
  // per row one broadcast word + one broadcast (left, right) pair
  const int y0 = warp * B, y1 = min(n1, y0 + B);
  auto fill = [&](int y, uint32_t word, uint32_t lrv) {
    word &= vmask;
    const uint32_t le = word & le_mask, ge = word & ge_mask;
    const int left = le ? 32 * zc + 31 - __clz(le) : (int)(lrv & 0xFFFFu) - 1;
    const int rgt = ge ? 32 * zc + __ffs(ge) - 1 : (int)(lrv >> 16);
    int d = 0x7fffffff;
    if (left >= 0) d = z - left;
    if (rgt != 0xFFFF) d = min(d, rgt - z);
    dcol[y * 32] = (lane < nlines && d != 0x7fffffff) ? (uint32_t)(d * d) : kTileInf;
  };
  int y = y0;
  for (; y + 4 <= y1; y += 4) {
    uint32_t wd[4], lv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      wd[t] = load_bits_window(wbase + (int64_t)(y + t) * words_z, lo2 + 32 * zc, words_z);
      lv[t] = __ldg(lrbase + (int64_t)(y + t) * nw);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) fill(y + t, wd[t], lv[t]);
  }
  for (; y < y1; ++y)
    fill(y, load_bits_window(wbase + (int64_t)y * words_z, lo2 + 32 * zc, words_z), __ldg(lrbase + (int64_t)y * nw));
  __syncthreads();
  int32_t *dst = out + (x * n1) * (int64_t)n2 + zc * 32;
  segmented_fh<int32_t, WIDE>(tile, segs, n1, nlines, dst, n2);
}

// Pass X: CTA = (z chunk, y); rows x of the tile are the 32 z values of
// g(x, y, zchunk) (one coalesced 128 B row each).
template <bool WIDE>
__global__ void __launch_bounds__(ETHREADS) edt_x_kernel(const int32_t *__restrict__ g, int n0, int n1, int n2,
                                                         float *__restrict__ out) {
  extern __shared__ uint32_t smem[];
  uint32_t *tile = smem;                                                // [n0][32]
  SegLine *segs = reinterpret_cast<SegLine *>(smem + (size_t)n0 * 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int zc = blockIdx.x;
  const int64_t y = blockIdx.y;
  const int nlines = min(32, n2 - zc * 32);
  const int B = (n0 + KSEG - 1) / KSEG;
  const int64_t row_stride = (int64_t)n1 * n2;
  const bool on = lane < nlines;
  // Stage the [n0][32] tile with asynchronous 16-byte copies (all rows in
  // flight at once; g holds -1 = kTileInf for "no source", so the copy is
  // raw).  Row x lands rotated by 8 * (segment of x) words, the column
  // layout segmented_fh expects.  Lanes past the line end are zero-filled
  // (inactive in the envelope).
  (void)on;
  const int32_t *gbase = g + y * n2 + zc * 32;
  const int bytes_row = nlines * 4;
  for (int i = tid; i < n0 * 8; i += ETHREADS) {
    const int r = i >> 3, piece = i & 7;  // 8 x 16 B per 128 B row
    const int sgm = r / B;
    const int col = (piece * 4 + 8 * sgm) & 31;
    const int rem = bytes_row - piece * 16;
    const int nb = rem >= 16 ? 16 : (rem > 0 ? rem : 0);
    const int32_t *src = nb > 0 ? gbase + (int64_t)r * row_stride + piece * 4 : g;
    const unsigned dst_s = (unsigned)__cvta_generic_to_shared(tile + r * 32 + col);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst_s), "l"(src), "r"(nb) : "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  float *dst = out + y * n2 + zc * 32;
  segmented_fh<float, WIDE>(tile, segs, n0, nlines, dst, row_stride);
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
  int rc;
  if (maxd <= 1024 && use_bits && n[0] <= 65535 && n[1] <= 65535 && n[2] % 4 == 0) {  // 16 B-aligned g rows
    VPB_REQUIRE(grid->occ_bits, "use_bits set but grid->occ_bits is null");
    // Pass Z+Y fused from the occupancy words, then pass X.
    const size_t smem_zy = (size_t)n[1] * 32 * 4 + sizeof(SegLine) * 32;
    const size_t smem_x = (size_t)n[0] * 32 * 4 + sizeof(SegLine) * 32;
    const bool wide = maxd > 512;
    auto kzy = wide ? edt_zy_kernel<true> : edt_zy_kernel<false>;
    auto kx = wide ? edt_x_kernel<true> : edt_x_kernel<false>;
    if (smem_zy > 48 * 1024) VPB_CUDA(cudaFuncSetAttribute(kzy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_zy));
    if (smem_x > 48 * 1024) VPB_CUDA(cudaFuncSetAttribute(kx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_x));
    const unsigned zch = (unsigned)((n[2] + 31) / 32);
    // per-line left/right source table (fits the u16 z-distance slot of the workspace)
    uint32_t *lr = reinterpret_cast<uint32_t *>(workspace);
    const int64_t lines = n[0] * n[1];
    edt_line_lr_kernel<<<(unsigned)ceil_div(lines, 256), 256, 0, s>>>(
        grid->occ_bits, grid->dims[1], ceil_div(grid->dims[2], 32), lo[0], lo[1], (int)lo[2], (int)n[0], (int)n[1],
        (int)n[2], lr);
    rc = check_launch("edt_line_lr_kernel");
    if (rc) return rc;
    kzy<<<dim3(zch, (unsigned)n[0]), ETHREADS, smem_zy, s>>>(grid->occ_bits, grid->dims[1], ceil_div(grid->dims[2], 32),
                                                             lo[0], lo[1], (int)lo[2], (int)n[1], (int)n[2], lr, g2);
    rc = check_launch("edt_zy_kernel");
    if (rc) return rc;
    kx<<<dim3(zch, (unsigned)n[1]), ETHREADS, smem_x, s>>>(g2, (int)n[0], (int)n[1], (int)n[2], out_sq);
    return check_launch("edt_x_kernel");
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
