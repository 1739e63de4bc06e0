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
__device__ __forceinline__ uint32_t load_bits_window(const uint32_t *__restrict__ w, int64_t z0) {
  // 32 bits of the line starting at global z0 (z0 may be unaligned).
  const int64_t wi = z0 >> 5;
  const int sh = (int)(z0 & 31);
  const uint32_t a = __ldg(w + wi);
  if (sh == 0) return a;
  const uint32_t b = __ldg(w + wi + 1);
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
  return align_up(vox * sizeof(uint16_t), 256) + align_up(vox * sizeof(int32_t), 256);
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
  int32_t *g2 = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(workspace) + align_up(vox * 2, 256));
  const int64_t lines_z = n[0] * n[1];
  if (use_bits) {
    VPB_REQUIRE(grid->occ_bits, "use_bits set but grid->occ_bits is null");
    if (n[2] <= 1024) {
      edt_pass_z_scan<<<dim3((unsigned)ceil_div(n[1], 8), (unsigned)n[0]), 256, 0, s>>>(grid->occ_bits, grid->dims[1],
                                                                     ceil_div(grid->dims[2], 32), lo[0], lo[1],
                                                                     (int)lo[2], n[0], n[1], (int)n[2], dz);
    } else {
      edt_pass_z_bits<<<(unsigned)ceil_div(lines_z, 8), 256, 0, s>>>(
          grid->occ_bits, grid->dims[1], ceil_div(grid->dims[2], 32), lo[0], lo[1], lo[2], n[0], n[1], n[2], dz);
    }
  } else {
    VPB_REQUIRE(grid->log_odds, "log_odds is null");
    edt_pass_z_logodds<<<(unsigned)ceil_div(lines_z, 8), 256, 0, s>>>(
        grid->log_odds, grid->dims[1], grid->dims[2], lo[0], lo[1], lo[2], n[0], n[1], n[2], thr, dz);
  }
  int rc = check_launch("edt_pass_z");
  if (rc) return rc;
  const int64_t maxd = n[0] > n[1] ? (n[0] > n[2] ? n[0] : n[2]) : (n[1] > n[2] ? n[1] : n[2]);
  if (maxd <= 1024) {
    // Pass Y: lines (x, z), element y at stride n2, outer stride n1*n2.
    rc = launch_fh_smem<uint16_t, int32_t>(dz, g2, n[0], n[1] * n[2], n[2], n[1], n[2], s);
    if (rc) return rc;
    // Pass X: lines (y, z), element x at stride n1*n2, outer stride n2.
    return launch_fh_smem<int32_t, float>(g2, out_sq, n[1], n[2], n[2], n[0], n[1] * n[2], s);
  }
  rc = launch_fh<uint16_t, int32_t>(dz, g2, n[0], n[1] * n[2], n[2], n[1], n[2], maxd, s);
  if (rc) return rc;
  return launch_fh<int32_t, float>(g2, out_sq, n[1], n[2], n[2], n[0], n[1] * n[2], maxd, s);
}

}  // extern "C"
