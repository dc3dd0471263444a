// K1: per-frame energy codes (luma, Sobel gradient, motion difference).
//
// Replaces energy.py:23-37 (to_luma), :40-59 (gradient_energy), :62-87 (motion_energy).
// The fp64 motion energy is a pure function of two bytes per pixel:
//   e = min(fl(fl(wm*|dL|) + fl(wg*g)), 255)   (g = pure Sobel on the clip's first frame)
// so one streaming pass writes a 2-byte code (|dL| << 8 | g) per pixel and every later
// consumer (window statistics, uniform map) decodes e in registers.
//
// Layout: frames (T, H, W, C) uint8, row-major; codes (T, H, W) uint16.
// Work is (tile, frame) units: a tile is 32 rows x 128 columns; a persistent CTA takes a
// contiguous range of units (consecutive frames of one tile, sometimes two tiles), keeps
// each thread's previous-frame luma in registers for the motion term, and streams the RGB
// tile (+1 row / +16 columns of halo) through a 2-slot ring filled by 3-D TMA boxes one
// frame ahead.  Frame borders replicate (np.pad mode="edge" in gradient_energy): the luma
// pass reads clamped coordinates, so the TMA's zero fill outside the frame is never used.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "scpl_common.cuh"
#include "scpl_kernels.h"

namespace scpl {

constexpr int kCW = 128, kCH = 32;      // output tile
constexpr int kCRows = kCH + 2;         // luma rows incl. halo
constexpr int kRawPx = kCW + 32;        // raw columns: c0-16 .. c0+143 (16-aligned box start)
constexpr int kLumStride = 144;         // bytes per luma row in shared memory
constexpr int kCodesThreads = 256;      // 8 warps: warp = 4 output rows, lane = 4 columns

template <int C>
struct RawGeo {
  static constexpr int kRowBytes = kRawPx * C;              // 480 / 160
  static constexpr int kBox = C == 3 ? 240 : 160;            // TMA box inner bytes (<= 256)
  static constexpr int kNBox = kRowBytes / kBox;             // 2 / 1
  static constexpr int kRegion = ((kCRows * kBox + 127) / 128) * 128;  // one box (TMA dst: 128-B aligned)
  static constexpr int kSlot = kNBox * kRegion;
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// byte x of raw row k in a slot (boxes are stored one after the other)
template <int C>
__device__ __forceinline__ int raw_off(int k, int x) {
  using G = RawGeo<C>;
  const int b = x / G::kBox;
  return b * G::kRegion + k * G::kBox + (x - b * G::kBox);
}

// luma of 4 RGB pixels packed in 12 bytes (a, b, c), energy.py:35 exactly: X + 500 =
// 256 (r + 2g) + (43 r + 75 g + 114 b) + 500 by byte dot products, the nearest integer of
// X / 1000 is floor((X + 500) / 1000) = umulhi(X + 500, 4294968) (exact for X + 500 <
// 256001, checked exhaustively); the rare ties X % 1000 == 500 take luma_of's fp64 path.
__device__ __forceinline__ uint32_t luma_t(uint32_t px, uint32_t c_hi, uint32_t c_lo, uint32_t& rem) {
  const uint32_t t = (__dp4a(px, c_hi, 0u) << 8) + __dp4a(px, c_lo, 500u);
  const uint32_t q = __umulhi(t, 4294968u);
  rem = t - q * 1000u;
  return q;
}
__device__ __forceinline__ uint32_t luma4_rgb(uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t p1 = __byte_perm(a, b, 0x0543);  // r1 g1 b1 (a3 b0 b1)
  const uint32_t p2 = __byte_perm(b, c, 0x0432);  // r2 g2 b2 (b2 b3 c0)
  uint32_t m0, m1, m2, m3;
  uint32_t q0 = luma_t(a, 0x00000201u, 0x00724B2Bu, m0);
  uint32_t q1 = luma_t(p1, 0x00000201u, 0x00724B2Bu, m1);
  uint32_t q2 = luma_t(p2, 0x00000201u, 0x00724B2Bu, m2);
  uint32_t q3 = luma_t(c, 0x00020100u, 0x724B2B00u, m3);  // r3 g3 b3 = c1 c2 c3
  if (__builtin_expect(m0 == 0u || m1 == 0u || m2 == 0u || m3 == 0u, 0)) {  // X % 1000 == 500
    if (m0 == 0u) q0 = luma_of(a & 255u, (a >> 8) & 255u, (a >> 16) & 255u);
    if (m1 == 0u) q1 = luma_of(a >> 24, b & 255u, (b >> 8) & 255u);
    if (m2 == 0u) q2 = luma_of((b >> 16) & 255u, b >> 24, c & 255u);
    if (m3 == 0u) q3 = luma_of((c >> 8) & 255u, (c >> 16) & 255u, c >> 24);
  }
  return __byte_perm(__byte_perm(q0, q1, 0x0040), __byte_perm(q2, q3, 0x0040), 0x5410);
}

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
}

// luma of the pixel at raw column rp (0 .. kRawPx-1) of raw row rk
template <int C>
__device__ __forceinline__ uint32_t raw_luma1(uint32_t raw_s, int rk, int rp) {
  const int x = rp * C;
  if (C == 3)
    return luma_of(lds8(raw_s + raw_off<C>(rk, x)), lds8(raw_s + raw_off<C>(rk, x + 1)),
                   lds8(raw_s + raw_off<C>(rk, x + 2)));
  return lds8(raw_s + raw_off<C>(rk, x));
}

// luma of a raw tile -> lum[kCRows][kLumStride] (column index = pixel - (c0 - 4)):
// warp = rows, lane = 4 columns c0 + 4 lane ..; then threads 0 .. 2*kCRows-1 add the halo
// pixels c0 - 1 and c0 + 128 of every row.  Frame borders replicate: rows and columns are
// clamped into the frame.  src0 = this lane's group in raw row 0 of the slot.
template <int C>
__device__ __forceinline__ void codes_luma(uint32_t raw_s, uint32_t src0, uint32_t lum_s, int r0, int c0, int H,
                                           int W) {
  using G = RawGeo<C>;
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  const int px0 = c0 + 4 * lane;
  const uint32_t dst0 = lum_s + 4 * lane + 4;
  if (px0 + 3 < W) {
#pragma unroll 1
    for (int k = wy; k < kCRows; k += kCodesThreads / 32) {
      const int rk = min(max(r0 - 1 + k, 0), H - 1) - (r0 - 1);  // clamped frame row
      const uint32_t src = src0 + rk * G::kBox;
      sts32(dst0 + k * kLumStride, C == 3 ? luma4_rgb(lds32(src), lds32(src + 4), lds32(src + 8)) : lds32(src));
    }
  } else {  // right frame border: clamped columns
#pragma unroll 1
    for (int k = wy; k < kCRows; k += kCodesThreads / 32) {
      const int rk = min(max(r0 - 1 + k, 0), H - 1) - (r0 - 1);
      uint32_t word = 0;
      for (int u = 0; u < 4; ++u) word |= raw_luma1<C>(raw_s, rk, min(px0 + u, W - 1) - (c0 - 16)) << (8 * u);
      sts32(dst0 + k * kLumStride, word);
    }
  }
  if (threadIdx.x < 2 * kCRows) {
    const int k = threadIdx.x >> 1, side = threadIdx.x & 1;
    const int rk = min(max(r0 - 1 + k, 0), H - 1) - (r0 - 1);
    const int px = min(max(side == 0 ? c0 - 1 : c0 + kCW, 0), W - 1);
    sts8(lum_s + k * kLumStride + (side == 0 ? 3 : kCW + 4), raw_luma1<C>(raw_s, rk, px - (c0 - 16)));
  }
}

// codes of one frame for this thread's 4 rows x 4 columns; prev[i] = previous luma word.
// Sobel in 16-bit lane pairs (even / odd columns): per luma row k, S_k = l + 2m + r
// (horizontal smoothing) and D_k = r - l (+256 bias); then gx = D_a + 2 D_b + D_c and
// gy = S_c - S_a (+1024 bias each), |g| = max(g', 2048 - g') - 1024 lane-wise, and
// min(|gx| + |gy|, 255) -- the same integers as gradient_energy's int32 Sobel.
// |dL| for 4 pixels is one byte-SIMD absolute difference.
__device__ __forceinline__ void codes_tile(uint32_t lum_s, uint32_t (&prev)[4], bool emit, bool have_prev,
                                           int r0, int c0, int H, int W, uint16_t* __restrict__ out,
                                           bool vec_out) {
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  uint32_t SE[6], SO[6], DE[6], DO[6], M[6];  // rows stream through: at most 3 live at once
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const uint32_t row = lum_s + (4 * wy + k) * kLumStride + 4 * lane;
    const uint32_t lo = lds32(row), mid = lds32(row + 4), hi = lds32(row + 8);
    const uint32_t wl = __byte_perm(lo, mid, 0x6543);  // columns -1 .. 2
    const uint32_t wr = __byte_perm(mid, hi, 0x4321);  // columns 1 .. 4
    const uint32_t le = __byte_perm(wl, 0, 0x4240), lo_ = __byte_perm(wl, 0, 0x4341);
    const uint32_t me = __byte_perm(mid, 0, 0x4240), mo = __byte_perm(mid, 0, 0x4341);
    const uint32_t re = __byte_perm(wr, 0, 0x4240), ro = __byte_perm(wr, 0, 0x4341);
    SE[k] = le + 2u * me + re;
    SO[k] = lo_ + 2u * mo + ro;
    DE[k] = re + 0x01000100u - le;
    DO[k] = ro + 0x01000100u - lo_;
    M[k] = mid;
    if (k < 2) continue;
    const int i = k - 2;
    const uint32_t gxe = DE[i] + 2u * DE[i + 1] + DE[i + 2], gxo = DO[i] + 2u * DO[i + 1] + DO[i + 2];
    const uint32_t gye = SE[i + 2] + 0x04000400u - SE[i], gyo = SO[i + 2] + 0x04000400u - SO[i];
    const uint32_t ae = __vmaxu2(gxe, 0x08000800u - gxe) + __vmaxu2(gye, 0x08000800u - gye) - 0x08000800u;
    const uint32_t ao = __vmaxu2(gxo, 0x08000800u - gxo) + __vmaxu2(gyo, 0x08000800u - gyo) - 0x08000800u;
    const uint32_t g = __byte_perm(__vminu2(ae, 0x00FF00FFu), __vminu2(ao, 0x00FF00FFu), 0x6240);
    const uint32_t d = have_prev ? __vabsdiffu4(M[i + 1], prev[i]) : 0u;
    prev[i] = M[i + 1];
    const uint32_t w0 = __byte_perm(g, d, 0x5140), w1 = __byte_perm(g, d, 0x7362);
    const int r = r0 + 4 * wy + i, c = c0 + 4 * lane;
    if (emit && r < H) {
      uint16_t* o = out + (size_t)i * W;  // out: this thread's first pixel
      if (vec_out && c + 3 < W) {
        *reinterpret_cast<uint2*>(o) = make_uint2(w0, w1);
      } else {
        const uint32_t v[4] = {w0 & 0xffffu, w0 >> 16, w1 & 0xffffu, w1 >> 16};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c + u < W) o[u] = (uint16_t)v[u];
      }
    }
  }
}

// plain (non-TMA) fill of a raw slot: frames with unaligned rows, or the API's separate
// previous-frame pointer.  Out-of-frame bytes are left as they are (never read).
template <int C>
__device__ __forceinline__ void codes_load_plain(const uint8_t* frame, uint8_t* raw, int r0, int c0, int H, int W) {
  constexpr int kRow = RawGeo<C>::kRowBytes;
  for (int q = threadIdx.x; q < kCRows * kRow; q += kCodesThreads) {
    const int k = q / kRow, x = q - k * kRow;
    const int r = r0 - 1 + k, px = c0 - 16 + x / C;
    if (r >= 0 && r < H && px >= 0 && px < W) raw[raw_off<C>(k, x)] = frame[((size_t)r * W + px) * C + x % C];
  }
}

template <int C>
__global__ void __launch_bounds__(kCodesThreads, 4) codes_kernel(const __grid_constant__ CUtensorMap tm,
                                                              const uint8_t* __restrict__ frames,
                                                              const uint8_t* __restrict__ prev_frame, int t0,
                                                              int n, int H, int W, int tiles_x, long units,
                                                              int use_tma, uint16_t* __restrict__ codes) {
  using G = RawGeo<C>;
  extern __shared__ __align__(128) uint8_t smem[];
  auto raw = [&](uint32_t s) { return smem + (s & 1u) * G::kSlot; };
  // two luma buffers: frame q's luma pass writes one while frame q-1's tile pass may still read
  // the other, so one block barrier per frame suffices
  auto lum = [&](uint32_t s) { return smem + 2 * G::kSlot + (s & 1u) * (kCRows * kLumStride); };
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * G::kSlot + 2 * kCRows * kLumStride);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const bool vec_out = (W & 3) == 0;
  const size_t fpx = (size_t)H * W;
  // this lane's 4-pixel group in raw row 0 of slot 0 (a group never straddles two boxes)
  const int gx_ = (4 * (threadIdx.x & 31) + 16) * C, gb_ = gx_ / G::kBox;
  const uint32_t src_lane = smem_u32(smem) + gb_ * G::kRegion + (gx_ - gb_ * G::kBox);
  uint32_t phase = 0;  // bit s: parity of slot s
  uint32_t seq = 0;    // frames consumed so far (slot = seq & 1)

  // unit u = tile * n + (t - t0); this CTA owns [u0, u1)
  const long per = (units + gridDim.x - 1) / gridDim.x;
  long u = (long)blockIdx.x * per;
  const long u1 = min(units, u + per);
  while (u < u1) {
    const int tile = (int)(u / n);
    const int tb = t0 + (int)(u - (long)tile * n);
    const int te = t0 + (int)min((long)n, (long)(tb - t0) + (u1 - u));
    u += te - tb;
    const int r0 = (tile / tiles_x) * kCH, c0 = (tile % tiles_x) * kCW;
    // frame sequence: q = 0 is frame tb-1 (if any), then tb .. te-1
    const bool prev_in_clip = tb > 0;
    const bool have_prev0 = prev_in_clip || prev_frame != nullptr;
    const int q0 = have_prev0 ? 0 : 1, q1 = te - tb;
    auto fill = [&](int q, uint32_t s) {
      const int t = tb + q - 1;
      if (q == 0 && !prev_in_clip) {
        codes_load_plain<C>(prev_frame, raw(s), r0, c0, H, W);
      } else if (use_tma) {
        if (threadIdx.x == 0) {
          mbar_arrive_tx(&bar[s & 1], (uint32_t)(G::kNBox * kCRows * G::kBox));
#pragma unroll
          for (int b = 0; b < G::kNBox; ++b)
            tma_load_3d(raw(s) + b * G::kRegion, &tm, (c0 - 16) * C + b * G::kBox, r0 - 1, t, &bar[s & 1]);
        }
      } else {
        codes_load_plain<C>(frames + (size_t)t * fpx * C, raw(s), r0, c0, H, W);
      }
    };
    auto tma_slot = [&](int q) { return use_tma && !(q == 0 && !prev_in_clip); };
    uint32_t prev[4] = {0, 0, 0, 0};
    // One barrier per frame (B_q, after the luma pass): the raw slot of frame q+1 was last read by
    // frame q-1's luma pass and the luma buffer of frame q by frame q-2's tile pass, both before
    // B_{q-1}; a plain (cooperative) fill of frame q+1 is made visible by B_q.
    fill(q0, seq);
    if (!tma_slot(q0)) __syncthreads();
    for (int q = q0; q <= q1; ++q, ++seq) {
      if (q + 1 <= q1) fill(q + 1, seq + 1);
      if (tma_slot(q)) {
        mbar_wait(&bar[seq & 1], (phase >> (seq & 1)) & 1u);
        phase ^= 1u << (seq & 1);
      }
      codes_luma<C>(smem_u32(raw(seq)), src_lane + (seq & 1u) * G::kSlot, smem_u32(lum(seq)), r0, c0, H, W);
      __syncthreads();  // B_q
      const int t = tb + q - 1;
      codes_tile(smem_u32(lum(seq)), prev, q >= 1, q > 1 || have_prev0, r0, c0, H, W,
                 codes + (size_t)t * fpx + (size_t)(r0 + 4 * (threadIdx.x >> 5)) * W + c0 + 4 * (threadIdx.x & 31),
                 vec_out);
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 codes_tmap_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    SCPL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    SCPL_ARG(q == cudaDriverEntryPointSuccess && p != nullptr, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <int C>
static void launch_codes_c(const uint8_t* frames, const uint8_t* prev_frame, int t0, int n, int H, int W,
                           uint16_t* codes, int num_sms, cudaStream_t st) {
  using G = RawGeo<C>;
  const size_t row_bytes = (size_t)W * C;
  const bool tma = (row_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(frames) & 15) == 0);
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  if (tma) {
    cuuint64_t dims[3] = {(cuuint64_t)row_bytes, (cuuint64_t)H, (cuuint64_t)(t0 + n)};
    cuuint64_t strides[2] = {(cuuint64_t)row_bytes, (cuuint64_t)row_bytes * H};
    cuuint32_t box[3] = {(cuuint32_t)G::kBox, (cuuint32_t)kCRows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = codes_tmap_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(frames), dims,
                                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SCPL_ARG(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed for the clip");
  }
  const size_t smem = 2 * (size_t)G::kSlot + 2 * (size_t)kCRows * kLumStride + 16;
  const int tiles_x = cdiv(W, kCW), tiles = tiles_x * cdiv(H, kCH);
  const long units = (long)tiles * n;
  static std::atomic<int> per_sm_cache{0};  // resident CTAs per SM (same on every B200)
  int per_sm = per_sm_cache.load();
  smem_optin(reinterpret_cast<const void*>(codes_kernel<C>));  // (once per device)
  if (per_sm == 0) {
    SCPL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, codes_kernel<C>, kCodesThreads, smem));
    if (per_sm < 1) per_sm = 1;
    per_sm_cache.store(per_sm);
  }
  const long grid = std::min<long>(units, (long)num_sms * per_sm);
  codes_kernel<C><<<(int)grid, kCodesThreads, smem, st>>>(tm, frames, prev_frame, t0, n, H, W, tiles_x, units,
                                                           tma ? 1 : 0, codes);
  SCPL_CHECK_LAUNCH();
}

void launch_codes(const uint8_t* frames, const uint8_t* prev_frame, int t0, int n, int H, int W, int C,
                  uint16_t* codes, int num_sms, cudaStream_t st) {
  if (n <= 0) return;
  if (C == 3)
    launch_codes_c<3>(frames, prev_frame, t0, n, H, W, codes, num_sms, st);
  else
    launch_codes_c<1>(frames, prev_frame, t0, n, H, W, codes, num_sms, st);
}

// ---------------------------------------------------------------- API-level kernels

// to_luma over npx pixels (energy.py:23-37)
__global__ void luma_kernel(const uint8_t* __restrict__ rgb, long npx, int C, uint8_t* __restrict__ out) {
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < npx; p += (long)gridDim.x * blockDim.x) {
    if (C == 3)
      out[p] = (uint8_t)luma_of(rgb[3 * p], rgb[3 * p + 1], rgb[3 * p + 2]);
    else
      out[p] = rgb[p * C];
  }
}

void launch_luma(const uint8_t* rgb, long npx, int C, uint8_t* out, cudaStream_t st) {
  if (npx <= 0) return;
  int blocks = (int)std::min<long>(cdiv(npx, 256), 148L * 16);
  luma_kernel<<<blocks, 256, 0, st>>>(rgb, npx, C, out);
  SCPL_CHECK_LAUNCH();
}

// decode codes -> float64 energy maps (motion_energy's return value)
__global__ void decode_kernel(const uint16_t* __restrict__ codes, long per_frame, int T, int first_pure,
                              double wm, double wg, double* __restrict__ out) {
  long n = per_frame * T;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
    uint32_t c = codes[p];
    bool pure = first_pure && p < per_frame;
    uint32_t g = c & 255u, d = c >> 8;
    double e;
    if (pure) {
      e = (double)g;
    } else {
      e = __dadd_rn(__dmul_rn(wm, (double)d), __dmul_rn(wg, (double)g));
      e = e <= 255.0 ? e : 255.0;
    }
    out[p] = e;
  }
}

void launch_decode(const uint16_t* codes, long per_frame, int T, int first_pure, double wm, double wg,
                   double* out, cudaStream_t st) {
  long n = per_frame * T;
  if (n <= 0) return;
  int blocks = (int)std::min<long>(cdiv(n, 256), 148L * 16);
  decode_kernel<<<blocks, 256, 0, st>>>(codes, per_frame, T, first_pure, wm, wg, out);
  SCPL_CHECK_LAUNCH();
}

// jitter (bench.py:39-57): per consecutive frame pair, the exact integer sum over pixels of
// |luma(t+1) - luma(t)| (the reference takes the float64 mean of these integers, which is
// exact up to the one division done on the host)
template <int C>
__global__ void jitter_sums_kernel(const uint8_t* __restrict__ frames, long npx, unsigned long long* __restrict__ sums) {
  const int t = blockIdx.y;
  const uint8_t* a = frames + (size_t)t * npx * C;
  const uint8_t* b = a + (size_t)npx * C;
  unsigned long long acc = 0;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < npx; p += (long)gridDim.x * blockDim.x) {
    int la, lb;
    if (C == 3) {
      la = (int)luma_of(a[3 * p], a[3 * p + 1], a[3 * p + 2]);
      lb = (int)luma_of(b[3 * p], b[3 * p + 1], b[3 * p + 2]);
    } else {
      la = a[p];
      lb = b[p];
    }
    acc += (unsigned long long)abs(lb - la);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&sums[t], acc);
}

void launch_jitter_sums(const uint8_t* frames, int T, long npx, int C, unsigned long long* sums, cudaStream_t st) {
  if (T < 2) return;
  SCPL_CUDA(cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * (T - 1), st));
  dim3 grid((unsigned)std::min<long>(cdiv(npx, 256), 256), T - 1);
  if (C == 3)
    jitter_sums_kernel<3><<<grid, 256, 0, st>>>(frames, npx, sums);
  else
    jitter_sums_kernel<1><<<grid, 256, 0, st>>>(frames, npx, sums);
  SCPL_CHECK_LAUNCH();
}

// gradient_energy of a luma plane, as float64 (API) -- energy.py:40-59
__global__ void sobel_f64_kernel(const uint8_t* __restrict__ luma, int H, int W, double* __restrict__ out) {
  long n = (long)H * W;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
    int i = (int)(p / W), j = (int)(p - (long)i * W);
    int im = max(i - 1, 0), ip = min(i + 1, H - 1), jm = max(j - 1, 0), jp = min(j + 1, W - 1);
    const uint8_t* a = luma + (long)im * W;
    const uint8_t* b = luma + (long)i * W;
    const uint8_t* c = luma + (long)ip * W;
    int gx = (a[jp] + 2 * b[jp] + c[jp]) - (a[jm] + 2 * b[jm] + c[jm]);
    int gy = (c[jm] + 2 * c[j] + c[jp]) - (a[jm] + 2 * a[j] + a[jp]);
    int g = abs(gx) + abs(gy);
    out[p] = (double)(g > 255 ? 255 : g);
  }
}

void launch_sobel_f64(const uint8_t* luma, int H, int W, double* out, cudaStream_t st) {
  long n = (long)H * W;
  if (n <= 0) return;
  int blocks = (int)std::min<long>(cdiv(n, 256), 148L * 16);
  sobel_f64_kernel<<<blocks, 256, 0, st>>>(luma, H, W, out);
  SCPL_CHECK_LAUNCH();
}

}  // namespace scpl
