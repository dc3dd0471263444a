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
constexpr int kLumW = kCW + 8;          // luma columns: c0-4 .. c0+131
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

// luma of raw tile -> lum[kCRows][kLumStride], replicating the frame border
template <int C>
__device__ __forceinline__ void codes_luma(const uint8_t* raw, uint8_t* lum, int r0, int c0, int H, int W) {
  constexpr int kGroups = kLumW / 4;  // 34 groups of 4 luma columns per row
  for (int q = threadIdx.x; q < kCRows * kGroups; q += kCodesThreads) {
    const int k = q / kGroups, g = q - k * kGroups;
    const int gr = min(max(r0 - 1 + k, 0), H - 1);  // clamped frame row
    const int rk = gr - (r0 - 1);                   // its raw row
    const int px0 = c0 - 4 + 4 * g;                 // first pixel of the group
    uint32_t word;
    if (px0 >= 0 && px0 + 3 < W) {
      const int x = (px0 - (c0 - 16)) * C;  // 4-byte aligned, never straddles a box
      const uint32_t* src = reinterpret_cast<const uint32_t*>(raw + raw_off<C>(rk, x));
      if (C == 3) {
        const uint32_t a = src[0], b = src[1], c = src[2];
        const uint32_t l0 = luma_of(a & 255u, (a >> 8) & 255u, (a >> 16) & 255u);
        const uint32_t l1 = luma_of(a >> 24, b & 255u, (b >> 8) & 255u);
        const uint32_t l2 = luma_of((b >> 16) & 255u, b >> 24, c & 255u);
        const uint32_t l3 = luma_of((c >> 8) & 255u, (c >> 16) & 255u, c >> 24);
        word = l0 | (l1 << 8) | (l2 << 16) | (l3 << 24);
      } else {
        word = src[0];
      }
    } else {  // frame border: clamped columns
      word = 0;
      for (int u = 0; u < 4; ++u) {
        const int px = min(max(px0 + u, 0), W - 1);
        const int x = (px - (c0 - 16)) * C;
        uint32_t l;
        if (px - (c0 - 16) < 0 || px - (c0 - 16) >= kRawPx) {
          l = 0;  // outside the loaded box: never read by an in-frame output
        } else if (C == 3) {
          l = luma_of(raw[raw_off<C>(rk, x)], raw[raw_off<C>(rk, x + 1)], raw[raw_off<C>(rk, x + 2)]);
        } else {
          l = raw[raw_off<C>(rk, x)];
        }
        word |= l << (8 * u);
      }
    }
    *reinterpret_cast<uint32_t*>(lum + k * kLumStride + 4 * g) = word;
  }
}

// codes of one frame for this thread's 4 rows x 4 columns; prev[i] = previous luma word
__device__ __forceinline__ void codes_tile(const uint8_t* lum, uint32_t (&prev)[4], bool emit, bool have_prev,
                                           int r0, int c0, int H, int W, uint16_t* __restrict__ out,
                                           bool vec_out) {
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  int v[6][6];  // [lum row 4wy .. 4wy+5][col -1 .. 4]
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const uint32_t* row = reinterpret_cast<const uint32_t*>(lum + (4 * wy + k) * kLumStride);
    const uint32_t lo = row[lane], mid = row[lane + 1], hi = row[lane + 2];
    v[k][0] = lo >> 24;
    v[k][1] = mid & 255;
    v[k][2] = (mid >> 8) & 255;
    v[k][3] = (mid >> 16) & 255;
    v[k][4] = mid >> 24;
    v[k][5] = hi & 255;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int cs[6], cd[6];
#pragma unroll
    for (int u = 0; u < 6; ++u) {
      cs[u] = v[i][u] + 2 * v[i + 1][u] + v[i + 2][u];
      cd[u] = v[i + 2][u] - v[i][u];
    }
    const uint32_t cur = (uint32_t)v[i + 1][1] | ((uint32_t)v[i + 1][2] << 8) | ((uint32_t)v[i + 1][3] << 16) |
                         ((uint32_t)v[i + 1][4] << 24);
    uint32_t code[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int gx = cs[u + 2] - cs[u];
      const int gy = cd[u] + 2 * cd[u + 1] + cd[u + 2];
      const int g = min(abs(gx) + abs(gy), 255);
      const int d = have_prev ? abs(v[i + 1][u + 1] - (int)((prev[i] >> (8 * u)) & 255u)) : 0;
      code[u] = ((uint32_t)d << 8) | (uint32_t)g;
    }
    prev[i] = cur;
    const int r = r0 + 4 * wy + i, c = c0 + 4 * lane;
    if (emit && r < H) {
      uint16_t* o = out + (size_t)r * W + c;
      if (vec_out && c + 3 < W) {
        *reinterpret_cast<uint2*>(o) = make_uint2(code[0] | (code[1] << 16), code[2] | (code[3] << 16));
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c + u < W) o[u] = (uint16_t)code[u];
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
  uint8_t* lum = smem + 2 * G::kSlot;
  uint64_t* bar = reinterpret_cast<uint64_t*>(lum + kCRows * kLumStride);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const bool vec_out = (W & 3) == 0;
  const size_t fpx = (size_t)H * W;
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
    fill(q0, seq);
    for (int q = q0; q <= q1; ++q, ++seq) {
      if (q + 1 <= q1) fill(q + 1, seq + 1);  // the slot was released by the sync ending frame q-1
      if (tma_slot(q)) {
        mbar_wait(&bar[seq & 1], (phase >> (seq & 1)) & 1u);
        phase ^= 1u << (seq & 1);
      }
      __syncthreads();  // plain fills visible
      codes_luma<C>(raw(seq), lum, r0, c0, H, W);
      __syncthreads();
      const int t = tb + q - 1;
      codes_tile(lum, prev, q >= 1, q > 1 || have_prev0, r0, c0, H, W, codes + (size_t)t * fpx, vec_out);
      __syncthreads();  // lum and raw(seq) free
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
  const size_t smem = 2 * (size_t)G::kSlot + (size_t)kCRows * kLumStride + 16;
  const int tiles_x = cdiv(W, kCW), tiles = tiles_x * cdiv(H, kCH);
  const long units = (long)tiles * n;
  int per_sm = 0;
  SCPL_CUDA(cudaFuncSetAttribute(codes_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SCPL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, codes_kernel<C>, kCodesThreads, smem));
  if (per_sm < 1) per_sm = 1;
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
