// K1: per-frame energy codes (luma, Sobel gradient, motion difference).
//
// Replaces energy.py:23-37 (to_luma), :40-59 (gradient_energy), :62-87 (motion_energy).
// The fp64 motion energy is a pure function of two bytes per pixel:
//   e = min(fl(fl(wm*|dL|) + fl(wg*g)), 255)   (g = pure Sobel on the clip's first frame)
// so one streaming pass writes a 2-byte code (|dL| << 8 | g) per pixel and every later
// consumer (window statistics, uniform map) decodes e in registers.
//
// Layout: frames (T, H, W, C) uint8, row-major; codes (T, H, W) uint16.  A CTA owns a
// band of RB rows and walks a range of frames, keeping the previous frame's luma band in
// shared memory (the motion term needs luma(t-1)); the next frame's RGB band (+1 halo row
// each side) is prefetched with cp.async.bulk (TMA bulk copy) while the current one is
// processed.
#include "scpl_common.cuh"
#include "scpl_kernels.h"

namespace scpl {

struct CodesSmem {
  uint8_t* raw[2];
  uint8_t* lum[2];
  uint64_t* bar;
};

template <int C>
__device__ __forceinline__ void luma_band(const uint8_t* raw, uint8_t* lum, int rows, int W) {
  int n = rows * W;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    if (C == 3) {
      lum[p] = (uint8_t)luma_of(raw[3 * p], raw[3 * p + 1], raw[3 * p + 2]);
    } else {
      lum[p] = raw[p];
    }
  }
}

// Sobel (edge replicated) + |dL| for band rows 1..nrows of `lc` (rows 0 and nrows+1 are
// the halo); writes codes rows r0..r0+nrows-1.
__device__ __forceinline__ void codes_band(const uint8_t* lc, const uint8_t* lp, bool have_prev, int nrows,
                                           int W, uint16_t* out) {
  const int groups = (W + 7) >> 3;
  const int n = nrows * groups;
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    int k = q / groups + 1;
    int j0 = (q - (k - 1) * groups) << 3;
    const uint8_t* a = lc + (k - 1) * W;
    const uint8_t* b = lc + k * W;
    const uint8_t* c = lc + (k + 1) * W;
    uint16_t v[8];
    // column sums for j0-1 .. j0+8 (clamped)
    int cs[10], cd[10];
#pragma unroll
    for (int u = 0; u < 10; ++u) {
      int j = j0 - 1 + u;
      j = j < 0 ? 0 : (j > W - 1 ? W - 1 : j);
      int A = a[j], B = b[j], Cc = c[j];
      cs[u] = A + 2 * B + Cc;  // vertical [1,2,1]
      cd[u] = Cc - A;          // bottom - top
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      int j = j0 + u;
      if (j < W) {
        // right/left neighbours clamp at the border: u+2 maps to column min(j+1, W-1)
        int ur = (j + 1 <= W - 1) ? u + 2 : u + 1;
        int ul = (j - 1 >= 0) ? u : u + 1;
        int gx = cs[ur] - cs[ul];
        int gy = cd[ul] + 2 * cd[u + 1] + cd[ur];
        int g = abs(gx) + abs(gy);
        g = g > 255 ? 255 : g;
        int d = have_prev ? abs((int)b[j] - (int)lp[k * W + j]) : 0;
        v[u] = (uint16_t)((d << 8) | g);
      }
    }
    uint16_t* o = out + (size_t)(k - 1) * W + j0;
    if (j0 + 8 <= W && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
      uint4 pk;
      pk.x = v[0] | ((uint32_t)v[1] << 16);
      pk.y = v[2] | ((uint32_t)v[3] << 16);
      pk.z = v[4] | ((uint32_t)v[5] << 16);
      pk.w = v[6] | ((uint32_t)v[7] << 16);
      *reinterpret_cast<uint4*>(o) = pk;
    } else {
      for (int u = 0; u < 8 && j0 + u < W; ++u) o[u] = v[u];
    }
  }
}

template <int C>
__global__ void __launch_bounds__(256) codes_kernel(const uint8_t* __restrict__ frames,
                                                    const uint8_t* __restrict__ prev_frame, int T, int H,
                                                    int W, int RB, int fpg, int use_bulk,
                                                    uint16_t* __restrict__ codes) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int band = blockIdx.x;
  const int r0 = band * RB;
  const int nrows = min(RB, H - r0);
  const int t_begin = blockIdx.y * fpg;
  const int t_end = min(T, t_begin + fpg);
  if (t_begin >= T) return;
  const size_t row_bytes = (size_t)W * C;
  const size_t band_bytes = (size_t)(RB + 2) * row_bytes;
  const size_t frame_bytes = (size_t)H * row_bytes;

  CodesSmem s;
  s.raw[0] = smem;
  s.raw[1] = smem + band_bytes;
  s.lum[0] = smem + 2 * band_bytes;
  s.lum[1] = s.lum[0] + (size_t)(RB + 2) * W;
  s.bar = reinterpret_cast<uint64_t*>(s.lum[1] + (((size_t)(RB + 2) * W + 15) & ~(size_t)15));

  // sequence q = 0 is the previous frame (may be absent), q >= 1 is frame t_begin + q - 1
  const bool have_prev0 = (t_begin > 0) || (prev_frame != nullptr);
  auto src_of = [&](int q) -> const uint8_t* {
    if (q == 0) return t_begin > 0 ? frames + (size_t)(t_begin - 1) * frame_bytes : prev_frame;
    return frames + (size_t)(t_begin + q - 1) * frame_bytes;
  };
  const int q_first = have_prev0 ? 0 : 1;
  const int q_last = t_end - t_begin;  // inclusive

  auto issue = [&](int q, int slot) {
    // one bulk copy per band row (+ halo), rows clamped at the frame borders
    const uint8_t* src = src_of(q);
    if (threadIdx.x == 0) {
      fence_proxy_async();
      mbar_arrive_tx(&s.bar[slot], (uint32_t)((nrows + 2) * row_bytes));
      for (int k = 0; k < nrows + 2; ++k) {
        int r = r0 - 1 + k;
        r = r < 0 ? 0 : (r > H - 1 ? H - 1 : r);
        bulk_g2s(s.raw[slot] + k * row_bytes, src + (size_t)r * row_bytes, (uint32_t)row_bytes, &s.bar[slot]);
      }
    }
  };
  auto load_plain = [&](int q, int slot) {
    const uint8_t* src = src_of(q);
    const int n = (nrows + 2) * (int)row_bytes;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      int k = p / (int)row_bytes, o = p - k * (int)row_bytes;
      int r = r0 - 1 + k;
      r = r < 0 ? 0 : (r > H - 1 ? H - 1 : r);
      s.raw[slot][p] = src[(size_t)r * row_bytes + o];
    }
  };

  if (use_bulk) {
    if (threadIdx.x == 0) {
      mbar_init(&s.bar[0], 1);
      mbar_init(&s.bar[1], 1);
      fence_mbar_init();
    }
    __syncthreads();
    issue(q_first, q_first & 1);
  }
  uint32_t phase[2] = {0, 0};
  int cur = 0;  // lum buffer holding the most recent luma band
  for (int q = q_first; q <= q_last; ++q) {
    const int slot = q & 1;
    if (use_bulk) {
      if (q + 1 <= q_last) issue(q + 1, (q + 1) & 1);
      mbar_wait(&s.bar[slot], phase[slot]);
      phase[slot] ^= 1;
    } else {
      load_plain(q, slot);
      __syncthreads();
    }
    const int nxt = cur ^ 1;
    luma_band<C>(s.raw[slot], s.lum[nxt], nrows + 2, W);
    __syncthreads();
    if (q >= 1) {
      const int t = t_begin + q - 1;
      bool have_prev = (q > 1) || have_prev0;
      codes_band(s.lum[nxt], s.lum[cur], have_prev, nrows, W, codes + ((size_t)t * H + r0) * W);
    }
    cur = nxt;
    __syncthreads();  // raw[slot] and lum[cur^1] free for reuse
  }
}

void launch_codes(const uint8_t* frames, const uint8_t* prev_frame, int T, int H, int W, int C,
                  uint16_t* codes, int num_sms, cudaStream_t st) {
  if (T <= 0) return;
  const int RB = 4;
  const size_t row_bytes = (size_t)W * C;
  bool bulk = (row_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(frames) & 15) == 0) &&
              (prev_frame == nullptr || (reinterpret_cast<uintptr_t>(prev_frame) & 15) == 0);
  size_t lum_bytes = (((size_t)(RB + 2) * W + 15) & ~(size_t)15);
  size_t smem = 2 * (size_t)(RB + 2) * row_bytes + 2 * lum_bytes + 16;
  SCPL_ARG(smem <= 227 * 1024, "frame too wide for the energy kernel's shared-memory band");
  int bands = cdiv(H, RB);
  int per_sm = (int)((228 * 1024) / (smem + 1024));
  per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);
  int slots = num_sms * per_sm;
  int groups = slots / bands;
  if (groups < 1) groups = 1;
  if (groups > (T + 7) / 8) groups = (T + 7) / 8;
  if (groups < 1) groups = 1;
  int fpg = cdiv(T, groups);
  groups = cdiv(T, fpg);
  dim3 grid(bands, groups);
  if (C == 3) {
    SCPL_CUDA(cudaFuncSetAttribute(codes_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    codes_kernel<3><<<grid, 256, smem, st>>>(frames, prev_frame, T, H, W, RB, fpg, bulk ? 1 : 0, codes);
  } else {
    SCPL_CUDA(cudaFuncSetAttribute(codes_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    codes_kernel<1><<<grid, 256, smem, st>>>(frames, prev_frame, T, H, W, RB, fpg, bulk ? 1 : 0, codes);
  }
  SCPL_CHECK_LAUNCH();
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
