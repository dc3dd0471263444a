// K8: replay a run's batches on every frame of the run.
//
// Replaces replay_batches (pipeline.py:140-154), which calls remove_batch once per frame
// per batch (75% of the reference's buffered wall time).  Within a batch the removed
// columns address the frame the batch was selected on, so replaying all batches equals
// one gather through the composed original-column index map; one pass per frame reads
// H*W*C bytes and writes H*W'*C bytes.
//
// Width phase: out[t][i][y] = in[t][i][idx[i][y]] -- a CTA stages input rows in shared
// memory with 16-byte loads, gathers, and writes the output rows with 16-byte stores.
// Height phase (carve on the transposed frame): out[t][y][j] = in[t][idx[j][y]][j] --
// 32x32 tiles of the index map are transposed through shared memory so both the index
// reads and the pixel writes are coalesced.
#include <algorithm>

#include "scpl_common.cuh"
#include "scpl_kernels.h"

namespace scpl {

constexpr int kReplayRows = 4;

template <int C>
__global__ void __launch_bounds__(256) replay_rows_kernel(const uint8_t* __restrict__ in,
                                                          uint8_t* __restrict__ out, int H, int W,
                                                          const int16_t* __restrict__ idx, int stride, int tw,
                                                          int vec) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* rin = smem;
  uint8_t* rout = smem + (((size_t)W * C + 15) & ~(size_t)15);
  const int t = blockIdx.y;
  const size_t in_row = (size_t)W * C, out_row = (size_t)tw * C;
  for (int rr = 0; rr < kReplayRows; ++rr) {
    const int i = blockIdx.x * kReplayRows + rr;
    if (i >= H) break;
    const uint8_t* src = in + ((size_t)t * H + i) * in_row;
    uint8_t* dst = out + ((size_t)t * H + i) * out_row;
    if (vec) {
      for (size_t q = threadIdx.x; q < in_row / 16; q += blockDim.x)
        reinterpret_cast<uint4*>(rin)[q] = reinterpret_cast<const uint4*>(src)[q];
    } else {
      for (size_t q = threadIdx.x; q < in_row; q += blockDim.x) rin[q] = src[q];
    }
    __syncthreads();
    const int16_t* ir = idx + (size_t)i * stride;
    for (int y = threadIdx.x; y < tw; y += blockDim.x) {
      int s = ir[y];
      SCPL_DCHECK(s >= 0 && s < W, "replay index inside the row");
#pragma unroll
      for (int c = 0; c < C; ++c) rout[y * C + c] = rin[s * C + c];
    }
    __syncthreads();
    if (vec) {
      for (size_t q = threadIdx.x; q < out_row / 16; q += blockDim.x)
        reinterpret_cast<uint4*>(dst)[q] = reinterpret_cast<const uint4*>(rout)[q];
    } else {
      for (size_t q = threadIdx.x; q < out_row; q += blockDim.x) dst[q] = rout[q];
    }
    __syncthreads();
  }
}

// Width phase, vectorised (W*C and tw*C multiples of 16): the index row is the same for every
// frame of the run, so a CTA owns one row i for all the run's frames.  Each thread owns 16
// consecutive output pixels, keeps their 16 source columns in registers, and per frame gathers
// 16*C bytes from the staged input row into registers and writes them with 16-byte stores.
// Input rows arrive by 1-D bulk copies (TMA) into a kRing-slot ring, kRing-1 frames ahead.
constexpr int kRing = 4;  // 3 frames ahead: a short run's rows are all in flight at once
constexpr int kRpPx = 16;  // output pixels per thread

template <int C>
__global__ void __launch_bounds__(128) replay_rows_vec_kernel(const uint8_t* __restrict__ in,
                                                              uint8_t* __restrict__ out, int T, int H, int W,
                                                              const int16_t* __restrict__ idx, int stride, int tw) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[kRing];
  const int i = blockIdx.x;
  const int tid = threadIdx.x;
  const uint32_t in_row = (uint32_t)W * C;
  const size_t out_row = (size_t)tw * C;
  const uint32_t slot = (in_row + 127) & ~127u;
  if (tid == 0) {
    for (int k = 0; k < kRing; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
    for (int t = 0; t < kRing - 1 && t < T; ++t) {
      mbar_arrive_tx(&bar[t], in_row);
      bulk_g2s(smem + (size_t)t * slot, in + ((size_t)t * H + i) * in_row, in_row, &bar[t]);
    }
  }
  // this thread's source columns (byte offsets in the staged row)
  const int y0 = tid * kRpPx;
  const bool active = y0 < tw;
  int src[kRpPx];
  if (active && y0 + kRpPx <= tw && (stride & 7) == 0) {  // two 16-byte loads of the index row
    const uint4* ip = reinterpret_cast<const uint4*>(idx + (size_t)i * stride + y0);
    const uint4 a = __ldg(ip), b = __ldg(ip + 1);
    const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < kRpPx; ++k) src[k] = (int)(int16_t)(wv[k >> 1] >> (16 * (k & 1))) * C;
  } else {
#pragma unroll
    for (int k = 0; k < kRpPx; ++k) src[k] = active && y0 + k < tw ? (int)idx[(size_t)i * stride + y0 + k] * C : 0;
  }
#pragma unroll
  for (int k = 0; k < kRpPx; ++k)
    SCPL_DCHECK(src[k] >= 0 && src[k] < W * C && (k == 0 || y0 + k >= tw || src[k] > src[k - 1]),
                "replay index map strictly increasing inside the row");
  __syncthreads();
  for (int t = 0; t < T; ++t) {
    const int sl = t % kRing;
    if (tid == 0 && t + kRing - 1 < T) {  // the slot of frame t-1 is free: every thread passed its gather
      const int tn = t + kRing - 1, sn = tn % kRing;
      fence_proxy_async();  // (the generic reads of that slot before the async refill)
      mbar_arrive_tx(&bar[sn], in_row);
      bulk_g2s(smem + (size_t)sn * slot, in + ((size_t)tn * H + i) * in_row, in_row, &bar[sn]);
    }
    mbar_wait(&bar[sl], (uint32_t)((t / kRing) & 1));
    const uint8_t* row = smem + (size_t)sl * slot;
    if (active) {
      uint32_t wv[kRpPx * C / 4];
#pragma unroll
      for (int w = 0; w < kRpPx * C / 4; ++w) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int byte = 4 * w + b, k = byte / C, c = byte - k * C;
          v |= (uint32_t)row[src[k] + c] << (8 * b);
        }
        wv[w] = v;
      }
      uint4* dst = reinterpret_cast<uint4*>(out + ((size_t)t * H + i) * out_row + (size_t)y0 * C);
      const int nvec = min(kRpPx, tw - y0) * C / 16;  // (tw*C is a multiple of 16; y0*C too)
#pragma unroll
      for (int v = 0; v < kRpPx * C / 16; ++v)
        if (v < nvec) __stcs(dst + v, make_uint4(wv[4 * v], wv[4 * v + 1], wv[4 * v + 2], wv[4 * v + 3]));
    }
    __syncthreads();  // slot sl is read by everyone before it is refilled (frame t + kRing)
  }
}

template <int C>
__global__ void replay_cols_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int H, int W,
                                   const int16_t* __restrict__ idx, int stride, int th) {
  __shared__ int16_t tile[32][33];
  const int t = blockIdx.z;
  const int j0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  // idx is (W, stride): carve row j = original column j, entries = original rows
  for (int r = threadIdx.y; r < 32; r += 8) {
    int j = j0 + r, y = y0 + threadIdx.x;
    tile[r][threadIdx.x] = (j < W && y < th) ? idx[(size_t)j * stride + y] : (int16_t)0;
  }
  __syncthreads();
  const uint8_t* src = in + (size_t)t * H * W * C;
  uint8_t* dst = out + (size_t)t * th * W * C;
  for (int r = threadIdx.y; r < 32; r += 8) {
    int y = y0 + r, j = j0 + threadIdx.x;
    if (y < th && j < W) {
      int s = tile[threadIdx.x][r];
#pragma unroll
      for (int c = 0; c < C; ++c) dst[((size_t)y * W + j) * C + c] = src[((size_t)s * W + j) * C + c];
    }
  }
}

void launch_replay(const uint8_t* in, uint8_t* out, int T, int H, int W, int C, const int16_t* idx, int stride,
                   int target, int transposed, cudaStream_t st) {
  if (T <= 0) return;
  if (!transposed) {
    bool vec = ((size_t)W * C % 16 == 0) && ((size_t)target * C % 16 == 0) &&
               ((reinterpret_cast<uintptr_t>(in) & 15) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    size_t smem = (((size_t)W * C + 15) & ~(size_t)15) + (size_t)target * C + 16;
    SCPL_ARG(smem <= 227 * 1024, "frame too wide for the replay kernel");
    // (kRpPx pixels per thread: C*16 bytes, whole 16-byte stores when tw*C % 16 == 0; at most
    // 128 threads, so widths <= 2048 output pixels)
    if (vec && target <= 128 * kRpPx && (size_t)kRing * (((size_t)W * C + 127) & ~(size_t)127) <= 200 * 1024) {
      const size_t rs = (size_t)kRing * (((size_t)W * C + 127) & ~(size_t)127);
      const int threads = std::max(32, (cdiv(target, kRpPx) + 31) / 32 * 32);
      if (C == 3) {
        smem_optin(reinterpret_cast<const void*>(replay_rows_vec_kernel<3>));
        replay_rows_vec_kernel<3><<<H, threads, rs, st>>>(in, out, T, H, W, idx, stride, target);
      } else {
        smem_optin(reinterpret_cast<const void*>(replay_rows_vec_kernel<1>));
        replay_rows_vec_kernel<1><<<H, threads, rs, st>>>(in, out, T, H, W, idx, stride, target);
      }
      SCPL_CHECK_LAUNCH();
      return;
    }
    dim3 grid(cdiv(H, kReplayRows), T);
    if (C == 3) {
      smem_optin(reinterpret_cast<const void*>(replay_rows_kernel<3>));
      replay_rows_kernel<3><<<grid, 256, smem, st>>>(in, out, H, W, idx, stride, target, vec ? 1 : 0);
    } else {
      smem_optin(reinterpret_cast<const void*>(replay_rows_kernel<1>));
      replay_rows_kernel<1><<<grid, 256, smem, st>>>(in, out, H, W, idx, stride, target, vec ? 1 : 0);
    }
  } else {
    dim3 grid(cdiv(W, 32), cdiv(target, 32), T);
    if (C == 3)
      replay_cols_kernel<3><<<grid, dim3(32, 8), 0, st>>>(in, out, H, W, idx, stride, target);
    else
      replay_cols_kernel<1><<<grid, dim3(32, 8), 0, st>>>(in, out, H, W, idx, stride, target);
  }
  SCPL_CHECK_LAUNCH();
}

}  // namespace scpl
