// K4-K7: the SCPL carve loop of every run, batched across runs.
//
// Replaces batch_carve (batching.py:118-153) and what it calls: cumulative_energy
// (seams.py:39-65), label_parents (batching.py:39-46), select_batch (:49-73),
// trace_columns (seams.py:68-81), remove_batch on the representative frame (:76-107) and
// default_energy (:110-115).  One host iteration = one DP pass of every active run:
//
//   gradient  (all runs, all pixels)  Sobel of the compacted luma plane        [parallel]
//   dp        (one CTA per run)       row-sequential min/argmin, leftmost tie  [row chain]
//                                     break, 2-bit back codes folded into one
//                                     32-bit path word per column every 16 rows
//   select    (one CTA per run)       labels by chaining block landing deltas,
//                                     per-parent leftmost min (labels are
//                                     monotone, so segments), k-truncation by
//                                     (cost, col), trace by decoding path words
//   compact   (one warp per row)      remove the batch's columns from luma and
//                                     the composed original-column index map   [parallel]
//
// The first pass of a buffered run runs on the fp64 uniform map (fp64 DP, IEEE adds,
// no contraction); every later pass on integer gradient energy, where an int32 DP is
// bit-identical to the reference's float64 one (values are integers < 2^31).
#include <cfloat>

#include "scpl_common.cuh"
#include "scpl_kernels.h"

namespace scpl {

constexpr int kDpThreads = 1024;
constexpr int kDpCols = 4;  // columns per thread => max width 4096

// ------------------------------------------------------------------ setup
__global__ void setup_luma_kernel(const uint8_t* __restrict__ frame, int H, int W, int C, int transposed,
                                  uint8_t* __restrict__ luma, int16_t* __restrict__ idx) {
  __shared__ uint8_t tile[32][33];
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    int i = i0 + r, j = j0 + threadIdx.x;
    uint8_t v = 0;
    if (i < H && j < W) {
      const uint8_t* px = frame + ((long)i * W + j) * C;
      v = C == 3 ? (uint8_t)luma_of(px[0], px[1], px[2]) : px[0];
      if (!transposed) {
        luma[(long)i * W + j] = v;
        idx[(long)i * W + j] = (int16_t)j;
      }
    }
    tile[r][threadIdx.x] = v;
  }
  if (!transposed) return;
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    int j = j0 + r, i = i0 + threadIdx.x;  // carve row j, carve col i
    if (i < H && j < W) {
      luma[(long)j * H + i] = tile[threadIdx.x][r];
      idx[(long)j * H + i] = (int16_t)i;
    }
  }
}

void launch_carve_setup_luma(const uint8_t* frame, int H, int W, int C, int transposed, uint8_t* luma,
                             int16_t* idx, cudaStream_t st) {
  dim3 grid(cdiv(W, 32), cdiv(H, 32));
  setup_luma_kernel<<<grid, dim3(32, 8), 0, st>>>(frame, H, W, C, transposed, luma, idx);
  SCPL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ gradient
// default_energy (batching.py:110-115) on the compacted plane: Sobel with edge
// replication inside [0,rows) x [0,width); zero map when either side is < 3.
__global__ void carve_gradient_kernel(RunCarve* __restrict__ runs, int first_iter) {
  RunCarve& R = runs[blockIdx.z];
  if (R.done) return;
  if (first_iter && R.U != nullptr) return;  // first pass runs on the fp64 map
  const int i = blockIdx.y;
  const int rows = R.rows, w = R.width, stride = R.stride;
  if (i >= rows) return;
  const bool zero = rows < 3 || w < 3;
  const uint8_t* a = R.luma + (long)max(i - 1, 0) * stride;
  const uint8_t* b = R.luma + (long)i * stride;
  const uint8_t* c = R.luma + (long)min(i + 1, rows - 1) * stride;
  uint8_t* out = R.grad + (long)i * stride;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < w; j += gridDim.x * blockDim.x) {
    int g = 0;
    if (!zero) {
      int jm = max(j - 1, 0), jp = min(j + 1, w - 1);
      int gx = (a[jp] + 2 * b[jp] + c[jp]) - (a[jm] + 2 * b[jm] + c[jm]);
      int gy = (c[jm] + 2 * c[j] + c[jp]) - (a[jm] + 2 * a[j] + a[jp]);
      g = abs(gx) + abs(gy);
      g = g > 255 ? 255 : g;
    }
    out[j] = (uint8_t)g;
  }
}

void launch_carve_gradient(RunCarve* runs, int nruns, int max_rows, int max_stride, int first_iter,
                           cudaStream_t st) {
  dim3 grid(cdiv(max_stride, 256), max_rows, nruns);
  carve_gradient_kernel<<<grid, 256, 0, st>>>(runs, first_iter);
  SCPL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ DP
template <bool F64>
struct DpT;
template <>
struct DpT<true> {
  using V = double;
  static __device__ __forceinline__ V inf() { return __longlong_as_double(0x7ff0000000000000ll); }
  static __device__ __forceinline__ V load(const RunCarve& R, long p) { return R.U[p]; }
  static __device__ __forceinline__ V add(V a, V b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double out(V v) { return v; }
};
template <>
struct DpT<false> {
  using V = int;
  static __device__ __forceinline__ V inf() { return 0x7fffffff; }
  static __device__ __forceinline__ V load(const RunCarve& R, long p) { return (int)R.grad[p]; }
  static __device__ __forceinline__ V add(V a, V b) { return a + b; }
  static __device__ __forceinline__ double out(V v) { return (double)v; }
};

template <bool F64>
__global__ void __launch_bounds__(kDpThreads) carve_dp_kernel(RunCarve* __restrict__ runs) {
  using T = DpT<F64>;
  using V = typename T::V;
  RunCarve& R = runs[blockIdx.x];
  if (R.done) return;
  // the fp64 pass is only the first pass of a run that has a uniform map
  if (F64 != (R.U != nullptr && R.iters == 0)) return;
  extern __shared__ __align__(16) uint8_t smem[];
  const int w = R.width, rows = R.rows, stride = R.stride;
  V* ce[2] = {reinterpret_cast<V*>(smem), reinterpret_cast<V*>(smem) + stride};
  uint32_t* pb[2] = {reinterpret_cast<uint32_t*>(smem + 2 * sizeof(V) * stride),
                     reinterpret_cast<uint32_t*>(smem + 2 * sizeof(V) * stride) + stride};
  const int tid = threadIdx.x;
  V e_nx[kDpCols];
#pragma unroll
  for (int k = 0; k < kDpCols; ++k) {
    int j = tid + k * kDpThreads;
    if (j < w) ce[0][j] = T::load(R, j);
    e_nx[k] = (j < w && rows > 1) ? T::load(R, (long)stride + j) : V(0);
  }
  __syncthreads();
  for (int i = 1; i < rows; ++i) {
    V e_cur[kDpCols];
#pragma unroll
    for (int k = 0; k < kDpCols; ++k) {
      int j = tid + k * kDpThreads;
      e_cur[k] = e_nx[k];
      e_nx[k] = (j < w && i + 1 < rows) ? T::load(R, (long)(i + 1) * stride + j) : V(0);
    }
    const V* prv = ce[(i - 1) & 1];
    V* cur = ce[i & 1];
    const uint32_t* pprv = pb[(i - 1) & 1];
    uint32_t* pcur = pb[i & 1];
    const int within = (i - 1) & (kBlockRows - 1);
    const int blk = (i - 1) / kBlockRows;
    const bool bstart = within == 0;
    const bool bend = within == kBlockRows - 1 || i == rows - 1;
#pragma unroll
    for (int k = 0; k < kDpCols; ++k) {
      int j = tid + k * kDpThreads;
      if (j < w) {
        V l = j > 0 ? prv[j - 1] : T::inf();
        V c = prv[j];
        V r = j + 1 < w ? prv[j + 1] : T::inf();
        uint32_t code = 0;
        V m = l;
        if (c < m) { m = c; code = 1; }   // strict: the smaller delta wins ties (seams.py:62)
        if (r < m) { m = r; code = 2; }
        cur[j] = T::add(e_cur[k], m);
        uint32_t po = bstart ? 0u : pprv[j - 1 + (int)code];
        uint32_t pn = (po << 2) | code;
        pcur[j] = pn;
        if (bend) {
          int sum = __popc(pn & 0x55555555u) + 2 * __popc(pn & 0xAAAAAAAAu);
          R.pw[(long)blk * stride + j] = pn;
          R.delta[(long)blk * stride + j] = (int8_t)(sum - (within + 1));
        }
      }
    }
    __syncthreads();
  }
  const V* last = ce[(rows - 1) & 1];
#pragma unroll
  for (int k = 0; k < kDpCols; ++k) {
    int j = tid + k * kDpThreads;
    if (j < w) R.lastce[j] = T::out(last[j]);
  }
}

void launch_carve_dp(RunCarve* runs, int nruns, bool fp64, int max_stride, cudaStream_t st) {
  SCPL_ARG(max_stride <= kDpThreads * kDpCols, "carve width above 4096 is not supported");
  if (fp64) {
    size_t smem = 2 * sizeof(double) * max_stride + 2 * sizeof(uint32_t) * max_stride;
    SCPL_CUDA(cudaFuncSetAttribute(carve_dp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    carve_dp_kernel<true><<<nruns, kDpThreads, smem, st>>>(runs);
  } else {
    size_t smem = 2 * sizeof(int) * max_stride + 2 * sizeof(uint32_t) * max_stride;
    SCPL_CUDA(cudaFuncSetAttribute(carve_dp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    carve_dp_kernel<false><<<nruns, kDpThreads, smem, st>>>(runs);
  }
  SCPL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ select + trace
// exclusive block scan over 1024 threads (one value each); returns the total
__device__ int block_scan_excl(int v, int* warp_sums, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = (lane < (int)(blockDim.x >> 5)) ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_sums[lane] = s;  // inclusive
  }
  __syncthreads();
  int base = wid > 0 ? warp_sums[wid - 1] : 0;
  total = warp_sums[(blockDim.x >> 5) - 1];
  __syncthreads();
  return base + x - v;
}

constexpr int kSelThreads = 1024;

__global__ void __launch_bounds__(kSelThreads) carve_select_kernel(RunCarve* __restrict__ runs) {
  RunCarve& R = runs[blockIdx.x];
  if (R.done) {
    if (threadIdx.x == 0) R.b = 0;
    return;
  }
  extern __shared__ __align__(16) uint8_t smem[];
  const int w = R.width, rows = R.rows, stride = R.stride;
  const int nblk = (rows - 1 + kBlockRows - 1) / kBlockRows;
  double* lce = reinterpret_cast<double*>(smem);                 // w
  unsigned long long* segmin = reinterpret_cast<unsigned long long*>(lce + stride);  // w
  int* lab = reinterpret_cast<int*>(segmin + stride);            // w
  int* segarg = lab + stride;                                     // w
  int* cand = segarg + stride;                                    // w
  int* sel = cand + stride;                                       // w
  __shared__ int warp_sums[32];
  __shared__ int s_P, s_b;
  __shared__ double s_bestv;
  __shared__ int s_bestc;
  const int tid = threadIdx.x;

  for (int j = tid; j < w; j += kSelThreads) {
    lce[j] = R.lastce[j];
    segmin[j] = ~0ull;
    segarg[j] = INT_MAX;
  }
  // labels (batching.py:39-46) by chaining block landing deltas bottom-up, recording the
  // block-end column of every last-row column's path for the trace
  for (int j = tid; j < w; j += kSelThreads) {
    int c = j;
    for (int b = nblk - 1; b >= 0; --b) {
      R.col_end[(long)b * stride + j] = (int16_t)c;
      c += R.delta[(long)b * stride + c];
    }
    lab[j] = c;
  }
  __syncthreads();

  int b;
  if (R.kmax == 1) {
    // min_seam (seams.py:84-89): leftmost global minimum
    if (tid == 0) {
      s_bestv = DBL_MAX;
      s_bestc = INT_MAX;
    }
    __syncthreads();
    for (int j = tid; j < w; j += kSelThreads)
      atomicMin(&segmin[0], (unsigned long long)__double_as_longlong(lce[j]));
    __syncthreads();
    for (int j = tid; j < w; j += kSelThreads)
      if ((unsigned long long)__double_as_longlong(lce[j]) == segmin[0]) atomicMin(&segarg[0], j);
    __syncthreads();
    if (tid == 0) sel[0] = segarg[0];
    b = 1;
  } else {
    // per-parent leftmost strict minimum (batching.py:59-64); doubles >= 0 order as u64
    for (int j = tid; j < w; j += kSelThreads)
      atomicMin(&segmin[lab[j]], (unsigned long long)__double_as_longlong(lce[j]));
    __syncthreads();
    for (int j = tid; j < w; j += kSelThreads)
      if ((unsigned long long)__double_as_longlong(lce[j]) == segmin[lab[j]]) atomicMin(&segarg[lab[j]], j);
    __syncthreads();
    // candidates in label order == column order
    const int per = (w + kSelThreads - 1) / kSelThreads;
    int cnt = 0;
    for (int u = 0; u < per; ++u) {
      int l = tid * per + u;
      if (l < w && segarg[l] != INT_MAX) ++cnt;
    }
    int tot;
    int pos = block_scan_excl(cnt, warp_sums, tot);
    for (int u = 0; u < per; ++u) {
      int l = tid * per + u;
      if (l < w && segarg[l] != INT_MAX) cand[pos++] = segarg[l];
    }
    const int P = tot;
    const int k = w - R.target;
    __syncthreads();
    if (P <= k) {
      for (int q = tid; q < P; q += kSelThreads) sel[q] = cand[q];
      b = P;
    } else {
      // keep the k cheapest by (cost, col) (batching.py:66-68), then back to column order
      const int perq = (P + kSelThreads - 1) / kSelThreads;
      int keep = 0;
      for (int u = 0; u < perq; ++u) {
        int q = tid * perq + u;
        if (q < P) {
          double cq = lce[cand[q]];
          int rank = 0;
          for (int o = 0; o < P; ++o) {
            double co = lce[cand[o]];
            rank += (co < cq) || (co == cq && o < q);
          }
          if (rank < k) keep |= 1 << u;
        }
      }
      int kc = __popc(keep);
      int tot2;
      int p2 = block_scan_excl(kc, warp_sums, tot2);
      for (int u = 0; u < perq; ++u)
        if (keep >> u & 1) sel[p2++] = cand[tid * perq + u];
      b = k;
    }
  }
  __syncthreads();

  // trace (seams.py:68-81): decode each selected seam's path word per block
  const int bnb = b * nblk;
  for (int q = tid; q < bnb; q += kSelThreads) {
    int s = q / nblk, blk = q - s * nblk;
    int c = R.col_end[(long)blk * stride + sel[s]];
    uint32_t pw = R.pw[(long)blk * stride + c];
    int i_start = 1 + blk * kBlockRows;
    int i_end = min(i_start + kBlockRows, rows) - 1;
    for (int i = i_end; i >= i_start; --i) {
      R.rem[(long)i * b + s] = (int16_t)c;
      c += (int)(pw & 3u) - 1;
      pw >>= 2;
    }
  }
  for (int s = tid; s < b; s += kSelThreads) R.rem[s] = (int16_t)lab[sel[s]];  // row 0
  if (R.dbg_sizes != nullptr) {
    for (int s = tid; s < b; s += kSelThreads) {
      R.dbg_cols[R.nremoved + s] = (int16_t)sel[s];
      R.dbg_costs[R.nremoved + s] = lce[sel[s]];
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (R.dbg_sizes != nullptr) R.dbg_sizes[R.iters] = b;
    R.b = b;
    R.width = w - b;
    R.iters += 1;
    R.nremoved += b;
    R.done = (w - b) <= R.target;
  }
}

void launch_carve_select(RunCarve* runs, int nruns, int max_stride, int max_rows, cudaStream_t st) {
  size_t smem = (size_t)max_stride * (8 + 8 + 4 * 4);
  SCPL_ARG(smem <= 227 * 1024, "carve width too large for the select kernel");
  SCPL_CUDA(cudaFuncSetAttribute(carve_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  carve_select_kernel<<<nruns, kSelThreads, smem, st>>>(runs);
  SCPL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ compact
// remove_batch (batching.py:76-107) on the representative's luma plane and on the
// composed index map: a warp per row walks the row in 32-column chunks left to right,
// so in-place writes (to y <= x) never overtake pending reads.
__global__ void carve_compact_kernel(RunCarve* __restrict__ runs) {
  RunCarve& R = runs[blockIdx.y];
  const int b = R.b;
  if (b == 0) return;
  const int warps = blockDim.x >> 5;
  const int i = blockIdx.x * warps + (threadIdx.x >> 5);
  if (i >= R.rows) return;
  const int lane = threadIdx.x & 31;
  const int w0 = R.width + b;
  uint8_t* lrow = R.luma + (long)i * R.stride;
  int16_t* irow = R.idx + (long)i * R.stride;
  const int16_t* rr = R.rem + (long)i * b;
  int ptr = 0, before = 0;
  int nxt = rr[0];
  for (int x0 = 0; x0 < w0; x0 += 32) {
    unsigned mask = 0;
    while (ptr < b && nxt < x0 + 32) {
      mask |= 1u << (nxt - x0);
      ++ptr;
      nxt = ptr < b ? rr[ptr] : INT_MAX;
    }
    const int x = x0 + lane;
    const bool live = x < w0 && !((mask >> lane) & 1u);
    uint8_t lv = 0;
    int16_t iv = 0;
    if (x < w0) {
      lv = lrow[x];
      iv = irow[x];
    }
    __syncwarp();
    if (live) {
      int y = x - before - __popc(mask & ((1u << lane) - 1u));
      lrow[y] = lv;
      irow[y] = iv;
    }
    before += __popc(mask);
    __syncwarp();
  }
}

void launch_carve_compact(RunCarve* runs, int nruns, int max_rows, cudaStream_t st) {
  dim3 grid(cdiv(max_rows, 8), nruns);
  carve_compact_kernel<<<grid, 256, 0, st>>>(runs);
  SCPL_CHECK_LAUNCH();
}

}  // namespace scpl
