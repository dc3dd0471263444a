// K4-K7 (v2): the whole SCPL carve loop of a run in ONE persistent cluster kernel.
//
// Replaces batch_carve (batching.py:118-153) with everything it calls: cumulative_energy
// (seams.py:39-65), label_parents (batching.py:39-46), select_batch (:49-73),
// trace_columns (seams.py:68-81), remove_batch on the representative frame (:76-107) and
// default_energy (:110-115).
//
// One thread-block cluster of CL CTAs (CL SMs) carves one run; runs are independent, so a
// launch holds every run of a clip (grid = runs x CL).  Per DP pass:
//
//  1. DP, column-split.  Each warp owns 96 columns and computes a 128-column window
//     (owned +-16) for 16 rows without any barrier: neighbours come from register shuffles,
//     the window's valid region shrinks by one column per row, and after 16 rows exactly
//     the owned columns remain valid ("trapezoid" tiling).  Every 16 rows (one path-word
//     block) warps publish their owned cumulative energies to shared memory -- and the 16
//     columns next to a CTA edge into the neighbour CTA through DSMEM -- then one cluster
//     barrier.  The reference's argmin-first tie-break (seams.py:62) is strict '<' in the
//     order -1, 0, +1.  Back pointers never leave registers: each column carries a 32-bit
//     path word (2 bits per row) that is reset at every block start; at a block's last row
//     the owned words and their landing deltas go to global memory.
//     First pass of a buffered run: float64 on the uniform map (IEEE adds, no FMA);
//     later passes: int32 on gradient energy (integer-valued, so bit-identical).
//  2. Select (every CTA redundantly, no broadcast needed): labels by chaining the landing
//     deltas bottom-up (table staged in shared memory), per-parent leftmost minimum via
//     shared-memory atomics (labels are monotone, so parents are segments), k-truncation
//     by (cost, col), then each CTA decodes its share of (seam, block) path words into the
//     removed-column log.
//  3. Compact, row-split: luma, gradient and the original-column index map drop the
//     batch's columns in place (warp per row, 32-column chunks left to right).
//  4. Gradient, row-split and incremental: a pixel's Sobel value changes only if a removed
//     pixel of rows i-1..i+1 lay within one column of it; only those are recomputed.
#include <cfloat>
#include <climits>

#include "scpl_common.cuh"
#include "scpl_kernels.h"

namespace scpl {

constexpr int kLanesCols = 4;                     // columns per lane in a warp window
constexpr int kWin = 32 * kLanesCols;             // 128-column window
constexpr int kHalo = kBlockRows;                 // 16 = rows per exchange
constexpr int kOwn = kWin - 2 * kHalo;            // 96 owned columns per warp
constexpr int kIntInf = 0x3fffffff;
constexpr int kMaxWarps = 16;                    // 512 threads: <= 128 registers per thread

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

// ------------------------------------------------------------------ DP value traits
template <bool F64>
struct Val;
template <>
struct Val<false> {
  using T = int;
  static __device__ __forceinline__ T inf() { return kIntInf; }
  static __device__ __forceinline__ T add(T a, T b) { return a + b; }
  static __device__ __forceinline__ double to_d(T v) { return (double)v; }
};
template <>
struct Val<true> {
  using T = double;
  static __device__ __forceinline__ T inf() { return __longlong_as_double(0x7ff0000000000000ll); }
  static __device__ __forceinline__ T add(T a, T b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double to_d(T v) { return v; }
};

struct Geo {  // per-pass column ownership
  int w;          // current width
  int cta_lo, cta_hi;  // owned by this CTA
  int own_lo, own_hi;  // owned by this warp (own_lo >= own_hi: idle)
  int win_lo;          // first window column of this warp (own_lo - 16)
};

// raw energy of one lane's 4 window columns in row i: int path = one 32-bit word of the
// u8 gradient plane, fp64 path = 4 doubles of the uniform map.  Columns outside [0, w) are
// masked by the caller; only in-row addresses are touched.
__device__ __forceinline__ uint32_t load_e_int(const CarveRun& R, int i, int j0, int w) {
  if (j0 < 0 || j0 >= w) return 0u;
  return __ldg(reinterpret_cast<const uint32_t*>(R.grad + (long)i * R.pitch + j0));
}
__device__ __forceinline__ void load_e_f64(const CarveRun& R, int i, int j0, int w, double (&e)[kLanesCols]) {
  const double* row = R.U + (long)i * R.pitch;
  if (j0 >= 0 && j0 + 3 < w) {
    double2 a = __ldg(reinterpret_cast<const double2*>(row + j0));
    double2 b = __ldg(reinterpret_cast<const double2*>(row + j0 + 2));
    e[0] = a.x; e[1] = a.y; e[2] = b.x; e[3] = b.y;
  } else {
#pragma unroll
    for (int k = 0; k < kLanesCols; ++k) e[k] = (j0 + k >= 0 && j0 + k < w) ? row[j0 + k] : 0.0;
  }
}

template <bool F64>
struct ERow;
template <>
struct ERow<false> {
  uint32_t v;
  __device__ __forceinline__ void load(const CarveRun& R, int i, int j0, int w) { v = load_e_int(R, i, j0, w); }
  __device__ __forceinline__ int get(int k) const { return (int)((v >> (8 * k)) & 255u); }
};
template <>
struct ERow<true> {
  double v[kLanesCols];
  __device__ __forceinline__ void load(const CarveRun& R, int i, int j0, int w) { load_e_f64(R, i, j0, w, v); }
  __device__ __forceinline__ double get(int k) const { return v[k]; }
};

// one DP row for a lane's 4 columns (seams.py:54-64): strict '<' in the order -1, 0, +1
template <bool F64>
__device__ __forceinline__ void dp_row(typename Val<F64>::T (&ce)[kLanesCols], uint32_t (&pw)[kLanesCols],
                                       const ERow<F64>& e, const bool (&in)[kLanesCols], int lane) {
  using V = Val<F64>;
  using T = typename V::T;
  T left = __shfl_up_sync(0xffffffffu, ce[kLanesCols - 1], 1);
  T right = __shfl_down_sync(0xffffffffu, ce[0], 1);
  uint32_t pleft = __shfl_up_sync(0xffffffffu, pw[kLanesCols - 1], 1);
  uint32_t pright = __shfl_down_sync(0xffffffffu, pw[0], 1);
  if (lane == 0) left = V::inf();
  if (lane == 31) right = V::inf();
  T nce[kLanesCols];
  uint32_t npw[kLanesCols];
#pragma unroll
  for (int k = 0; k < kLanesCols; ++k) {
    T l = k > 0 ? ce[k - 1] : left;
    T c = ce[k];
    T r = k + 1 < kLanesCols ? ce[k + 1] : right;
    uint32_t pl = k > 0 ? pw[k - 1] : pleft;
    uint32_t pc = pw[k];
    uint32_t pr = k + 1 < kLanesCols ? pw[k + 1] : pright;
    bool p1 = c < l;
    T m = p1 ? c : l;
    uint32_t ps = p1 ? pc : pl;
    uint32_t code = p1 ? 1u : 0u;
    bool p2 = r < m;
    m = p2 ? r : m;
    ps = p2 ? pr : ps;
    code = p2 ? 2u : code;
    nce[k] = in[k] ? V::add((T)e.get(k), m) : V::inf();
    npw[k] = (ps << 2) | code;
  }
#pragma unroll
  for (int k = 0; k < kLanesCols; ++k) {
    ce[k] = nce[k];
    pw[k] = npw[k];
  }
}

// One DP pass over all rows for this warp's window. ceX: smem exchange rows [2][pitch].
template <bool F64>
__device__ void dp_pass(const CarveRun& R, const Geo& g, typename Val<F64>::T* ceX, int CL, uint32_t rank,
                        int per_cta) {
  using V = Val<F64>;
  using T = typename V::T;
  constexpr int PF = F64 ? 4 : kBlockRows;  // rows of energy in flight
  const int lane = threadIdx.x & 31;
  const int rows = R.rows, w = g.w;
  const bool active = g.own_lo < g.own_hi;
  const int j0 = g.win_lo + lane * kLanesCols;
  T ce[kLanesCols];
  uint32_t pw[kLanesCols];
  bool in[kLanesCols];
#pragma unroll
  for (int k = 0; k < kLanesCols; ++k) in[k] = (j0 + k >= 0) && (j0 + k < w);
  ERow<F64> ring[PF];
  if (active) {
    ERow<F64> e0;
    e0.load(R, 0, j0, w);
#pragma unroll
    for (int k = 0; k < kLanesCols; ++k) ce[k] = in[k] ? (T)e0.get(k) : V::inf();
#pragma unroll
    for (int q = 0; q < PF; ++q)
      if (1 + q < rows) ring[q].load(R, 1 + q, j0, w);
  }
  const int nblk = (rows - 1 + kBlockRows - 1) / kBlockRows;
  for (int blk = 0; blk < nblk; ++blk) {
    const int i0 = 1 + blk * kBlockRows;
    const int nr = min(kBlockRows, rows - i0);
    if (active) {
      if (blk > 0) {
        const T* src = ceX + (size_t)((blk - 1) & 1) * R.pitch;
#pragma unroll
        for (int k = 0; k < kLanesCols; ++k) ce[k] = in[k] ? src[j0 + k] : V::inf();
      }
#pragma unroll
      for (int k = 0; k < kLanesCols; ++k) pw[k] = 0u;
      if constexpr (F64) {
#pragma unroll
        for (int r = 0; r < kBlockRows; ++r) {
          if (r < nr) {
            ERow<true> e = ring[r % PF];
            if (i0 + r + PF < rows) ring[r % PF].load(R, i0 + r + PF, j0, w);
            dp_row<true>(ce, pw, e, in, lane);
          }
        }
      } else {
        ERow<false> cur[kBlockRows];
#pragma unroll
        for (int r = 0; r < kBlockRows; ++r) cur[r] = ring[r];
        // next block's energy rows in flight while this block computes
#pragma unroll
        for (int r = 0; r < kBlockRows; ++r)
          if (i0 + kBlockRows + r < rows) ring[r].load(R, i0 + kBlockRows + r, j0, w);
#pragma unroll
        for (int r = 0; r < kBlockRows; ++r)
          if (r < nr) dp_row<false>(ce, pw, cur[r], in, lane);
      }
      // block end: owned columns publish path words, landing deltas and ce
      T* dst = ceX + (size_t)(blk & 1) * R.pitch;
#pragma unroll
      for (int k = 0; k < kLanesCols; ++k) {
        int j = j0 + k;
        if (j >= g.own_lo && j < g.own_hi) {
          int sum = __popc(pw[k] & 0x55555555u) + 2 * __popc(pw[k] & 0xAAAAAAAAu);
          R.pw[(long)blk * R.pitch + j] = pw[k];
          R.delta[(long)blk * R.pitch + j] = (int8_t)(sum - nr);
          dst[j] = ce[k];
          // halo for every other CTA whose warps' windows reach column j
          for (int q = 0; q < CL; ++q) {
            if (q == (int)rank) continue;
            int lo = min(w, q * per_cta), hi = min(w, lo + per_cta);
            if (lo < hi && j >= lo - kHalo && j < hi + kHalo) st_cluster(map_rank(&dst[j], q), ce[k]);
          }
        }
      }
    }
    cluster_sync();
  }
  // last row
  if (active) {
#pragma unroll
    for (int k = 0; k < kLanesCols; ++k) {
      int j = j0 + k;
      if (j >= g.own_lo && j < g.own_hi) R.lastce[j] = V::to_d(ce[k]);
    }
  }
}

// ------------------------------------------------------------------ block helpers
__device__ int block_excl_scan(int v, int* ws, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < nw ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    ws[lane] = s;
  }
  __syncthreads();
  int base = wid > 0 ? ws[wid - 1] : 0;
  total = ws[nw - 1];
  __syncthreads();
  return base + x - v;
}

// ------------------------------------------------------------------ the persistent kernel
struct SelSmem {
  double* lce;
  unsigned long long* segmin;
  int* lab;
  int* segarg;
  int* cand;
  int* sel;
  int8_t* dtab;    // staged delta table [nblk][pitch] (or nullptr: chain in global)
};

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// warp-inclusive scan of v over lanes
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Alive-column bitmask of one row (nw32 words, <= 32*kMaxAliveWordsPerLane): the lanes hold
// words m = lane + 32u; wv/pre (per-warp smem) receive the words and exclusive popcounts.
constexpr int kMaxAliveWordsPerLane = 4;  // widths up to 4096
__device__ __forceinline__ void alive_row_prefix(const uint32_t* row, int nw32, uint32_t* wv, int* pre) {
  const int lane = threadIdx.x & 31;
  int running = 0;
#pragma unroll
  for (int u = 0; u < kMaxAliveWordsPerLane; ++u) {
    int m = lane + 32 * u;
    uint32_t wd = m < nw32 ? row[m] : 0u;
    int p = __popc(wd);
    int incl = warp_incl_scan(p);
    if (m < nw32) {
      wv[m] = wd;
      pre[m] = running + incl - p;
    }
    running += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
}

// original column of current column c (the c-th alive bit), given wv/pre of the row
__device__ __forceinline__ int alive_select(const uint32_t* wv, const int* pre, int nw32, int c) {
  int lo = 0, hi = nw32 - 1;  // largest m with pre[m] <= c
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= c) lo = mid; else hi = mid - 1;
  }
  return lo * 32 + (int)__fns(wv[lo], 0, c - pre[lo] + 1);
}

__global__ void __launch_bounds__(kMaxWarps * 32, 1) carve_cluster_kernel(CarveRun* __restrict__ runs, int CL) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int ws[32];
  __shared__ __align__(8) uint64_t s_bar[kMaxWarps * 2];
  const uint32_t rank = cluster_rank();
  CarveRun& Rg = runs[blockIdx.x / CL];
  const CarveRun R = Rg;  // static fields in registers
  const int rows = R.rows, pitch = R.pitch;
  const int nblk = (rows - 1 + kBlockRows - 1) / kBlockRows;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int nw32 = (R.width0 + 31) >> 5;
  const int rlo = (int)((long)rows * rank / CL), rhi = (int)((long)rows * (rank + 1) / CL);
  const bool stage_dtab = R.stage_dtab != 0;
  const int RB = ((pitch + 15) & ~15) + 16;  // staged row bytes (compaction)
  int w = R.width0;
  int iters = 0, removed = 0;
  long long prof[4] = {0, 0, 0, 0};
  long long tp = clock64();

  // all columns alive; per-warp mbarriers for the staged compaction
  for (int i = rlo + wid; i < rhi; i += nw)
    for (int m = lane; m < nw32; m += 32) {
      int hi = R.width0 - 32 * m;
      R.alive[(long)i * R.alive_pitch + m] = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
    }
  if (lane == 0) {
    mbar_init(&s_bar[2 * wid], 1);
    mbar_init(&s_bar[2 * wid + 1], 1);
    fence_mbar_init();
  }
  uint32_t phase[2] = {0u, 0u};
  cluster_sync();

  while (w > R.target) {
    // ---------------- 1. DP
    Geo g;
    g.w = w;
    const int per = ((w + CL - 1) / CL + 3) & ~3;
    g.cta_lo = min(w, (int)rank * per);
    g.cta_hi = min(w, g.cta_lo + per);
    g.own_lo = g.cta_lo + wid * kOwn;
    g.own_hi = min(g.cta_hi, g.own_lo + kOwn);
    g.win_lo = g.own_lo - kHalo;
    if (iters == 0 && R.U != nullptr)
      dp_pass<true>(R, g, reinterpret_cast<double*>(smem), CL, rank, per);
    else
      dp_pass<false>(R, g, reinterpret_cast<int*>(smem), CL, rank, per);
    cluster_sync();  // lastce / pw / delta of all CTAs visible
    if (tid == 0) { long long t = clock64(); prof[0] += t - tp; tp = t; }

    // ---------------- 2. select (redundant per CTA)
    SelSmem S;
    {
      uint8_t* p = smem;
      S.lce = reinterpret_cast<double*>(p);
      p += 8 * (size_t)pitch;
      S.segmin = reinterpret_cast<unsigned long long*>(p);
      p += 8 * (size_t)pitch;
      S.lab = reinterpret_cast<int*>(p);
      p += 4 * (size_t)pitch;
      S.segarg = reinterpret_cast<int*>(p);
      p += 4 * (size_t)pitch;
      S.cand = reinterpret_cast<int*>(p);
      p += 4 * (size_t)pitch;
      S.sel = reinterpret_cast<int*>(p);
      p += 4 * (size_t)pitch;
      S.dtab = stage_dtab ? reinterpret_cast<int8_t*>(p) : nullptr;
    }
    for (int j = tid; j < w; j += blockDim.x) {
      S.lce[j] = R.lastce[j];
      S.segmin[j] = ~0ull;
      S.segarg[j] = INT_MAX;
    }
    const int8_t* dsrc = R.delta;
    if (stage_dtab) {
      const int per_row = (w + 15) >> 4;  // 16-byte copies; pitch is a multiple of 16
      for (int q = tid; q < nblk * per_row; q += blockDim.x) {
        int bl = q / per_row, c = (q - bl * per_row) << 4;
        *reinterpret_cast<uint4*>(S.dtab + (size_t)bl * pitch + c) =
            *reinterpret_cast<const uint4*>(R.delta + (size_t)bl * pitch + c);
      }
      dsrc = S.dtab;
    }
    __syncthreads();
    // labels (batching.py:39-46): chain the block landing deltas, 8 columns per thread in flight
    for (int jb = tid; jb < w; jb += 8 * blockDim.x) {
      int c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) c[u] = jb + u * (int)blockDim.x;
      for (int bl = nblk - 1; bl >= 0; --bl) {
        const int8_t* drow = dsrc + (size_t)bl * pitch;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (jb + u * (int)blockDim.x < w) c[u] += drow[c[u]];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (jb + u * (int)blockDim.x < w) S.lab[jb + u * blockDim.x] = c[u];
    }
    __syncthreads();
    int b;
    if (R.kmax == 1) {  // raw mode: min_seam, leftmost global minimum (seams.py:84-89)
      for (int j = tid; j < w; j += blockDim.x)
        atomicMin(&S.segmin[0], (unsigned long long)__double_as_longlong(S.lce[j]));
      __syncthreads();
      for (int j = tid; j < w; j += blockDim.x)
        if ((unsigned long long)__double_as_longlong(S.lce[j]) == S.segmin[0]) atomicMin(&S.segarg[0], j);
      __syncthreads();
      if (tid == 0) S.sel[0] = S.segarg[0];
      b = 1;
    } else {
      // per parent the leftmost strict minimum (batching.py:59-64); doubles >= 0 order as u64
      for (int j = tid; j < w; j += blockDim.x)
        atomicMin(&S.segmin[S.lab[j]], (unsigned long long)__double_as_longlong(S.lce[j]));
      __syncthreads();
      for (int j = tid; j < w; j += blockDim.x)
        if ((unsigned long long)__double_as_longlong(S.lce[j]) == S.segmin[S.lab[j]])
          atomicMin(&S.segarg[S.lab[j]], j);
      __syncthreads();
      const int perq0 = (w + blockDim.x - 1) / blockDim.x;
      int cnt = 0;
      for (int u = 0; u < perq0; ++u) {
        int l = tid * perq0 + u;
        if (l < w && S.segarg[l] != INT_MAX) ++cnt;
      }
      int P;
      int pos = block_excl_scan(cnt, ws, P);
      for (int u = 0; u < perq0; ++u) {
        int l = tid * perq0 + u;
        if (l < w && S.segarg[l] != INT_MAX) S.cand[pos++] = S.segarg[l];
      }
      __syncthreads();
      const int k = w - R.target;
      if (P <= k) {
        for (int q = tid; q < P; q += blockDim.x) S.sel[q] = S.cand[q];
        b = P;
      } else {  // keep the k cheapest by (cost, col) (batching.py:66-68)
        const int perq = (P + blockDim.x - 1) / blockDim.x;
        unsigned keep = 0;
        for (int u = 0; u < perq; ++u) {
          int q = tid * perq + u;
          if (q < P) {
            double cq = S.lce[S.cand[q]];
            int rk = 0;
            for (int o = 0; o < P; ++o) {
              double co = S.lce[S.cand[o]];
              rk += (co < cq) || (co == cq && o < q);
            }
            if (rk < k) keep |= 1u << u;
          }
        }
        int tot;
        int p2 = block_excl_scan(__popc(keep), ws, tot);
        for (int u = 0; u < perq; ++u)
          if (keep >> u & 1u) S.sel[p2++] = S.cand[tid * perq + u];
        b = k;
      }
    }
    __syncthreads();
    // trace (seams.py:68-81): walk each seam's block-end columns through the staged deltas,
    // keeping those of this CTA's blocks (bl % CL == rank); then decode (seam, block) pairs
    // in parallel into the removed-column log
    int16_t* log = R.rem;  // rows x rem_cap, this batch's columns at [removed, removed + b)
    for (int s = tid; s < b; s += blockDim.x) {
      int c = S.sel[s];
      for (int bl = nblk - 1; bl >= 0; --bl) {
        if (bl % CL == (int)rank) R.cend[(long)bl * pitch + s] = (int16_t)c;
        c += dsrc[(size_t)bl * pitch + c];
      }
      if (rank == 0) log[removed + s] = (int16_t)c;  // row 0 (== the seam's label)
    }
    __syncthreads();
    const int myblk = nblk > (int)rank ? (nblk - 1 - (int)rank) / CL + 1 : 0;
    for (int q = tid; q < b * myblk; q += blockDim.x) {
      int s = q / myblk, bl = (int)rank + (q - s * myblk) * CL;
      int c = R.cend[(long)bl * pitch + s];
      uint32_t word = R.pw[(long)bl * pitch + c];
      int i_start = 1 + bl * kBlockRows;
      int i_end = min(i_start + kBlockRows, rows) - 1;
      for (int i = i_end; i >= i_start; --i) {
        log[(long)i * R.rem_cap + removed + s] = (int16_t)c;
        c += (int)(word & 3u) - 1;
        word >>= 2;
      }
    }
    if (rank == 0 && R.sizes != nullptr) {
      for (int s = tid; s < b; s += blockDim.x) {
        R.cols[removed + s] = (int16_t)S.sel[s];
        R.costs[removed + s] = S.lce[S.sel[s]];
      }
      if (tid == 0) R.sizes[iters] = b;
    }
    cluster_sync();  // the whole batch's log is visible
    if (tid == 0) { long long t = clock64(); prof[1] += t - tp; tp = t; }

    // ---------------- 3. compact luma + grad in place, update the alive bitmask
    // (remove_batch, batching.py:76-107).  Warp per row; the row pair is staged in shared
    // memory by a TMA bulk copy (next row prefetched while this one is written back), and
    // every output word is one funnel shift of two staged words unless a removed column
    // falls inside it.
    const int w0 = w;
    const int wn = w - b;
    {
      uint8_t* wbuf = smem + (size_t)wid * (4 * RB + 1024);
      uint32_t* wv = reinterpret_cast<uint32_t*>(wbuf + 4 * RB);
      int* pre = reinterpret_cast<int*>(wbuf + 4 * RB + 512);
      const uint32_t nbytes = (uint32_t)((w0 + 15) & ~15);
      auto issue = [&](int row, int slot) {
        if (lane == 0) {
          fence_proxy_async_global();
          mbar_arrive_tx(&s_bar[2 * wid + slot], 2 * nbytes);
          bulk_g2s(wbuf + (size_t)slot * 2 * RB, R.luma + (long)row * pitch, nbytes, &s_bar[2 * wid + slot]);
          bulk_g2s(wbuf + (size_t)slot * 2 * RB + RB, R.grad + (long)row * pitch, nbytes, &s_bar[2 * wid + slot]);
        }
      };
      int kk = 0;
      if (rlo + wid < rhi) issue(rlo + wid, 0);
      for (int i = rlo + wid; i < rhi; i += nw, ++kk) {
        const int slot = kk & 1;
        if (i + nw < rhi) issue(i + nw, slot ^ 1);
        mbar_wait(&s_bar[2 * wid + slot], phase[slot]);
        phase[slot] ^= 1u;
        const uint8_t* Ls = wbuf + (size_t)slot * 2 * RB;
        const uint8_t* Gs = Ls + RB;
        uint32_t* Lg = reinterpret_cast<uint32_t*>(R.luma + (long)i * pitch);
        uint32_t* Gg = reinterpret_cast<uint32_t*>(R.grad + (long)i * pitch);
        const int16_t* rr = log + (long)i * R.rem_cap + removed;  // sorted, old coordinates
        // output byte y reads input byte y + #{t : rr[t] - t <= y}
        int tptr = 0;  // warp-uniform: entries with rr[t]-t < chunk start
        const int nwo = (wn + 3) >> 2;
        for (int q0 = 0; q0 < nwo; q0 += 32) {
          const int y0 = 4 * (q0 + lane);
          const int cend = 4 * (q0 + 32);
          int s4[4] = {tptr, tptr, tptr, tptr};
          int t = tptr;
          while (t < b) {
            int a = rr[t] - t;
            if (a >= cend) break;
#pragma unroll
            for (int u = 0; u < 4; ++u) s4[u] += (a <= y0 + u);
            ++t;
          }
          tptr = t;  // warp-uniform: all lanes walked the same entries
          // entries with a < chunk start are counted in the base; recount the in-chunk ones
          if (q0 + lane < nwo) {
            uint32_t lo, go;
            if (s4[0] == s4[3]) {
              const int x0 = y0 + s4[0];
              const uint32_t* L32 = reinterpret_cast<const uint32_t*>(Ls) + (x0 >> 2);
              const uint32_t* G32 = reinterpret_cast<const uint32_t*>(Gs) + (x0 >> 2);
              const uint32_t sh = (uint32_t)(x0 & 3) * 8u;
              lo = __funnelshift_r(L32[0], L32[1], sh);
              go = __funnelshift_r(G32[0], G32[1], sh);
            } else {
              lo = go = 0u;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                lo |= (uint32_t)Ls[y0 + u + s4[u]] << (8 * u);
                go |= (uint32_t)Gs[y0 + u + s4[u]] << (8 * u);
              }
            }
            Lg[q0 + lane] = lo;
            Gg[q0 + lane] = go;
          }
        }
        // alive bitmask: clear the original columns of this batch's removed pixels
        uint32_t* arow = R.alive + (long)i * R.alive_pitch;
        alive_row_prefix(arow, nw32, wv, pre);
        // highest seams first: clearing bits above a target never moves the target's
        // select, so the prefix counts taken before the batch stay valid
        for (int base = b - 1; base >= 0; base -= 32) {
          const int s = base - lane;
          int o = 0;
          if (s >= 0) o = alive_select(wv, pre, nw32, rr[s]);
          __syncwarp();
          if (s >= 0) atomicAnd(&wv[o >> 5], ~(1u << (o & 31)));
          __syncwarp();
        }
        for (int m = lane; m < nw32; m += 32) arow[m] = wv[m];
        __syncwarp();
      }
    }
    cluster_sync();  // compacted luma of every row visible
    if (tid == 0) { long long t = clock64(); prof[2] += t - tp; tp = t; }

    // ---------------- 4. incremental gradient (batching.py:110-115 on the carved frame)
    if (wn > R.target) {
      const bool zero = rows < 3 || wn < 3;
      for (int i = rlo + wid; i < rhi; i += nw) {
        uint8_t* gr = R.grad + (long)i * pitch;
        if (zero) {
          for (int y = lane; y < wn; y += 32) gr[y] = 0;
          continue;
        }
        const int16_t* ri = log + (long)i * R.rem_cap + removed;  // row i's removed (sorted)
        const int ia = max(i - 1, 0), ib = min(i + 1, rows - 1);
        const uint8_t* la = R.luma + (long)ia * pitch;
        const uint8_t* lb = R.luma + (long)i * pitch;
        const uint8_t* lc = R.luma + (long)ib * pitch;
        // candidates: rows {i-1, i, i+1} x seams x offsets {-1, 0, +1}, in old columns
        const int ncand = 9 * b;
        for (int q = lane; q < ncand; q += 32) {
          int rsel = q / (3 * b), rem = q - rsel * 3 * b;
          int s = rem / 3, off = rem - s * 3 - 1;
          int r = rsel == 0 ? ia : (rsel == 1 ? i : ib);
          int x = log[(long)r * R.rem_cap + removed + s] + off;
          if (x < 0 || x >= w0) continue;
          int lo = 0, hi = b;  // number of row-i removed columns < x
          while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (ri[mid] < x) lo = mid + 1; else hi = mid;
          }
          if (lo < b && ri[lo] == x) continue;  // removed itself
          int y = x - lo;
          int ym = max(y - 1, 0), yp = min(y + 1, wn - 1);
          int gx = (la[yp] + 2 * lb[yp] + lc[yp]) - (la[ym] + 2 * lb[ym] + lc[ym]);
          int gy = (lc[ym] + 2 * lc[y] + lc[yp]) - (la[ym] + 2 * la[y] + la[yp]);
          int gv = abs(gx) + abs(gy);
          gr[y] = (uint8_t)(gv > 255 ? 255 : gv);
        }
      }
    }
    removed += b;
    ++iters;
    w = wn;
    cluster_sync();
    if (tid == 0) { long long t = clock64(); prof[3] += t - tp; tp = t; }
  }

  // final index map (original column of every kept column) from the alive bitmask
  {
    uint8_t* wbuf = smem + (size_t)wid * (4 * RB + 1024);
    uint32_t* wv = reinterpret_cast<uint32_t*>(wbuf + 4 * RB);
    int* pre = reinterpret_cast<int*>(wbuf + 4 * RB + 512);
    for (int i = rlo + wid; i < rhi; i += nw) {
      alive_row_prefix(R.alive + (long)i * R.alive_pitch, nw32, wv, pre);
      int16_t* ir = R.idx + (long)i * pitch;
      for (int m = lane; m < nw32; m += 32) {
        uint32_t wd = wv[m];
        int o = pre[m];
        while (wd) {
          int bit = __ffs(wd) - 1;
          ir[o++] = (int16_t)(m * 32 + bit);
          wd &= wd - 1;
        }
      }
      __syncwarp();
    }
  }
  if (rank == 0 && tid == 0) {
    Rg.iters = iters;
    Rg.removed = removed;
    if (R.prof)
      for (int k = 0; k < 4; ++k) R.prof[k] = prof[k];
  }
}

// ------------------------------------------------------------------ setup + launch
// luma / index / gradient planes of one representative frame in carve orientation.
// codes (nullable): the frame's energy codes (low byte = Sobel of its luma); else the
// gradient is computed here (transpose commutes with the edge-replicated Sobel).
__global__ void run_setup_kernel(const uint8_t* __restrict__ frame, int H, int W, int C, int transposed,
                                 const uint16_t* __restrict__ codes, int pitch, uint8_t* __restrict__ luma,
                                 uint8_t* __restrict__ grad, int16_t* __restrict__ idx) {
  __shared__ uint8_t tl[32][33], tg[32][33];
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    int i = i0 + r, j = j0 + threadIdx.x;
    uint8_t v = 0, gv = 0;
    if (i < H && j < W) {
      const uint8_t* px = frame + ((long)i * W + j) * C;
      v = C == 3 ? (uint8_t)luma_of(px[0], px[1], px[2]) : px[0];
      gv = codes ? (uint8_t)(codes[(long)i * W + j] & 255u) : 0;
      if (!transposed) {
        luma[(long)i * pitch + j] = v;
        grad[(long)i * pitch + j] = gv;
        idx[(long)i * pitch + j] = (int16_t)j;
      }
    }
    tl[r][threadIdx.x] = v;
    tg[r][threadIdx.x] = gv;
  }
  if (!transposed) return;
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    int j = j0 + r, i = i0 + threadIdx.x;  // carve row j, carve col i
    if (i < H && j < W) {
      luma[(long)j * pitch + i] = tl[threadIdx.x][r];
      grad[(long)j * pitch + i] = tg[threadIdx.x][r];
      idx[(long)j * pitch + i] = (int16_t)i;
    }
  }
}

// full Sobel of a carve-orientation luma plane (runs without energy codes)
__global__ void plane_sobel_kernel(const uint8_t* __restrict__ luma, int rows, int cols, int pitch,
                                   uint8_t* __restrict__ grad) {
  const int i = blockIdx.y;
  const bool zero = rows < 3 || cols < 3;
  const uint8_t* a = luma + (long)max(i - 1, 0) * pitch;
  const uint8_t* b = luma + (long)i * pitch;
  const uint8_t* c = luma + (long)min(i + 1, rows - 1) * pitch;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x) {
    int g = 0;
    if (!zero) {
      int jm = max(j - 1, 0), jp = min(j + 1, cols - 1);
      int gx = (a[jp] + 2 * b[jp] + c[jp]) - (a[jm] + 2 * b[jm] + c[jm]);
      int gy = (c[jm] + 2 * c[j] + c[jp]) - (a[jm] + 2 * a[j] + a[jp]);
      g = abs(gx) + abs(gy);
      g = g > 255 ? 255 : g;
    }
    grad[(long)i * pitch + j] = (uint8_t)g;
  }
}

void launch_run_setup(const uint8_t* frame, int H, int W, int C, int transposed, const uint16_t* codes,
                      const CarveRun& R, cudaStream_t st) {
  dim3 grid(cdiv(W, 32), cdiv(H, 32));
  run_setup_kernel<<<grid, dim3(32, 8), 0, st>>>(frame, H, W, C, transposed, codes, R.pitch, R.luma, R.grad,
                                                 R.idx);
  SCPL_CHECK_LAUNCH();
  if (!codes) {
    plane_sobel_kernel<<<dim3(cdiv(R.width0, 256), R.rows), 256, 0, st>>>(R.luma, R.rows, R.width0, R.pitch,
                                                                         R.grad);
    SCPL_CHECK_LAUNCH();
  }
}

int carve_cluster_size(int nruns, int width, int num_sms) {
  int cl = 1;
  while (cl < 8 && (long)nruns * cl * 2 <= num_sms) cl <<= 1;  // one cluster per run, all resident
  while ((long)kOwn * kMaxWarps * cl < width && cl < 8) cl <<= 1;  // <= kMaxWarps warps per CTA
  return cl;
}

size_t carve_smem_bytes(int rows, int pitch, bool stage, int warps) {
  const int nblk = (rows - 1 + kBlockRows - 1) / kBlockRows;
  size_t dp = 2 * sizeof(double) * (size_t)pitch;
  size_t sel = (size_t)pitch * (8 + 8 + 4 * 4) + 16;
  if (stage) sel += (size_t)nblk * pitch;
  const size_t RB = (((size_t)pitch + 15) & ~(size_t)15) + 16;
  size_t comp = (size_t)warps * (4 * RB + 1024);
  size_t m = dp > sel ? dp : sel;
  return m > comp ? m : comp;
}

int carve_warps(int width, int cl) {
  const int per_cta = (((width + cl - 1) / cl) + 3) & ~3;
  int warps = (per_cta + kOwn - 1) / kOwn;
  return warps < 4 ? 4 : warps;
}

bool carve_stage_dtab(int rows, int pitch, int warps) {
  return carve_smem_bytes(rows, pitch, true, warps) <= 220 * 1024;
}

void launch_carve_cluster(CarveRun* runs_d, int nruns, int rows, int pitch, int width, int cl, cudaStream_t st) {
  if (nruns == 0) return;
  const int warps = carve_warps(width, cl);
  SCPL_ARG(warps <= kMaxWarps, "carve width too large for the cluster size");
  const bool stage = carve_stage_dtab(rows, pitch, warps);
  size_t smem = carve_smem_bytes(rows, pitch, stage, warps);
  SCPL_ARG(smem <= 227 * 1024, "carve plane too large for shared memory");
  SCPL_CUDA(cudaFuncSetAttribute(carve_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nruns * cl);
  cfg.blockDim = dim3(warps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SCPL_CUDA(cudaLaunchKernelEx(&cfg, carve_cluster_kernel, runs_d, cl));
  SCPL_CHECK_LAUNCH();
}

}  // namespace scpl
