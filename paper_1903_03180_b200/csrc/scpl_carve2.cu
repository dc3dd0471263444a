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

constexpr int kC = 6;                             // columns per lane in a DP warp window
constexpr int kWin = 32 * kC;                     // 192-column window
constexpr int kXRows = 32;                        // rows between boundary exchanges (= halo)
constexpr int kOwn = kWin - 2 * kXRows;           // 128 owned columns per DP warp
constexpr int kDpWarps = 4;                       // DP warps per CTA: one per SM sub-partition
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

// neighbour exchange barriers: release/acquire at cluster scope, local or remote arrive
__device__ __forceinline__ void mbar_arrive_cluster_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster_remote(uint64_t* bar, uint32_t rank) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(map_rank(bar, rank))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITX_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITX_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
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

// ------------------------------------------------------------------ DP (v3)
// Window layout: a DP warp owns kOwn = 128 columns and computes a 192-column window
// (owned +- 32), 6 contiguous columns per lane, for kXRows = 32 rows between exchanges.
// Energy rows reach shared memory through TMA bulk copies (one 1-D copy per window row,
// issued by lane 0 a stage ahead); async-proxy copies do not hold back the release of the
// block-boundary exchange, and the lanes read them with plain LDS.
template <bool F64>
struct DpCfg;
template <>
struct DpCfg<false> {
  static constexpr int kStageRows = 32, kStages = 2;  // a whole exchange block in flight
};
template <>
struct DpCfg<true> {
  static constexpr int kStageRows = 4, kStages = 6;   // fp64 rows are 8x larger: finer ring
};
template <bool F64>
__host__ __device__ constexpr size_t dp_ring_bytes() {
  return (size_t)DpCfg<F64>::kStages * DpCfg<F64>::kStageRows * kWin * (F64 ? 8 : 1);
}

// issue stage `st` (rows 1 + st*RS ...) of this warp's energy window into ring slot st % S
template <bool F64>
__device__ __forceinline__ void dp_issue_stage(const CarveRun& R, int st, int win_lo, uint8_t* ring,
                                               uint64_t* bars) {
  constexpr int RS = DpCfg<F64>::kStageRows, S = DpCfg<F64>::kStages;
  constexpr int sz = F64 ? 8 : 1;
  const int slot = st % S;
  const int i0 = 1 + st * RS;
  const int nrow = min(RS, R.rows - i0);
  if (nrow <= 0) return;
  const int c0 = max(win_lo, 0);
  const int c1 = min(win_lo + kWin, R.pitch);
  const uint32_t bytes = (uint32_t)((c1 - c0) * sz);
  const uint8_t* base = F64 ? reinterpret_cast<const uint8_t*>(R.U) : R.grad;
  uint8_t* dst0 = ring + (size_t)slot * RS * kWin * sz + (size_t)(c0 - win_lo) * sz;
  fence_proxy_async_global();
  mbar_arrive_tx(&bars[slot], bytes * nrow);
  for (int r = 0; r < nrow; ++r)
    bulk_g2s(dst0 + (size_t)r * kWin * sz, base + ((size_t)(i0 + r) * R.pitch + c0) * sz, bytes, &bars[slot]);
}

// one DP row for a lane's kC columns (seams.py:54-64): strict '<' in the order -1, 0, +1
template <bool F64, bool EDGE>
__device__ __forceinline__ void dp_row(typename Val<F64>::T (&ce)[kC], uint32_t (&pw)[kC],
                                       const uint8_t* erow, const bool (&in)[kC], int lane) {
  using V = Val<F64>;
  using T = typename V::T;
  T e[kC];
  if constexpr (F64) {
    const double2* p = reinterpret_cast<const double2*>(erow) + lane * (kC / 2);
#pragma unroll
    for (int q = 0; q < kC / 2; ++q) {
      double2 v = p[q];
      e[2 * q] = v.x;
      e[2 * q + 1] = v.y;
    }
  } else {
    const uint16_t* p = reinterpret_cast<const uint16_t*>(erow) + lane * (kC / 2);
#pragma unroll
    for (int q = 0; q < kC / 2; ++q) {
      uint32_t v = p[q];
      e[2 * q] = (int)(v & 255u);
      e[2 * q + 1] = (int)(v >> 8);
    }
  }
  T left = __shfl_up_sync(0xffffffffu, ce[kC - 1], 1);
  T right = __shfl_down_sync(0xffffffffu, ce[0], 1);
  uint32_t pleft = __shfl_up_sync(0xffffffffu, pw[kC - 1], 1);
  uint32_t pright = __shfl_down_sync(0xffffffffu, pw[0], 1);
  if (lane == 0) left = V::inf();
  if (lane == 31) right = V::inf();
  T nce[kC];
  uint32_t npw[kC];
#pragma unroll
  for (int k = 0; k < kC; ++k) {
    T l = k > 0 ? ce[k - 1] : left;
    T c = ce[k];
    T r = k + 1 < kC ? ce[k + 1] : right;
    uint32_t pl = k > 0 ? pw[k - 1] : pleft;
    uint32_t pc = pw[k];
    uint32_t pr = k + 1 < kC ? pw[k + 1] : pright;
    bool p1 = c < l;
    T m = p1 ? c : l;
    uint32_t ps = p1 ? pc : pl;
    uint32_t code = p1 ? 1u : 0u;
    bool p2 = r < m;
    m = p2 ? r : m;
    ps = p2 ? pr : ps;
    code = p2 ? 2u : code;
    T v = V::add(e[k], m);
    nce[k] = (!EDGE || in[k]) ? v : V::inf();
    npw[k] = (ps << 2) | code;
  }
#pragma unroll
  for (int k = 0; k < kC; ++k) {
    ce[k] = nce[k];
    pw[k] = npw[k];
  }
}

// One DP pass for this warp's window.  ceX: smem exchange rows [2][pitch]; ring: this
// warp's energy ring; bars: its S ring mbarriers (phase bits in rph); xbar/xc: the
// neighbour-exchange barriers and exchange counter (buffer = xc & 1, parity = (xc>>1) & 1).
// Exchange blocks of 32 rows: when every CTA owns >= 32 columns only adjacent CTAs supply
// halo and each CTA waits on its own mbarrier for its warps plus the adjacent CTAs' warps
// (release/acquire at cluster scope).  Tiny widths fall back to a cluster barrier.
template <bool F64, bool EDGE>
__device__ void dp_rows(const CarveRun& R, const Geo& g, typename Val<F64>::T* ceX, int CL, uint32_t rank,
                        int per_cta, uint64_t* xbar, uint32_t& xc, uint8_t* ring, uint64_t* bars, uint32_t& rph,
                        bool dp_warp, long long* dprof) {
  using V = Val<F64>;
  using T = typename V::T;
  constexpr int RS = DpCfg<F64>::kStageRows, S = DpCfg<F64>::kStages;
  constexpr int sz = F64 ? 8 : 1;
  static_assert(kXRows % RS == 0 && kBlockRows % RS == 0 || RS == kXRows, "stage layout");
  const int lane = threadIdx.x & 31;
  const int rows = R.rows, w = g.w;
  const bool active = dp_warp && g.own_lo < g.own_hi;
  const int j0 = g.win_lo + lane * kC;
  const bool nb_mode = per_cta >= kXRows;
  T ce[kC];
  uint32_t pw[kC];
  bool in[kC];
#pragma unroll
  for (int k = 0; k < kC; ++k) in[k] = (j0 + k >= 0) && (j0 + k < w);
  const int nstage = (rows - 1 + RS - 1) / RS;
  int issued = 0;  // stages issued so far (lane 0's view; uniform enough for the loop below)
  if (active) {
#pragma unroll
    for (int k = 0; k < kC; ++k) {
      T v;
      if constexpr (F64)
        v = in[k] ? R.U[j0 + k] : 0.0;
      else
        v = in[k] ? (int)R.grad[j0 + k] : 0;
      ce[k] = in[k] ? v : V::inf();
    }
    issued = min(S - 1, nstage);
    if (lane == 0)
      for (int st = 0; st < issued; ++st) dp_issue_stage<F64>(R, st, g.win_lo, ring, bars);
  }
  // wait for stage st (issuing the one S-1 ahead first) and return its ring rows
  auto stage_rows = [&](int st) -> const uint8_t* {
    __syncwarp();
    if (lane == 0 && st + S - 1 < nstage) dp_issue_stage<F64>(R, st + S - 1, g.win_lo, ring, bars);
    const int slot = st % S;
    long long tq = clock64();
    mbar_wait(&bars[slot], (rph >> slot) & 1u);
    __syncwarp();  // reconverge after the per-lane wait loop: the row shuffles need a converged warp
    dprof[1] += clock64() - tq;
    rph ^= 1u << slot;
    return ring + (size_t)slot * RS * kWin * sz;
  };
  const int nx = (rows - 1 + kXRows - 1) / kXRows;
  for (int xb = 0; xb < nx; ++xb) {
    long long tx = clock64();
    if (xb > 0 && nb_mode) {
      const uint32_t e = xc - 1;
      mbar_wait_cluster(&xbar[e & 1], (e >> 1) & 1);
    }
    __syncwarp();
    dprof[0] += clock64() - tx;
    if (active) {
      if (xb > 0) {
        const T* src = ceX + (size_t)((xc - 1) & 1) * R.pitch;
#pragma unroll
        for (int k = 0; k < kC; ++k) ce[k] = in[k] ? src[j0 + k] : V::inf();
      }
      const uint8_t* stage = nullptr;
      if constexpr (RS == kXRows) stage = stage_rows(xb);
#pragma unroll 1
      for (int pb = 0; pb < kXRows / kBlockRows; ++pb) {
        const int i0 = 1 + xb * kXRows + pb * kBlockRows;
        const int nr = min(kBlockRows, rows - i0);
        if (nr <= 0) break;
#pragma unroll
        for (int k = 0; k < kC; ++k) pw[k] = 0u;  // path words restart every 16 rows
        if (nr == kBlockRows) {
#pragma unroll
          for (int r = 0; r < kBlockRows; ++r) {
            const uint8_t* erow;
            if constexpr (RS == kXRows) {
              erow = stage + (size_t)(pb * kBlockRows + r) * kWin * sz;
            } else {
              if (r % RS == 0) stage = stage_rows((i0 - 1) / RS + r / RS);
              erow = stage + (size_t)(r % RS) * kWin * sz;
            }
            dp_row<F64, EDGE>(ce, pw, erow, in, lane);
          }
        } else {
#pragma unroll 1
          for (int r = 0; r < nr; ++r) {
            const int i = i0 + r;
            const uint8_t* erow;
            if constexpr (RS == kXRows) {
              erow = stage + (size_t)(pb * kBlockRows + r) * kWin * sz;
            } else {
              if ((i - 1) % RS == 0) stage = stage_rows((i - 1) / RS);
              erow = stage + (size_t)((i - 1) % RS) * kWin * sz;
            }
            dp_row<F64, EDGE>(ce, pw, erow, in, lane);
          }
        }
        // path-word block end: owned words and landing deltas (read after the pass)
        const int pbi = (i0 - 1) / kBlockRows;
#pragma unroll
        for (int k = 0; k < kC; ++k) {
          int j = j0 + k;
          if (j >= g.own_lo && j < g.own_hi) {
            int sum = __popc(pw[k] & 0x55555555u) + 2 * __popc(pw[k] & 0xAAAAAAAAu);
            R.pw[(long)pbi * R.pitch + j] = pw[k];
            R.delta[(long)pbi * R.pitch + j] = (int8_t)(sum - nr);
          }
        }
      }
      dprof[2] += clock64() - tx;  // waits + rows of this exchange block
      // exchange-block end: owned ce to this CTA's buffer, halo to the adjacent CTAs
      T* dst = ceX + (size_t)(xc & 1) * R.pitch;
#pragma unroll
      for (int k = 0; k < kC; ++k) {
        int j = j0 + k;
        if (j >= g.own_lo && j < g.own_hi) {
          dst[j] = ce[k];
          if (nb_mode) {
            if (rank > 0 && j < g.cta_lo + kXRows) st_cluster(map_rank(&dst[j], rank - 1), ce[k]);
            if ((int)rank + 1 < CL && j >= g.cta_hi - kXRows) st_cluster(map_rank(&dst[j], rank + 1), ce[k]);
          } else {
            for (int q = 0; q < CL; ++q) {
              if (q == (int)rank) continue;
              int lo = min(w, q * per_cta), hi = min(w, lo + per_cta);
              if (lo < hi && j >= lo - kXRows && j < hi + kXRows) st_cluster(map_rank(&dst[j], q), ce[k]);
            }
          }
        }
      }
    }
    if (nb_mode) {
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_cluster_local(&xbar[xc & 1]);
        if (rank > 0) mbar_arrive_cluster_remote(&xbar[xc & 1], rank - 1);
        if ((int)rank + 1 < CL) mbar_arrive_cluster_remote(&xbar[xc & 1], rank + 1);
      }
    } else {
      cluster_sync();
    }
    ++xc;
  }
  if (active) {
#pragma unroll
    for (int k = 0; k < kC; ++k) {
      int j = j0 + k;
      if (j >= g.own_lo && j < g.own_hi) R.lastce[j] = V::to_d(ce[k]);
    }
  }
  (void)issued;
}

template <bool F64>
__device__ void dp_pass(const CarveRun& R, const Geo& g, typename Val<F64>::T* ceX, int CL, uint32_t rank,
                        int per_cta, uint64_t* xbar, uint32_t& xc, uint8_t* ring, uint64_t* bars, uint32_t& rph,
                        bool dp_warp, long long* dprof) {
  // interior windows skip the per-column range masks
  const bool edge = g.win_lo < 0 || g.win_lo + kWin > g.w;
  if (__any_sync(0xffffffffu, edge))
    dp_rows<F64, true>(R, g, ceX, CL, rank, per_cta, xbar, xc, ring, bars, rph, dp_warp, dprof);
  else
    dp_rows<F64, false>(R, g, ceX, CL, rank, per_cta, xbar, xc, ring, bars, rph, dp_warp, dprof);
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
constexpr int kListCap = 192;             // per-warp staged removal-list entries per row
constexpr int kWarpScratch = 1024 + 3 * kListCap * 2;  // wv + pre + three row lists
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

__global__ void __launch_bounds__(kMaxWarps * 32, 1) carve_cluster_kernel(CarveRun* __restrict__ runs, int CL, int ncw) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int ws[32];
  __shared__ __align__(8) uint64_t s_bar[kMaxWarps * 2];
  __shared__ __align__(8) uint64_t s_xbar[2];
  __shared__ __align__(8) uint64_t s_rbar[kMaxWarps * 6];
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
  long long dprof[3] = {0, 0, 0};

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
  }
  // DP warps own 128 columns each; the ring buffers exist for the first ndp warps
  const int ndp = min(kMaxWarps, (((R.width0 + CL - 1) / CL + 15) / 16 * 16 + kOwn - 1) / kOwn);
  if (tid == 0) {  // every DP warp of this CTA and of the adjacent CTAs arrives per exchange
    const int nadj = (rank > 0 ? 1 : 0) + ((int)rank + 1 < CL ? 1 : 0);
    mbar_init(&s_xbar[0], (uint32_t)(ndp * (1 + nadj)));
    mbar_init(&s_xbar[1], (uint32_t)(ndp * (1 + nadj)));
  }
  if (lane == 0)
    for (int k = 0; k < 6; ++k) mbar_init(&s_rbar[wid * 6 + k], 1);
  if (lane == 0) fence_mbar_init();
  uint32_t xc = 0, rph = 0;
  uint32_t phase[2] = {0u, 0u};
  cluster_sync();

  while (w > R.target) {
    // ---------------- 1. DP
    Geo g;
    g.w = w;
    const int per = ((w + CL - 1) / CL + 15) & ~15;
    g.cta_lo = min(w, (int)rank * per);
    g.cta_hi = min(w, g.cta_lo + per);
    g.own_lo = g.cta_lo + wid * kOwn;
    g.own_hi = min(g.cta_hi, g.own_lo + kOwn);
    g.win_lo = g.own_lo - kXRows;
    // warps outside the DP go straight to the cluster barrier -- unless the pass falls back
    // to cluster barriers per exchange (tiny widths), which every thread must join
    const bool in_dp = wid < ndp || per < kXRows;
    if (in_dp) {
      uint8_t* ring = smem + 2 * sizeof(double) * (size_t)pitch;
      if (iters == 0 && R.U != nullptr)
        dp_pass<true>(R, g, reinterpret_cast<double*>(smem), CL, rank, per, s_xbar, xc,
                      ring + (size_t)wid * dp_ring_bytes<true>(), &s_rbar[wid * 6], rph, wid < ndp, dprof);
      else
        dp_pass<false>(R, g, reinterpret_cast<int*>(smem), CL, rank, per, s_xbar, xc,
                       ring + (size_t)wid * dp_ring_bytes<false>(), &s_rbar[wid * 6], rph, wid < ndp, dprof);
    }
    // warps outside the DP park on a named barrier (descheduled, no issue slots taken)
    // until the DP warps are done; then everyone joins the cluster barrier
    if (in_dp)
      asm volatile("bar.arrive 1, %0;" ::"r"(blockDim.x) : "memory");
    else
      asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
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
      uint8_t* wbuf = smem + (size_t)wid * (4 * RB + kWarpScratch);
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
      if (wid < ncw && rlo + wid < rhi) issue(rlo + wid, 0);
      for (int i = rlo + wid; wid < ncw && i < rhi; i += ncw, ++kk) {
        const int slot = kk & 1;
        if (i + ncw < rhi) issue(i + ncw, slot ^ 1);
        mbar_wait(&s_bar[2 * wid + slot], phase[slot]);
        phase[slot] ^= 1u;
        const uint8_t* Ls = wbuf + (size_t)slot * 2 * RB;
        const uint8_t* Gs = Ls + RB;
        uint32_t* Lg = reinterpret_cast<uint32_t*>(R.luma + (long)i * pitch);
        uint32_t* Gg = reinterpret_cast<uint32_t*>(R.grad + (long)i * pitch);
        const int16_t* rg = log + (long)i * R.rem_cap + removed;  // sorted, old coordinates
        int16_t* lst = reinterpret_cast<int16_t*>(wbuf + 4 * RB + 1024);
        const int16_t* rr = rg;
        if (b <= kListCap) {  // stage the list: the walk below is a dependent chain
          for (int t = lane; t < b; t += 32) lst[t] = rg[t];
          __syncwarp();
          rr = lst;
        }
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
      for (int i = rlo + wid; wid < ncw && i < rhi; i += ncw) {
        uint8_t* gr = R.grad + (long)i * pitch;
        if (zero) {
          for (int y = lane; y < wn; y += 32) gr[y] = 0;
          continue;
        }
        const int ia = max(i - 1, 0), ib = min(i + 1, rows - 1);
        // rows {i-1, i, i+1}'s removed columns (sorted), staged per warp when they fit
        const int16_t* l3[3] = {log + (long)ia * R.rem_cap + removed, log + (long)i * R.rem_cap + removed,
                                log + (long)ib * R.rem_cap + removed};
        if (b <= kListCap) {
          int16_t* lst = reinterpret_cast<int16_t*>(smem + (size_t)wid * (4 * RB + kWarpScratch) + 4 * RB + 1024);
          for (int t = lane; t < 3 * b; t += 32) {
            int rs = t / b;
            lst[rs * kListCap + (t - rs * b)] = l3[rs][t - rs * b];
          }
          __syncwarp();
          l3[0] = lst;
          l3[1] = lst + kListCap;
          l3[2] = lst + 2 * kListCap;
        }
        const int16_t* ri = l3[1];
        const uint8_t* la = R.luma + (long)ia * pitch;
        const uint8_t* lb = R.luma + (long)i * pitch;
        const uint8_t* lc = R.luma + (long)ib * pitch;
        // candidates: rows {i-1, i, i+1} x seams x offsets {-1, 0, +1}, in old columns
        const int ncand = 9 * b;
        for (int q = lane; q < ncand; q += 32) {
          int rsel = q / (3 * b), rem = q - rsel * 3 * b;
          int s = rem / 3, off = rem - s * 3 - 1;
          int x = l3[rsel][s] + off;
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
        __syncwarp();  // the staged lists are reused by the next row
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
    uint8_t* wbuf = smem + (size_t)wid * (4 * RB + kWarpScratch);
    uint32_t* wv = reinterpret_cast<uint32_t*>(wbuf + 4 * RB);
    int* pre = reinterpret_cast<int*>(wbuf + 4 * RB + 512);
    for (int i = rlo + wid; wid < ncw && i < rhi; i += ncw) {
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
  if (rank == 0 && tid == 32 && R.prof)
    for (int k = 0; k < 3; ++k) R.prof[8 + k] = dprof[k];
  if (rank == 0 && tid == 0) {
    Rg.iters = iters;
    Rg.removed = removed;
    if (R.prof) {
      for (int k = 0; k < 4; ++k) R.prof[k] = prof[k];
      for (int k = 0; k < 3; ++k) R.prof[4 + k] = dprof[k];

    }
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
  // one DP warp per SM sub-partition: kDpWarps x 128 columns per CTA, at most 8 CTAs
  int cl = (width + kOwn * kDpWarps - 1) / (kOwn * kDpWarps);
  return cl < 1 ? 1 : (cl > 8 ? 8 : cl);
}

int carve_dp_warps(int width, int cl) {
  const int per = ((width + cl - 1) / cl + 15) & ~15;
  return (per + kOwn - 1) / kOwn;
}

constexpr size_t kSmemBudget = 220 * 1024;

// warps that stage rows for the compaction / gradient phases (4 staged rows each)
int carve_comp_warps(int pitch) {
  const size_t RB = (((size_t)pitch + 15) & ~(size_t)15) + 16;
  size_t n = kSmemBudget / (4 * RB + kWarpScratch);
  return (int)(n > (size_t)kMaxWarps ? kMaxWarps : n);
}

size_t carve_smem_bytes(int rows, int pitch, bool stage, int warps, int dp_warps) {
  const int nblk = (rows - 1 + kBlockRows - 1) / kBlockRows;
  size_t dp = 2 * sizeof(double) * (size_t)pitch + (size_t)dp_warps * dp_ring_bytes<true>();
  size_t sel = (size_t)pitch * (8 + 8 + 4 * 4) + 16;
  if (stage) sel += (size_t)nblk * pitch;
  const size_t RB = (((size_t)pitch + 15) & ~(size_t)15) + 16;
  size_t comp = (size_t)warps * (4 * RB + kWarpScratch);
  size_t m = dp > sel ? dp : sel;
  return m > comp ? m : comp;
}

int carve_warps(int width, int cl) { return carve_dp_warps(width, cl); }

bool carve_stage_dtab(int rows, int pitch, int cl) {
  return carve_smem_bytes(rows, pitch, true, carve_comp_warps(pitch), carve_dp_warps(pitch, cl)) <= kSmemBudget;
}

void launch_carve_cluster(CarveRun* runs_d, int nruns, int rows, int pitch, int width, int cl, cudaStream_t st) {
  if (nruns == 0) return;
  // the DP needs carve_dp_warps() warps (128 owned columns each); the row-parallel phases
  // use every warp, so the CTA always runs kMaxWarps (DP-idle warps skip the DP)
  const int dpw = carve_dp_warps(width, cl);
  SCPL_ARG(dpw <= kMaxWarps, "carve width too large for the cluster size");
  const int warps = kMaxWarps;
  const int ncw = carve_comp_warps(pitch);
  SCPL_ARG(ncw >= 1, "carve plane too wide for the compaction stage");
  const bool stage = carve_stage_dtab(rows, pitch, cl);
  size_t smem = carve_smem_bytes(rows, pitch, stage, ncw, dpw);
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
  SCPL_CUDA(cudaLaunchKernelEx(&cfg, carve_cluster_kernel, runs_d, cl, ncw));
  SCPL_CHECK_LAUNCH();
}

}  // namespace scpl
