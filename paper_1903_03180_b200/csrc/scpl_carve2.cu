// K4-K7: the SCPL carve loop of a run -- one cluster kernel per DP pass plus row kernels.
//
// Replaces batch_carve (batching.py:118-153) with everything it calls: cumulative_energy
// (seams.py:39-65), label_parents (batching.py:39-46), select_batch (:49-73),
// trace_columns (seams.py:68-81), remove_batch on the representative frame (:76-107) and
// default_energy (:110-115).
//
// One thread-block cluster of CL CTAs (CL SMs) carves one run; runs are independent, so a
// launch holds every run of a carve group (grid = runs x CL).  Per pass (carve_pass_kernel):
//
//  1. DP, column-split.  Each DP warp owns kOwn columns (128 / 64 / 32 for the kc6 / kc4 / kc3
//     builds) and computes a window 64 columns wider for 32 rows without any barrier:
//     neighbours come from register shuffles, the window's valid region shrinks by one column
//     per row, and after 32 rows exactly the owned columns remain valid ("trapezoid" tiling).
//     Every 32 rows warps publish their owned cumulative energies to shared memory -- and the
//     32 columns next to a CTA edge into the neighbour CTA with st.async on its mbarrier.  The
//     reference's argmin-first tie-break (seams.py:62) is strict '<' in the order -1, 0, +1.
//     First pass of a buffered run: float64 on the uniform map (IEEE adds, no FMA), carrying
//     path words; later passes: packed int keys on gradient energy (integer-valued, so
//     bit-identical) with per-column choice words.  Block-end words and landing deltas go to
//     global memory through helper warps.
//  2. Select + trace (select_trace, every CTA redundantly): labels by chaining the landing
//     deltas bottom-up (table staged in shared memory), per-parent leftmost minimum via
//     shared-memory atomics (labels are monotone, so parents are segments), k-truncation by
//     (cost, col), then each CTA decodes its share of (seam, block) pairs into the
//     removed-column log.
// Between passes (row kernels, whole GPU):
//  3. Compact (carve_compact_kernel): luma and gradient drop the batch's columns in place.
//  4. Gradient (carve_dirty_kernel), incremental: a pixel's Sobel value changes only if a
//     removed pixel of rows i-1..i+1 lay within one column of it; only those are recomputed.
// The original-column index map is rebuilt once per run at the end (carve_index_kernel).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <climits>

#include "scpl_common.cuh"
#include "scpl_kernels.h"

// Compiled twice (build_ext.py): SCPL_KC = 6 (namespace scpl::kc6, the default: 128 owned
// columns per DP warp, fewest SMs per run) and SCPL_KC = 4 (scpl::kc4: 64 owned columns, a third
// fewer instructions per DP row on twice the SMs -- for runs carved alone, where SMs are free).
#ifndef SCPL_KC
#define SCPL_KC 6
#endif
#if SCPL_KC == 4
#define SCPL_KC_NS kc4
#elif SCPL_KC == 3
#define SCPL_KC_NS kc3
#else
#define SCPL_KC_NS kc6
#endif

namespace scpl {
namespace SCPL_KC_NS {

constexpr int kC = SCPL_KC;                       // columns per lane in a DP warp window
constexpr int kWin = 32 * kC;                     // 192-column window (kC = 6)
constexpr int kXRows = 32;                        // rows between boundary exchanges (= halo)
constexpr int kOwn = kWin - 2 * kXRows;           // 128 owned columns per DP warp (kC = 6)
constexpr int kDpWarps = 4;                       // DP warps per CTA: one per SM sub-partition
constexpr int kRingW = kWin + 16;                 // ring row: a 16-aligned superset of the window
constexpr int kIntInf = 0x3fffffff;
constexpr int kMaxWarps = 8;                     // 256 threads (<= 128 registers): room on the SM for row and scan CTAs

// Fine-grained DP timers (SCPL_CARVE_PROF builds only): clock64 reads and a local-memory
// accumulator array would otherwise sit on the DP's critical path.
#ifdef SCPL_CARVE_PROF
#define DP_CLOCK() clock64()
#define DP_PROF(i, v) (dprof[i] += (v))
#else
#define DP_CLOCK() 0ll
#define DP_PROF(i, v) ((void)0)
#endif
// select sub-phase timers (thread 0 of each CTA; SCPL_CARVE_PROF builds): slots 12..16
#ifdef SCPL_CARVE_PROF
#define SEL_PROF(k)                                   \
  do {                                                \
    if (tid == 0 && R.prof) {                         \
      const long long t_ = clock64();                 \
      atomicAdd((unsigned long long*)&R.prof[12 + (k)], (unsigned long long)(t_ - ts)); \
      ts = t_;                                        \
    }                                                 \
  } while (0)
#else
#define SEL_PROF(k) ((void)0)
#endif

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
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
// remote store that completes 4/8 bytes on the target CTA's mbarrier (no fence needed)
__device__ __forceinline__ void st_async_remote(const int* local_dst, int v, uint64_t* local_bar, uint32_t rank) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                   map_rank(local_dst, rank)),
               "r"(v), "r"(map_rank(local_bar, rank))
               : "memory");
}
__device__ __forceinline__ void st_async_remote(const double* local_dst, double v, uint64_t* local_bar,
                                                uint32_t rank) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                   map_rank(local_dst, rank)),
               "l"(__double_as_longlong(v)), "r"(map_rank(local_bar, rank))
               : "memory");
}
__device__ __forceinline__ uint32_t lds32_u(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t lds64_u(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds_s8(uint32_t a) {
  int v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t map_rank_pure(const void* p, uint32_t rank) {
  uint32_t out;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void st_async_addr(uint32_t raddr, int v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_addr(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
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

__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

// A DP warp's block-end staging (choice / path words, dir sums, then a 4-word header holding
// the block index and row count), double buffered when a helper warp stores it.
constexpr int kPwStageWords = 3 * kWin + 4;  // 64-bit words, dir sums, header
// Int-pass keys: K = ce << kKeyShift | dir << kDirShift | sumdir (the dir sum of the path within
// the current 32-row block, <= 64: 7 bits).
constexpr int kKeyShift = 9, kDirShift = 7, kSumMask = (1 << kDirShift) - 1;
constexpr int kSubRows = 16;  // int passes: rows per 32-bit choice word (two per block)

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
  static constexpr int kStageRows = 4, kStages = 3;   // fp64 rows are 8x larger: finer ring
};
template <bool F64>
__host__ __device__ constexpr size_t dp_ring_bytes() {
  return (size_t)DpCfg<F64>::kStages * DpCfg<F64>::kStageRows * kRingW * (F64 ? 8 : 1);
}

// issue stage `st` (rows 1 + st*RS ...) of this warp's energy window into ring slot st % S:
// one 2-D TMA box (kRingW columns from the 16-aligned column at or below the window start,
// RS rows); out-of-range columns and rows land as 0
template <bool F64>
__device__ __forceinline__ void dp_issue_stage(const CarveRun& Rg, int plane, int rows, int st, int win_lo,
                                               uint8_t* ring, uint64_t* bars) {
  constexpr int RS = DpCfg<F64>::kStageRows, S = DpCfg<F64>::kStages;
  constexpr int sz = F64 ? 8 : 1;
  const int slot = st % S;
  const int i0 = 1 + st * RS;
  if (i0 >= rows) return;
  fence_proxy_async_global();
  mbar_arrive_tx(&bars[slot], (uint32_t)(RS * kRingW * sz));
  tma_load_2d(ring + (size_t)slot * RS * kRingW * sz, F64 ? &Rg.tm_U : &Rg.tm_grad[plane], win_lo & ~15, i0,
              &bars[slot]);
}

// one DP row for a lane's kC columns (seams.py:54-64): strict '<' in the order -1, 0, +1
// float64 pass (first pass of a buffered run): ce values with path words pw carried along
// (2 bits per row of the seam ending in the column).
template <bool F64, bool EDGE>
__device__ __forceinline__ void dp_row(typename Val<F64>::T (&ce)[kC], uint64_t (&pw)[kC],
                                       const uint8_t* erow, const bool (&in)[kC], int lane) {
  using V = Val<F64>;
  using T = typename V::T;
  T e[kC];
  if constexpr (F64) {
    const double* p = reinterpret_cast<const double*>(erow) + lane * kC;
#pragma unroll
    for (int k = 0; k < kC; ++k) e[k] = p[k];
  } else {
    const uint8_t* p = erow + lane * kC;
#pragma unroll
    for (int k = 0; k < kC; ++k) e[k] = (int)p[k];
  }
  T left = __shfl_up_sync(0xffffffffu, ce[kC - 1], 1);
  T right = __shfl_down_sync(0xffffffffu, ce[0], 1);
  uint64_t pleft = __shfl_up_sync(0xffffffffu, pw[kC - 1], 1);
  uint64_t pright = __shfl_down_sync(0xffffffffu, pw[0], 1);
  if (lane == 0) left = V::inf();
  if (lane == 31) right = V::inf();
  T nce[kC];
  uint64_t npw[kC];
#pragma unroll
  for (int k = 0; k < kC; ++k) {
    T l = k > 0 ? ce[k - 1] : left;
    T c = ce[k];
    T r = k + 1 < kC ? ce[k + 1] : right;
    uint64_t pl = k > 0 ? pw[k - 1] : pleft;
    uint64_t pc = pw[k];
    uint64_t pr = k + 1 < kC ? pw[k + 1] : pright;
    bool p1 = c < l;
    T m = p1 ? c : l;
    uint64_t ps = p1 ? pc : pl;
    uint32_t code = p1 ? 1u : 0u;
    bool p2 = r < m;
    m = p2 ? r : m;
    ps = p2 ? pr : ps;
    code = p2 ? 2u : code;
    T v = V::add(e[k], m);
    nce[k] = (!EDGE || in[k]) ? v : V::inf();
    npw[k] = (ps << 2) | (uint64_t)code;
  }
#pragma unroll
  for (int k = 0; k < kC; ++k) {
    ce[k] = nce[k];
    pw[k] = npw[k];
  }
}

// int32 passes: one packed key per column, K = ce << 9 | dir << 7 | sumdir.  The three
// candidates of a cell are K[j-1] (dir 0), K[j] + 129 (dir 1) and K[j+1] + 258 (dir 2); their
// minimum is the minimum cost with ties going to the lower dir -- exactly the reference's
// strict '<' in the order -1, 0, +1 (seams.py:54-64) -- and carries the predecessor's sum of
// dirs within the current 32-row block, so the block's landing delta (sumdir - rows) needs
// no path word.  cw collects this column's own dir per row (the choice word, latest row in
// the low bits); the trace walks the choice words of the columns a seam visits.
// MASK (bit 0: left, bit 1: right): the window's left / right end is an image border (always
// both with the EDGE layout): the lane at that end sees +inf beyond it.  Any other window end
// is a decaying halo -- whatever value enters there reaches at most column r of the window after
// r rows, never the owned columns (kXRows in from each end) within a 32-row block -- so it takes
// the shuffled key unmasked, and the neighbour keys enter the minimum last (one dependent op
// per row after the shuffle).
template <bool EDGE, int MASK>
__device__ __forceinline__ void dp_row_key(int (&K)[kC], uint32_t (&cw)[kC], const uint8_t* erow,
                                           const bool (&in)[kC], int lane) {
  int e[kC];
  const uint8_t* p = erow + lane * kC;
#pragma unroll
  for (int k = 0; k < kC; ++k) e[k] = (int)p[k];
  int left = __shfl_up_sync(0xffffffffu, K[kC - 1], 1);
  int right = __shfl_down_sync(0xffffffffu, K[0], 1);
  if ((MASK & 1) && lane == 0) left = kIntInf;
  if ((MASK & 2) && lane == 31) right = kIntInf;
  int n[kC];
#pragma unroll
  for (int k = 0; k < kC; ++k) {
    // the candidates' biases add dir to the dir field and to the dir sum at once (sumdir + dir
    // <= 64 + 2 never carries into the dir field, so ties still go to the lower dir); the new
    // key is the minimum with its dir field cleared plus the energy.  The lane's own candidates
    // are combined first, the shuffled neighbour last (integer min: the order does not matter)
    constexpr int kBc = (1 << kDirShift) + 1, kBr = (2 << kDirShift) + 2;
    int m;
    if (kC == 1) {
      m = min(min(K[0] + kBc, right + kBr), left);
    } else if (k == 0) {
      m = min(min(K[0] + kBc, K[1] + kBr), left);
    } else if (k == kC - 1) {
      m = min(min(K[k - 1], K[k] + kBc), right + kBr);
    } else {
      m = min(min(K[k - 1], K[k] + kBc), K[k + 1] + kBr);
    }
    const int d = m & (3 << kDirShift);
    int v;  // m - d + e * 512 as two multiply-adds (FMA pipe; the ALU pipe is the DP's bottleneck)
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(v) : "r"(e[k]), "r"(1 << kKeyShift), "r"(m));
    asm("mad.lo.s32 %0, %1, -1, %2;" : "=r"(v) : "r"(d), "r"(v));
    n[k] = (!EDGE || in[k]) ? v : kIntInf;
    cw[k] = cw[k] * 4u + __umulhi((uint32_t)d, 1u << (32 - kDirShift));  // d >> kDirShift
  }
#pragma unroll
  for (int k = 0; k < kC; ++k) K[k] = n[k];
}

// one row of either pass (the fp64 pass always masks)
template <bool F64, bool EDGE, int MASK, class PW>
__device__ __forceinline__ void dp_step(typename Val<F64>::T (&ce)[kC], PW (&pw)[kC], const uint8_t* erow,
                                        const bool (&in)[kC], int lane) {
  if constexpr (F64)
    dp_row<true, EDGE>(ce, pw, erow, in, lane);
  else
    dp_row_key<EDGE, MASK>(ce, pw, erow, in, lane);
}

// One DP pass for this warp's window.  ceX: smem exchange rows [2][pitch]; ring: this
// warp's energy ring; bars: its S ring mbarriers (phase bits in rph); xbar/xc: the
// neighbour-exchange barriers and exchange counter (buffer = xc & 1, parity = (xc>>1) & 1).
// Exchange blocks of 32 rows: when every CTA owns >= 32 columns only adjacent CTAs supply
// halo and each CTA waits on its own mbarrier for its warps plus the adjacent CTAs' warps
// (release/acquire at cluster scope).  Tiny widths fall back to a cluster barrier.
// halo bytes a CTA receives per exchange at width w: the adjacent CTAs' owned columns
// within 32 of its own range (only adjacent CTAs reach when every CTA owns >= 32 columns)
__device__ __forceinline__ uint32_t halo_bytes_for(int w, int CL, uint32_t rank, int sz) {
  const int per = ((w + CL - 1) / CL + 15) & ~15;
  const int lo_me = min(w, (int)rank * per), hi_me = min(w, lo_me + per);
  uint32_t bytes = 0;
  for (int q = (int)rank - 1; q <= (int)rank + 1; q += 2) {
    if (q < 0 || q >= CL) continue;
    int lo = min(w, q * per), hi = min(w, lo + per);
    int a = max(lo, lo_me - kXRows), b = min(hi, hi_me + kXRows);
    if (b > a) bytes += (uint32_t)((b - a) * sz);
  }
  return bytes;
}

// Global stores of one staged block end (the lane-contiguous words transposed through the
// staging row so the stores coalesce): owned columns' words and landing deltas.
// stg: 64-bit words of the window's columns (2 bits per row, the block's last row in the low
// bits), then their dir sums (int passes), then the header.
template <bool F64>
__device__ __forceinline__ void store_block_end(const CarveRun& R, const Geo& g, const uint32_t* stg, int pbi,
                                                int nrb) {
  const int lane = threadIdx.x & 31;
  const uint64_t* w64 = reinterpret_cast<const uint64_t*>(stg);
  uint64_t* gpw = R.pw + (long)pbi * R.pitch + g.win_lo;
  int8_t* gdl = R.delta + (long)pbi * R.pitch + g.win_lo;
#pragma unroll
  for (int k = 0; k < kC; ++k) {
    const int c = lane + 32 * k;
    const int j = g.win_lo + c;
    if (j >= g.own_lo && j < g.own_hi) {  // (transposed column: not this lane's own[])
      const uint64_t word = w64[c];
      gpw[c] = word;
      const int sumdir = F64 ? __popcll(word & 0x5555555555555555ull) + 2 * __popcll(word & 0xAAAAAAAAAAAAAAAAull)
                             : (int)stg[2 * kWin + c];
      gdl[c] = (int8_t)(sumdir - nrb);
    }
  }
}

// Helper warp of one DP warp: performs its block-end global stores (the DP warp only fills a
// staging buffer and moves on).  hbar: full[2] (32 DP-lane arrivals), empty[2] (32 helper-
// lane arrivals); a header of ~0 ends the pass.
template <bool F64>
__device__ __forceinline__ bool pw_service(const CarveRun& R, const Geo& g, const uint32_t* stage, uint64_t* hbar,
                                           uint32_t& n) {
  mbar_wait_sleep(&hbar[n & 1], (n >> 1) & 1);
  const uint32_t* stg = stage + (n & 1) * kPwStageWords;
  const uint32_t hdr = stg[3 * kWin];
  if (hdr == 0xffffffffu) return false;
  store_block_end<F64>(R, g, stg, (int)hdr, (int)stg[3 * kWin + 1]);
  mbar_arrive(&hbar[2 + (n & 1)]);
  ++n;
  return true;
}
template <bool F64>
__device__ void pw_helper(const CarveRun& R, const Geo& g, const uint32_t* stage, uint64_t* hbar) {
  uint32_t n = 0;
  while (pw_service<F64>(R, g, stage, hbar, n)) {
  }
}

// ------------------------------------------------------------------ fused producer (int passes)
// default_energy (batching.py:110-115) of the carved frame without compaction / gradient
// kernels: while the DP warps work on block k, the producer warps build block k+1's energy rows
// for this CTA's windows.  Per row: the previous batch (remove_batch, batching.py:76-107) is
// removed from the source luma plane row (only the columns the CTA's windows need, +-1), the
// compacted row goes to a luma ring in shared memory (and the CTA's own columns to the other
// luma plane, for the next pass), then the Sobel energy (energy.py:40-59, edge replication)
// of the ring rows goes into the DP's energy ring.  Luma of a pixel commutes with compaction,
// so this is default_energy of the carved RGB frame.
// The fused pass kernel has kFusedWarps warps: warpgroup 0 = the DP warps (setmaxnreg: 128
// registers), warpgroups 1-2 = kProdWarps producer warps (56 registers); producer q < 4 also
// stores DP warp q's block ends (helper duty).  Launch allocation: 80 registers per thread.
constexpr int kFusedWarps = 12;
constexpr int kProdWarps = 8;
constexpr int kProdFirst = 4;   // first producer warp
constexpr int kRegDp = 128, kRegProd = 56, kRegFused = 80;
constexpr int kLumRing = 34;    // luma ring rows: block k's Sobel needs rows 32k .. 32k+33
constexpr int kProdBar = 3;     // named barrier of the producer warps
// Every input of a producer (the source luma rows, the previous batch's removed columns) exists
// when the pass starts, so the producers stage block k+1's inputs with cp.async while they
// work on block k: per compaction row the source columns the CTA needs (a superset fixed per
// pass: the new columns [d0, d1) come from [d0, d1 + b)) and the row's removed-column list.
// Batches larger than kProdBcap read global memory directly (slower, same results).
constexpr int kProdBcap = 64;
constexpr int kStageRows = 34;  // compaction rows per block (block 0: rows 0 .. 33)
__host__ __device__ inline int fused_stage_sw(int rw) { return (rw + 48 + kProdBcap + 15) & ~15; }
__host__ __device__ inline int fused_stage_slot(int rw) { return fused_stage_sw(rw) + 2 * kProdBcap + 32; }

struct ProdGeo {
  int g_lo;   // image column of energy-ring column 0 (16-aligned, may be negative)
  int rw;     // energy-ring row stride; luma-ring row stride rw + 32 (column c <-> image c + g_lo - 16)
  int cta_lo, cta_hi;
};

// the CTA's energy columns [g_lo, g_hi) at width w: the union of its active DP warps' windows
__host__ __device__ inline bool fused_cta_range(int w, int CL, int rank, int& g_lo, int& g_hi) {
  const int per = ((w + CL - 1) / CL + 15) & ~15;
  const int cta_lo = w < rank * per ? w : rank * per;
  const int cta_hi = w < cta_lo + per ? w : cta_lo + per;
  bool any = false;
  for (int dw = 0; dw < kMaxWarps; ++dw) {
    const int own_lo = cta_lo + dw * kOwn;
    const int own_hi = cta_hi < own_lo + kOwn ? cta_hi : own_lo + kOwn;
    if (own_lo >= own_hi) break;
    int wl = own_lo - kXRows;
    if (w >= kWin) wl = wl < 0 ? 0 : (wl > w - kWin ? w - kWin : wl);
    const int lo = wl & ~15, hi = wl + kWin;
    if (!any || lo < g_lo) g_lo = lo;
    if (!any || hi > g_hi) g_hi = hi;
    any = true;
  }
  return any;
}

// DP-phase shared memory of a fused int pass: exchange rows (2 x 4 B x pitch), the helper
// staging of kProdWarps DP warps, the energy ring (1 + 2 x 32 rows of rw), the luma ring
// (kLumRing rows of rw + 32), the per-row breakpoint table, two blocks of staged inputs
__host__ __device__ inline size_t fused_off_stage(int pitch) { return 8 * (size_t)pitch; }
__host__ __device__ inline size_t fused_off_ering(int pitch) {
  return fused_off_stage(pitch) + (size_t)kDpWarps * 2 * kPwStageWords * 4;
}
__host__ __device__ inline size_t fused_off_lring(int pitch, int rw) {
  return fused_off_ering(pitch) + (size_t)(1 + 2 * kXRows) * rw;
}
__host__ __device__ inline size_t fused_off_rowtab(int pitch, int rw) {
  return fused_off_lring(pitch, rw) + (size_t)kLumRing * (rw + 32);
}
__host__ __device__ inline size_t fused_off_pstage(int pitch, int rw) {
  return fused_off_rowtab(pitch, rw) + ((kStageRows * 8 + 15) & ~15);
}
__host__ __device__ inline size_t fused_dp_bytes(int pitch, int rw) {
  return fused_off_pstage(pitch, rw) + (size_t)2 * kStageRows * fused_stage_slot(rw);
}

__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint32_t lds32p(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// (no "memory" clobber: the producers' shared-memory phases are ordered by prod_bar, whose asm
// is a compiler barrier; a clobber here would force every CarveRun field to be re-read)
__device__ __forceinline__ uint32_t lds16p(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32p(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void prod_bar() {
  asm volatile("bar.sync %0, %1;" ::"n"(kProdBar), "n"(kProdWarps * 32) : "memory");
}

// One luma row's horizontal Sobel terms around 4 columns (even / odd columns in 16-bit lanes):
// S = l + 2m + r and D = r - l + 256, from the luma-ring words at a - 4, a, a + 4.
__device__ __forceinline__ void sobel_prep(uint32_t a, uint32_t& se, uint32_t& so, uint32_t& de, uint32_t& dO) {
  const uint32_t lo = lds32p(a - 4), mid = lds32p(a), hi = lds32p(a + 4);
  const uint32_t wl = __byte_perm(lo, mid, 0x6543);  // columns -1 .. 2
  const uint32_t wr = __byte_perm(mid, hi, 0x4321);  // columns 1 .. 4
  const uint32_t le = __byte_perm(wl, 0, 0x4240), lo_ = __byte_perm(wl, 0, 0x4341);
  const uint32_t me = __byte_perm(mid, 0, 0x4240), mo = __byte_perm(mid, 0, 0x4341);
  const uint32_t re = __byte_perm(wr, 0, 0x4240), ro = __byte_perm(wr, 0, 0x4341);
  se = le + 2u * me + re;
  so = lo_ + 2u * mo + ro;
  de = re + 0x01000100u - le;
  dO = ro + 0x01000100u - lo_;
}

// The producer warps of a fused int pass (tp = 0 .. 255 over kProdWarps warps).  Per block k
// (DP rows 1+32k .. 32k+32), all producer threads share every phase:
//   wait for block k's staged inputs, stage block k+1 (cp.async: the source columns the CTA
//   needs, [d0, d1 + b), and the removed-column lists of compaction rows a0(k) .. a1(k));
//   A1 warp per row: the previous batch's breakpoints a_t = rr[t] - t below / inside [d0, d1)
//      by ballots, then lane per 4-column word: source shift s(y) = #{a_t <= y}, one funnel
//      shift of two staged words (byte-wise where s changes inside the word) into the luma ring;
//   A2 edge replication (np.pad "edge"), the CTA's own columns to the next plane;
//   wait until the DP is done with the slot's previous block; B Sobel (8-row streams, lane per
//   4-column word) from the luma ring into the energy ring; full[slot]; helper duty.
// Compaction rows: block 0 rows 0 .. 33, block k rows 32k+2 .. 32k+33 (block k's Sobel needs
// luma rows 32k .. 32k+33; the luma ring holds kLumRing = 34 rows).
__device__ void produce_pass(const CarveRun& R, int w, int b, int off, const ProdGeo& P, uint8_t* ering,
                             uint8_t* lring, uint8_t* pstage, uint64_t* full, uint64_t* empty, int tp, bool helper,
                             const Geo& hg, const uint32_t* hstage, uint64_t* hbar, bool active_cta,
                             long long* prof) {
  constexpr int NT = kProdWarps * 32;
  // (SCPL_PROF: producer thread 0 of rank 0 times its phases into prof[17..25])
  long long pt = prof ? clock64() : 0;
  auto ph = [&](int i) {
    if (prof) {
      const long long u = clock64();
      prof[17 + i] += u - pt;
      pt = u;
    }
  };
  // every CarveRun field in registers (the cp.async / barrier asm are compiler barriers)
  const int rows = R.rows, pitch = R.pitch, rw = P.rw, lw = P.rw + 32, lo = P.g_lo - 16;
  const int g_lo = P.g_lo, cta_lo = P.cta_lo, cta_hi = P.cta_hi;
  const int16_t* const rem = R.rem;
  const long rem_cap = R.rem_cap;
  const uint8_t* src = R.luma[R.lsel];
  uint8_t* dst = R.luma[R.lsel ^ 1];
  const int nstage = active_cta ? (rows - 1 + kXRows - 1) / kXRows : 0;
  const int d0 = max(g_lo - 1, 0), d1 = min(g_lo + rw + 1, w);
  const int y0 = d0 & ~3;
  const bool staged = b <= kProdBcap;
  const int X0 = d0 & ~15, X1 = min((d1 + b + 15) & ~15, pitch);
  const int nch = (X1 - X0) >> 4;                 // staged 16-byte source chunks per row
  const int ncr = b > 0 ? (b + 14) / 8 + 1 : 0;   // staged 16-byte removed-list chunks per row
  const int per_row = nch + ncr;
  const int sw = fused_stage_sw(rw), slot = fused_stage_slot(rw);
  const bool tiny = rows < 3 || w < 3;  // zero energy below the 3x3 Sobel domain
  const int lane = tp & 31, pw = tp >> 5;  // producer warp 0 .. kProdWarps-1
  const int fdbg = R.fdbg;
  auto a0f = [&](int k) { return k == 0 ? 0 : kXRows * k + 2; };
  auto a1f = [&](int k) { return min(kXRows * k + 34, rows); };
  auto erow = [&](int r) -> uint8_t* {
    return ering + (size_t)(r == 0 ? 0 : 1 + kXRows * (((r - 1) / kXRows) & 1) + (r - 1) % kXRows) * rw;
  };
  auto stage_block = [&](int k) {
    if (staged && k < nstage) {
      uint8_t* buf = pstage + (size_t)(k & 1) * kStageRows * slot;
      const int r0 = a0f(k), nr = a1f(k) - r0;
      for (int p = tp; p < nr * per_row; p += NT) {
        const int j = p / per_row, c = p - j * per_row;
        uint8_t* sl = buf + (size_t)j * slot;
        if (c < nch)
          cp_async16(sl + 16 * c, src + (size_t)(r0 + j) * pitch + X0 + 16 * c);
        else
          cp_async16(sl + sw + 16 * (c - nch), rem + (((long)(r0 + j) * rem_cap + off) & ~7L) + 8 * (c - nch));
      }
    }
    cp_async_commit();
  };
  uint32_t hn = 0;
  bool hdone = !helper;
  const uint32_t lsm = smem_u32(lring);
  stage_block(0);
  for (int k = 0; k < nstage; ++k) {
    cp_async_wait<0>();
    prod_bar();  // block k's staged rows (every thread's copies) are visible
    ph(0);
    if (!(fdbg & 4)) stage_block(k + 1);
    ph(1);
    const uint8_t* buf = pstage + (size_t)(k & 1) * kStageRows * slot;
    const int r0 = a0f(k), nr = a1f(k) - r0;
    // A1: warp per row
    for (int j = pw; j < nr && !(fdbg & 8); j += kProdWarps) {
      long long tq0 = prof ? clock64() : 0;
      const long e = (long)(r0 + j) * rem_cap + off;
      const int16_t* rr = staged ? reinterpret_cast<const int16_t*>(buf + (size_t)j * slot + sw) + (e & 7L) : rem + e;
      // breakpoints: lane t holds a_t (t < 64 in registers; larger batches walk rr)
      const uint32_t rrs = smem_u32(rr);
      int alo = INT_MAX, ahi = INT_MAX;
      if (staged) {
        if (lane < b) alo = (int)(int16_t)lds16p(rrs + 2 * lane) - lane;
        if (lane + 32 < b) ahi = (int)(int16_t)lds16p(rrs + 2 * (lane + 32)) - (lane + 32);
      } else {
        if (lane < b) alo = (int)rr[lane] - lane;
        if (lane + 32 < b) ahi = (int)rr[lane + 32] - (lane + 32);
      }
      SCPL_DCHECK(lane >= b || ((int)rr[lane] >= lane && (int)rr[lane] < w + b && (lane == 0 || rr[lane - 1] < rr[lane])),
                  "removed columns disjoint and in range (fused)");
      int n_lt, m;
      if (b <= 32) {
        n_lt = __popc(__ballot_sync(0xffffffffu, alo < d0));
        m = __popc(__ballot_sync(0xffffffffu, alo < d1)) - n_lt;
      } else if (b <= 64) {
        n_lt = __popc(__ballot_sync(0xffffffffu, alo < d0)) + __popc(__ballot_sync(0xffffffffu, ahi < d0));
        m = __popc(__ballot_sync(0xffffffffu, alo < d1)) + __popc(__ballot_sync(0xffffffffu, ahi < d1)) - n_lt;
      } else {
        n_lt = 0;
        m = 0;
        for (int t = lane; t < b; t += 32) {
          const int a = (int)rr[t] - t;
          n_lt += a < d0;
          m += a >= d0 && a < d1;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          n_lt += __shfl_xor_sync(0xffffffffu, n_lt, o);
          m += __shfl_xor_sync(0xffffffffu, m, o);
        }
      }
      // the first (up to) 2 in-range breakpoints in warp-uniform registers; more: walk rr
      const bool few = m <= 2 && b <= 64;
      int bp0 = INT_MAX, bp1 = INT_MAX;
      if (few && m >= 1) {
        const int t = n_lt;
        bp0 = t < 32 ? __shfl_sync(0xffffffffu, alo, t & 31) : __shfl_sync(0xffffffffu, ahi, t & 31);
        if (m >= 2) {
          const int t1 = n_lt + 1;
          bp1 = t1 < 32 ? __shfl_sync(0xffffffffu, alo, t1 & 31) : __shfl_sync(0xffffffffu, ahi, t1 & 31);
        }
      }
      const uint8_t* sr = buf + (size_t)j * slot;  // staged: source column x at sr[x - X0]
      const uint8_t* gsr = src + (size_t)(r0 + j) * pitch;
      const uint32_t srs = smem_u32(sr), lrs = lsm + (uint32_t)(((r0 + j) % kLumRing) * lw - lo);
      if (prof) {
        const long long u = clock64();
        prof[27] += u - tq0;
        tq0 = u;
      }
      auto shift_at = [&](int y) {  // s(y) = #{a_t <= y}
        if (few) return n_lt + (bp0 <= y) + (bp1 <= y);
        int sy = n_lt;
        for (int t = n_lt; t < n_lt + m; ++t) sy += (int)rr[t] - t <= y;
        return sy;
      };
      for (int y4 = y0 + 4 * lane; y4 < d1 && !(fdbg & 1); y4 += 128) {
        int s0 = n_lt, s3 = n_lt;
        if (m > 0) {
          s0 = shift_at(y4);
          s3 = shift_at(y4 + 3);
        }
        uint32_t v;
        if (staged && s0 == s3) {
          const int x = y4 + s0 - X0;
          const uint32_t a = srs + (uint32_t)(x & ~3);
          v = __funnelshift_r(lds32p(a), lds32p(a + 4), (uint32_t)(x & 3) * 8u);
        } else {  // the shift changes inside the word (or an unstaged row): byte by byte
          const int xs[4] = {y4 + s0, y4 + 1 + shift_at(y4 + 1), y4 + 2 + shift_at(y4 + 2), y4 + 3 + s3};
          v = 0u;
          if (staged) {
#pragma unroll
            for (int u = 0; u < 4; ++u) v |= (uint32_t)sr[xs[u] - X0] << (8 * u);
          } else {
            const int w0 = w + b;
#pragma unroll
            for (int u = 0; u < 4; ++u) v |= (xs[u] < w0 ? (uint32_t)gsr[xs[u]] : 0u) << (8 * u);
          }
        }
        sts32p(lrs + (uint32_t)y4, v);
      }
      __syncwarp();
      if (prof) {
        const long long u = clock64();
        prof[28] += u - tq0;
        tq0 = u;
      }
      // edge replication (np.pad "edge") of this row: the same warp wrote it
      if (d0 == 0 || d1 == w) {
        uint8_t* lrow = lring + (size_t)((r0 + j) % kLumRing) * lw;
        if (d0 == 0) {
          const uint8_t v = lrow[-lo];
          for (int c = lane; c < -lo; c += 32) lrow[c] = v;
        }
        if (d1 == w) {
          const uint8_t v = lrow[w - 1 - lo];
          for (int c = w - lo + lane; c < lw; c += 32) lrow[c] = v;
        }
      }
      if (prof) prof[29] += clock64() - tq0;
    }
    if (prof) prof[30] += clock64() - pt;
    prod_bar();
    ph(3);
    if (fdbg & 4) stage_block(k + 1);
    // A2: the CTA's own columns to the next plane in 16-byte chunks (cta_lo and its ring column
    // are 16-aligned; the last CTA may write up to 15 bytes past w -- never read)
    {
      const int nco = (cta_hi - cta_lo + 15) >> 4, c0 = cta_lo - lo;
      for (int p = tp; p < nr * nco; p += NT) {
        const int j = p / nco, c = p - j * nco;
        *reinterpret_cast<uint4*>(dst + (size_t)(r0 + j) * pitch + cta_lo + 16 * c) =
            *reinterpret_cast<const uint4*>(lring + (size_t)((r0 + j) % kLumRing) * lw + c0 + 16 * c);
      }
    }
    ph(4);
    if (k >= 2) mbar_wait_sleep(&empty[k & 1], ((k >> 1) - 1) & 1);
    ph(5);
    // B: Sobel of the block's rows (block 0 also row 0): groups of 8 rows, each shared by two
    // warps (interleaved 4-column words), rows streamed
    {
      const int s0 = k == 0 ? 0 : 1 + kXRows * k, s1 = min(1 + kXRows * (k + 1), rows);
      const int ngr = (s1 - s0 + 7) >> 3;
      for (int g = pw >> 1; g < ngr; g += kProdWarps / 2) {
        const int ra = s0 + 8 * g, rb = min(ra + 8, s1);
        for (int c = 4 * (lane + 32 * (pw & 1)); c < rw; c += 256) {
          if (tiny) {
            for (int r = ra; r < rb; ++r) *reinterpret_cast<uint32_t*>(erow(r) + c) = 0u;
            continue;
          }
          auto la = [&](int r) { return lsm + (uint32_t)((r % kLumRing) * lw + c + 16); };
          uint32_t SEa, SOa, DEa, DOa, SEb, SOb, DEb, DOb;
          sobel_prep(la(max(ra - 1, 0)), SEa, SOa, DEa, DOa);
          sobel_prep(la(ra), SEb, SOb, DEb, DOb);
          auto one = [&](int r) {
            uint32_t SEc, SOc, DEc, DOc;
            sobel_prep(la(min(r + 1, rows - 1)), SEc, SOc, DEc, DOc);
            const uint32_t gxe = DEa + 2u * DEb + DEc, gxo = DOa + 2u * DOb + DOc;
            const uint32_t gye = SEc + 0x04000400u - SEa, gyo = SOc + 0x04000400u - SOa;
            const uint32_t ae = __vmaxu2(gxe, 0x08000800u - gxe) + __vmaxu2(gye, 0x08000800u - gye) - 0x08000800u;
            const uint32_t ao = __vmaxu2(gxo, 0x08000800u - gxo) + __vmaxu2(gyo, 0x08000800u - gyo) - 0x08000800u;
            *reinterpret_cast<uint32_t*>(erow(r) + c) =
                __byte_perm(__vminu2(ae, 0x00FF00FFu), __vminu2(ao, 0x00FF00FFu), 0x6240);
            SEa = SEb; SOa = SOb; DEa = DEb; DOa = DOb;
            SEb = SEc; SOb = SOc; DEb = DEc; DOb = DOc;
          };
          if (rb - ra == 8) {
#pragma unroll
            for (int r = 0; r < 8; ++r) one(ra + r);
          } else {
            for (int r = ra; r < rb; ++r) one(r);
          }
        }
      }
    }
    ph(6);
    mbar_arrive(&full[k & 1]);
    prod_bar();  // (the next block's A1 overwrites luma-ring rows this Sobel read)
    ph(7);
    if (!hdone && k >= 1) hdone = !pw_service<false>(R, hg, hstage, hbar, hn);
    ph(8);
  }
  while (!hdone) hdone = !pw_service<false>(R, hg, hstage, hbar, hn);
  ph(8);
  cp_async_wait<0>();  // (only empty groups can remain: the select phase reuses the staging)
}

// Fused int passes: the DP warps read their energy rows from the CTA's shared ring, which the
// producer warps fill (ring row 0 = image row 0, then two slots of 32 rows: block k in slot
// k & 1, full[slot] completing once per use, empty[slot] when every active DP warp is done).
struct FusedRing {
  const uint8_t* ring;  // nullptr: per-warp TMA rings
  int rw;               // ring row stride
  int off;              // ring column of this warp's window start (win_lo - g_lo)
  uint64_t* full;       // [2] producer -> DP
  uint64_t* empty;      // [2] DP -> producer
  long long* prof;      // (SCPL_PROF, one DP warp of rank 0) ring waits into prof[26]
};

template <bool F64, bool EDGE, int MASK>
__device__ void dp_rows(const CarveRun& R, const CarveRun& Rg, const Geo& g, int plane, typename Val<F64>::T* ceX, int CL,
                        uint32_t rank, int per_cta, uint64_t* xbar, uint32_t& xc, uint32_t& xm, uint8_t* ring,
                        uint64_t* bars, uint32_t& rph, int ndp, long long* dprof, uint32_t* pw_stage,
                        uint64_t* hbar, const FusedRing& F) {
  using V = Val<F64>;
  using T = typename V::T;
  constexpr int RS = DpCfg<F64>::kStageRows, S = DpCfg<F64>::kStages;
  constexpr int sz = F64 ? 8 : 1;
  static_assert(kXRows % RS == 0 && kBlockRows % RS == 0 || RS == kXRows, "stage layout");
  static_assert(kBlockRows == kXRows && kBlockRows == 2 * kSubRows, "one block per exchange, two choice words");
  const int lane = threadIdx.x & 31;
  const int rows = R.rows, w = g.w, pitch = R.pitch;
  const bool active = g.own_lo < g.own_hi;
  const int j0 = g.win_lo + lane * kC;
  const bool nb_mode = per_cta >= kXRows;
  T ce[kC];
  using PW = std::conditional_t<F64, uint64_t, uint32_t>;
  PW pw[kC];          // F64: path words of the block; int: choice words of the 16-row sub-block
  uint32_t cwh[kC];   // int: choice words of the block's first sub-block
  bool in[kC];
#pragma unroll
  for (int k = 0; k < kC; ++k) in[k] = (j0 + k >= 0) && (j0 + k < w);
  bool own[kC];
#pragma unroll
  for (int k = 0; k < kC; ++k) own[k] = (j0 + k >= g.own_lo) && (j0 + k < g.own_hi);
  const bool send_lo = nb_mode && active && rank > 0 && g.own_lo < g.cta_lo + kXRows;
  const bool send_hi = nb_mode && active && (int)rank + 1 < CL && g.own_hi > g.cta_hi - kXRows;
  const int nstage = (rows - 1 + RS - 1) / RS;
  const bool fused = !F64 && F.ring != nullptr;
  const int rsw = fused ? F.rw : kRingW;  // energy ring row stride
  if (active) {
    if (fused) {  // row 0 comes with the first block
      mbar_wait_sleep(&F.full[0], 0);
      __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < kC; ++k) {
      T v;
      if constexpr (F64)
        v = in[k] ? R.U[j0 + k] : 0.0;
      else
        v = in[k] ? (int)(fused ? F.ring[F.off + lane * kC + k] : R.grad[plane][j0 + k]) << kKeyShift
                  : 0;  // key of row 0
      ce[k] = in[k] ? v : V::inf();
    }
    if (lane == 0 && !fused)
      for (int st = 0; st < S - 1 && st < nstage; ++st) dp_issue_stage<F64>(Rg, plane, rows, st, g.win_lo, ring, bars);
  }
  // Exchange protocol (nb_mode): exchange e alternates between two mbarriers (e & 1); a
  // CTA announces the bytes of exchange e + 1 at the end of block e, right after its local
  // barrier (for e = 0, before the cluster barrier that precedes the pass).
  const uint32_t halo_bytes = nb_mode ? halo_bytes_for(w, CL, rank, (int)sizeof(T)) : 0u;
  // wait for stage st (issuing the one S-1 ahead first) and return its ring rows
  auto stage_rows = [&](int st) -> const uint8_t* {
    if (fused) {
      const long long tq = F.prof ? clock64() : 0;
      mbar_wait_sleep(&F.full[st & 1], (st >> 1) & 1);
      __syncwarp();
      if (F.prof && lane == 0) F.prof[26] += clock64() - tq;
      return F.ring + (size_t)(1 + kXRows * (st & 1)) * F.rw + F.off;
    }
    __syncwarp();
    if (lane == 0 && st + S - 1 < nstage) dp_issue_stage<F64>(Rg, plane, rows, st + S - 1, g.win_lo, ring, bars);
    const int slot = st % S;
    [[maybe_unused]] long long tq = DP_CLOCK();
    mbar_wait(&bars[slot], (rph >> slot) & 1u);
    __syncwarp();
    DP_PROF(1, DP_CLOCK() - tq);
    rph ^= 1u << slot;
    return ring + ((size_t)slot * RS * kRingW + (g.win_lo & 15)) * sz;
  };
  // block-end path words and landing deltas of the owned columns: the lane-contiguous words
  // are transposed through this warp's staging row so the global stores coalesce
  // block-end path words and landing deltas of the owned columns: the lane-contiguous words
  // are transposed through this warp's staging row so the global stores coalesce
  uint32_t hu = 0;  // staged block ends handed to the helper warp
  auto next_stage = [&]() -> uint32_t* {  // helper mode: a free staging buffer
    uint32_t* stg = pw_stage + (hu & 1) * kPwStageWords;
    if (hu >= 2) mbar_wait(&hbar[2 + (hu & 1)], ((hu >> 1) - 1) & 1);
    return stg;
  };
  auto store_pw = [&](int pbi, int nrb) {
    [[maybe_unused]] long long t7 = DP_CLOCK();
    uint32_t* stg = hbar ? next_stage() : pw_stage;
    uint64_t* s64 = reinterpret_cast<uint64_t*>(stg);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kC; ++k) {
      uint64_t word;
      if constexpr (F64) {
        word = pw[k];
      } else {  // rows of the second sub-block in the low bits, contiguous with the first's
        const int n2 = nrb - kSubRows;
        word = n2 > 0 ? ((uint64_t)cwh[k] << (2 * n2)) | pw[k] : (uint64_t)pw[k];
      }
      s64[lane * kC + k] = word;
    }
    if constexpr (!F64) {
#pragma unroll
      for (int k = 0; k < kC; ++k) stg[2 * kWin + lane * kC + k] = (uint32_t)(ce[k] & kSumMask);
    }
    if (hbar) {
      if (lane == 0) {
        stg[3 * kWin] = (uint32_t)pbi;
        stg[3 * kWin + 1] = (uint32_t)nrb;
      }
      mbar_arrive(&hbar[hu & 1]);
      ++hu;
    } else {
      __syncwarp();
      store_block_end<F64>(R, g, stg, pbi, nrb);
    }
    DP_PROF(7, DP_CLOCK() - t7);
  };
  int last_pbi = -1, last_nr = 0;
  const int nx = (rows - 1 + kXRows - 1) / kXRows;
  for (int xb = 0; xb < nx; ++xb) {
    [[maybe_unused]] long long tx = DP_CLOCK();
    if (nb_mode) {
      if (xb > 0) {  // halo of the previous exchange landed (st.async completion)
        const uint32_t e = xm - 1;
        mbar_wait(&xbar[e & 1], (e >> 1) & 1);
        __syncwarp();
      }
    }
    DP_PROF(0, DP_CLOCK() - tx);
    if (active) {
      if (xb > 0) {
        const T* src = ceX + (size_t)((xc - 1) & 1) * pitch;
#pragma unroll
        for (int k = 0; k < kC; ++k) ce[k] = in[k] ? src[j0 + k] : V::inf();
      }
      const uint8_t* stage = nullptr;
      if constexpr (RS == kXRows) stage = stage_rows(xb);
      // one 32-row block per exchange block: path words / dir sums restart here; int passes
      // fill a 32-bit choice word per 16-row sub-block
      const int i0 = 1 + xb * kXRows;
      const int nrb = min(kBlockRows, rows - i0);
#pragma unroll
      for (int k = 0; k < kC; ++k) {
        pw[k] = 0;
        if constexpr (!F64) ce[k] &= ~kSumMask;
      }
#pragma unroll 1
      for (int sb = 0; sb * kSubRows < nrb; ++sb) {
        const int s0 = i0 + sb * kSubRows;
        const int nr = min(kSubRows, rows - s0);
        if constexpr (!F64) {
          if (sb == 1) {
#pragma unroll
            for (int k = 0; k < kC; ++k) {
              cwh[k] = pw[k];
              pw[k] = 0u;
            }
          }
        }
        if (nr == kSubRows) {
          // 4 rows unrolled per step: short enough for the instruction cache
#pragma unroll 1
          for (int r4 = 0; r4 < kSubRows; r4 += 4) {
            const uint8_t* ebase;
            if constexpr (RS == kXRows) {
              ebase = stage + (size_t)(sb * kSubRows + r4) * rsw * sz;
            } else {
              static_assert(RS == 4, "fp64 stages hold 4 rows");
              ebase = stage_rows((s0 - 1 + r4) / RS);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) dp_step<F64, EDGE, MASK>(ce, pw, ebase + (size_t)r * rsw * sz, in, lane);
          }
        } else {
#pragma unroll 1
          for (int r = 0; r < nr; ++r) {
            const int i = s0 + r;
            const uint8_t* erow;
            if constexpr (RS == kXRows) {
              erow = stage + (size_t)(sb * kSubRows + r) * rsw * sz;
            } else {
              if ((i - 1) % RS == 0) stage = stage_rows((i - 1) / RS);
              erow = stage + (size_t)((i - 1) % RS) * kRingW * sz;
            }
            dp_step<F64, EDGE, MASK>(ce, pw, erow, in, lane);
          }
        }
      }
      if constexpr (!F64) {
        if (nrb <= kSubRows) {  // a single sub-block: its words are the block's
#pragma unroll
          for (int k = 0; k < kC; ++k) cwh[k] = 0u;
        }
      }
      if (fused) mbar_arrive(&F.empty[xb & 1]);  // this block's energy rows are consumed
      // block end: owned words and landing deltas (read after the pass), stored after the
      // exchange below
      last_pbi = xb;
      last_nr = nrb;
      DP_PROF(2, DP_CLOCK() - tx);
      tx = DP_CLOCK();
    }
    DP_PROF(4, DP_CLOCK() - tx);
    if (active) {
      // exchange-block end: owned ce into this CTA's buffer (the halo sends follow the barrier;
      // tiny widths: cluster stores before a cluster barrier)
      T* dst = ceX + (size_t)(xc & 1) * pitch;
#pragma unroll
      for (int k = 0; k < kC; ++k)
        if (own[k]) dst[j0 + k] = ce[k];
      if (!nb_mode) {
#pragma unroll 1
        for (int q = 0; q < CL; ++q) {
          if (q == (int)rank) continue;
          const int lo = min(w, q * per_cta), hi = min(w, lo + per_cta);
          const uint32_t rd = map_rank_pure(dst, q);
#pragma unroll
          for (int k = 0; k < kC; ++k) {
            const int j = j0 + k;
            if (own[k] && lo < hi && j >= lo - kXRows && j < hi + kXRows) st_cluster(rd + (uint32_t)(j * sizeof(T)), ce[k]);
          }
        }
      }
    }
    DP_PROF(5, DP_CLOCK() - tx);
    // One barrier per exchange: this CTA's DP warps' values are in its buffer, and every local
    // warp has passed its wait on exchange e-1 (block start), so thread 0 may announce the
    // bytes of exchange e+1 on the barrier slot e-1 used (a phase completing at once can no
    // longer overtake a slow waiter's parity).  The announcement and the neighbours' sends
    // may land in either order: the barrier's transaction count is signed.
    if (nb_mode) {
      asm volatile("bar.sync 2, %0;" ::"r"(ndp * 32) : "memory");
      if (threadIdx.x == 0 && xb + 1 < nx) mbar_arrive_tx(&xbar[(xm + 1) & 1], halo_bytes);
    } else {
      cluster_sync();
    }
    if (nb_mode && active) {
      // halo columns straight into the adjacent CTAs' buffers with st.async, completing bytes
      // on their exchange barrier -- after the local barrier, so the sends (edge warps only)
      // do not hold up this CTA's other warps; only the CTA's first / last warp owns columns
      // within kXRows of a CTA edge
      T* dst = ceX + (size_t)(xc & 1) * pitch;
      if (send_lo) {
        const uint32_t rd = map_rank_pure(dst, rank - 1), rb = map_rank_pure(&xbar[xm & 1], rank - 1);
#pragma unroll
        for (int k = 0; k < kC; ++k)
          if (own[k] && j0 + k < g.cta_lo + kXRows) st_async_addr(rd + (uint32_t)((j0 + k) * sizeof(T)), ce[k], rb);
      }
      if (send_hi) {
        const uint32_t rd = map_rank_pure(dst, rank + 1), rb = map_rank_pure(&xbar[xm & 1], rank + 1);
#pragma unroll
        for (int k = 0; k < kC; ++k)
          if (own[k] && j0 + k >= g.cta_hi - kXRows) st_async_addr(rd + (uint32_t)((j0 + k) * sizeof(T)), ce[k], rb);
      }
    }
    DP_PROF(6, DP_CLOCK() - tx);
    if (active && last_pbi >= 0) {
      store_pw(last_pbi, last_nr);
      last_pbi = -1;
    }
    if (active) DP_PROF(3, DP_CLOCK() - tx);
    ++xc;
    if (nb_mode) ++xm;
  }
  if (hbar) {  // end of the pass for the helper warp
    uint32_t* stg = next_stage();
    if (lane == 0) stg[3 * kWin] = 0xffffffffu;
    mbar_arrive(&hbar[hu & 1]);
  }
  if (nb_mode && nx > 0) {  // the last exchange must be complete before the smem is reused
    const uint32_t e = xm - 1;
    mbar_wait(&xbar[e & 1], (e >> 1) & 1);
    __syncwarp();
  }
  if (active) {
#pragma unroll
    for (int k = 0; k < kC; ++k) {
      int j = j0 + k;
      if (j >= g.own_lo && j < g.own_hi) {
        if constexpr (F64)
          R.lastce[j] = ce[k];
        else
          R.lastce[j] = (double)(ce[k] >> kKeyShift);
      }
    }
  }
}

template <bool F64>
__device__ void dp_pass(const CarveRun& R, const CarveRun& Rg, const Geo& g, int plane, typename Val<F64>::T* ceX, int CL,
                        uint32_t rank, int per_cta, uint64_t* xbar, uint32_t& xc, uint32_t& xm, uint8_t* ring,
                        uint64_t* bars, uint32_t& rph, int ndp, long long* dprof, uint32_t* pw_stage,
                        uint64_t* hbar, const FusedRing& F) {
  // windows lie inside [0, w) unless the plane is narrower than one window
  if (g.w < kWin)
    dp_rows<F64, true, 3>(R, Rg, g, plane, ceX, CL, rank, per_cta, xbar, xc, xm, ring, bars, rph, ndp, dprof,
                       pw_stage, hbar, F);
  else if constexpr (F64)  // (the fp64 pass always masks both ends)
    dp_rows<true, false, 3>(R, Rg, g, plane, ceX, CL, rank, per_cta, xbar, xc, xm, ring, bars, rph, ndp, dprof,
                            pw_stage, hbar, F);
  else {
    // which window ends are image borders
    const int mask = (g.win_lo <= 0 ? 1 : 0) | (g.win_lo + kWin >= g.w ? 2 : 0);
    if (mask == 0)
      dp_rows<false, false, 0>(R, Rg, g, plane, ceX, CL, rank, per_cta, xbar, xc, xm, ring, bars, rph, ndp, dprof,
                               pw_stage, hbar, F);
    else if (mask == 1)
      dp_rows<false, false, 1>(R, Rg, g, plane, ceX, CL, rank, per_cta, xbar, xc, xm, ring, bars, rph, ndp, dprof,
                               pw_stage, hbar, F);
    else if (mask == 2)
      dp_rows<false, false, 2>(R, Rg, g, plane, ceX, CL, rank, per_cta, xbar, xc, xm, ring, bars, rph, ndp, dprof,
                               pw_stage, hbar, F);
    else
      dp_rows<false, false, 3>(R, Rg, g, plane, ceX, CL, rank, per_cta, xbar, xc, xm, ring, bars, rph, ndp, dprof,
                               pw_stage, hbar, F);
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
// Select-phase shared memory (after the DP; it reuses the DP's space).  Costs are doubles on
// the fp64 pass and ints on the int passes (integer-valued ce, seams.py:39-65); per-parent
// minima are atomicMin on the cost's bit pattern (costs >= 0 order as unsigned).  Column
// indices (labels, candidates, selected seams) fit int16 (widths <= 4096).
template <bool F64>
struct SelSmem {
  using Cost = std::conditional_t<F64, double, int>;
  using Bits = std::conditional_t<F64, unsigned long long, unsigned int>;
  Cost* lce;
  Bits* segmin;
  int* segarg;
  int16_t* lab;
  int16_t* cand;
  int16_t* sel;
  int8_t* dtab;  // staged delta table [nblk][pitch] (or nullptr: chain in global)
  static __host__ __device__ constexpr size_t bytes_per_col() { return 2 * sizeof(Cost) + 4 + 3 * 2; }
  __device__ void carve(uint8_t* base, int pitch, bool stage) {
    uint8_t* p = base;
    lce = reinterpret_cast<Cost*>(p);
    p += sizeof(Cost) * (size_t)pitch;
    segmin = reinterpret_cast<Bits*>(p);
    p += sizeof(Bits) * (size_t)pitch;
    segarg = reinterpret_cast<int*>(p);
    p += 4 * (size_t)pitch;
    lab = reinterpret_cast<int16_t*>(p);
    p += 2 * (size_t)pitch;
    cand = reinterpret_cast<int16_t*>(p);
    p += 2 * (size_t)pitch;
    sel = reinterpret_cast<int16_t*>(p);
    p += 2 * (size_t)pitch;
    dtab = stage ? reinterpret_cast<int8_t*>(base + ((p - base + 15) & ~(size_t)15)) : nullptr;
  }
};
template <bool F64>
__host__ __device__ constexpr size_t sel_bytes(int pitch) {
  return SelSmem<F64>::bytes_per_col() * (size_t)pitch + 16;
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

// ------------------------------------------------------------------ row kernels
// Compact one row of luma and gradient in place (remove_batch, batching.py:76-107).  Output
// byte y reads input byte y + s(y), s(y) = #{t : a_t <= y}, a_t = rem[t] - t.  The warp
// stages the source row in shared memory (TMA bulk copy, so the in-place writes cannot race
// the reads), counts a_t per output word in a packed histogram (low half: a_t <= 4q, high
// half: a_t <= 4q + 3), prefix-sums it, and writes each output word as one funnel shift of
// two source words -- or byte by byte when its shift changes inside the word.
constexpr int kRowWarps = 8;

// The compaction CTA is small (kCompWarps warps, shared memory sized by the pitch) so that it
// fits next to a resident pass CTA: the row kernels of one group then run on SMs that other
// groups' (latency-bound) passes hold, instead of queueing for free SMs.
constexpr int kCompWarps = 4;
constexpr int kRowListCap = 256;  // removed-column list staged in shared memory (rows of batches up to this)
__host__ __device__ __forceinline__ size_t compact_warp_bytes(int pitch) {
  // rows, histogram (nwo + 1 words), barrier, removed-column list
  return 2 * (size_t)pitch + 4 * (size_t)((pitch >> 2) + 4) + 16 + 2 * kRowListCap;
}
size_t carve_compact_smem(int pitch) { return (size_t)kCompWarps * compact_warp_bytes(pitch); }

// Stage one row of luma and gradient (lane 0; whole 16-byte chunks of the w0 columns).
__device__ __forceinline__ void compact_issue(const uint8_t* L, const uint8_t* G, int w0, uint8_t* sL, uint8_t* sG,
                                              uint64_t* bar) {
  const uint32_t rbytes = (uint32_t)(((w0 + 15) >> 4) << 4);
  mbar_arrive_tx(bar, 2 * rbytes);
  bulk_g2s(sL, L, rbytes, bar);
  bulk_g2s(sG, G, rbytes, bar);
}

// One warp compacts one staged row in place: rg = the row's b removed columns (ascending, in
// the w0 = wn + b column frame); the staging completes on bar (phase `parity`).
// (bar == nullptr: the row is already staged; G / sG == nullptr: luma only; L2: a second luma
// destination; rs: kRowListCap int16 of shared memory where a global list is staged for the
// words whose shift changes inside them -- else a chain of dependent global loads per word)
__device__ __forceinline__ void compact_row(uint8_t* L, uint8_t* G, const int16_t* rg, int b, int wn,
                                            const uint8_t* sL, const uint8_t* sG, uint32_t* hist, uint64_t* bar,
                                            uint32_t parity, uint8_t* L2 = nullptr, int16_t* rs = nullptr) {
  const int lane = threadIdx.x & 31;
  const int w0 = wn + b;
  const int nwo = (wn + 3) >> 2;
  for (int q = lane; q <= nwo; q += 32) hist[q] = 0u;
  __syncwarp();
  const bool stage_list = rs != nullptr && b <= kRowListCap;
  // b <= 255: four 8-bit fields, field u counting a_t <= 4q + u, so every output byte's shift is
  // known (no search when a removed column falls inside a word); else two 16-bit fields (u = 0, 3)
  const bool f4 = b <= 255;
  for (int t = lane; t < b; t += 32) {
    const int16_t rv = rg[t];
    // the batch's seams are pairwise disjoint (batching.py:104): strictly increasing per row
    SCPL_DCHECK(rv >= t && rv < w0 && (t == 0 || rg[t - 1] < rv), "removed columns disjoint and in range");
    if (stage_list) rs[t] = rv;
    const int at = rv - t;  // >= 0
    if (f4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // a_t <= 4q + u  <=>  q >= (a_t - u + 3) >> 2
        const int qu = (at - u + 3) >> 2;
        if (qu <= nwo) atomicAdd(&hist[qu], 1u << (8 * u));
      }
    } else {
      const int q1 = (at + 3) >> 2, q2 = at >> 2;  // a_t <= 4q  <=>  q >= q1;  a_t <= 4q+3  <=>  q >= q2
      if (q1 <= nwo) atomicAdd(&hist[q1], 1u);
      if (q2 <= nwo) atomicAdd(&hist[q2], 0x10000u);
    }
  }
  __syncwarp();
  // inclusive prefix over q = 0 .. nwo-1: lane owns a contiguous segment
  const int per = (nwo + 31) >> 5;
  const int q0 = min(nwo, lane * per), q1 = min(nwo, q0 + per);
  uint32_t run = 0;
  for (int q = q0; q < q1; ++q) run += hist[q];
  uint32_t incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  run = incl - run;
  for (int q = q0; q < q1; ++q) {
    run += hist[q];
    hist[q] = run;
  }
  if (bar) mbar_wait(bar, parity);
  __syncwarp();
  if (stage_list) rg = rs;  // (staged before the histogram's __syncwarp)
  const uint32_t* Lw = reinterpret_cast<const uint32_t*>(sL);
  const uint32_t* Gw = reinterpret_cast<const uint32_t*>(sG);
  const int nwi = (w0 + 3) >> 2;
  for (int q = lane; q < nwo; q += 32) {
    const uint32_t h = hist[q];
    const int s0 = f4 ? (int)(h & 255u) : (int)(h & 0xffffu), s3 = f4 ? (int)(h >> 24) : (int)(h >> 16);
    uint32_t lv, gv;
    if (s0 == s3) {
      const int x0 = 4 * q + s0, wq = x0 >> 2;
      const uint32_t sh = (uint32_t)(x0 & 3) * 8u;
      const bool nx = wq + 1 < nwi;
      lv = __funnelshift_r(Lw[wq], nx ? Lw[wq + 1] : 0u, sh);
      gv = G ? __funnelshift_r(Gw[wq], nx ? Gw[wq + 1] : 0u, sh) : 0u;
    } else if (f4) {  // byte u from 4q + u + s(4q + u)
      lv = 0u;
      gv = 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = 4 * q + u + (int)((h >> (8 * u)) & 255u);
        if (x < w0) {
          lv |= (uint32_t)sL[x] << (8 * u);
          if (G) gv |= (uint32_t)sG[x] << (8 * u);
        }
      }
    } else {  // s(4q + u) for u = 0..3 from the removed list
      int t = s0;
      lv = 0u;
      gv = 0u;
      for (int u = 0; u < 4; ++u) {
        while (t < b && rg[t] - t <= 4 * q + u) ++t;
        const int x = 4 * q + u + t;
        if (x < w0) {
          lv |= (uint32_t)sL[x] << (8 * u);
          if (G) gv |= (uint32_t)sG[x] << (8 * u);
        }
      }
    }
    reinterpret_cast<uint32_t*>(L)[q] = lv;
    if (L2) reinterpret_cast<uint32_t*>(L2)[q] = lv;
    if (G) reinterpret_cast<uint32_t*>(G)[q] = gv;
  }
  __syncwarp();  // hist and the staged row are free again
}

constexpr int kDirtyCap = 256;
// la / lb / lc: the compacted luma rows i-1, i, i+1 (clamped), gr: the gradient row i to patch;
// ra / ri / rc: the batch's removed columns of those rows (b each, ascending, w0 frame).
__device__ __forceinline__ void dirty_row_at(const uint8_t* la, const uint8_t* lb, const uint8_t* lc, uint8_t* gr,
                                             const int16_t* ra, const int16_t* ri, const int16_t* rc, int b, int wn,
                                             bool tiny, int16_t* stage) {
  const int lane = threadIdx.x & 31;
  const int w0 = wn + b;
  if (tiny) {  // fewer than 3 rows or columns: zero energy (default_energy)
    for (int y = lane; y < wn; y += 32) gr[y] = 0;
    return;
  }
  if (b <= kDirtyCap) {
    for (int t = lane; t < b; t += 32) {
      const int16_t va = ra[t], vi = ri[t], vc = rc[t];
      stage[t] = va;
      stage[kDirtyCap + t] = vi;
      stage[2 * kDirtyCap + t] = vc;
    }
    __syncwarp();
    ra = stage;
    ri = stage + kDirtyCap;
    rc = stage + 2 * kDirtyCap;
  }
  for (int q = lane; q < 9 * b; q += 32) {
    const int rsel = q / (3 * b), rem = q - rsel * 3 * b;
    const int s = rem / 3, offc = rem - s * 3 - 1;
    const int x = (rsel == 0 ? ra : rsel == 1 ? ri : rc)[s] + offc;
    if (x < 0 || x >= w0) continue;
    int lo = 0, hi = b;  // row-i removed columns < x
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (ri[mid] < x) lo = mid + 1; else hi = mid;
    }
    if (lo < b && ri[lo] == x) continue;  // removed itself
    const int y = x - lo;
    const int ym = max(y - 1, 0), yp = min(y + 1, wn - 1);
    const int gx = (la[yp] + 2 * lb[yp] + lc[yp]) - (la[ym] + 2 * lb[ym] + lc[ym]);
    const int gy = (lc[ym] + 2 * lc[y] + lc[yp]) - (la[ym] + 2 * la[y] + la[yp]);
    const int gv = abs(gx) + abs(gy);
    gr[y] = (uint8_t)(gv > 255 ? 255 : gv);
  }
  __syncwarp();  // the staged lists are free again
}

// default_energy (batching.py:110-115) of row i of the carved frame, incrementally: a pixel's
// Sobel value changes only if a removed pixel of rows i-1..i+1 lay within one column of it.
// `lum`/`gra` are the frame's planes, off = the batch's offset in the removed-column log.
// The three rows' removed-column lists are staged in the warp's shared memory (`stage`, 3 x
// kDirtyCap entries) when they fit, so the binary searches do not chain global loads.
__device__ __forceinline__ void dirty_row(const CarveRun& R, const uint8_t* lum, uint8_t* gra, int i, int b, int wn,
                                          int off, int16_t* stage) {
  const int rows = R.rows;
  const int ia = max(i - 1, 0), ib = min(i + 1, rows - 1);
  dirty_row_at(lum + (long)ia * R.pitch, lum + (long)i * R.pitch, lum + (long)ib * R.pitch, gra + (long)i * R.pitch,
               R.rem + (long)ia * R.rem_cap + off, R.rem + (long)i * R.rem_cap + off,
               R.rem + (long)ib * R.rem_cap + off, b, wn, rows < 3 || wn < 3, stage);
}

// Select + trace of one pass (every CTA of the cluster redundantly; no broadcast needed):
// labels (batching.py:39-46) by chaining the landing deltas, per-parent leftmost minimum
// (:59-64), k-truncation by (cost, col) (:66-68), then the removed-column log (seams.py:68-81).
// Returns the batch size.
template <bool F64>
__device__ int select_trace(const CarveRun& R, uint8_t* smem, int* ws, uint64_t* dbar, int w, int iters, int removed,
                            uint32_t rank, int CL, int nblk) {
  using Sel = SelSmem<F64>;
  using Cost = typename Sel::Cost;
  using Bits = typename Sel::Bits;
  const int tid = threadIdx.x;
  const int rows = R.rows, pitch = R.pitch;
  // (the fp64 pass chains the deltas in global memory: its shared memory stays small enough for
  // two pass CTAs per SM; it is one pass per run)
  const bool stage_dtab = R.stage_dtab != 0 && !F64;
  Sel S;
  S.carve(smem, pitch, stage_dtab);
  const int8_t* dsrc = R.delta;
  if (stage_dtab && tid == 0) {
    // one bulk copy of the whole landing-delta table; the DP's generic-proxy stores (every
    // CTA, published by the cluster barrier) are ordered before the async-proxy read
    fence_proxy_async_global();
    mbar_arrive_tx(dbar, (uint32_t)((size_t)nblk * pitch));
    bulk_g2s(S.dtab, R.delta, (uint32_t)((size_t)nblk * pitch), dbar);
  }
  for (int j = tid; j < w; j += blockDim.x) {
    S.lce[j] = (Cost)R.lastce[j];
    S.segmin[j] = ~(Bits)0;
    S.segarg[j] = INT_MAX;
  }
  if (stage_dtab) {
    mbar_wait(dbar, 0);
    dsrc = S.dtab;
  }
  __syncthreads();
  [[maybe_unused]] long long ts = DP_CLOCK();
  // labels (batching.py:39-46): chain the block landing deltas, 8 columns per thread in flight
  // (shared-memory table: 32-bit shared addresses, no generic-address resolution per step)
  for (int jb = tid; jb < w; jb += 8 * blockDim.x) {
    int c[8];
    bool ok[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      c[u] = jb + u * (int)blockDim.x;
      ok[u] = c[u] < w;
      if (!ok[u]) c[u] = 0;
    }
    if (stage_dtab) {
      uint32_t row = smem_u32(S.dtab) + (uint32_t)(nblk - 1) * (uint32_t)pitch;
      for (int bl = nblk - 1; bl >= 0; --bl, row -= (uint32_t)pitch) {
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] += lds_s8(row + (uint32_t)c[u]);
      }
    } else {
      for (int bl = nblk - 1; bl >= 0; --bl) {
        const int8_t* drow = dsrc + (size_t)bl * pitch;
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] += drow[c[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (ok[u]) S.lab[jb + u * blockDim.x] = (int16_t)c[u];
  }
  __syncthreads();
  SEL_PROF(0);
  if (rank == 0 && R.labs != nullptr)  // seam dump: this pass's labels (label_parents)
    for (int j = tid; j < w; j += blockDim.x) R.labs[(long)iters * R.width0 + j] = S.lab[j];
  auto bits = [](Cost v) -> Bits {
    if constexpr (F64)
      return (Bits)__double_as_longlong(v);
    else
      return (Bits)v;
  };
  int b;
  if (R.kmax == 1) {  // raw mode: min_seam, leftmost global minimum (seams.py:84-89)
    for (int j = tid; j < w; j += blockDim.x) atomicMin(&S.segmin[0], bits(S.lce[j]));
    __syncthreads();
    for (int j = tid; j < w; j += blockDim.x)
      if (bits(S.lce[j]) == S.segmin[0]) atomicMin(&S.segarg[0], j);
    __syncthreads();
    if (tid == 0) S.sel[0] = (int16_t)S.segarg[0];
    b = 1;
  } else {
    // per parent the leftmost strict minimum (batching.py:59-64); costs >= 0 order as unsigned
    for (int j = tid; j < w; j += blockDim.x) atomicMin(&S.segmin[S.lab[j]], bits(S.lce[j]));
    __syncthreads();
    for (int j = tid; j < w; j += blockDim.x)
      if (bits(S.lce[j]) == S.segmin[S.lab[j]]) atomicMin(&S.segarg[S.lab[j]], j);
    __syncthreads();
    SEL_PROF(1);
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
      if (l < w && S.segarg[l] != INT_MAX) S.cand[pos++] = (int16_t)S.segarg[l];
    }
    __syncthreads();
    SEL_PROF(2);
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
          const Cost cq = S.lce[S.cand[q]];
          int rk = 0;
          for (int o = 0; o < P; ++o) {
            const Cost co = S.lce[S.cand[o]];
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
  SEL_PROF(3);
  // trace (seams.py:68-81): walk each seam's block-end columns through the staged deltas,
  // keeping those of this CTA's blocks (bl % CL == rank); then decode (seam, block) pairs
  // in parallel into the removed-column log
  int16_t* log = R.rem;  // rows x rem_cap, this batch's columns at [removed, removed + b)
  for (int s = tid; s < b; s += blockDim.x) {
    int c = S.sel[s];
    int next_mine = (nblk - 1) - ((nblk - 1 - (int)rank) % CL + CL) % CL;  // highest block with bl % CL == rank
    for (int bl = nblk - 1; bl >= 0; --bl) {
      if (bl == next_mine) {
        R.cend[(long)bl * pitch + s] = (int16_t)c;
        next_mine -= CL;
      }
      c += stage_dtab ? lds_s8(smem_u32(S.dtab) + (uint32_t)bl * (uint32_t)pitch + (uint32_t)c)
                      : (int)dsrc[(size_t)bl * pitch + c];
    }
    if (rank == 0) log[removed + s] = (int16_t)c;  // row 0 (== the seam's label)
  }
  __syncthreads();
  const int myblk = nblk > (int)rank ? (nblk - 1 - (int)rank) / CL + 1 : 0;
  // each thread walks one (seam, block) pair: path words (fp64 pass: one word per pair) or the
  // choice words of the columns the seam visits (int passes; L1/L2-resident, just written)
  for (int q = tid; q < b * myblk; q += blockDim.x) {
    int s = q / myblk, bl = (int)rank + (q - s * myblk) * CL;
    int c = R.cend[(long)bl * pitch + s];
    const uint64_t* pwb = R.pw + (long)bl * pitch;
    int i_start = 1 + bl * kBlockRows;
    int i_end = min(i_start + kBlockRows, rows) - 1;
    if constexpr (F64) {  // path word of the seam's end column
      uint64_t word = pwb[c];
      for (int i = i_end; i >= i_start; --i) {
        SCPL_DCHECK(c >= 0 && c < w, "trace column inside the row (fp64 pass)");
        log[(long)i * R.rem_cap + removed + s] = (int16_t)c;
        c += (int)(word & 3u) - 1;
        word >>= 2;
      }
    } else {
      for (int i = i_end, qq = 0; i >= i_start; --i, ++qq) {
        SCPL_DCHECK(c >= 0 && c < w, "trace column inside the row");
        log[(long)i * R.rem_cap + removed + s] = (int16_t)c;
        c += (int)((pwb[c] >> (2 * qq)) & 3u) - 1;
      }
    }
  }
  SEL_PROF(4);
  if (rank == 0 && R.cols != nullptr)
    for (int s = tid; s < b; s += blockDim.x) {
      R.cols[removed + s] = S.sel[s];
      R.costs[removed + s] = (double)S.lce[S.sel[s]];
    }
  if (rank == 0 && tid == 0) R.sizes[iters] = b;  // every CTA reads them in the final phase
  return b;
}

__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Shared-memory barriers of a pass (static shared memory of the carve kernels)
struct PassBars {
  uint64_t* xbar;  // [2] neighbour exchange
  uint64_t* rbar;  // [kMaxWarps * 6] DP energy rings
  uint64_t* dbar;  // [1] delta-table staging
  uint64_t* hbar;  // [kMaxWarps * 4] DP warp -> helper warp
};

// One DP pass + select + trace of run Rg on this CTA's cluster, at width w after `iters` passes
// and `removed` seams: returns the batch size (every CTA computes the same).  The barriers are
// initialised here (reinit: they held the previous pass's phases; every use of them is complete
// -- the caller synchronised the cluster).  Ends with a cluster barrier: the batch's removed-
// column log is complete.
// FK: the fused kernel (kFusedWarps warps, fused int passes only); else the plain kernel
// (kMaxWarps warps: fp64 passes and unfused int passes).
template <bool FK>
__device__ int cluster_pass(CarveRun& Rg, int CL, uint32_t rank, int w, int iters, int removed, bool fp64,
                            uint8_t* smem, int* ws, const PassBars& B, bool reinit, long long& t_dp,
                            long long& t_sel) {
  const CarveRun& R = Rg;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rows = R.rows;
  const int nblk = (rows - 1 + kBlockRows - 1) / kBlockRows;
  const int plane = 0;  // planes are compacted in place
  long long dprof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tp = clock64();
  if (R.prof && rank == 0 && tid == 0 && iters < 500) R.prof[32 + 2 * iters] = (long long)globaltimer_ns();

  const int per = ((w + CL - 1) / CL + 15) & ~15;
  const int ndp = min(kMaxWarps, (per + kOwn - 1) / kOwn);
  // fused int pass: the host guarantees per >= kXRows and ndp <= kDpWarps at every width, and
  // launches the fused kernel for exactly these passes
  constexpr bool fused = FK;
  if (FK != (!fp64 && R.fused != 0) || (FK && (per < kXRows || ndp > kDpWarps))) __trap();
  int n_act = 0;  // DP warps with columns (they arrive on the ring's empty barriers)
  {
    const int clo = min(w, (int)rank * per), chi = min(w, clo + per);
    for (int q = 0; q < ndp; ++q) n_act += clo + q * kOwn < chi;
  }
  if (tid == 0) {
    if (reinit) {
      mbar_inval(&B.xbar[0]);
      mbar_inval(&B.xbar[1]);
      mbar_inval(B.dbar);
    }
    mbar_init(&B.xbar[0], 1);
    mbar_init(&B.xbar[1], 1);
    mbar_init(B.dbar, 1);
    if (rows > 1 && per >= kXRows)  // the pass's first exchange, announced before it can start
      mbar_arrive_tx(&B.xbar[0], halo_bytes_for(w, CL, rank, fp64 ? 8 : 4));
  }
  if (fused) {  // rbar[0..1]: ring full (producer threads), rbar[2..3]: ring empty (DP lanes)
    if (tid == 0)
      for (int k = 0; k < 4; ++k) {
        if (reinit) mbar_inval(&B.rbar[k]);
        mbar_init(&B.rbar[k], k < 2 ? kProdWarps * 32 : max(n_act, 1) * 32);
      }
  } else if (lane == 0) {
    for (int k = 0; k < 6; ++k) {
      if (reinit) mbar_inval(&B.rbar[wid * 6 + k]);
      mbar_init(&B.rbar[wid * 6 + k], 1);
    }
  }
  if (lane == 0 && wid < kMaxWarps) {
    for (int k = 0; k < 4; ++k) {
      if (reinit) mbar_inval(&B.hbar[wid * 4 + k]);
      mbar_init(&B.hbar[wid * 4 + k], 32);
    }
    fence_mbar_init();
  }
  uint32_t xc = 0, xm = 0, rph = 0;
  cluster_sync();

  // ---------------- 1. DP
  {
    auto geo = [&](int dw) {
      Geo g;
      g.w = w;
      g.cta_lo = min(w, (int)rank * per);
      g.cta_hi = min(w, g.cta_lo + per);
      g.own_lo = g.cta_lo + dw * kOwn;
      g.own_hi = min(g.cta_hi, g.own_lo + kOwn);
      // window: owned +- 32, shifted inside [0, w) when the plane is wide enough, so that a
      // window edge is either an image border (exact +inf) or a decaying halo -- no masks
      g.win_lo = w >= kWin ? min(max(g.own_lo - kXRows, 0), w - kWin) : g.own_lo - kXRows;
      return g;
    };
    const bool in_dp = wid < ndp || per < kXRows;
    // helper warps: the block-end global stores of DP warp (wid - ndp), off its critical path
    const bool helpers = per >= kXRows && 2 * ndp <= kMaxWarps;
    const int pitch = R.pitch;
    if constexpr (FK) {
      ProdGeo P;
      P.rw = R.ring_w;
      int g_hi = 0;
      P.g_lo = 0;
      const bool act = fused_cta_range(w, CL, (int)rank, P.g_lo, g_hi);
      if (act && g_hi - P.g_lo > P.rw) __trap();  // (host bug: ring_w below the CTA's range)
      P.cta_lo = min(w, (int)rank * per);
      P.cta_hi = min(w, P.cta_lo + per);
      uint32_t* stage0 = reinterpret_cast<uint32_t*>(smem + fused_off_stage(pitch));
      uint8_t* ering = smem + fused_off_ering(pitch);
      // register split (setmaxnreg, warpgroup-uniform): DP warpgroup up, producers down, then
      // both back to the launch allocation for the select phase
      if (wid < kProdFirst) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegDp));
        if (wid < ndp) {
          const Geo g = geo(wid);
          const FusedRing F{ering, P.rw, g.win_lo - P.g_lo, &B.rbar[0], &B.rbar[2],
                            R.prof && rank == 0 && wid == 0 ? R.prof : nullptr};
          // (a DP warp without columns gets no helper: it would only send the end marker, after
          // the other DP warps' blocks -- which its producer, blocked on that marker, must build)
          dp_pass<false>(R, Rg, g, plane, reinterpret_cast<int*>(smem), CL, rank, per, B.xbar, xc, xm, nullptr,
                         nullptr, rph, ndp, dprof, stage0 + wid * 2 * kPwStageWords,
                         wid < n_act ? &B.hbar[wid * 4] : nullptr, F);
        }
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegFused));
      } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegProd));
        const int q = wid - kProdFirst;
        produce_pass(R, w, R.b, removed - R.b, P, ering, smem + fused_off_lring(pitch, P.rw),
                     smem + fused_off_pstage(pitch, P.rw), &B.rbar[0], &B.rbar[2], tid - kProdFirst * 32,
                     q < n_act, geo(min(q, ndp - 1)), stage0 + min(q, kDpWarps - 1) * 2 * kPwStageWords,
                     &B.hbar[min(q, kDpWarps - 1) * 4], act,
                     R.prof && rank == 0 && tid == kProdFirst * 32 ? R.prof : nullptr);
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegFused));
      }
    } else {
    if (fused) __trap();
    uint8_t* ring = smem + 2 * (fp64 ? 8 : 4) * (size_t)pitch;
    uint32_t* pw_stage0 = reinterpret_cast<uint32_t*>(ring + (size_t)ndp * (fp64 ? dp_ring_bytes<true>()
                                                                                 : dp_ring_bytes<false>()));
    if (in_dp) {
      const Geo g = geo(wid);
      uint32_t* pw_stage = pw_stage0 + wid * 2 * kPwStageWords;
      uint64_t* hb = helpers ? &B.hbar[wid * 4] : nullptr;
      if (fp64)
        dp_pass<true>(R, Rg, g, plane, reinterpret_cast<double*>(smem), CL, rank, per, B.xbar, xc, xm,
                      ring + (size_t)wid * dp_ring_bytes<true>(), &B.rbar[wid * 6], rph, ndp, dprof, pw_stage, hb,
                      FusedRing{});
      else
        dp_pass<false>(R, Rg, g, plane, reinterpret_cast<int*>(smem), CL, rank, per, B.xbar, xc, xm,
                       ring + (size_t)wid * dp_ring_bytes<false>(), &B.rbar[wid * 6], rph, ndp, dprof, pw_stage, hb,
                       FusedRing{});
    } else if (helpers && wid < 2 * ndp) {
      const int dw = wid - ndp;
      const uint32_t* stage = pw_stage0 + dw * 2 * kPwStageWords;
      if (fp64)
        pw_helper<true>(R, geo(dw), stage, &B.hbar[dw * 4]);
      else
        pw_helper<false>(R, geo(dw), stage, &B.hbar[dw * 4]);
    }
    }
  }
  cluster_sync();  // lastce / pw / delta of all CTAs visible
  t_dp += clock64() - tp;
  tp = clock64();

  // ---------------- 2. select + trace (redundant per CTA)
  const int b = fp64 ? select_trace<true>(R, smem, ws, B.dbar, w, iters, removed, rank, CL, nblk)
                     : select_trace<false>(R, smem, ws, B.dbar, w, iters, removed, rank, CL, nblk);
  cluster_sync();  // the batch's log is complete before the rows are compacted
  t_sel += clock64() - tp;
  if (rank == 0 && tid == 0 && R.prof) {
    for (int k = 0; k < 8; ++k) R.prof[4 + k] += dprof[k];
    if (iters < 500) R.prof[33 + 2 * iters] = (long long)globaltimer_ns();
  }
  return b;
}

// One DP pass + select + trace for every active run (one cluster per run).  Per-run state
// (width, iters, removed) is read at entry and written back at exit.
// fp64_smem: this launch's dynamic shared memory holds the fp64 layouts (a buffered run's first
// pass, every pass with reaverage_energy); int-pass launches get the smaller int layout, so two
// pass CTAs fit on an SM.
template <bool FK>
__device__ __forceinline__ void pass_body(CarveRun* __restrict__ runs, int CL, int fp64_smem, uint8_t* smem,
                                          const PassBars& B, int* ws) {
  const uint32_t rank = cluster_rank();
  CarveRun& Rg = runs[blockIdx.x / CL];
  const int w = Rg.width, iters = Rg.iters, removed = Rg.removed;
  if (w <= Rg.target) {  // done: nothing this iteration
    if (rank == 0 && threadIdx.x == 0) Rg.b = 0;
    return;
  }
  const bool fp64 = Rg.U != nullptr && (iters == 0 || Rg.reaverage);  // reaverage: every pass on the mean
  if (fp64 && !fp64_smem) __trap();  // (launcher bug: an int-sized launch reached an fp64 pass)
  long long t_dp = 0, t_sel = 0;
  const int b = cluster_pass<FK>(Rg, CL, rank, w, iters, removed, fp64, smem, ws, B, false, t_dp, t_sel);
  if (rank == 0 && threadIdx.x == 0) {
    if (FK) Rg.lsel ^= 1;  // the compacted luma went to the other plane
    Rg.b = b;
    Rg.width = w - b;
    Rg.iters = iters + 1;
    Rg.removed = removed + b;
    Rg.cyc_dp += t_dp;
    Rg.cyc_sel += t_sel;
  }
}

__global__ void __launch_bounds__(kMaxWarps * 32, 2) carve_pass_kernel(CarveRun* __restrict__ runs, int CL,
                                                                       int fp64_smem) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int ws[32];
  __shared__ __align__(8) uint64_t s_xbar[2];
  __shared__ __align__(8) uint64_t s_rbar[kMaxWarps * 6];
  __shared__ __align__(8) uint64_t s_dbar;  // delta-table staging (select phase)
  __shared__ __align__(8) uint64_t s_hbar[kMaxWarps * 4];  // DP warp -> helper warp staging
  pass_body<false>(runs, CL, fp64_smem, smem, PassBars{s_xbar, s_rbar, &s_dbar, s_hbar}, ws);
}

// Fused int passes: 4 DP warps + kProdWarps producer warps; launched at kRegFused registers per
// thread (two CTAs per SM), split by setmaxnreg inside the DP phase.
__global__ void __launch_bounds__(kFusedWarps * 32, 2) carve_pass_fused_kernel(CarveRun* __restrict__ runs,
                                                                               int CL) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int ws[32];
  __shared__ __align__(8) uint64_t s_xbar[2];
  __shared__ __align__(8) uint64_t s_rbar[4];
  __shared__ __align__(8) uint64_t s_dbar;
  __shared__ __align__(8) uint64_t s_hbar[kMaxWarps * 4];
  pass_body<true>(runs, CL, 0, smem, PassBars{s_xbar, s_rbar, &s_dbar, s_hbar}, ws);
}

// Programmatic dependent launch: the row kernels and the loop check are launched while the
// kernel before them drains (their CTAs wait here for its results), hiding a launch latency per
// kernel boundary of every carve iteration.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(kCompWarps * 32) carve_compact_kernel(CarveRun* __restrict__ runs) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t csm[];
  const CarveRun& R = runs[blockIdx.y];
  const int b = R.b;
  if (b == 0 || R.width <= R.target) return;  // nothing removed / no further pass reads the planes
  if ((int)blockIdx.z >= R.nfr) return;       // frame of the run's plane stack (reaverage)
  const long long fo = (long long)blockIdx.z * R.fstride;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int i = blockIdx.x * kCompWarps + wl;
  if (i >= R.rows) return;
  const int pitch = R.pitch;
  uint8_t* base = csm + (size_t)wl * compact_warp_bytes(pitch);
  uint8_t* sL = base;
  uint8_t* sG = base + pitch;
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + 2 * (size_t)pitch);
  uint64_t* bar = reinterpret_cast<uint64_t*>(hist + (pitch >> 2) + 4);
  uint8_t* L = R.luma[0] + fo + (long)i * pitch;
  uint8_t* G = R.grad[0] + fo + (long)i * pitch;
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    compact_issue(L, G, R.width + b, sL, sG, bar);
  }
  int16_t* rs = reinterpret_cast<int16_t*>(base + compact_warp_bytes(pitch) - 2 * kRowListCap);
  compact_row(L, G, R.rem + (long)i * R.rem_cap + (R.removed - b), b, R.width, sL, sG, hist, bar, 0, nullptr, rs);
}

__global__ void __launch_bounds__(kRowWarps * 32) carve_dirty_kernel(CarveRun* __restrict__ runs) {
  pdl_wait();
  const CarveRun& R = runs[blockIdx.y];
  const int b = R.b;
  if (b == 0 || R.width <= R.target) return;  // no further pass reads this gradient
  if ((int)blockIdx.z >= R.nfr) return;
  const long long fo = (long long)blockIdx.z * R.fstride;
  __shared__ int16_t s_lists[kRowWarps][3 * kDirtyCap];
  const int i = blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (i >= R.rows) return;
  dirty_row(R, R.luma[0] + fo, R.grad[0] + fo, i, b, R.width, R.removed - b, s_lists[threadIdx.x >> 5]);
}

// Final index map (original column of every kept column): replay each row's batches on an
// alive-column bitmask in shared memory.  A batch's columns are "the c-th alive column" of
// the frame it was selected on; clearing the highest first keeps the prefix counts taken
// before the batch valid for the lower ones.
__global__ void __launch_bounds__(kRowWarps * 32) carve_index_kernel(CarveRun* __restrict__ runs) {
  __shared__ uint32_t s_wv[kRowWarps][32 * kMaxAliveWordsPerLane];
  __shared__ int s_pre[kRowWarps][32 * kMaxAliveWordsPerLane];
  const CarveRun& R = runs[blockIdx.y];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int i = blockIdx.x * kRowWarps + wl;
  if (i >= R.rows) return;
  uint32_t* wv = s_wv[wl];
  int* pre = s_pre[wl];
  const int nw32 = (R.width0 + 31) >> 5;
  for (int m = lane; m < nw32; m += 32) {
    int hi = R.width0 - 32 * m;
    wv[m] = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
  }
  __syncwarp();
  const int16_t* lg = R.rem + (long)i * R.rem_cap;
  auto prefix = [&]() {
    int running = 0;
#pragma unroll
    for (int u = 0; u < kMaxAliveWordsPerLane; ++u) {
      int m = lane + 32 * u;
      int p = m < nw32 ? __popc(wv[m]) : 0;
      int incl = warp_incl_scan(p);
      if (m < nw32) pre[m] = running + incl - p;
      running += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
  };
  int off = 0;
  for (int k = 0; k < R.iters; ++k) {
    const int bk = R.sizes[k];
    prefix();
    for (int base = bk - 1; base >= 0; base -= 32) {
      const int sidx = base - lane;
      int o = 0;
      if (sidx >= 0) o = alive_select(wv, pre, nw32, lg[off + sidx]);
      SCPL_DCHECK(sidx < 0 || (o >= 0 && o < R.width0 && (wv[o >> 5] >> (o & 31) & 1u)),
                  "index map: removed column is an alive original column");
      __syncwarp();
      if (sidx >= 0) atomicAnd(&wv[o >> 5], ~(1u << (o & 31)));
      __syncwarp();
    }
    off += bk;
  }
  prefix();
  int16_t* ir = R.idx + (long)i * R.pitch;
  for (int m = lane; m < nw32; m += 32) {
    uint32_t wd = wv[m];
    int o = pre[m];
    while (wd) {
      int bit = __ffs(wd) - 1;
      ir[o++] = (int16_t)(m * 32 + bit);
      wd &= wd - 1;
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
        if (idx) idx[(long)i * pitch + j] = (int16_t)j;
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
      if (idx) idx[(long)j * pitch + i] = (int16_t)i;
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
                      const CarveRun& R, cudaStream_t st, int f) {
  dim3 grid(cdiv(W, 32), cdiv(H, 32));
  uint8_t* L = R.luma[0] + (long long)f * R.fstride;
  uint8_t* G = R.grad[0] + (long long)f * R.fstride;
  // the index map is the run's (one per run); frame f > 0 of a reaverage stack only needs planes
  run_setup_kernel<<<grid, dim3(32, 8), 0, st>>>(frame, H, W, C, transposed, codes, R.pitch, L, G,
                                                 f == 0 ? R.idx : nullptr);
  SCPL_CHECK_LAUNCH();
  if (!codes) {
    plane_sobel_kernel<<<dim3(cdiv(R.width0, 256), R.rows), 256, 0, st>>>(L, R.rows, R.width0, R.pitch, G);
    SCPL_CHECK_LAUNCH();
  }
}

// reaverage_energy (pipeline.py:289-290): U = np.stack(default_energy of every carved frame)
// .mean(0).  The gradients are integers, so the per-pixel sum over the stack is exact in any
// order and the mean is one correctly rounded division, as numpy's.
__global__ void carve_mean_kernel(CarveRun* __restrict__ runs) {
  const CarveRun& R = runs[blockIdx.y];
  if (!R.reaverage || R.width <= R.target) return;
  const int i = blockIdx.x;
  if (i >= R.rows) return;
  const double dn = (double)R.nfr;
  double* u = const_cast<double*>(R.U) + (long)i * R.pitch;
  for (int j = threadIdx.x; j < R.width; j += blockDim.x) {
    uint32_t sum = 0;
    const uint8_t* g = R.grad[0] + (long)i * R.pitch + j;
    for (int f = 0; f < R.nfr; ++f) sum += g[(long long)f * R.fstride];
    u[j] = __ddiv_rn((double)sum, dn);
  }
}

void launch_carve_mean(CarveRun* runs_d, int nruns, int rows, cudaStream_t st) {
  carve_mean_kernel<<<dim3(rows, nruns), 256, 0, st>>>(runs_d);
  SCPL_CHECK_LAUNCH();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
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

static void encode_plane(CUtensorMap* tm, const void* base, CUtensorMapDataType dt, int esz, int cols, int rows,
                         int pitch, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * esz};
  cuuint32_t box[2] = {(cuuint32_t)kRingW, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = tmap_encode()(tm, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SCPL_ARG(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed for a carve plane");
}

void encode_carve_tensor_maps(CarveRun& R) {
  for (int p = 0; p < 2; ++p)
    encode_plane(&R.tm_grad[p], R.grad[p], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, R.width0, R.rows, R.pitch,
                 DpCfg<false>::kStageRows);
  encode_carve_tensor_map_U(R);
}

// the fp64 plane's map alone (box = this variant's ring row): the fp64 first pass may run with
// another variant than the int passes
void encode_carve_tensor_map_U(CarveRun& R) {
  if (R.U)
    encode_plane(&R.tm_U, R.U, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, R.width0, R.rows, R.pitch,
                 DpCfg<true>::kStageRows);
}

int carve_dp_warps(int width, int cl) {
  const int per = ((width + cl - 1) / cl + 15) & ~15;
  return (per + kOwn - 1) / kOwn;
}

// the narrow variants need up to 16 CTAs per run (kc3 at 1080p, kc4 at 4K): a non-portable
// cluster size
constexpr int kMaxCluster = SCPL_KC <= 4 ? 16 : 8;

int carve_cluster_size(int nruns, int width, int num_sms) {
  // one DP warp per SM sub-partition: kDpWarps x kOwn columns per CTA
  int cl = (width + kOwn * kDpWarps - 1) / (kOwn * kDpWarps);
  if (const char* e = getenv("SCPL_CARVE_CL")) {  // experiments: fewer CTAs, more DP warps each
    const int want = atoi(e);
    if (want >= 1 && want <= kMaxCluster && carve_dp_warps(width, want) <= kMaxWarps) cl = want;
  }
  return cl < 1 ? 1 : (cl > kMaxCluster ? kMaxCluster : cl);
}


// Int-pass launches fit two pass CTAs on an SM (228 KB of shared memory, 1 KB reserved per
// CTA, the static barriers); fp64 launches may take the whole opt-in.
constexpr size_t kSmemBudgetInt = 111 * 1024;
constexpr size_t kSmemBudgetF64 = 220 * 1024;

size_t dp_smem_bytes(int pitch, int dp_warps, bool f64) {
  return 2 * (size_t)(f64 ? 8 : 4) * pitch +
         (size_t)dp_warps * ((f64 ? dp_ring_bytes<true>() : dp_ring_bytes<false>()) + 8 * kPwStageWords);
}

size_t carve_smem_bytes(int rows, int pitch, bool stage, int dp_warps, bool f64) {
  const int nblk = (rows - 1 + kBlockRows - 1) / kBlockRows;
  const size_t dp = dp_smem_bytes(pitch, dp_warps, f64);
  // (the fp64 pass never stages the delta table: select_trace)
  const size_t sel = f64 ? sel_bytes<true>(pitch) : sel_bytes<false>(pitch) + (stage ? (size_t)nblk * pitch : 0);
  return dp > sel ? dp : sel;
}

// shared memory of this variant's fp64 pass (the first pass of a run with a uniform map): the
// launcher runs that pass with the narrowest variant that keeps it within the two-CTA budget
size_t carve_f64_smem(int width, int cl) { return carve_smem_bytes(2, (width + 15) & ~15, false, carve_dp_warps(width, cl), true); }
bool carve_f64_fits_pair(int width, int cl) { return carve_f64_smem(width, cl) <= kSmemBudgetInt; }

int carve_warps(int width, int cl) { return carve_dp_warps(width, cl); }

// Fused int passes need, at every width the run's int passes see (target < w <= width0): at
// least kXRows columns per CTA (neighbour exchanges) and at most kProdWarps DP warps.
static int fused_ring_cap(int width0, int cl);
// Opt-in (SCPL_FUSED=1): bit-exact, but measured slower than the separate row kernels -- the
// producer warps are latency-bound next to the DP warps.
bool carve_fused_ok(int width0, int target, int cl) {
  if (!getenv("SCPL_FUSED")) return false;
  const int per_min = ((target + 1 + cl - 1) / cl + 15) & ~15;
  return per_min >= kXRows && carve_dp_warps(width0, cl) <= kDpWarps &&
         fused_dp_bytes((width0 + 15) & ~15, fused_ring_cap(width0, cl)) <= kSmemBudgetInt;
}

// energy-ring row stride: the widest CTA range over every width up to width0 (a function of the
// initial width and cluster size only, so launchers size the shared memory from them)
static int fused_ring_cap(int width0, int cl) {
  thread_local int c_w = -1, c_cl = -1, c_rw = 0;  // (launchers ask per iteration in host loops)
  if (width0 == c_w && cl == c_cl) return c_rw;
  int rw = 16;
  for (int w = 1; w <= width0; ++w)
    for (int r = 0; r < cl; ++r) {
      int lo = 0, hi = 0;
      if (fused_cta_range(w, cl, r, lo, hi)) rw = std::max(rw, (hi - lo + 15) & ~15);
    }
  c_w = width0;
  c_cl = cl;
  c_rw = rw;
  return rw;
}
int carve_fused_ring_w(int width0, int target, int cl) {
  (void)target;
  return fused_ring_cap(width0, cl);
}

// pass, compact, gradient, check (+ mean with reaverage_energy)
int carve_kernels_per_iteration(bool reaverage) { return reaverage ? 5 : 4; }

// the landing-delta table is staged in shared memory when the int layout still fits two CTAs
// per SM with it (and the fp64 layout the opt-in)
bool carve_stage_dtab(int rows, int pitch, int cl) {
  return carve_smem_bytes(rows, pitch, true, carve_dp_warps(pitch, cl), false) <= kSmemBudgetInt;
}

// one carve iteration (pass, compaction, gradient [, mean]); f64 = the pass may be an fp64 one
// (first pass of runs with a uniform map, or reaverage_energy): the larger shared-memory layout
// Loop condition of the device-side carve loop: another iteration while any run is above its
// target (bounded by max_iters: every pass removes at least one seam).
__global__ void carve_check_kernel(const CarveRun* __restrict__ runs, int nruns, int max_iters, int* iters,
                                   cudaGraphConditionalHandle loop) {
  pdl_wait();
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < nruns; r += blockDim.x)
    if (runs[r].width > runs[r].target) any = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int n = ++*iters;
    cudaGraphSetConditional(loop, (any && n < max_iters) ? 1u : 0u);
  }
}

static void launch_carve_check(CarveRun* runs_d, int nruns, int max_iters, int* iters_d,
                               cudaGraphConditionalHandle h, cudaStream_t cs, bool pdl = true) {
  if (!pdl) {
    carve_check_kernel<<<1, 256, 0, cs>>>((const CarveRun*)runs_d, nruns, max_iters, iters_d, h);
    SCPL_CUDA(cudaGetLastError());
    return;
  }
  cudaLaunchAttribute pa[1];
  pa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pa[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cc = {};
  cc.gridDim = dim3(1);
  cc.blockDim = dim3(256);
  cc.stream = cs;
  cc.attrs = pa;
  cc.numAttrs = 1;
  SCPL_CUDA(cudaLaunchKernelEx(&cc, carve_check_kernel, (const CarveRun*)runs_d, nruns, max_iters, iters_d, h));
}

void launch_carve_iteration(CarveRun* runs_d, int nruns, int rows, int pitch, int width, int cl, cudaStream_t st,
                            int max_fr, bool reaverage, bool f64, const RowsLoop* loop, bool fused) {
  if (nruns == 0) return;
  const int dpw = carve_dp_warps(width, cl);
  SCPL_ARG(dpw <= kMaxWarps, "carve width too large for the cluster size");
  const bool stage = carve_stage_dtab(rows, pitch, cl);
  f64 = f64 || reaverage;
  size_t smem = carve_smem_bytes(rows, pitch, stage, dpw, f64);
  const bool fk = fused && !f64;  // the fused kernel: its DP phase holds the producer rings
  if (fk) smem = std::max(carve_smem_bytes(rows, pitch, stage, dpw, false), fused_dp_bytes(pitch, fused_ring_cap(width, cl)));
  SCPL_ARG(smem <= 227 * 1024, "carve plane too large for shared memory");
  smem_optin(reinterpret_cast<const void*>(carve_pass_kernel));
  smem_optin(reinterpret_cast<const void*>(carve_pass_fused_kernel));
  if (cl > 8 && once_per_device(reinterpret_cast<const void*>(&launch_carve_iteration))) {
    SCPL_CUDA(cudaFuncSetAttribute(carve_pass_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SCPL_CUDA(cudaFuncSetAttribute(carve_pass_fused_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nruns * cl);
  cfg.blockDim = dim3((fk ? kFusedWarps : kMaxWarps) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (fk)
    SCPL_CUDA(cudaLaunchKernelEx(&cfg, carve_pass_fused_kernel, runs_d, cl));
  else
    SCPL_CUDA(cudaLaunchKernelEx(&cfg, carve_pass_kernel, runs_d, cl, f64 ? 1 : 0));
  SCPL_CHECK_LAUNCH();
  const bool fork = loop && loop->side && !fused && !reaverage;
  if (fork) {  // the widths are final once the pass is done: the loop condition on a side branch
    SCPL_CUDA(cudaEventRecord(loop->e_fork, st));
    SCPL_CUDA(cudaStreamWaitEvent(loop->side, loop->e_fork, 0));
    launch_carve_check(runs_d, nruns, loop->max_iters, loop->counters, loop->handle, loop->side, false);
    SCPL_CUDA(cudaEventRecord(loop->e_join, loop->side));
  }
  if (fused) {  // the next pass's producers remove this batch: no row kernels
    if (reaverage) launch_carve_mean(runs_d, nruns, rows, st);
    if (loop) launch_carve_check(runs_d, nruns, loop->max_iters, loop->counters, loop->handle, st);
    return;
  }
  const size_t csmem = carve_compact_smem(pitch);
  smem_optin(reinterpret_cast<const void*>(carve_compact_kernel));
  cudaLaunchAttribute pa[1];
  pa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pa[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t rc = {};
  rc.gridDim = dim3(cdiv(rows, kCompWarps), nruns, max_fr);
  rc.blockDim = dim3(kCompWarps * 32);
  rc.dynamicSmemBytes = csmem;
  rc.stream = st;
  rc.attrs = pa;
  rc.numAttrs = 1;
  SCPL_CUDA(cudaLaunchKernelEx(&rc, carve_compact_kernel, runs_d));
  SCPL_CHECK_LAUNCH();
  rc.gridDim = dim3(cdiv(rows, kRowWarps), nruns, max_fr);
  rc.blockDim = dim3(kRowWarps * 32);
  rc.dynamicSmemBytes = 0;
  SCPL_CUDA(cudaLaunchKernelEx(&rc, carve_dirty_kernel, runs_d));
  SCPL_CHECK_LAUNCH();
  if (reaverage) launch_carve_mean(runs_d, nruns, rows, st);
  if (fork)
    SCPL_CUDA(cudaStreamWaitEvent(st, loop->e_join, 0));
  else if (loop)
    launch_carve_check(runs_d, nruns, loop->max_iters, loop->counters, loop->handle, st);
}

// Word copy by the SMs.  Small control transfers between device memory and mapped pinned
// host memory go through here instead of the copy engines, so they never queue behind the
// clip's bulk host<->device copies.
__global__ void word_copy_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

void launch_word_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  const size_t n = (bytes + 3) / 4;
  word_copy_kernel<<<(int)std::min<size_t>(cdiv((long)n, 256), 64), 256, 0, st>>>(
      reinterpret_cast<uint32_t*>(dst), reinterpret_cast<const uint32_t*>(src), n);
  SCPL_CHECK_LAUNCH();
}

// carve every run to its target in ONE graph launch: [first iteration with the fp64-sized
// pass, then] while (any run above target) { pass; compact; gradient } -- no host round trip
// per iteration.  first_f64: the runs' first pass is an fp64 one (they carry a uniform map).
cudaGraphExec_t build_carve_loop(CarveRun* runs_d, int nruns, int rows, int pitch, int width, int cl, int max_iters,
                                 int* iters_d, int max_fr, bool reaverage, bool first_f64, FirstIter first,
                                 int first_cl, bool fused, int prio) {
  cudaGraph_t g;
  SCPL_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  SCPL_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaStream_t cs = capture_stream(prio);
  const long before = g_launches.load();
  cudaGraphNode_t pro_last = nullptr;
  if (first_f64 && !reaverage) {  // prologue: the fp64 pass, then the condition for the loop
    SCPL_CUDA(cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    const RowsLoop lp{max_iters, iters_d, h};
    (first ? first : launch_carve_iteration)(runs_d, nruns, rows, pitch, width, first ? first_cl : cl, cs, max_fr,
                                             reaverage, true, &lp, fused);
    cudaStreamCaptureStatus cst;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    SCPL_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps));
    SCPL_ARG(ndeps == 1, "internal: carve prologue must end in one node");
    pro_last = deps[0];  // the kernel that sets the condition
    SCPL_CUDA(cudaStreamEndCapture(cs, &g));
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cond;
  SCPL_CUDA(cudaGraphAddNode(&cond, g, pro_last ? &pro_last : nullptr, pro_last ? 1 : 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  SCPL_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  {
    // the loop condition on a side branch of the body (SCPL_CHECK_FORK=0: after the row kernels)
    static const bool check_fork = !(getenv("SCPL_CHECK_FORK") && atoi(getenv("SCPL_CHECK_FORK")) == 0);
    RowsLoop lp{max_iters, iters_d, h};
    if (check_fork) {
      SCPL_CUDA(cudaStreamCreateWithFlags(&lp.side, cudaStreamNonBlocking));
      SCPL_CUDA(cudaEventCreateWithFlags(&lp.e_fork, cudaEventDisableTiming));
      SCPL_CUDA(cudaEventCreateWithFlags(&lp.e_join, cudaEventDisableTiming));
    }
    // (unrolled bodies: the loop's re-evaluation is paid once per carve_unroll() iterations; only
    // the last one carries the condition kernel)
    const int unroll = carve_unroll();
    for (int u = 0; u < unroll; ++u)
      launch_carve_iteration(runs_d, nruns, rows, pitch, width, cl, cs, max_fr, reaverage, false,
                             u == unroll - 1 ? &lp : nullptr, fused);
    SCPL_CUDA(cudaStreamEndCapture(cs, &body));
    if (check_fork) {
      cudaEventDestroy(lp.e_fork);
      cudaEventDestroy(lp.e_join);
      cudaStreamDestroy(lp.side);
    }
  }
  graph_set_priority(g, prio);
  graph_set_priority(body, prio);
  g_launches.store(before);  // counted per executed iteration by the caller
  cudaGraphExec_t ex;
  SCPL_CUDA(cudaGraphInstantiate(&ex, g, 0));
  cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  return ex;
}

void launch_carve_index(CarveRun* runs_d, int nruns, int rows, cudaStream_t st) {
  if (nruns == 0) return;
  carve_index_kernel<<<dim3(cdiv(rows, kRowWarps), nruns), kRowWarps * 32, 0, st>>>(runs_d);
  SCPL_CHECK_LAUNCH();
}

}  // namespace SCPL_KC_NS
}  // namespace scpl
