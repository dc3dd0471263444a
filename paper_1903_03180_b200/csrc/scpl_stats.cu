// K2: window statistics for the spatio-temporal buffer scan (ASDE), bit-exact.
//
// Replaces SpatioTemporalBuffer.push's candidate test (buffering.py:115-119) and
// _asde_from_sums (buffering.py:174-176).  For a run start s with n_acc frames already
// accepted, one launch evaluates L candidate lengths n = n_acc+1 .. n_acc+L:
//   S += e_t, Q += fl(e_t*e_t)                      (per pixel, stream order; :116-117)
//   var = fl(Q/n) - fl(fl(S/n)^2); std = sqrt(max(var, 0))
//   ASDE(n) = pairwise_sum(std over the row-major map) / (H*W)   (numpy's tree)
// numpy's pairwise tree splits [0, N) recursively (n2 = n/2 rounded down to a multiple of
// 8) into leaves of <= 128 elements, each summed with 8 strided accumulators.  The host
// enumerates the leaves once per shape; here a group of 8 lanes owns one leaf, lane j
// holding accumulator r[j] and the S,Q of its pixels in registers across all L
// candidates.  A second kernel folds the leaf sums with the same tree (one CTA per
// candidate).  The per-pixel S,Q after the chunk are checkpointed so the next chunk of
// the same run resumes without re-reading earlier frames.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstddef>
#include <vector>

#include "scpl_common.cuh"
#include "scpl_kernels.h"

namespace scpl {

// ------------------------------------------------------------ host: pairwise plan
static void plan_rec(long off, long n, std::vector<int2>& leaves) {
  if (n <= 128) {
    leaves.push_back(make_int2((int)off, (int)n));
    return;
  }
  long h = n / 2;
  h -= h % 8;
  plan_rec(off, h, leaves);
  plan_rec(off + h, n - h, leaves);
}

static long count_leaves(long n) {
  if (n <= 128) return 1;
  long h = n / 2;
  h -= h % 8;
  return count_leaves(h) + count_leaves(n - h);
}

// virtual complete tree of depth D over the recursion: node v (D bits, MSB = first split)
static void vnodes_rec(long n, int depth, int D, int v, long first_leaf, std::vector<PwVnode>& out) {
  if (depth == D) {
    out[v] = PwVnode{(int)first_leaf, n};
    return;
  }
  if (n <= 128) {
    // leaf above depth D: the leftmost descendant carries it, the rest add +0.0 (exact)
    int shift = D - depth;
    out[v << shift] = PwVnode{(int)first_leaf, n};
    return;
  }
  long h = n / 2;
  h -= h % 8;
  vnodes_rec(h, depth + 1, D, 2 * v, first_leaf, out);
  vnodes_rec(n - h, depth + 1, D, 2 * v + 1, first_leaf + count_leaves(h), out);
}

void build_pairwise_plan(long N, std::vector<int2>& leaves, std::vector<PwVnode>& vnodes) {
  leaves.clear();
  plan_rec(0, N, leaves);
  vnodes.assign(1 << kPwDepth, PwVnode{0, 0});
  vnodes_rec(N, 0, kPwDepth, 0, 0, vnodes);
}

// ------------------------------------------------------------ device: leaf sums
// A CTA's 32 leaves cover one contiguous pixel range (<= 4096 pixels).  The codes of every
// frame a launch reads (the run's first frame when it starts a run, then the L candidates)
// stream into an 8-stage shared-memory ring by 1-D TMA bulk copies issued up front, so the
// fp64 work never waits on a global load; lanes then read their strided elements from
// shared memory.  Rows of N not divisible by 8 fall back to cooperative plain copies.
// Screening bound (APPROX).  With u = 2^-53, X = Q/n <= 255^2 (every e <= 255) and
// M = S/n, the screened variance fma(-m, m, RN(Q*rn)) (m = RN(S*rn), rn = RN(1/n)) and the
// reference's RN(RN(Q/n) - RN(RN(S/n)^2)) differ by at most 5.03uX + 9.12uM^2 <= 14.2uX
// (+ O(u^2)) <= 1.03e-10; kScanDelta doubles that.  For x, y >= 0, |sqrt(x) - sqrt(y)| <=
// min(sqrt|x-y|, |x-y| / sqrt(x)), and max(., 0) does not increase the distance, so per pixel
// |std~ - std| <= min(sqrt(delta), delta / std~) plus relative roundings (f32 conversion,
// rsqrt.approx (budgeted at 2^-20), the <= 9-term per-lane f32 sum: < 1.6e-6 of std~), which
// the decision adds separately with a 5x margin.
constexpr float kScanDelta = 2.0e-10f;
constexpr float kScanSqrtDelta = 1.4143e-5f;  // > sqrt(kScanDelta)

constexpr int kLeafLanes = 16;     // lanes per leaf: accumulator j = lanes j (first half) and j + 8
constexpr int kHalfMax = 8;        // elements per lane and accumulator half (a leaf has <= 16 per accumulator)
constexpr int kStatStages = 4;
constexpr int kStatStageBytes = (256 / kLeafLanes) * 128 * 2;  // one CTA's pixels of one frame
// ring, its barriers, the A / B energy tables; screened windows add (sum std~, sum bound) per
// candidate and warp (kStatRed per candidate).  ~21 KB at spec 8: a scan CTA fits on an SM
// next to a resident carve-pass CTA.
constexpr size_t kStatSmem = (size_t)kStatStages * kStatStageBytes + 8 * kStatStages + 2 * 256 * sizeof(double) +
                             kScanMaxL * sizeof(double) + 64;  // (+ slot / window counters)  // (+ the screened body's 1 / n table)
constexpr size_t kStatRed = 16 * sizeof(double);

// numpy's leaf sum (pairwise_sum, n <= 128): r[j] = a[j] + a[j+8] + ... (sequential), then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail elements in order.  Here lane
// (h, j) of a leaf's 16 lanes holds accumulator j's elements m in [h ? m0 : 0, h ? nmain : m0)
// (m0 = ceil(nmain/2)): the first half sums its part, hands the partial to the second half,
// which continues the same sequential sum -- the bracketing is numpy's exactly, with half the
// registers per lane (so twice the resident warps hide the fp64 latency).
//
// APPROX (screening, scan only): per candidate the CTA adds sum(std~) and sum(bound) into
// asum/bsum, where std~ = sqrt_f32(f32(fma(-m, m, Q*rn))), m = S*rn, rn = RN(1/n), and bound
// is a per-pixel bound on |std~ - std| (std = the reference's fl(sqrt(max(var, 0))), see
// kScanDelta) -- see scan_step_kernel for how the decision uses them.  S, Q themselves are
// accumulated exactly as in the exact kernel, so the checkpoint is the reference's.
// The checkpoint is read from ckS/ckQ (runs continued from an earlier window) and written to
// ckSo/ckQo (the same arrays for an in-place update).
template <bool APPROX>
__device__ __forceinline__ void window_stats_body(const uint16_t* __restrict__ codes, long N,
                                                  const int2* __restrict__ leaves, int nleaves, int s, int n_acc,
                                                  int L, int first_pure, int init, double wm, double wg,
                                                  const double* ckS, const double* ckQ, double* ckSo, double* ckQo,
                                                  double* __restrict__ leafsum, double* asum, double* bsum) {
  extern __shared__ __align__(128) uint8_t st_ring[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(st_ring + kStatStages * kStatStageBytes);
  double* A = reinterpret_cast<double*>(bars + kStatStages);
  double* B = A + 256;
  for (int k = threadIdx.x; k < 256; k += blockDim.x) {
    A[k] = __dmul_rn(wm, (double)k);
    B[k] = __dmul_rn(wg, (double)k);
  }
  const int leaves_per_cta = blockDim.x / kLeafLanes;
  const int first = blockIdx.x * leaves_per_cta;
  const int last = min(nleaves, first + leaves_per_cta) - 1;
  const long p_lo = leaves[first].x;
  const int2 lf_last = leaves[last];
  const int npx = (int)(lf_last.x + lf_last.y - p_lo);
  const uint32_t bytes = (uint32_t)((npx * 2 + 15) & ~15);
  const bool bulk = (N & 7) == 0;  // frame rows 16-byte aligned (leaf starts are multiples of 8)
  const int M = L + (init ? 1 : 0);  // frames read: [s if init], s+n_acc .. s+n_acc+L-1
  auto frame_of = [&](int i) { return init ? (i == 0 ? s : s + n_acc + i - 1) : s + n_acc + i; };
  if (bulk) {
    if (threadIdx.x == 0) {
      for (int k = 0; k < kStatStages; ++k) mbar_init(&bars[k], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < M && i < kStatStages; ++i) {
        mbar_arrive_tx(&bars[i], bytes);
        bulk_g2s(st_ring + i * kStatStageBytes, codes + (size_t)frame_of(i) * N + p_lo, bytes, &bars[i]);
      }
    }
  } else {
    __syncthreads();
  }
  // stage i: wait for it (bulk) or fill it cooperatively (plain); returns its base
  auto acquire = [&](int i) -> const uint16_t* {
    uint8_t* st = st_ring + (i % kStatStages) * kStatStageBytes;
    if (bulk) {
      mbar_wait(&bars[i % kStatStages], (uint32_t)(i / kStatStages) & 1u);
    } else {
      const uint16_t* src = codes + (size_t)frame_of(i) * N + p_lo;
      for (int q = threadIdx.x; q < npx; q += blockDim.x) reinterpret_cast<uint16_t*>(st)[q] = src[q];
      __syncthreads();
    }
    return reinterpret_cast<const uint16_t*>(st);
  };
  // stage i fully consumed: refill it with frame i + kStatStages
  auto release = [&](int i) {
    __syncthreads();
    if (bulk && threadIdx.x == 0 && i + kStatStages < M) {
      const int j = i + kStatStages;
      mbar_arrive_tx(&bars[j % kStatStages], bytes);
      bulk_g2s(st_ring + (j % kStatStages) * kStatStageBytes, codes + (size_t)frame_of(j) * N + p_lo, bytes,
               &bars[j % kStatStages]);
    }
  };

  const int lane = threadIdx.x & 31;
  const int sub = lane & 15, j = sub & 7, h = sub >> 3;
  const int leaf = (blockIdx.x * blockDim.x + threadIdx.x) / kLeafLanes;
  const bool active = leaf < nleaves;
  int2 lf = active ? leaves[leaf] : make_int2((int)p_lo, 8);
  const int len = lf.y;
  const int nmain = len >> 3;     // elements per accumulator
  const int ntail = len & 7;      // sequential tail: element 8*nmain + t held by lane (0, t)
  const int m0 = (nmain + 1) >> 1;
  const int mb = h ? m0 : 0, cnt = h ? nmain - m0 : m0;  // this lane's elements
  const long base = lf.x;
  const int lb = (int)(base - p_lo);  // leaf start within the CTA range
  const bool has_tail = active && h == 0 && j < ntail;
  auto off = [&](int k) { return k < kHalfMax ? lb + 8 * (mb + k) + j : lb + 8 * nmain + j; };
  auto valid = [&](int k) { return k < kHalfMax ? (active && k < cnt) : has_tail; };

  double S[kHalfMax + 1], Q[kHalfMax + 1];
  int ci = 0;  // next stage
  if (init) {
    const uint16_t* st = acquire(ci);
#pragma unroll
    for (int k = 0; k <= kHalfMax; ++k) {
      const double e = valid(k) ? energy_of(st[off(k)], first_pure && s == 0, A, B) : 0.0;
      S[k] = e;
      Q[k] = __dmul_rn(e, e);
    }
    release(ci++);
  } else {
#pragma unroll
    for (int k = 0; k <= kHalfMax; ++k) {
      const long p = p_lo + off(k);
      S[k] = valid(k) ? ckS[p] : 0.0;
      Q[k] = valid(k) ? ckQ[p] : 0.0;
    }
  }

  const int g0 = lane & ~15;  // first lane of this leaf's group
  double* red = B + 256;  // APPROX: per candidate and warp, (sum std~, sum bound)
  for (int c = 0; c < L; ++c, ++ci) {
    const int t = s + n_acc + c;
    const int n = n_acc + c + 1;
    const double dn = (double)n;
    const double rn = __ddiv_rn(1.0, dn);
    const uint16_t* ct = acquire(ci);
    const bool pure = first_pure && t == 0;
    if constexpr (APPROX) {
      float as = 0.f, ab = 0.f;
#pragma unroll
      for (int k = 0; k <= kHalfMax; ++k) {
        if (valid(k)) {
          // the tables' products recomputed on the fp64 pipe (A[d] == fl(wm * d) exactly): no
          // bank-conflicted table loads
          const uint32_t code = ct[off(k)];
          const double e = pure ? (double)(code & 255u)
                                : fmin(__dadd_rn(__dmul_rn(wm, (double)(code >> 8)), __dmul_rn(wg, (double)(code & 255u))),
                                       255.0);
          S[k] = __dadd_rn(S[k], e);
          Q[k] = __dadd_rn(Q[k], __dmul_rn(e, e));
          const double m = __dmul_rn(S[k], rn);
          const double var = __fma_rn(-m, m, __dmul_rn(Q[k], rn));
          // std~ = v * rsqrt(v) (MUFU; v > 0 so no 0 * inf); a variance <= 0 gives std~ ~ 1e-15
          // and the bound sqrt(delta), which covers the reference's std <= sqrt(delta) there
          const float v = fmaxf(__double2float_rn(var), 1e-30f);
          float rs;
          asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(v));
          as += v * rs;
          ab += fminf(kScanSqrtDelta, kScanDelta * rs);
        }
      }
      release(ci);
      double ds = (double)as, db = (double)ab;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ds += __shfl_xor_sync(0xffffffffu, ds, o);
        db += __shfl_xor_sync(0xffffffffu, db, o);
      }
      if (lane == 0) {
        red[(c * 8 + (threadIdx.x >> 5)) * 2] = ds;
        red[(c * 8 + (threadIdx.x >> 5)) * 2 + 1] = db;
      }
      continue;
    }
    double sd[kHalfMax + 1];
#pragma unroll
    for (int k = 0; k <= kHalfMax; ++k) {
      sd[k] = 0.0;
      if (valid(k)) {
        const double e = energy_of(ct[off(k)], pure, A, B);
        S[k] = __dadd_rn(S[k], e);
        Q[k] = __dadd_rn(Q[k], __dmul_rn(e, e));
        const double m = div_small(S[k], dn, rn);
        const double var = __dsub_rn(div_small(Q[k], dn, rn), __dmul_rn(m, m));
        sd[k] = __dsqrt_rn(var >= 0.0 ? var : 0.0);
      }
    }
    release(ci);
    // first half: r_j's leading part; second half continues the sequential sum
    double acc = sd[0];
#pragma unroll
    for (int k = 1; k < kHalfMax; ++k)
      if (h == 0 && k < cnt) acc = __dadd_rn(acc, sd[k]);
    const double part = __shfl_sync(0xffffffffu, acc, g0 + j);
    if (h == 1) {
      acc = part;
#pragma unroll
      for (int k = 0; k < kHalfMax; ++k)
        if (k < cnt) acc = __dadd_rn(acc, sd[k]);
    }
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) in the second half (xor within lanes 8..15)
    double x = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
    x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 2));
    x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 4));
    if (nmain == 0) x = 0.0;  // n < 8: numpy's plain loop from 0
    for (int k = 0; k < 7; ++k) {  // tail elements in order (uniform trip count for shuffles)
      const double tv = __shfl_sync(0xffffffffu, sd[kHalfMax], g0 + k);
      if (k < ntail) x = __dadd_rn(x, tv);
    }
    if (active && sub == 8) leafsum[(size_t)c * nleaves + leaf] = x;
  }

  if constexpr (APPROX) {  // this CTA's per-candidate sums (release() synchronised the warps)
    __syncthreads();
    for (int c = threadIdx.x; c < L; c += blockDim.x) {
      double ds = 0.0, db = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        ds += red[(c * 8 + w) * 2];
        db += red[(c * 8 + w) * 2 + 1];
      }
      atomicAdd(&asum[c], ds);
      atomicAdd(&bsum[c], db);
    }
  }
  // checkpoint S,Q after n_acc + L frames
#pragma unroll
  for (int k = 0; k <= kHalfMax; ++k) {
    if (valid(k)) {
      const long p = p_lo + off(k);
      ckSo[p] = S[k];
      ckQo[p] = Q[k];
    }
  }
}

// ------------------------------------------------------------ device: screened windows
// The screened (APPROX) evaluation of a window does not need numpy's summation tree: only
// S and Q per pixel are exact (they are the checkpoint); sum(std~) and sum(bound) may be
// added in any order (their f32 roundings are part of scan_step_kernel's margin).  So this
// body drops the leaf layout: a CTA owns `chunk` consecutive pixels (a multiple of 8, sized so
// the grid is a whole number of waves), thread t the pixel pairs 2 (t + 256 k), k = 0..3 --
// one 32-bit shared-memory load per pair and frame, one 16-byte checkpoint load / store per
// pair, no per-pixel branches (warps skip whole k slots past the chunk; only the one warp on
// the chunk's edge runs the masked variant).  Per pixel and candidate: 2 I2F, 9 fp64
// operations (e, S, Q, m, Q/n, var), F2F, MUFU.RSQ and 5 f32 operations.
//   * the clamp min(e, 255) is a no-op when wm, wg >= 0 and fl(fl(255 wm) + fl(255 wg)) <= 255
//     (rounding is monotone, so every e is <= that value): CLAMP = false drops it;
//   * a pure-gradient frame (the clip's first, energy.py:79-80) is wm = 0, wg = 1 (exact);
//   * the bound min(sqrt(delta), delta * rs) is accumulated as min(1 / sqrt(delta), rs) and
//     scaled by delta once per CTA: kScrCap * kScanDelta == kScanSqrtDelta, and the f32 sums'
//     relative rounding (< 2e-6) is far inside kScanDelta's factor 2 over the proven bound.
constexpr int kScrPairs = 4;                          // pixel pairs per thread
constexpr int kScrMaxChunk = 256 * 2 * kScrPairs;     // 2048 pixels per CTA at most
constexpr float kScrCap = 70715.0f;                   // kScanSqrtDelta / kScanDelta
// The screened body's ring holds a whole default window (8 candidates + the initial frame start
// with every copy in flight): the kernel is bound by memory latency, not by a pipe (ncu round
// 2d: SMs active 75% of the time, issue slots 50%, DRAM 18%), so nothing waits on a refill.
constexpr int kScrStages = 8;
constexpr size_t kScrSmem = (size_t)kScrStages * kStatStageBytes + 8 * kScrStages + kScanMaxL * 8 * 2 * sizeof(float) +
                            kScanMaxL * sizeof(double) + 64;  // (+ slot / window counters)
static_assert(kScrMaxChunk * 2 <= kStatStageBytes, "a chunk's codes of one frame fit a ring stage");

// CTAs' pixels for a frame of N pixels: the smallest whole number of waves (4 CTAs per SM)
// that keeps a chunk within kScrMaxChunk; a multiple of 8 pixels (16-byte bulk copies)
int screen_chunk(long N, int num_sms) {
  const long wave = (long)std::max(1, num_sms) * 4;
  long g = wave;
  while (cdiv(N, g) > kScrMaxChunk) g += wave;
  long chunk = cdiv(N, g);
  chunk = (chunk + 7) & ~7L;
  return (int)std::min<long>(kScrMaxChunk, std::max<long>(512, chunk));
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// Integer -> double and double -> float without the conversion unit: the window kernel was
// bound by the XU pipe (I2F.F64, F2F.F32.F64 and MUFU share it: 68% busy, ncu round 2d) while
// the fp64 pipe idled.  u8_f64: 2^52 + k is exact in the low mantissa bits, minus 2^52 (exact).
// f64_f32_floor: max(var, ~1e-30) on the high word (doubles order like sign-magnitude integers,
// a negative variance has the sign bit set), then the f32 bit pattern by re-biasing the exponent
// and a funnel shift: truncation instead of rounding, a relative error < 2^-23 that is part of
// the decision's relative margin (see below).
__device__ __forceinline__ double u8_f64(uint32_t k) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)k), 4503599627370496.0);
}
__device__ __forceinline__ float f64_f32_floor(double var) {
  const int hi = max(__double2hiint(var), 0x39B4484B);  // high word of 1e-30
  return __uint_as_float(__funnelshift_l((uint32_t)__double2loint(var), (uint32_t)(hi - 0x38000000), 3));
}

// Relative f32 errors of one pixel's std~ and of the sums: truncation 2^-23, rsqrt.approx 2^-20
// (budget), the fused multiply-add, the 8-term per-lane sum, 5 shuffle adds -- < 2e-6 in total;
// scan_decide_plan budgets 8e-6.
template <bool CLAMP>
__device__ __forceinline__ void screen_px(uint32_t d, uint32_t g, double wm, double wg, double rn, double& S,
                                          double& Q, float& as, float& ab, float mask, bool masked) {
  double e = __dadd_rn(__dmul_rn(wm, u8_f64(d)), __dmul_rn(wg, u8_f64(g)));
  if (CLAMP) e = e > 255.0 ? 255.0 : e;  // (never NaN)
  S = __dadd_rn(S, e);
  Q = __dadd_rn(Q, __dmul_rn(e, e));
  const double m = __dmul_rn(S, rn);
  const double var = __fma_rn(-m, m, __dmul_rn(Q, rn));
  // std~ = v * rsqrt(v) (v > 0, so no 0 * inf); a variance <= 0 gives std~ ~ 1e-15 and the
  // bound sqrt(delta), which covers the reference's std <= sqrt(delta) there
  const float v = f64_f32_floor(var);
  float rs;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(v));
  if (masked) {
    as = __fmaf_rn(__fmul_rn(v, rs), mask, as);
    ab = __fmaf_rn(fminf(kScrCap, rs), mask, ab);
  } else {
    as = __fmaf_rn(v, rs, as);
    ab = __fadd_rn(ab, fminf(kScrCap, rs));
  }
}

// Every CTA of a window launch checks in once its sums (or leaf sums) are written -- also the
// CTAs with nothing to do for this window's layout, so that no CTA can read the scan state
// after it has been advanced.  True (block-uniform) for the last CTA of the grid.
__device__ __forceinline__ bool scan_window_arrive(ScanState* S) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&S->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  return s_last != 0;
}

__device__ void scan_screen_finish_warp(ScanState* S, cudaGraphConditionalHandle loop, int in_graph);

// one candidate frame for this thread's K full pixel pairs (no masks)
template <bool CLAMP, int K>
__device__ __forceinline__ void screen_frame_full(uint32_t a, double wm, double wg, double rn, double (&S)[8],
                                                  double (&Q)[8], float& as, float& ab) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t w = lds_u32(a + 1024 * k);
    screen_px<CLAMP>(__byte_perm(w, 0u, 0x4441), w & 255u, wm, wg, rn, S[2 * k], Q[2 * k], as, ab, 1.f, false);
    screen_px<CLAMP>(w >> 24, __byte_perm(w, 0u, 0x4442), wm, wg, rn, S[2 * k + 1], Q[2 * k + 1], as, ab, 1.f, false);
  }
}

template <bool CLAMP>
__device__ __forceinline__ bool window_screen_body(const uint16_t* __restrict__ codes, long N, int chunk, int s,
                                                   int n_acc, int L, int init, double wm0, double wg0,
                                                   const double* ckS, const double* ckQ, double* ckSo,
                                                   double* ckQo, double* asum, double* bsum, ScanState* Sg,
                                                   cudaGraphConditionalHandle loop, int in_graph) {
  extern __shared__ __align__(128) uint8_t st_ring[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(st_ring + kScrStages * kStatStageBytes);
  float* red = reinterpret_cast<float*>(bars + kScrStages);             // [L][8 warps][2]
  double* rns = reinterpret_cast<double*>(red + kScanMaxL * 8 * 2);      // [L]: RN(1 / n)
  int* cnt = reinterpret_cast<int*>(rns + kScanMaxL);                    // [stages]: warps done with a slot
  int* done = cnt + kScrStages;                                          // warps done with the window
  const long p0 = (long)blockIdx.x * chunk;
  if (p0 >= N) return scan_window_arrive(Sg);
  const int npx = (int)min((long)chunk, N - p0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // slot k of this warp covers chunk pixels [512 k + 64 warp, + 64): nfull slots are entirely
  // inside the chunk (warp-uniform: 4 or 3 of them run the unmasked code), the next one may be
  // partly inside (edge: masked), the rest are skipped
  const int wb = 64 * warp;
  const int nfull = npx >= wb + 64 ? min(kScrPairs, (npx - wb - 64) / 512 + 1) : 0;
  const bool edge = nfull < kScrPairs && 512 * nfull + wb < npx;
  const int i0e = 512 * nfull + 2 * (int)threadIdx.x - 64 * warp + wb;  // this thread's first edge-slot pixel
  const float mk0 = edge && i0e < npx ? 1.f : 0.f, mk1 = edge && i0e + 1 < npx ? 1.f : 0.f;
  auto slot_on = [&](int k) { return k < nfull || (k == nfull && edge); };
  auto px_on = [&](int k, int u) { return k < nfull || (k == nfull && (u ? mk1 : mk0) != 0.f); };
  const bool vec = ((N & 1) == 0) && ((reinterpret_cast<uintptr_t>(ckS) | reinterpret_cast<uintptr_t>(ckQ) |
                                       reinterpret_cast<uintptr_t>(ckSo) | reinterpret_cast<uintptr_t>(ckQo)) &
                                      15) == 0;
  double S[2 * kScrPairs], Q[2 * kScrPairs];
  // the checkpoint first: its loads are in flight while the ring is set up
  if (!init) {
#pragma unroll
    for (int k = 0; k < kScrPairs; ++k) {
      S[2 * k] = S[2 * k + 1] = Q[2 * k] = Q[2 * k + 1] = 0.0;
      if (!slot_on(k)) continue;
      const long p = p0 + 512 * k + 2 * (int)threadIdx.x;
      if (k < nfull && vec) {
        const double2 sv = *reinterpret_cast<const double2*>(ckS + p);
        const double2 qv = *reinterpret_cast<const double2*>(ckQ + p);
        S[2 * k] = sv.x, S[2 * k + 1] = sv.y, Q[2 * k] = qv.x, Q[2 * k + 1] = qv.y;
      } else {
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (px_on(k, u)) S[2 * k + u] = ckS[p + u], Q[2 * k + u] = ckQ[p + u];
      }
    }
  }

  const uint32_t bytes = (uint32_t)((npx * 2 + 15) & ~15);
  const bool bulk = (N & 7) == 0;  // frame rows 16-byte aligned (chunk starts are multiples of 8)
  const int M = L + (init ? 1 : 0);  // frames read: [s if init], s+n_acc .. s+n_acc+L-1
  auto frame_of = [&](int i) { return init ? (i == 0 ? s : s + n_acc + i - 1) : s + n_acc + i; };
  for (int c = threadIdx.x; c < L; c += blockDim.x) rns[c] = __ddiv_rn(1.0, (double)(n_acc + c + 1));
  if (threadIdx.x <= kScrStages) cnt[threadIdx.x] = 0;  // (cnt[kScrStages] is `done`)
  if (bulk) {
    if (threadIdx.x == 0) {
      for (int k = 0; k < kScrStages; ++k) mbar_init(&bars[k], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < M && i < kScrStages; ++i) {
        mbar_arrive_tx(&bars[i], bytes);
        bulk_g2s(st_ring + i * kStatStageBytes, codes + (size_t)frame_of(i) * N + p0, bytes, &bars[i]);
      }
    }
  } else {
    __syncthreads();
  }
  const uint32_t ring_s = smem_u32(st_ring) + 4 * threadIdx.x;
  auto acquire = [&](int i) -> uint32_t {  // this thread's first pair in stage i
    const int slot = i % kScrStages;
    if (bulk) {
      mbar_wait(&bars[slot], (uint32_t)(i / kScrStages) & 1u);
    } else {
      const uint16_t* src = codes + (size_t)frame_of(i) * N + p0;
      uint16_t* st = reinterpret_cast<uint16_t*>(st_ring + slot * kStatStageBytes);
      for (int q = threadIdx.x; q < npx; q += blockDim.x) st[q] = src[q];
      __syncthreads();
    }
    return ring_s + slot * kStatStageBytes;
  };
  // stage i consumed.  No block barrier anywhere in the window: a slot that is needed again
  // (windows longer than the ring) is refilled by the LAST warp to finish with it (a shared
  // counter per slot), so the warps run through the window's frames on their own, waiting only
  // on the frames' copies.  (Plain fills: a thread refilling slot i has passed the barrier of
  // acquire(i + kScrStages - 1), which every thread reaches after its frame i.)
  const int nwarps = (int)(blockDim.x >> 5);
  auto release = [&](int i) {
    if (bulk && i + kScrStages < M) {
      __syncwarp();
      if (lane == 0) {
        const int slot = i % kScrStages;
        __threadfence_block();
        if (atomicAdd(&cnt[slot], 1) == nwarps - 1) {
          cnt[slot] = 0;
          __threadfence_block();
          fence_proxy_async();  // (the warps' reads of the slot before the async refill)
          const int j = i + kScrStages;
          mbar_arrive_tx(&bars[slot], bytes);
          bulk_g2s(st_ring + slot * kStatStageBytes, codes + (size_t)frame_of(j) * N + p0, bytes, &bars[slot]);
        }
      }
    }
  };

  int ci = 0;  // next stage
  if (init) {
    const uint32_t a = acquire(ci);
    const bool pure0 = s == 0;  // (the clip's first frame is pure gradient: wm = 0, wg = 1)
    const double wm = pure0 ? 0.0 : wm0, wg = pure0 ? 1.0 : wg0;
#pragma unroll
    for (int k = 0; k < kScrPairs; ++k) {
      S[2 * k] = S[2 * k + 1] = Q[2 * k] = Q[2 * k + 1] = 0.0;
      if (!slot_on(k)) continue;
      const uint32_t w = lds_u32(a + 1024 * k);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t c16 = u ? w >> 16 : w & 0xffffu;
        double e = __dadd_rn(__dmul_rn(wm, (double)(c16 >> 8)), __dmul_rn(wg, (double)(c16 & 255u)));
        e = e > 255.0 ? 255.0 : e;
        S[2 * k + u] = e;
        Q[2 * k + u] = __dmul_rn(e, e);
      }
    }
    release(ci++);
  }

  // (a candidate is never the clip's first frame: the scan state keeps n_acc >= 1, so the
  // pure-gradient frame 0 only ever enters as a run's initial frame above)
  SCPL_DCHECK(s + n_acc >= 1, "screened candidate at frame 0");
  const double wm = wm0, wg = wg0;
  const int path = nfull == kScrPairs ? 0 : (nfull == kScrPairs - 1 && !edge ? 1 : 2);
  for (int c = 0; c < L; ++c, ++ci) {
    const uint32_t a = acquire(ci);
    const double rn = rns[c];
    float as = 0.f, ab = 0.f;
    if (path == 0) {
      screen_frame_full<CLAMP, kScrPairs>(a, wm, wg, rn, S, Q, as, ab);
    } else if (path == 1) {
      screen_frame_full<CLAMP, kScrPairs - 1>(a, wm, wg, rn, S, Q, as, ab);
    } else {
#pragma unroll
      for (int k = 0; k < kScrPairs; ++k) {
        if (!slot_on(k)) continue;
        const uint32_t w = lds_u32(a + 1024 * k);
        const bool m = k >= nfull;
        screen_px<CLAMP>(__byte_perm(w, 0u, 0x4441), w & 255u, wm, wg, rn, S[2 * k], Q[2 * k], as, ab,
                         m ? mk0 : 1.f, true);
        screen_px<CLAMP>(w >> 24, __byte_perm(w, 0u, 0x4442), wm, wg, rn, S[2 * k + 1], Q[2 * k + 1], as, ab,
                         m ? mk1 : 1.f, true);
      }
    }
    release(ci);
    // warp sums of (as, ab): lanes 0-15 fold as, lanes 16-31 fold ab
    const bool hi = (lane & 16) != 0;
    float x = hi ? ab : as;
    const float y = hi ? as : ab;
    x = __fadd_rn(x, __shfl_xor_sync(0xffffffffu, y, 16));
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) x = __fadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
    if ((lane & 15) == 0) red[(c * 8 + warp) * 2 + (lane >> 4)] = x;
  }

  // The last warp of the CTA to finish the window adds the CTA's sums to the global ones and
  // checks the CTA in (scan_window_arrive's ticket); every warp then stores its checkpoint (the
  // deciding warp only needs the sums; the stores are ordered before the next window by the
  // kernel boundary).  The last warp of the last CTA decides and plans.
  __syncwarp();
  int flag = 0;
  if (lane == 0) {
    __threadfence_block();
    flag = atomicAdd(done, 1) == nwarps - 1;
  }
  const bool cta_last = __shfl_sync(0xffffffffu, flag, 0) != 0;
  bool grid_last = false;
  if (cta_last) {
    __threadfence_block();
    for (int c = lane; c < L; c += 32) {
      double ds = 0.0, db = 0.0;
      for (int w = 0; w < nwarps; ++w) {
        ds += (double)red[(c * 8 + w) * 2];
        db += (double)red[(c * 8 + w) * 2 + 1];
      }
      atomicAdd(&asum[c], ds);
      atomicAdd(&bsum[c], db * (double)kScanDelta);
    }
    __syncwarp();
    flag = 0;
    if (lane == 0) {
      __threadfence();
      flag = atomicAdd(&Sg->ticket, 1u) == gridDim.x - 1;
    }
    grid_last = __shfl_sync(0xffffffffu, flag, 0) != 0;
  }
  // checkpoint S,Q after n_acc + L frames
#pragma unroll
  for (int k = 0; k < kScrPairs; ++k) {
    if (!slot_on(k)) continue;
    const long p = p0 + 512 * k + 2 * (int)threadIdx.x;
    if (k < nfull && vec) {
      *reinterpret_cast<double2*>(ckSo + p) = make_double2(S[2 * k], S[2 * k + 1]);
      *reinterpret_cast<double2*>(ckQo + p) = make_double2(Q[2 * k], Q[2 * k + 1]);
    } else {
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (px_on(k, u)) ckSo[p + u] = S[2 * k + u], ckQo[p + u] = Q[2 * k + u];
    }
  }
  if (grid_last) scan_screen_finish_warp(Sg, loop, in_graph);
  return false;  // (decided here if this was the last CTA)
}

__device__ __forceinline__ bool screen_noclamp(double wm, double wg) {
  return __double2hiint(wm) >= 0 && __double2hiint(wg) >= 0 &&
         __dadd_rn(__dmul_rn(wm, 255.0), __dmul_rn(wg, 255.0)) <= 255.0;  // (false for NaN weights)
}

__global__ void __launch_bounds__(256, 3) window_stats_kernel(const uint16_t* __restrict__ codes, long N,
                                                           const int2* __restrict__ leaves, int nleaves,
                                                           int s, int n_acc, int L, int first_pure, int init,
                                                           double wm, double wg, double* __restrict__ ckS,
                                                           double* __restrict__ ckQ,
                                                           double* __restrict__ leafsum) {
  window_stats_body<false>(codes, N, leaves, nleaves, s, n_acc, L, first_pure, init, wm, wg, ckS, ckQ, ckS, ckQ,
                           leafsum, nullptr, nullptr);
}

// Scan variant: the window comes from the device-side scan state (no host round trip).  The grid
// covers both layouts (scan_grid): exact windows by leaves, screened windows by pixel chunks.
__device__ void scan_window_finish(ScanState* S, int nleaves, const PwVnode* __restrict__ vnodes,
                                   cudaGraphConditionalHandle loop, int in_graph, double* scratch);
__global__ void __launch_bounds__(256, 4) window_stats_scan_kernel(ScanState* S,
                                                                const int2* __restrict__ leaves, int nleaves,
                                                                int chunk, const PwVnode* __restrict__ vnodes,
                                                                cudaGraphConditionalHandle loop, int in_graph) {
  extern __shared__ __align__(128) uint8_t st_ring[];
  // the window, read once up front (one round trip; the deciding CTA rewrites the state only
  // after every CTA of the grid has checked in)
  const int L = S->L, approx = S->approx, exact = S->exact, s = S->s, n_acc = S->n_acc, init = S->init;
  const long N = S->N;
  const double wm = S->wm, wg = S->wg;
  const uint16_t* codes = S->codes;
  double *ckS = S->ckS, *ckQ = S->ckQ, *ckS2 = S->ckS2, *ckQ2 = S->ckQ2;
  if (L <= 0) return;
  const bool by_leaf = (long)blockIdx.x * (blockDim.x / kLeafLanes) < nleaves;
  bool last;
  if (!approx || exact) {
    if (by_leaf)
      window_stats_body<false>(codes, N, leaves, nleaves, s, n_acc, L, 1, init, wm, wg, ckS, ckQ, ckS2, ckQ2,
                               S->leafsum, nullptr, nullptr);
    last = scan_window_arrive(S);
  } else if (chunk <= 0) {  // (SCPL_SCAN_LEAF_SCREEN=1: the leaf-layout screening body)
    if (by_leaf)
      window_stats_body<true>(codes, N, leaves, nleaves, s, n_acc, L, 1, init, wm, wg, ckS, ckQ, ckS2, ckQ2,
                              nullptr, S->asum, S->bsum);
    last = scan_window_arrive(S);
  } else if (screen_noclamp(wm, wg)) {
    last = window_screen_body<false>(codes, N, chunk, s, n_acc, L, init, wm, wg, ckS, ckQ, ckS2, ckQ2, S->asum,
                                     S->bsum, S, loop, in_graph);
  } else {
    last = window_screen_body<true>(codes, N, chunk, s, n_acc, L, init, wm, wg, ckS, ckQ, ckS2, ckQ2, S->asum,
                                    S->bsum, S, loop, in_graph);
  }
  if (last) scan_window_finish(S, nleaves, vnodes, loop, in_graph, reinterpret_cast<double*>(st_ring));
}

// grid of a scan window launch and the screened body's chunk (0: leaf-layout screening)
static int scan_grid(long N, int nleaves, int& chunk) {
  static const bool leaf_screen = getenv("SCPL_SCAN_LEAF_SCREEN") != nullptr;  // (experiments)
  int dev = 0, sms = 0;
  SCPL_CUDA(cudaGetDevice(&dev));
  SCPL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  chunk = leaf_screen ? 0 : screen_chunk(N, sms);
  const int by_leaves = cdiv((long)nleaves * kLeafLanes, 256);
  return chunk > 0 ? std::max(by_leaves, (int)cdiv(N, (long)chunk)) : by_leaves;
}

static void stats_smem_attr() {
  smem_optin(reinterpret_cast<const void*>(window_stats_kernel));  // (once per device)
  smem_optin(reinterpret_cast<const void*>(window_stats_scan_kernel));
}

// ------------------------------------------------------------ device: tree fold
// The leaf sums are folded along a virtual complete tree of depth kPwDepth over numpy's
// recursion (build_pairwise_plan): node v's value is the pairwise sum of its subtree, an
// empty node adds +0.0 (exact for the non-negative sums here).  kPwFoldCtas CTAs per
// candidate each fold one complete subtree of depth kPwDepth - kPwTop to a partial; the
// root folds the kPwFoldCtas partials (again a complete tree, so the bracketing is numpy's).
__device__ double pw_eval(long n, const double* __restrict__ ls, int& li) {
  if (n <= 128) return __ldcg(&ls[li++]);  // (L2: the fused tail reads other CTAs' leaf sums)
  long h = n / 2;
  h -= h % 8;
  double a = pw_eval(h, ls, li);
  double b = pw_eval(n - h, ls, li);
  return __dadd_rn(a, b);
}

constexpr int kPwSub = (1 << kPwDepth) / kPwFoldCtas;  // vnodes per CTA

// one subtree (fold CTA index b) of candidate sums ls folded in v[kPwSub] (shared); returns the
// subtree's sum in v[0] (valid for thread 0 after the last barrier)
__device__ __forceinline__ void fold_subtree(const double* ls, const PwVnode* __restrict__ vnodes, int b, double* v) {
  const int v0 = b * kPwSub;
  for (int t = threadIdx.x; t < kPwSub; t += blockDim.x) {
    PwVnode vn = vnodes[v0 + t];
    double x = 0.0;
    if (vn.n > 0) {
      int li = vn.first_leaf;
      x = pw_eval(vn.n, ls, li);
    }
    v[t] = x;
  }
  __syncthreads();
  // fold in place at the left child's slot: v[2ts] = v[2ts] + v[2ts+s]
  for (int s = 1; s < kPwSub; s <<= 1) {
    for (int t = threadIdx.x; t < (kPwSub >> 1) / s; t += blockDim.x)
      v[2 * t * s] = __dadd_rn(v[2 * t * s], v[2 * t * s + s]);
    __syncthreads();
  }
}

// grid (kPwFoldCtas, L)
__global__ void __launch_bounds__(256) fold_partial_kernel(const double* leafsum, int nleaves,
                                                           const PwVnode* __restrict__ vnodes, double* partial) {
  __shared__ double v[kPwSub];
  const int c = blockIdx.y;
  fold_subtree(leafsum + (size_t)c * nleaves, vnodes, blockIdx.x, v);
  if (threadIdx.x == 0) partial[(size_t)c * kPwFoldCtas + blockIdx.x] = v[0];
}

__device__ __forceinline__ double fold_root(const double* partial, int c, long N) {
  double v[kPwFoldCtas];
#pragma unroll
  for (int k = 0; k < kPwFoldCtas; ++k) v[k] = partial[(size_t)c * kPwFoldCtas + k];
#pragma unroll
  for (int s = 1; s < kPwFoldCtas; s <<= 1)
#pragma unroll
    for (int k = 0; k < kPwFoldCtas; k += 2 * s) v[k] = __dadd_rn(v[k], v[k + s]);
  return __ddiv_rn(__dadd_rn(0.0, v[0]), (double)N);
}

__global__ void fold_root_kernel(const double* __restrict__ partial, int L, long N, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < L) out[c] = fold_root(partial, c, N);
}

void launch_pairwise_fold(const double* leafsum, int nleaves, const PwVnode* vnodes, long N, int L,
                          double* partial, double* out, cudaStream_t st) {
  fold_partial_kernel<<<dim3(kPwFoldCtas, L), 256, 0, st>>>(leafsum, nleaves, vnodes, partial);
  SCPL_CHECK_LAUNCH();
  fold_root_kernel<<<cdiv(L, 64), 64, 0, st>>>(partial, L, N, out);
  SCPL_CHECK_LAUNCH();
}

void launch_window_stats(const uint16_t* codes, long N, const int2* leaves, int nleaves, int s, int n_acc,
                         int L, int first_pure, int init, double wm, double wg, double* ckS, double* ckQ,
                         double* leafsum, const PwVnode* vnodes, double* partial, double* asde_out,
                         cudaStream_t st) {
  int threads = 256;
  int blocks = cdiv((long)nleaves * kLeafLanes, threads);
  stats_smem_attr();
  window_stats_kernel<<<blocks, threads, kStatSmem, st>>>(codes, N, leaves, nleaves, s, n_acc, L, first_pure, init,
                                                          wm, wg, ckS, ckQ, leafsum);
  SCPL_CHECK_LAUNCH();
  launch_pairwise_fold(leafsum, nleaves, vnodes, N, L, partial, asde_out, st);
}

// ------------------------------------------------------------ device-side buffer scan
// SpatioTemporalBuffer.push/flush (buffering.py:93-138) as a state machine in device
// memory: plan the next window of candidates, or consume the latest ASDEs and decide.
// Candidate n is accepted while asde(n) <= threshold(n) (buffering.py:119); a breach
// closes the run before the offending frame, which starts the next run.  A window never
// reaches past `avail` (frames whose codes are on the device), so the host can feed the
// clip in chunks; the ASDE of a length is independent of how the lengths were chunked.
__device__ void scan_plan(ScanState* S) {
  while (!S->done) {
    const int remaining = S->T - (S->s + S->n_acc);
    if (remaining == 0) {  // end of clip: flush (pipeline.py:131-133)
      S->runs[2 * S->nruns] = S->s;
      S->runs[2 * S->nruns + 1] = S->n_acc;
      S->nruns++;
      S->done = 1;
      break;
    }
    if (S->n_acc >= S->max_len) {  // the next push would exceed the cap: flush
      S->runs[2 * S->nruns] = S->s;
      S->runs[2 * S->nruns + 1] = S->n_acc;
      S->nruns++;
      S->s += S->n_acc;
      S->n_acc = 1;
      S->init = 1;
      continue;
    }
    int L = min(S->spec, min(remaining, S->max_len - S->n_acc));
    // a run's first window stops where the previous run broke (runs tend to repeat their
    // length; an evaluated candidate past the breach is wasted work); the ASDE of a length
    // does not depend on how the lengths are split into windows
    if (S->n_acc == 1 && S->nruns > 0) L = min(L, max(2, S->runs[2 * S->nruns - 1]));
    L = min(L, S->avail - (S->s + S->n_acc));
    if (L <= 0) break;  // wait for more frames
    S->L = L;
    for (int c = 0; c < L; ++c) S->asum[c] = S->bsum[c] = 0.0;
    return;
  }
  S->L = 0;
}

// Screened window, candidate c: the reference accepts it iff asde(c) <= phi; with
// |asde~ - asde| <= marg (kScanDelta's per-pixel bounds, the relative f32 roundings of std~
// with a 4x margin, and the reference's own fp64 rounding) the test is settled when
// asde~ + marg < phi (0: accepted) or asde~ - marg > phi (1: breach); otherwise 2 (the window
// is re-run exactly).  asum / bsum are other CTAs' atomics, read past L1.
__device__ __forceinline__ int scan_screen_status(const ScanState* S, int c) {
  const double invN = 1.0 / (double)S->N;
  const double a = *(const volatile double*)&S->asum[c] * invN;
  const double marg = 2.0 * *(const volatile double*)&S->bsum[c] * invN + 8e-6 * a + 1e-9;
  const double phi = S->phi[S->n_acc + c + 1];
  return a + marg < phi ? 0 : (a - marg > phi ? 1 : 2);
}

// Thread 0 of the deciding CTA: consume the window's results (asde[c]: exact ASDEs of an exact
// window), decide, plan the next window and set the loop condition.
__device__ void scan_decide_plan(ScanState* S, const double* asde, const int* status,
                                 cudaGraphConditionalHandle loop, int decide, int in_graph) {
  const int L = S->L;
  const bool exact = !S->approx || S->exact;
  if (decide && L > 0) {
    int breach = -1;
    if (exact) {
      for (int c = 0; c < L; ++c) {
        if (!(asde[c] <= S->phi[S->n_acc + c + 1])) {
          breach = c;
          break;
        }
      }
    } else {
      // screened window: status[c] (scan_screen_status, evaluated by the CTA's threads in
      // parallel) is 0 = accepted, 1 = breach, 2 = the bound cannot settle the threshold test
      bool unsure = S->force_fallback != 0;
      for (int c = 0; c < L && !unsure; ++c) {
        if (status[c] == 0) continue;
        if (status[c] == 1) {
          breach = c;
          break;
        }
        unsure = true;
      }
      if (unsure) {  // same window again, exact kernel (the checkpoint read is untouched)
        S->exact = 1;
        S->fallbacks++;
        S->steps++;
        if (in_graph) cudaGraphSetConditional(loop, 1u);
        return;
      }
    }
    S->exact = 0;
    if (breach < 0) {  // every candidate accepted: the written checkpoint becomes current
      S->n_acc += L;
      S->init = 0;
      double* t = S->ckS;
      S->ckS = S->ckS2;
      S->ckS2 = t;
      t = S->ckQ;
      S->ckQ = S->ckQ2;
      S->ckQ2 = t;
    } else {
      S->runs[2 * S->nruns] = S->s;
      S->runs[2 * S->nruns + 1] = S->n_acc + breach;
      S->nruns++;
      S->s += S->n_acc + breach;
      S->n_acc = 1;
      S->init = 1;
    }
    S->L = 0;
    S->steps++;
  }
  scan_plan(S);
  if (in_graph) cudaGraphSetConditional(loop, S->L > 0 ? 1u : 0u);
}

// The head of a scan launch: plan the first window of the chunk.
__global__ void scan_step_kernel(ScanState* S, cudaGraphConditionalHandle loop, int in_graph) {
  if (threadIdx.x == 0) scan_decide_plan(S, nullptr, nullptr, loop, 0, in_graph);
}

// The deciding CTA of a window launch (scan_window_arrive): folds an exact window's leaf sums
// (one CTA: exact windows are the rare fallback), decides and plans -- the loop body is ONE
// kernel, no fold / step launches per window.
__device__ void scan_window_finish(ScanState* S, int nleaves, const PwVnode* __restrict__ vnodes,
                                   cudaGraphConditionalHandle loop, int in_graph, double* scratch) {
  __shared__ double asde[kScanMaxL];
  __shared__ int status[kScanMaxL];
  __syncthreads();  // (the ring is free: scratch)
  __threadfence();
  const int L = S->L;
  if (!S->approx || S->exact) {
    for (int c = 0; c < L; ++c)
      for (int b = 0; b < kPwFoldCtas; ++b) {
        fold_subtree(S->leafsum + (size_t)c * nleaves, vnodes, b, scratch);
        if (threadIdx.x == 0) S->partial[(size_t)c * kPwFoldCtas + b] = scratch[0];
        __syncthreads();
      }
    for (int c = threadIdx.x; c < L; c += blockDim.x) asde[c] = fold_root(S->partial, c, S->N);
  } else {  // one thread per candidate: the loads of the sums and thresholds in parallel
    for (int c = threadIdx.x; c < L; c += blockDim.x) status[c] = scan_screen_status(S, c);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    S->ticket = 0;
    scan_decide_plan(S, asde, status, loop, 1, in_graph);
  }
}

// The same for a screened window decided by ONE warp (the last warp of the last CTA to finish:
// window_screen_body has no block barriers): a lane per candidate evaluates the threshold tests.
__device__ void scan_screen_finish_warp(ScanState* S, cudaGraphConditionalHandle loop, int in_graph) {
  __shared__ int status[kScanMaxL];
  __threadfence();
  const int L = S->L;
  for (int c = threadIdx.x & 31; c < L; c += 32) status[c] = scan_screen_status(S, c);
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    S->ticket = 0;
    scan_decide_plan(S, nullptr, status, loop, 1, in_graph);
  }
}

__global__ void scan_reset_kernel(ScanState* S, ScanState init) { *S = init; }
__global__ void scan_avail_kernel(ScanState* S, int avail) { S->avail = avail; }

// graph: step(plan) -> while (L > 0) { window statistics; its last CTA decides and plans }
cudaGraphExec_t build_scan_graph(ScanState* S, long N, const int2* leaves, int nleaves, const PwVnode* vnodes,
                                 int spec, int prio) {
  SCPL_ARG(spec >= 1 && spec <= 64, "spec_len must be in 1..64");
  cudaGraph_t g;
  SCPL_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  SCPL_CUDA(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
  cudaStream_t cs = capture_stream(prio);
  // head: plan
  SCPL_CUDA(cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  scan_step_kernel<<<1, 32, 0, cs>>>(S, h, 1);
  SCPL_CUDA(cudaGetLastError());  // captured, counted per graph launch
  SCPL_CUDA(cudaStreamEndCapture(cs, &g));
  cudaGraphNode_t head;
  size_t nn = 1;
  SCPL_CUDA(cudaGraphGetNodes(g, &head, &nn));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cond;
  SCPL_CUDA(cudaGraphAddNode(&cond, g, &head, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  SCPL_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  stats_smem_attr();
  int chunk = 0;
  const int grid = scan_grid(N, nleaves, chunk);
  const size_t smem = std::max(kStatSmem + spec * kStatRed, kScrSmem);
  // SCPL_SCAN_UNROLL=n (experiments): n windows per execution of the loop body (a window kernel
  // that finds nothing planned, L == 0, returns at once).  Unlike the carve loop's unrolling this
  // gains nothing (the kernels that find no window cost what the loop's re-evaluation saves): 1
  static const int unroll = getenv("SCPL_SCAN_UNROLL") ? std::min(8, std::max(1, atoi(getenv("SCPL_SCAN_UNROLL")))) : 1;
  for (int u = 0; u < unroll; ++u) {
    window_stats_scan_kernel<<<grid, 256, smem, cs>>>(S, leaves, nleaves, chunk, vnodes, h, 1);
    SCPL_CUDA(cudaGetLastError());  // captured, counted per graph launch
  }
  SCPL_CUDA(cudaStreamEndCapture(cs, &body));
  graph_set_priority(g, prio);
  graph_set_priority(body, prio);
  cudaGraphExec_t ex;
  SCPL_CUDA(cudaGraphInstantiate(&ex, g, 0));
  cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  return ex;
}

// Host-driven equivalent of one scan graph launch (SCPL_HOST_LOOPS: profiling, where the
// conditional graph would hide the kernels from the profiler): the host reads L back.
void run_scan_host(ScanState* S, long N, const int2* leaves, int nleaves, const PwVnode* vnodes, int spec, int* h_L,
                   cudaStream_t st) {
  scan_step_kernel<<<1, 32, 0, st>>>(S, 0, 0);
  SCPL_CHECK_LAUNCH();
  stats_smem_attr();
  int chunk = 0;
  const int grid = scan_grid(N, nleaves, chunk);
  const size_t smem = std::max(kStatSmem + spec * kStatRed, kScrSmem);
  while (true) {
    SCPL_CUDA(cudaMemcpyAsync(h_L, reinterpret_cast<uint8_t*>(S) + offsetof(ScanState, L), sizeof(int),
                              cudaMemcpyDeviceToHost, st));
    SCPL_CUDA(cudaStreamSynchronize(st));
    if (*h_L <= 0) break;
    window_stats_scan_kernel<<<grid, 256, smem, st>>>(S, leaves, nleaves, chunk, vnodes, 0, 0);
    SCPL_CHECK_LAUNCH();
  }
}

void launch_scan_reset(ScanState* S, const ScanState& init, cudaStream_t st) {
  scan_reset_kernel<<<1, 1, 0, st>>>(S, init);
  SCPL_CHECK_LAUNCH();
}
void launch_scan_avail(ScanState* S, int avail, cudaStream_t st) {
  scan_avail_kernel<<<1, 1, 0, st>>>(S, avail);
  SCPL_CHECK_LAUNCH();
}

// ------------------------------------------------------------ K3: uniform map
// FixedRun.uniform_energy (buffering.py:69-71): sequential per-pixel sum over the run's
// frames, divided by T (equal to np.stack(maps).mean(axis=0) bit for bit).  Written in
// the carve orientation (transposed for a height phase) with a 32x32 smem tile.
__global__ void uniform_kernel(const uint16_t* __restrict__ codes, int H, int W, int s, int n, int first_pure,
                               double wm, double wg, int transposed, double* __restrict__ out, int pitch) {
  __shared__ double A[256], B[256];
  __shared__ double tile[32][33];
  for (int k = threadIdx.y * 32 + threadIdx.x; k < 256; k += 256) {
    A[k] = __dmul_rn(wm, (double)k);
    B[k] = __dmul_rn(wg, (double)k);
  }
  __syncthreads();
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  const long N = (long)H * W;
  const double dn = (double)n;
  for (int r = threadIdx.y; r < 32; r += 8) {
    int i = i0 + r, j = j0 + threadIdx.x;
    double acc = 0.0;
    if (i < H && j < W) {
      long p = (long)i * W + j;
      acc = energy_of(codes[(size_t)s * N + p], first_pure && s == 0, A, B);
      for (int t = s + 1; t < s + n; ++t) acc = __dadd_rn(acc, energy_of(codes[(size_t)t * N + p], false, A, B));
      acc = __ddiv_rn(acc, dn);
      if (!transposed) out[(long)i * pitch + j] = acc;
    }
    tile[r][threadIdx.x] = acc;
  }
  if (!transposed) return;
  __syncthreads();
  // out is (W, H): out[j][i]
  for (int r = threadIdx.y; r < 32; r += 8) {
    int j = j0 + r, i = i0 + threadIdx.x;
    if (i < H && j < W) out[(long)j * pitch + i] = tile[threadIdx.x][r];
  }
}

// Width phases (the common case): each thread owns 8 consecutive pixels of a row, reads their
// codes with one 16-byte load per frame (four frames in flight), keeps 8 sequential fp64 sums
// (the reference's per-pixel order, buffering.py:71) and writes 8 means with 16-byte stores.
// e is recomputed on the fp64 pipe (energy.py:86-87) instead of table loads.
constexpr int kUniPx = 8;
__device__ __forceinline__ double energy_fp64(uint32_t code, bool pure, double wm, double wg) {
  const uint32_t g = code & 255u;
  if (pure) return (double)g;
  return fmin(__dadd_rn(__dmul_rn(wm, (double)(code >> 8)), __dmul_rn(wg, (double)g)), 255.0);
}
// CLAMP = false (wm, wg non-negative with fl(fl(255 wm) + fl(255 wg)) <= 255, uniform_noclamp):
// min(e, 255) is a no-op and every e is >= +0.0, so the sum may start from +0.0 (0 + e == e bit
// for bit); bytes become doubles on the fp64 pipe (u8_f64) -- 8 instructions per pixel and
// frame instead of 16.  A pure-gradient frame (the clip's first) is wm = 0, wg = 1.
template <bool CLAMP>
__global__ void __launch_bounds__(256, 4) uniform_vec_kernel(const uint16_t* __restrict__ codes, int H, int W, int s,
                                                          int n, int first_pure, double wm0, double wg0,
                                                          double* __restrict__ out, int pitch) {
  const long N = (long)H * W;
  const long q = blockIdx.x * (long)blockDim.x + threadIdx.x;  // 8-pixel group
  if (q * kUniPx >= N) return;
  const long p = q * kUniPx;
  const uint4* src = reinterpret_cast<const uint4*>(codes + (size_t)s * N + p);
  const size_t fstride = (size_t)N / kUniPx;  // uint4 per frame
  double acc[kUniPx];
#pragma unroll
  for (int k = 0; k < kUniPx; ++k) acc[k] = 0.0;
  // frames in chunks of 4 with every load of a chunk in flight (a short run is one or two round
  // trips), then the sequential fp64 sum in frame order (buffering.py:69-71)
  const bool pure0 = first_pure && s == 0;
  for (int t0 = 0; t0 < n; t0 += 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t0 + u < n) v[u] = __ldcs(src + (size_t)(t0 + u) * fstride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (t0 + u >= n) break;
      const uint32_t w4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
      const bool pure = pure0 && t0 + u == 0;
      if (CLAMP) {
#pragma unroll
        for (int k = 0; k < kUniPx; ++k) {
          const double e = energy_fp64((w4[k >> 1] >> (16 * (k & 1))) & 0xffffu, pure, wm0, wg0);
          acc[k] = t0 + u == 0 ? e : __dadd_rn(acc[k], e);
        }
      } else {
        const double wm = pure ? 0.0 : wm0, wg = pure ? 1.0 : wg0;
#pragma unroll
        for (int k = 0; k < kUniPx; k += 2) {
          const uint32_t w = w4[k >> 1];
          const double e0 = __dadd_rn(__dmul_rn(wm, u8_f64(__byte_perm(w, 0u, 0x4441))), __dmul_rn(wg, u8_f64(w & 255u)));
          const double e1 = __dadd_rn(__dmul_rn(wm, u8_f64(w >> 24)), __dmul_rn(wg, u8_f64(__byte_perm(w, 0u, 0x4442))));
          acc[k] = __dadd_rn(acc[k], e0);
          acc[k + 1] = __dadd_rn(acc[k + 1], e1);
        }
      }
    }
  }
  const double dn = (double)n;
  const int i = (int)(p / W), j = (int)(p - (long)i * W);
  double2* o = reinterpret_cast<double2*>(out + (long)i * pitch + j);
#pragma unroll
  for (int k = 0; k < kUniPx; k += 2) o[k / 2] = make_double2(__ddiv_rn(acc[k], dn), __ddiv_rn(acc[k + 1], dn));
}

// wm, wg with a clear sign bit and fl(fl(255 wm) + fl(255 wg)) <= 255 (separate roundings, as the
// device computes e): rounding is monotone, so no e exceeds 255 and none is -0.0
static bool uniform_noclamp(double wm, double wg) {
  if (std::signbit(wm) || std::signbit(wg) || !(wm == wm) || !(wg == wg)) return false;
  volatile double a = wm * 255.0, b = wg * 255.0;
  volatile double c = a + b;
  return c <= 255.0;
}

void launch_uniform(const uint16_t* codes, int H, int W, int s, int n, int first_pure, double wm, double wg,
                    int transposed, double* out, cudaStream_t st, int pitch) {
  if (pitch <= 0) pitch = transposed ? H : W;
  const long N = (long)H * W;
  if (!transposed && W % kUniPx == 0 && pitch % 2 == 0 && (reinterpret_cast<uintptr_t>(codes) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    if (uniform_noclamp(wm, wg))
      uniform_vec_kernel<false><<<cdiv(N / kUniPx, 256), 256, 0, st>>>(codes, H, W, s, n, first_pure, wm, wg, out, pitch);
    else
      uniform_vec_kernel<true><<<cdiv(N / kUniPx, 256), 256, 0, st>>>(codes, H, W, s, n, first_pure, wm, wg, out, pitch);
    SCPL_CHECK_LAUNCH();
    return;
  }
  dim3 grid(cdiv(W, 32), cdiv(H, 32));
  uniform_kernel<<<grid, dim3(32, 8), 0, st>>>(codes, H, W, s, n, first_pure, wm, wg, transposed, out, pitch);
  SCPL_CHECK_LAUNCH();
}

}  // namespace scpl
