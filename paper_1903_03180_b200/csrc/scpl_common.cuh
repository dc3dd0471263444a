// Shared helpers for the sm_100a SCPL kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include <atomic>
#include <string>

namespace scpl {

// ---------------------------------------------------------------- error plumbing
void set_error(const std::string& msg);
extern std::atomic<long> g_launches;  // kernels launched by this library (bench evidence)
struct Error {
  int code;  // 1 = invalid argument (ValueError), 2 = CUDA/runtime (RuntimeError)
  std::string msg;
};

#define SCPL_CUDA(x)                                                                        \
  do {                                                                                      \
    cudaError_t _e = (x);                                                                   \
    if (_e != cudaSuccess)                                                                  \
      throw ::scpl::Error{2, std::string(#x) + ": " + cudaGetErrorString(_e)};              \
  } while (0)
#define SCPL_CHECK_LAUNCH()                                  \
  do {                                                       \
    ::scpl::g_launches.fetch_add(1, std::memory_order_relaxed); \
    SCPL_CUDA(cudaGetLastError());                           \
  } while (0)
#define SCPL_ARG(cond, msg)                                      \
  do {                                                           \
    if (!(cond)) throw ::scpl::Error{1, std::string(msg)};       \
  } while (0)

static inline int cdiv(long a, long b) { return (int)((a + b - 1) / b); }

// Device-side invariant checks of the checked build (libscpl_checked.so, -DSCPL_CHECKS; loaded
// with SCPL_CHECKED=1): a violated invariant prints and traps, which fails the call with a
// CUDA error.  Compiled out of the product build.
#ifdef SCPL_CHECKS
#define SCPL_DCHECK(cond, what)                                                                   \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("SCPL_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                  \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define SCPL_DCHECK(cond, what) ((void)0)
#endif

// Opt a kernel into the full 227 KB of dynamic shared memory, once per process: setting a
// function attribute while that kernel runs on another stream can serialise the host.
void smem_optin(const void* kernel);
// true the first time (current device, key) is seen (per-device one-time attribute setup)
bool once_per_device(const void* key);
// Kernel nodes of a captured graph run at the priority recorded in the node, not at the
// priority of the stream the graph is launched into: give every kernel node of g this one
// (SCPL_GRAPH_PRIO=1; see scpl_api.cu).
void graph_set_priority(cudaGraph_t g, int prio);
// the capture stream for a graph whose kernels should run at prio (only with SCPL_GRAPH_PRIO=1)
cudaStream_t capture_stream(int prio);

// ---------------------------------------------------------------- exact arithmetic
// energy.py:35 -- luma = rint(fma(b,.114, fma(r,.299, g*.587))).  Outside the exact
// half cases (299r+587g+114b == 500 mod 1000) the rounded value is the nearest integer
// of X/1000, so integer arithmetic decides; the 16,782 half cases take the fp64 path.
__device__ __forceinline__ uint32_t luma_of(uint32_t r, uint32_t g, uint32_t b) {
  uint32_t x = 299u * r + 587u * g + 114u * b;
  uint32_t q = x / 1000u;
  uint32_t rem = x - q * 1000u;
  if (rem != 500u) return q + (rem > 500u ? 1u : 0u);
  double acc = __dmul_rn((double)g, 0.587);
  acc = __fma_rn((double)r, 0.299, acc);
  acc = __fma_rn((double)b, 0.114, acc);
  return (uint32_t)__double2uint_rn(acc);  // round-half-even == np.rint
}

// Correctly rounded x / n for a small positive integer n given rn = RN(1/n):
// Markstein correction q' = RN(q + RN(x - n*q) * rn) (exact remainder by FMA).
// Checked against IEEE division on 1.28e9 samples for every n in 1..64
// (DESIGN.md "exactness"); the parity tests re-check it end to end.
__device__ __forceinline__ double div_small(double x, double n, double rn) {
  double q = __dmul_rn(x, rn);
  double r = __fma_rn(-q, n, x);
  return __fma_rn(r, rn, q);
}

// motion energy of one pixel from its code (|dL| << 8 | grad), energy.py:79-87.
// A[d] = fl(wm*d), B[g] = fl(wg*g) precomputed; pure gradient on the clip's first frame.
__device__ __forceinline__ double energy_of(uint32_t code, bool pure, const double* A, const double* B) {
  uint32_t g = code & 255u;
  if (pure) return (double)g;
  return fmin(__dadd_rn(A[code >> 8], B[g]), 255.0);  // e is never NaN: fmin == the clamp
}

// ---------------------------------------------------------------- async copy helpers (TMA bulk)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// mbar_wait with a suspend-time hint: the waiting warp sleeps until the phase completes (or
// the hint expires) instead of spinning on try_wait, leaving the SM sub-partition's issue
// slots to the warps that do the work (the carve's producer warps share them with DP warps)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

}  // namespace scpl
