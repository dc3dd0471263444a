// C-ABI (include/scpl.h) and the native orchestrator of the buffered SCPL path.
//
// retarget_video (pipeline.py:92-137) runs here, on the host side of the .so:
//   1. energy codes for every frame                       (K1, one streaming pass)
//   2. the spatio-temporal buffer scan                    (K2 chunks + exact host decision
//      against the caller's phi table, buffering.py:93-138)
//   3. per carved axis (width first unless height_first, pipeline.py:192-193):
//        per run: representative luma plane + index map (+ uniform map on the first
//        carved axis, K3), then the carve loop batched across all runs (K4-K7),
//        then the replay gather of every frame of the run (K8)
//   4. RunMetrics.dp_passes = total DP passes.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <list>
#include <array>
#include <deque>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/scpl.h"
#include "scpl_common.cuh"
#include "scpl_kernels.h"

using namespace scpl;

namespace scpl {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
void smem_optin(const void* kernel) {
  static std::mutex mu;
  static std::set<const void*> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(kernel)) return;
  int dev = 0, optin = 0;
  SCPL_CUDA(cudaGetDevice(&dev));
  SCPL_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  SCPL_CUDA(cudaFuncGetAttributes(&fa, kernel));
  SCPL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - (int)fa.sharedSizeBytes));
  done.insert(kernel);
}
std::atomic<long> g_launches{0};
}  // namespace scpl

struct PwPlan {
  int2* leaves = nullptr;
  PwVnode* vnodes = nullptr;
  int nleaves = 0;
};

struct scpl_ctx {
  int device = 0;
  int num_sms = 148;
  int clock_khz = 0;  // base SM clock (queried once: the query costs milliseconds of host time)
  int prio_lo = 0, prio_hi = 0;
  bool prio_known = false;
  cudaStream_t s_h2d = nullptr, s_codes = nullptr, s_d2h = nullptr, s_scan = nullptr;  // pipeline streams
  double* h_asde = nullptr;  // pinned
  int h_asde_cap = 0;
  std::map<long, PwPlan> plans;
  // device-side buffer scan
  ScanState* scan = nullptr;                       // device
  double* phi_d = nullptr;
  std::vector<double> phi_h;                       // contents of phi_d
  std::map<std::pair<long, int>, cudaGraphExec_t> scan_graphs;  // (N, spec)
  uint8_t* pin = nullptr;  // pinned scratch (pinned_scratch)
  size_t pin_cap = 0;
  std::vector<cudaStream_t> s_carve;  // concurrent run groups
  // Instantiated carve loops kept for reuse (instantiating / destroying a conditional graph
  // costs host time on every group): free entries by shape, each with its own run-state
  // memory that the graph's kernels point at.
  struct CarveLoop {
    cudaGraphExec_t ex = nullptr;
    void* mem = nullptr;  // nruns CarveRuns + the iteration counter
  };
  std::multimap<std::array<int, 8>, CarveLoop> loop_pool;
  std::deque<std::array<int, 8>> loop_order;  // free entries, oldest first (eviction)
  std::vector<cudaEvent_t> ev_pool[2];         // free events: [0] no timing, [1] timing
};

namespace {

// stream-ordered device buffer
struct DBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DBuf() = default;
  DBuf(size_t bytes, cudaStream_t s) : st(s) {
    if (bytes) SCPL_CUDA(cudaMallocAsync(&p, bytes, s));
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), st(o.st) { o.p = nullptr; }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    p = o.p;
    st = o.st;
    o.p = nullptr;
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

template <class F>
int guarded(scpl_ctx* ctx, F&& f) {
  try {
    if (ctx) SCPL_CUDA(cudaSetDevice(ctx->device));
    f();
    return 0;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return 2;
  }
}

const PwPlan& plan_for(scpl_ctx* ctx, long N) {
  auto it = ctx->plans.find(N);
  if (it != ctx->plans.end()) return it->second;
  std::vector<int2> leaves;
  std::vector<PwVnode> vnodes;
  build_pairwise_plan(N, leaves, vnodes);
  PwPlan p;
  p.nleaves = (int)leaves.size();
  SCPL_CUDA(cudaMalloc(&p.leaves, sizeof(int2) * leaves.size()));
  SCPL_CUDA(cudaMalloc(&p.vnodes, sizeof(PwVnode) * vnodes.size()));
  SCPL_CUDA(cudaMemcpy(p.leaves, leaves.data(), sizeof(int2) * leaves.size(), cudaMemcpyHostToDevice));
  SCPL_CUDA(cudaMemcpy(p.vnodes, vnodes.data(), sizeof(PwVnode) * vnodes.size(), cudaMemcpyHostToDevice));
  return ctx->plans.emplace(N, p).first->second;
}

double* pinned_asde(scpl_ctx* ctx, int n) {
  if (ctx->h_asde_cap < n) {
    if (ctx->h_asde) cudaFreeHost(ctx->h_asde);
    ctx->h_asde = nullptr;
    SCPL_CUDA(cudaMallocHost(&ctx->h_asde, sizeof(double) * n));
    ctx->h_asde_cap = n;
  }
  return ctx->h_asde;
}

// SCPL_HOST_LOOPS=1: drive the scan and carve loops from the host instead of conditional
// graphs (identical results; lets a profiler see every kernel)
bool host_loops() { return getenv("SCPL_HOST_LOOPS") != nullptr; }

// grow-only pinned scratch (one user at a time: the current C-ABI call)
uint8_t* pinned_scratch(scpl_ctx* ctx, size_t bytes) {
  if (ctx->pin_cap < bytes) {
    if (ctx->pin) cudaFreeHost(ctx->pin);
    ctx->pin = nullptr;
    ctx->pin_cap = 0;
    SCPL_CUDA(cudaMallocHost(&ctx->pin, bytes));
    ctx->pin_cap = bytes;
  }
  return ctx->pin;
}

// ------------------------------------------------------------------ buffer scan
// SpatioTemporalBuffer.push/flush over the whole clip (buffering.py:93-138), decided on
// the device: each scan_chunk launch runs the scan as far as the frames whose codes are on
// the device allow (a conditional while node around stats -> fold -> decide), then copies
// the run count (and the append-only run list) to pinned memory, so the host can hand
// closed runs to the carve while the scan goes on -- it never waits on an ASDE.
struct ScanStream {
  DBuf ck, leafsum, partial, runs_d;
  cudaGraphExec_t graph = nullptr;
  const PwPlan* plan = nullptr;
  int spec = 8;
  int* h_L = nullptr;  // pinned (host-driven loops)
  int T = 0;
  int* h_n = nullptr;     // pinned: run count after each chunk
  int* h_runs = nullptr;  // pinned: (start, len) pairs, 2T ints
  ScanState* h_state = nullptr;
};

void scan_start(scpl_ctx* ctx, ScanStream& S, const uint16_t* codes, int T, int H, int W,
                const scpl_video_params& P, cudaStream_t st) {
  const long N = (long)H * W;
  const PwPlan& plan = plan_for(ctx, N);
  const int spec = P.spec_len > 0 ? P.spec_len : 8;
  SCPL_ARG(spec <= 64, "spec_len must be <= 64");
  if (!ctx->scan) SCPL_CUDA(cudaMalloc(&ctx->scan, sizeof(ScanState)));
  std::vector<double> phi(P.phi, P.phi + P.max_len + 1);
  if (phi != ctx->phi_h) {
    if (ctx->phi_h.size() < phi.size()) {
      if (ctx->phi_d) cudaFree(ctx->phi_d);
      ctx->phi_d = nullptr;
      SCPL_CUDA(cudaMalloc(&ctx->phi_d, sizeof(double) * phi.size()));
    }
    SCPL_CUDA(cudaMemcpy(ctx->phi_d, phi.data(), sizeof(double) * phi.size(), cudaMemcpyHostToDevice));
    ctx->phi_h = phi;
  }
  auto key = std::make_pair(N, spec);
  auto it = ctx->scan_graphs.find(key);
  if (it == ctx->scan_graphs.end())
    it = ctx->scan_graphs.emplace(key, build_scan_graph(ctx->scan, plan.leaves, plan.nleaves, plan.vnodes, spec))
             .first;
  S.graph = it->second;
  S.plan = &plan;
  S.spec = spec;
  S.T = T;
  S.ck = DBuf(sizeof(double) * 4 * N, st);
  S.leafsum = DBuf(sizeof(double) * spec * plan.nleaves, st);
  S.partial = DBuf(sizeof(double) * spec * kPwFoldCtas, st);
  S.runs_d = DBuf(sizeof(int) * 2 * T, st);
  ScanState init{};
  init.codes = codes;
  init.N = N;
  init.ckS = S.ck.as<double>();
  init.ckQ = S.ck.as<double>() + N;
  init.ckS2 = S.ck.as<double>() + 2 * N;
  init.ckQ2 = S.ck.as<double>() + 3 * N;
  // screened windows (exact re-run only when the bound cannot settle a threshold test);
  // SCPL_SCAN_EXACT=1 evaluates every window exactly, SCPL_SCAN_FORCE_FALLBACK=1 screens
  // every window and then re-runs it exactly (tests of both paths)
  init.approx = getenv("SCPL_SCAN_EXACT") ? 0 : 1;
  init.force_fallback = getenv("SCPL_SCAN_FORCE_FALLBACK") ? 1 : 0;
  init.leafsum = S.leafsum.as<double>();
  init.partial = S.partial.as<double>();
  init.phi = ctx->phi_d;
  init.runs = S.runs_d.as<int>();
  init.wm = P.w_motion;
  init.wg = P.w_grad;
  init.T = T;
  init.max_len = P.max_len;
  init.spec = spec;
  init.avail = 0;
  init.s = 0;
  init.n_acc = 1;
  init.init = 1;
  launch_scan_reset(ctx->scan, init, st);
}

void scan_chunk(scpl_ctx* ctx, ScanStream& S, int c, int avail, cudaStream_t st) {
  launch_scan_avail(ctx->scan, avail, st);
  if (host_loops())
    run_scan_host(ctx->scan, S.plan->leaves, S.plan->nleaves, S.plan->vnodes, S.spec, S.h_L, st);
  else
    SCPL_CUDA(cudaGraphLaunch(S.graph, st));
  // (SM copies into mapped pinned memory: no copy-engine queueing behind the clip's copies)
  kc6::launch_word_copy(&S.h_n[c], reinterpret_cast<uint8_t*>(ctx->scan) + offsetof(ScanState, nruns), sizeof(int), st);
  kc6::launch_word_copy(S.h_runs, S.runs_d.p, sizeof(int) * 2 * S.T, st);
}

void scan_end(scpl_ctx* ctx, ScanStream& S, cudaStream_t st) {
  kc6::launch_word_copy(S.h_state, ctx->scan, sizeof(ScanState), st);
}

// after the stream is done
void scan_finish(ScanStream& S, int chunks, scpl_video_result* result) {
  const ScanState& R = *S.h_state;
  if (!(R.done == 1 && R.nruns >= 1 && R.nruns <= S.T)) throw Error{2, "buffer scan did not finish"};
  g_launches.fetch_add((long)chunks + 3L * R.steps, std::memory_order_relaxed);
  result->scan_windows = R.steps;
  result->scan_fallbacks = R.fallbacks;
}

// ------------------------------------------------------------------ carve driver
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Planes for `nruns` carves of rows x cols (carve orientation) in one stream-ordered slab.
constexpr size_t kProfBytes = 8192;  // SCPL_PROF: 32 counters + (entry, exit) timestamps per pass

struct CarveSet {
  DBuf mem;
  std::vector<CarveRun> runs;
  int rows = 0, cols = 0, pitch = 0, target = 0, cl = 1;
  size_t planes_bytes = 0;  // luma + gradient planes of every run, at the start of mem
  int max_fr = 1;           // most frames carved together by one run (reaverage)
  bool reaverage = false;
  bool has_uniform = false;  // U holds a uniform map for the first pass (else the mean gradient)
  int kc = 6;                // DP window variant (scpl_carve2.cu: kc6 / kc4)
  long long prof[4] = {0, 0, 0, 0};
  scpl_ctx* ctx = nullptr;
  std::array<int, 8> loop_key{};
  scpl_ctx::CarveLoop loop;        // device-side iteration loop + run states (back to the pool
                                   // once the work is complete: sets outlive the final sync)
  CarveRun* h_runs = nullptr;      // pinned: run state after the carve (read once the stream is done)
  int* h_iters = nullptr;          // pinned: loop iterations executed
  CarveSet() = default;
  CarveSet(const CarveSet&) = delete;
  CarveSet& operator=(const CarveSet&) = delete;
  ~CarveSet() {
    if (!loop.mem) return;
    constexpr size_t kPoolCap = 64;
    ctx->loop_pool.emplace(loop_key, loop);
    ctx->loop_order.push_back(loop_key);
    while (ctx->loop_order.size() > kPoolCap) {
      auto it = ctx->loop_pool.find(ctx->loop_order.front());
      ctx->loop_order.pop_front();
      if (it == ctx->loop_pool.end()) continue;
      if (it->second.ex) cudaGraphExecDestroy(it->second.ex);
      cudaFree(it->second.mem);
      ctx->loop_pool.erase(it);
    }
  }
};

// DP window variants (scpl_carve2.cu compiled per width): kc6 = 128 owned columns per DP warp
// (4 CTAs for 1080p), kc4 = 64 (8 CTAs; 15 at 4K), kc3 = 32 (15 CTAs at 1080p); more than 8
// CTAs is a non-portable cluster size.  The DP row
// is latency-bound on one warp per SM sub-partition, so narrower windows shorten a pass (fewer
// instructions per row) at the price of SM-time.  A group takes the narrowest variant whose
// clusters, for the clip's runs extrapolated from this group's density (nruns over `span` of
// the T frames; a host clip's last group: just its own runs), would hold at most half the SMs --
// long runs (C4, C5, a lone last run) go narrow, C2's burst of 4-frame runs stays kc6.
// SCPL_CARVE_KC=3|4|6 forces one.
#define SCPL_CARVE_FN(kc, fn) ((kc) == 4 ? kc4::fn : (kc) == 3 ? kc3::fn : kc6::fn)
int carve_cluster(int kc, int nruns, int cols, int num_sms) {
  return SCPL_CARVE_FN(kc, carve_cluster_size)(nruns, cols, num_sms);
}
int carve_variant(int nruns, int cols, int span, int T, int num_sms, bool final_group) {
  const bool fit4 = cols <= 16 * 4 * 64, fit3 = cols <= 16 * 4 * 32;
  if (const char* e = getenv("SCPL_CARVE_KC")) {
    const int k = atoi(e);
    return k == 3 && fit3 ? 3 : (k == 3 || k == 4) && fit4 ? 4 : 6;
  }
  // the last group of a clip (scan finished) carves with nothing left to come
  const double est_runs = final_group ? (double)nruns : (double)nruns * T / std::max(1, span);
  auto fits = [&](int kc) { return est_runs * carve_cluster(kc, 1, cols, num_sms) <= 0.5 * num_sms; };
  if (fit3 && fits(3)) return 3;
  if (fit4 && fits(4)) return 4;
  return 6;
}

// nfr (nullable): frames carved together per run (reaverage_energy), else one each
void carve_alloc(CarveSet& S, int nruns, int rows, int cols, int target, int kmax, bool with_U, bool dbg,
                 int cl, cudaStream_t st, const int* nfr = nullptr, bool reaverage = false, int kc = 6) {
  SCPL_ARG(cols <= 4096, "frames wider than 4096 columns (in the carve orientation) are not supported");
  // int-pass keys hold the path cost (<= 255 per row) above 9 bits of direction data
  SCPL_ARG(rows <= 8192, "frames taller than 8192 rows (in the carve orientation) are not supported");
  const int pitch = (cols + 15) & ~15;
  const int nblk = std::max(1, (rows - 1 + kBlockRows - 1) / kBlockRows);
  const int rem_cap = std::max(1, cols - target);
  const int alive_pitch = ((cols + 31) / 32 + 3) & ~3;
  const size_t plane = (size_t)rows * pitch;
  // every run's luma and gradient plane first (compacted in place; one contiguous range for
  // the L2 persistence window), then each run's tables
  const size_t plane_al = align256(plane);
  long total_fr = 0;
  int max_fr = 1;
  for (int r = 0; r < nruns; ++r) {
    const int n = nfr ? std::max(1, nfr[r]) : 1;
    total_fr += n;
    max_fr = std::max(max_fr, n);
  }
  const size_t planes_bytes = (size_t)total_fr * 2 * plane_al;
  const bool uniform_given = with_U;
  if (reaverage) with_U = true;  // U = the mean gradient, recomputed every pass
  size_t per = align256(plane * 2) + align256((size_t)nblk * pitch * 8) +
               align256((size_t)nblk * pitch) + align256((size_t)pitch * 8) + align256((size_t)rows * rem_cap * 2) +
               align256((size_t)rows * alive_pitch * 4) + align256((size_t)nblk * pitch * 2) + align256(kProfBytes) +
               (with_U ? align256(plane * 8) : 0) + align256((size_t)cols * 4) +
               (dbg ? align256((size_t)cols * 2) + align256((size_t)cols * 8) : 0);
  S.mem = DBuf(planes_bytes + per * nruns, st);
  S.planes_bytes = planes_bytes;
  S.rows = rows;
  S.cols = cols;
  S.pitch = pitch;
  S.target = target;
  S.cl = cl;
  S.max_fr = max_fr;
  S.reaverage = reaverage;
  S.has_uniform = uniform_given;
  S.kc = kc;
  S.runs.assign(nruns, CarveRun{});
  uint8_t* base = S.mem.as<uint8_t>();
  size_t plane_off = 0;
  const int stage = SCPL_CARVE_FN(kc, carve_stage_dtab)(rows, pitch, cl) ? 1 : 0;
  for (int r = 0; r < nruns; ++r) {
    uint8_t* p = base + planes_bytes + per * r;
    auto take = [&](size_t bytes) {
      uint8_t* q = p;
      p += align256(bytes);
      return q;
    };
    CarveRun& R = S.runs[r];
    R.rows = rows;
    R.pitch = pitch;
    R.width0 = cols;
    R.target = target;
    R.kmax = kmax;
    R.stage_dtab = stage;
    R.nfr = nfr ? std::max(1, nfr[r]) : 1;
    R.reaverage = reaverage ? 1 : 0;
    R.fstride = (long long)plane_al;
    R.luma[0] = R.luma[1] = base + plane_off;
    R.grad[0] = R.grad[1] = base + plane_off + (size_t)R.nfr * plane_al;
    plane_off += (size_t)R.nfr * 2 * plane_al;
    R.width = cols;
    R.idx = reinterpret_cast<int16_t*>(take(plane * 2));
    R.pw = reinterpret_cast<uint64_t*>(take((size_t)nblk * pitch * 8));
    R.delta = reinterpret_cast<int8_t*>(take((size_t)nblk * pitch));
    R.lastce = reinterpret_cast<double*>(take((size_t)pitch * 8));
    R.rem = reinterpret_cast<int16_t*>(take((size_t)rows * rem_cap * 2));
    R.rem_cap = rem_cap;
    R.alive = reinterpret_cast<uint32_t*>(take((size_t)rows * alive_pitch * 4));
    R.alive_pitch = alive_pitch;
    R.cend = reinterpret_cast<int16_t*>(take((size_t)nblk * pitch * 2));
    R.prof = reinterpret_cast<long long*>(take(kProfBytes));
    if (!getenv("SCPL_PROF")) R.prof = nullptr;
    R.U = with_U ? reinterpret_cast<double*>(take(plane * 8)) : nullptr;
    R.sizes = reinterpret_cast<int*>(take((size_t)cols * 4));
    if (dbg) {
      R.cols = reinterpret_cast<int16_t*>(take((size_t)cols * 2));
      R.costs = reinterpret_cast<double*>(take((size_t)cols * 8));
    }
    SCPL_CARVE_FN(kc, encode_carve_tensor_maps)(R);
  }
}

// Carve every run of a set to its target, asynchronously on st: one graph launch runs the
// iteration loop on the device (pass, compaction, gradient until every run is done), then
// the index kernel; the final run states and the iteration count land in pinned memory
// (h_state: nruns CarveRuns + 16 bytes; read by carve_finish once the stream is done).
void carve_launch(scpl_ctx* ctx, CarveSet& S, void* h_state, cudaStream_t st) {
  const int nruns = (int)S.runs.size();
  CarveRun* h_runs = reinterpret_cast<CarveRun*>(h_state);
  S.h_runs = h_runs;
  S.h_iters = reinterpret_cast<int*>(h_runs + nruns);
  *S.h_iters = 0;
  if (nruns == 0) return;
  for (auto& R : S.runs) {
    R.cyc_dp = R.cyc_sel = 0;
    if (R.prof) SCPL_CUDA(cudaMemsetAsync(R.prof, 0, kProfBytes, st));
  }
  const bool graph = S.cols > S.target && !host_loops();
  S.ctx = ctx;
  S.loop_key = {nruns, S.rows, S.pitch, S.cols, S.cl, S.cols - S.target + 1, S.max_fr,
                (int)S.reaverage + 2 * graph + 4 * S.kc};
  auto it = ctx->loop_pool.find(S.loop_key);
  if (it != ctx->loop_pool.end()) {
    S.loop = it->second;
    ctx->loop_pool.erase(it);
    for (auto o = ctx->loop_order.begin(); o != ctx->loop_order.end(); ++o)
      if (*o == S.loop_key) {
        ctx->loop_order.erase(o);
        break;
      }
  } else {
    SCPL_CUDA(cudaMalloc(&S.loop.mem, sizeof(CarveRun) * nruns + 16));
  }
  CarveRun* runs_d = reinterpret_cast<CarveRun*>(S.loop.mem);
  int* iters_d = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(S.loop.mem) + sizeof(CarveRun) * nruns);
  std::memcpy(h_runs, S.runs.data(), sizeof(CarveRun) * nruns);
  // run states and the zeroed counter from mapped pinned memory
  kc6::launch_word_copy(runs_d, h_runs, sizeof(CarveRun) * nruns + sizeof(int), st);
  if (S.reaverage && !S.has_uniform)  // first pass on the mean gradient too (pipeline.py:289-290)
    kc6::launch_carve_mean(runs_d, nruns, S.rows, st);
  if (S.cols > S.target && host_loops()) {  // bursts of 8 iterations, host checks the widths
    int done_iters = 0;
    while (true) {
      for (int k = 0; k < 8; ++k)
        SCPL_CARVE_FN(S.kc, launch_carve_iteration)(runs_d, nruns, S.rows, S.pitch, S.cols, S.cl, st, S.max_fr,
                                                    S.reaverage);
      done_iters += 8;
      kc6::launch_word_copy(h_runs, runs_d, sizeof(CarveRun) * nruns, st);
      SCPL_CUDA(cudaStreamSynchronize(st));
      bool all = true;
      for (int r = 0; r < nruns; ++r) all &= h_runs[r].width <= h_runs[r].target;
      if (all || done_iters > S.cols) break;
    }
  } else if (graph) {
    if (!S.loop.ex)
      S.loop.ex = SCPL_CARVE_FN(S.kc, build_carve_loop)(runs_d, nruns, S.rows, S.pitch, S.cols, S.cl,
                                                        S.cols - S.target + 1, iters_d, S.max_fr, S.reaverage);
    SCPL_CUDA(cudaGraphLaunch(S.loop.ex, st));
  }
  kc6::launch_carve_index(runs_d, nruns, S.rows, st);
  kc6::launch_word_copy(h_runs, runs_d, sizeof(CarveRun) * nruns + sizeof(int), st);  // states + counter
}

// after the stream is done: run states back into S.runs, launch accounting, profile
void carve_finish(CarveSet& S) {
  const int nruns = (int)S.runs.size();
  if (nruns == 0) return;
  std::memcpy(S.runs.data(), S.h_runs, sizeof(CarveRun) * nruns);
  g_launches.fetch_add((long)kc6::carve_kernels_per_iteration(S.reaverage) * *S.h_iters, std::memory_order_relaxed);
  for (auto& R : S.runs)
    if (R.width > R.target) throw Error{2, "carve loop stopped before every run reached its target"};
  long long best = -1;
  for (auto& R : S.runs) {
    long long c[17] = {};
    if (R.prof) {
      SCPL_CUDA(cudaMemcpy(c, R.prof, sizeof(c), cudaMemcpyDeviceToHost));
      c[0] = R.cyc_dp;
      c[1] = R.cyc_sel;
      fprintf(stderr,
              "carve prof: iters %d rows %d | dp %lld sel %lld | xwait %lld ringwait %lld rows %lld publish %lld"
              " [bar1 %lld stores %lld bar2 %lld] store_pw %lld | sel: labels %lld min %lld cand %lld trunc %lld"
              " trace %lld (x CTAs)\n",
              R.iters, R.rows, c[0], c[1], c[4], c[5], c[6], c[7], c[8], c[9], c[10], c[11], c[12], c[13], c[14],
              c[15], c[16]);
      // pass timestamps (globaltimer ns at entry / exit of each pass): time inside passes vs gaps
      const int n = std::min(R.iters, (int)(kProfBytes / 16) - 16);
      std::vector<long long> ts(2 * (size_t)n);
      if (n > 0) {
        SCPL_CUDA(cudaMemcpy(ts.data(), R.prof + 32, sizeof(long long) * 2 * n, cudaMemcpyDeviceToHost));
        long long in = 0, gap = 0;
        for (int k = 0; k < n; ++k) {
          in += ts[2 * k + 1] - ts[2 * k];
          if (k > 0) gap += ts[2 * k] - ts[2 * k - 1];
        }
        fprintf(stderr, "carve ts: iters %d span %.3f ms in-pass %.3f ms gaps %.3f ms (first start %.3f ms)\n", n,
                (ts[2 * n - 1] - ts[0]) * 1e-6, in * 1e-6, gap * 1e-6, (ts[0] % 1000000000LL) * 1e-6);
      }
    }
    long long tot = R.cyc_dp + R.cyc_sel;
    if (tot > best) {
      best = tot;
      S.prof[0] = R.cyc_dp;
      S.prof[1] = R.cyc_sel;
      S.prof[2] = R.iters;  // passes of that run
      S.prof[3] = 0;
    }
  }
}

void carve_run_all(scpl_ctx* ctx, CarveSet& S, cudaStream_t st) {
  const int nruns = (int)S.runs.size();
  uint8_t* pin = pinned_scratch(ctx, sizeof(CarveRun) * (size_t)std::max(nruns, 1) + 64);
  carve_launch(ctx, S, pin, st);
  SCPL_CUDA(cudaStreamSynchronize(st));
  carve_finish(S);
}

}  // namespace

// ================================================================== C-ABI
extern "C" {

int scpl_version(void) { return 1; }
long scpl_kernel_launches(void) { return g_launches.load(); }
const char* scpl_last_error(void) { return g_err.c_str(); }

int scpl_create(int device, scpl_ctx** out) {
  return guarded(nullptr, [&] {
    SCPL_ARG(out != nullptr, "out is NULL");
    int n = 0;
    SCPL_CUDA(cudaGetDeviceCount(&n));
    SCPL_ARG(device >= 0 && device < n, "no such CUDA device");
    SCPL_CUDA(cudaSetDevice(device));
    auto* c = new scpl_ctx();
    c->device = device;
    SCPL_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    SCPL_CUDA(cudaDeviceGetAttribute(&c->clock_khz, cudaDevAttrClockRate, device));
    // keep freed workspace in the stream-ordered pool (no unmap/remap of GBs per clip)
    cudaMemPool_t pool;
    SCPL_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    SCPL_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    *out = c;
  });
}

void scpl_destroy(scpl_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (auto& kv : ctx->plans) {
    cudaFree(kv.second.leaves);
    cudaFree(kv.second.vnodes);
  }
  if (ctx->h_asde) cudaFreeHost(ctx->h_asde);
  if (ctx->pin) cudaFreeHost(ctx->pin);
  for (cudaStream_t x : ctx->s_carve) cudaStreamDestroy(x);
  for (auto& kv : ctx->scan_graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : ctx->loop_pool) {
    if (kv.second.ex) cudaGraphExecDestroy(kv.second.ex);
    cudaFree(kv.second.mem);
  }
  for (auto& pool : ctx->ev_pool)
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  if (ctx->scan) cudaFree(ctx->scan);
  if (ctx->phi_d) cudaFree(ctx->phi_d);
  for (cudaStream_t x : {ctx->s_h2d, ctx->s_codes, ctx->s_d2h, ctx->s_scan})
    if (x) cudaStreamDestroy(x);
  delete ctx;
}

int scpl_to_luma(scpl_ctx* ctx, const uint8_t* pixels, long npx, int channels, uint8_t* luma_out, void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(channels == 1 || channels == 3, "unsupported channel count: expected 1 or 3");
    launch_luma(pixels, npx, channels, luma_out, (cudaStream_t)stream);
  });
}

int scpl_gradient_energy(scpl_ctx* ctx, const uint8_t* luma, int h, int w, double* out, void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(h >= 3 && w >= 3, "frame too small for 3x3 Sobel");
    launch_sobel_f64(luma, h, w, out, (cudaStream_t)stream);
  });
}

int scpl_energy_codes(scpl_ctx* ctx, const uint8_t* frames, const uint8_t* prev, int T, int h, int w,
                      int channels, uint16_t* codes, void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(channels == 1 || channels == 3, "unsupported channel count: expected 1 or 3");
    SCPL_ARG(h >= 3 && w >= 3, "frame too small for 3x3 Sobel");
    launch_codes(frames, prev, 0, T, h, w, channels, codes, ctx->num_sms, (cudaStream_t)stream);
  });
}

int scpl_decode_energy(scpl_ctx* ctx, const uint16_t* codes, int T, int h, int w, int first_pure, double w_motion,
                       double w_grad, double* out, void* stream) {
  return guarded(ctx, [&] {
    launch_decode(codes, (long)h * w, T, first_pure, w_motion, w_grad, out, (cudaStream_t)stream);
  });
}

int scpl_window_asde(scpl_ctx* ctx, const uint16_t* codes, int T, int h, int w, int start, int n_acc, int count,
                     double w_motion, double w_grad, double* state, int init, double* asde_out, void* stream) {
  return guarded(ctx, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    SCPL_ARG(count >= 1 && n_acc >= 1 && start >= 0 && start + n_acc + count <= T, "window out of range");
    SCPL_ARG(!init || n_acc == 1, "init requires n_acc == 1");
    const long N = (long)h * w;
    const PwPlan& plan = plan_for(ctx, N);
    DBuf leafsum(sizeof(double) * count * plan.nleaves, st);
    DBuf partial(sizeof(double) * count * kPwFoldCtas, st);
    DBuf asde_d(sizeof(double) * count, st);
    launch_window_stats(codes, N, plan.leaves, plan.nleaves, start, n_acc, count, 1, init, w_motion, w_grad,
                        state, state + N, leafsum.as<double>(), plan.vnodes, partial.as<double>(),
                        asde_d.as<double>(), st);
    SCPL_CUDA(cudaMemcpyAsync(asde_out, asde_d.p, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
    SCPL_CUDA(cudaStreamSynchronize(st));
  });
}

int scpl_uniform_energy(scpl_ctx* ctx, const uint16_t* codes, int h, int w, int start, int n, double w_motion,
                        double w_grad, int transposed, double* out, void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(n >= 1, "empty run");
    launch_uniform(codes, h, w, start, n, 1, w_motion, w_grad, transposed, out, (cudaStream_t)stream);
  });
}

int scpl_replay(scpl_ctx* ctx, const uint8_t* in, int T, int h, int w, int channels, const int16_t* index,
                int stride, int target, int transposed, uint8_t* out, void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(channels == 1 || channels == 3, "unsupported channel count: expected 1 or 3");
    launch_replay(in, out, T, h, w, channels, index, stride, target, transposed, (cudaStream_t)stream);
  });
}

int scpl_batch_carve(scpl_ctx* ctx, const uint8_t* frame, int h, int w, int channels, int target,
                     const double* energy, int kmax, int16_t* index_out, int* n_batches, int* batch_sizes,
                     int16_t* batch_cols, double* batch_costs, int16_t* offsets, void* stream) {
  return guarded(ctx, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    SCPL_ARG(channels == 1 || channels == 3, "unsupported channel count: expected 1 or 3");
    SCPL_ARG(target >= 1, "target width must be >= 1");
    SCPL_ARG(target <= w, "target width exceeds frame width");
    SCPL_ARG(h >= 1 && w >= 1, "empty frame");
    CarveSet S;
    const int kc = carve_variant(1, w, 1, 1, ctx->num_sms, true);
    carve_alloc(S, 1, h, w, target, kmax, energy != nullptr, true, carve_cluster(kc, 1, w, ctx->num_sms), st, nullptr,
                false, kc);
    CarveRun& R = S.runs[0];
    kc6::launch_run_setup(frame, h, w, channels, 0, nullptr, R, st);
    if (energy)
      SCPL_CUDA(cudaMemcpy2DAsync(const_cast<double*>(R.U), sizeof(double) * R.pitch, energy, sizeof(double) * w,
                                  sizeof(double) * w, h, cudaMemcpyDeviceToDevice, st));
    carve_run_all(ctx, S, st);
    const CarveRun& Rh = S.runs[0];
    const int iters = w > target ? Rh.iters : 0, removed = w > target ? Rh.removed : 0;
    *n_batches = iters;
    if (iters) {
      SCPL_CUDA(cudaMemcpyAsync(batch_sizes, Rh.sizes, sizeof(int) * iters, cudaMemcpyDeviceToHost, st));
      SCPL_CUDA(cudaMemcpyAsync(batch_cols, Rh.cols, sizeof(int16_t) * removed, cudaMemcpyDeviceToHost, st));
      SCPL_CUDA(cudaMemcpyAsync(batch_costs, Rh.costs, sizeof(double) * removed, cudaMemcpyDeviceToHost, st));
    }
    SCPL_CUDA(cudaMemcpy2DAsync(index_out, sizeof(int16_t) * target, Rh.idx, sizeof(int16_t) * Rh.pitch,
                                sizeof(int16_t) * target, h, cudaMemcpyDeviceToDevice, st));
    if (offsets && removed) {
      std::vector<int16_t> log((size_t)h * Rh.rem_cap);
      SCPL_CUDA(cudaMemcpyAsync(log.data(), Rh.rem, sizeof(int16_t) * log.size(), cudaMemcpyDeviceToHost, st));
      SCPL_CUDA(cudaStreamSynchronize(st));
      for (int s = 0; s < removed; ++s)
        for (int i = 0; i < h; ++i) offsets[(size_t)s * h + i] = log[(size_t)i * Rh.rem_cap + s];
    }
    SCPL_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"

namespace {

// retarget_video (pipeline.py:92-137), streamed.  The clip (device buffer, or pinned host
// buffer copied in 16-frame chunks on a copy stream) gets its energy codes and the device-
// side buffer scan chunk by chunk; whenever the scan has closed enough runs, the host hands
// them as one group to a carve stream: per phase (width, then height, or the reverse) a
// run set is carved by the device-side iteration loop and replayed into the output, and
// with host buffers the group's output frames leave on a second copy stream.  Groups carve
// concurrently with the scan, the copies and each other (each carve is latency bound on a
// few SMs).  Runs are independent, so the results do not depend on the grouping.
struct Group {
  std::list<CarveSet> sets;
  std::list<DBuf> bufs;
  cudaStream_t st = nullptr;
};

void retarget_core(scpl_ctx* ctx, const uint8_t* frames_dev, const uint8_t* frames_host, int T, int h, int w,
                   int channels, const scpl_video_params& P, uint8_t* out_dev, uint8_t* out_host,
                   scpl_video_result* result, cudaStream_t st) {
  const bool timeline = getenv("SCPL_TIMELINE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;  // (label, timing event)
  const auto t_host0 = std::chrono::steady_clock::now();
  auto hmark = [&](const std::string& label) {
    if (!timeline) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    fprintf(stderr, "host %8.3f ms  %s\n", ms, label.c_str());
  };
  SCPL_ARG(channels == 1 || channels == 3, "unsupported channel count: expected 1 or 3");
  SCPL_ARG(h >= 3 && w >= 3, "frame too small to carve");
  SCPL_ARG(P.target_width >= 1 && P.target_width <= w, "target width out of range");
  SCPL_ARG(P.target_height >= 1 && P.target_height <= h, "target height out of range");
  SCPL_ARG(P.mode >= 0 && P.mode <= 2, "unknown mode");
  SCPL_ARG(P.max_len >= 1, "max_len must be >= 1");
  SCPL_ARG(P.mode != 2 || P.phi != nullptr, "phi table required for buffered mode");
  SCPL_ARG(P.shard_count <= 1 || (P.shard_rank >= 0 && P.shard_rank < P.shard_count),
           "shard_rank must be in 0 .. shard_count-1");
  const int shards = std::max(1, P.shard_count);
  result->dp_passes = 0;
  result->n_runs = 0;
  for (float& x : result->phase_ms) x = 0.f;
  for (long long& x : result->carve_cycles) x = 0;
  result->carve_cluster = 0;
  result->scan_windows = result->scan_fallbacks = 0;
  if (T <= 0) return;
  const int C = channels;
  const int tw = P.target_width, th = P.target_height;
  const size_t fbytes0 = (size_t)h * w * C;
  const bool host_in = frames_host != nullptr, host_out = out_host != nullptr;
  const bool buffered = P.mode == 2;
  // Priorities: the scan feeds everything (it releases the runs), so codes and scan get the
  // highest; carve groups are ordered by start frame (see dispatch) -- the carve passes
  // compete for whole SMs.
  // Levels: prio_hi (scan) .. prio_lo; carve groups use prio_hi+1 .. prio_lo (or all if the
  // range is tiny), kStreamsPerLevel streams each.
  if (!ctx->prio_known) {
    SCPL_CUDA(cudaDeviceGetStreamPriorityRange(&ctx->prio_lo, &ctx->prio_hi));
    ctx->prio_known = true;
  }
  const int prio_lo = ctx->prio_lo, prio_hi = ctx->prio_hi;
  for (cudaStream_t* x : {&ctx->s_h2d, &ctx->s_d2h})
    if (!*x) SCPL_CUDA(cudaStreamCreateWithFlags(x, cudaStreamNonBlocking));
  for (cudaStream_t* x : {&ctx->s_codes, &ctx->s_scan})
    if (!*x) SCPL_CUDA(cudaStreamCreateWithPriority(x, cudaStreamNonBlocking, prio_hi));
  const int carve_hi = prio_lo - prio_hi >= 2 ? prio_hi + 1 : prio_hi;
  const int nlevels = prio_lo - carve_hi + 1;  // levels carve_hi .. prio_lo
  const int kStreamsPerLevel = 4;
  while ((int)ctx->s_carve.size() < nlevels * kStreamsPerLevel) {
    const int level = (int)ctx->s_carve.size() / kStreamsPerLevel;  // 0 = lowest priority
    cudaStream_t x;
    SCPL_CUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, prio_lo - level));
    ctx->s_carve.push_back(x);
  }
  std::vector<int> phases;  // 0 width, 1 height (pipeline.py:192-193, 246-277)
  for (int ax : (P.height_first ? std::vector<int>{1, 0} : std::vector<int>{0, 1})) {
    if (ax == 0 && tw < w) phases.push_back(0);
    if (ax == 1 && th < h) phases.push_back(1);
  }
  const int chunk = 16;
  const int nchunk = (T + chunk - 1) / chunk;

  // pinned scratch: scan readbacks, then per group and phase the carve-run states
  const size_t scan_pin = 64 + ((sizeof(int) * (nchunk + 2 * (size_t)T) + 63) & ~(size_t)63) + sizeof(ScanState);
  const size_t need = scan_pin + (phases.size() + 1) * (size_t)T * (sizeof(CarveRun) + 64) + 4096;
  uint8_t* pin = pinned_scratch(ctx, need);
  size_t pin_used = 0;
  auto pin_take = [&](size_t bytes) {
    uint8_t* q = pin + pin_used;
    pin_used += (bytes + 63) & ~(size_t)63;
    SCPL_ARG(pin_used <= need, "internal: pinned scratch exhausted");
    return q;
  };

  // events come from (and go back to) the context's pools: every use is complete once the
  // call returns (final synchronize, or the drain guard on the error path)
  std::vector<std::pair<cudaEvent_t, bool>> events;
  struct EvGuard {
    scpl_ctx* ctx;
    std::vector<std::pair<cudaEvent_t, bool>>& e;
    ~EvGuard() {
      for (auto& x : e) ctx->ev_pool[x.second].push_back(x.first);
    }
  } evg{ctx, events};
  auto new_event = [&](bool timing) {
    cudaEvent_t e;
    auto& pool = ctx->ev_pool[timing];
    if (!pool.empty()) {
      e = pool.back();
      pool.pop_back();
    } else {
      SCPL_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
    }
    events.push_back({e, timing});
    return e;
  };
  cudaEvent_t ev_start = new_event(true), ev_codes = new_event(true), ev_scan = new_event(true),
              ev_end = new_event(true);
  SCPL_CUDA(cudaEventRecord(ev_start, st));
  hmark("start recorded");

  // buffers (stream-ordered on st; every other stream waits for ev_alloc)
  DBuf frames_buf, codes, out_buf;
  const uint8_t* frames = frames_dev;
  if (host_in) {
    frames_buf = DBuf(fbytes0 * T, st);
    frames = frames_buf.as<uint8_t>();
  }
  if (P.mode != 0) codes = DBuf(sizeof(uint16_t) * (size_t)T * h * w, st);
  uint8_t* out = out_dev;
  if (host_out) {
    out_buf = DBuf((size_t)T * th * tw * C, st);
    out = out_buf.as<uint8_t>();
  }
  ScanStream scan;
  if (buffered) {
    scan.h_n = reinterpret_cast<int*>(pin_take(sizeof(int) * nchunk));
    scan.h_runs = reinterpret_cast<int*>(pin_take(sizeof(int) * 2 * (size_t)T));
    scan.h_state = reinterpret_cast<ScanState*>(pin_take(sizeof(ScanState)));
    scan.h_L = reinterpret_cast<int*>(pin_take(sizeof(int)));
    scan_start(ctx, scan, codes.as<uint16_t>(), T, h, w, P, st);
  }
  std::list<Group> groups;
  auto mark = [&](const std::string& label, cudaStream_t sm) {
    if (!timeline) return;
    cudaEvent_t e = new_event(true);
    SCPL_CUDA(cudaEventRecord(e, sm));
    marks.push_back({label, e});
  };
  // from here on, anything that unwinds must first let the queued work finish
  struct DrainGuard {
    bool armed = true;
    ~DrainGuard() {
      if (armed) cudaDeviceSynchronize();
    }
  } drain;
  cudaEvent_t ev_alloc = new_event(false);
  SCPL_CUDA(cudaEventRecord(ev_alloc, st));

  // 1. frames in (host) and energy codes, chunk by chunk (the scan starts on the first chunk)
  std::vector<cudaEvent_t> ev_chunk_codes(nchunk, nullptr);
  if (host_in) SCPL_CUDA(cudaStreamWaitEvent(ctx->s_h2d, ev_alloc, 0));
  SCPL_CUDA(cudaStreamWaitEvent(ctx->s_codes, ev_alloc, 0));
  for (int c = 0; c < nchunk; ++c) {
    const int t0 = c * chunk, n = std::min(chunk, T - t0);
    if (host_in) {
      SCPL_CUDA(cudaMemcpyAsync(const_cast<uint8_t*>(frames) + fbytes0 * t0, frames_host + fbytes0 * t0,
                                fbytes0 * n, cudaMemcpyHostToDevice, ctx->s_h2d));
      mark("h2d " + std::to_string(c), ctx->s_h2d);
      cudaEvent_t e = new_event(false);
      SCPL_CUDA(cudaEventRecord(e, ctx->s_h2d));
      SCPL_CUDA(cudaStreamWaitEvent(ctx->s_codes, e, 0));
    }
    if (P.mode != 0)
      launch_codes(frames, nullptr, t0, n, h, w, C, codes.as<uint16_t>(), ctx->num_sms, ctx->s_codes);
    ev_chunk_codes[c] = new_event(false);
    SCPL_CUDA(cudaEventRecord(ev_chunk_codes[c], ctx->s_codes));
  }
  cudaStream_t ss = ctx->s_scan;
  SCPL_CUDA(cudaStreamWaitEvent(ss, ev_alloc, 0));
  SCPL_CUDA(cudaStreamWaitEvent(ss, ev_chunk_codes[0], 0));
  SCPL_CUDA(cudaEventRecord(ev_codes, ss));  // (first chunk's codes)

  // 2. buffer scan, chunk by chunk (fixed one-frame runs for scpl / raw)
  std::vector<cudaEvent_t> ev_chunk(nchunk, nullptr);
  if (buffered) {
    for (int c = 0; c < nchunk; ++c) {
      SCPL_CUDA(cudaStreamWaitEvent(ss, ev_chunk_codes[c], 0));
      scan_chunk(ctx, scan, c, std::min(T, (c + 1) * chunk), ss);
      mark("scan " + std::to_string(c), ss);
      ev_chunk[c] = new_event(false);
      SCPL_CUDA(cudaEventRecord(ev_chunk[c], ss));
    }
    scan_end(ctx, scan, ss);
  } else {
    SCPL_CUDA(cudaStreamWaitEvent(ss, ev_chunk_codes[nchunk - 1], 0));
  }
  SCPL_CUDA(cudaEventRecord(ev_scan, ss));

  // 3. carve + replay, one run group at a time as runs close
  std::vector<std::pair<int, int>> runs;
  int next_stream = 0;
  auto dispatch = [&](int r0, int r1, cudaEvent_t ready, bool final_group) {
    if (r1 <= r0) return;
    Group& G = groups.emplace_back();
    {  // later groups (by first frame) on higher-priority streams
      const int ta0 = runs[r0].first;
      int level = std::min(nlevels - 1, (int)((long)ta0 * nlevels / std::max(T, 1)));
      // a device clip's runs are all closed within the scan, and then every group competes for
      // SMs: the earliest groups go first (measured ~2% faster on C2 than the other order, and
      // equal priorities are ~30% slower); a host clip's last group closes alone after the
      // copies and is the critical path, so there the later groups go first
      if (!host_in) level = nlevels - 1 - level;
      G.st = ctx->s_carve[level * kStreamsPerLevel + (next_stream++ % kStreamsPerLevel)];
    }
    cudaStream_t gs = G.st;
    SCPL_CUDA(cudaStreamWaitEvent(gs, ev_alloc, 0));
    SCPL_CUDA(cudaStreamWaitEvent(gs, ready, 0));
    const int nr = r1 - r0;
    const int ta = runs[r0].first, tb = runs[r1 - 1].first + runs[r1 - 1].second;
    mark("group " + std::to_string(groups.size() - 1) + " start", gs);
    auto ship = [&](size_t off, size_t bytes) {  // D2H of finished output frames
      if (!host_out) return;
      cudaEvent_t e = new_event(false);
      SCPL_CUDA(cudaEventRecord(e, gs));
      SCPL_CUDA(cudaStreamWaitEvent(ctx->s_d2h, e, 0));
      SCPL_CUDA(cudaMemcpyAsync(out_host + off, out + off, bytes, cudaMemcpyDeviceToHost, ctx->s_d2h));
    };
    if (phases.empty()) {
      SCPL_CUDA(cudaMemcpyAsync(out + fbytes0 * ta, frames + fbytes0 * ta, fbytes0 * (tb - ta),
                                cudaMemcpyDeviceToDevice, gs));
      ship(fbytes0 * ta, fbytes0 * (tb - ta));
      return;
    }
    const uint8_t* cur = frames;
    int cur_t0 = 0, curH = h, curW = w;
    for (size_t ph = 0; ph < phases.size(); ++ph) {
      const bool height = phases[ph] == 1;
      const int rows = height ? curW : curH, cols = height ? curH : curW;
      const int target = height ? th : tw;
      const bool with_U = (ph == 0) && P.mode != 0;
      CarveSet& S = G.sets.emplace_back();
      hmark("group alloc");
      const bool rea = P.reaverage != 0 && P.mode != 0;  // raw mode ignores it (pipeline.py:120-132)
      std::vector<int> nfr;
      if (rea)
        for (int r = r0; r < r1; ++r) nfr.push_back(runs[r].second);
      const int kc = carve_variant(nr, cols, tb - ta, T, ctx->num_sms, final_group);
      carve_alloc(S, nr, rows, cols, target, P.mode == 0 ? 1 : 0, with_U, false,
                  carve_cluster(kc, nr, cols, ctx->num_sms), gs, rea ? nfr.data() : nullptr, rea, kc);
      hmark("group setup");
      const size_t fbytes = (size_t)curH * curW * C;
      for (int r = r0; r < r1; ++r) {
        CarveRun& R = S.runs[r - r0];
        const int s0 = runs[r].first;
        // the first carved axis works on the original frames, whose energy codes carry the
        // Sobel gradient of every frame (so the carve's gradient plane needs no recompute);
        // reaverage carves every frame of the run, otherwise its first frame represents it
        for (int f = 0; f < R.nfr; ++f) {
          const uint16_t* fcodes =
              (ph == 0 && P.mode != 0) ? codes.as<uint16_t>() + (size_t)(s0 + f) * h * w : nullptr;
          kc6::launch_run_setup(cur + fbytes * (s0 + f - cur_t0), curH, curW, C, height ? 1 : 0, fcodes, R, gs, f);
        }
        if (with_U)
          launch_uniform(codes.as<uint16_t>(), h, w, s0, runs[r].second, 1, P.w_motion, P.w_grad, height ? 1 : 0,
                         const_cast<double*>(R.U), gs, R.pitch);
      }
      mark("group " + std::to_string(groups.size() - 1) + " setup done", gs);
      hmark("group carve_launch");
      carve_launch(ctx, S, pin_take(sizeof(CarveRun) * nr + 16), gs);
      hmark("group replay");
      mark("group " + std::to_string(groups.size() - 1) + " carve done", gs);
      const int nH = height ? th : curH, nW = height ? curW : tw;
      const bool last = ph + 1 == phases.size();
      uint8_t* dst = out;
      int dst_t0 = 0;
      if (!last) {
        dst = G.bufs.emplace_back((size_t)(tb - ta) * nH * nW * C, gs).as<uint8_t>();
        dst_t0 = ta;
      }
      const size_t obytes = (size_t)nH * nW * C;
      for (int r = r0; r < r1; ++r) {
        const CarveRun& R = S.runs[r - r0];
        const int s0 = runs[r].first, n = runs[r].second;
        launch_replay(cur + fbytes * (s0 - cur_t0), dst + obytes * (s0 - dst_t0), n, curH, curW, C, R.idx, R.pitch,
                      target, height ? 1 : 0, gs);
        if (last) ship(obytes * s0, obytes * n);
      }
      mark("group " + std::to_string(groups.size() - 1) + " phase " + std::to_string(ph) + " runs " +
               std::to_string(nr), gs);
      cur = dst;
      cur_t0 = dst_t0;
      curH = nH;
      curW = nW;
    }
    if (host_out) mark("d2h group " + std::to_string(groups.size() - 1), ctx->s_d2h);
  };
  if (buffered) {
    // host clips: every closed run goes out at once (the copies are the bottleneck); device
    // clips: groups of >= 4 runs (fewer, larger carve sets)
    int min_group = host_in ? 1 : 4;
    if (const char* e = getenv("SCPL_GROUP_MIN")) min_group = std::max(1, atoi(e));
    int done = 0;
    for (int c = 0; c < nchunk; ++c) {
      hmark("wait chunk " + std::to_string(c));
      SCPL_CUDA(cudaEventSynchronize(ev_chunk[c]));
      const int n = scan.h_n[c];
      for (int r = (int)runs.size(); r < n; ++r) runs.push_back({scan.h_runs[2 * r], scan.h_runs[2 * r + 1]});
      if (shards > 1) {  // this rank's runs (round-robin by run index), each as it closes
        for (int r = done; r < n; ++r)
          if (r % shards == P.shard_rank) dispatch(r, r + 1, ev_chunk[c], host_in && c + 1 == nchunk);
        done = n;
      } else if (n - done >= min_group || (c + 1 == nchunk && n > done)) {
        // (a device clip's scan ends long before its groups do: only a host clip's last group,
        // closed after the copies, carves with the GPU to itself)
        dispatch(done, n, ev_chunk[c], host_in && c + 1 == nchunk);
        done = n;
      }
    }
  } else {
    for (int t = 0; t < T; ++t) runs.push_back({t, 1});
    // sharded: a contiguous block of frames per rank
    dispatch((int)((long)T * P.shard_rank / shards), (int)((long)T * (P.shard_rank + 1) / shards), ev_scan, false);
  }
  SCPL_CUDA(cudaStreamWaitEvent(st, ev_scan, 0));
  for (Group& G : groups) {
    cudaEvent_t e = new_event(false);
    SCPL_CUDA(cudaEventRecord(e, G.st));
    SCPL_CUDA(cudaStreamWaitEvent(st, e, 0));
  }
  if (host_out) {
    cudaEvent_t e = new_event(false);
    SCPL_CUDA(cudaEventRecord(e, ctx->s_d2h));
    SCPL_CUDA(cudaStreamWaitEvent(st, e, 0));
  }
  SCPL_CUDA(cudaEventRecord(ev_end, st));
  hmark("all queued");
  SCPL_CUDA(cudaStreamSynchronize(st));
  drain.armed = false;
  hmark("synchronized");

  // 4. results
  if (buffered) scan_finish(scan, nchunk, result);
  result->n_runs = (int)runs.size();
  if (result->run_start && result->run_len)
    for (size_t r = 0; r < runs.size(); ++r) {
      result->run_start[r] = runs[r].first;
      result->run_len[r] = runs[r].second;
    }
  long dp = 0, pass_launches = 0;
  long long pass_cyc = 0;
  for (Group& G : groups)
    for (CarveSet& S : G.sets) {
      carve_finish(S);
      long long slow = 0;
      int launches = 0;
      for (auto& R : S.runs) {
        dp += R.iters;
        slow = std::max(slow, R.cyc_dp + R.cyc_sel);
        launches = std::max(launches, R.iters);
      }
      pass_cyc += slow;  // a launch lasts as long as its slowest cluster
      pass_launches += launches;
      if (S.prof[0] + S.prof[1] > result->carve_cycles[0] + result->carve_cycles[1])
        for (int k = 0; k < 3; ++k) result->carve_cycles[k] = S.prof[k];
      result->carve_cluster = S.cl;
    }
  result->dp_passes = dp;
  result->carve_cycles[3] = pass_launches;
  if (pass_launches > 0) result->phase_ms[3] = (float)((double)pass_cyc / pass_launches / std::max(ctx->clock_khz, 1));
  for (auto& m : marks) {
    float ms = 0.f;
    SCPL_CUDA(cudaEventElapsedTime(&ms, ev_start, m.second));
    fprintf(stderr, "timeline %8.3f ms  %s\n", ms, m.first.c_str());
  }
  SCPL_CUDA(cudaEventElapsedTime(&result->phase_ms[0], ev_start, ev_codes));
  SCPL_CUDA(cudaEventElapsedTime(&result->phase_ms[1], ev_codes, ev_scan));
  SCPL_CUDA(cudaEventElapsedTime(&result->phase_ms[2], ev_scan, ev_end));
  if (timeline) {
    float ms = 0.f;
    SCPL_CUDA(cudaEventElapsedTime(&ms, ev_start, ev_end));
    fprintf(stderr, "timeline %8.3f ms  end\n", ms);
  }
  hmark("results");
}

}  // namespace

extern "C" {

int scpl_jitter_sums(scpl_ctx* ctx, const uint8_t* frames, int T, int h, int w, int channels,
                     unsigned long long* sums, void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(channels == 1 || channels == 3, "unsupported channel count: expected 1 or 3");
    SCPL_ARG(T >= 2, "need at least 2 frames");
    launch_jitter_sums(frames, T, (long)h * w, channels, sums, (cudaStream_t)stream);
  });
}

int scpl_retarget_video(scpl_ctx* ctx, const uint8_t* frames, int T, int h, int w, int channels,
                        const scpl_video_params* params, uint8_t* out, scpl_video_result* result, void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(params != nullptr && result != nullptr, "params/result is NULL");
    const auto t0 = std::chrono::steady_clock::now();
    retarget_core(ctx, frames, nullptr, T, h, w, channels, *params, out, nullptr, result, (cudaStream_t)stream);
    if (getenv("SCPL_TIMELINE"))
      fprintf(stderr, "host %8.3f ms  returned (after cleanup)\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  });
}

int scpl_retarget_video_host(scpl_ctx* ctx, const uint8_t* frames, int T, int h, int w, int channels,
                             const scpl_video_params* params, uint8_t* out, scpl_video_result* result,
                             void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(params != nullptr && result != nullptr, "params/result is NULL");
    SCPL_ARG(frames != nullptr && out != nullptr, "frames/out is NULL");
    retarget_core(ctx, nullptr, frames, T, h, w, channels, *params, nullptr, out, result, (cudaStream_t)stream);
  });
}

int scpl_cumulative_energy(scpl_ctx* ctx, const double* energy, int h, int w, double* ce, int8_t* back,
                           void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(h >= 1 && w >= 1, "expected a non-empty 2-d energy map");
    launch_dp_tables(energy, h, w, ce, back, (cudaStream_t)stream);
  });
}

int scpl_label_parents(scpl_ctx* ctx, const int8_t* back, int h, int w, int64_t* labels, void* stream) {
  return guarded(ctx, [&] { launch_labels(back, h, w, (long*)labels, (cudaStream_t)stream); });
}

int scpl_trace_columns(scpl_ctx* ctx, const int8_t* back, int h, int w, const int64_t* cols, int b,
                       int64_t* offsets, void* stream) {
  return guarded(ctx, [&] { launch_trace(back, h, w, (const long*)cols, b, (long*)offsets, (cudaStream_t)stream); });
}

int scpl_select_batch(scpl_ctx* ctx, const double* last, const int64_t* labels, int w, int k, int64_t* cols,
                      double* costs, int* nb, void* stream) {
  return guarded(ctx, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    DBuf d_nb(sizeof(int), st);
    launch_select_tables(last, (const long*)labels, w, k, (long*)cols, costs, d_nb.as<int>(), st);
    SCPL_CUDA(cudaMemcpyAsync(nb, d_nb.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    SCPL_CUDA(cudaStreamSynchronize(st));
  });
}

int scpl_remove_columns(scpl_ctx* ctx, const uint8_t* in, int h, int w, int channels, const int64_t* offsets, int b,
                        uint8_t* out, int* rowcount, void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(b >= 0 && b <= w, "batch larger than the frame");
    launch_remove_cols(in, h, w, channels, (const long*)offsets, b, out, rowcount, (cudaStream_t)stream);
  });
}

int scpl_sums_start(scpl_ctx* ctx, const double* e, long n, double* S, double* Q, void* stream) {
  return guarded(ctx, [&] { launch_sums(e, n, nullptr, nullptr, S, Q, (cudaStream_t)stream); });
}

int scpl_sums_push(scpl_ctx* ctx, const double* e, long n, const double* S_in, const double* Q_in, double* S,
                   double* Q, void* stream) {
  return guarded(ctx, [&] { launch_sums(e, n, S_in, Q_in, S, Q, (cudaStream_t)stream); });
}

int scpl_sums_map(scpl_ctx* ctx, const double* S, const double* Q, long N, int n, int what, double* out,
                  void* stream) {
  return guarded(ctx, [&] { launch_sums_map(S, Q, N, n, what, out, (cudaStream_t)stream); });
}

int scpl_asde_from_sums(scpl_ctx* ctx, const double* S, const double* Q, long N, int n, double* out, void* stream) {
  return guarded(ctx, [&] {
    cudaStream_t st = (cudaStream_t)stream;
    SCPL_ARG(N >= 1 && n >= 1, "empty buffer");
    const PwPlan& plan = plan_for(ctx, N);
    DBuf leafsum(sizeof(double) * plan.nleaves, st);
    DBuf partial(sizeof(double) * kPwFoldCtas, st);
    DBuf d(sizeof(double), st);
    launch_asde_sums(S, Q, N, n, plan.leaves, plan.nleaves, plan.vnodes, leafsum.as<double>(), partial.as<double>(),
                     d.as<double>(), st);
    SCPL_CUDA(cudaMemcpyAsync(out, d.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    SCPL_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
