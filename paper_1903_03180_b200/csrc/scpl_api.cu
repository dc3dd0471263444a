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
#include <tuple>
#include <string>
#include <thread>
#include <vector>

#include "../../include/scpl.h"
#include "scpl_common.cuh"
#include "scpl_kernels.h"

using namespace scpl;

namespace scpl {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
// true the first time (current device, key) is seen: per-device function attributes (one
// process may drive several GPUs)
bool once_per_device(const void* key) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  SCPL_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  return done.insert({dev, key}).second;
}
void smem_optin(const void* kernel) {
  static std::mutex mu;  // (serialises the attribute calls of concurrent first launches)
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  SCPL_CUDA(cudaGetDevice(&dev));
  static std::set<std::pair<int, const void*>> done;
  if (done.count({dev, kernel})) return;
  int optin = 0;
  SCPL_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  SCPL_CUDA(cudaFuncGetAttributes(&fa, kernel));
  SCPL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - (int)fa.sharedSizeBytes));
  done.insert({dev, kernel});
}
// SCPL_GRAPH_PRIO=1 (experiments): the kernel nodes of the scan / carve loop graphs carry the
// priority of the stream they are launched into (captured nodes otherwise run at the capture
// stream's default priority).  Measured: no gain on any config, and the carve loops' pool then
// holds one graph per (shape, priority), so a C4 batch step now and then instantiates graphs
// (52 -> 96 ms outliers); off by default.
static bool graph_prio_on() {
  static const bool on = getenv("SCPL_GRAPH_PRIO") && atoi(getenv("SCPL_GRAPH_PRIO")) != 0;
  return on;
}
void graph_set_priority(cudaGraph_t g, int prio) {
  if (!graph_prio_on()) return;
  static const bool dbg = getenv("SCPL_DEBUG_PRIO") != nullptr;
  size_t n = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  std::vector<cudaGraphNode_t> nodes(n);
  if (n && cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  for (cudaGraphNode_t nd : nodes) {
    // (not every node type answers the attribute calls: those are skipped)
    cudaKernelNodeAttrValue v = {};
    const cudaError_t e0 = cudaGraphKernelNodeGetAttribute(nd, cudaKernelNodeAttributePriority, &v);
    const int had = v.priority;
    if (e0 != cudaSuccess) {
      cudaGetLastError();
      if (dbg) fprintf(stderr, "scpl prio: node skipped (%s)\n", cudaGetErrorString(e0));
      continue;
    }
    v.priority = prio;
    const cudaError_t e1 = cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributePriority, &v);
    if (e1 != cudaSuccess) cudaGetLastError();
    if (dbg) fprintf(stderr, "scpl prio: kernel node %d -> %d (%s)\n", had, prio, cudaGetErrorString(e1));
  }
}
cudaStream_t capture_stream(int prio) {
  cudaStream_t cs;
  if (graph_prio_on())
    SCPL_CUDA(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, prio));
  else
    SCPL_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  return cs;
}
std::atomic<long> g_launches{0};
int carve_unroll() {
  static const int u = getenv("SCPL_CARVE_UNROLL") ? std::min(8, std::max(1, atoi(getenv("SCPL_CARVE_UNROLL")))) : 4;
  return u;
}
}  // namespace scpl

struct PwPlan {
  int2* leaves = nullptr;
  PwVnode* vnodes = nullptr;
  int nleaves = 0;
};

// A lane: what one clip in flight needs for itself -- its codes and scan streams and its
// device-side scan state (several clips' scans run at once in a batch).
struct ScanLane {
  cudaStream_t s_codes = nullptr, s_scan = nullptr;
  ScanState* scan = nullptr;  // device
};

struct scpl_ctx {
  std::mutex mu;  // one C-ABI call at a time per context (entry points lock it)
  int device = 0;
  int num_sms = 148;
  int clock_khz = 0;  // base SM clock (queried once: the query costs milliseconds of host time)
  int prio_lo = 0, prio_hi = 0;
  bool prio_known = false;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // copy streams
  std::vector<ScanLane> lanes;
  std::map<long, PwPlan> plans;
  double* phi_d = nullptr;
  std::vector<double> phi_h;                       // contents of phi_d
  std::map<std::tuple<long, int, const void*>, cudaGraphExec_t> scan_graphs;  // (N, spec, lane state)
  uint8_t* pin = nullptr;  // pinned scratch (pinned_scratch)
  size_t pin_cap = 0;
  std::vector<std::vector<cudaStream_t>> s_carve;  // concurrent run groups, per priority level
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

// restores the calling thread's current device (the caller -- e.g. torch -- may be on another)
struct DeviceRestore {
  int dev = -1;
  ~DeviceRestore() {
    if (dev >= 0) cudaSetDevice(dev);
  }
};

template <class F>
int guarded(scpl_ctx* ctx, F&& f) {
  try {
    std::unique_lock<std::mutex> lock;
    DeviceRestore restore;
    if (ctx) {
      lock = std::unique_lock<std::mutex>(ctx->mu);
      SCPL_CUDA(cudaGetDevice(&restore.dev));
      if (restore.dev == ctx->device) restore.dev = -1;
      else SCPL_CUDA(cudaSetDevice(ctx->device));
    }
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
  long N = 0;
  cudaGraphExec_t graph = nullptr;
  const PwPlan* plan = nullptr;
  ScanState* state = nullptr;  // the lane's device state
  int spec = 8;
  int* h_L = nullptr;  // pinned (host-driven loops)
  int T = 0;
  int* h_n = nullptr;     // pinned: run count after each chunk
  int* h_runs = nullptr;  // pinned: (start, len) pairs, 2T ints
  ScanState* h_state = nullptr;
};

// the phi table (threshold(n), n = 0..max_len) on the device; shared by every lane of a call
void upload_phi(scpl_ctx* ctx, const scpl_video_params& P) {
  std::vector<double> phi(P.phi, P.phi + P.max_len + 1);
  if (phi == ctx->phi_h) return;
  if (ctx->phi_h.size() < phi.size()) {
    if (ctx->phi_d) cudaFree(ctx->phi_d);
    ctx->phi_d = nullptr;
    SCPL_CUDA(cudaMalloc(&ctx->phi_d, sizeof(double) * phi.size()));
  }
  SCPL_CUDA(cudaMemcpy(ctx->phi_d, phi.data(), sizeof(double) * phi.size(), cudaMemcpyHostToDevice));
  ctx->phi_h = phi;
}

void scan_start(scpl_ctx* ctx, ScanStream& S, ScanLane& lane, const uint16_t* codes, int T, int H, int W,
                const scpl_video_params& P, cudaStream_t st) {
  const long N = (long)H * W;
  const PwPlan& plan = plan_for(ctx, N);
  // candidates per scan window (speculation length): params, else SCPL_SPEC (experiments), else 16
  // (a window's fixed cost -- launch, checkpoint, decision -- is ~7 candidates' worth of work; a
  // run's first window is still capped by the previous run's length)
  static const int spec_env = getenv("SCPL_SPEC") ? atoi(getenv("SCPL_SPEC")) : 0;
  const int spec = P.spec_len > 0 ? P.spec_len : (spec_env > 0 ? spec_env : 16);
  SCPL_ARG(spec <= 64, "spec_len must be <= 64");
  if (!lane.scan) SCPL_CUDA(cudaMalloc(&lane.scan, sizeof(ScanState)));
  auto key = std::make_tuple(N, spec, (const void*)lane.scan);
  auto it = ctx->scan_graphs.find(key);
  if (it == ctx->scan_graphs.end())
    it = ctx->scan_graphs.emplace(key, build_scan_graph(lane.scan, N, plan.leaves, plan.nleaves, plan.vnodes, spec,
                                                         ctx->prio_known ? ctx->prio_hi : 0))
             .first;
  S.graph = it->second;
  S.plan = &plan;
  S.N = N;
  S.state = lane.scan;
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
  launch_scan_reset(S.state, init, st);
}

void scan_chunk(ScanStream& S, int c, int avail, cudaStream_t st) {
  launch_scan_avail(S.state, avail, st);
  if (host_loops())
    run_scan_host(S.state, S.N, S.plan->leaves, S.plan->nleaves, S.plan->vnodes, S.spec, S.h_L, st);
  else
    SCPL_CUDA(cudaGraphLaunch(S.graph, st));
  // (SM copies into mapped pinned memory: no copy-engine queueing behind the clip's copies)
  kc6::launch_word_copy(&S.h_n[c], reinterpret_cast<uint8_t*>(S.state) + offsetof(ScanState, nruns), sizeof(int), st);
  kc6::launch_word_copy(S.h_runs, S.runs_d.p, sizeof(int) * 2 * S.T, st);
}

void scan_end(ScanStream& S, cudaStream_t st) { kc6::launch_word_copy(S.h_state, S.state, sizeof(ScanState), st); }

// after the stream is done
void scan_finish(ScanStream& S, int chunks, scpl_video_result* result) {
  const ScanState& R = *S.h_state;
  if (!(R.done == 1 && R.nruns >= 1 && R.nruns <= S.T)) throw Error{2, "buffer scan did not finish"};
  g_launches.fetch_add((long)chunks + (long)R.steps, std::memory_order_relaxed);
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
  bool bucket = false;       // pad the run count to carve_bucket (batches: many group sizes)
  int kc = 6;                // DP window variant (scpl_carve2.cu: kc6 / kc4 / kc3)
  int kc_first = 6, cl_first = 1;  // variant + cluster of the fp64 first pass (uniform map)
  bool fused = false;        // fused int passes (no compaction / gradient kernels)
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
    constexpr size_t kPoolCap = 256;
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
// est_runs: runs expected to carve at the same time as this group (the group's density over
// the frames it covers, extrapolated to everything in flight)
int carve_variant(double est_runs, int cols, int num_sms) {
  const bool fit4 = cols <= 16 * 4 * 64, fit3 = cols <= 16 * 4 * 32;
  if (const char* e = getenv("SCPL_CARVE_KC")) {
    const int k = atoi(e);
    return k == 3 && fit3 ? 3 : (k == 3 || k == 4) && fit4 ? 4 : 6;
  }
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
               (dbg ? align256((size_t)cols * 2) + align256((size_t)cols * 8) +
                          align256((size_t)rem_cap * cols * 2)
                    : 0);
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
  // the fp64 first pass takes the first variant (the group's, then narrower ones) whose fp64
  // layout still fits two pass CTAs per SM: otherwise it waits for a whole free SM while the
  // other groups' int passes hold every SM (measured: the last run of C2 started ~7 ms late)
  S.kc_first = kc;
  S.cl_first = cl;
  static const bool first_same = getenv("SCPL_FIRST_SAME") != nullptr;  // (experiments)
  if (with_U && !reaverage && !first_same) {
    const bool fit4 = cols <= 16 * 4 * 64, fit3 = cols <= 16 * 4 * 32;
    for (int k : {kc, 4, 3}) {
      if ((k == 4 && !fit4) || (k == 3 && !fit3)) continue;
      const int c = carve_cluster(k, nruns, cols, 148);
      if (SCPL_CARVE_FN(k, carve_f64_fits_pair)(cols, c)) {
        S.kc_first = k;
        S.cl_first = c;
        break;
      }
    }
  }
  S.runs.assign(nruns, CarveRun{});
  // fused int passes (one frame per run): the pass kernel removes the previous batch and computes
  // the energy itself; the gradient plane's memory becomes the second luma plane
  S.fused = !reaverage && max_fr == 1 && rows >= 2 && SCPL_CARVE_FN(kc, carve_fused_ok)(cols, target, cl);
  const int ring_w = S.fused ? SCPL_CARVE_FN(kc, carve_fused_ring_w)(cols, target, cl) : 0;
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
    R.fused = S.fused ? 1 : 0;
    R.ring_w = ring_w;
    R.lsel = 0;
    R.fdbg = getenv("SCPL_FDBG") ? atoi(getenv("SCPL_FDBG")) : 0;
    if (S.fused) R.luma[1] = R.grad[0];
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
      R.labs = reinterpret_cast<int16_t*>(take((size_t)rem_cap * cols * 2));  // passes <= seams removed
    }
    SCPL_CARVE_FN(kc, encode_carve_tensor_maps)(R);
    if (S.kc_first != kc) SCPL_CARVE_FN(S.kc_first, encode_carve_tensor_map_U)(R);
  }
}

// run-count bucket of the pooled carve loops: the next power of two (multiples of 64 above)
int carve_bucket(int nruns) {
  if (nruns > 64) return (nruns + 63) / 64 * 64;
  int b = 1;
  while (b < nruns) b <<= 1;
  return b;
}

// Carve every run of a set to its target, asynchronously on st: one graph launch runs the
// iteration loop on the device (pass, compaction, gradient until every run is done), then
// the index kernel; the final run states and the iteration count land in pinned memory
// (h_state: nruns CarveRuns + 16 bytes; read by carve_finish once the stream is done).
void carve_launch(scpl_ctx* ctx, CarveSet& S, void* h_state, cudaStream_t st) {
  const int nruns = (int)S.runs.size();
  const bool graph = S.cols > S.target && !host_loops();
  // graph loops are instantiated for a bucketed run count (padding runs are already "done", so
  // every kernel skips them): the pooled graphs then serve any group size up to the bucket
  // instead of instantiating a conditional graph (~1 ms of host time) per new group size
  const int nb = graph && S.bucket ? carve_bucket(nruns) : nruns;
  CarveRun* h_runs = reinterpret_cast<CarveRun*>(h_state);
  S.h_runs = h_runs;
  S.h_iters = reinterpret_cast<int*>(h_runs + nb);
  *S.h_iters = 0;
  if (nruns == 0) return;
  for (auto& R : S.runs) {
    R.cyc_dp = R.cyc_sel = 0;
    if (R.prof) SCPL_CUDA(cudaMemsetAsync(R.prof, 0, kProfBytes, st));
  }
  S.ctx = ctx;
  int prio = 0;  // the loop's kernel nodes carry the group stream's priority (part of the pool key)
  if (graph_prio_on()) SCPL_CUDA(cudaStreamGetPriority(st, &prio));
  S.loop_key = {nb, S.rows, S.pitch, S.cols, S.cl, S.cols - S.target + 1, S.max_fr,
                (int)S.reaverage + 2 * graph + 4 * S.kc + 64 * (int)S.has_uniform + 128 * S.kc_first +
                    2048 * S.cl_first + 65536 * (int)S.fused + (1 << 20) * (prio & 15)};
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
    SCPL_CUDA(cudaMalloc(&S.loop.mem, sizeof(CarveRun) * nb + 16));
  }
  CarveRun* runs_d = reinterpret_cast<CarveRun*>(S.loop.mem);
  int* iters_d = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(S.loop.mem) + sizeof(CarveRun) * nb);
  std::memcpy(h_runs, S.runs.data(), sizeof(CarveRun) * nruns);
  for (int r = nruns; r < nb; ++r) h_runs[r] = CarveRun{};  // padding: width == target == 0
  // run states and the zeroed loop counters (iterations, CTAs done) from mapped pinned memory
  S.h_iters[1] = 0;
  kc6::launch_word_copy(runs_d, h_runs, sizeof(CarveRun) * nb + 2 * sizeof(int), st);
  if (S.reaverage && !S.has_uniform)  // first pass on the mean gradient too (pipeline.py:289-290)
    kc6::launch_carve_mean(runs_d, nruns, S.rows, st);
  if (S.cols > S.target && host_loops()) {  // bursts of 8 iterations, host checks the widths
    int done_iters = 0;
    while (true) {
      for (int k = 0; k < 8; ++k) {  // (a uniform map's first pass is an fp64 one)
        const bool first = done_iters + k == 0 && S.has_uniform && !S.reaverage;
        SCPL_CARVE_FN(first ? S.kc_first : S.kc, launch_carve_iteration)(
            runs_d, nruns, S.rows, S.pitch, S.cols, first ? S.cl_first : S.cl, st, S.max_fr, S.reaverage, first,
            nullptr, S.fused);
      }
      done_iters += 8;
      kc6::launch_word_copy(h_runs, runs_d, sizeof(CarveRun) * nruns, st);
      SCPL_CUDA(cudaStreamSynchronize(st));
      bool all = true;
      for (int r = 0; r < nruns; ++r) all &= h_runs[r].width <= h_runs[r].target;
      if (all || done_iters > S.cols) break;
    }
  } else if (graph) {
    if (!S.loop.ex)
      S.loop.ex = SCPL_CARVE_FN(S.kc, build_carve_loop)(
          runs_d, nb, S.rows, S.pitch, S.cols, S.cl, S.cols - S.target + 1, iters_d, S.max_fr, S.reaverage,
          S.has_uniform, SCPL_CARVE_FN(S.kc_first, launch_carve_iteration), S.cl_first, S.fused, prio);
    SCPL_CUDA(cudaGraphLaunch(S.loop.ex, st));
  }
  kc6::launch_carve_index(runs_d, nruns, S.rows, st);
  kc6::launch_word_copy(h_runs, runs_d, sizeof(CarveRun) * nb + sizeof(int), st);  // states + counter
}

// after the stream is done: run states back into S.runs, launch accounting, profile
void carve_finish(CarveSet& S) {
  const int nruns = (int)S.runs.size();
  if (nruns == 0) return;
  std::memcpy(S.runs.data(), S.h_runs, sizeof(CarveRun) * nruns);
  {  // kernels per executed loop body: the unrolled iterations' kernels + one condition kernel
    const long per_iter = (S.fused ? 2 : kc6::carve_kernels_per_iteration(S.reaverage)) - 1;
    g_launches.fetch_add((per_iter * carve_unroll() + 1) * *S.h_iters, std::memory_order_relaxed);
  }
  for (auto& R : S.runs)
    if (R.width > R.target) throw Error{2, "carve loop stopped before every run reached its target"};
  long long best = -1;
  for (auto& R : S.runs) {
    long long c[31] = {};
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
      if (R.fused)
        fprintf(stderr,
                "carve prod (rank 0 thread 0, cycles): stagewait %lld issue %lld A0 %lld A1 %lld A2 %lld empty %lld"
                " B %lld full %lld svc %lld | dp ringwait %lld | A1 setup %lld words %lld edge %lld own %lld\n",
                c[17], c[18], c[19], c[20], c[21], c[22], c[23], c[24], c[25], c[26], c[27], c[28], c[29], c[30]);
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
  uint8_t* pin = pinned_scratch(ctx, sizeof(CarveRun) * (size_t)carve_bucket(std::max(nruns, 1)) + 64);
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
  if (ctx->pin) cudaFreeHost(ctx->pin);
  for (auto& lv : ctx->s_carve)
    for (cudaStream_t x : lv) cudaStreamDestroy(x);
  for (auto& kv : ctx->scan_graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : ctx->loop_pool) {
    if (kv.second.ex) cudaGraphExecDestroy(kv.second.ex);
    cudaFree(kv.second.mem);
  }
  for (auto& pool : ctx->ev_pool)
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  for (auto& l : ctx->lanes) {
    if (l.scan) cudaFree(l.scan);
    for (cudaStream_t x : {l.s_codes, l.s_scan})
      if (x) cudaStreamDestroy(x);
  }
  if (ctx->phi_d) cudaFree(ctx->phi_d);
  for (cudaStream_t x : {ctx->s_h2d, ctx->s_d2h})
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
    const int kc = carve_variant(1.0, w, ctx->num_sms);
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

// retarget_video (pipeline.py:92-137), streamed, for one clip or a batch of clips of one shape.
// Every clip (device buffer, or pinned host buffer copied in 16-frame chunks on a copy stream)
// gets its energy codes and its device-side buffer scan chunk by chunk on its own lane (codes
// and scan streams, scan state); whenever the scans have closed enough runs, the host hands
// them -- from any clip -- as one group to a carve stream: per phase (width, then height, or
// the reverse) the group's runs are carved together by the device-side iteration loop and
// replayed into their clips' outputs, and with host buffers each run's output frames leave on
// a second copy stream.  Groups carve concurrently with the scans, the copies and each other
// (each carve is latency bound on a few SMs).  Runs are independent, so the results do not
// depend on the grouping.
struct ClipJob {
  const uint8_t* frames_dev = nullptr;
  const uint8_t* frames_host = nullptr;
  uint8_t* out_dev = nullptr;
  uint8_t* out_host = nullptr;
  scpl_video_result* result = nullptr;
  int index = 0;
  // state
  const uint8_t* frames = nullptr;  // device frames
  uint8_t* out = nullptr;           // device output
  DBuf frames_buf, codes, out_buf;
  ScanStream scan;
  ScanLane* lane = nullptr;
  std::vector<cudaEvent_t> ev_chunk_codes, ev_chunk;
  cudaEvent_t ev_codes = nullptr, ev_scan = nullptr;
  std::vector<std::pair<int, int>> runs;
  int done = 0;  // runs considered for dispatch so far
  long dp = 0;
};

struct RunRef {
  ClipJob* job;
  int r;  // index into job->runs
};

struct Group {
  std::list<CarveSet> sets;  // one per carved axis, in phase order
  std::vector<int> axes;
  std::list<DBuf> bufs;
  std::vector<RunRef> runs;
  cudaStream_t st = nullptr;
};

// append one seam-dump record (include/scpl.h, scpl_video_result) for run R of a carve set
void dump_record(scpl_video_result* res, int run, int axis, const CarveRun& R) {
  const int rows = R.rows, cols = R.width0, iters = R.width0 > R.target ? R.iters : 0;
  const int removed = R.width0 > R.target ? R.removed : 0;
  auto pad8 = [](size_t x) { return (x + 7) & ~(size_t)7; };
  const size_t bytes = 32 + pad8(4 * (size_t)iters) + pad8(2 * (size_t)removed) + 8 * (size_t)removed +
                       pad8(2 * (size_t)rows * removed) + pad8(2 * (size_t)iters * cols);
  SCPL_ARG(res->seam_dump_used + bytes <= res->seam_dump_cap, "seam_dump buffer too small");
  uint8_t* p = static_cast<uint8_t*>(res->seam_dump) + res->seam_dump_used;
  std::memset(p, 0, bytes);
  const int32_t hdr[8] = {run, axis, rows, cols, iters, removed, 0, 0};
  std::memcpy(p, hdr, sizeof(hdr));
  p += 32;
  if (iters) SCPL_CUDA(cudaMemcpy(p, R.sizes, 4 * (size_t)iters, cudaMemcpyDeviceToHost));
  p += pad8(4 * (size_t)iters);
  if (removed) SCPL_CUDA(cudaMemcpy(p, R.cols, 2 * (size_t)removed, cudaMemcpyDeviceToHost));
  p += pad8(2 * (size_t)removed);
  if (removed) SCPL_CUDA(cudaMemcpy(p, R.costs, 8 * (size_t)removed, cudaMemcpyDeviceToHost));
  p += 8 * (size_t)removed;
  if (removed)  // the removed-column log is rows x rem_cap, rem_cap == removed
    SCPL_CUDA(cudaMemcpy2D(p, 2 * (size_t)removed, R.rem, 2 * (size_t)R.rem_cap, 2 * (size_t)removed, rows,
                           cudaMemcpyDeviceToHost));
  p += pad8(2 * (size_t)rows * removed);
  if (iters) SCPL_CUDA(cudaMemcpy(p, R.labs, 2 * (size_t)iters * cols, cudaMemcpyDeviceToHost));
  res->seam_dump_used += bytes;
}

void retarget_jobs(scpl_ctx* ctx, std::vector<ClipJob>& jobs, int T, int h, int w, int channels,
                   const scpl_video_params& P, cudaStream_t st) {
  const bool timeline = getenv("SCPL_TIMELINE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;  // (label, timing event)
  const auto t_host0 = std::chrono::steady_clock::now();
  auto hmark = [&](const std::string& label) {
    if (!timeline) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    fprintf(stderr, "host %8.3f ms  %s\n", ms, label.c_str());
  };
  const int njobs = (int)jobs.size();
  SCPL_ARG(njobs >= 1, "no clips");
  SCPL_ARG(channels == 1 || channels == 3, "unsupported channel count: expected 1 or 3");
  SCPL_ARG(h >= 3 && w >= 3, "frame too small to carve");
  SCPL_ARG(P.target_width >= 1 && P.target_width <= w, "target width out of range");
  SCPL_ARG(P.target_height >= 1 && P.target_height <= h, "target height out of range");
  SCPL_ARG(P.mode >= 0 && P.mode <= 2, "unknown mode");
  SCPL_ARG(P.max_len >= 1, "max_len must be >= 1");
  SCPL_ARG(P.mode != 2 || P.phi != nullptr, "phi table required for buffered mode");
  SCPL_ARG(P.shard_count <= 1 || (P.shard_rank >= 0 && P.shard_rank < P.shard_count),
           "shard_rank must be in 0 .. shard_count-1");
  SCPL_ARG(njobs == 1 || (P.shard_count <= 1 && P.runs_in == nullptr && !P.scan_only),
           "shard_*, runs_in and scan_only apply to single-clip calls");
  const bool buffered = P.mode == 2;
  const bool given = buffered && P.runs_in != nullptr;
  const bool scan_only = P.scan_only != 0;
  SCPL_ARG(!scan_only || (buffered && !given), "scan_only needs buffered mode without runs_in");
  if (given) {
    SCPL_ARG(P.n_runs_in >= 0, "n_runs_in must be >= 0");
    for (int r = 0; r < P.n_runs_in; ++r) {
      const int a = P.runs_in[2 * r], n = P.runs_in[2 * r + 1];
      SCPL_ARG(a >= 0 && n >= 1 && n <= P.max_len && a + n <= T, "runs_in: run out of range");
    }
  }
  const int shards = std::max(1, P.shard_count);
  for (auto& J : jobs) {
    scpl_video_result* result = J.result;
    result->dp_passes = 0;
    result->n_runs = 0;
    for (float& x : result->phase_ms) x = 0.f;
    for (long long& x : result->carve_cycles) x = 0;
    result->carve_cluster = 0;
    result->scan_windows = result->scan_fallbacks = 0;
    result->seam_dump_used = 0;
  }
  if (T <= 0) return;
  const int C = channels;
  const int tw = P.target_width, th = P.target_height;
  const size_t fbytes0 = (size_t)h * w * C;
  const bool host_in = jobs[0].frames_host != nullptr, host_out = jobs[0].out_host != nullptr;
  bool dump = false;
  for (auto& J : jobs) dump |= J.result->seam_dump != nullptr;
  // Priorities: the scans feed everything (they release the runs), so codes and scans get the
  // highest; carve groups are ordered by position in the batch (see dispatch) -- the carve
  // passes compete for whole SMs.  Levels: prio_hi (scan) .. prio_lo; carve groups use
  // prio_hi+1 .. prio_lo (or all if the range is tiny).
  if (!ctx->prio_known) {
    SCPL_CUDA(cudaDeviceGetStreamPriorityRange(&ctx->prio_lo, &ctx->prio_hi));
    ctx->prio_known = true;
  }
  const int prio_lo = ctx->prio_lo, prio_hi = ctx->prio_hi;
  for (cudaStream_t* x : {&ctx->s_h2d, &ctx->s_d2h})
    if (!*x) SCPL_CUDA(cudaStreamCreateWithFlags(x, cudaStreamNonBlocking));
  // Clips in flight: a batch's clips take the lanes in turn (clip j on lane j % L), so the
  // scans of later clips queue behind earlier ones on their lane while the earlier clips' runs
  // carve -- scans and carves overlap instead of running as two phases.
  int nlanes = njobs > 1 ? 8 : 1;
  if (const char* e = getenv("SCPL_LANES")) nlanes = std::max(1, atoi(e));
  nlanes = std::min(nlanes, njobs);
  while ((int)ctx->lanes.size() < nlanes) {
    ScanLane l;
    SCPL_CUDA(cudaStreamCreateWithPriority(&l.s_codes, cudaStreamNonBlocking, prio_hi));
    SCPL_CUDA(cudaStreamCreateWithPriority(&l.s_scan, cudaStreamNonBlocking, prio_hi));
    ctx->lanes.push_back(l);
  }
  for (int j = 0; j < njobs; ++j) {
    jobs[j].lane = &ctx->lanes[j % nlanes];
    jobs[j].index = j;
  }
  const int carve_hi = prio_lo - prio_hi >= 2 ? prio_hi + 1 : prio_hi;
  const int nlevels = prio_lo - carve_hi + 1;  // levels carve_hi .. prio_lo
  // Every group of a call gets a stream of its own (groups sharing a stream would carve one
  // after the other: measured, C2's last run waited ~7 ms for an earlier group that way), up to
  // kMaxStreamsPerLevel per priority level, created on demand.
  const int kMaxStreamsPerLevel = 16;
  if ((int)ctx->s_carve.size() < nlevels) ctx->s_carve.resize(nlevels);
  std::vector<int> used_at(nlevels, 0);
  // SCPL_CARVE_STREAMS=N (experiments): groups take N streams in turn instead (group g on stream
  // g % N, all at the carve priority), bounding how many groups carve at once
  static const int n_streams = getenv("SCPL_CARVE_STREAMS") ? std::max(1, atoi(getenv("SCPL_CARVE_STREAMS"))) : 0;
  int group_count = 0;
  auto carve_stream = [&](int level) {
    if (n_streams > 0) level = nlevels - 1;
    auto& v = ctx->s_carve[level];
    if (n_streams > 0) {
      const int k = group_count++ % n_streams;
      while ((int)v.size() <= k) {
        cudaStream_t x;
        SCPL_CUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, prio_lo - level));
        v.push_back(x);
      }
      return v[k];
    }
    const int k = used_at[level]++;
    if (k >= kMaxStreamsPerLevel) return v[k % kMaxStreamsPerLevel];
    if ((int)v.size() <= k) {
      cudaStream_t x;
      SCPL_CUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, prio_lo - level));  // 0 = lowest
      v.push_back(x);
    }
    return v[k];
  };
  std::vector<int> phases;  // 0 width, 1 height (pipeline.py:192-193, 246-277)
  if (!scan_only)
    for (int ax : (P.height_first ? std::vector<int>{1, 0} : std::vector<int>{0, 1})) {
      if (ax == 0 && tw < w) phases.push_back(0);
      if (ax == 1 && th < h) phases.push_back(1);
    }
  // chunks of 16 frames: a host clip's copies overlap its codes and scan, and a single clip's
  // runs reach the carve while its scan goes on; a batch of device clips is scanned clip by clip
  // in one piece (other clips' runs keep the carve busy; a chunk costs host API calls per clip)
  // SCPL_CHUNK=N (experiments): frames per chunk of a single / host clip
  static const int chunk_env = getenv("SCPL_CHUNK") ? std::max(1, atoi(getenv("SCPL_CHUNK"))) : 0;
  const int chunk = (njobs > 1 && !host_in) ? std::max(T, 1) : (chunk_env > 0 ? std::min(chunk_env, std::max(T, 1)) : 16);
  const int nchunk = (T + chunk - 1) / chunk;
  if (buffered && !given) upload_phi(ctx, P);

  // pinned scratch: scan readbacks, then per group and phase the carve-run states
  const size_t scan_pin = 64 + ((sizeof(int) * (nchunk + 2 * (size_t)T) + 63) & ~(size_t)63) + sizeof(ScanState) + 64;
  // (carve states: at most twice the runs per phase with the bucket padding, + 64 B per group)
  const size_t need = njobs * scan_pin + (2 * phases.size() + 1) * (size_t)T * njobs * (sizeof(CarveRun) + 64) +
                      4096 * (size_t)njobs;
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
  cudaEvent_t ev_start = new_event(true), ev_end = new_event(true);
  SCPL_CUDA(cudaEventRecord(ev_start, st));
  hmark("start recorded");

  // buffers (stream-ordered on st; every other stream waits for ev_alloc)
  for (auto& J : jobs) {
    J.frames = J.frames_dev;
    if (host_in) {
      J.frames_buf = DBuf(fbytes0 * T, st);
      J.frames = J.frames_buf.as<uint8_t>();
    }
    if (P.mode != 0) J.codes = DBuf(sizeof(uint16_t) * (size_t)T * h * w, st);
    J.out = J.out_dev;
    if (host_out && !scan_only) {
      J.out_buf = DBuf((size_t)T * th * tw * C, st);
      J.out = J.out_buf.as<uint8_t>();
    }
    if (buffered && !given) {
      J.scan.h_n = reinterpret_cast<int*>(pin_take(sizeof(int) * nchunk));
      J.scan.h_runs = reinterpret_cast<int*>(pin_take(sizeof(int) * 2 * (size_t)T));
      J.scan.h_state = reinterpret_cast<ScanState*>(pin_take(sizeof(ScanState)));
      J.scan.h_L = reinterpret_cast<int*>(pin_take(sizeof(int)));
    }
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

  // 1. frames in (host): every clip's chunks on the copy stream, clip by clip, so the first
  // clips' scans start first
  std::vector<std::vector<cudaEvent_t>> ev_h2d(njobs);
  if (host_in) {
    SCPL_CUDA(cudaStreamWaitEvent(ctx->s_h2d, ev_alloc, 0));
    for (auto& J : jobs)
      for (int c = 0; c < nchunk; ++c) {
        const int t0 = c * chunk, n = std::min(chunk, T - t0);
        SCPL_CUDA(cudaMemcpyAsync(const_cast<uint8_t*>(J.frames) + fbytes0 * t0, J.frames_host + fbytes0 * t0,
                                  fbytes0 * n, cudaMemcpyHostToDevice, ctx->s_h2d));
        if (njobs == 1) mark("h2d " + std::to_string(c), ctx->s_h2d);
        cudaEvent_t e = new_event(false);
        SCPL_CUDA(cudaEventRecord(e, ctx->s_h2d));
        ev_h2d[J.index].push_back(e);
      }
  }
  // 2. per clip, on its lane: energy codes chunk by chunk, then the buffer scan chunk by chunk
  // (each scan chunk waits for its codes; fixed one-frame runs for scpl / raw; given runs: no
  // scan).  A lane's scans run one clip after another (its scan state is reset in stream order).
  // A batch's clips are started lazily (at most two per lane ahead of the harvested ones): the
  // host's API calls for later clips then overlap the GPU work instead of delaying the first
  // dispatch.
  auto start_job = [&](ClipJob& J) {
    cudaStream_t sc = J.lane->s_codes;
    SCPL_CUDA(cudaStreamWaitEvent(sc, ev_alloc, 0));
    J.ev_chunk_codes.assign(nchunk, nullptr);
    for (int c = 0; c < nchunk; ++c) {
      const int t0 = c * chunk, n = std::min(chunk, T - t0);
      if (host_in) SCPL_CUDA(cudaStreamWaitEvent(sc, ev_h2d[J.index][c], 0));
      if (P.mode != 0) launch_codes(J.frames, nullptr, t0, n, h, w, C, J.codes.as<uint16_t>(), ctx->num_sms, sc);
      J.ev_chunk_codes[c] = new_event(false);
      SCPL_CUDA(cudaEventRecord(J.ev_chunk_codes[c], sc));
    }
    cudaStream_t ss = J.lane->s_scan;
    J.ev_codes = new_event(true);
    J.ev_scan = new_event(true);
    SCPL_CUDA(cudaStreamWaitEvent(ss, ev_alloc, 0));
    if (buffered && !given) scan_start(ctx, J.scan, *J.lane, J.codes.as<uint16_t>(), T, h, w, P, ss);
    SCPL_CUDA(cudaStreamWaitEvent(ss, J.ev_chunk_codes[0], 0));
    SCPL_CUDA(cudaEventRecord(J.ev_codes, ss));  // (first chunk's codes)
    J.ev_chunk.assign(nchunk, nullptr);
    if (buffered && !given) {
      for (int c = 0; c < nchunk; ++c) {
        SCPL_CUDA(cudaStreamWaitEvent(ss, J.ev_chunk_codes[c], 0));
        scan_chunk(J.scan, c, std::min(T, (c + 1) * chunk), ss);
        if (njobs == 1) mark("scan " + std::to_string(c), ss);
        J.ev_chunk[c] = new_event(false);
        SCPL_CUDA(cudaEventRecord(J.ev_chunk[c], ss));
      }
      scan_end(J.scan, ss);
    } else {
      SCPL_CUDA(cudaStreamWaitEvent(ss, J.ev_chunk_codes[nchunk - 1], 0));
    }
    SCPL_CUDA(cudaEventRecord(J.ev_scan, ss));
  };
  const bool polled = buffered && !given && !scan_only;
  const int ahead = 2 * nlanes;
  int started = 0;
  for (; started < njobs && (!polled || started < ahead); ++started) start_job(jobs[started]);

  // 3. carve + replay, one run group at a time as runs close
  const long total_frames = (long)T * njobs;
  auto dispatch = [&](std::vector<RunRef> rr, std::vector<cudaEvent_t> ready, bool final_group) {
    if (rr.empty()) return;
    std::sort(ready.begin(), ready.end());
    ready.erase(std::unique(ready.begin(), ready.end()), ready.end());
    Group& G = groups.emplace_back();
    G.runs = rr;
    const int gi = (int)groups.size() - 1;
    long covered = 0;
    for (auto& x : rr) covered += x.job->runs[x.r].second;
    {  // priority level by position in the batch
      const long pos = (long)rr[0].job->index * T + rr[0].job->runs[rr[0].r].first;
      int level = std::min(nlevels - 1, (int)(pos * nlevels / std::max(total_frames, 1L)));
      // device clips: every group competes for SMs once the scans are through, and the earliest
      // groups go first (measured ~2% faster on C2 than the other order, and equal priorities
      // are ~30% slower); a host clip's last group closes alone after the copies and is the
      // critical path, so there the later groups go first
      static const bool late_first = getenv("SCPL_PRIO_LATE") != nullptr;  // (experiments)
      if (!host_in && !late_first) level = nlevels - 1 - level;
      if (final_group) level = nlevels - 1;  // (the critical path: top carve priority)
      G.st = carve_stream(level);
    }
    cudaStream_t gs = G.st;
    SCPL_CUDA(cudaStreamWaitEvent(gs, ev_alloc, 0));
    for (cudaEvent_t e : ready) SCPL_CUDA(cudaStreamWaitEvent(gs, e, 0));
    const int nr = (int)rr.size();
    mark("group " + std::to_string(gi) + " start", gs);
    auto ship = [&](ClipJob* J, size_t off, size_t bytes) {  // D2H of finished output frames
      if (!host_out) return;
      cudaEvent_t e = new_event(false);
      SCPL_CUDA(cudaEventRecord(e, gs));
      SCPL_CUDA(cudaStreamWaitEvent(ctx->s_d2h, e, 0));
      SCPL_CUDA(cudaMemcpyAsync(J->out_host + off, J->out + off, bytes, cudaMemcpyDeviceToHost, ctx->s_d2h));
    };
    if (phases.empty()) {
      for (auto& x : rr) {
        const int s0 = x.job->runs[x.r].first, n = x.job->runs[x.r].second;
        SCPL_CUDA(cudaMemcpyAsync(x.job->out + fbytes0 * s0, x.job->frames + fbytes0 * s0, fbytes0 * n,
                                  cudaMemcpyDeviceToDevice, gs));
        ship(x.job, fbytes0 * s0, fbytes0 * n);
      }
      return;
    }
    // per run: where its current frames are (the clip, then the previous phase's buffer)
    std::vector<const uint8_t*> src(nr);
    for (int k = 0; k < nr; ++k) src[k] = rr[k].job->frames + fbytes0 * rr[k].job->runs[rr[k].r].first;
    int curH = h, curW = w;
    const double est = final_group ? (double)nr : (double)nr * total_frames / std::max(1L, covered);
    const int kc = carve_variant(est, (phases[0] == 1 ? h : w), ctx->num_sms);
    for (size_t ph = 0; ph < phases.size(); ++ph) {
      const bool height = phases[ph] == 1;
      const int rows = height ? curW : curH, cols = height ? curH : curW;
      const int target = height ? th : tw;
      const bool with_U = (ph == 0) && P.mode != 0;
      CarveSet& S = G.sets.emplace_back();
      G.axes.push_back(phases[ph]);
      hmark("group alloc");
      const bool rea = P.reaverage != 0 && P.mode != 0;  // raw mode ignores it (pipeline.py:120-132)
      std::vector<int> nfr;
      if (rea)
        for (auto& x : rr) nfr.push_back(x.job->runs[x.r].second);
      const int kcp = ph == 0 ? kc : carve_variant(est, cols, ctx->num_sms);
      carve_alloc(S, nr, rows, cols, target, P.mode == 0 ? 1 : 0, with_U, dump,
                  carve_cluster(kcp, nr, cols, ctx->num_sms), gs, rea ? nfr.data() : nullptr, rea, kcp);
      hmark("group setup");
      const size_t fbytes = (size_t)curH * curW * C;
      for (int k = 0; k < nr; ++k) {
        CarveRun& R = S.runs[k];
        ClipJob* J = rr[k].job;
        const int s0 = J->runs[rr[k].r].first;
        // the first carved axis works on the original frames, whose energy codes carry the
        // Sobel gradient of every frame (so the carve's gradient plane needs no recompute);
        // reaverage carves every frame of the run, otherwise its first frame represents it
        for (int f = 0; f < R.nfr; ++f) {
          const uint16_t* fcodes =
              (ph == 0 && P.mode != 0) ? J->codes.as<uint16_t>() + (size_t)(s0 + f) * h * w : nullptr;
          kc6::launch_run_setup(src[k] + fbytes * f, curH, curW, C, height ? 1 : 0, fcodes, R, gs, f);
        }
        if (with_U)
          launch_uniform(J->codes.as<uint16_t>(), h, w, s0, J->runs[rr[k].r].second, 1, P.w_motion, P.w_grad,
                         height ? 1 : 0, const_cast<double*>(R.U), gs, R.pitch);
      }
      mark("group " + std::to_string(gi) + " setup done", gs);
      hmark("group carve_launch");
      // (a batch's groups come in many sizes: their pooled graphs are shared per bucket; the
      // padding clusters cost a single clip's few group sizes more than they save)
      S.bucket = njobs > 1;
      carve_launch(ctx, S, pin_take(sizeof(CarveRun) * (S.bucket ? carve_bucket(nr) : nr) + 16), gs);
      hmark("group replay");
      mark("group " + std::to_string(gi) + " carve done", gs);
      const int nH = height ? th : curH, nW = height ? curW : tw;
      const bool last = ph + 1 == phases.size();
      const size_t obytes = (size_t)nH * nW * C;
      uint8_t* inter = nullptr;
      if (!last) inter = G.bufs.emplace_back((size_t)covered * obytes, gs).as<uint8_t>();
      size_t ioff = 0;
      for (int k = 0; k < nr; ++k) {
        const CarveRun& R = S.runs[k];
        ClipJob* J = rr[k].job;
        const int s0 = J->runs[rr[k].r].first, n = J->runs[rr[k].r].second;
        uint8_t* dst = last ? J->out + obytes * s0 : inter + ioff;
        launch_replay(src[k], dst, n, curH, curW, C, R.idx, R.pitch, target, height ? 1 : 0, gs);
        if (last) ship(J, obytes * s0, obytes * n);
        src[k] = dst;
        ioff += obytes * n;
      }
      mark("group " + std::to_string(gi) + " phase " + std::to_string(ph) + " runs " + std::to_string(nr), gs);
      curH = nH;
      curW = nW;
    }
    if (host_out) mark("d2h group " + std::to_string(gi), ctx->s_d2h);
  };
  // a single clip split across GPUs: runs go, as they close, to the least-loaded rank (every
  // rank sees the same run list, so every rank computes the same assignment); a run's cost is
  // dominated by its carve (about as long as replaying ~1000 frames), the length breaks ties
  std::vector<double> load(shards, 0.0);
  auto mine = [&](const std::pair<int, int>& run) {
    if (shards <= 1) return true;
    int best = 0;
    for (int k = 1; k < shards; ++k)
      if (load[k] < load[best]) best = k;
    load[best] += 1000.0 + run.second;
    return best == P.shard_rank;
  };
  if (scan_only) {
    // nothing to carve
  } else if (given) {
    ClipJob& J = jobs[0];
    for (int r = 0; r < P.n_runs_in; ++r) J.runs.push_back({P.runs_in[2 * r], P.runs_in[2 * r + 1]});
    std::vector<RunRef> rr;
    for (int r = 0; r < (int)J.runs.size(); ++r) rr.push_back({&J, r});
    dispatch(rr, {J.ev_scan}, true);
  } else if (buffered) {
    // host clips: every closed run goes out at once (the copies are the bottleneck); device
    // clips: groups of >= 4 runs (fewer, larger carve sets), >= 8 across a batch of clips
    // device clips: pairs of runs, but a run of >= 48 frames at once and short runs (< 8 frames
    // on average, e.g. a panning segment's 4-frame runs) as they close -- a group carves until its
    // slowest run is done (measured: C2 13.8 ms with singles vs 14.9 with groups of 4; C5 16.9 ms
    // with pairs vs 19.2 singles / 17.7 fours)
    int min_group = host_in ? 1 : (njobs > 1 ? 8 : 2);
    const bool fixed_min = getenv("SCPL_GROUP_MIN") != nullptr;
    if (fixed_min) min_group = std::max(1, atoi(getenv("SCPL_GROUP_MIN")));
    // a batch's closed runs go out in groups of at most max_group (each group's carve loop is
    // one serial chain of pass / row kernels: more groups, more chains in flight)
    int max_group = 1 << 30;
    if (const char* e = getenv("SCPL_GROUP_MAX")) max_group = std::max(1, atoi(e));
    // event-driven: harvest every clip's chunks as they complete (any order), dispatch groups
    std::vector<int> next(njobs, 0);
    int remaining = njobs * nchunk, harvested_jobs = 0;
    std::vector<RunRef> pending;
    std::vector<cudaEvent_t> ready;
    while (remaining > 0) {
      bool progress = false;
      for (int ji = 0; ji < started; ++ji) {
        ClipJob& J = jobs[ji];
        while (next[J.index] < nchunk) {
          const int c = next[J.index];
          const cudaError_t q = cudaEventQuery(J.ev_chunk[c]);
          if (q == cudaErrorNotReady) break;
          SCPL_CUDA(q);
          const int n = J.scan.h_n[c];
          for (int r = (int)J.runs.size(); r < n; ++r)
            J.runs.push_back({J.scan.h_runs[2 * r], J.scan.h_runs[2 * r + 1]});
          ++next[J.index];
          --remaining;
          progress = true;
          if (next[J.index] == nchunk) ++harvested_jobs;
          if (shards > 1) {  // this rank's runs (a single clip), each as it closes
            for (int r = J.done; r < (int)J.runs.size(); ++r)
              if (mine(J.runs[r])) dispatch({{&J, r}}, {J.ev_chunk[c]}, host_in && remaining == 0);
            J.done = (int)J.runs.size();
            continue;
          }
          for (int r = J.done; r < (int)J.runs.size(); ++r) {
            pending.push_back({&J, r});
            ready.push_back(J.ev_chunk[c]);
          }
          J.done = (int)J.runs.size();
        }
      }
      // (a device clip's scan ends long before its groups do: only a host clip's last group,
      // closed after the copies, carves with the GPU to itself)
      int want = min_group;
      if (!fixed_min && !host_in && njobs == 1 && !pending.empty()) {
        long fr = 0;
        int longest = 0;
        for (auto& x : pending) {
          fr += x.job->runs[x.r].second;
          longest = std::max(longest, x.job->runs[x.r].second);
        }
        // a long run goes at once (the clip's critical paths), so do bursts of short runs
        if (longest >= 48 || fr < 8L * (long)pending.size()) want = 1;
      }
      while ((int)pending.size() >= want || (remaining == 0 && !pending.empty())) {
        const size_t k = std::min(pending.size(), (size_t)max_group);
        std::vector<RunRef> grp(pending.begin(), pending.begin() + k);
        std::vector<cudaEvent_t> ev(ready.begin(), ready.begin() + k);
        pending.erase(pending.begin(), pending.begin() + k);
        ready.erase(ready.begin(), ready.begin() + k);
        // the clip's last group (closed by the end of the scan) is the critical path of a single
        // clip: SCPL_LAST_WIDE=1 carves it with the narrowest window at the top carve priority
        static const bool last_wide = getenv("SCPL_LAST_WIDE") != nullptr;
        const bool last = remaining == 0 && pending.empty() && njobs == 1;
        dispatch(grp, ev, last && (host_in || last_wide));
      }
      while (started < njobs && started < harvested_jobs + ahead) start_job(jobs[started++]);
      if (!progress && remaining > 0) std::this_thread::yield();
    }
  } else {
    ClipJob& J = jobs[0];
    std::vector<RunRef> rr;
    for (auto& Jx : jobs)
      for (int t = 0; t < T; ++t) Jx.runs.push_back({t, 1});
    // sharded: a contiguous block of frames per rank
    std::vector<cudaEvent_t> ready;
    for (auto& Jx : jobs) {
      const int a = njobs == 1 ? (int)((long)T * P.shard_rank / shards) : 0;
      const int b = njobs == 1 ? (int)((long)T * (P.shard_rank + 1) / shards) : T;
      for (int t = a; t < b; ++t) rr.push_back({&Jx, t});
      ready.push_back(Jx.ev_scan);
    }
    (void)J;
    dispatch(rr, ready, false);
  }
  for (auto& J : jobs) SCPL_CUDA(cudaStreamWaitEvent(st, J.ev_scan, 0));
  for (Group& G : groups) {
    cudaEvent_t e = new_event(false);
    SCPL_CUDA(cudaEventRecord(e, G.st));
    SCPL_CUDA(cudaStreamWaitEvent(st, e, 0));
  }
  if (host_out && !scan_only) {
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
  for (auto& J : jobs) {
    if (buffered && !given) {
      scan_finish(J.scan, nchunk, J.result);
      if (scan_only)  // every run of the scan
        for (int r = (int)J.runs.size(); r < J.scan.h_state->nruns; ++r)
          J.runs.push_back({J.scan.h_runs[2 * r], J.scan.h_runs[2 * r + 1]});
    }
    J.result->n_runs = (int)J.runs.size();
    if (J.result->run_start && J.result->run_len)
      for (size_t r = 0; r < J.runs.size(); ++r) {
        J.result->run_start[r] = J.runs[r].first;
        J.result->run_len[r] = J.runs[r].second;
      }
  }
  long pass_launches = 0;
  long long pass_cyc = 0, best_cyc = 0, best[3] = {0, 0, 0};
  int cluster = 0;
  for (Group& G : groups) {
    auto ax = G.axes.begin();
    for (CarveSet& S : G.sets) {
      carve_finish(S);
      long long slow = 0;
      int launches = 0;
      for (size_t k = 0; k < S.runs.size(); ++k) {
        const CarveRun& R = S.runs[k];
        ClipJob* J = G.runs[k].job;
        J->dp += R.iters;
        slow = std::max(slow, R.cyc_dp + R.cyc_sel);
        launches = std::max(launches, R.iters);
        if (J->result->seam_dump) dump_record(J->result, G.runs[k].r, *ax, R);
      }
      pass_cyc += slow;  // a launch lasts as long as its slowest cluster
      pass_launches += launches;
      if (S.prof[0] + S.prof[1] > best_cyc) {
        best_cyc = S.prof[0] + S.prof[1];
        for (int k = 0; k < 3; ++k) best[k] = S.prof[k];
      }
      cluster = S.cl;
      ++ax;
    }
  }
  float ms_end = 0.f;
  for (auto& m : marks) {
    float ms = 0.f;
    SCPL_CUDA(cudaEventElapsedTime(&ms, ev_start, m.second));
    fprintf(stderr, "timeline %8.3f ms  %s\n", ms, m.first.c_str());
  }
  SCPL_CUDA(cudaEventElapsedTime(&ms_end, ev_start, ev_end));
  for (auto& J : jobs) {
    scpl_video_result* res = J.result;
    res->dp_passes = J.dp;
    for (int k = 0; k < 3; ++k) res->carve_cycles[k] = best[k];
    res->carve_cycles[3] = pass_launches;
    res->carve_cluster = cluster;
    if (pass_launches > 0)
      res->phase_ms[3] = (float)((double)pass_cyc / pass_launches / std::max(ctx->clock_khz, 1));
    SCPL_CUDA(cudaEventElapsedTime(&res->phase_ms[0], ev_start, J.ev_codes));
    SCPL_CUDA(cudaEventElapsedTime(&res->phase_ms[1], J.ev_codes, J.ev_scan));
    float scan_end_ms = 0.f;
    SCPL_CUDA(cudaEventElapsedTime(&scan_end_ms, ev_start, J.ev_scan));
    res->phase_ms[2] = ms_end - scan_end_ms;
  }
  if (timeline) fprintf(stderr, "timeline %8.3f ms  end\n", ms_end);
  hmark("results");
}

void retarget_core(scpl_ctx* ctx, const uint8_t* frames_dev, const uint8_t* frames_host, int T, int h, int w,
                   int channels, const scpl_video_params& P, uint8_t* out_dev, uint8_t* out_host,
                   scpl_video_result* result, cudaStream_t st) {
  std::vector<ClipJob> jobs(1);
  jobs[0].frames_dev = frames_dev;
  jobs[0].frames_host = frames_host;
  jobs[0].out_dev = out_dev;
  jobs[0].out_host = out_host;
  jobs[0].result = result;
  retarget_jobs(ctx, jobs, T, h, w, channels, P, st);
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

int scpl_retarget_batch(scpl_ctx* ctx, int nclips, const uint8_t* const* clips, int T, int h, int w, int channels,
                        const scpl_video_params* params, uint8_t* const* outs, scpl_video_result* results,
                        int host_buffers, void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(params != nullptr && results != nullptr && clips != nullptr && outs != nullptr,
             "params/results/clips/outs is NULL");
    SCPL_ARG(nclips >= 1, "nclips must be >= 1");
    std::vector<ClipJob> jobs(nclips);
    for (int i = 0; i < nclips; ++i) {
      SCPL_ARG(clips[i] != nullptr && (outs[i] != nullptr || params->scan_only), "clip or output is NULL");
      (host_buffers ? jobs[i].frames_host : jobs[i].frames_dev) = clips[i];
      (host_buffers ? jobs[i].out_host : jobs[i].out_dev) = outs[i];
      jobs[i].result = &results[i];
    }
    retarget_jobs(ctx, jobs, T, h, w, channels, *params, (cudaStream_t)stream);
  });
}

int scpl_retarget_video_host(scpl_ctx* ctx, const uint8_t* frames, int T, int h, int w, int channels,
                             const scpl_video_params* params, uint8_t* out, scpl_video_result* result,
                             void* stream) {
  return guarded(ctx, [&] {
    SCPL_ARG(params != nullptr && result != nullptr, "params/result is NULL");
    SCPL_ARG(frames != nullptr && (out != nullptr || params->scan_only), "frames/out is NULL");
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
    SCPL_ARG(channels >= 1, "bytes per pixel must be >= 1");
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
