// Internal kernel launchers (not part of the C-ABI; see include/scpl.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace scpl {

constexpr int kPwDepth = 14;   // virtual complete tree depth for the pairwise fold
constexpr int kPwFoldCtas = 16;  // CTAs per candidate folding one depth-10 subtree each
constexpr int kBlockRows = 32; // DP rows per 64-bit path / choice word (2 bits per row)

struct PwVnode {
  int first_leaf;
  long n;  // 0 => contributes +0.0
};

void build_pairwise_plan(long N, std::vector<int2>& leaves, std::vector<PwVnode>& vnodes);

// codes of frames t0 .. t0+n-1 of the clip starting at `frames` into codes (frame 0 based);
// the frame before t0 is frames[t0-1], or prev_frame (nullable) when t0 == 0
void launch_codes(const uint8_t* frames, const uint8_t* prev_frame, int t0, int n, int H, int W, int C,
                  uint16_t* codes, int num_sms, cudaStream_t st);
void launch_luma(const uint8_t* rgb, long npx, int C, uint8_t* out, cudaStream_t st);
void launch_decode(const uint16_t* codes, long per_frame, int T, int first_pure, double wm, double wg,
                   double* out, cudaStream_t st);
void launch_sobel_f64(const uint8_t* luma, int H, int W, double* out, cudaStream_t st);
void launch_jitter_sums(const uint8_t* frames, int T, long npx, int C, unsigned long long* sums, cudaStream_t st);

void launch_window_stats(const uint16_t* codes, long N, const int2* leaves, int nleaves, int s, int n_acc,
                         int L, int first_pure, int init, double wm, double wg, double* ckS, double* ckQ,
                         double* leafsum, const PwVnode* vnodes, double* partial, double* asde_out,
                         cudaStream_t st);
// leaf sums (L x nleaves) -> L ASDE values; partial holds L x kPwFoldCtas doubles
void launch_pairwise_fold(const double* leafsum, int nleaves, const PwVnode* vnodes, long N, int L,
                          double* partial, double* out, cudaStream_t st);

// Device-side buffer scan state (scpl_stats.cu).  runs holds (start, len) pairs.
constexpr int kScanMaxL = 64;  // candidates per window (spec_len <= 64)
struct ScanState {
  const uint16_t* codes;
  long N;
  double *ckS, *ckQ;    // S, Q after the accepted frames (read by a window that continues a run)
  double *ckS2, *ckQ2;  // written by every window; swapped with ckS/ckQ when all its candidates pass
  double *leafsum, *partial;
  const double* phi;  // threshold(n), n = 0..max_len
  int* runs;
  double wm, wg;
  int T, max_len, spec, avail;
  int s, n_acc, init, L, done, nruns;
  int steps;      // loop-body executions (one window kernel each; its last CTA decides and plans)
  // Screened windows: a window is first evaluated by the cheap bounded kernel (approximate
  // ASDE + a rigorous bound on its distance to the reference's value); only a window with a
  // candidate whose threshold test the bound cannot settle is re-run exactly.
  int approx;     // screening enabled
  int exact;      // the current window runs the exact kernel (screening was inconclusive)
  int force_fallback;  // testing: treat every screened window as inconclusive
  int fallbacks;  // windows re-run exactly
  double asum[kScanMaxL], bsum[kScanMaxL];  // per candidate: sum of approximate std, of bounds
  unsigned int ticket;  // CTAs of the current window launch that are done (the last one decides)
};
cudaGraphExec_t build_scan_graph(ScanState* S, long N, const int2* leaves, int nleaves, const PwVnode* vnodes,
                                 int spec, int prio = 0);
void launch_scan_reset(ScanState* S, const ScanState& init, cudaStream_t st);
void launch_scan_avail(ScanState* S, int avail, cudaStream_t st);
void run_scan_host(ScanState* S, long N, const int2* leaves, int nleaves, const PwVnode* vnodes, int spec, int* h_L,
                   cudaStream_t st);
void launch_uniform(const uint16_t* codes, int H, int W, int s, int n, int first_pure, double wm, double wg,
                    int transposed, double* out, cudaStream_t st, int pitch = 0);

// ------------------------------------------------------------------ carve v2 (scpl_carve2.cu)
// One run's carve state; planes are rows x pitch (pitch >= width0, multiple of 16).
struct alignas(64) CarveRun {
  CUtensorMap tm_grad[2];  // 2-D TMA descriptors of the energy planes (DP windows, OOB -> 0)
  CUtensorMap tm_U;
  int rows, pitch, width0, target;
  int kmax;             // 0 = SCPL batch (k = remaining), 1 = raw (one min seam per pass)
  int nfr;              // frames carved together (reaverage_energy: the run's frames; else 1)
  int reaverage;        // every pass on U = mean gradient of the nfr carved frames (fp64 DP)
  long long fstride;    // bytes between consecutive frames' luma (and gradient) planes
  int stage_dtab;       // stage the landing-delta table in shared memory (set by the launcher)
  const double* U;      // fp64 energy of the first pass, or nullptr (gradient from the start)
  uint8_t* luma[2];     // luma plane(s) of the carved frame(s), compacted in place ([1] == [0])
  uint8_t* grad[2];     // their gradients (incrementally maintained; [1] == [0])
  int16_t* idx;         // output: original column of each kept column (rows x pitch)
  uint32_t* alive;      // rows x alive_pitch bitmask of surviving original columns
  int alive_pitch;
  int16_t* cend;        // nblk x pitch scratch: block-end columns of the selected seams
  long long* prof;      // optional (SCPL_PROF): detailed phase cycles
  uint64_t* pw;         // nblk x pitch path / choice words of each block (2 bits per row)
  int8_t* delta;        // nblk x pitch landing deltas
  double* lastce;       // pitch
  int16_t* rem;         // rows x rem_cap: removed columns of every batch, in that batch's coordinates
  int rem_cap;          // >= width0 - target
  int* sizes;           // optional per-batch sizes (capacity width0)
  int16_t* cols;        // optional per-seam last-row column (capacity width0)
  double* costs;        // optional per-seam cost
  int16_t* labs;        // optional (seam dump): parent labels of every pass, passes x width0
  // Fused int passes (fused != 0): the pass kernel's producer warps remove the previous batch
  // from the luma plane luma[lsel] while the DP runs, write the compacted rows to luma[lsel ^ 1]
  // and compute their Sobel energy straight into the DP's shared-memory ring (row stride
  // ring_w) -- no compaction / gradient kernels, no gradient plane.
  int fused;
  int ring_w;
  int lsel;
  int fdbg;             // (experiments: SCPL_FDBG timing variants of the producer; results invalid)
  // state (read at every kernel entry, advanced by the pass kernel)
  int width;            // current width
  int iters;            // DP passes done
  int removed;          // seams removed so far (offset of the next batch in the log)
  int b;                // size of the batch selected by the latest pass (0: none)
  long long cyc_dp, cyc_sel;  // SM cycles of the DP and select/trace phases, summed over passes
};
// Device-side carve loop plumbing: the iteration's last kernel sets the loop's condition
// (counters[0]: iterations executed)
struct RowsLoop {
  int max_iters;
  int* counters;
  cudaGraphConditionalHandle handle;
  // loop body only: the loop condition is evaluated on a side branch right after the pass (which
  // writes the widths), next to the row kernels instead of after them (SCPL_CHECK_FORK=0: after)
  cudaStream_t side = nullptr;
  cudaEvent_t e_fork = nullptr, e_join = nullptr;
};
// carve iterations per execution of the device-side loop's body (SCPL_CARVE_UNROLL; runs that are
// done skip every kernel, so the extra iterations of the last body are no-ops)
int carve_unroll();
// one carve iteration of some DP window variant (the fp64 first pass may use another variant)
using FirstIter = void (*)(CarveRun* runs_d, int nruns, int rows, int pitch, int width, int cl, cudaStream_t st,
                           int max_fr, bool reaverage, bool f64, const RowsLoop* loop, bool fused);
// carve launchers (scpl_carve2.cu), compiled once per DP window width: kc6 (default) and kc4
#define SCPL_CARVE_DECLS \
  void launch_run_setup(const uint8_t* frame, int H, int W, int C, int transposed, const uint16_t* codes, \
                        const CarveRun& R, cudaStream_t st, int f = 0); \
  void launch_carve_mean(CarveRun* runs_d, int nruns, int rows, cudaStream_t st); \
  int carve_cluster_size(int nruns, int width, int num_sms); \
  void encode_carve_tensor_maps(CarveRun& R); \
  void launch_carve_iteration(CarveRun* runs_d, int nruns, int rows, int pitch, int width, int cl, cudaStream_t st, \
                              int max_fr = 1, bool reaverage = false, bool f64 = false, \
                              const RowsLoop* loop = nullptr, bool fused = false); \
  void launch_carve_index(CarveRun* runs_d, int nruns, int rows, cudaStream_t st); \
  void launch_word_copy(void* dst, const void* src, size_t bytes, cudaStream_t st); \
  cudaGraphExec_t build_carve_loop(CarveRun* runs_d, int nruns, int rows, int pitch, int width, int cl, int max_iters, \
                                   int* iters_d, int max_fr = 1, bool reaverage = false, bool first_f64 = false, \
                                   FirstIter first = nullptr, int first_cl = 0, bool fused = false, \
                                   int prio = 0); \
  bool carve_fused_ok(int width0, int target, int cl); \
  int carve_fused_ring_w(int width0, int target, int cl); \
  void encode_carve_tensor_map_U(CarveRun& R); \
  bool carve_f64_fits_pair(int width, int cl); \
  bool carve_stage_dtab(int rows, int pitch, int cl); \
  int carve_kernels_per_iteration(bool reaverage); \
  int carve_warps(int width, int cl); \

namespace kc6 {
SCPL_CARVE_DECLS
}
namespace kc4 {
SCPL_CARVE_DECLS
}
namespace kc3 {
SCPL_CARVE_DECLS
}
#undef SCPL_CARVE_DECLS

void launch_replay(const uint8_t* in, uint8_t* out, int T, int H, int W, int C, const int16_t* idx, int stride,
                   int tw, int transposed, cudaStream_t st);

// API-level table kernels (scpl_tables.cu)
void launch_dp_tables(const double* e, int h, int w, double* ce, int8_t* back, cudaStream_t st);
void launch_labels(const int8_t* back, int h, int w, long* labels, cudaStream_t st);
void launch_trace(const int8_t* back, int h, int w, const long* cols, int b, long* offsets, cudaStream_t st);
void launch_select_tables(const double* last, const long* labels, int w, int k, long* cols, double* costs, int* nb,
                          cudaStream_t st);
void launch_remove_cols(const uint8_t* in, int h, int w, int C, const long* offsets, int b, uint8_t* out,
                        int* rowcount, cudaStream_t st);
void launch_sums(const double* e, long N, const double* S_in, const double* Q_in, double* S, double* Q,
                 cudaStream_t st);
void launch_sums_map(const double* S, const double* Q, long N, int n, int what, double* out, cudaStream_t st);
void launch_asde_sums(const double* S, const double* Q, long N, int n, const int2* leaves, int nleaves,
                      const PwVnode* vnodes, double* leafsum, double* partial, double* out, cudaStream_t st);

}  // namespace scpl
