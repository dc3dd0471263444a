/*
 * scpl.h -- C-ABI of libscpl.so, the sm_100a (B200) implementation of the buffered
 * seam-carving-with-parental-labeling (SCPL) video retargeting path of arXiv 1903.03180.
 *
 * The reference (`vidcarve` 0.1.0, /root/reference/pkg/src/vidcarve) is a pure-Python
 * package; its "operator API" is the Python function surface re-exported by
 * vidcarve/__init__.py:9-29.  It has no FFI layer, so each entry point below names the
 * reference function(s) it replaces; the Python package paper_1903_03180_b200 binds them
 * with ctypes and keeps the reference's signatures and errors.
 *
 * Conventions
 *   - Plain pointers and sizes; no torch types.  Pointers marked (dev) are CUDA device
 *     pointers owned by the caller; (host) are host pointers.  Frames are row-major
 *     (T, H, W, C) uint8 with C = 1 (gray) or 3 (RGB).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls enqueue work and
 *     return; results in device memory are valid once the stream has been synchronised.
 *     Entry points that return host results synchronise the stream themselves.
 *   - Return codes: 0 ok, 1 invalid argument (the Python layer raises ValueError with
 *     the message), 2 CUDA/runtime failure (RuntimeError).  scpl_last_error() returns a
 *     thread-local message for the last failing call.
 *   - One context per device; calls on a context are serialised by its owner.
 *   - Everything is bit-exact with the reference on the same inputs.
 */
#ifndef SCPL_H
#define SCPL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct scpl_ctx scpl_ctx;

int scpl_version(void);
long scpl_kernel_launches(void); /* kernels this library has launched so far (process-wide) */
const char* scpl_last_error(void);
int scpl_create(int device, scpl_ctx** out);
void scpl_destroy(scpl_ctx* ctx);

/* vidcarve.energy.to_luma (energy.py:23-37): luma_out[p] for npx pixels of `channels`
 * bytes each (3: BT.601 rint, bit-exact with the reference's float64 matmul; 1: copy). */
int scpl_to_luma(scpl_ctx* ctx, const uint8_t* pixels /*dev*/, long npx, int channels,
                 uint8_t* luma_out /*dev*/, void* stream);

/* vidcarve.energy.gradient_energy (energy.py:40-59): float64 (h,w) Sobel map. */
int scpl_gradient_energy(scpl_ctx* ctx, const uint8_t* luma /*dev h*w*/, int h, int w,
                         double* out /*dev h*w*/, void* stream);

/* Energy codes of a clip: codes[t][p] = |luma_t - luma_{t-1}| << 8 | sobel(luma_t).
 * `prev` (dev, nullable) is the frame before frames[0]; without it frame 0's motion
 * byte is 0 and consumers treat it as the stream's first frame (energy.py:79-80). */
int scpl_energy_codes(scpl_ctx* ctx, const uint8_t* frames /*dev*/, const uint8_t* prev /*dev|NULL*/,
                      int T, int h, int w, int channels, uint16_t* codes /*dev T*h*w*/, void* stream);

/* vidcarve.energy.motion_energy (energy.py:62-87) of codes: float64 maps for T frames;
 * first_pure=1 makes frame 0 the pure-gradient first frame. */
int scpl_decode_energy(scpl_ctx* ctx, const uint16_t* codes /*dev*/, int T, int h, int w, int first_pure,
                       double w_motion, double w_grad, double* out /*dev T*h*w*/, void* stream);

/* SpatioTemporalBuffer.push candidate test (buffering.py:115-119, 174-176): ASDE of the
 * windows [start, start+n) for n = n_acc+1 .. n_acc+count over the codes of frames
 * 0..T-1 (frame 0 = stream start).  state (dev, 2*h*w doubles) holds the per-pixel
 * sums S,Q of the accepted window: init=1 starts it from frame `start` (n_acc must be 1),
 * else it resumes; on return it holds the sums after n_acc+count frames.
 * asde_out (host, count doubles). */
int scpl_window_asde(scpl_ctx* ctx, const uint16_t* codes /*dev*/, int T, int h, int w, int start, int n_acc,
                     int count, double w_motion, double w_grad, double* state /*dev*/, int init,
                     double* asde_out /*host*/, void* stream);

/* FixedRun.uniform_energy (buffering.py:69-71): mean of frames [start, start+n)'s
 * motion energy, written (h,w) or transposed (w,h). */
int scpl_uniform_energy(scpl_ctx* ctx, const uint16_t* codes /*dev*/, int h, int w, int start, int n,
                        double w_motion, double w_grad, int transposed, double* out /*dev*/, void* stream);

/* vidcarve.batching.batch_carve (batching.py:118-153): carve `frame` (h,w,channels) to
 * `target` columns.  energy (dev h*w float64, nullable) is the first pass's map, later
 * passes use the gradient of the carved frame.  kmax=1 gives raw mode's one-seam-per-pass
 * loop (pipeline.py:229-243, min_seam).  Outputs:
 *   index_out (dev h*target int16): original column of each kept pixel per row;
 *   n_batches (host): number of DP passes;  batch_sizes (host, capacity w);
 *   batch_cols / batch_costs (host, capacity w): last-row column and cost of every seam,
 *   batches concatenated in order, columns ascending within a batch;
 *   offsets (host, capacity w*h, nullable): offsets[(seam)*h + row], same seam order. */
int scpl_batch_carve(scpl_ctx* ctx, const uint8_t* frame /*dev*/, int h, int w, int channels, int target,
                     const double* energy /*dev|NULL*/, int kmax, int16_t* index_out /*dev*/,
                     int* n_batches, int* batch_sizes, int16_t* batch_cols, double* batch_costs,
                     int16_t* offsets, void* stream);

/* replay_batches (pipeline.py:140-154) as one gather through a composed index map:
 * width: out[t][i][y] = in[t][i][index[i*stride+y]]             (transposed = 0)
 * height: out[t][y][j] = in[t][index[j*stride+y]][j]            (transposed = 1) */
int scpl_replay(scpl_ctx* ctx, const uint8_t* in /*dev*/, int T, int h, int w, int channels,
                const int16_t* index /*dev*/, int stride, int target, int transposed, uint8_t* out /*dev*/,
                void* stream);

typedef struct {
  int target_width;   /* <= w */
  int target_height;  /* <= h */
  int mode;           /* 0 raw, 1 scpl, 2 buffered (pipeline.py:39 MODES) */
  int height_first;
  int max_len;        /* BufferPolicy.max_len */
  double w_motion, w_grad;
  const double* phi;  /* host, max_len+1 entries: threshold(n, policy) as the reference computes it */
  int spec_len;       /* window candidates evaluated per stats launch (0 = default) */
  int reaverage;      /* RetargetConfig.reaverage_energy (pipeline.py:269-270, 280-296) */
  int shard_rank;     /* multi-GPU split of ONE clip: every rank computes the codes and */
  int shard_count;    /* the whole buffer scan, then carves and replays only its share of the runs
                         (longest-processing-time first over the closed runs, see sharding.py;
                         scpl/raw: a contiguous block of frames); other runs' output frames are
                         left untouched.  0 or 1: all runs */
  const int* runs_in; /* host, nullable (buffered mode): (start, len) pairs of runs found by an
                         earlier scan of the same clip (scan_only, or another rank).  The scan is
                         skipped and exactly these runs are carved and replayed (a rank's share
                         of a clip split across GPUs); other frames of out are left untouched */
  int n_runs_in;
  int scan_only;      /* 1: energy codes + buffer scan only (run boundaries in the result; out is
                         not written and may be NULL) */
} scpl_video_params;

typedef struct {
  long dp_passes;      /* RunMetrics.dp_passes */
  int n_runs;
  int* run_start;      /* host, capacity T (nullable) */
  int* run_len;        /* host, capacity T (nullable) */
  float phase_ms[4];   /* device ms: start -> codes done, -> scan done, scan done -> all carved and
                          replayed (groups overlap the scan), mean carve-pass launch duration (SM
                          clock cycles of the slowest cluster / base clock rate) */
  long long carve_cycles[4]; /* slowest run: dp cycles, select cycles, its pass count; then the
                                number of carve-pass kernel launches (dp_passes / launches = runs
                                per launch) */
  int carve_cluster;   /* CTAs per run cluster used by the carve */
  int scan_windows;    /* buffered: windows the buffer scan evaluated (screened or exact) */
  int scan_fallbacks;  /* buffered: screened windows re-run exactly (bound inconclusive) */
  /* Seam-dump parity mode (in: seam_dump, seam_dump_cap; out: seam_dump_used).  When seam_dump
   * (host) is set, every carved (run, axis) appends one record -- everything batch_carve
   * (batching.py:118-153) decides for that run's representative frame -- in little-endian
   * sections each padded to 8 bytes:
   *   int32 hdr[8] = {run, axis (0 width, 1 height), rows, cols, passes, removed, 0, 0}
   *   int32 sizes[passes]             batch sizes (SeamBatch lengths)
   *   int16 last_cols[removed]        last-row column of each seam, batches concatenated
   *   double costs[removed]           Seam.cost
   *   int16 offsets[rows][removed]    Seam.offsets (column per row, in the batch's frame)
   *   int16 labels[passes][cols]      label_parents of each pass (first source_width valid)
   * Records are in no particular order; the call fails (code 1) if seam_dump_cap is too small. */
  void* seam_dump;
  size_t seam_dump_cap;
  size_t seam_dump_used;
} scpl_video_result;

/* vidcarve.pipeline.retarget_video (pipeline.py:92-137), buffered / scpl / raw modes,
 * reaverage_energy = False: frames (dev T*h*w*channels) -> out (dev T*th*tw*channels). */
int scpl_retarget_video(scpl_ctx* ctx, const uint8_t* frames /*dev*/, int T, int h, int w, int channels,
                        const scpl_video_params* params, uint8_t* out /*dev*/, scpl_video_result* result,
                        void* stream);

/* Same call with HOST buffers (pinned for asynchronous copies): frames are copied in
 * 16-frame chunks on a copy stream while the energy codes and the buffer scan run on the
 * chunks already resident; each run's output frames are copied back on a second copy stream
 * as soon as the run is replayed.  Returns once out is complete. */
int scpl_retarget_video_host(scpl_ctx* ctx, const uint8_t* frames /*host*/, int T, int h, int w, int channels,
                             const scpl_video_params* params, uint8_t* out /*host*/, scpl_video_result* result,
                             void* stream);

/* Many independent clips in one call (BASELINE config C4: a batch of clips of one shape):
 * clips[i] (dev, or host when host_buffers = 1: pinned for asynchronous copies) ->
 * outs[i] (same kind), results[i] per clip.  Equivalent to one scpl_retarget_video(_host) call
 * per clip, but every clip's codes and buffer scan run at once and closed runs of all clips
 * share carve groups, so many runs are in flight on the GPU.  params is shared by all clips
 * (shard_* / runs_in / scan_only must be unset). */
int scpl_retarget_batch(scpl_ctx* ctx, int nclips, const uint8_t* const* clips, int T, int h, int w,
                        int channels, const scpl_video_params* params, uint8_t* const* outs,
                        scpl_video_result* results, int host_buffers, void* stream);

/* bench.jitter (bench.py:39-57): sums[t] = sum over pixels of |luma(t+1) - luma(t)| for
 * t < T-1 (exact integers; the caller divides by h*w and averages windows as the reference). */
int scpl_jitter_sums(scpl_ctx* ctx, const uint8_t* frames /*dev*/, int T, int h, int w, int channels,
                     unsigned long long* sums /*dev, T-1*/, void* stream);

/* ---- lower-level reference functions (API completeness; not on the hot path) ---- */

/* seams.cumulative_energy (seams.py:39-65): full float64 ce and int8 back tables. */
int scpl_cumulative_energy(scpl_ctx* ctx, const double* energy /*dev h*w*/, int h, int w, double* ce /*dev*/,
                           int8_t* back /*dev*/, void* stream);
/* batching.label_parents (batching.py:39-46): first-row landing column per last-row column. */
int scpl_label_parents(scpl_ctx* ctx, const int8_t* back /*dev*/, int h, int w, int64_t* labels /*dev w*/,
                       void* stream);
/* seams.trace_columns (seams.py:68-81): offsets[s*h + i] for b last-row columns. */
int scpl_trace_columns(scpl_ctx* ctx, const int8_t* back /*dev*/, int h, int w, const int64_t* cols /*dev b*/,
                       int b, int64_t* offsets /*dev b*h*/, void* stream);
/* batching.select_batch (batching.py:49-73) without the trace: selected last-row columns
 * (ascending, dev) and costs (dev); k <= 0 means unbounded; *nb (host) = batch size. */
int scpl_select_batch(scpl_ctx* ctx, const double* last_row /*dev w*/, const int64_t* labels /*dev w*/, int w,
                      int k, int64_t* cols /*dev*/, double* costs /*dev*/, int* nb /*host*/, void* stream);
/* batching.remove_batch / seams.remove_seam (batching.py:76-107, seams.py:92-105):
 * `channels` is the pixel size in bytes (any dtype: pixels move as raw bytes);
 * rowcount[i] (dev) = distinct removed columns in row i (caller asserts == b). */
int scpl_remove_columns(scpl_ctx* ctx, const uint8_t* in /*dev*/, int h, int w, int channels,
                        const int64_t* offsets /*dev b*h*/, int b, uint8_t* out /*dev h*(w-b)*channels*/,
                        int* rowcount /*dev h*/, void* stream);
/* SpatioTemporalBuffer accumulators on float64 maps (buffering.py:116-117, 163-167). */
int scpl_sums_start(scpl_ctx* ctx, const double* e, long n, double* S, double* Q, void* stream);
int scpl_sums_push(scpl_ctx* ctx, const double* e, long n, const double* S_in, const double* Q_in, double* S,
                   double* Q, void* stream);
/* what = 0: S/n (uniform_energy, buffering.py:158-161); 1: std map (:140-145). */
int scpl_sums_map(scpl_ctx* ctx, const double* S, const double* Q, long N, int n, int what, double* out,
                  void* stream);
/* _asde_from_sums (buffering.py:174-176), numpy pairwise mean; *out host. */
int scpl_asde_from_sums(scpl_ctx* ctx, const double* S, const double* Q, long N, int n, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
