// Internal kernel launchers (not part of the C-ABI; see include/scpl.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace scpl {

constexpr int kPwDepth = 10;   // virtual complete tree depth for the pairwise fold
constexpr int kBlockRows = 16; // DP rows per 32-bit path word (2 bits per row)

struct PwVnode {
  int first_leaf;
  long n;  // 0 => contributes +0.0
};

void build_pairwise_plan(long N, std::vector<int2>& leaves, std::vector<PwVnode>& vnodes);

void launch_codes(const uint8_t* frames, const uint8_t* prev_frame, int T, int H, int W, int C,
                  uint16_t* codes, int num_sms, cudaStream_t st);
void launch_luma(const uint8_t* rgb, long npx, int C, uint8_t* out, cudaStream_t st);
void launch_decode(const uint16_t* codes, long per_frame, int T, int first_pure, double wm, double wg,
                   double* out, cudaStream_t st);
void launch_sobel_f64(const uint8_t* luma, int H, int W, double* out, cudaStream_t st);

void launch_window_stats(const uint16_t* codes, long N, const int2* leaves, int nleaves, int s, int n_acc,
                         int L, int first_pure, int init, double wm, double wg, double* ckS, double* ckQ,
                         double* leafsum, const PwVnode* vnodes, double* asde_out, cudaStream_t st);
void launch_uniform(const uint16_t* codes, int H, int W, int s, int n, int first_pure, double wm, double wg,
                    int transposed, double* out, cudaStream_t st);

// ------------------------------------------------------------------ carve state (one per run)
// Carve orientation: `rows` x `cols` where a vertical seam removes one column per row
// (for a height phase the planes are the transposed frame).  Planes have row stride
// `stride` (= the initial cols).
struct RunCarve {
  // static
  int rows, stride, target;
  int kmax;             // 0 = SCPL batch (k = remaining), 1 = raw (one min seam per pass)
  const double* U;      // fp64 energy for the first pass, or nullptr (gradient from the start)
  uint8_t* luma;        // rows x stride, compacted in place
  uint8_t* grad;        // rows x stride, gradient of the compacted luma
  int16_t* idx;         // rows x stride, original column of each current column
  uint32_t* pw;         // nblk x stride path words at block-end rows
  int8_t* delta;        // nblk x stride landing delta of each block-end column
  int16_t* col_end;     // nblk x stride block-end column of each last-row column's path
  int16_t* rem;         // rows x stride removed columns of the current batch (row-major, b per row)
  double* lastce;       // stride
  double* dbg_costs;    // optional: per batch costs (sum over batches <= stride) or nullptr
  int16_t* dbg_cols;    // optional: per batch last-row columns
  int* dbg_sizes;       // optional: per batch size
  // dynamic
  int width;            // current width
  int iters;            // DP passes done
  int b;                // size of the current batch
  int done;
  int nremoved;         // total removed so far (offset into dbg arrays)
};

void launch_carve_gradient(RunCarve* runs, int nruns, int max_rows, int max_stride, int first_iter,
                           cudaStream_t st);
void launch_carve_dp(RunCarve* runs, int nruns, bool fp64, int max_stride, cudaStream_t st);
void launch_carve_select(RunCarve* runs, int nruns, int max_stride, int max_rows, cudaStream_t st);
void launch_carve_compact(RunCarve* runs, int nruns, int max_rows, cudaStream_t st);
void launch_carve_setup_luma(const uint8_t* frame, int H, int W, int C, int transposed, uint8_t* luma,
                             int16_t* idx, cudaStream_t st);

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
                      const PwVnode* vnodes, double* leafsum, double* out, cudaStream_t st);

}  // namespace scpl
