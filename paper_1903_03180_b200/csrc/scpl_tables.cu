// API-level kernels behind the reference's lower-level functions (not on the hot path,
// which never materialises these tables):
//   cumulative_energy -> full (ce, back) tables          seams.py:39-65
//   label_parents     -> per-column chain over back       batching.py:39-46
//   select_batch      -> per-parent min, k-truncation, trace   batching.py:49-73
//   trace_columns     -> bottom-up walk                   seams.py:68-81
//   remove_batch      -> per-row compaction + disjointness count   batching.py:76-107
//   buffer sums / ASDE / std / mean on arbitrary float64 maps     buffering.py:93-176
#include <cfloat>
#include <climits>

#include "scpl_common.cuh"
#include "scpl_kernels.h"

namespace scpl {

// ------------------------------------------------------------------ DP tables
__global__ void __launch_bounds__(1024) dp_tables_kernel(const double* __restrict__ e, int h, int w,
                                                         double* __restrict__ ce, int8_t* __restrict__ back) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  for (int j = threadIdx.x; j < w; j += blockDim.x) {
    ce[j] = e[j];
    back[j] = 0;
  }
  __syncthreads();
  for (int i = 1; i < h; ++i) {
    const double* prv = ce + (long)(i - 1) * w;
    for (int j = threadIdx.x; j < w; j += blockDim.x) {
      double l = j > 0 ? prv[j - 1] : INF, c = prv[j], r = j + 1 < w ? prv[j + 1] : INF;
      int d = -1;
      double m = l;
      if (c < m) { m = c; d = 0; }
      if (r < m) { m = r; d = 1; }
      ce[(long)i * w + j] = __dadd_rn(e[(long)i * w + j], m);
      back[(long)i * w + j] = (int8_t)d;
    }
    __syncthreads();
  }
}

void launch_dp_tables(const double* e, int h, int w, double* ce, int8_t* back, cudaStream_t st) {
  dp_tables_kernel<<<1, 1024, 0, st>>>(e, h, w, ce, back);
  SCPL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ trace / labels
// cols (b) last-row columns -> offsets[s*h + i]
__global__ void trace_kernel(const int8_t* __restrict__ back, int h, int w, const long* __restrict__ cols, int b,
                             long* __restrict__ offsets) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= b) return;
  long c = cols[s];
  offsets[(long)s * h + h - 1] = c;
  for (int i = h - 1; i > 0; --i) {
    c += back[(long)i * w + c];
    offsets[(long)s * h + i - 1] = c;
  }
}

__global__ void labels_kernel(const int8_t* __restrict__ back, int h, int w, long* __restrict__ labels) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= w) return;
  long c = j;
  for (int i = h - 1; i > 0; --i) c += back[(long)i * w + c];
  labels[j] = c;
}

void launch_labels(const int8_t* back, int h, int w, long* labels, cudaStream_t st) {
  labels_kernel<<<cdiv(w, 128), 128, 0, st>>>(back, h, w, labels);
  SCPL_CHECK_LAUNCH();
}

void launch_trace(const int8_t* back, int h, int w, const long* cols, int b, long* offsets, cudaStream_t st) {
  if (b <= 0) return;
  trace_kernel<<<cdiv(b, 128), 128, 0, st>>>(back, h, w, cols, b, offsets);
  SCPL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ select (per-parent min + k)
// Single CTA. Outputs the selected last-row columns (ascending) and their costs.
__global__ void __launch_bounds__(1024) select_tables_kernel(const double* __restrict__ last,
                                                             const long* __restrict__ labels, int w, int k,
                                                             long* __restrict__ cols_out, double* __restrict__ costs_out,
                                                             int* __restrict__ nb_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  unsigned long long* segmin = reinterpret_cast<unsigned long long*>(smem);
  int* segarg = reinterpret_cast<int*>(segmin + w);
  int* cand = segarg + w;
  __shared__ int s_n;
  for (int j = threadIdx.x; j < w; j += blockDim.x) {
    segmin[j] = ~0ull;
    segarg[j] = INT_MAX;
  }
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < w; j += blockDim.x)
    atomicMin(&segmin[labels[j]], (unsigned long long)__double_as_longlong(last[j]));
  __syncthreads();
  for (int j = threadIdx.x; j < w; j += blockDim.x)
    if ((unsigned long long)__double_as_longlong(last[j]) == segmin[labels[j]]) atomicMin(&segarg[labels[j]], j);
  __syncthreads();
  if (threadIdx.x == 0) {  // candidates in label (== column) order; API path, serial is fine
    int n = 0;
    for (int l = 0; l < w; ++l)
      if (segarg[l] != INT_MAX) cand[n++] = segarg[l];
    s_n = n;
  }
  __syncthreads();
  const int P = s_n;
  const int kk = (k <= 0 || k > P) ? P : k;
  // rank by (cost, col); keep rank < kk
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    double cq = last[cand[q]];
    int rank = 0;
    for (int o = 0; o < P; ++o) {
      double co = last[cand[o]];
      rank += (co < cq) || (co == cq && o < q);
    }
    segarg[q] = rank < kk ? 1 : 0;  // reuse as keep flags
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int q = 0; q < P; ++q)
      if (segarg[q]) {
        cols_out[n] = cand[q];
        costs_out[n] = last[cand[q]];
        ++n;
      }
    *nb_out = n;
  }
}

void launch_select_tables(const double* last, const long* labels, int w, int k, long* cols, double* costs, int* nb,
                          cudaStream_t st) {
  size_t smem = (size_t)w * (8 + 4 + 4);
  SCPL_ARG(smem <= 227 * 1024, "map too wide for select_batch");
  smem_optin(reinterpret_cast<const void*>(select_tables_kernel));
  select_tables_kernel<<<1, 1024, smem, st>>>(last, labels, w, k, cols, costs, nb);
  SCPL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ remove columns
// out[i] = in[i] without columns offsets[s*h+i]; rowcount[i] = number of distinct removed
// columns in row i (the caller asserts it equals b, batching.py:104).
__global__ void remove_cols_kernel(const uint8_t* __restrict__ in, int h, int w, int C,
                                   const long* __restrict__ offsets, int b, uint8_t* __restrict__ out,
                                   int* __restrict__ rowcount) {
  extern __shared__ uint8_t mark[];
  const int i = blockIdx.x;
  for (int j = threadIdx.x; j < w; j += blockDim.x) mark[j] = 0;
  __syncthreads();
  for (int s = threadIdx.x; s < b; s += blockDim.x) mark[offsets[(long)s * h + i]] = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    int cnt = 0, y = 0;
    for (int j = 0; j < w; ++j) {
      if (mark[j]) {
        ++cnt;
        continue;
      }
      if (y < w - b)
        for (int c = 0; c < C; ++c) out[((long)i * (w - b) + y) * C + c] = in[((long)i * w + j) * C + c];
      ++y;
    }
    rowcount[i] = cnt;
  }
}

void launch_remove_cols(const uint8_t* in, int h, int w, int C, const long* offsets, int b, uint8_t* out,
                        int* rowcount, cudaStream_t st) {
  remove_cols_kernel<<<h, 128, w, st>>>(in, h, w, C, offsets, b, out, rowcount);
  SCPL_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ buffer statistics on float64 maps
__global__ void sums_kernel(const double* __restrict__ e, long N, const double* __restrict__ S_in,
                            const double* __restrict__ Q_in, double* __restrict__ S, double* __restrict__ Q) {
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < N; p += (long)gridDim.x * blockDim.x) {
    double x = e[p];
    double x2 = __dmul_rn(x, x);
    if (S_in) {
      S[p] = __dadd_rn(S_in[p], x);   // buffering.py:116-117
      Q[p] = __dadd_rn(Q_in[p], x2);
    } else {
      S[p] = x;                        // buffering.py:163-167
      Q[p] = x2;
    }
  }
}

void launch_sums(const double* e, long N, const double* S_in, const double* Q_in, double* S, double* Q,
                 cudaStream_t st) {
  int blocks = (int)std::min<long>(cdiv(N, 256), 148L * 8);
  sums_kernel<<<blocks, 256, 0, st>>>(e, N, S_in, Q_in, S, Q);
  SCPL_CHECK_LAUNCH();
}

__device__ __forceinline__ double std_of(double S, double Q, double n) {
  double m = __ddiv_rn(S, n);
  double var = __dsub_rn(__ddiv_rn(Q, n), __dmul_rn(m, m));
  return __dsqrt_rn(var >= 0.0 ? var : 0.0);
}

// what: 0 mean (S/n), 1 std
__global__ void sums_map_kernel(const double* __restrict__ S, const double* __restrict__ Q, long N, int n, int what,
                                double* __restrict__ out) {
  const double dn = (double)n;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < N; p += (long)gridDim.x * blockDim.x)
    out[p] = what == 0 ? __ddiv_rn(S[p], dn) : std_of(S[p], Q[p], dn);
}

void launch_sums_map(const double* S, const double* Q, long N, int n, int what, double* out, cudaStream_t st) {
  int blocks = (int)std::min<long>(cdiv(N, 256), 148L * 8);
  sums_map_kernel<<<blocks, 256, 0, st>>>(S, Q, N, n, what, out);
  SCPL_CHECK_LAUNCH();
}

// leaf sums of std(S,Q) with numpy's 8-accumulator pattern (one 8-lane group per leaf)
__global__ void sums_leaf_kernel(const double* __restrict__ S, const double* __restrict__ Q, const int2* leaves,
                                 int nleaves, int n, double* __restrict__ leafsum) {
  const int lane = threadIdx.x & 31, sub = lane & 7;
  const int leaf = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const bool active = leaf < nleaves;
  int2 lf = active ? leaves[leaf] : make_int2(0, 8);
  const int nmain = lf.y >> 3, ntail = lf.y & 7;
  const double dn = (double)n;
  double acc = 0.0, tail = 0.0;
  if (active) {
    for (int k = 0; k < nmain; ++k) {
      long p = lf.x + sub + 8 * k;
      double sd = std_of(S[p], Q[p], dn);
      acc = k == 0 ? sd : __dadd_rn(acc, sd);
    }
    if (sub < ntail) {
      long p = lf.x + 8 * nmain + sub;
      tail = std_of(S[p], Q[p], dn);
    }
  }
  double x = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
  x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 2));
  x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 4));
  const int g0 = lane & ~7;
  for (int k = 0; k < 7; ++k) {
    double tv = __shfl_sync(0xffffffffu, tail, g0 + k);
    if (k < ntail) x = __dadd_rn(x, tv);
  }
  if (active && sub == 0) leafsum[leaf] = x;
}

void launch_asde_sums(const double* S, const double* Q, long N, int n, const int2* leaves, int nleaves,
                      const PwVnode* vnodes, double* leafsum, double* partial, double* out, cudaStream_t st) {
  sums_leaf_kernel<<<cdiv((long)nleaves * 8, 256), 256, 0, st>>>(S, Q, leaves, nleaves, n, leafsum);
  SCPL_CHECK_LAUNCH();
  launch_pairwise_fold(leafsum, nleaves, vnodes, N, 1, partial, out, st);
}

}  // namespace scpl
