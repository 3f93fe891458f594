// Launch wrappers of the sm_100a kernels (preprocess.cu, draw.cu, stream.cu, verify.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fstg {

// ---- preprocessing (preprocess.cu) ----
cudaError_t launch_qtables(const uint32_t* revtab, int k, int64_t nbases, uint32_t* qplain, uint32_t* qtrans,
                           cudaStream_t st);
template <typename T>
cudaError_t launch_fwht_sketch(int k, const T* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                               int64_t basis_begin, int64_t basis_end, T* cols, int64_t ldc, cudaStream_t st);
// Retain-sampled FWHT: only requested columns (sorted by ell; basis s owns
// [req_start[s], req_start[s+1])) are written, to out[req_pos[r] * ldc], for
// rows [row0, m) (row i lands at out[... + i - row0]). req_rec (optional, the
// fp32 k = 12 / 14 kernels) holds the same requests packed as (w = ell mod d,
// slot) u32 pairs; those kernels prefetch the next basis' records into shared
// memory while transforming the current one.
template <typename T>
cudaError_t launch_fwht_retain(int k, const T* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                               int64_t nbases, T* out, int64_t ldc, const int64_t* req_start, const int64_t* req_ell,
                               const int64_t* req_pos, cudaStream_t st, int64_t row0 = 0,
                               const uint2* req_rec = nullptr);
template <typename T>
cudaError_t launch_identity(const T* a, int64_t lda, int64_t m, int64_t n, int64_t d, int64_t nk, T* cols,
                            int64_t ldc, cudaStream_t st);
template <typename T>
cudaError_t launch_row_norms(const T* a, int64_t lda, int64_t m, int64_t n, double* out, cudaStream_t st);

// Experiment readout of the stream kernel's per-role mbarrier wait cycles
// (FSTG_STREAM_DEBUG bit 8; 14 counters, see stream.cu WaitSite); resets them.
void stream_wait_profile(unsigned long long* out, int count);

// ---- design verifiers (verify.cu) ----
// Per basis pair (explicit list, or pb == nullptr: the upper triangle incl.
// the diagonal) the d-point integer FWHT of (-1)^(Q_b + Q_b2): acc (8 u64 =
// 4 u128) += {sum F^2 within, sum F^4 within, sum F^2 cross, sum F^4 cross};
// stats = {max |F - d delta| within, min F^2 cross, max F^2 cross}.
cudaError_t launch_verify_pairs(int k, const uint32_t* qplain, int64_t nk, int64_t npairs, const int32_t* pb,
                                const int32_t* pb2, unsigned long long* acc, int* stats, cudaStream_t st);
// Sampled column pairs (ia[i], ib[i]): acc (4 u64) += {sum F^2, sum F^4}, F = d <u_a, u_b>.
cudaError_t launch_verify_samples(int k, const uint32_t* qplain, const int64_t* ia, const int64_t* ib, int64_t count,
                                  unsigned long long* acc, cudaStream_t st);
// Pairs a < b of Kerdock matrices (nk x k row words) whose sum has rank < k.
cudaError_t launch_verify_ranks(int k, const uint32_t* rows, int64_t nk, unsigned long long* bad, cudaStream_t st);

// ---- public helpers (helpers.cu): stream.hpp:86-162, kerdock.hpp:156-167 ----
cudaError_t launch_inner_product(const double* x, int64_t n, int64_t d, const uint32_t* rev, uint64_t wpos,
                                 double* out, cudaStream_t st);
cudaError_t launch_median_of_means(const double* samples, int64_t m, int64_t J, int64_t K, double* out,
                                   cudaStream_t st);
cudaError_t launch_hard_threshold(const double* v, int64_t len, double eps, double* out, cudaStream_t st);
cudaError_t launch_design_column(int64_t n, int64_t d, int identity, const uint32_t* rev, int k, uint64_t wpos,
                                 double sqrt_d, double* out, cudaStream_t st);

// ---- draws (draw.cu) ----
template <typename IdxT>
cudaError_t launch_draw(const uint64_t* seeds, uint64_t seed_base, int64_t B, int64_t N, uint64_t L, IdxT* out,
                        cudaStream_t st);
cudaError_t launch_narrow_indices(const int64_t* in, int64_t count, int64_t L, uint32_t* out, int* bad,
                                  cudaStream_t st);

// ---- streaming estimator (stream.cu) ----
template <typename T>
struct StreamArgs {
  // sketch
  const T* cols;
  int64_t ldc;  // column stride (elements), multiple of 16 bytes
  const T* a;
  int64_t lda;  // row stride of the embedded A (elements), multiple of 16 bytes
  // fp32 only: bf16 (RN) copy of A for the refinement's screening pass, row stride ldab
  // (elements, multiple of 8); null = screen on the fp32 rows (or no screening, debug bit 16)
  const uint16_t* ab;
  int64_t ldab;
  const float* abn;  // |ab row i|_2, rounded up (with ab)
  const uint32_t* qplain;
  const uint32_t* qtrans;
  const uint32_t* revtab;
  int k;
  int64_t d, L, m, n, kb;  // kb = (d/2)*d, first identity index
  // params
  int64_t J, K, N;
  int64_t want;
  double epsilon;
  // batch
  const T* X;
  int64_t ldx;
  const uint32_t* idx;  // B x N
  const T* gathered;    // optional: B x N x ldc columns (draw_and_gather buffer); null -> cols + ell * ldc
  int64_t B;
  // outputs (device)
  int32_t* counts;
  int32_t* support;  // B x want
  T* values;         // B x want
  int32_t* cands;    // optional B x want
  T* mu;             // optional B x m
  // scratch: gridDim.x x 2 slots x (K + 1) x m_pad (batch means + mu)
  T* means;
  int64_t m_pad;
  // pipeline
  int stages;
  int stage_stride;  // bytes between ring stages (>= one segment, 128-byte multiple)
  int rstride;       // bytes per refinement-ring stage (one row of A); 0 = direct loads
  int rstages;       // refinement-ring stages in use (<= kRStages), set by stream_grid_size
  int rrows;         // rows per refinement-ring stage (2 for bf16 screening rows), set by stream_grid_size
  int xbufs;         // x buffers in shared memory
  int nseg;
  int chunk;
  // Row-blocked design-only transform (fstg_transform_design_batch):
  //   kMeansFull    the whole pipeline (default)
  //   kMeansPartial columns hold rows [row0, row0 + m) only (m_pad = their padded height);
  //                 the batch means of those rows go to means_io, no tail
  //   kMeansTail    no columns: median / select / refinement from means_io (m_pad = m_io)
  // means_io: B x (K + 1) x m_io (K batch means, then mu written by the tail).
  int means_mode;
  T* means_io;
  int64_t m_io, row0;
  int64_t means_vstride;  // elements between vectors in means_io (0: (K + 1) * m_io)
  // With kMeansPartial: 1 = every (vector, batch) pair is its own work item (small batches:
  // B < #SMs), item w = v * K + b covering samples [b * J, (b + 1) * J) of vector v.
  int batch_split;
  // experiment switches (env FSTG_STREAM_DEBUG; 0 in production):
  // bit 0: column pipeline only (coefficient warps idle, t = 1)
  // bit 1: coefficient pipeline only (no column loads, consumers skip the ring)
  // bit 2: no refinement; bit 3: per-role mbarrier wait profile; bit 4: no screening;
  // bit 5: no exact dots after screening; bit 6: screening rows loaded but not screened
  int debug;
};
enum MeansMode { kMeansFull = 0, kMeansPartial = 1, kMeansTail = 2 };

template <typename T>
cudaError_t launch_stream(const StreamArgs<T>& args, bool strict, int grid, cudaStream_t st);
// Elements of the `means` scratch the kernel needs for `grid` CTAs.
template <typename T>
int64_t stream_scratch_elems(const StreamArgs<T>& args, int grid);
// Persistent grid size the stream kernel wants for this configuration.
template <typename T>
int stream_grid_size(StreamArgs<T>& args, bool strict, int64_t B, size_t* smem_bytes, int* stages,
                     int* stage_stride, int* rstride, int* xbufs);

}  // namespace fstg
