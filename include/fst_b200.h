/*
 * fst_b200.h — C-ABI of the B200-native thresholded-Ax hot path
 * (arXiv 2105.05879; reference: /root/reference/proj/include/fst).
 *
 * Plain pointers and sizes only; no torch, no Eigen, no C++ types. Every entry
 * point names the reference interface it replaces (file:line, relative to
 * /root/reference/proj/include/fst/). The C++ mirror of the reference API
 * (`fst_b200.hpp`) and the Python mirror (`paper_2105_05879_b200/fst.py`) sit
 * on top of this header; INTEGRATION.md shows the binding a reference
 * maintainer would add.
 *
 * Residency: every `const void* X` / output pointer may be HOST or DEVICE
 * memory (detected with cudaPointerGetAttributes); device buffers are used in
 * place. Host buffers are copied in chunks (the end-to-end path) on two
 * copy streams, chunk i+1's input copy and kernel overlapping chunk i's
 * compute and output copy. The copies run straight from / to the caller's
 * buffers: page-locked (cudaHostAlloc / cudaHostRegister) host memory gets
 * fully asynchronous DMA; pageable memory still overlaps compute (each
 * chunk's output copy is issued only after the next chunk's kernel is
 * queued) but costs the driver's staging copy.
 *
 * Errors: every function returns an fstg_status; the message of the last
 * failure on the calling thread is returned by fstg_last_error(). There is no
 * CPU fallback: without a usable sm_100 device the compute entry points fail
 * with FSTG_ERR_CUDA.
 */
#ifndef FST_B200_H_
#define FST_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSTG_ABI_VERSION 1

/* Status codes map 1:1 onto the reference's exception classes. */
typedef enum fstg_status {
  FSTG_OK = 0,
  FSTG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (stream.hpp:30-38, sketch.hpp:152-153) */
  FSTG_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range (sketch.hpp:115, kerdock.hpp:122) */
  FSTG_ERR_OVERFLOW = 3,         /* std::overflow_error (stream.hpp:340-341) */
  FSTG_ERR_RUNTIME = 4,          /* std::runtime_error: allocation (sketch.hpp:162-165) */
  FSTG_ERR_CUDA = 5,             /* CUDA runtime failure / no sm_100 device */
  FSTG_ERR_NOT_SUPPORTED = 6,    /* shape outside this build's GPU limits */
  FSTG_ERR_IO = 7,               /* IoError (io.hpp:23): open/read/write failure */
  FSTG_ERR_MAGIC = 8,            /* MagicMismatchError (io.hpp:26) */
  FSTG_ERR_VERSION = 9,          /* VersionUnsupportedError (io.hpp:29) */
  FSTG_ERR_TRUNCATED = 10,       /* TruncatedPayloadError (io.hpp:32) */
  FSTG_ERR_MALFORMED = 11,       /* MalformedHeaderError (io.hpp:35) */
  FSTG_ERR_NO_MATRIX = 12        /* std::logic_error "Sketch: no embedded matrix" (sketch.hpp:109) */
} fstg_status;

typedef enum fstg_dtype { FSTG_F32 = 0, FSTG_F64 = 1 } fstg_dtype;

/* Arithmetic mode of the streaming estimator.
 *  FAST   : warp-parallel sample coefficients, FMA accumulation (fp32 default).
 *  STRICT : the reference's exact operation order — Gray-code sequential
 *           coefficient sums (stream.hpp:89-103), separately rounded
 *           multiply/add in j order (stream.hpp:232-234); bit-identical
 *           estimator and candidate set to the reference arithmetic (fp64
 *           default). */
typedef enum fstg_mode { FSTG_MODE_DEFAULT = 0, FSTG_MODE_FAST = 1, FSTG_MODE_STRICT = 2 } fstg_mode;

/* Mirrors fst::StreamParams (stream.hpp:22-39); `seed` is the per-call seed. */
typedef struct fstg_stream_params {
  double epsilon;
  double delta;
  int64_t s;
  int64_t J;
  int64_t K;
  int64_t widen;
  uint64_t seed;
  int32_t mode; /* fstg_mode */
  int32_t reserved;
} fstg_stream_params;

typedef struct fstg_sketch fstg_sketch; /* opaque; owns device buffers; immutable after create */

typedef struct fstg_sketch_info {
  int64_t m, n, d, L;         /* sketch.hpp:98-102 */
  int32_t k;
  int32_t dtype;              /* fstg_dtype */
  double row_norm_max;        /* sketch.hpp:105 */
  int32_t device;
  int32_t reserved;
  int64_t column_stride;      /* elements between consecutive columns (>= m, 16-byte multiple) */
  uint64_t device_bytes;      /* total HBM held by the sketch */
  double preprocess_ms;       /* device time of the last preprocess, CUDA events */
} fstg_sketch_info;

/* ---------------------------------------------------------------- misc ---- */
const char* fstg_last_error(void);
const char* fstg_version(void);
/* Number of usable sm_100 devices (0 when none; never falls back to CPU). */
int fstg_device_count(int* count);

/* ------------------------------------------- host-side design parameters -- */
/* sketch.hpp:58-63 even_log2_ceil */
int fstg_even_log2_ceil(int64_t n, int* k);
/* kerdock.hpp:26-31 DesignParams::make -> d, L */
int fstg_design_params(int k, int64_t* d, int64_t* L);
/* kerdock.hpp:55-84 kerdock_matrix: k rows, bit j of row i = entry (i,j) */
int fstg_kerdock_matrix(int k, uint64_t s, uint64_t* rows);
/* stream.hpp:58-69 choose_params */
int fstg_choose_params(double row_norm_max, double gamma, double eta, int64_t m, int64_t* J, int64_t* K);
/* stream.hpp:30-38 StreamParams::validate */
int fstg_validate_params(const fstg_stream_params* p);
/* stream.hpp:245-246 candidate count `want` */
int64_t fstg_candidate_count(int64_t s, int64_t widen, int64_t m);

/* ------------------------------------------------------- preprocessing ---- */
/* Replaces fst::preprocess (sketch.hpp:149-211). `a` is m x n row-major of
 * `dtype` (host or device). The sketch {A s_l}, column-major m x L, is built in
 * HBM on `device` by the in-shared-memory FWHT kernels; the embedded A is
 * kept for refinement. `stream` may be NULL (library stream). */
int fstg_preprocess(const void* a, int dtype, int64_t m, int64_t n, int device, void* stream,
                    fstg_sketch** out);
/* Builds only Kerdock bases [basis_begin, basis_end) (and the identity block
 * when include_identity != 0) into a full-size sketch: the basis-sharded
 * preprocessing of a multi-GPU replica. The columns of
 * the other bases are left unwritten; they are filled in place by the NVLink
 * all-gather (paper_2105_05879_b200/parallel.py) through
 * fstg_sketch_device_columns. */
int fstg_preprocess_shard(const void* a, int dtype, int64_t m, int64_t n, int device, void* stream,
                          int64_t basis_begin, int64_t basis_end, int include_identity, fstg_sketch** out);
/* Design-only sketch: embedded A + Kerdock tables, NO materialised columns —
 * for n where the m x L sketch cannot exist (n = 16384: 8.8 TB). Columns are
 * then produced on demand by fstg_sample_columns (retain-sampled
 * preprocessing) and consumed by
 * fstg_transform_gathered_batch. */
int fstg_preprocess_design(const void* a, int dtype, int64_t m, int64_t n, int device, void* stream,
                           fstg_sketch** out);
int fstg_sketch_info_get(const fstg_sketch* sk, fstg_sketch_info* info);
/* Sketch::row_norm_max (sketch.hpp:105) */
int fstg_row_norm_max(const fstg_sketch* sk, double* out);
/* sketch.hpp:107-111 Sketch::embedded_matrix: A (m x n row-major, the sketch's
 * dtype) into out (host or device); FSTG_ERR_NO_MATRIX without one. */
int fstg_sketch_embedded_matrix(const fstg_sketch* sk, void* out);
/* Sketch::column (sketch.hpp:114-117): copies column ell (m values) to `out`. */
int fstg_sketch_column(const fstg_sketch* sk, int64_t ell, void* out);
/* Raw device pointers (column-major, stride column_stride) for zero-copy use
 * by collectives (all-gather of basis shards) and tests. */
int fstg_sketch_device_columns(const fstg_sketch* sk, void** columns);
/* draw_and_gather (stream.hpp:184-191): copies columns indices[0..count) into
 * out (count x m, row j = column indices[j]); out may be host or device. */
int fstg_sketch_gather(const fstg_sketch* sk, const int64_t* indices, int64_t count, void* out, void* stream);
/* Retain-sampled preprocessing: computes only the requested columns A s_ell,
 * ell = indices[0..count), by running the FWHT over every Kerdock basis that
 * holds a request (requests radix-sorted by ell) and keeping the sampled
 * outputs; out is count x column_stride (device or host), column j at
 * j * column_stride — the draw_and_gather buffer of stream.hpp:184-191. Works
 * for design-only and materialised sketches (identical values). */
int fstg_sample_columns(const fstg_sketch* sk, const int64_t* indices, int64_t count, void* out, void* stream);
/* Device time of the last preprocess (ms, CUDA events). */
int fstg_sketch_preprocess_ms(const fstg_sketch* sk, double* ms);
void fstg_destroy(fstg_sketch* sk);

/* ---------------------------------------------------- FSTK persistence ---- */
/* save (sketch.hpp:213-232): FSTK, little-endian: "FSTK", u32 version, u64 m n
 * k d L, u8 hasEmbeddedA, L columns of m values, then the m x n row-major A.
 * version 1 = the reference's format (float64 payload; an fp32 sketch is
 * widened exactly), readable by fst::load. version 2 = the same layout with a
 * float32 payload (half the bytes; the reference rejects it with
 * VersionUnsupportedError). Columns stream device -> pinned host -> file. */
int fstg_save(const fstg_sketch* sk, const char* path, int version);
/* load (sketch.hpp:241-302) straight into HBM on `device`, with the
 * reference's header validation and error classes. `dtype` selects the
 * device representation (FSTG_F64 keeps a v1 payload as is; FSTG_F32 rounds it
 * to float32 on the GPU; a v2 file is always fp32). A file without an embedded
 * A loads, but transforms on it fail with FSTG_ERR_NO_MATRIX (sketch.hpp:109). */
int fstg_load(const char* path, int dtype, int device, void* stream, fstg_sketch** out);

/* ------------------------------------------------------------ streaming ---- */
/* draw_samples (stream.hpp:173-182) for B vectors: vector v uses seeds[v] in
 * place of p->seed. indices: B x (J*K) int64 (host or device). */
int fstg_draw_samples(const fstg_sketch* sk, const fstg_stream_params* p, const uint64_t* seeds, int64_t B,
                      int64_t* indices, void* stream);

/* transform (stream.hpp:272-275) over a batch of B vectors X (B x n row-major,
 * sketch dtype). Vector v draws its indices from seeds[v] (seeds == NULL ->
 * p->seed for every vector). Outputs (want = fstg_candidate_count):
 *   counts[B]            support size of each vector
 *   support[B x want]    sorted ascending support indices (first counts[v] valid)
 *   values[B x want]     exact (Ax)_i for the support, sketch dtype
 *   candidates[B x want] optional (NULL): the sorted candidate set
 *   mu[B x m]            optional (NULL): the median-of-means estimate
 * Any pointer may be host or device memory. */
int fstg_transform_batch(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                         const uint64_t* seeds, int32_t* counts, int32_t* support, void* values,
                         int32_t* candidates, void* mu, void* stream);

/* transform_with_samples (stream.hpp:197-268): as above with pre-drawn
 * indices (B x J*K int64, host or device) instead of seeds. */
int fstg_transform_with_samples_batch(const fstg_sketch* sk, const void* X, int64_t B,
                                      const fstg_stream_params* p, const int64_t* indices, int32_t* counts,
                                      int32_t* support, void* values, int32_t* candidates, void* mu,
                                      void* stream);

/* ------------------------------------------------- synthetic inputs (host) -- */
/* SeededRng(seed).gaussian() x count (reference rng.hpp:31-43, fill order of
 * generators.hpp:22-25). */
int fstg_gen_gaussian(uint64_t seed, int64_t count, double* out);
/* B target vectors y (B x m): s distinct rows by partial Fisher-Yates
 * (generators.hpp:44-53) valued +-1/sqrt(s) (value_kind 0) or N(0,1)
 * (value_kind 1), plus noise_sigma * N(0,1) on every entry. */
int fstg_gen_sparse_targets(const uint64_t* seeds, int64_t B, int64_t m, int64_t s, int value_kind,
                            double noise_sigma, double* Y);

/* gen_mixture's target draw (generators.hpp:60-78), unnormalised. */
int fstg_gen_mixture_targets(const uint64_t* seeds, int64_t B, int64_t m, double p, double* Y);

/* transform_with_samples with drawn.use_gathered (stream.hpp:197-268, 235-236):
 * vector v's sample j reads its column from gathered[(v * J*K + j) *
 * column_stride] (device memory, e.g. filled by fstg_sample_columns) instead of
 * the sketch; indices (B x J*K int64) still drive the coefficients. */
int fstg_transform_gathered_batch(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                                  const int64_t* indices, const void* gathered, int32_t* counts, int32_t* support,
                                  void* values, int32_t* candidates, void* mu, void* stream);

/* transform (stream.hpp:272-275) for a batch on a sketch whose columns need not
 * exist (fstg_preprocess_design; n = 16384): the draws, then per block of
 * row_block rows (0 = as many as ~70% of free device memory holds) the
 * retain-sampled FWHT of those rows of every sampled column and the estimator's
 * batch sums for those rows, then median / top-want / refinement. One Kerdock
 * pass per call; batch means bit-identical to fstg_transform_batch on the full
 * sketch. X, seeds and outputs in device memory. */
int fstg_transform_design_batch(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                                const uint64_t* seeds, int64_t row_block, int32_t* counts, int32_t* support,
                                void* values, int32_t* candidates, void* mu, void* stream);

/* The two halves of fstg_transform_design_batch, for row-sharded multi-GPU use:
 * rows [row_begin, row_end) of every vector's K batch means (vector v, batch b,
 * row r at means[v * vstride + b * ld + r - row_begin]; ld >= row_end - row_begin,
 * vstride >= K * ld), then median / top-want / refinement from complete means
 * (means[v * vstride + b * ld + row], ld >= m and a multiple of 16 bytes,
 * vstride >= (K + 1) * ld; slot K receives mu). Device memory. */
int fstg_design_partial_means(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                              const uint64_t* seeds, int64_t row_begin, int64_t row_end, int64_t row_block,
                              void* means, int64_t vstride, int64_t ld, void* stream);
int fstg_transform_from_means(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                              void* means, int64_t vstride, int64_t ld, int32_t* counts, int32_t* support, void* values,
                              int32_t* candidates, void* mu, void* stream);

/* ------------------------------------------------------- public helpers ---- */
/* The reference's smaller public functions on this path, as GPU kernels (host
 * or device pointers; device selects the GPU). */
/* stream.hpp:109-121 inner_product_with_design: s_ell^T x, the Kerdock case by
 * the reference's sequential Gray-code walk (bit-exact fp64). */
int fstg_inner_product_with_design(int k, const double* x, int64_t n, int64_t ell, double* out, int device);
/* stream.hpp:147-155 median_of_means: samples m x (J*K), column j at samples + j*m. */
int fstg_median_of_means(const double* samples, int64_t m, int64_t J, int64_t K, double* out, int device);
/* stream.hpp:158-162 hard_threshold (|t| = eps kept). */
int fstg_hard_threshold(const double* v, int64_t len, double eps, double* out, int device);
/* kerdock.hpp:156-167 projected_design_column: s_ell, n entries. */
int fstg_projected_design_column(int k, int64_t n, int64_t ell, double* out, int device);

/* ------------------------------------------------------ design verifiers --- */
/* kerdock.hpp:198-317, cli.hpp:45-82, on the GPU (sign tables of the design
 * expanded on `device`). All reported quantities are exact: every inner
 * product of unit design vectors is F/d with F an integer (one integer FWHT
 * per basis pair yields a whole cross Gram). Policies: */
#define FSTG_VERIFY_REFERENCE 0  /* the reference's: exhaustive for k <= 6, sampled above (same seeds/draws) */
#define FSTG_VERIFY_EXHAUSTIVE 1 /* every basis pair / every column pair for any k <= cap (k <= 14) */

/* kerdock.hpp:199-208 MubReport */
typedef struct fstg_mub_report {
  double max_within_gram_dev; /* max |B^T B - I| over every basis */
  double min_cross_sq;        /* extremes of squared cross-basis inner products */
  double max_cross_sq;
  double max_cross_dev;       /* max |<x,y>^2 - 1/d| */
  int32_t exhaustive;         /* 0 when basis pairs were sampled */
  int32_t reserved;
  int64_t basis_pairs;        /* cross-basis pairs checked */
} fstg_mub_report;

/* kerdock.hpp:261-266 MomentReport */
typedef struct fstg_moment_report {
  double m1;
  double m2;
  int32_t exact;              /* 0 for the sampled estimate */
  int32_t reserved;
  int64_t pairs;              /* ordered column pairs summed */
} fstg_moment_report;

/* kerdock.hpp:213-256 verify_mub. k > cap -> FSTG_ERR_INVALID_ARGUMENT
 * (the reference's invalid_argument); k > 14 -> FSTG_ERR_NOT_SUPPORTED. */
int fstg_verify_mub(int k, int cap, int policy, int device, fstg_mub_report* out);
/* kerdock.hpp:301-315 verify_design_moments (same errors). */
int fstg_verify_design_moments(int k, int cap, int policy, int device, fstg_moment_report* out);
/* kerdock.hpp:267-276 design_moment_target c_{d,k}. */
double fstg_design_moment_target(int64_t d, int k);
/* cli.hpp:45-60: every Kerdock matrix zero-diagonal and symmetric
 * (*skew_symmetric = 1), and the number of basis pairs a < b whose sum is
 * rank-deficient (must be 0). Ranks on the GPU. */
int fstg_verify_kerdock_set(int k, int device, int* skew_symmetric, int64_t* bad_pairs);

/* ------------------------------------------------------------ profiling ---- */
/* When enabled, the library brackets each launch of its kernels with CUDA
 * events on the launching stream; fstg_profile_read returns the accumulated
 * device milliseconds and launch count of kernel `name` ("preprocess_fwht",
 * "draw", "stream", ...) since the last reset. */
int fstg_profile_enable(int enable);
int fstg_profile_reset(void);
int fstg_profile_read(const char* name, double* ms, int64_t* launches);
/* Total kernel launches issued by the library since the last reset. */
int fstg_launch_count(int64_t* launches);

/* ----------------------------------------------------------- memory pool --- */
/* Calls with very large transient buffers (the design-only transforms: ~70% of
 * free HBM of retained columns) trim the library's stream-ordered pool on
 * return so the caller can allocate that HBM again (default, retain = 0). With
 * retain = 1 the pool keeps them cached for the next call: a stream of
 * design-only batches then skips re-mapping ~100 GB per call (config 4:
 * 4.8 -> 2.5 s per 8192-vector step), at the cost of that HBM staying reserved
 * until retain is cleared (which trims at once). Process-wide. */
int fstg_set_pool_retain(int retain);

#ifdef __cplusplus
}
#endif

#endif /* FST_B200_H_ */
