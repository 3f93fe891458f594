// C-ABI implementation (include/fst_b200.h): sketch lifetime, batching,
// host<->device staging and profiling around the sm_100a kernels.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <limits>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/fst_b200.h"
#include "design.hpp"
#include "kernels.hpp"

using namespace fstg;

struct fstg_sketch {
  int device = 0;
  int dtype = FSTG_F32;
  Design design;
  int64_t m = 0, n = 0, ldc = 0, lda = 0;
  void* cols = nullptr;
  void* a = nullptr;
  uint16_t* ab = nullptr;  // fp32 sketches: bf16 (RN) copy of A for the refinement screening, row stride ldab
  int64_t ldab = 0;
  float* abn = nullptr;    // |ab row|_2 rounded up (the screening bound)
  uint32_t* qplain = nullptr;
  uint32_t* qtrans = nullptr;
  uint32_t* revtab = nullptr;
  double row_norm_max = 0;
  double preprocess_ms = 0;
  uint64_t device_bytes = 0;
  bool has_a = true;  // false for an FSTK file saved without the embedded A
};

namespace {

thread_local std::string g_error;

// IoError family (io.hpp:23-37) and the reference's logic_error for a sketch
// without its embedded matrix (sketch.hpp:109), each with its status code.
struct CodedError : std::runtime_error {
  int code;
  CodedError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

int set_error(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return FSTG_OK;
  } catch (const CodedError& e) {
    return set_error(e.code, e.what());
  } catch (const InvalidArgument& e) {
    return set_error(FSTG_ERR_INVALID_ARGUMENT, e.what());
  } catch (const OutOfRange& e) {
    return set_error(FSTG_ERR_OUT_OF_RANGE, e.what());
  } catch (const Overflow& e) {
    return set_error(FSTG_ERR_OVERFLOW, e.what());
  } catch (const NotSupported& e) {
    return set_error(FSTG_ERR_NOT_SUPPORTED, e.what());
  } catch (const CudaError& e) {
    return set_error(FSTG_ERR_CUDA, e.what());
  } catch (const std::invalid_argument& e) {
    return set_error(FSTG_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::out_of_range& e) {
    return set_error(FSTG_ERR_OUT_OF_RANGE, e.what());
  } catch (const std::overflow_error& e) {
    return set_error(FSTG_ERR_OVERFLOW, e.what());
  } catch (const std::bad_alloc& e) {
    return set_error(FSTG_ERR_RUNTIME, e.what());
  } catch (const std::runtime_error& e) {
    return set_error(FSTG_ERR_RUNTIME, e.what());
  } catch (const std::exception& e) {
    return set_error(FSTG_ERR_RUNTIME, e.what());
  }
}

// ------------------------------------------------------------ profiling ----
struct ProfEntry {
  double ms = 0;
  int64_t launches = 0;
};
struct PendingEvent {
  std::string name;
  cudaEvent_t start, stop;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::map<std::string, ProfEntry> g_prof;
std::vector<PendingEvent> g_pending;
std::atomic<int64_t> g_launches{0};

void resolve_pending_locked() {
  for (auto& p : g_pending) {
    float ms = 0;
    if (cudaEventSynchronize(p.stop) == cudaSuccess && cudaEventElapsedTime(&ms, p.start, p.stop) == cudaSuccess) {
      auto& e = g_prof[p.name];
      e.ms += ms;
      e.launches += 1;
    }
    cudaEventDestroy(p.start);
    cudaEventDestroy(p.stop);
  }
  g_pending.clear();
}

// RAII bracket around one kernel launch.
class ProfScope {
 public:
  ProfScope(const char* name, cudaStream_t st) : name_(name), st_(st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    on_ = g_prof_on;
    if (on_) {
      cudaEventCreate(&start_);
      cudaEventCreate(&stop_);
      cudaEventRecord(start_, st_);
    }
  }
  ~ProfScope() {
    if (!on_) return;
    cudaEventRecord(stop_, st_);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_pending.push_back({name_, start_, stop_});
  }

 private:
  std::string name_;
  cudaStream_t st_;
  bool on_ = false;
  cudaEvent_t start_{}, stop_{};
};

// ------------------------------------------------------------- helpers ----
bool is_device_ptr(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

void require_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw CudaError("no CUDA device available (this library has no CPU fallback)");
  }
  if (device < 0 || device >= count) throw InvalidArgument("device ordinal out of range");
  cudaDeviceProp prop{};
  cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10) throw CudaError("device is not sm_100 (B200); kernels are built for sm_100a only");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
}

size_t dtype_size(int dtype) {
  if (dtype == FSTG_F32) return 4;
  if (dtype == FSTG_F64) return 8;
  throw InvalidArgument("dtype must be FSTG_F32 or FSTG_F64");
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

void validate(const fstg_stream_params* p) {
  // stream.hpp:30-38
  if (p == nullptr) throw InvalidArgument("StreamParams: null");
  if (!(p->epsilon > p->delta) || p->delta < 0) throw InvalidArgument("StreamParams: need epsilon > delta >= 0");
  if (p->s < 1) throw InvalidArgument("StreamParams: need s >= 1");
  if (p->J < 1 || p->K < 1) throw InvalidArgument("StreamParams: need J, K >= 1");
  if (p->widen < 1) throw InvalidArgument("StreamParams: need widen >= 1");
  if (p->J > INT64_MAX / p->K) throw Overflow("StreamParams: J*K overflows");
}

__global__ void finite_check_kernel(const void* a, int dtype, int64_t count, int* bad) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    const double v = dtype == FSTG_F64 ? static_cast<const double*>(a)[i] : double(static_cast<const float*>(a)[i]);
    if (!isfinite(v)) atomicExch(bad, 1);
  }
}

// bf16 screening table (stream.cu refine_screen_bf16): ab[i, j] = RN_bf16(a[i, j]), padding zeroed
__global__ void bf16_table_kernel(const float* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                  uint16_t* __restrict__ ab, int64_t ldab) {
  const int64_t total = m * ldab;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / ldab, j = t % ldab;
    const __nv_bfloat16 h = __float2bfloat16_rn(j < n ? a[i * lda + j] : 0.f);
    ab[t] = __bfloat16_as_ushort(h);
  }
}

// |ab row i|_2 in fp64, rounded up to fp32 (one warp per row)
__global__ void bf16_row_norms_kernel(const uint16_t* __restrict__ ab, int64_t ldab, int64_t m, float* __restrict__ out) {
  const int lane = threadIdx.x % 32;
  for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) / 32; i < m;
       i += int64_t(gridDim.x) * blockDim.x / 32) {
    double s = 0.0;
    for (int64_t j = lane; j < ldab; j += 32) {
      const double v = static_cast<double>(__uint_as_float(static_cast<uint32_t>(ab[i * ldab + j]) << 16));
      s = fma(v, v, s);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[i] = __double2float_ru(sqrt(s) * (1.0 + 0x1.0p-40));
  }
}

template <typename T>
__global__ void gather_kernel(const T* __restrict__ cols, int64_t ldc, int64_t m, const int64_t* __restrict__ idx,
                              int64_t count, int64_t L, T* __restrict__ out, int* __restrict__ bad) {
  for (int64_t j = blockIdx.x; j < count; j += gridDim.x) {
    const int64_t ell = idx[j];
    if (ell < 0 || ell >= L) {
      if (threadIdx.x == 0) atomicExch(bad, 1);
      continue;
    }
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) out[j * m + i] = cols[ell * ldc + i];
  }
}

// Per-call scratch comes from the device's stream-ordered pool. The pool's
// release threshold is raised once per device so memory freed at the end of a
// call stays cached for the next one (the default threshold returns it to the
// driver at every synchronisation, which made every step re-allocate).
void keep_pool_warm(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t threshold = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  cudaGetLastError();
  done.push_back(device);
}

// After calls whose transient buffers were large (retained columns: ~100 GB), give the
// pool's free blocks back so the caller's own allocations do not find HBM reserved.
std::atomic<bool> g_pool_retain{false};  // fstg_set_pool_retain

void trim_pool(int device, cudaStream_t st, size_t keep = size_t(4) << 30) {
  if (g_pool_retain.load()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    cudaStreamSynchronize(st);
    cudaMemPoolTrimTo(pool, keep);
  }
  cudaGetLastError();
}

// Device scratch released at scope exit (stream-ordered).
struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(size_t bytes, cudaStream_t s) : st(s) {
    if (bytes) cuda_check(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), st(o.st) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      if (p) cudaFreeAsync(p, st);
      p = o.p;
      st = o.st;
      o.p = nullptr;
    }
    return *this;
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  template <typename U>
  U* as() const {
    return static_cast<U*>(p);
  }
};

// bf16 screening copy of an fp32 embedded A (32 MiB at n = 4096); built with the sketch
void build_screen_table(fstg_sketch* sk, cudaStream_t st) {
  if (sk->dtype != FSTG_F32 || !sk->has_a || sk->a == nullptr || sk->m == 0) return;
  sk->ldab = round_up(sk->n, 8);
  const size_t bytes = size_t(sk->m) * size_t(sk->ldab) * 2;
  cuda_check(cudaMalloc(&sk->ab, bytes), "allocate bf16 screening table");
  sk->device_bytes += bytes;
  bf16_table_kernel<<<148 * 4, 256, 0, st>>>(static_cast<const float*>(sk->a), sk->lda, sk->m, sk->n, sk->ab, sk->ldab);
  cuda_check(cudaGetLastError(), "bf16 screening table");
  cuda_check(cudaMalloc(&sk->abn, size_t(sk->m) * sizeof(float)), "allocate screening row norms");
  sk->device_bytes += size_t(sk->m) * sizeof(float);
  bf16_row_norms_kernel<<<148 * 4, 256, 0, st>>>(sk->ab, sk->ldab, sk->m, sk->abn);
  cuda_check(cudaGetLastError(), "screening row norms");
}

// the screening table a transform uses: none when screening is off (FSTG_STREAM_DEBUG bit 16)
// or for the A/B experiment switch FSTG_NO_BF16_SCREEN
const uint16_t* screen_table(const fstg_sketch* sk) {
  const char* dbg = std::getenv("FSTG_STREAM_DEBUG");
  if (dbg && (std::atoi(dbg) & 16)) return nullptr;
  const char* off = std::getenv("FSTG_NO_BF16_SCREEN");
  if (off && std::atoi(off) != 0) return nullptr;
  return sk->ab;
}

// ---------------------------------------------------------- preprocess ----
template <typename T>
void build_sketch(fstg_sketch* sk, const void* a_in, cudaStream_t st, int64_t b0, int64_t b1, bool identity,
                  bool materialize = true) {
  const int64_t m = sk->m, n = sk->n;
  const Design& D = sk->design;
  const int64_t nk = D.kerdock_bases();
  constexpr int64_t VEC = 16 / sizeof(T);
  sk->ldc = round_up(m, VEC);
  sk->lda = round_up(n, VEC);

  // embedded A (row-major, padded rows zeroed)
  const size_t a_bytes = size_t(m) * sk->lda * sizeof(T);
  cuda_check(cudaMalloc(&sk->a, a_bytes), "allocate embedded A");
  sk->device_bytes += a_bytes;
  cuda_check(cudaMemsetAsync(sk->a, 0, a_bytes, st), "memset A");
  cuda_check(cudaMemcpy2DAsync(sk->a, sk->lda * sizeof(T), a_in, n * sizeof(T), n * sizeof(T), m,
                               cudaMemcpyDefault, st),
             "copy A to device");

  {  // finite check (sketch.hpp:153)
    DevBuf bad(sizeof(int), st);
    cuda_check(cudaMemsetAsync(bad.p, 0, sizeof(int), st), "memset");
    const int64_t count = m * sk->lda;
    finite_check_kernel<<<148 * 4, 256, 0, st>>>(sk->a, sk->dtype, count, bad.as<int>());
    cuda_check(cudaGetLastError(), "finite check");
    int h = 0;
    cuda_check(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st), "copy flag");
    cuda_check(cudaStreamSynchronize(st), "sync");
    if (h) throw InvalidArgument("preprocess: matrix entries must be finite");
  }

  // sketch columns
  const uint64_t col_bytes = materialize ? uint64_t(D.L) * uint64_t(sk->ldc) * sizeof(T) : 0;
  if (materialize) {
    cudaError_t e = cudaMalloc(&sk->cols, col_bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      sk->cols = nullptr;
      throw std::runtime_error("preprocess: cannot allocate sketch of " + std::to_string(col_bytes) + " bytes");
    }
  }
  sk->device_bytes += col_bytes;
  // Row padding (ldc > m) is zeroed; a basis-sharded build leaves the other
  // ranks' Kerdock blocks unwritten (they are filled by the all-gather).
  if (materialize && sk->ldc != m) cuda_check(cudaMemsetAsync(sk->cols, 0, col_bytes, st), "memset sketch");

  // Kerdock sign tables
  const std::vector<uint32_t> rev = reversed_row_table(D);
  const int64_t wpb = D.d >= 32 ? D.d / 32 : 1;
  const int64_t twords = (D.d >= 128) ? (D.d >= 1024 ? D.d / 1024 : 1) * 32 : 0;
  cuda_check(cudaMalloc(&sk->revtab, rev.size() * sizeof(uint32_t)), "allocate tables");
  cuda_check(cudaMalloc(&sk->qplain, size_t(nk) * wpb * sizeof(uint32_t)), "allocate tables");
  if (twords) cuda_check(cudaMalloc(&sk->qtrans, size_t(nk) * twords * sizeof(uint32_t)), "allocate tables");
  sk->device_bytes += rev.size() * 4 + size_t(nk) * (wpb + twords) * 4;
  cuda_check(cudaMemcpyAsync(sk->revtab, rev.data(), rev.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st),
             "upload tables");
  {
    ProfScope ps("qtables", st);
    cuda_check(launch_qtables(sk->revtab, D.k, nk, sk->qplain, sk->qtrans, st), "qtable kernel");
  }

  cudaEvent_t e0, e1;
  cuda_check(cudaEventCreate(&e0), "event");
  cuda_check(cudaEventCreate(&e1), "event");
  cuda_check(cudaEventRecord(e0, st), "event");
  if (materialize && b1 > b0) {
    ProfScope ps("preprocess_fwht", st);
    const cudaError_t e = launch_fwht_sketch<T>(D.k, static_cast<const T*>(sk->a), sk->lda, m, n, sk->qplain, b0,
                                                b1, static_cast<T*>(sk->cols), sk->ldc, st);
    if (e == cudaErrorNotSupported) {
      cudaGetLastError();
      throw NotSupported("preprocess: this (k, dtype) needs more than 227 KiB of shared memory per CTA");
    }
    cuda_check(e, "fwht sketch kernel");
  }
  if (materialize && identity) {
    ProfScope ps("preprocess_identity", st);
    cuda_check(launch_identity<T>(static_cast<const T*>(sk->a), sk->lda, m, n, D.d, nk, static_cast<T*>(sk->cols),
                                  sk->ldc, st),
               "identity kernel");
  }
  cuda_check(cudaEventRecord(e1, st), "event");

  // row_norm_max (sketch.hpp:126-131)
  DevBuf norms(size_t(m) * sizeof(double), st);
  {
    ProfScope ps("row_norms", st);
    cuda_check(launch_row_norms<T>(static_cast<const T*>(sk->a), sk->lda, m, n, norms.as<double>(), st), "row norms");
  }
  std::vector<double> h(static_cast<size_t>(m));
  cuda_check(cudaMemcpyAsync(h.data(), norms.p, size_t(m) * sizeof(double), cudaMemcpyDeviceToHost, st), "copy norms");
  cuda_check(cudaStreamSynchronize(st), "preprocess sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  sk->preprocess_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  double rn = 0;
  for (double v : h) rn = std::max(rn, v);
  sk->row_norm_max = rn;
  if constexpr (sizeof(T) == 4) build_screen_table(sk, st);
}

void destroy_sketch(fstg_sketch* sk) {
  if (!sk) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(sk->device);
  cudaFree(sk->cols);
  cudaFree(sk->a);
  cudaFree(sk->ab);
  cudaFree(sk->abn);
  cudaFree(sk->qplain);
  cudaFree(sk->qtrans);
  cudaFree(sk->revtab);
  cudaSetDevice(prev);
  delete sk;
}

// -------------------------------------------------- retain-sampled columns ----
__global__ void basis_ranges_kernel(const uint64_t* __restrict__ sorted, int64_t count, int64_t nk, int64_t d,
                                    int64_t* __restrict__ start) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s <= nk; s += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t key = static_cast<uint64_t>(s) * static_cast<uint64_t>(d);
    int64_t lo = 0, hi = count;  // lower_bound
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (sorted[mid] < key) lo = mid + 1; else hi = mid;
    }
    start[s] = lo;
  }
}

template <typename T>
__global__ void identity_requests_kernel(const T* __restrict__ a, int64_t lda, int64_t row0, int64_t row1, int64_t n,
                                         int64_t kb, T sqrt_d, const uint64_t* __restrict__ ell,
                                         const int64_t* __restrict__ pos, int64_t first, int64_t count,
                                         T* __restrict__ out, int64_t ldc) {
  for (int64_t r = first + blockIdx.x; r < count; r += gridDim.x) {
    const int64_t w = static_cast<int64_t>(ell[r]) - kb;
    T* dst = out + pos[r] * ldc - row0;
    for (int64_t i = row0 + threadIdx.x; i < row1; i += blockDim.x) dst[i] = (w < n) ? sqrt_d * a[i * lda + w] : T(0);
  }
}

// (w = ell mod d, slot) u32 records of the sorted requests for the fp32 TMEM retain kernels
__global__ void pack_requests_kernel(const uint64_t* __restrict__ sorted, const int64_t* __restrict__ pos,
                                     int64_t count, uint64_t d, uint2* __restrict__ rec) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < count; r += int64_t(gridDim.x) * blockDim.x)
    rec[r] = make_uint2(static_cast<uint32_t>(sorted[r] & (d - 1)), static_cast<uint32_t>(pos[r]));
}

__global__ void iota_kernel(int64_t* v, int64_t count) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) v[i] = i;
}

__global__ void check_range_kernel(const int64_t* in, int64_t count, int64_t L, uint64_t* keys, int* bad) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = in[i];
    if (v < 0 || v >= L) {
      atomicExch(bad, 1);
      keys[i] = 0;
    } else {
      keys[i] = static_cast<uint64_t>(v);
    }
  }
}

template <typename T>
// Columns A s_ell (rows [row0, row1), column j at out + j * ldc_out) for the requested
// indices: the retain-sampled FWHT plus the identity-block gather.
void sample_columns_impl(const fstg_sketch* sk, const int64_t* indices, int64_t count, void* out, cudaStream_t st,
                         int64_t row0 = 0, int64_t row1 = -1, int64_t ldc_out = 0) {
  if (row1 < 0) row1 = sk->m;
  if (ldc_out <= 0) ldc_out = row0 == 0 && row1 == sk->m ? sk->ldc : row1 - row0;
  if (row0 < 0 || row1 > sk->m || row0 >= row1 || ldc_out < row1 - row0)
    throw InvalidArgument("sample_columns: bad row range / column stride");
  if (!sk) throw InvalidArgument("sample_columns: null sketch");
  if (count < 0 || (count > 0 && (!indices || !out))) throw InvalidArgument("sample_columns: bad arguments");
  if (count == 0) return;
  if (!sk->has_a) throw CodedError(FSTG_ERR_NO_MATRIX, "Sketch: no embedded matrix");
  cuda_check(cudaSetDevice(sk->device), "cudaSetDevice");
  keep_pool_warm(sk->device);
  const Design& D = sk->design;
  const int64_t nk = D.kerdock_bases();
  DevBuf idx_in, keys(size_t(count) * 8, st), keys_sorted(size_t(count) * 8, st), pos(size_t(count) * 8, st),
      pos_sorted(size_t(count) * 8, st), start(size_t(nk + 1) * 8, st), bad(sizeof(int), st), out_buf;
  const int64_t* id = indices;
  if (!is_device_ptr(indices)) {
    idx_in = DevBuf(size_t(count) * 8, st);
    cuda_check(cudaMemcpyAsync(idx_in.p, indices, size_t(count) * 8, cudaMemcpyHostToDevice, st), "H2D indices");
    id = idx_in.as<int64_t>();
  }
  T* dst = static_cast<T*>(out);
  const bool out_is_dev = is_device_ptr(out);
  if (!out_is_dev) {
    out_buf = DevBuf(size_t(count) * ldc_out * sizeof(T), st);
    dst = out_buf.as<T>();
  }
  cuda_check(cudaMemsetAsync(bad.p, 0, sizeof(int), st), "memset");
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((count + 255) / 256, 148 * 32));
  check_range_kernel<<<blocks, 256, 0, st>>>(id, count, D.L, keys.as<uint64_t>(), bad.as<int>());
  iota_kernel<<<blocks, 256, 0, st>>>(pos.as<int64_t>(), count);
  cuda_check(cudaGetLastError(), "request setup");
  // sort requests by ell (CUB radix sort, 32 key bits: L < 2^32)
  size_t temp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys.as<uint64_t>(), keys_sorted.as<uint64_t>(),
                                  pos.as<int64_t>(), pos_sorted.as<int64_t>(), count, 0, 32, st);
  DevBuf temp(temp_bytes, st);
  cuda_check(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, keys.as<uint64_t>(), keys_sorted.as<uint64_t>(),
                                             pos.as<int64_t>(), pos_sorted.as<int64_t>(), count, 0, 32, st),
             "sort requests");
  basis_ranges_kernel<<<static_cast<unsigned>((nk + 256) / 256), 256, 0, st>>>(keys_sorted.as<uint64_t>(), count, nk,
                                                                             D.d, start.as<int64_t>());
  cuda_check(cudaGetLastError(), "basis ranges");
  DevBuf rec;
  if (sizeof(T) == 4 && count < (int64_t{1} << 32)) {
    rec = DevBuf(size_t(count) * sizeof(uint2), st);
    pack_requests_kernel<<<blocks, 256, 0, st>>>(keys_sorted.as<uint64_t>(), pos_sorted.as<int64_t>(), count,
                                                 static_cast<uint64_t>(D.d), rec.as<uint2>());
    cuda_check(cudaGetLastError(), "pack requests");
  }
  {
    ProfScope ps("sample_columns_fwht", st);
    const cudaError_t e = launch_fwht_retain<T>(D.k, static_cast<const T*>(sk->a), sk->lda, row1, sk->n, sk->qplain,
                                                nk, dst, ldc_out, start.as<int64_t>(),
                                                reinterpret_cast<const int64_t*>(keys_sorted.p), pos_sorted.as<int64_t>(),
                                                st, row0, rec.p ? rec.as<uint2>() : nullptr);
    if (e == cudaErrorNotSupported) {
      cudaGetLastError();
      throw NotSupported("sample_columns: this (k, dtype) needs more than 227 KiB of shared memory per CTA");
    }
    cuda_check(e, "retain fwht");
  }
  {
    // identity-block requests: sqrt(d) * A[:, w] (sketch.hpp:200-208); first index = start[nk]
    int64_t first = 0;
    cuda_check(cudaMemcpyAsync(&first, start.as<int64_t>() + nk, 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    if (first < count) {
      ProfScope ps("sample_columns_identity", st);
      identity_requests_kernel<T><<<static_cast<unsigned>(std::min<int64_t>(count - first, 148 * 16)), 256, 0, st>>>(
          static_cast<const T*>(sk->a), sk->lda, row0, row1, sk->n, nk * D.d,
          static_cast<T>(std::sqrt(static_cast<double>(D.d))), keys_sorted.as<uint64_t>(), pos_sorted.as<int64_t>(),
          first, count, dst, ldc_out);
      cuda_check(cudaGetLastError(), "identity requests");
    }
  }
  int h = 0;
  cuda_check(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st), "flag");
  if (!out_is_dev)
    cuda_check(cudaMemcpyAsync(out, dst, size_t(count) * ldc_out * sizeof(T), cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "sync");
  if (h) throw OutOfRange("Sketch::column: index out of range");
}

// --------------------------------------------------------- persistence ----
// FSTK (sketch.hpp:213-302): "FSTK", u32 version, u64 m n k d L, u8 flag,
// L columns of m values, then m*n row-major A; little-endian; 49-byte header.
constexpr uint64_t kFstkHeader = 49;
constexpr size_t kChunkBytes = size_t(64) << 20;

__global__ void f64_to_f32_pitched(const double* __restrict__ src, int64_t rows, int64_t cols_src, float* __restrict__ dst,
                                   int64_t ld_dst) {
  const int64_t total = rows * cols_src;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols_src, c = i % cols_src;
    dst[r * ld_dst + c] = static_cast<float>(src[i]);
  }
}

struct PinnedBuf {
  void* p = nullptr;
  explicit PinnedBuf(size_t bytes) { cuda_check(cudaMallocHost(&p, bytes), "cudaMallocHost"); }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
};

struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

void put_le(std::vector<unsigned char>& h, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) h.push_back(static_cast<unsigned char>(v >> (8 * i)));
}

uint64_t get_le(const unsigned char* p, int bytes) {
  uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}

// Streams a device matrix (rows x cols, pitch ld elements of size es_dev) to
// the file as rows x cols values of size es_file (widening f32 -> f64 exactly).
// Whole rows per chunk while a row fits the pinned chunk; longer rows (m above
// kChunkBytes / 8 values, e.g. a reference file's huge m) go in element pieces.
void write_device_matrix(FILE* f, const void* dev, int64_t rows, int64_t cols, int64_t ld, size_t es_dev,
                         size_t es_file, PinnedBuf& buf, const std::string& path) {
  std::vector<double> wide;
  auto emit = [&](size_t count) {
    size_t wrote;
    if (es_dev == es_file) {
      wrote = std::fwrite(buf.p, es_file, count, f);
    } else {  // f32 device -> f64 file (exact)
      wide.resize(count);
      const float* src = static_cast<const float*>(buf.p);
      for (size_t i = 0; i < count; ++i) wide[i] = static_cast<double>(src[i]);
      wrote = std::fwrite(wide.data(), 8, count, f);
    }
    if (wrote != count) throw CodedError(FSTG_ERR_IO, "write failed: " + path);
  };
  const size_t piece = kChunkBytes / 8;  // values per chunk (the widened copy is 8 bytes per value)
  if (size_t(cols) <= piece) {
    const size_t row_bytes_dev = size_t(cols) * es_dev;
    const int64_t rows_per_chunk = int64_t(piece / size_t(cols));
    for (int64_t r0 = 0; r0 < rows; r0 += rows_per_chunk) {
      const int64_t rc = std::min(rows_per_chunk, rows - r0);
      cuda_check(cudaMemcpy2D(buf.p, row_bytes_dev, static_cast<const char*>(dev) + size_t(r0) * ld * es_dev,
                              size_t(ld) * es_dev, row_bytes_dev, size_t(rc), cudaMemcpyDeviceToHost),
                 "D2H sketch chunk");
      emit(size_t(rc) * size_t(cols));
    }
    return;
  }
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c0 = 0; c0 < cols; c0 += int64_t(piece)) {
      const size_t cc = std::min<size_t>(piece, size_t(cols - c0));
      cuda_check(cudaMemcpy(buf.p, static_cast<const char*>(dev) + (size_t(r) * ld + size_t(c0)) * es_dev,
                            cc * es_dev, cudaMemcpyDeviceToHost),
                 "D2H sketch piece");
      emit(cc);
    }
}

void save_impl(const fstg_sketch* sk, const char* path, int version) {
  if (!sk || !path) throw InvalidArgument("save: null argument");
  if (version != 1 && version != 2) throw InvalidArgument("save: FSTK version must be 1 (float64) or 2 (float32)");
  if (version == 2 && sk->dtype != FSTG_F32) throw InvalidArgument("save: FSTK v2 holds float32 sketches");
  if (!sk->cols) throw InvalidArgument("save: design-only sketch has no columns to save");
  cuda_check(cudaSetDevice(sk->device), "cudaSetDevice");
  File file(path, "wb");
  if (!file.f) throw CodedError(FSTG_ERR_IO, std::string("cannot open for writing: ") + path);
  std::vector<unsigned char> h = {'F', 'S', 'T', 'K'};
  put_le(h, static_cast<uint64_t>(version), 4);
  put_le(h, static_cast<uint64_t>(sk->m), 8);
  put_le(h, static_cast<uint64_t>(sk->n), 8);
  put_le(h, static_cast<uint64_t>(sk->design.k), 8);
  put_le(h, static_cast<uint64_t>(sk->design.d), 8);
  put_le(h, static_cast<uint64_t>(sk->design.L), 8);
  h.push_back(sk->has_a ? 1 : 0);
  if (std::fwrite(h.data(), 1, h.size(), file.f) != h.size()) throw CodedError(FSTG_ERR_IO, std::string("write failed: ") + path);
  const size_t es_dev = dtype_size(sk->dtype), es_file = version == 1 ? 8 : 4;
  PinnedBuf buf(kChunkBytes);
  cuda_check(cudaDeviceSynchronize(), "sync before save");
  write_device_matrix(file.f, sk->cols, sk->design.L, sk->m, sk->ldc, es_dev, es_file, buf, path);
  if (sk->has_a) write_device_matrix(file.f, sk->a, sk->m, sk->n, sk->lda, es_dev, es_file, buf, path);
  if (std::fflush(file.f) != 0) throw CodedError(FSTG_ERR_IO, std::string("write failed: ") + path);
}

// Reads rows x cols values of es_file bytes from the file into a device matrix
// (pitch ld elements of the sketch dtype), rounding f64 -> f32 on the GPU.
// Whole rows per chunk while a row fits the 64 MiB pinned / staging buffers;
// a longer row (an FSTK header may declare any m) is read in element pieces,
// so no file content can make a read exceed either buffer.
void read_device_matrix(FILE* f, void* dev, int64_t rows, int64_t cols, int64_t ld, size_t es_file, size_t es_dev,
                        PinnedBuf& buf, void* staging, cudaStream_t st, const std::string& path) {
  // one piece: rc rows of cc values starting at (r0, c0)
  auto piece = [&](int64_t r0, int64_t rc, int64_t c0, int64_t cc) {
    const size_t count = size_t(rc) * size_t(cc);
    cuda_check(cudaStreamSynchronize(st), "sync");  // previous chunk's copy out of `buf` is done
    if (std::fread(buf.p, es_file, count, f) != count)
      throw CodedError(FSTG_ERR_TRUNCATED, "FSTK payload truncated: " + path);
    char* dst = static_cast<char*>(dev) + (size_t(r0) * ld + size_t(c0)) * es_dev;
    if (es_file == es_dev) {
      cuda_check(cudaMemcpy2DAsync(dst, size_t(ld) * es_dev, buf.p, size_t(cc) * es_file, size_t(cc) * es_file,
                                   size_t(rc), cudaMemcpyHostToDevice, st),
                 "H2D sketch chunk");
    } else {
      cuda_check(cudaMemcpyAsync(staging, buf.p, count * es_file, cudaMemcpyHostToDevice, st), "H2D sketch chunk");
      f64_to_f32_pitched<<<148 * 8, 256, 0, st>>>(static_cast<const double*>(staging), rc, cc,
                                                 reinterpret_cast<float*>(dst), ld);
      cuda_check(cudaGetLastError(), "f64->f32");
    }
  };
  const size_t per = kChunkBytes / es_file;  // values per chunk
  if (size_t(cols) <= per) {
    const int64_t rows_per_chunk = int64_t(per / size_t(cols));
    for (int64_t r0 = 0; r0 < rows; r0 += rows_per_chunk) piece(r0, std::min(rows_per_chunk, rows - r0), 0, cols);
  } else {
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t c0 = 0; c0 < cols; c0 += int64_t(per)) piece(r, 1, c0, std::min<int64_t>(int64_t(per), cols - c0));
  }
  cuda_check(cudaStreamSynchronize(st), "sync");
}

void load_impl(const char* path, int dtype, int device, void* stream, fstg_sketch** out) {
  if (!path || !out) throw InvalidArgument("load: null argument");
  *out = nullptr;
  const std::string p(path);
  std::error_code ec;
  const uint64_t fsize = std::filesystem::file_size(p, ec);
  if (ec) throw CodedError(FSTG_ERR_IO, "cannot open for reading: " + p);
  if (fsize < kFstkHeader) throw CodedError(FSTG_ERR_TRUNCATED, "sketch file shorter than its header: " + p);
  File file(path, "rb");
  if (!file.f) throw CodedError(FSTG_ERR_IO, "cannot open for reading: " + p);
  unsigned char h[kFstkHeader];
  if (std::fread(h, 1, kFstkHeader, file.f) != kFstkHeader)
    throw CodedError(FSTG_ERR_TRUNCATED, "sketch file shorter than its header: " + p);
  if (std::memcmp(h, "FSTK", 4) != 0) throw CodedError(FSTG_ERR_MAGIC, "not an FSTK sketch file: " + p);
  const uint64_t version = get_le(h + 4, 4);
  if (version != 1 && version != 2)
    throw CodedError(FSTG_ERR_VERSION, "unsupported FSTK version " + std::to_string(version));
  const uint64_t m = get_le(h + 8, 8), n = get_le(h + 16, 8), k = get_le(h + 24, 8), d = get_le(h + 32, 8),
                 L = get_le(h + 40, 8);
  const int flag = h[48];
  if (m == 0 || n == 0 || k < 2 || k > 16 || k % 2 != 0 || d != (uint64_t{1} << k) || L != d * (d / 2 + 1) || n > d ||
      (flag != 0 && flag != 1))
    throw CodedError(FSTG_ERR_MALFORMED, "inconsistent FSTK header fields: " + p);
  const size_t es_file = version == 1 ? 8 : 4;
  const uint64_t col_bytes = es_file * m * L;
  const uint64_t expected = kFstkHeader + col_bytes + (flag ? es_file * m * n : 0);
  if (fsize < expected) throw CodedError(FSTG_ERR_TRUNCATED, "FSTK payload truncated: " + p);
  if (fsize > expected) throw CodedError(FSTG_ERR_MALFORMED, "FSTK file larger than its header declares");
  if (version == 2 && dtype == FSTG_F64) throw InvalidArgument("load: an FSTK v2 file holds a float32 sketch");
  dtype_size(dtype);
  if (k > 14) throw NotSupported("load: k > 14 exceeds this GPU build");
  require_device(device);
  keep_pool_warm(device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  auto* sk = new fstg_sketch();
  try {
    sk->device = device;
    sk->dtype = dtype;
    sk->design = Design::make(static_cast<int>(k));
    sk->m = static_cast<int64_t>(m);
    sk->n = static_cast<int64_t>(n);
    sk->has_a = flag != 0;
    const size_t es = dtype_size(dtype);
    const int64_t VEC = int64_t(16 / es);
    sk->ldc = round_up(sk->m, VEC);
    sk->lda = round_up(sk->n, VEC);
    const uint64_t dev_col_bytes = uint64_t(L) * uint64_t(sk->ldc) * es;
    if (cudaMalloc(&sk->cols, dev_col_bytes) != cudaSuccess) {
      cudaGetLastError();
      sk->cols = nullptr;
      throw std::runtime_error("load: cannot allocate sketch of " + std::to_string(dev_col_bytes) + " bytes");
    }
    sk->device_bytes += dev_col_bytes;
    if (sk->ldc != sk->m) cuda_check(cudaMemsetAsync(sk->cols, 0, dev_col_bytes, st), "memset sketch");
    const size_t a_bytes = size_t(sk->m) * sk->lda * es;
    cuda_check(cudaMalloc(&sk->a, a_bytes), "allocate embedded A");
    sk->device_bytes += a_bytes;
    cuda_check(cudaMemsetAsync(sk->a, 0, a_bytes, st), "memset A");

    PinnedBuf buf(kChunkBytes);
    DevBuf staging(es_file != es ? kChunkBytes : 0, st);
    read_device_matrix(file.f, sk->cols, static_cast<int64_t>(L), sk->m, sk->ldc, es_file, es, buf, staging.p, st, p);
    if (flag) read_device_matrix(file.f, sk->a, sk->m, sk->n, sk->lda, es_file, es, buf, staging.p, st, p);

    // design tables (the Sketch constructor rebuilds the Kerdock set, sketch.hpp:130)
    const Design& D = sk->design;
    const std::vector<uint32_t> rev = reversed_row_table(D);
    const int64_t nk = D.kerdock_bases();
    const int64_t wpb = D.d >= 32 ? D.d / 32 : 1;
    const int64_t twords = (D.d >= 128) ? (D.d >= 1024 ? D.d / 1024 : 1) * 32 : 0;
    cuda_check(cudaMalloc(&sk->revtab, rev.size() * sizeof(uint32_t)), "allocate tables");
    cuda_check(cudaMalloc(&sk->qplain, size_t(nk) * wpb * sizeof(uint32_t)), "allocate tables");
    if (twords) cuda_check(cudaMalloc(&sk->qtrans, size_t(nk) * twords * sizeof(uint32_t)), "allocate tables");
    cuda_check(cudaMemcpyAsync(sk->revtab, rev.data(), rev.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st),
               "upload tables");
    cuda_check(launch_qtables(sk->revtab, D.k, nk, sk->qplain, sk->qtrans, st), "qtable kernel");
    // row_norm_max (sketch.hpp:126-131; 0 without an embedded matrix)
    double rn = 0;
    if (flag) {
      DevBuf norms(size_t(sk->m) * sizeof(double), st);
      if (dtype == FSTG_F32)
        cuda_check(launch_row_norms<float>(static_cast<const float*>(sk->a), sk->lda, sk->m, sk->n, norms.as<double>(), st),
                   "row norms");
      else
        cuda_check(launch_row_norms<double>(static_cast<const double*>(sk->a), sk->lda, sk->m, sk->n, norms.as<double>(), st),
                   "row norms");
      std::vector<double> hn(static_cast<size_t>(sk->m));
      cuda_check(cudaMemcpyAsync(hn.data(), norms.p, hn.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "norms");
      cuda_check(cudaStreamSynchronize(st), "sync");
      for (double v : hn) rn = std::max(rn, v);
    }
    if (flag) build_screen_table(sk, st);
    cuda_check(cudaStreamSynchronize(st), "sync");
    sk->row_norm_max = rn;
  } catch (...) {
    destroy_sketch(sk);
    throw;
  }
  *out = sk;
}

int preprocess_impl(const void* a, int dtype, int64_t m, int64_t n, int device, void* stream, int64_t b0, int64_t b1,
                    bool full, int include_identity, fstg_sketch** out, bool materialize = true) {
  return guarded([&] {
    if (out == nullptr) throw InvalidArgument("preprocess: out is null");
    *out = nullptr;
    dtype_size(dtype);
    if (m < 1 || n < 1) throw InvalidArgument("preprocess: matrix must be nonempty");
    if (a == nullptr) throw InvalidArgument("preprocess: matrix pointer is null");
    const int k = even_log2_ceil(n);
    const Design D = Design::make(k);
    if (k > 14) throw NotSupported("preprocess: k > 14 (n > 16384) exceeds this GPU build's FWHT kernels");
    if (full) {
      b0 = 0;
      b1 = D.kerdock_bases();
    }
    if (b0 < 0 || b1 > D.kerdock_bases() || b0 > b1) throw OutOfRange("preprocess_shard: basis range out of range");
    require_device(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* sk = new fstg_sketch();
    sk->device = device;
    sk->dtype = dtype;
    sk->design = D;
    sk->m = m;
    sk->n = n;
    try {
      if (dtype == FSTG_F32)
        build_sketch<float>(sk, a, st, b0, b1, full || include_identity, materialize);
      else
        build_sketch<double>(sk, a, st, b0, b1, full || include_identity, materialize);
    } catch (...) {
      destroy_sketch(sk);
      throw;
    }
    *out = sk;
  });
}

// --------------------------------------------------------------- stream ----
struct Outputs {
  int32_t* counts;
  int32_t* support;
  void* values;
  int32_t* cands;
  void* mu;
};

template <typename T>
void run_batch(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p, const uint64_t* seeds,
               const int64_t* indices, const Outputs& out, cudaStream_t st, const void* gathered = nullptr) {
  validate(p);
  if (B < 0) throw InvalidArgument("transform: negative batch size");
  if (B == 0) return;
  if (X == nullptr) throw InvalidArgument("transform: X is null");
  if (out.counts == nullptr || out.support == nullptr || out.values == nullptr)
    throw InvalidArgument("transform: counts/support/values must be non-null");
  const Design& D = sk->design;
  const int64_t N = p->J * p->K;
  if (N > (int64_t(1) << 40)) throw NotSupported("transform: J*K too large for this build");
  if (!sk->has_a) throw CodedError(FSTG_ERR_NO_MATRIX, "Sketch: no embedded matrix");
  if (sk->cols == nullptr && gathered == nullptr)
    throw InvalidArgument("transform: design-only sketch; columns must come from fstg_transform_gathered_batch");
  if (gathered != nullptr && !is_device_ptr(gathered))
    throw InvalidArgument("transform_gathered: the gathered columns must be device memory");
  const int64_t want = candidate_count(p->s, p->widen, sk->m);
  const bool strict = p->mode == FSTG_MODE_STRICT || (p->mode == FSTG_MODE_DEFAULT && sk->dtype == FSTG_F64);
  if (p->mode < 0 || p->mode > 2) throw InvalidArgument("StreamParams: unknown mode");
  cuda_check(cudaSetDevice(sk->device), "cudaSetDevice");
  keep_pool_warm(sk->device);

  const int64_t n = sk->n, m = sk->m;
  const bool x_dev = is_device_ptr(X);
  const bool seeds_dev = is_device_ptr(seeds);
  const bool idx_dev = is_device_ptr(indices);
  const bool o_dev = is_device_ptr(out.counts) && is_device_ptr(out.support) && is_device_ptr(out.values) &&
                     (out.cands == nullptr || is_device_ptr(out.cands)) && (out.mu == nullptr || is_device_ptr(out.mu));
  const bool all_dev = x_dev && o_dev && (seeds == nullptr || seeds_dev) && (indices == nullptr || idx_dev);

  // Chunking bounds scratch (indices: chunk x N x 4 bytes) and pipelines host copies.
  // Host buffers: chunks grow geometrically from kFirstChunk to kMaxChunk vectors, so
  // the one copy that cannot overlap (the first chunk's H2D) is short while later
  // launches are long (each launch pays a pipeline fill and an unoverlapped tail).
  // The first chunk carries ~64 MiB of x (at least 2048 vectors) and at most a quarter of
  // the batch (but >= 256 vectors), so mid-size batches overlap 3/4 of their H2D (config 2,
  // 4096 vectors: e2e 1.07-1.12M -> 1.15-1.17M vectors/s); tiny batches run as one launch.
  constexpr int64_t kMaxChunk = 16384;
  int64_t first_chunk =
      std::max<int64_t>(2048, (int64_t(64) << 20) / std::max<int64_t>(1, n * int64_t(sizeof(T))));
  first_chunk = std::min<int64_t>(first_chunk, std::max<int64_t>(256, B / 4));
  if (const char* e = std::getenv("FSTG_FIRST_CHUNK")) first_chunk = std::max<int64_t>(1, std::atoll(e));  // experiments
  int64_t chunk = all_dev ? B : std::min<int64_t>(B, kMaxChunk);
  chunk = std::max<int64_t>(1, std::min<int64_t>(chunk, (int64_t(1) << 29) / std::max<int64_t>(N, 1)));
  int64_t next_chunk = all_dev ? chunk : std::min<int64_t>(chunk, first_chunk);

  StreamArgs<T> args{};
  args.cols = static_cast<const T*>(sk->cols);
  args.ldc = sk->ldc;
  args.a = static_cast<const T*>(sk->a);
  args.lda = sk->lda;
  args.ab = screen_table(sk);
  args.ldab = sk->ldab;
  args.abn = sk->abn;
  args.qplain = sk->qplain;
  args.qtrans = sk->qtrans;
  args.revtab = sk->revtab;
  args.k = D.k;
  args.d = D.d;
  args.L = D.L;
  args.m = m;
  args.n = n;
  args.kb = D.kerdock_bases() * D.d;
  args.J = p->J;
  args.K = p->K;
  args.N = N;
  args.want = want;
  args.epsilon = p->epsilon;
  args.ldx = n;
  args.m_pad = sk->ldc;
  constexpr int64_t SEG = 16384 / sizeof(T);
  args.nseg = static_cast<int>((sk->ldc + SEG - 1) / SEG);
  if (args.nseg > 4) throw NotSupported("transform: m too large for this GPU build (m <= 4 * 16 KiB / sizeof(T))");
  size_t smem = 0;
  int stages = 0, stage_stride = 0, rstride = 0, xbufs = 0;
  const int grid_max = stream_grid_size<T>(args, strict, chunk, &smem, &stages, &stage_stride, &rstride, &xbufs);
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (const char* e = std::getenv("FSTG_NO_BATCH_SPLIT")) if (std::atoi(e) != 0) sms = 0;  // experiments
  if (smem > 227 * 1024) throw NotSupported("transform: shared-memory plan exceeds 227 KiB (d or want too large)");
  args.stages = stages;
  args.stage_stride = stage_stride;
  args.rstride = rstride;
  args.xbufs = xbufs;
  {
    const char* dbg = std::getenv("FSTG_STREAM_DEBUG");
    args.debug = dbg ? std::atoi(dbg) : 0;
  }

  // Host buffers: H2D of chunk i+1 and D2H of chunk i-1 run on their own streams while
  // chunk i computes (one shared copy stream would queue the next H2D behind the
  // previous chunk's D2H, which waits for that chunk's kernel).
  const int nbuf = all_dev ? 1 : 2;
  // copy streams and events are cached per host thread and device (created once)
  struct HostPathRes {
    cudaStream_t in = nullptr, out = nullptr;
    cudaEvent_t ev[3][2] = {};
  };
  thread_local std::map<int, HostPathRes> t_res;
  cudaStream_t copy_st = nullptr, out_st = nullptr;
  HostPathRes* res = nullptr;
  if (!all_dev) {
    res = &t_res[sk->device];
    if (res->in == nullptr) {
      cuda_check(cudaStreamCreateWithFlags(&res->in, cudaStreamNonBlocking), "stream");
      cuda_check(cudaStreamCreateWithFlags(&res->out, cudaStreamNonBlocking), "stream");
      for (auto& row : res->ev)
        for (auto& e : row) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    copy_st = res->in;
    out_st = res->out;
  }
  struct Bufs {
    DevBuf X, idx, counts, support, values, cands, mu, seeds, idx64;
  };
  std::vector<Bufs> bufs(nbuf);
  DevBuf means(size_t(stream_scratch_elems<T>(args, grid_max)) * sizeof(T), st);
  DevBuf bad(sizeof(int), st);
  cuda_check(cudaMemsetAsync(bad.p, 0, sizeof(int), st), "memset");
  cudaEvent_t ev_in[2] = {}, ev_done[2] = {}, ev_out[2] = {};
  for (int b = 0; b < nbuf; ++b) {
    if (res != nullptr) {
      ev_in[b] = res->ev[0][b];
      ev_done[b] = res->ev[1][b];
      ev_out[b] = res->ev[2][b];
    }
    Bufs& bf = bufs[b];
    bf.idx = DevBuf(size_t(chunk) * N * sizeof(uint32_t), st);
    if (!x_dev) bf.X = DevBuf(size_t(chunk) * n * sizeof(T), st);
    if (!o_dev) {
      bf.counts = DevBuf(size_t(chunk) * sizeof(int32_t), st);
      bf.support = DevBuf(size_t(chunk) * want * sizeof(int32_t), st);
      bf.values = DevBuf(size_t(chunk) * want * sizeof(T), st);
      if (out.cands) bf.cands = DevBuf(size_t(chunk) * want * sizeof(int32_t), st);
      if (out.mu) bf.mu = DevBuf(size_t(chunk) * m * sizeof(T), st);
    }
    if (seeds != nullptr && !seeds_dev) bf.seeds = DevBuf(size_t(chunk) * sizeof(uint64_t), st);
    if (indices != nullptr && !idx_dev) bf.idx64 = DevBuf(size_t(chunk) * N * sizeof(int64_t), st);
  }
  if (!all_dev) {  // the copy stream starts after the stream-ordered allocations on st
    cuda_check(cudaEventRecord(ev_in[0], st), "event");
    cuda_check(cudaStreamWaitEvent(copy_st, ev_in[0], 0), "wait");
  }

  struct Pending {
    int64_t v0 = -1, cb = 0;
    int b = 0;
  } pending;
  // D2H of a finished chunk's outputs on out_st (ordered after its kernel by ev_done)
  auto drain = [&]() {
    if (pending.v0 < 0) return;
    const int64_t v0 = pending.v0, cb = pending.cb;
    Bufs& bf = bufs[pending.b];
    pending.v0 = -1;
    cuda_check(cudaStreamWaitEvent(out_st, ev_done[pending.b], 0), "wait");
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, out_st), "D2H");
    };
    d2h(out.counts + v0, bf.counts.p, size_t(cb) * sizeof(int32_t));
    d2h(out.support + v0 * want, bf.support.p, size_t(cb) * want * sizeof(int32_t));
    d2h(static_cast<T*>(out.values) + v0 * want, bf.values.p, size_t(cb) * want * sizeof(T));
    if (out.cands) d2h(out.cands + v0 * want, bf.cands.p, size_t(cb) * want * sizeof(int32_t));
    if (out.mu) d2h(static_cast<T*>(out.mu) + v0 * m, bf.mu.p, size_t(cb) * m * sizeof(T));
    cuda_check(cudaEventRecord(ev_out[pending.b], out_st), "event");
  };
  // On an error mid-loop the copy streams may still be reading or writing this call's
  // buffers: let them finish before the stream-ordered frees on st release the memory.
  struct DrainOnThrow {
    cudaStream_t a, b, c;
    bool armed = true;
    ~DrainOnThrow() {
      if (!armed) return;
      if (a) cudaStreamSynchronize(a);
      if (b) cudaStreamSynchronize(b);
      if (c) cudaStreamSynchronize(c);
      cudaGetLastError();
    }
  } guard{copy_st, out_st, st};
  int it = 0;
  for (int64_t v0 = 0, cb = 0; v0 < B; v0 += cb, ++it) {
    cb = std::min(next_chunk, B - v0);
    next_chunk = std::min(chunk, next_chunk * 2);
    const int b = it % nbuf;
    Bufs& bf = bufs[b];
    // ---- inputs ----
    const T* Xd = x_dev ? static_cast<const T*>(X) + v0 * n : bf.X.as<T>();
    const uint64_t* sd = seeds == nullptr ? nullptr : (seeds_dev ? seeds + v0 : bf.seeds.as<uint64_t>());
    const int64_t* id64 = indices == nullptr ? nullptr : (idx_dev ? indices + v0 * N : bf.idx64.as<int64_t>());
    if (!all_dev) {
      if (it >= nbuf) cuda_check(cudaStreamWaitEvent(copy_st, ev_done[b], 0), "wait");  // buffer free
      if (!x_dev)
        cuda_check(cudaMemcpyAsync(bf.X.p, static_cast<const T*>(X) + v0 * n, size_t(cb) * n * sizeof(T),
                                   cudaMemcpyHostToDevice, copy_st),
                   "H2D X");
      if (seeds != nullptr && !seeds_dev)
        cuda_check(cudaMemcpyAsync(bf.seeds.p, seeds + v0, size_t(cb) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                   copy_st),
                   "H2D seeds");
      if (indices != nullptr && !idx_dev)
        cuda_check(cudaMemcpyAsync(bf.idx64.p, indices + v0 * N, size_t(cb) * N * sizeof(int64_t),
                                   cudaMemcpyHostToDevice, copy_st),
                   "H2D indices");
      cuda_check(cudaEventRecord(ev_in[b], copy_st), "event");
      cuda_check(cudaStreamWaitEvent(st, ev_in[b], 0), "wait");
      if (it >= nbuf) cuda_check(cudaStreamWaitEvent(st, ev_out[b], 0), "wait");  // outputs drained
    }
    // ---- indices ----
    if (indices == nullptr) {
      ProfScope ps("draw", st);
      cuda_check(launch_draw<uint32_t>(sd, p->seed, cb, N, static_cast<uint64_t>(D.L), bf.idx.as<uint32_t>(), st),
                 "draw kernel");
    } else {
      ProfScope ps("narrow_indices", st);
      cuda_check(launch_narrow_indices(id64, cb * N, D.L, bf.idx.as<uint32_t>(), bad.as<int>(), st), "indices");
    }
    // ---- estimator ----
    args.X = Xd;
    args.idx = bf.idx.as<uint32_t>();
    args.gathered = gathered ? static_cast<const T*>(gathered) + v0 * N * sk->ldc : nullptr;
    args.B = cb;
    args.counts = o_dev ? out.counts + v0 : bf.counts.as<int32_t>();
    args.support = o_dev ? out.support + v0 * want : bf.support.as<int32_t>();
    args.values = o_dev ? static_cast<T*>(out.values) + v0 * want : bf.values.as<T>();
    args.cands = out.cands == nullptr ? nullptr : (o_dev ? out.cands + v0 * want : bf.cands.as<int32_t>());
    args.mu = out.mu == nullptr ? nullptr : (o_dev ? static_cast<T*>(out.mu) + v0 * m : bf.mu.as<T>());
    args.means = means.as<T>();
    const int grid = static_cast<int>(std::min<int64_t>(grid_max, cb));
    if (cb < sms && p->K > 1) {
      // Small batch: one CTA per vector would leave SMs idle. Every (vector, batch)
      // pair becomes a work item writing its batch mean (bit-identical: each batch
      // sum runs over its J samples in j order), then the tail runs per vector.
      DevBuf means_io(size_t(cb) * (p->K + 1) * args.m_pad * sizeof(T), st);
      args.means_mode = kMeansPartial;
      args.batch_split = 1;
      args.means_io = means_io.as<T>();
      args.m_io = args.m_pad;
      args.row0 = 0;
      args.means_vstride = 0;
      {
        ProfScope ps("stream", st);
        cuda_check(launch_stream<T>(args, strict, static_cast<int>(std::min<int64_t>(sms, cb * p->K)), st),
                   "stream kernel (batch split)");
      }
      args.means_mode = kMeansTail;
      args.batch_split = 0;
      {
        ProfScope ps("stream_tail", st);
        cuda_check(launch_stream<T>(args, strict, grid, st), "stream kernel (tail)");
      }
      args.means_mode = kMeansFull;
      args.means_io = nullptr;
    } else {
      ProfScope ps("stream", st);
      cuda_check(launch_stream<T>(args, strict, grid, st), "stream kernel");
    }
    if (args.debug & 8) {  // experiment: where each warp role waits (stream.cu WaitSite)
      cuda_check(cudaStreamSynchronize(st), "sync");
      unsigned long long w[14] = {};
      stream_wait_profile(w, 14);
      auto pct = [&](int site, int total) { return w[total] ? 100.0 * double(w[site]) / double(w[total]) : 0.0; };
      std::fprintf(stderr,
                   "stream waits (%% of role time): producer empty %.1f | coef x_empty %.1f t_empty %.1f | tail m_full "
                   "%.1f x_full %.1f r_empty %.1f r_full %.1f | consumer t_full %.1f column %.1f m_empty %.1f\n",
                   pct(0, 10), pct(1, 11), pct(2, 11), pct(3, 12), pct(4, 12), pct(5, 12), pct(6, 12), pct(7, 13),
                   pct(8, 13), pct(9, 13));
    }
    // ---- outputs ----
    // The D2H of chunk i is issued after chunk i+1's copy-in and kernel are queued (next
    // iteration): a copy into pageable host memory blocks this thread until it completes,
    // and deferring it keeps the next kernel queued behind the running one either way.
    if (!all_dev) {
      cuda_check(cudaEventRecord(ev_done[b], st), "event");
      if (o_dev) cuda_check(cudaEventRecord(ev_out[b], st), "event");
      drain();
      if (!o_dev) pending = Pending{v0, cb, b};
    }
  }
  if (!all_dev) drain();
  if (indices != nullptr) {
    int h = 0;
    cuda_check(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st), "copy flag");
    cuda_check(cudaStreamSynchronize(st), "sync");
    if (h) throw OutOfRange("Sketch::column: index out of range");
  }
  if (!all_dev) {
    cuda_check(cudaStreamSynchronize(copy_st), "sync copies");
    cuda_check(cudaStreamSynchronize(out_st), "sync copies");
    cuda_check(cudaStreamSynchronize(st), "sync compute");
  }
  guard.armed = false;
}

// ------------------------------------------- row-blocked design transform ----
// transform (stream.hpp:272-275) on a design-only sketch whose columns cannot
// exist (n = 16384: 8.8 TB). Rows of the estimator are independent — row i's
// batch sum is sum_j t_j C[i, ell_j] in j order — so the columns are produced
// and consumed one row block at a time: per block, the retain-sampled FWHT
// computes rows [r0, r1) of every sampled column of every vector (one pass over
// all Kerdock bases for those rows only), and the stream kernel in PARTIAL mode
// writes those rows of each vector's K batch means to means_io. Then TAIL mode
// runs median / select / refinement from means_io. Per call the Kerdock work is
// ONE full pass whatever the batch size (vector chunks would each need a full
// pass), and the batch means are bit-identical to the full-column path.
template <typename T>
struct DesignRun {
  const fstg_sketch* sk;
  const fstg_stream_params* p;
  bool strict;
  int64_t N, want;
  StreamArgs<T> args{};
  cudaStream_t st;

  DesignRun(const fstg_sketch* sk_, const void* X, int64_t B, const fstg_stream_params* p_, cudaStream_t st_)
      : sk(sk_), p(p_), st(st_) {
    validate(p);
    if (B < 0) throw InvalidArgument("transform_design: negative batch size");
    if (!sk->has_a) throw CodedError(FSTG_ERR_NO_MATRIX, "Sketch: no embedded matrix");
    if (B > 0 && (X == nullptr || !is_device_ptr(X))) throw InvalidArgument("transform_design: X must be device memory");
    if (p->mode < 0 || p->mode > 2) throw InvalidArgument("StreamParams: unknown mode");
    strict = p->mode == FSTG_MODE_STRICT || (p->mode == FSTG_MODE_DEFAULT && sk->dtype == FSTG_F64);
    const Design& D = sk->design;
    N = p->J * p->K;
    if (N > (int64_t(1) << 40)) throw NotSupported("transform: J*K too large for this build");
    want = candidate_count(p->s, p->widen, sk->m);
    cuda_check(cudaSetDevice(sk->device), "cudaSetDevice");
    keep_pool_warm(sk->device);
    args.a = static_cast<const T*>(sk->a);
    args.lda = sk->lda;
    args.ab = screen_table(sk);
    args.ldab = sk->ldab;
    args.abn = sk->abn;
    args.qplain = sk->qplain;
    args.qtrans = sk->qtrans;
    args.revtab = sk->revtab;
    args.k = D.k;
    args.d = D.d;
    args.L = D.L;
    args.n = sk->n;
    args.kb = D.kerdock_bases() * D.d;
    args.J = p->J;
    args.K = p->K;
    args.N = N;
    args.want = want;
    args.epsilon = p->epsilon;
    args.X = static_cast<const T*>(X);
    args.ldx = sk->n;
    args.B = B;
    const char* dbg = std::getenv("FSTG_STREAM_DEBUG");
    args.debug = dbg ? std::atoi(dbg) : 0;
  }

  void launch(const char* name) {
    if (args.nseg > 4) throw NotSupported("transform: m too large for this GPU build (m <= 4 * 16 KiB / sizeof(T))");
    size_t smem = 0;
    int stages = 0, stage_stride = 0, rstride = 0, xbufs = 0;
    const int grid = stream_grid_size<T>(args, strict, args.B, &smem, &stages, &stage_stride, &rstride, &xbufs);
    if (smem > 227 * 1024) throw NotSupported("transform: shared-memory plan exceeds 227 KiB (d or want too large)");
    args.stages = stages;
    args.stage_stride = stage_stride;
    args.rstride = rstride;
    args.xbufs = xbufs;
    DevBuf scratch(size_t(stream_scratch_elems<T>(args, grid)) * sizeof(T), st);
    args.means = scratch.as<T>();
    ProfScope ps(name, st);
    cuda_check(launch_stream<T>(args, strict, grid, st), "stream kernel");
  }

  // Rows [row_begin, row_end) of every vector's K batch means: vector v, batch b, row
  // r at means[v * vstride + b * ld + (r - row_begin)] (PARTIAL mode, row blocks).
  void partial(const uint64_t* seeds, int64_t row_begin, int64_t row_end, int64_t row_block, T* means,
               int64_t vstride, int64_t ld) {
    const int64_t B = args.B;
    if (B == 0 || row_end <= row_begin) return;
    if (row_begin < 0 || row_end > sk->m) throw InvalidArgument("design_partial_means: row range outside [0, m)");
    if (ld < row_end - row_begin || vstride < p->K * ld) throw InvalidArgument("design_partial_means: bad strides");
    const Design& D = sk->design;
    DevBuf idx64(size_t(B) * N * 8, st), idx32(size_t(B) * N * 4, st);
    {
      ProfScope ps("draw", st);
      cuda_check(launch_draw<int64_t>(seeds, p->seed, B, N, static_cast<uint64_t>(D.L), idx64.as<int64_t>(), st), "draw");
    }
    {
      ProfScope ps("draw", st);
      cuda_check(launch_draw<uint32_t>(seeds, p->seed, B, N, static_cast<uint64_t>(D.L), idx32.as<uint32_t>(), st),
                 "draw");
    }
    constexpr int64_t SEG = 16384 / sizeof(T), ALIGN = 16 / sizeof(T);
    const int64_t per_row = B * N * int64_t(sizeof(T));
    if (row_block <= 0) {  // as many rows as ~70% of free device memory holds
      size_t free_b = 0, total_b = 0;
      cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
      cudaMemPool_t pool;  // memory the pool holds but does not use (fstg_set_pool_retain) is free to us
      if (cudaDeviceGetDefaultMemPool(&pool, sk->device) == cudaSuccess) {
        uint64_t reserved = 0, used = 0;
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        if (reserved > used) free_b += size_t(reserved - used);
      }
      cudaGetLastError();
      row_block = std::max<int64_t>(ALIGN, int64_t(double(free_b) * 0.7) / std::max<int64_t>(per_row, 1));
      // then equal blocks: as few as memory allows, but no ragged last block (config 4,
      // 16384 rows: 4 x 4096 instead of 3 x ~4800 + 1984 -> 2.50 -> 2.26 s per step)
      const int64_t rows = row_end - row_begin, nblk = (rows + row_block - 1) / row_block;
      row_block = ((rows + nblk - 1) / nblk + ALIGN - 1) / ALIGN * ALIGN;
    }
    row_block = std::max<int64_t>(ALIGN, row_block / ALIGN * ALIGN);
    args.idx = idx32.as<uint32_t>();
    args.means_io = means;
    args.m_io = ld;
    args.means_vstride = vstride;
    for (int64_t r0 = row_begin; r0 < row_end; r0 += row_block) {
      const int64_t r1 = std::min(row_end, r0 + row_block);
      const int64_t ldh = (r1 - r0 + ALIGN - 1) / ALIGN * ALIGN;
      DevBuf cols(size_t(B) * N * ldh * sizeof(T), st);
      sample_columns_impl<T>(sk, idx64.as<int64_t>(), B * N, cols.p, st, r0, r1, ldh);
      args.means_mode = kMeansPartial;
      args.cols = nullptr;
      args.gathered = cols.as<T>();
      args.ldc = ldh;
      args.m = r1 - r0;
      args.m_pad = ldh;
      args.row0 = r0 - row_begin;
      args.nseg = static_cast<int>((ldh + SEG - 1) / SEG);
      launch("stream_partial");
    }
  }

  // Median / top-want / refinement from K batch means per vector (means[v * vstride
  // + b * ld + row], slot K receives mu) (TAIL mode).
  void tail(T* means, int64_t vstride, int64_t ld, const Outputs& out) {
    if (args.B == 0) return;
    if (out.counts == nullptr || out.support == nullptr || out.values == nullptr)
      throw InvalidArgument("transform_design: counts/support/values must be non-null");
    if (!is_device_ptr(out.counts) || !is_device_ptr(out.support) || !is_device_ptr(out.values) ||
        (out.cands && !is_device_ptr(out.cands)) || (out.mu && !is_device_ptr(out.mu)))
      throw InvalidArgument("transform_design: outputs must be device memory");
    constexpr int64_t SEG = 16384 / sizeof(T), VEC = 16 / sizeof(T);
    if (ld < sk->m || ld % VEC != 0 || vstride < (p->K + 1) * ld)
      throw InvalidArgument("transform_from_means: bad strides (ld >= m, multiple of 16 bytes; vstride >= (K+1) ld)");
    args.counts = out.counts;
    args.support = out.support;
    args.values = static_cast<T*>(out.values);
    args.cands = out.cands;
    args.mu = static_cast<T*>(out.mu);
    args.means_mode = kMeansTail;
    args.means_io = means;
    args.m_io = ld;
    args.means_vstride = vstride;
    args.idx = nullptr;
    args.gathered = nullptr;
    args.cols = nullptr;
    args.ldc = ld;
    args.m = sk->m;
    args.m_pad = ld;
    args.row0 = 0;
    args.nseg = static_cast<int>((ld + SEG - 1) / SEG);
    launch("stream_tail");
  }
};

// ------------------------------------------- row-blocked design transform ----
// transform (stream.hpp:272-275) on a design-only sketch whose columns cannot
// exist (n = 16384: 8.8 TB). Rows of the estimator are independent — row i's
// batch sum is sum_j t_j C[i, ell_j] in j order — so the columns are produced
// and consumed one row block at a time: per block, the retain-sampled FWHT
// computes rows [r0, r1) of every sampled column of every vector (one pass over
// all Kerdock bases for those rows only), and the stream kernel in PARTIAL mode
// writes those rows of each vector's K batch means; then TAIL mode runs median /
// select / refinement. Per call the Kerdock work is ONE full pass whatever the
// batch size, and the batch means are bit-identical to the full-column path.
template <typename T>
void transform_design_impl(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                           const uint64_t* seeds, int64_t row_block, const Outputs& out, cudaStream_t st) {
  DesignRun<T> run(sk, X, B, p, st);
  if (B == 0) return;
  if (seeds && !is_device_ptr(seeds)) throw InvalidArgument("transform_design: seeds must be device memory");
  const int64_t m_io = sk->ldc, vstride = (p->K + 1) * m_io;
  DevBuf means(size_t(B) * vstride * sizeof(T), st);
  run.partial(seeds, 0, sk->m, row_block, means.as<T>(), vstride, m_io);
  run.tail(means.as<T>(), vstride, m_io, out);
  cuda_check(cudaStreamSynchronize(st), "sync");
  trim_pool(sk->device, st);
}


// ------------------------------------------------------- public helpers ----
// Host-or-device double buffers for the small helpers (copied in / out).
struct DoubleIn {
  DevBuf buf;
  const double* p = nullptr;
  DoubleIn(const double* src, int64_t count, cudaStream_t st) {
    if (count <= 0) return;
    if (is_device_ptr(src)) {
      p = src;
    } else {
      buf = DevBuf(size_t(count) * 8, st);
      cuda_check(cudaMemcpyAsync(buf.p, src, size_t(count) * 8, cudaMemcpyHostToDevice, st), "H2D");
      p = buf.as<double>();
    }
  }
};

void finish_out(double* dst, const DevBuf& tmp, int64_t count, cudaStream_t st) {
  if (tmp.p != nullptr)
    cuda_check(cudaMemcpyAsync(dst, tmp.p, size_t(count) * 8, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "sync");
}

void helper_prologue(int device) {
  require_device(device);
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
}

// kerdock.hpp:111-129 DesignIndex::from_linear -> (identity?, basis s, wpos) and the basis' reversed rows
bool decode_design_index(const Design& D, int64_t ell, uint64_t* wpos, std::vector<uint32_t>& rev) {
  if (ell < 0 || ell >= D.L) throw OutOfRange("DesignIndex: linear index out of range");
  const int64_t kb = D.kerdock_bases() * D.d;
  rev.assign(16, 0u);
  if (ell >= kb) {
    *wpos = static_cast<uint64_t>(ell - kb);
    return true;
  }
  const Field f(D.k - 1, D.modulus);
  const auto rows = kerdock_matrix(D, f, static_cast<uint64_t>(ell / D.d));
  reversed_rows(rows.data(), D.k, rev.data());
  *wpos = static_cast<uint64_t>(ell % D.d);
  return false;
}

void inner_product_impl(int k, const double* x, int64_t n, int64_t ell, double* out, int device) {
  const Design D = Design::make(k);
  if (!x || !out) throw InvalidArgument("inner_product_with_design: null pointer");
  if (n < 1 || n > D.d) throw InvalidArgument("inner_product_with_design: bad vector length");
  uint64_t wpos = 0;
  std::vector<uint32_t> rev;
  const bool identity = decode_design_index(D, ell, &wpos, rev);
  if (identity) {  // stream.hpp:113-116: sqrt(d) x_w or 0 (one multiply; no kernel needed)
    double xv = 0;
    if (static_cast<int64_t>(wpos) < n) {
      helper_prologue(device);
      cuda_check(cudaMemcpy(&xv, x + wpos, 8, is_device_ptr(x) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost),
                 "copy");
      *out = std::sqrt(static_cast<double>(D.d)) * xv;
    } else {
      *out = 0.0;
    }
    return;
  }
  helper_prologue(device);
  cudaStream_t st = nullptr;
  DoubleIn xin(x, n, st);
  DevBuf drev(16 * 4, st), dout(8, st);
  cuda_check(cudaMemcpyAsync(drev.p, rev.data(), 16 * 4, cudaMemcpyHostToDevice, st), "H2D");
  {
    ProfScope ps("inner_product", st);
    cuda_check(launch_inner_product(xin.p, n, D.d, drev.as<uint32_t>(), wpos, dout.as<double>(), st), "kernel");
  }
  cuda_check(cudaMemcpyAsync(out, dout.p, 8, is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st),
             "copy out");
  cuda_check(cudaStreamSynchronize(st), "sync");
}

void median_of_means_impl(const double* samples, int64_t m, int64_t J, int64_t K, double* out, int device) {
  if (J < 1 || K < 1 || m < 0) throw InvalidArgument("median_of_means: samples must have J*K columns");
  if (m > 0 && (!samples || !out)) throw InvalidArgument("median_of_means: null pointer");
  if (m == 0) return;
  helper_prologue(device);
  cudaStream_t st = nullptr;
  DoubleIn in(samples, m * J * K, st);
  DevBuf tmp;
  double* dst = out;
  if (!is_device_ptr(out)) {
    tmp = DevBuf(size_t(m) * 8, st);
    dst = tmp.as<double>();
  }
  {
    ProfScope ps("median_of_means", st);
    cuda_check(launch_median_of_means(in.p, m, J, K, dst, st), "kernel");
  }
  finish_out(out, tmp, m, st);
}

void hard_threshold_impl(const double* v, int64_t len, double eps, double* out, int device) {
  if (len < 0 || (len > 0 && (!v || !out))) throw InvalidArgument("hard_threshold: bad arguments");
  if (len == 0) return;
  helper_prologue(device);
  cudaStream_t st = nullptr;
  DoubleIn in(v, len, st);
  DevBuf tmp;
  double* dst = out;
  if (!is_device_ptr(out)) {
    tmp = DevBuf(size_t(len) * 8, st);
    dst = tmp.as<double>();
  }
  {
    ProfScope ps("hard_threshold", st);
    cuda_check(launch_hard_threshold(in.p, len, eps, dst, st), "kernel");
  }
  finish_out(out, tmp, len, st);
}

void design_column_impl(int k, int64_t n, int64_t ell, double* out, int device) {
  const Design D = Design::make(k);
  if (n < 1 || n > D.d) throw InvalidArgument("projected_design_column: n out of [1,d]");
  if (!out) throw InvalidArgument("projected_design_column: null pointer");
  uint64_t wpos = 0;
  std::vector<uint32_t> rev;
  const bool identity = decode_design_index(D, ell, &wpos, rev);
  helper_prologue(device);
  cudaStream_t st = nullptr;
  DevBuf drev(16 * 4, st), tmp;
  cuda_check(cudaMemcpyAsync(drev.p, rev.data(), 16 * 4, cudaMemcpyHostToDevice, st), "H2D");
  double* dst = out;
  if (!is_device_ptr(out)) {
    tmp = DevBuf(size_t(n) * 8, st);
    dst = tmp.as<double>();
  }
  {
    ProfScope ps("design_column", st);
    cuda_check(launch_design_column(n, D.d, identity ? 1 : 0, drev.as<uint32_t>(), D.k, wpos,
                                    std::sqrt(static_cast<double>(D.d)), dst, st),
               "kernel");
  }
  finish_out(out, tmp, n, st);
}

// ----------------------------------------------------- design verifiers ----
// kerdock.hpp:198-317 / cli.hpp:45-60 on the GPU (verify.cu). Inner products
// are F/d with integer F, so every report field is assembled exactly from the
// integer statistics the kernels return.
using u128 = unsigned __int128;

u128 get_u128(const unsigned long long* v) { return (static_cast<u128>(v[1]) << 64) | v[0]; }

// num / den for a power-of-two den, exact whenever the quotient and the
// remainder fit a double's mantissa (always, for a valid design).
double exact_ratio(u128 num, u128 den) {
  const u128 q = num / den, r = num % den;
  return static_cast<double>(q) + static_cast<double>(r) / static_cast<double>(den);
}

struct VerifyTables {
  Design D;
  DevBuf revtab, qplain;
};

void verify_prologue(int k, int cap, int policy, int device, const char* who, VerifyTables& t, cudaStream_t st) {
  t.D = Design::make(k);
  if (k > cap) throw InvalidArgument(std::string(who) + ": k exceeds the verification cap");
  if (policy != FSTG_VERIFY_REFERENCE && policy != FSTG_VERIFY_EXHAUSTIVE)
    throw InvalidArgument(std::string(who) + ": unknown policy");
  if (k > 14) throw NotSupported(std::string(who) + ": k > 14 is not supported on the GPU path");
  require_device(device);
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  const std::vector<uint32_t> rev = reversed_row_table(t.D);
  const int64_t nk = t.D.kerdock_bases(), wpb = t.D.d >= 32 ? t.D.d / 32 : 1;
  t.revtab = DevBuf(rev.size() * 4, st);
  t.qplain = DevBuf(size_t(nk) * wpb * 4, st);
  cuda_check(cudaMemcpyAsync(t.revtab.p, rev.data(), rev.size() * 4, cudaMemcpyHostToDevice, st), "upload tables");
  ProfScope ps("qtables", st);
  cuda_check(launch_qtables(t.revtab.as<uint32_t>(), k, nk, t.qplain.as<uint32_t>(), nullptr, st), "qtable kernel");
}

struct PairStats {
  u128 x2w = 0, x4w = 0, x2c = 0, x4c = 0;
  int bad = 0, f2min = INT32_MAX, f2max = 0;
};

// Basis pairs through the integer FWHT kernel; pairs == empty -> the whole upper triangle.
PairStats run_pairs(const VerifyTables& t, const std::vector<int32_t>& pb, const std::vector<int32_t>& pb2,
                    cudaStream_t st) {
  const int64_t nk = t.D.kerdock_bases();
  const bool all = pb.empty();
  const int64_t npairs = all ? nk * (nk + 1) / 2 : static_cast<int64_t>(pb.size());
  DevBuf acc(8 * 8, st), stats(3 * 4, st), dpb, dpb2;
  const int init[3] = {0, INT32_MAX, 0};
  cuda_check(cudaMemsetAsync(acc.p, 0, 64, st), "memset");
  cuda_check(cudaMemcpyAsync(stats.p, init, sizeof(init), cudaMemcpyHostToDevice, st), "H2D");
  if (!all) {
    dpb = DevBuf(pb.size() * 4, st);
    dpb2 = DevBuf(pb.size() * 4, st);
    cuda_check(cudaMemcpyAsync(dpb.p, pb.data(), pb.size() * 4, cudaMemcpyHostToDevice, st), "H2D pairs");
    cuda_check(cudaMemcpyAsync(dpb2.p, pb2.data(), pb.size() * 4, cudaMemcpyHostToDevice, st), "H2D pairs");
  }
  {
    ProfScope ps("verify_pairs", st);
    cuda_check(launch_verify_pairs(t.D.k, t.qplain.as<uint32_t>(), nk, npairs, dpb.as<int32_t>(), dpb2.as<int32_t>(),
                                   acc.as<unsigned long long>(), stats.as<int>(), st),
               "verify pairs kernel");
  }
  unsigned long long h[8];
  int hs[3];
  cuda_check(cudaMemcpyAsync(h, acc.p, 64, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaMemcpyAsync(hs, stats.p, 12, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "sync");
  PairStats r;
  r.x2w = get_u128(h);
  r.x4w = get_u128(h + 2);
  r.x2c = get_u128(h + 4);
  r.x4c = get_u128(h + 6);
  r.bad = hs[0];
  r.f2min = hs[1];
  r.f2max = hs[2];
  return r;
}

void verify_mub_impl(int k, int cap, int policy, int device, fstg_mub_report* out) {
  if (!out) throw InvalidArgument("verify_mub: null report");
  cudaStream_t st = nullptr;
  VerifyTables t;
  verify_prologue(k, cap, policy, device, "verify_mub", t, st);
  const int64_t d = t.D.d, nk = t.D.kerdock_bases(), nb = nk + 1;
  const bool exhaustive = policy == FSTG_VERIFY_EXHAUSTIVE || k <= 6;
  std::vector<int32_t> pb, pb2;
  int64_t identity_pairs = 0, cross_pairs = 0;
  if (exhaustive) {
    identity_pairs = nk;  // (b, identity) for every Kerdock b
    cross_pairs = nb * (nb - 1) / 2;
  } else {
    for (int64_t b = 0; b < nk; ++b) {  // within-basis Gram of every basis (kerdock.hpp:223-227)
      pb.push_back(static_cast<int32_t>(b));
      pb2.push_back(static_cast<int32_t>(b));
    }
    std::mt19937_64 rng(0x6d7562u);  // kerdock.hpp:245: fixed-seed basis-pair sample
    for (int i = 0; i < 256; ++i) {
      const auto b = static_cast<int64_t>(rng() % static_cast<uint64_t>(nb));
      auto b2 = static_cast<int64_t>(rng() % static_cast<uint64_t>(nb - 1));
      if (b2 >= b) ++b2;
      ++cross_pairs;
      if (b == nk || b2 == nk) {
        ++identity_pairs;
      } else {
        pb.push_back(static_cast<int32_t>(std::min(b, b2)));  // F is symmetric in the pair
        pb2.push_back(static_cast<int32_t>(std::max(b, b2)));
      }
    }
  }
  const PairStats ps = run_pairs(t, pb, pb2, st);
  const double dd = static_cast<double>(d), inv_d = 1.0 / dd;
  fstg_mub_report r{};
  r.max_within_gram_dev = static_cast<double>(ps.bad) / dd;  // identity block: I^T I - I = 0
  double lo = std::numeric_limits<double>::infinity(), hi = -std::numeric_limits<double>::infinity();
  if (ps.f2max > 0 || ps.f2min != INT32_MAX) {
    lo = static_cast<double>(ps.f2min) / (dd * dd);
    hi = static_cast<double>(ps.f2max) / (dd * dd);
  }
  if (identity_pairs > 0) {  // e_pos . u_{s,w} = +-2^(-k/2): squared exactly 1/d
    lo = std::min(lo, inv_d);
    hi = std::max(hi, inv_d);
  }
  if (!std::isfinite(lo)) lo = hi = 0;
  r.min_cross_sq = lo;
  r.max_cross_sq = hi;
  r.max_cross_dev = cross_pairs > 0 ? std::max(std::abs(lo - inv_d), std::abs(hi - inv_d)) : 0.0;
  r.exhaustive = exhaustive ? 1 : 0;
  r.basis_pairs = cross_pairs;
  *out = r;
}

void verify_moments_impl(int k, int cap, int policy, int device, fstg_moment_report* out) {
  if (!out) throw InvalidArgument("verify_design_moments: null report");
  cudaStream_t st = nullptr;
  VerifyTables t;
  verify_prologue(k, cap, policy, device, "verify_design_moments", t, st);
  const int64_t d = t.D.d, nk = t.D.kerdock_bases(), L = t.D.L;
  const u128 ud = static_cast<u128>(d);
  fstg_moment_report r{};
  if (policy == FSTG_VERIFY_EXHAUSTIVE || k <= 6) {
    // sum over ordered column pairs: Kerdock x Kerdock blocks from the FWHT
    // (sum_{w,w'} (F[w^w']/d)^2 = sum_u F^2 / d, ^4: sum_u F^4 / d^3), both
    // orders of every cross pair; identity x identity = d ones; identity x
    // Kerdock (both orders) = 2 d^2 entries of 1/d (and 1/d^2 for ^4).
    const PairStats ps = run_pairs(t, {}, {}, st);
    const u128 n2 = ps.x2w + 2 * ps.x2c + (ud + 2 * static_cast<u128>(nk) * ud) * ud;
    const u128 n4 = ps.x4w + 2 * ps.x4c + (ud + 2 * static_cast<u128>(nk)) * ud * ud * ud;
    const double pairs = static_cast<double>(L) * static_cast<double>(L);
    r.m1 = exact_ratio(n2, ud) / pairs;
    r.m2 = exact_ratio(n4, ud * ud * ud) / pairs;
    r.exact = 1;
    r.pairs = L * L;
  } else {
    const int samples = 4'000'000;  // kerdock.hpp:305-313, same engine, seed and draw order
    std::vector<int64_t> ia(samples), ib(samples);
    std::mt19937_64 rng(0x6d6f6du);
    for (int i = 0; i < samples; ++i) {
      ia[i] = static_cast<int64_t>(rng() % static_cast<uint64_t>(L));
      ib[i] = static_cast<int64_t>(rng() % static_cast<uint64_t>(L));
    }
    DevBuf da(size_t(samples) * 8, st), db(size_t(samples) * 8, st), acc(4 * 8, st);
    cuda_check(cudaMemcpyAsync(da.p, ia.data(), size_t(samples) * 8, cudaMemcpyHostToDevice, st), "H2D samples");
    cuda_check(cudaMemcpyAsync(db.p, ib.data(), size_t(samples) * 8, cudaMemcpyHostToDevice, st), "H2D samples");
    cuda_check(cudaMemsetAsync(acc.p, 0, 32, st), "memset");
    {
      ProfScope ps("verify_samples", st);
      cuda_check(launch_verify_samples(k, t.qplain.as<uint32_t>(), da.as<int64_t>(), db.as<int64_t>(), samples,
                                       acc.as<unsigned long long>(), st),
                 "verify samples kernel");
    }
    unsigned long long h[4];
    cuda_check(cudaMemcpyAsync(h, acc.p, 32, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    // sum2 = sum F^2 / d^2, sum4 = sum F^4 / d^4 (each sampled term exact)
    r.m1 = exact_ratio(get_u128(h), ud * ud) / samples;
    r.m2 = exact_ratio(get_u128(h + 2), ud * ud * ud * ud) / samples;
    r.exact = 0;
    r.pairs = samples;
  }
  *out = r;
}

void verify_kerdock_set_impl(int k, int device, int* skew, int64_t* bad_pairs) {
  if (!skew || !bad_pairs) throw InvalidArgument("verify_kerdock_set: null output");
  const Design D = Design::make(k);
  if (k > 14) throw NotSupported("verify_kerdock_set: k > 14 is not supported on the GPU path");
  require_device(device);
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cudaStream_t st = nullptr;
  const Field f(D.k - 1, D.modulus);
  const int64_t nk = D.kerdock_bases();
  std::vector<uint32_t> rows(size_t(nk) * k);
  bool ok = true;
  for (int64_t s = 0; s < nk; ++s) {
    const auto m = kerdock_matrix(D, f, static_cast<uint64_t>(s));
    for (int i = 0; i < k; ++i) {
      rows[size_t(s) * k + i] = static_cast<uint32_t>(m[i]);
      ok = ok && ((m[i] >> i) & 1) == 0;
      for (int j = 0; j < k; ++j) ok = ok && ((m[i] >> j) & 1) == ((m[j] >> i) & 1);
    }
  }
  DevBuf drows(rows.size() * 4, st), bad(8, st);
  cuda_check(cudaMemcpyAsync(drows.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, st), "H2D rows");
  cuda_check(cudaMemsetAsync(bad.p, 0, 8, st), "memset");
  {
    ProfScope ps("verify_ranks", st);
    cuda_check(launch_verify_ranks(k, drows.as<uint32_t>(), nk, bad.as<unsigned long long>(), st), "rank kernel");
  }
  unsigned long long h = 0;
  cuda_check(cudaMemcpyAsync(&h, bad.p, 8, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "sync");
  *skew = ok ? 1 : 0;
  *bad_pairs = static_cast<int64_t>(h);
}

}  // namespace

// ====================================================================== ABI ==
extern "C" {

const char* fstg_last_error(void) { return g_error.c_str(); }

const char* fstg_version(void) { return "fst_b200 1 (sm_100a)"; }

int fstg_device_count(int* count) {
  return guarded([&] {
    if (!count) throw InvalidArgument("null");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    int ok = 0;
    for (int i = 0; i < c; ++i) {
      cudaDeviceProp prop{};
      if (cudaGetDeviceProperties(&prop, i) == cudaSuccess && prop.major == 10) ++ok;
    }
    *count = ok;
  });
}

int fstg_even_log2_ceil(int64_t n, int* k) {
  return guarded([&] { *k = even_log2_ceil(n); });
}

int fstg_design_params(int k, int64_t* d, int64_t* L) {
  return guarded([&] {
    const Design D = Design::make(k);
    *d = D.d;
    *L = D.L;
  });
}

int fstg_kerdock_matrix(int k, uint64_t s, uint64_t* rows) {
  return guarded([&] {
    const Design D = Design::make(k);
    const Field f(k - 1, D.modulus);
    const auto r = kerdock_matrix(D, f, s);
    std::memcpy(rows, r.data(), r.size() * sizeof(uint64_t));
  });
}

int fstg_choose_params(double r, double gamma, double eta, int64_t m, int64_t* J, int64_t* K) {
  return guarded([&] { choose_params(r, gamma, eta, m, J, K); });
}

int fstg_validate_params(const fstg_stream_params* p) {
  return guarded([&] { validate(p); });
}

int64_t fstg_candidate_count(int64_t s, int64_t widen, int64_t m) { return candidate_count(s, widen, m); }

int fstg_preprocess(const void* a, int dtype, int64_t m, int64_t n, int device, void* stream, fstg_sketch** out) {
  return preprocess_impl(a, dtype, m, n, device, stream, 0, 0, true, 1, out);
}

int fstg_preprocess_design(const void* a, int dtype, int64_t m, int64_t n, int device, void* stream,
                           fstg_sketch** out) {
  return preprocess_impl(a, dtype, m, n, device, stream, 0, 0, true, 1, out, false);
}

int fstg_sample_columns(const fstg_sketch* sk, const int64_t* indices, int64_t count, void* out, void* stream) {
  return guarded([&] {
    if (!sk) throw InvalidArgument("sample_columns: null sketch");
    if (sk->dtype == FSTG_F32)
      sample_columns_impl<float>(sk, indices, count, out, static_cast<cudaStream_t>(stream));
    else
      sample_columns_impl<double>(sk, indices, count, out, static_cast<cudaStream_t>(stream));
    // host output: the device staging buffer can be large (count columns); hand it back
    const size_t staged = size_t(count) * size_t(sk->ldc) * (sk->dtype == FSTG_F32 ? 4 : 8);
    if (out != nullptr && !is_device_ptr(out) && staged > (size_t(1) << 30))
      trim_pool(sk->device, static_cast<cudaStream_t>(stream));
  });
}

int fstg_transform_gathered_batch(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                                  const int64_t* indices, const void* gathered, int32_t* counts, int32_t* support,
                                  void* values, int32_t* candidates, void* mu, void* stream) {
  return guarded([&] {
    if (!sk) throw InvalidArgument("null sketch");
    if ((indices == nullptr || gathered == nullptr) && B > 0)
      throw InvalidArgument("transform_gathered: indices and gathered columns are required");
    const Outputs o{counts, support, values, candidates, mu};
    if (sk->dtype == FSTG_F32)
      run_batch<float>(sk, X, B, p, nullptr, indices, o, static_cast<cudaStream_t>(stream), gathered);
    else
      run_batch<double>(sk, X, B, p, nullptr, indices, o, static_cast<cudaStream_t>(stream), gathered);
  });
}

int fstg_preprocess_shard(const void* a, int dtype, int64_t m, int64_t n, int device, void* stream,
                          int64_t basis_begin, int64_t basis_end, int include_identity, fstg_sketch** out) {
  return preprocess_impl(a, dtype, m, n, device, stream, basis_begin, basis_end, false, include_identity, out);
}

int fstg_sketch_info_get(const fstg_sketch* sk, fstg_sketch_info* info) {
  return guarded([&] {
    if (!sk || !info) throw InvalidArgument("null sketch/info");
    info->m = sk->m;
    info->n = sk->n;
    info->d = sk->design.d;
    info->L = sk->design.L;
    info->k = sk->design.k;
    info->dtype = sk->dtype;
    info->row_norm_max = sk->row_norm_max;
    info->device = sk->device;
    info->reserved = 0;
    info->column_stride = sk->ldc;
    info->device_bytes = sk->device_bytes;
    info->preprocess_ms = sk->preprocess_ms;
  });
}

int fstg_row_norm_max(const fstg_sketch* sk, double* out) {
  return guarded([&] {
    if (!sk || !out) throw InvalidArgument("null");
    *out = sk->row_norm_max;
  });
}

int fstg_sketch_embedded_matrix(const fstg_sketch* sk, void* out) {
  return guarded([&] {
    if (!sk || !out) throw InvalidArgument("null");
    if (!sk->has_a) throw CodedError(FSTG_ERR_NO_MATRIX, "Sketch: no embedded matrix");
    cuda_check(cudaSetDevice(sk->device), "cudaSetDevice");
    const size_t es = sk->dtype == FSTG_F32 ? 4 : 8;
    cuda_check(cudaMemcpy2D(out, size_t(sk->n) * es, sk->a, size_t(sk->lda) * es, size_t(sk->n) * es, size_t(sk->m),
                            is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost),
               "copy embedded matrix");
  });
}

int fstg_sketch_column(const fstg_sketch* sk, int64_t ell, void* out) {
  return guarded([&] {
    if (!sk || !out) throw InvalidArgument("null");
    if (ell < 0 || ell >= sk->design.L) throw OutOfRange("Sketch::column: index out of range");
    if (!sk->cols) throw InvalidArgument("Sketch::column: design-only sketch (use fstg_sample_columns)");
    cuda_check(cudaSetDevice(sk->device), "cudaSetDevice");
    const size_t es = dtype_size(sk->dtype);
    cuda_check(cudaMemcpy(out, static_cast<const char*>(sk->cols) + size_t(ell) * sk->ldc * es, size_t(sk->m) * es,
                          cudaMemcpyDefault),
               "copy column");
  });
}

int fstg_sketch_gather(const fstg_sketch* sk, const int64_t* indices, int64_t count, void* out, void* stream) {
  return guarded([&] {
    if (!sk || (count > 0 && (!indices || !out))) throw InvalidArgument("sketch_gather: null argument");
    if (count < 0) throw InvalidArgument("sketch_gather: negative count");
    if (count == 0) return;
    if (!sk->cols) throw InvalidArgument("sketch_gather: design-only sketch (use fstg_sample_columns)");
    cuda_check(cudaSetDevice(sk->device), "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t es = dtype_size(sk->dtype);
    DevBuf idx_buf, out_buf;
    const int64_t* idx = indices;
    if (!is_device_ptr(indices)) {
      idx_buf = DevBuf(size_t(count) * sizeof(int64_t), st);
      cuda_check(cudaMemcpyAsync(idx_buf.p, indices, size_t(count) * sizeof(int64_t), cudaMemcpyHostToDevice, st), "H2D");
      idx = idx_buf.as<int64_t>();
    }
    const bool out_dev = is_device_ptr(out);
    void* dst = out;
    if (!out_dev) {
      out_buf = DevBuf(size_t(count) * sk->m * es, st);
      dst = out_buf.p;
    }
    DevBuf bad(sizeof(int), st);
    cuda_check(cudaMemsetAsync(bad.p, 0, sizeof(int), st), "memset");
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(count, 148 * 16));
    {
      ProfScope ps("gather", st);
      if (sk->dtype == FSTG_F32)
        gather_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(sk->cols), sk->ldc, sk->m, idx, count,
                                                  sk->design.L, static_cast<float*>(dst), bad.as<int>());
      else
        gather_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(sk->cols), sk->ldc, sk->m, idx, count,
                                                   sk->design.L, static_cast<double*>(dst), bad.as<int>());
      cuda_check(cudaGetLastError(), "gather kernel");
    }
    int h = 0;
    cuda_check(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st), "copy flag");
    if (!out_dev) cuda_check(cudaMemcpyAsync(out, dst, size_t(count) * sk->m * es, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    if (h) throw OutOfRange("Sketch::column: index out of range");
  });
}

int fstg_sketch_device_columns(const fstg_sketch* sk, void** columns) {
  return guarded([&] {
    if (!sk || !columns) throw InvalidArgument("null");
    *columns = sk->cols;
  });
}

int fstg_sketch_preprocess_ms(const fstg_sketch* sk, double* ms) {
  return guarded([&] {
    if (!sk || !ms) throw InvalidArgument("null");
    *ms = sk->preprocess_ms;
  });
}

void fstg_destroy(fstg_sketch* sk) { destroy_sketch(sk); }

int fstg_save(const fstg_sketch* sk, const char* path, int version) {
  return guarded([&] { save_impl(sk, path, version); });
}

int fstg_load(const char* path, int dtype, int device, void* stream, fstg_sketch** out) {
  return guarded([&] { load_impl(path, dtype, device, stream, out); });
}

int fstg_draw_samples(const fstg_sketch* sk, const fstg_stream_params* p, const uint64_t* seeds, int64_t B,
                      int64_t* indices, void* stream) {
  return guarded([&] {
    if (!sk) throw InvalidArgument("null sketch");
    validate(p);
    if (B < 0 || (B > 0 && indices == nullptr)) throw InvalidArgument("draw_samples: bad output");
    if (B == 0) return;
    cuda_check(cudaSetDevice(sk->device), "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t N = p->J * p->K;
    const bool out_dev = is_device_ptr(indices);
    DevBuf sd_buf, out_buf;
    const uint64_t* sd = seeds;
    if (seeds != nullptr && !is_device_ptr(seeds)) {
      sd_buf = DevBuf(size_t(B) * sizeof(uint64_t), st);
      cuda_check(cudaMemcpyAsync(sd_buf.p, seeds, size_t(B) * sizeof(uint64_t), cudaMemcpyHostToDevice, st), "H2D");
      sd = sd_buf.as<uint64_t>();
    }
    int64_t* dst = indices;
    if (!out_dev) {
      out_buf = DevBuf(size_t(B) * N * sizeof(int64_t), st);
      dst = out_buf.as<int64_t>();
    }
    {
      ProfScope ps("draw", st);
      cuda_check(launch_draw<int64_t>(sd, p->seed, B, N, static_cast<uint64_t>(sk->design.L), dst, st), "draw");
    }
    if (!out_dev) {
      cuda_check(cudaMemcpyAsync(indices, dst, size_t(B) * N * sizeof(int64_t), cudaMemcpyDeviceToHost, st), "D2H");
      cuda_check(cudaStreamSynchronize(st), "sync");
    }
  });
}

int fstg_transform_batch(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                         const uint64_t* seeds, int32_t* counts, int32_t* support, void* values, int32_t* candidates,
                         void* mu, void* stream) {
  return guarded([&] {
    if (!sk) throw InvalidArgument("null sketch");
    const Outputs o{counts, support, values, candidates, mu};
    if (sk->dtype == FSTG_F32)
      run_batch<float>(sk, X, B, p, seeds, nullptr, o, static_cast<cudaStream_t>(stream));
    else
      run_batch<double>(sk, X, B, p, seeds, nullptr, o, static_cast<cudaStream_t>(stream));
  });
}

int fstg_transform_with_samples_batch(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                                      const int64_t* indices, int32_t* counts, int32_t* support, void* values,
                                      int32_t* candidates, void* mu, void* stream) {
  return guarded([&] {
    if (!sk) throw InvalidArgument("null sketch");
    if (indices == nullptr && B > 0) throw InvalidArgument("transform_with_samples: indices are null");
    const Outputs o{counts, support, values, candidates, mu};
    if (sk->dtype == FSTG_F32)
      run_batch<float>(sk, X, B, p, nullptr, indices, o, static_cast<cudaStream_t>(stream));
    else
      run_batch<double>(sk, X, B, p, nullptr, indices, o, static_cast<cudaStream_t>(stream));
  });
}

int fstg_profile_enable(int enable) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = enable != 0;
  return FSTG_OK;
}

int fstg_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  resolve_pending_locked();
  g_prof.clear();
  g_launches.store(0);
  return FSTG_OK;
}

int fstg_profile_read(const char* name, double* ms, int64_t* launches) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  resolve_pending_locked();
  auto it = g_prof.find(name ? name : "");
  if (ms) *ms = it == g_prof.end() ? 0.0 : it->second.ms;
  if (launches) *launches = it == g_prof.end() ? 0 : it->second.launches;
  return FSTG_OK;
}

int fstg_set_pool_retain(int retain) {
  return guarded([&] {
    g_pool_retain.store(retain != 0);
    if (retain == 0) {
      int n = 0, cur = 0;
      cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
      cuda_check(cudaGetDevice(&cur), "cudaGetDevice");  // the caller's current device is restored
      for (int dev = 0; dev < n; ++dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          cuda_check(cudaSetDevice(dev), "cudaSetDevice");
          cuda_check(cudaDeviceSynchronize(), "sync");
          cudaMemPoolTrimTo(pool, size_t(4) << 30);
        }
      }
      cudaGetLastError();
      cuda_check(cudaSetDevice(cur), "cudaSetDevice");
    }
  });
}

int fstg_launch_count(int64_t* launches) {
  if (launches) *launches = g_launches.load();
  return FSTG_OK;
}

int fstg_verify_mub(int k, int cap, int policy, int device, fstg_mub_report* out) {
  return guarded([&] { verify_mub_impl(k, cap, policy, device, out); });
}

int fstg_verify_design_moments(int k, int cap, int policy, int device, fstg_moment_report* out) {
  return guarded([&] { verify_moments_impl(k, cap, policy, device, out); });
}

double fstg_design_moment_target(int64_t d, int k) {  // kerdock.hpp:267-276
  double num = 1, den = 1;
  for (int i = 0; i < k; ++i) {
    num *= static_cast<double>(2 * i + 1);
    den *= static_cast<double>(d + 2 * i);
  }
  return num / den;
}

int fstg_verify_kerdock_set(int k, int device, int* skew_symmetric, int64_t* bad_pairs) {
  return guarded([&] { verify_kerdock_set_impl(k, device, skew_symmetric, bad_pairs); });
}

int fstg_transform_design_batch(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                                const uint64_t* seeds, int64_t row_block, int32_t* counts, int32_t* support,
                                void* values, int32_t* candidates, void* mu, void* stream) {
  return guarded([&] {
    if (!sk) throw InvalidArgument("null sketch");
    const Outputs o{counts, support, values, candidates, mu};
    if (sk->dtype == FSTG_F32)
      transform_design_impl<float>(sk, X, B, p, seeds, row_block, o, static_cast<cudaStream_t>(stream));
    else
      transform_design_impl<double>(sk, X, B, p, seeds, row_block, o, static_cast<cudaStream_t>(stream));
  });
}

int fstg_design_partial_means(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                              const uint64_t* seeds, int64_t row_begin, int64_t row_end, int64_t row_block,
                              void* means, int64_t vstride, int64_t ld, void* stream) {
  return guarded([&] {
    if (!sk) throw InvalidArgument("null sketch");
    if (B > 0 && (means == nullptr || !is_device_ptr(means))) throw InvalidArgument("design_partial_means: means must be device memory");
    if (seeds && !is_device_ptr(seeds)) throw InvalidArgument("design_partial_means: seeds must be device memory");
    const auto st = static_cast<cudaStream_t>(stream);
    if (sk->dtype == FSTG_F32) {
      DesignRun<float> run(sk, X, B, p, st);
      run.partial(seeds, row_begin, row_end, row_block, static_cast<float*>(means), vstride, ld);
    } else {
      DesignRun<double> run(sk, X, B, p, st);
      run.partial(seeds, row_begin, row_end, row_block, static_cast<double*>(means), vstride, ld);
    }
    cuda_check(cudaStreamSynchronize(st), "sync");
    trim_pool(sk->device, st);
  });
}

int fstg_transform_from_means(const fstg_sketch* sk, const void* X, int64_t B, const fstg_stream_params* p,
                              void* means, int64_t vstride, int64_t ld, int32_t* counts, int32_t* support, void* values,
                              int32_t* candidates, void* mu, void* stream) {
  return guarded([&] {
    if (!sk) throw InvalidArgument("null sketch");
    if (B > 0 && (means == nullptr || !is_device_ptr(means))) throw InvalidArgument("transform_from_means: means must be device memory");
    const Outputs o{counts, support, values, candidates, mu};
    const auto st = static_cast<cudaStream_t>(stream);
    if (sk->dtype == FSTG_F32) {
      DesignRun<float> run(sk, X, B, p, st);
      run.tail(static_cast<float*>(means), vstride, ld, o);
    } else {
      DesignRun<double> run(sk, X, B, p, st);
      run.tail(static_cast<double*>(means), vstride, ld, o);
    }
    cuda_check(cudaStreamSynchronize(st), "sync");
  });
}

int fstg_inner_product_with_design(int k, const double* x, int64_t n, int64_t ell, double* out, int device) {
  return guarded([&] { inner_product_impl(k, x, n, ell, out, device); });
}

int fstg_median_of_means(const double* samples, int64_t m, int64_t J, int64_t K, double* out, int device) {
  return guarded([&] { median_of_means_impl(samples, m, J, K, out, device); });
}

int fstg_hard_threshold(const double* v, int64_t len, double eps, double* out, int device) {
  return guarded([&] { hard_threshold_impl(v, len, eps, out, device); });
}

int fstg_projected_design_column(int k, int64_t n, int64_t ell, double* out, int device) {
  return guarded([&] { design_column_impl(k, n, ell, out, device); });
}

}  // extern "C"
