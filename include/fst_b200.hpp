// fst_b200.hpp — C++ mirror of the reference `fst` API for the thresholded-Ax
// hot path, implemented over the C-ABI in fst_b200.h (libfst_b200.so).
//
// Same names, argument meaning and exception classes as
// /root/reference/proj/include/fst/{sketch,stream}.hpp, minus Eigen: matrices
// are row-major spans (pointer + m + n), vectors are std::vector<double>.
//   fst::preprocess              sketch.hpp:149   -> fst_b200::preprocess
//   fst::Sketch                  sketch.hpp:70    -> fst_b200::Sketch (device-resident, move-only)
//   fst::StreamParams            stream.hpp:22    -> fst_b200::StreamParams
//   fst::choose_params           stream.hpp:58    -> fst_b200::choose_params
//   fst::draw_samples            stream.hpp:173   -> fst_b200::draw_samples
//   fst::transform               stream.hpp:272   -> fst_b200::transform
//   fst::transform_with_samples  stream.hpp:197   -> fst_b200::transform_with_samples
//   fst::TransformResult         stream.hpp:53    -> fst_b200::TransformResult
//   fst::save / fst::load        sketch.hpp:215,241 -> fst_b200::save / load (FSTK, into HBM)
//   inner_product_with_design, median_of_means, hard_threshold (stream.hpp:109-162),
//   projected_design_column (kerdock.hpp:156), verify_mub / verify_design_moments
// plus the batched entry points transform_batch / transform_design_batch. Errors are rethrown as
// std::invalid_argument / std::out_of_range / std::overflow_error /
// std::runtime_error exactly where the reference throws them; CUDA failures
// (no CPU fallback exists) throw fst_b200::cuda_error.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fst_b200.h"

namespace fst_b200 {

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct not_supported : std::runtime_error {
  using std::runtime_error::runtime_error;
};
/// io.hpp:23-37 IoError family (FSTK load/save)
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct MagicMismatchError : IoError {
  using IoError::IoError;
};
struct VersionUnsupportedError : IoError {
  using IoError::IoError;
};
struct TruncatedPayloadError : IoError {
  using IoError::IoError;
};
struct MalformedHeaderError : IoError {
  using IoError::IoError;
};

inline void check(int rc) {
  if (rc == FSTG_OK) return;
  const std::string msg = fstg_last_error();
  switch (rc) {
    case FSTG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case FSTG_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case FSTG_ERR_OVERFLOW: throw std::overflow_error(msg);
    case FSTG_ERR_RUNTIME: throw std::runtime_error(msg);
    case FSTG_ERR_NOT_SUPPORTED: throw not_supported(msg);
    case FSTG_ERR_IO: throw IoError(msg);
    case FSTG_ERR_MAGIC: throw MagicMismatchError(msg);
    case FSTG_ERR_VERSION: throw VersionUnsupportedError(msg);
    case FSTG_ERR_TRUNCATED: throw TruncatedPayloadError(msg);
    case FSTG_ERR_MALFORMED: throw MalformedHeaderError(msg);
    case FSTG_ERR_NO_MATRIX: throw std::logic_error(msg);  // sketch.hpp:109
    default: throw cuda_error(msg);
  }
}

/// stream.hpp:22-39
struct StreamParams {
  double epsilon = 0;
  double delta = 0;
  std::int64_t s = 1;
  std::int64_t J = 1;
  std::int64_t K = 1;
  std::int64_t widen = 10;
  std::uint64_t seed = 0;
  int mode = FSTG_MODE_DEFAULT;

  fstg_stream_params c() const { return {epsilon, delta, s, J, K, widen, seed, mode, 0}; }
  void validate() const {
    const fstg_stream_params p = c();
    check(fstg_validate_params(&p));
  }
};

/// stream.hpp:41-54 (values are double for an fp64 sketch, widened from fp32 otherwise)
struct TransformResult {
  std::vector<std::int64_t> support;
  std::vector<double> values;
  std::vector<std::int64_t> candidate_set;
  std::vector<double> mu;
  std::int64_t samples_used = 0;
};

/// sketch.hpp:70-142 — owns the device-resident sketch; immutable, move-only.
class Sketch {
 public:
  Sketch() = default;
  explicit Sketch(fstg_sketch* h) : h_(h) { check(fstg_sketch_info_get(h_, &info_)); }
  Sketch(Sketch&& o) noexcept : h_(o.h_), info_(o.info_) { o.h_ = nullptr; }
  Sketch& operator=(Sketch&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = o.h_;
      info_ = o.info_;
      o.h_ = nullptr;
    }
    return *this;
  }
  Sketch(const Sketch&) = delete;
  Sketch& operator=(const Sketch&) = delete;
  ~Sketch() { reset(); }

  std::int64_t m() const { return info_.m; }
  std::int64_t n() const { return info_.n; }
  int k() const { return info_.k; }
  std::int64_t d() const { return info_.d; }
  std::int64_t L() const { return info_.L; }
  bool is_f64() const { return info_.dtype == FSTG_F64; }
  double row_norm_max() const { return info_.row_norm_max; }
  double preprocess_ms() const { return info_.preprocess_ms; }
  const fstg_sketch* handle() const { return h_; }

  /// Sketch::column (sketch.hpp:114-117), copied to the host as double.
  std::vector<double> column(std::int64_t ell) const {
    std::vector<double> out(static_cast<std::size_t>(m()));
    if (is_f64()) {
      check(fstg_sketch_column(h_, ell, out.data()));
    } else {
      std::vector<float> f(out.size());
      check(fstg_sketch_column(h_, ell, f.data()));
      for (std::size_t i = 0; i < f.size(); ++i) out[i] = f[i];
    }
    return out;
  }

  /// Sketch::embedded_matrix (sketch.hpp:107-111): A, m x n row-major, as double.
  std::vector<double> embedded_matrix() const {
    std::vector<double> out(static_cast<std::size_t>(m() * n()));
    if (is_f64()) {
      check(fstg_sketch_embedded_matrix(h_, out.data()));
    } else {
      std::vector<float> f(out.size());
      check(fstg_sketch_embedded_matrix(h_, f.data()));
      for (std::size_t i = 0; i < f.size(); ++i) out[i] = f[i];
    }
    return out;
  }

  /// Retain-sampled columns A s_ell (any sketch, including a design-only one):
  /// indices.size() x m, row j = column indices[j], as double.
  std::vector<double> sample_columns(const std::vector<std::int64_t>& indices) const {
    const std::int64_t ldc = info_.column_stride;
    std::vector<double> out(indices.size() * static_cast<std::size_t>(m()));
    if (is_f64()) {
      std::vector<double> buf(indices.size() * static_cast<std::size_t>(ldc));
      check(fstg_sample_columns(h_, indices.data(), static_cast<std::int64_t>(indices.size()), buf.data(), nullptr));
      for (std::size_t j = 0; j < indices.size(); ++j)
        for (std::int64_t i = 0; i < m(); ++i) out[j * m() + i] = buf[j * ldc + i];
    } else {
      std::vector<float> buf(indices.size() * static_cast<std::size_t>(ldc));
      check(fstg_sample_columns(h_, indices.data(), static_cast<std::int64_t>(indices.size()), buf.data(), nullptr));
      for (std::size_t j = 0; j < indices.size(); ++j)
        for (std::int64_t i = 0; i < m(); ++i) out[j * m() + i] = buf[j * ldc + i];
    }
    return out;
  }

 private:
  void reset() {
    if (h_) fstg_destroy(h_);
    h_ = nullptr;
  }
  fstg_sketch* h_ = nullptr;
  fstg_sketch_info info_{};
};

/// sketch.hpp:149-211 on device `device`; `a` is m x n row-major double.
inline Sketch preprocess(const double* a, std::int64_t m, std::int64_t n, int device = 0) {
  fstg_sketch* h = nullptr;
  check(fstg_preprocess(a, FSTG_F64, m, n, device, nullptr, &h));
  return Sketch(h);
}
/// fp32 sketch (the B200 headline configuration).
inline Sketch preprocess(const float* a, std::int64_t m, std::int64_t n, int device = 0) {
  fstg_sketch* h = nullptr;
  check(fstg_preprocess(a, FSTG_F32, m, n, device, nullptr, &h));
  return Sketch(h);
}

/// Design-only sketch (embedded A + Kerdock tables, no columns) for n whose sketch
/// cannot exist (n = 16384); use sample_columns / transform_design_batch on it.
inline Sketch preprocess_design(const float* a, std::int64_t m, std::int64_t n, int device = 0) {
  fstg_sketch* h = nullptr;
  check(fstg_preprocess_design(a, FSTG_F32, m, n, device, nullptr, &h));
  return Sketch(h);
}

/// sketch.hpp:215-232: FSTK v1 (float64, the reference's file) or v2 (float32).
inline void save(const Sketch& sk, const std::string& path, int version = 1) {
  check(fstg_save(sk.handle(), path.c_str(), version));
}
/// sketch.hpp:241-302 straight into HBM (dtype FSTG_F64 or FSTG_F32).
inline Sketch load(const std::string& path, int dtype = FSTG_F64, int device = 0) {
  fstg_sketch* h = nullptr;
  check(fstg_load(path.c_str(), dtype, device, nullptr, &h));
  return Sketch(h);
}

/// stream.hpp:109-121 (Kerdock index: the reference's Gray-code walk, bit-exact).
inline double inner_product_with_design(const std::vector<double>& x, int k, std::int64_t ell, int device = 0) {
  double out = 0;
  check(fstg_inner_product_with_design(k, x.data(), static_cast<std::int64_t>(x.size()), ell, &out, device));
  return out;
}
/// stream.hpp:147-155: samples m x (J*K), column-major (column j at j*m).
inline std::vector<double> median_of_means(const std::vector<double>& samples, std::int64_t m, std::int64_t J,
                                           std::int64_t K, int device = 0) {
  if (J < 1 || K < 1 || static_cast<std::int64_t>(samples.size()) != m * J * K)
    throw std::invalid_argument("median_of_means: samples must have J*K columns");
  std::vector<double> out(static_cast<std::size_t>(m));
  check(fstg_median_of_means(samples.data(), m, J, K, out.data(), device));
  return out;
}
/// stream.hpp:158-162
inline std::vector<double> hard_threshold(const std::vector<double>& v, double eps, int device = 0) {
  std::vector<double> out(v.size());
  check(fstg_hard_threshold(v.data(), static_cast<std::int64_t>(v.size()), eps, out.data(), device));
  return out;
}
/// kerdock.hpp:156-167
inline std::vector<double> projected_design_column(int k, std::int64_t n, std::int64_t ell, int device = 0) {
  std::vector<double> out(static_cast<std::size_t>(n));
  check(fstg_projected_design_column(k, n, ell, out.data(), device));
  return out;
}

/// stream.hpp:58-69
inline std::pair<std::int64_t, std::int64_t> choose_params(double row_norm_max, double gamma, double eta,
                                                           std::int64_t m) {
  std::int64_t J = 0, K = 0;
  check(fstg_choose_params(row_norm_max, gamma, eta, m, &J, &K));
  return {J, K};
}

/// stream.hpp:173-182
inline std::vector<std::int64_t> draw_samples(const Sketch& sk, const StreamParams& p) {
  p.validate();
  std::vector<std::int64_t> out(static_cast<std::size_t>(p.J * p.K));
  const fstg_stream_params c = p.c();
  check(fstg_draw_samples(sk.handle(), &c, &p.seed, 1, out.data(), nullptr));
  return out;
}

namespace detail {
template <typename T>
TransformResult run_one(const Sketch& sk, const std::vector<T>& x, const StreamParams& p,
                        const std::vector<std::int64_t>* indices) {
  if (static_cast<std::int64_t>(x.size()) != sk.n())
    throw std::invalid_argument("transform: vector length does not match sketch");
  p.validate();
  const std::int64_t want = fstg_candidate_count(p.s, p.widen, sk.m());
  std::int32_t count = 0;
  std::vector<std::int32_t> support(static_cast<std::size_t>(want)), cand(static_cast<std::size_t>(want));
  std::vector<T> values(static_cast<std::size_t>(want)), mu(static_cast<std::size_t>(sk.m()));
  const fstg_stream_params c = p.c();
  if (indices)
    check(fstg_transform_with_samples_batch(sk.handle(), x.data(), 1, &c, indices->data(), &count, support.data(),
                                            values.data(), cand.data(), mu.data(), nullptr));
  else
    check(fstg_transform_batch(sk.handle(), x.data(), 1, &c, &p.seed, &count, support.data(), values.data(),
                               cand.data(), mu.data(), nullptr));
  TransformResult r;
  r.support.assign(support.begin(), support.begin() + count);
  r.values.assign(values.begin(), values.begin() + count);
  r.candidate_set.assign(cand.begin(), cand.end());
  r.mu.assign(mu.begin(), mu.end());
  r.samples_used = p.J * p.K;
  return r;
}
}  // namespace detail

/// stream.hpp:272-275 (x must match the sketch dtype: double for fp64, float for fp32)
inline TransformResult transform(const Sketch& sk, const std::vector<double>& x, const StreamParams& p) {
  if (!sk.is_f64()) throw std::invalid_argument("transform: fp32 sketch needs a float vector");
  return detail::run_one(sk, x, p, nullptr);
}
inline TransformResult transform(const Sketch& sk, const std::vector<float>& x, const StreamParams& p) {
  if (sk.is_f64()) throw std::invalid_argument("transform: fp64 sketch needs a double vector");
  return detail::run_one(sk, x, p, nullptr);
}

/// stream.hpp:197-268
inline TransformResult transform_with_samples(const Sketch& sk, const std::vector<double>& x, const StreamParams& p,
                                              const std::vector<std::int64_t>& indices) {
  if (static_cast<std::int64_t>(indices.size()) != p.J * p.K)
    throw std::invalid_argument("transform: drawn sample count does not match J*K");
  return detail::run_one(sk, x, p, &indices);
}

/// The batched stream: X is B x n row-major (host or device memory, sketch
/// dtype); per-vector seeds; outputs as documented in fst_b200.h.
inline void transform_batch(const Sketch& sk, const void* X, std::int64_t B, const StreamParams& p,
                            const std::uint64_t* seeds, std::int32_t* counts, std::int32_t* support, void* values,
                            void* stream = nullptr) {
  const fstg_stream_params c = p.c();
  check(fstg_transform_batch(sk.handle(), X, B, &c, seeds, counts, support, values, nullptr, nullptr, stream));
}

/// The batched stream on a design-only sketch (row blocks of sampled columns;
/// device memory; bit-identical to transform_batch on the full sketch).
inline void transform_design_batch(const Sketch& sk, const void* X, std::int64_t B, const StreamParams& p,
                                   const std::uint64_t* seeds, std::int32_t* counts, std::int32_t* support,
                                   void* values, std::int64_t row_block = 0, void* stream = nullptr) {
  const fstg_stream_params c = p.c();
  check(fstg_transform_design_batch(sk.handle(), X, B, &c, seeds, row_block, counts, support, values, nullptr,
                                    nullptr, stream));
}

// kerdock.hpp:198-317 design verifiers (GPU; policy FSTG_VERIFY_REFERENCE
// reproduces the reference's reports, FSTG_VERIFY_EXHAUSTIVE checks every pair).
using MubReport = fstg_mub_report;
using MomentReport = fstg_moment_report;

inline MubReport verify_mub(int k, int cap = 8, int policy = FSTG_VERIFY_REFERENCE, int device = 0) {
  MubReport r{};
  check(fstg_verify_mub(k, cap, policy, device, &r));
  return r;
}

inline MomentReport verify_design_moments(int k, int cap = 8, int policy = FSTG_VERIFY_REFERENCE, int device = 0) {
  MomentReport r{};
  check(fstg_verify_design_moments(k, cap, policy, device, &r));
  return r;
}

inline double design_moment_target(std::int64_t d, int k) { return fstg_design_moment_target(d, k); }

}  // namespace fst_b200
