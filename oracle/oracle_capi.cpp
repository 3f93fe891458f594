// ORACLE — TEST INFRASTRUCTURE ONLY. Flat C entry points over fst_oracle so
// tests/ and bench.py's CPU legs can drive the restatement through ctypes.
// Status codes mirror the reference's exception classes:
//   0 ok, 1 std::invalid_argument, 2 std::out_of_range, 3 std::overflow_error,
//   4 std::runtime_error, 5 std::logic_error / other.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "fst_oracle.hpp"

using namespace fst_oracle;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::overflow_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

StreamParams make_params(double eps, double delta, std::int64_t s, std::int64_t J, std::int64_t K,
                         std::int64_t widen, std::uint64_t seed) {
  StreamParams p;
  p.epsilon = eps;
  p.delta = delta;
  p.s = s;
  p.J = J;
  p.K = K;
  p.widen = widen;
  p.seed = seed;
  return p;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_modulus_for_degree(int q, std::uint64_t* out) {
  return guarded([&] { *out = modulus_for_degree(q); });
}
int orc_verify_irreducible(std::uint64_t poly, int degree, int* out) {
  return guarded([&] { *out = verify_irreducible(poly, degree) ? 1 : 0; });
}
int orc_field_mul(int q, std::uint64_t a, std::uint64_t b, std::uint64_t* out) {
  return guarded([&] { *out = field_mul(q, modulus_for_degree(q), a, b); });
}
int orc_field_trace(int q, std::uint64_t a, int* out) {
  return guarded([&] { *out = field_trace(q, modulus_for_degree(q), a); });
}
int orc_gf2_rank(const std::uint64_t* rows, int dim) { return gf2_rank(rows, dim); }
std::uint64_t orc_coords_of_position(std::uint64_t p, int k) { return coords_of_position(p, k); }
std::uint64_t orc_position_of_coords(std::uint64_t w, int k) { return position_of_coords(w, k); }

int orc_design_params(int k, std::int64_t* d, std::int64_t* L) {
  return guarded([&] {
    const DesignParams p = DesignParams::make(k);
    *d = p.d;
    *L = p.L;
  });
}
int orc_kerdock_matrix(int k, std::uint64_t s, std::uint64_t* rows_out) {
  return guarded([&] {
    const auto m = kerdock_matrix(DesignParams::make(k), s);
    std::memcpy(rows_out, m.data(), sizeof(std::uint64_t) * m.size());
  });
}
int orc_quadratic_form(const std::uint64_t* rows, int dim, std::uint64_t x) { return quadratic_form(rows, dim, x); }
int orc_reversed_q_rows(const std::uint64_t* rows, int k, std::uint64_t* rev) {
  reversed_q_rows(rows, k, rev);
  return 0;
}
int orc_decode_index(int k, std::int64_t ell, int* identity, std::uint64_t* s, std::uint64_t* wpos) {
  return guarded([&] {
    const auto r = decode_index(DesignParams::make(k), ell);
    *identity = r.identity ? 1 : 0;
    *s = r.s;
    *wpos = r.wpos;
  });
}
int orc_projected_design_column(int k, std::int64_t n, std::int64_t ell, double* out) {
  return guarded([&] {
    const auto v = projected_design_column(DesignParams::make(k), n, ell);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}
int orc_even_log2_ceil(std::int64_t n, int* out) {
  return guarded([&] { *out = even_log2_ceil(n); });
}
int orc_fwht_unnormalized_f64(double* data, std::size_t len) {
  return guarded([&] { fwht_unnormalized(data, len); });
}
int orc_fwht_unnormalized_f32(float* data, std::size_t len) {
  return guarded([&] { fwht_unnormalized(data, len); });
}
int orc_fwht_normalized_f64(double* data, std::size_t len) {
  return guarded([&] { fwht_normalized(data, len); });
}

// ---- sketch handles (owned by the oracle; freed by orc_sketch_free) ----
struct OrcSketch {
  int dtype;  // 0 f32, 1 f64
  Sketch<double> d;
  Sketch<float> f;
};

int orc_preprocess(const void* a, int dtype, std::int64_t m, std::int64_t n, int threads, void** out) {
  return guarded([&] {
    auto* h = new OrcSketch();
    h->dtype = dtype;
    try {
      if (dtype == 1)
        h->d = preprocess<double>(static_cast<const double*>(a), m, n, threads);
      else
        h->f = preprocess<float>(static_cast<const float*>(a), m, n, threads);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void orc_sketch_free(void* h) { delete static_cast<OrcSketch*>(h); }
int orc_sketch_info(void* hv, std::int64_t* m, std::int64_t* n, int* k, std::int64_t* d, std::int64_t* L,
                    double* row_norm_max) {
  auto* h = static_cast<OrcSketch*>(hv);
  const DesignParams& p = h->dtype == 1 ? h->d.design : h->f.design;
  *m = h->dtype == 1 ? h->d.m : h->f.m;
  *n = h->dtype == 1 ? h->d.n : h->f.n;
  *k = p.k;
  *d = p.d;
  *L = p.L;
  *row_norm_max = h->dtype == 1 ? h->d.row_norm_max : h->f.row_norm_max;
  return 0;
}
const void* orc_sketch_columns(void* hv) {
  auto* h = static_cast<OrcSketch*>(hv);
  return h->dtype == 1 ? static_cast<const void*>(h->d.columns.data()) : static_cast<const void*>(h->f.columns.data());
}
int orc_sketch_column(void* hv, std::int64_t ell, void* out) {
  return guarded([&] {
    auto* h = static_cast<OrcSketch*>(hv);
    if (h->dtype == 1)
      std::memcpy(out, h->d.column(ell), sizeof(double) * h->d.m);
    else
      std::memcpy(out, h->f.column(ell), sizeof(float) * h->f.m);
  });
}

// ---- rng ----
int orc_rng_u64(std::uint64_t seed, std::int64_t count, std::uint64_t* out) {
  SeededRng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.next_u64();
  return 0;
}
int orc_rng_index(std::uint64_t seed, std::uint64_t bound, std::int64_t count, std::uint64_t* out) {
  SeededRng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.index(bound);
  return 0;
}
int orc_rng_gaussian(std::uint64_t seed, std::int64_t count, double* out) {
  SeededRng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.gaussian();
  return 0;
}
int orc_rng_unit_double(std::uint64_t seed, std::int64_t count, double* out) {
  SeededRng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.unit_double();
  return 0;
}
int orc_rng_coin(std::uint64_t seed, std::int64_t count, std::uint8_t* out) {
  SeededRng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.coin() ? 1 : 0;
  return 0;
}
std::uint64_t orc_mix_seed(std::uint64_t z) { return mix_seed(z); }
std::uint64_t orc_gen_seed(std::uint64_t t) { return gen_seed(t); }
std::uint64_t orc_stream_seed(std::uint64_t t) { return stream_seed(t); }

// ---- stream ----
int orc_choose_params(double r, double gamma, double eta, std::int64_t m, std::int64_t* J, std::int64_t* K) {
  return guarded([&] {
    const auto jk = choose_params(r, gamma, eta, m);
    *J = jk.first;
    *K = jk.second;
  });
}
int orc_validate_params(double eps, double delta, std::int64_t s, std::int64_t J, std::int64_t K,
                        std::int64_t widen) {
  return guarded([&] { make_params(eps, delta, s, J, K, widen, 0).validate(); });
}
int orc_inner_product_with_design(const double* x, std::int64_t n, int k, std::int64_t ell, double* out) {
  return guarded([&] { *out = inner_product_with_design(x, n, DesignParams::make(k), ell); });
}
int orc_median_of_batch_means_f64(const double* means, std::int64_t m, std::int64_t K, double* mu) {
  return guarded([&] {
    const auto v = median_of_batch_means(means, m, K);
    std::memcpy(mu, v.data(), sizeof(double) * v.size());
  });
}
int orc_draw_samples(std::int64_t L, double eps, double delta, std::int64_t s, std::int64_t J, std::int64_t K,
                     std::int64_t widen, std::uint64_t seed, std::int64_t* out) {
  return guarded([&] {
    const auto v = draw_samples(L, make_params(eps, delta, s, J, K, widen, seed));
    std::memcpy(out, v.data(), sizeof(std::int64_t) * v.size());
  });
}
std::int64_t orc_candidate_count(std::int64_t s, std::int64_t widen, std::int64_t m) {
  return candidate_count(s, widen, m);
}

// Runs transform_with_samples (indices==nullptr -> draw_samples first).
// Outputs: mu[m], candidates[want], support[<=want], values[<=want], *nsupport.
int orc_transform(void* hv, const void* x, double eps, double delta, std::int64_t s, std::int64_t J,
                  std::int64_t K, std::int64_t widen, std::uint64_t seed, const std::int64_t* indices,
                  void* mu_out, std::int64_t* cand_out, std::int64_t* support_out, void* values_out,
                  std::int64_t* nsupport) {
  return guarded([&] {
    auto* h = static_cast<OrcSketch*>(hv);
    const StreamParams p = make_params(eps, delta, s, J, K, widen, seed);
    p.validate();
    const std::int64_t L = h->dtype == 1 ? h->d.design.L : h->f.design.L;
    std::vector<std::int64_t> idx;
    if (indices)
      idx.assign(indices, indices + p.J * p.K);
    else
      idx = draw_samples(L, p);
    auto emit = [&](const auto& r, auto* mu, auto* vals) {
      if (mu) std::memcpy(mu, r.mu.data(), sizeof(r.mu[0]) * r.mu.size());
      if (cand_out) std::memcpy(cand_out, r.candidate_set.data(), sizeof(std::int64_t) * r.candidate_set.size());
      if (support_out) std::memcpy(support_out, r.support.data(), sizeof(std::int64_t) * r.support.size());
      if (vals) std::memcpy(vals, r.values.data(), sizeof(r.values[0]) * r.values.size());
      *nsupport = static_cast<std::int64_t>(r.support.size());
    };
    if (h->dtype == 1)
      emit(transform_with_samples(h->d, static_cast<const double*>(x), p, idx), static_cast<double*>(mu_out),
           static_cast<double*>(values_out));
    else
      emit(transform_with_samples(h->f, static_cast<const float*>(x), p, idx), static_cast<float*>(mu_out),
           static_cast<float*>(values_out));
  });
}

// Stream of B vectors (row-major B x n) over T threads, each thread calling
// transform() on the shared read-only sketch (safe per test_stream.cpp:342-373).
// Per-vector seeds; only the support counts are returned. Returns wall seconds.
int orc_transform_stream(void* hv, const void* X, std::int64_t B, double eps, double delta, std::int64_t s,
                         std::int64_t J, std::int64_t K, std::int64_t widen, const std::uint64_t* seeds,
                         int threads, std::int64_t* counts_out, double* seconds) {
  return guarded([&] {
    auto* h = static_cast<OrcSketch*>(hv);
    const std::int64_t n = h->dtype == 1 ? h->d.n : h->f.n;
    const std::int64_t L = h->dtype == 1 ? h->d.design.L : h->f.design.L;
    const auto t0 = std::chrono::steady_clock::now();
    auto work = [&](std::int64_t first, std::int64_t last) {
      for (std::int64_t v = first; v < last; ++v) {
        StreamParams p = make_params(eps, delta, s, J, K, widen, seeds[v]);
        const auto idx = draw_samples(L, p);
        if (h->dtype == 1)
          counts_out[v] = static_cast<std::int64_t>(
              transform_with_samples(h->d, static_cast<const double*>(X) + v * n, p, idx).support.size());
        else
          counts_out[v] = static_cast<std::int64_t>(
              transform_with_samples(h->f, static_cast<const float*>(X) + v * n, p, idx).support.size());
      }
    };
    threads = std::max(1, threads);
    std::vector<std::thread> pool;
    const std::int64_t per = (B + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
      const std::int64_t f = t * per, l = std::min(B, f + per);
      if (f >= l) break;
      pool.emplace_back([&work, f, l] { work(f, l); });
    }
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

}  // extern "C"

template <typename T>
static void transform_gathered_out(const T* a, std::int64_t m, std::int64_t n, const T* x, const StreamParams& p,
                                   const std::int64_t* indices, const T* gathered, T* mu_out,
                                   std::int64_t* cand_out, std::int64_t* support_out, T* values_out,
                                   std::int64_t* nsupport) {
  p.validate();
  const std::vector<std::int64_t> idx(indices, indices + p.J * p.K);
  const auto r = transform_gathered<T>(a, m, n, x, p, idx, gathered);
  std::memcpy(mu_out, r.mu.data(), sizeof(T) * r.mu.size());
  std::memcpy(cand_out, r.candidate_set.data(), sizeof(std::int64_t) * r.candidate_set.size());
  std::memcpy(support_out, r.support.data(), sizeof(std::int64_t) * r.support.size());
  std::memcpy(values_out, r.values.data(), sizeof(T) * r.values.size());
  *nsupport = static_cast<std::int64_t>(r.support.size());
}

extern "C" {

int orc_transform_gathered(const double* a, std::int64_t m, std::int64_t n, const double* x, double eps,
                           double delta, std::int64_t s, std::int64_t J, std::int64_t K, std::int64_t widen,
                           const std::int64_t* indices, const double* gathered, double* mu_out,
                           std::int64_t* cand_out, std::int64_t* support_out, double* values_out,
                           std::int64_t* nsupport) {
  return guarded([&] {
    transform_gathered_out<double>(a, m, n, x, make_params(eps, delta, s, J, K, widen, 0), indices, gathered,
                                   mu_out, cand_out, support_out, values_out, nsupport);
  });
}

// The same draw_and_gather transform run in float (the reference arithmetic
// with Scalar = float: every product and sum rounded to fp32).
int orc_transform_gathered_f32(const float* a, std::int64_t m, std::int64_t n, const float* x, double eps,
                               double delta, std::int64_t s, std::int64_t J, std::int64_t K, std::int64_t widen,
                               const std::int64_t* indices, const float* gathered, float* mu_out,
                               std::int64_t* cand_out, std::int64_t* support_out, float* values_out,
                               std::int64_t* nsupport) {
  return guarded([&] {
    transform_gathered_out<float>(a, m, n, x, make_params(eps, delta, s, J, K, widen, 0), indices, gathered,
                                  mu_out, cand_out, support_out, values_out, nsupport);
  });
}

// One Kerdock basis block of the sketch (sketch.hpp:171-196 for a single s):
// out is column-major d x m (column w of the block at w*m), dtype 0 = f32, 1 = f64.
int orc_kerdock_block(const void* a, int dtype, std::int64_t m, std::int64_t n, std::int64_t s, void* out) {
  return guarded([&] {
    const DesignParams p = DesignParams::make(even_log2_ceil(n));
    if (s < 0 || s >= p.kerdock_bases()) throw std::out_of_range("kerdock_block: basis out of range");
    const auto mat = kerdock_matrix(p, static_cast<std::uint64_t>(s));
    if (dtype == 1) {
      std::vector<double> sign, tile;
      kerdock_block(static_cast<const double*>(a), m, n, p, mat.data(), static_cast<double*>(out), sign, tile);
    } else {
      std::vector<float> sign, tile;
      kerdock_block(static_cast<const float*>(a), m, n, p, mat.data(), static_cast<float*>(out), sign, tile);
    }
  });
}

double orc_design_moment_target(std::int64_t d, int k) { return design_moment_target(d, k); }
int orc_verify_kerdock_set(int k, int* skew, std::int64_t* bad_pairs) {
  return guarded([&] {
    bool ok = false;
    verify_kerdock_set(DesignParams::make(k), &ok, bad_pairs);
    *skew = ok ? 1 : 0;
  });
}

// Reference preprocessing timed on a bounded sample (bench.py's CPU leg): the
// first `bases` Kerdock bases of A's sketch (kerdock_matrix + kerdock_block,
// the reference's per-basis work) spread over `threads` threads, each writing
// into its own basis-sized scratch block. Wall seconds.
int orc_bench_preprocess(const double* a, std::int64_t m, std::int64_t n, std::int64_t bases, int threads,
                         double* seconds) {
  return guarded([&] {
    const DesignParams p = DesignParams::make(even_log2_ceil(n));
    bases = std::min<std::int64_t>(bases, p.kerdock_bases());
    threads = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(threads, bases)));
    std::vector<std::vector<double>> blocks(static_cast<std::size_t>(threads));
    for (auto& b : blocks) b.assign(static_cast<std::size_t>(p.d * m), 0.0);  // touched before timing
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        std::vector<double> sign, tile;
        for (std::int64_t s = t; s < bases; s += threads) {
          const auto mat = kerdock_matrix(p, static_cast<std::uint64_t>(s));
          kerdock_block(a, m, n, p, mat.data(), blocks[t].data(), sign, tile);
        }
      });
    }
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

}  // extern "C"
