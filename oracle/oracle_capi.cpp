// ORACLE — TEST INFRASTRUCTURE ONLY. Flat C entry points over fst_oracle so
// tests/ and bench.py's CPU legs can drive the restatement through ctypes.
// Status codes mirror the reference's exception classes:
//   0 ok, 1 std::invalid_argument, 2 std::out_of_range, 3 std::overflow_error,
//   4 std::runtime_error, 5 std::logic_error / other.
#include <algorithm>
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
// B sparse target vectors y (B x m, row-major) for the BASELINE configs: vector v
// draws from SeededRng(seeds[v]) the s distinct rows of gen_exact_sparse
// (generators.hpp:44-53: partial Fisher-Yates with index(m - i)), each value
// +-1/sqrt(s) by coin (value_kind 0) or gaussian() (value_kind 1), then, if
// noise_sigma > 0, noise_sigma * gaussian() added to every row in order (the
// configs' dense-noise extension; the reference has no noise generator).
// Threads over vectors; each vector's stream is independent of the split.
int orc_gen_sparse_targets(const std::uint64_t* seeds, std::int64_t B, std::int64_t m, std::int64_t s,
                           int value_kind, double noise_sigma, int threads, double* Y) {
  return guarded([&] {
    if (B < 0 || m < 1 || s < 1 || s > m || value_kind < 0 || value_kind > 1)
      throw std::invalid_argument("gen_sparse_targets: bad arguments");
    const double mag = 1.0 / std::sqrt(static_cast<double>(s));
    auto work = [&](std::int64_t first, std::int64_t last) {
      std::vector<std::int64_t> perm(static_cast<std::size_t>(m));
      for (std::int64_t v = first; v < last; ++v) {
        SeededRng rng(seeds[v]);
        double* y = Y + v * m;
        std::fill(y, y + m, 0.0);
        std::iota(perm.begin(), perm.end(), std::int64_t{0});
        for (std::int64_t i = 0; i < s; ++i) {
          const auto j = i + static_cast<std::int64_t>(rng.index(static_cast<std::uint64_t>(m - i)));
          std::swap(perm[i], perm[j]);
          y[perm[i]] = value_kind == 0 ? (rng.coin() ? mag : -mag) : rng.gaussian();
        }
        if (noise_sigma > 0)
          for (std::int64_t i = 0; i < m; ++i) y[i] += noise_sigma * rng.gaussian();
      }
    };
    threads = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(threads, B)));
    std::vector<std::thread> pool;
    const std::int64_t per = (B + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
      const std::int64_t f = t * per, l = std::min(B, f + per);
      if (f < l) pool.emplace_back([&work, f, l] { work(f, l); });
    }
    for (auto& th : pool) th.join();
  });
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

// ---------------------------------------------------------------------------
// The B200 FAST-mode arithmetic, restated (test infrastructure): the same
// transform as transform_gathered<float> (stream.hpp:197-268) with the
// summation orders of the sm_100a kernels instead of the reference's, so the
// fp32 FAST path can be checked bit for bit rather than to a tolerance:
//  * coefficient t = s_ell^T x (stream.cu coeff_fast_multi, d >= 128): lane l
//    of a warp visits x[128 i + 4 l + e] for i ascending, e = 0..3 (positions
//    >= n read as 0), summing all of them into tot and the negatively signed
//    ones into neg; its partial is fmaf(-2, neg, tot); the 32 lane partials are
//    combined by the xor butterfly (offsets 16, 8, 4, 2, 1). d < 128
//    (coeff_generic): lane l sums +-x[l + 32 r]. Identity indices:
//    float(sqrt(d)) * x[pos].
//  * accumulation: acc = fmaf(t, C[i, ell], acc) per element in j order (FAST
//    uses FMA), batch mean acc / J, median as the reference (stream.hpp:126-143).
//  * candidate rule and threshold as the reference (stream.hpp:245-266);
//    refined value (stream.cu refine_dot_exact): exact products in fp64, lane l
//    accumulating 4-element chunks q = l + 32 i into two chains by i parity,
//    chains added, xor butterfly; stored as float, |v| >= eps tested in double.
static float lane_tree_f(float (&a)[32]) {
  for (int o = 16; o > 0; o >>= 1) {
    float b[32];
    for (int l = 0; l < 32; ++l) b[l] = a[l] + a[l ^ o];
    std::memcpy(a, b, sizeof(b));
  }
  return a[0];
}
static double lane_tree_d(double (&a)[32]) {
  for (int o = 16; o > 0; o >>= 1) {
    double b[32];
    for (int l = 0; l < 32; ++l) b[l] = a[l] + a[l ^ o];
    std::memcpy(a, b, sizeof(b));
  }
  return a[0];
}

static void transform_gathered_fast_order(const float* a, std::int64_t m, std::int64_t n, const float* x,
                                          const StreamParams& p, const std::int64_t* indices, const float* gathered,
                                          float* mu_out, std::int64_t* cand_out, std::int64_t* support_out,
                                          float* values_out, std::int64_t* nsupport) {
  p.validate();
  const DesignParams design = DesignParams::make(even_log2_ceil(n));
  const std::int64_t d = design.d, kb = design.kerdock_bases() * d, N = p.J * p.K;
  std::vector<float> xs(static_cast<std::size_t>(d), 0.f);
  for (std::int64_t i = 0; i < n; ++i) xs[i] = x[i];
  std::vector<std::uint8_t> q(static_cast<std::size_t>(d));
  std::int64_t cached = -1;
  std::vector<float> means(static_cast<std::size_t>(m * p.K), 0.f);
  for (std::int64_t jj = 0; jj < N; ++jj) {
    const std::int64_t ell = indices[jj];
    if (ell < 0 || ell >= design.L) throw std::out_of_range("Sketch::column: index out of range");
    float t;
    if (ell >= kb) {
      const std::int64_t pos = ell - kb;
      t = pos < n ? static_cast<float>(std::sqrt(static_cast<double>(d))) * xs[pos] : 0.f;
    } else {
      const std::int64_t s = ell / d;
      const std::uint64_t w = static_cast<std::uint64_t>(ell % d);
      if (s != cached) {
        const auto mat = kerdock_matrix(design, static_cast<std::uint64_t>(s));
        for (std::int64_t pos = 0; pos < d; ++pos)
          q[pos] = static_cast<std::uint8_t>(
              quadratic_form(mat.data(), design.k, coords_of_position(static_cast<std::uint64_t>(pos), design.k)));
        cached = s;
      }
      auto negbit = [&](std::int64_t pos) {
        return (q[pos] ^ (__builtin_popcountll(w & static_cast<std::uint64_t>(pos)) & 1)) != 0;
      };
      auto term = [&](std::int64_t pos) { return negbit(pos) ? -xs[pos] : xs[pos]; };
      float lanes[32];
      for (int l = 0; l < 32; ++l) {
        float acc = 0.f;
        if (d >= 128) {
          float tot = 0.f, neg = 0.f;
          for (std::int64_t i = 0; i < d / 128; ++i)
            for (int e = 0; e < 4; ++e) {
              const std::int64_t pos = 128 * i + 4 * l + e;
              tot += xs[pos];
              if (negbit(pos)) neg += xs[pos];
            }
          acc = std::fmaf(-2.f, neg, tot);
        } else {
          for (std::int64_t pos = l; pos < d; pos += 32) acc += term(pos);
        }
        lanes[l] = acc;
      }
      t = lane_tree_f(lanes);
    }
    float* col_sum = means.data() + (jj / p.J) * m;
    const float* col = gathered + jj * m;
    for (std::int64_t i = 0; i < m; ++i) col_sum[i] = std::fmaf(t, col[i], col_sum[i]);
  }
  for (auto& v : means) v /= static_cast<float>(p.J);
  const std::vector<float> mu = median_of_batch_means(means.data(), m, p.K);
  std::memcpy(mu_out, mu.data(), sizeof(float) * static_cast<std::size_t>(m));
  const std::int64_t want = candidate_count(p.s, p.widen, m);
  std::vector<std::int64_t> order(static_cast<std::size_t>(m));
  for (std::int64_t i = 0; i < m; ++i) order[i] = i;
  std::nth_element(order.begin(), order.begin() + want, order.end(), [&mu](std::int64_t u, std::int64_t v) {
    const float a = std::fabs(mu[u]), b = std::fabs(mu[v]);
    return a != b ? a > b : u < v;
  });
  std::sort(order.begin(), order.begin() + want);
  std::int64_t ns = 0;
  for (std::int64_t c = 0; c < want; ++c) {
    const std::int64_t i = order[c];
    cand_out[c] = i;
    const std::int64_t nv = (n + 3) / 4;
    double lanes[32];
    for (int l = 0; l < 32; ++l) {
      double chain[2] = {0.0, 0.0};
      for (std::int64_t qq = l, it = 0; qq < nv; qq += 32, ++it)
        for (int e = 0; e < 4; ++e) {
          const std::int64_t pos = 4 * qq + e;
          const double av = pos < n ? static_cast<double>(a[i * n + pos]) : 0.0;
          const double xv = static_cast<double>(xs[pos < d ? pos : 0]) * (pos < n ? 1.0 : 0.0);
          chain[it & 1] = std::fma(av, xv, chain[it & 1]);
        }
      lanes[l] = chain[0] + chain[1];
    }
    const double v = lane_tree_d(lanes);
    if (std::fabs(v) >= p.epsilon) {
      support_out[ns] = i;
      values_out[ns] = static_cast<float>(v);
      ++ns;
    }
  }
  *nsupport = ns;
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

// transform_gathered run in the B200 FAST-mode summation orders (float).
int orc_transform_gathered_fast_order(const float* a, std::int64_t m, std::int64_t n, const float* x, double eps,
                                      double delta, std::int64_t s, std::int64_t J, std::int64_t K, std::int64_t widen,
                                      const std::int64_t* indices, const float* gathered, float* mu_out,
                                      std::int64_t* cand_out, std::int64_t* support_out, float* values_out,
                                      std::int64_t* nsupport) {
  return guarded([&] {
    transform_gathered_fast_order(a, m, n, x, make_params(eps, delta, s, J, K, widen, 0), indices, gathered, mu_out,
                                  cand_out, support_out, values_out, nsupport);
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

// s_ell for each requested index (count x n, row j = s_{ell_j}), kerdock.hpp:156-167.
int orc_design_columns(int k, std::int64_t n, const std::int64_t* ells, std::int64_t count, double* out) {
  return guarded([&] {
    const DesignParams p = DesignParams::make(k);
    if (n < 1 || n > p.d) throw std::invalid_argument("design_columns: n out of [1,d]");
    const double sqrt_d = std::sqrt(static_cast<double>(p.d));
    std::vector<std::uint8_t> qbits;
    std::int64_t cached = -1;
    for (std::int64_t j = 0; j < count; ++j) {
      const DecodedIndex idx = decode_index(p, ells[j]);
      double* v = out + j * n;
      if (idx.identity) {
        std::fill(v, v + n, 0.0);
        if (static_cast<std::int64_t>(idx.wpos) < n) v[idx.wpos] = sqrt_d;
        continue;
      }
      if (static_cast<std::int64_t>(idx.s) != cached) {
        const auto m = kerdock_matrix(p, idx.s);
        qbits.assign(static_cast<std::size_t>(n), 0);
        for (std::int64_t q = 0; q < n; ++q)
          qbits[q] = static_cast<std::uint8_t>(
              quadratic_form(m.data(), p.k, coords_of_position(static_cast<std::uint64_t>(q), p.k)));
        cached = static_cast<std::int64_t>(idx.s);
      }
      for (std::int64_t q = 0; q < n; ++q)
        v[q] = (qbits[q] ^ (__builtin_popcountll(idx.wpos & static_cast<std::uint64_t>(q)) & 1)) ? -1.0 : 1.0;
    }
  });
}

// CPU baseline over a pool of P prepared vectors (gathered columns in host
// DRAM, P x N x m): `threads` threads process `total` vectors, vector t taking
// pool entry t % P; each runs draw_samples + transform_with_samples (the
// reference's transform(), stream.hpp:272-275) with its columns read from the
// gathered buffer. Returns wall seconds and the support sizes of the pool.
int orc_bench_gathered(const double* a, std::int64_t m, std::int64_t n, const double* X, std::int64_t P,
                       double eps, double delta, std::int64_t s, std::int64_t J, std::int64_t K, std::int64_t widen,
                       const std::uint64_t* seeds, const double* gathered, std::int64_t L, int threads,
                       std::int64_t total, std::int64_t* counts_out, double* seconds, int predrawn) {
  return guarded([&] {
    const std::int64_t N = J * K;
    // predrawn: the paper's timing convention (experiment.hpp:178-181) - draws done before the clock
    std::vector<std::vector<std::int64_t>> drawn;
    if (predrawn)
      for (std::int64_t v = 0; v < P; ++v) drawn.push_back(draw_samples(L, make_params(eps, delta, s, J, K, widen, seeds[v])));
    // the Kerdock set is built once, outside the clock, as the reference's Sketch constructor does
    // (sketch.hpp:130); transform() only derives the reversed rows per basis change (stream.hpp:222-226)
    const DesignParams design = DesignParams::make(even_log2_ceil(n));
    std::vector<std::vector<std::uint64_t>> kset(static_cast<std::size_t>(design.kerdock_bases()));
    for (std::int64_t s = 0; s < design.kerdock_bases(); ++s)
      kset[static_cast<std::size_t>(s)] = kerdock_matrix(design, static_cast<std::uint64_t>(s));
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    threads = std::max(1, threads);
    std::atomic<int> failed{0};
    for (int th = 0; th < threads; ++th) {
      pool.emplace_back([&, th] {
        try {
          for (std::int64_t t = th; t < total; t += threads) {
            const std::int64_t v = t % P;
            StreamParams p = make_params(eps, delta, s, J, K, widen, seeds[v]);
            const auto r = predrawn ? transform_gathered(a, m, n, X + v * n, p, drawn[v], gathered + v * N * m, &kset)
                                    : transform_gathered(a, m, n, X + v * n, p, draw_samples(L, p),
                                                         gathered + v * N * m, &kset);
            if (t < P) counts_out[v] = static_cast<std::int64_t>(r.support.size());
          }
        } catch (...) {
          failed = 1;
        }
      });
    }
    for (auto& t : pool) t.join();
    if (failed) throw std::runtime_error("bench_gathered: worker failed");
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// ---- FSTK save/load (sketch.hpp:213-302), fp64 reference format ----
// status: 7 IoError, 8 MagicMismatch, 9 VersionUnsupported, 10 TruncatedPayload, 11 MalformedHeader
static void put_le(std::FILE* f, std::uint64_t v, int bytes) {
  unsigned char b[8];
  for (int i = 0; i < bytes; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
  std::fwrite(b, 1, bytes, f);
}

int orc_save(void* hv, const char* path, int with_a) {
  auto* h = static_cast<OrcSketch*>(hv);
  if (h->dtype != 1) { g_err = "oracle save: fp64 sketches only"; return 1; }
  std::FILE* f = std::fopen(path, "wb");
  if (!f) { g_err = std::string("cannot open for writing: ") + path; return 7; }
  const auto& sk = h->d;
  std::fwrite("FSTK", 1, 4, f);
  put_le(f, 1, 4);
  put_le(f, sk.m, 8); put_le(f, sk.n, 8); put_le(f, sk.design.k, 8); put_le(f, sk.design.d, 8); put_le(f, sk.design.L, 8);
  const unsigned char flag = with_a ? 1 : 0;
  std::fwrite(&flag, 1, 1, f);
  std::fwrite(sk.columns.data(), 8, sk.columns.size(), f);
  if (with_a) std::fwrite(sk.a.data(), 8, sk.a.size(), f);
  const bool ok = std::fclose(f) == 0;
  if (!ok) { g_err = std::string("write failed: ") + path; return 7; }
  return 0;
}

int orc_load(const char* path, void** out) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) { g_err = std::string("cannot open for reading: ") + path; return 7; }
  std::fseek(f, 0, SEEK_END);
  const std::uint64_t fsize = static_cast<std::uint64_t>(std::ftell(f));
  std::fseek(f, 0, SEEK_SET);
  auto fail = [&](int code, const std::string& msg) { std::fclose(f); g_err = msg; return code; };
  if (fsize < 49) return fail(10, std::string("sketch file shorter than its header: ") + path);
  unsigned char hd[49];
  if (std::fread(hd, 1, 49, f) != 49) return fail(10, "short header");
  auto get = [&](int off, int bytes) { std::uint64_t v = 0; for (int i = 0; i < bytes; ++i) v |= std::uint64_t(hd[off + i]) << (8 * i); return v; };
  if (std::memcmp(hd, "FSTK", 4) != 0) return fail(8, std::string("not an FSTK sketch file: ") + path);
  const std::uint64_t version = get(4, 4);
  if (version != 1) return fail(9, "unsupported FSTK version " + std::to_string(version));
  const std::uint64_t m = get(8, 8), n = get(16, 8), k = get(24, 8), d = get(32, 8), L = get(40, 8);
  const int flag = hd[48];
  if (m == 0 || n == 0 || k < 2 || k > 16 || k % 2 != 0 || d != (std::uint64_t{1} << k) || L != d * (d / 2 + 1) || n > d ||
      (flag != 0 && flag != 1))
    return fail(11, std::string("inconsistent FSTK header fields: ") + path);
  const std::uint64_t expected = 49 + 8 * m * L + (flag ? 8 * m * n : 0);
  if (fsize < expected) return fail(10, std::string("FSTK payload truncated: ") + path);
  if (fsize > expected) return fail(11, "FSTK file larger than its header declares");
  auto* h = new OrcSketch();
  h->dtype = 1;
  h->d.design = DesignParams::make(static_cast<int>(k));
  h->d.m = static_cast<std::int64_t>(m);
  h->d.n = static_cast<std::int64_t>(n);
  h->d.columns.resize(m * L);
  bool ok = std::fread(h->d.columns.data(), 8, m * L, f) == m * L;
  if (flag) {
    h->d.a.resize(m * n);
    ok = ok && std::fread(h->d.a.data(), 8, m * n, f) == m * n;
  }
  std::fclose(f);
  if (!ok) {
    delete h;
    g_err = std::string("FSTK payload truncated: ") + path;
    return 10;
  }
  for (std::int64_t s = 0; s < h->d.design.kerdock_bases(); ++s) h->d.kerdock.push_back(kerdock_matrix(h->d.design, s));
  double rn = 0;
  for (std::uint64_t i = 0; i < (flag ? m : 0); ++i) {
    double acc = 0;
    for (std::uint64_t j = 0; j < n; ++j) acc += h->d.a[i * n + j] * h->d.a[i * n + j];
    rn = std::max(rn, std::sqrt(acc));
  }
  h->d.row_norm_max = rn;
  *out = h;
  return 0;
}

// generators.hpp:60-85 gen_mixture: returns x (n) and truth (m), both / |x|.
int orc_gen_mixture(const double* a, std::int64_t m, std::int64_t n, double p, std::uint64_t seed, double* x_out,
                    double* truth_out) {
  return guarded([&] {
    if (!(p > 0) || p > 1) throw std::invalid_argument("gen_mixture: need 0 < p <= 1");
    std::vector<double> truth(static_cast<std::size_t>(m));
    for (std::uint64_t attempt = 0;; ++attempt) {
      SeededRng rng(mix_seed(seed) ^ (attempt * 0x9e3779b97f4a7c15ull));
      bool any = false;
      for (std::int64_t i = 0; i < m; ++i) {
        if (rng.unit_double() <= p) {
          truth[i] = rng.gaussian();
          any = true;
        } else {
          truth[i] = 0.0;
        }
      }
      if (any) break;
    }
    double nrm = 0;
    for (std::int64_t j = 0; j < n; ++j) {
      double acc = 0;
      for (std::int64_t i = 0; i < m; ++i) acc += a[i * n + j] * truth[i];
      x_out[j] = acc;
      nrm += acc * acc;
    }
    nrm = std::sqrt(nrm);
    for (std::int64_t j = 0; j < n; ++j) x_out[j] /= nrm;
    for (std::int64_t i = 0; i < m; ++i) truth_out[i] = truth[i] / nrm;
  });
}

// ---- generators ----
int orc_gen_orthogonal(std::int64_t n, std::uint64_t seed, double* out) {
  return guarded([&] {
    const auto v = gen_orthogonal(n, seed);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}
int orc_gen_exact_sparse(const double* a, std::int64_t m, std::int64_t n, std::int64_t s, std::uint64_t seed,
                         double* x_out, double* truth_out) {
  return guarded([&] {
    const auto t = gen_exact_sparse(a, m, n, s, seed, x_out);
    std::memcpy(truth_out, t.data(), sizeof(double) * t.size());
  });
}

// ---- design verifiers (kerdock.hpp:198-317, cli.hpp:45-60) ----
int orc_materialize_design(int k, double* out) {
  return guarded([&] {
    const auto u = materialize_design(DesignParams::make(k));
    std::memcpy(out, u.data(), sizeof(double) * u.size());
  });
}
int orc_verify_mub(int k, int cap, double* out4, int* exhaustive) {
  return guarded([&] {
    const MubReport r = verify_mub(DesignParams::make(k), cap);
    out4[0] = r.max_within_gram_dev;
    out4[1] = r.min_cross_sq;
    out4[2] = r.max_cross_sq;
    out4[3] = r.max_cross_dev;
    *exhaustive = r.exhaustive ? 1 : 0;
  });
}
int orc_verify_design_moments(int k, int cap, double* out2, int* exact) {
  return guarded([&] {
    const MomentReport r = verify_design_moments(DesignParams::make(k), cap);
    out2[0] = r.m1;
    out2[1] = r.m2;
    *exact = r.exact ? 1 : 0;
  });
}
int orc_design_moments_of(const double* u, std::int64_t d, std::int64_t L, double* out2) {
  return guarded([&] {
    const MomentReport r = design_moments_of(u, d, L);
    out2[0] = r.m1;
    out2[1] = r.m2;
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
