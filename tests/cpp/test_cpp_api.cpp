// C++ API test: the reference's stream/sketch tests (proj/tests/test_stream.cpp,
// test_sketch.cpp) re-expressed against fst_b200.hpp, i.e. through the C-ABI
// library on the GPU. Built and run by tests/test_cpp_api.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

#include "fst_b200.hpp"

using namespace fst_b200;

static int failures = 0;
#define CHECK(...)                                                 \
  do {                                                             \
    if (!(__VA_ARGS__)) {                                                  \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
      ++failures;                                                  \
    }                                                              \
  } while (0)

template <typename E, typename F>
static void check_throws(F&& f, const char* what) {
  try {
    f();
  } catch (const E&) {
    return;
  } catch (...) {
  }
  std::printf("expected exception not thrown: %s\n", what);
  ++failures;
}

// Haar-like orthogonal matrix by modified Gram-Schmidt of a seeded Gaussian (row-major).
static std::vector<double> random_orthogonal(int n, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> g;
  std::vector<double> q(static_cast<std::size_t>(n) * n);
  for (auto& v : q) v = g(rng);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < i; ++j) {
      double d = 0;
      for (int c = 0; c < n; ++c) d += q[i * n + c] * q[j * n + c];
      for (int c = 0; c < n; ++c) q[i * n + c] -= d * q[j * n + c];
    }
    double nr = 0;
    for (int c = 0; c < n; ++c) nr += q[i * n + c] * q[i * n + c];
    nr = std::sqrt(nr);
    for (int c = 0; c < n; ++c) q[i * n + c] /= nr;
  }
  return q;
}

static std::vector<double> random_unit(int n, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> g;
  std::vector<double> x(n);
  double nr = 0;
  for (auto& v : x) {
    v = g(rng);
    nr += v * v;
  }
  for (auto& v : x) v /= std::sqrt(nr);
  return x;
}

static std::vector<double> matvec(const std::vector<double>& a, const std::vector<double>& x, int m, int n) {
  std::vector<double> y(m, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) y[i] += a[i * n + j] * x[j];
  return y;
}

int main() {
  // test_sketch.cpp:47-60: preprocess of the identity reproduces +-1 Kerdock columns
  {
    std::vector<double> eye(16 * 16, 0.0);
    for (int i = 0; i < 16; ++i) eye[i * 16 + i] = 1.0;
    Sketch sk = preprocess(eye.data(), 16, 16);
    CHECK(sk.k() == 4 && sk.L() == 144);
    CHECK(std::abs(sk.row_norm_max() - 1.0) < 1e-12);
    for (std::int64_t ell = 0; ell < 8 * 16; ++ell)
      for (double v : sk.column(ell)) CHECK(std::abs(v) == 1.0);
    check_throws<std::out_of_range>([&] { sk.column(sk.L()); }, "column(L)");
  }
  // test_stream.cpp:40-53 choose_params fixed values
  {
    CHECK(choose_params(1.0, 1.0, 1.0, 1) == std::make_pair<std::int64_t, std::int64_t>(30, 1));
    CHECK(choose_params(1.0, 0.5, 0.01, 4096) == std::make_pair<std::int64_t, std::int64_t>(119, 26));
    check_throws<std::invalid_argument>([] { choose_params(1.0, 0.0, 0.5, 16); }, "gamma = 0");
  }
  // test_stream.cpp:162-189 widen*s >= m gives exact hard thresholding
  {
    const auto a = random_orthogonal(16, 1);
    Sketch sk = preprocess(a.data(), 16, 16);
    const auto x = random_unit(16, 2);
    StreamParams p;
    p.epsilon = 0.2;
    p.s = 2;
    p.widen = 8;
    p.J = 3;
    p.K = 2;
    p.seed = 42;
    const TransformResult r = transform(sk, x, p);
    const auto ax = matvec(a, x, 16, 16);
    CHECK(r.candidate_set.size() == 16);
    std::size_t found = 0;
    for (int i = 0; i < 16; ++i)
      if (std::abs(ax[i]) >= 0.2) {
        CHECK(found < r.support.size() && r.support[found] == i);
        if (found < r.values.size()) CHECK(std::abs(r.values[found] - ax[i]) <= 1e-12);
        ++found;
      }
    CHECK(found == r.support.size());
  }
  // test_stream.cpp:191-202 x = 0
  {
    Sketch sk = preprocess(random_orthogonal(16, 3).data(), 16, 16);
    StreamParams p;
    p.epsilon = 0.1;
    p.s = 2;
    p.J = 5;
    p.K = 2;
    const TransformResult r = transform(sk, std::vector<double>(16, 0.0), p);
    CHECK(r.support.empty() && r.values.empty());
    for (double v : r.mu) CHECK(v == 0.0);
  }
  // test_stream.cpp:204-225 one spike, 100 seeds
  {
    const auto a = random_orthogonal(16, 4);
    Sketch sk = preprocess(a.data(), 16, 16);
    std::vector<double> x(a.begin(), a.begin() + 16);
    StreamParams p;
    p.epsilon = 0.5;
    p.s = 1;
    p.J = 500;
    p.K = 3;
    int ok = 0;
    for (std::uint64_t seed = 0; seed < 100; ++seed) {
      p.seed = seed;
      const TransformResult r = transform(sk, x, p);
      ok += (r.support.size() == 1 && r.support[0] == 0 && std::abs(r.values[0] - 1.0) <= 1e-10);
    }
    CHECK(ok == 100);
  }
  // test_stream.cpp:290-315 determinism and gather-independence
  {
    const auto a = random_orthogonal(32, 10);
    Sketch sk = preprocess(a.data(), 32, 32);
    const auto x = random_unit(32, 11);
    StreamParams p;
    p.epsilon = 0.05;
    p.s = 3;
    p.J = 25;
    p.K = 4;
    p.seed = 1234;
    const auto r1 = transform(sk, x, p), r2 = transform(sk, x, p);
    const auto r3 = transform_with_samples(sk, x, p, draw_samples(sk, p));
    CHECK(r1.support == r2.support && r1.values == r2.values && r1.mu == r2.mu);
    CHECK(r1.support == r3.support && r1.values == r3.values && r1.mu == r3.mu);
  }
  // test_stream.cpp:382-401 validation errors
  {
    Sketch sk = preprocess(random_orthogonal(16, 14).data(), 16, 16);
    StreamParams p;
    p.epsilon = 0.1;
    p.s = 1;
    p.J = 2;
    p.K = 2;
    check_throws<std::invalid_argument>([&] { transform(sk, std::vector<double>(15, 0.0), p); }, "length");
    StreamParams bad = p;
    bad.epsilon = 0.0;
    check_throws<std::invalid_argument>([&] { transform(sk, std::vector<double>(16, 0.0), bad); }, "eps");
    bad = p;
    bad.J = INT64_MAX / 2;
    bad.K = 3;
    check_throws<std::overflow_error>([&] { transform(sk, std::vector<double>(16, 0.0), bad); }, "J*K");
  }
  // test_sketch.cpp:128-133 rejects empty / non-finite input
  {
    std::vector<double> bad = {1.0, NAN, 1.0, 1.0};
    check_throws<std::invalid_argument>([&] { preprocess(bad.data(), 2, 2); }, "nan");
    check_throws<std::invalid_argument>([&] { preprocess(bad.data(), 0, 2); }, "empty");
  }
  // kerdock.hpp:198-317 verifiers (test_kerdock.cpp:200-216, 231-247)
  {
    const MubReport mub = verify_mub(4);
    if (!mub.exhaustive || mub.max_within_gram_dev != 0.0 || mub.min_cross_sq != 1.0 / 16 || mub.max_cross_dev != 0.0) {
      std::printf("FAIL verify_mub(4)\n");
      ++failures;
    }
    const MomentReport mom = verify_design_moments(4);
    if (std::abs(mom.m1 - 1.0 / 16) > 1e-12 || std::abs(mom.m2 - 1.0 / 96) > 1e-12 ||
        design_moment_target(16, 2) != mom.m2) {
      std::printf("FAIL verify_design_moments(4)\n");
      ++failures;
    }
    check_throws<std::invalid_argument>([&] { verify_mub(6, 4); }, "cap");
  }
  // FSTK save/load round trip, embedded matrix, sampled columns, helpers
  {
    const std::vector<double> a = random_orthogonal(16, 21);
    Sketch sk = preprocess(a.data(), 16, 16);
    const std::string path = "/tmp/fst_b200_cpp_test.fstk";
    save(sk, path);
    Sketch back = load(path);
    const std::vector<std::int64_t> idx = {0, 5, 100, sk.L() - 1};
    const std::vector<double> c1 = sk.sample_columns(idx), c2 = back.sample_columns(idx);
    if (c1 != c2 || back.embedded_matrix() != a || c1.size() != idx.size() * 16) {
      std::printf("FAIL save/load/sample_columns\n");
      ++failures;
    }
    for (std::size_t j = 0; j < idx.size(); ++j) {
      const std::vector<double> col = sk.column(idx[j]);
      for (int i = 0; i < 16; ++i)
        if (col[i] != c1[j * 16 + i]) {
          std::printf("FAIL sample_columns vs column\n");
          ++failures;
          j = idx.size();
          break;
        }
    }
    check_throws<MagicMismatchError>([&] {
      std::FILE* f = std::fopen(path.c_str(), "r+b");
      std::fputc('X', f);
      std::fclose(f);
      load(path);
    }, "magic");
    std::vector<double> x(16, 0.0);
    x[3] = 1.0;
    const std::vector<double> s5 = projected_design_column(4, 16, 5);
    if (inner_product_with_design(x, 4, 5) != s5[3]) {
      std::printf("FAIL inner_product_with_design\n");
      ++failures;
    }
    const std::vector<double> h = hard_threshold({0.5, -0.05, 0.1}, 0.1);
    if (h[0] != 0.5 || h[1] != 0.0 || h[2] != 0.1) {
      std::printf("FAIL hard_threshold\n");
      ++failures;
    }
    const std::vector<double> mom = median_of_means({1, 2, 3, 4, 5, 6, 7, 8}, 2, 2, 2);  // m=2: means (2,3),(6,7)
    if (mom[0] != 4.0 || mom[1] != 5.0) {
      std::printf("FAIL median_of_means %g %g\n", mom[0], mom[1]);
      ++failures;
    }
  }
  std::printf("cpp api: %s (%d failures)\n", failures ? "FAIL" : "ok", failures);
  return failures ? 1 : 0;
}
