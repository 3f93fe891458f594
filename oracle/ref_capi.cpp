// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI over the REFERENCE's own hot-path code: proj/include/fst/{sketch,stream,
// kerdock,fwht,gf2,rng,io}.hpp compiled unmodified from /root/reference (nothing
// is copied into this repo) against the minimal Eigen-API shim in
// oracle/eigen_shim (Eigen is not installed here). Built by `make -C oracle ref`
// into oracle/_ref/libfst_ref.so. Used by
//   - tests/test_ref_pin.py: pins the oracle restatement (oracle/fst_oracle.cpp)
//     against the reference itself — sketch columns, draws, mu, candidates,
//     support, values;
//   - bench.py --impl reference / cpu_baseline: times the reference's own
//     transform_with_samples() on the host cores (cpu_baseline.kind "reference").
// Status codes follow oracle_capi.cpp: 1 invalid_argument, 2 out_of_range,
// 3 overflow_error, 4 runtime_error / other.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fst/sketch.hpp"
#include "fst/stream.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
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
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

fst::StreamParams params(double eps, double delta, std::int64_t s, std::int64_t J, std::int64_t K,
                         std::int64_t widen, std::uint64_t seed) {
  fst::StreamParams p;
  p.epsilon = eps;
  p.delta = delta;
  p.s = s;
  p.J = J;
  p.K = K;
  p.widen = widen;
  p.seed = seed;
  return p;
}

fst::RowMatrix row_matrix(const double* a, std::int64_t m, std::int64_t n) {
  fst::RowMatrix out(m, n);
  std::memcpy(out.data(), a, sizeof(double) * static_cast<std::size_t>(m * n));
  return out;
}

}  // namespace

extern "C" {

const char* fstref_last_error() { return g_err.c_str(); }

/// fst::preprocess (sketch.hpp:149-211) on a row-major m x n fp64 matrix, FST_THREADS = threads.
int fstref_preprocess(const double* a, std::int64_t m, std::int64_t n, int threads, void** out) {
  return guarded([&] {
    if (threads >= 1) setenv("FST_THREADS", std::to_string(threads).c_str(), 1);
    const fst::RowMatrix am = row_matrix(a, m, n);
    *out = new fst::Sketch(fst::preprocess(am));
  });
}

/// A reference Sketch whose column set is not materialised (the public constructor,
/// sketch.hpp:72-81, with an empty column vector): valid for transform_with_samples on
/// gathered columns (stream.hpp:231-232 never reads the sketch's columns then).
int fstref_sketch_without_columns(const double* a, std::int64_t m, std::int64_t n, void** out) {
  return guarded([&] {
    const fst::DesignParams design = fst::DesignParams::make(fst::even_log2_ceil(n));
    *out = new fst::Sketch(design, m, n, row_matrix(a, m, n), std::vector<double>{});
  });
}

void fstref_sketch_free(void* h) { delete static_cast<fst::Sketch*>(h); }

int fstref_sketch_info(void* h, std::int64_t* m, std::int64_t* n, std::int64_t* L, double* row_norm_max) {
  return guarded([&] {
    const auto* sk = static_cast<const fst::Sketch*>(h);
    *m = sk->m();
    *n = sk->n();
    *L = sk->L();
    *row_norm_max = sk->row_norm_max();
  });
}

/// Copies the column-major m x L column set (Sketch::column_data).
int fstref_sketch_columns(void* h, double* out) {
  return guarded([&] {
    const auto* sk = static_cast<const fst::Sketch*>(h);
    if (!sk->column_data()) throw std::invalid_argument("sketch has no materialised columns");
    std::memcpy(out, sk->column_data(), sizeof(double) * static_cast<std::size_t>(sk->m() * sk->L()));
  });
}

/// fst::draw_samples (stream.hpp:173-182).
int fstref_draw_samples(void* h, double eps, double delta, std::int64_t s, std::int64_t J, std::int64_t K,
                        std::int64_t widen, std::uint64_t seed, std::int64_t* out) {
  return guarded([&] {
    const auto d = fst::draw_samples(*static_cast<const fst::Sketch*>(h), params(eps, delta, s, J, K, widen, seed));
    std::memcpy(out, d.indices.data(), sizeof(std::int64_t) * d.indices.size());
  });
}

/// fst::transform (stream.hpp:272-275); gathered (N x m, row j = column of draw j) selects the
/// draw_and_gather form (stream.hpp:184-191) for sketches without materialised columns.
int fstref_transform(void* h, const double* x, std::int64_t nx, double eps, double delta, std::int64_t s, std::int64_t J,
                     std::int64_t K, std::int64_t widen, std::uint64_t seed, const double* gathered,
                     double* mu_out, std::int64_t* cand_out, std::int64_t* support_out, double* values_out,
                     std::int64_t* nsupport) {
  return guarded([&] {
    const auto& sk = *static_cast<const fst::Sketch*>(h);
    const fst::StreamParams p = params(eps, delta, s, J, K, widen, seed);
    const Eigen::Map<const Eigen::VectorXd> xv(x, nx);  // length checked by the reference (stream.hpp:201)
    fst::TransformResult r;
    if (gathered) {
      fst::DrawnSamples d = fst::draw_samples(sk, p);
      d.gathered = Eigen::Map<const Eigen::MatrixXd>(gathered, sk.m(), p.J * p.K);
      d.use_gathered = true;
      r = fst::transform_with_samples(sk, xv, p, d);
    } else {
      r = fst::transform(sk, xv, p);
    }
    if (mu_out) std::memcpy(mu_out, r.estimate.mu.data(), sizeof(double) * static_cast<std::size_t>(sk.m()));
    if (cand_out) std::memcpy(cand_out, r.candidate_set.data(), sizeof(std::int64_t) * r.candidate_set.size());
    if (support_out) std::memcpy(support_out, r.support.data(), sizeof(std::int64_t) * r.support.size());
    if (values_out) std::memcpy(values_out, r.values.data(), sizeof(double) * r.values.size());
    *nsupport = static_cast<std::int64_t>(r.support.size());
  });
}

int fstref_choose_params(double row_norm_max, double gamma, double eta, std::int64_t m, std::int64_t* J,
                         std::int64_t* K) {
  return guarded([&] {
    const auto jk = fst::choose_params(row_norm_max, gamma, eta, m);
    *J = jk.first;
    *K = jk.second;
  });
}

/// Times the reference's transform over `total` vectors cycling a pool of P vectors on `threads`
/// host threads. Per vector: the reference's draw_samples (timed, as transform() draws) and
/// transform_with_samples on that vector's DrawnSamples, built before the clock with its
/// sampled columns gathered (gathered: P x N x m; the fp64 sketch at n = 4096 is 275 GB, more
/// than host RAM, so the sketch object carries no column set). Returns pool support counts.
int fstref_bench_gathered(const double* a, std::int64_t m, std::int64_t n, const double* X, std::int64_t P,
                          double eps, double delta, std::int64_t s, std::int64_t J, std::int64_t K,
                          std::int64_t widen, const std::uint64_t* seeds, const double* gathered, int threads,
                          std::int64_t total, std::int64_t* counts_out, double* seconds) {
  return guarded([&] {
    const fst::DesignParams design = fst::DesignParams::make(fst::even_log2_ceil(n));
    const fst::Sketch sk(design, m, n, row_matrix(a, m, n), std::vector<double>{});  // Kerdock set built here
    const std::int64_t N = J * K;
    std::vector<fst::DrawnSamples> pre(static_cast<std::size_t>(P));
    for (std::int64_t v = 0; v < P; ++v) {
      const fst::StreamParams p = params(eps, delta, s, J, K, widen, seeds[v]);
      pre[v] = fst::draw_samples(sk, p);
      pre[v].gathered = Eigen::Map<const Eigen::MatrixXd>(gathered + v * N * m, m, N);
      pre[v].use_gathered = true;
    }
    threads = std::max(1, threads);
    std::atomic<int> failed{0};
    std::string first_error;
    std::atomic<bool> mismatch{false};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int th = 0; th < threads; ++th) {
      pool.emplace_back([&, th] {
        try {
          for (std::int64_t t = th; t < total; t += threads) {
            const std::int64_t v = t % P;
            const fst::StreamParams p = params(eps, delta, s, J, K, widen, seeds[v]);
            const fst::DrawnSamples drawn = fst::draw_samples(sk, p);  // timed: transform() draws per vector
            if (drawn.indices != pre[v].indices) mismatch = true;
            const Eigen::Map<const Eigen::VectorXd> xv(X + v * n, n);
            const fst::TransformResult r = fst::transform_with_samples(sk, xv, p, pre[v]);
            if (t < P) counts_out[v] = static_cast<std::int64_t>(r.support.size());
          }
        } catch (const std::exception& e) {
          if (failed.exchange(1) == 0) first_error = e.what();
        }
      });
    }
    for (auto& t : pool) t.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (failed) throw std::runtime_error("bench_gathered worker: " + first_error);
    if (mismatch) throw std::runtime_error("bench_gathered: draws differ from the prepared samples");
  });
}

}  // extern "C"
