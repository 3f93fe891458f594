// Host-side synthetic input generators (product code; BASELINE.json configs).
// They follow the reference's SeededRng conventions (rng.hpp: std::mt19937_64,
// multiply-shift bounded draws, Box-Muller normals, top-bit coin) and its
// gen_exact_sparse draw order (generators.hpp:44-53: partial Fisher-Yates,
// then the value). The dense noise term and the N(0,1)-valued targets are the
// configs' new generators (SURVEY.md §0 flag 6). Multithreaded over vectors.
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

#include "../../include/fst_b200.h"

namespace {

class Rng {
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  uint64_t index(uint64_t bound) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(eng_()) * bound) >> 64);
  }
  double unit_double() { return (static_cast<double>(eng_() >> 11) + 1.0) * 0x1.0p-53; }
  double gaussian() {
    if (have_) {
      have_ = false;
      return spare_;
    }
    const double u1 = unit_double(), u2 = unit_double();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * 3.141592653589793238462643383279502884 * u2;
    spare_ = r * std::sin(th);
    have_ = true;
    return r * std::cos(th);
  }
  bool coin() { return (eng_() >> 63) != 0; }

 private:
  std::mt19937_64 eng_;
  double spare_ = 0;
  bool have_ = false;
};

template <typename Fn>
void parallel_for(int64_t count, Fn&& fn) {
  const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
  const int64_t threads = std::min<int64_t>(hw, std::max<int64_t>(1, count / 64));
  if (threads <= 1) {
    fn(int64_t{0}, count);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t per = (count + threads - 1) / threads;
  for (int64_t t = 0; t < threads; ++t) {
    const int64_t f = t * per, l = std::min(count, f + per);
    if (f < l) pool.emplace_back([&fn, f, l] { fn(f, l); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// SeededRng(seed).gaussian() x count (the fill order of gen_orthogonal,
// generators.hpp:22-25).
// The engine stream is inherently sequential, the Box-Muller transform is not:
// normals 2p and 2p+1 are r cos(th) and r sin(th) of draws 2p and 2p+1, so the
// raw 64-bit draws are generated in chunks on this thread and the transform runs
// on all cores (bit-identical to the sequential Rng::gaussian loop; n = 16384
// fills 268M normals).
int fstg_gen_gaussian(uint64_t seed, int64_t count, double* out) {
  if (count < 0 || (count > 0 && out == nullptr)) return FSTG_ERR_INVALID_ARGUMENT;
  std::mt19937_64 eng(seed);
  constexpr int64_t kPairs = int64_t(1) << 22;  // pairs per chunk (64 MiB of raw draws)
  const int64_t pairs = (count + 1) / 2;
  std::vector<uint64_t> raw(static_cast<size_t>(2 * std::min(pairs, kPairs)));
  for (int64_t p0 = 0; p0 < pairs; p0 += kPairs) {
    const int64_t np = std::min(kPairs, pairs - p0);
    for (int64_t i = 0; i < 2 * np; ++i) raw[static_cast<size_t>(i)] = eng();
    parallel_for(np, [&](int64_t first, int64_t last) {
      for (int64_t q = first; q < last; ++q) {
        const double u1 = (static_cast<double>(raw[2 * q] >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = (static_cast<double>(raw[2 * q + 1] >> 11) + 1.0) * 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * 3.141592653589793238462643383279502884 * u2;
        const int64_t i = 2 * (p0 + q);
        out[i] = r * std::cos(th);
        if (i + 1 < count) out[i + 1] = r * std::sin(th);
      }
    });
  }
  return FSTG_OK;
}

// B sparse(+noise) target vectors y (B x m, row-major). Vector v uses
// SeededRng(seeds[v]): s distinct rows by partial Fisher-Yates with
// index(m - i); value +-1/sqrt(s) by coin (value_kind 0) or N(0,1)
// (value_kind 1); then, if noise_sigma > 0, noise_sigma * N(0,1) added to all
// m entries in row order.
int fstg_gen_sparse_targets(const uint64_t* seeds, int64_t B, int64_t m, int64_t s, int value_kind,
                            double noise_sigma, double* Y) {
  if (B < 0 || m < 1 || s < 1 || s > m || (B > 0 && (seeds == nullptr || Y == nullptr)) || value_kind < 0 ||
      value_kind > 1)
    return FSTG_ERR_INVALID_ARGUMENT;
  const double mag = 1.0 / std::sqrt(static_cast<double>(s));
  parallel_for(B, [&](int64_t first, int64_t last) {
    std::vector<int64_t> perm(static_cast<size_t>(m));
    for (int64_t v = first; v < last; ++v) {
      Rng r(seeds[v]);
      double* y = Y + v * m;
      std::fill(y, y + m, 0.0);
      std::iota(perm.begin(), perm.end(), int64_t{0});
      for (int64_t i = 0; i < s; ++i) {
        const int64_t j = i + static_cast<int64_t>(r.index(static_cast<uint64_t>(m - i)));
        std::swap(perm[i], perm[j]);
        y[perm[i]] = value_kind == 0 ? (r.coin() ? mag : -mag) : r.gaussian();
      }
      if (noise_sigma > 0)
        for (int64_t i = 0; i < m; ++i) y[i] += noise_sigma * r.gaussian();
    }
  });
  return FSTG_OK;
}

// gen_mixture's target draw (generators.hpp:60-78): entries are N(0,1) with
// probability p (unit_double() <= p, then gaussian()), else 0; an all-zero draw
// retries on SeededRng(mix_seed(seed) ^ attempt * 0x9e3779b97f4a7c15). The
// caller forms x = A^T y and rescales both by |x| (generators.hpp:80-83).
int fstg_gen_mixture_targets(const uint64_t* seeds, int64_t B, int64_t m, double p, double* Y) {
  if (B < 0 || m < 1 || !(p > 0) || p > 1 || (B > 0 && (seeds == nullptr || Y == nullptr)))
    return FSTG_ERR_INVALID_ARGUMENT;
  auto mix = [](uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  };
  parallel_for(B, [&](int64_t first, int64_t last) {
    for (int64_t v = first; v < last; ++v) {
      double* y = Y + v * m;
      for (uint64_t attempt = 0;; ++attempt) {
        Rng r(mix(seeds[v]) ^ (attempt * 0x9e3779b97f4a7c15ull));
        bool any = false;
        for (int64_t i = 0; i < m; ++i) {
          if (r.unit_double() <= p) {
            y[i] = r.gaussian();
            any = true;
          } else {
            y[i] = 0.0;
          }
        }
        if (any) break;
      }
    }
  });
  return FSTG_OK;
}

}  // extern "C"
