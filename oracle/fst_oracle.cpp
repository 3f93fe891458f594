// ORACLE — TEST INFRASTRUCTURE ONLY (see fst_oracle.hpp header).
// Restates /root/reference/proj/include/fst/*.hpp without Eigen. Every
// function cites the reference lines it follows.
#include "fst_oracle.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <thread>

namespace fst_oracle {

// ------------------------------------------------------------------ gf2 ----

std::uint64_t modulus_for_degree(int q) {  // gf2.hpp:205-218
  switch (q) {
    case 1: return 0b11ull;
    case 3: return 0b1011ull;
    case 5: return 0b100101ull;
    case 7: return 0b10000011ull;
    case 9: return 0b1000010001ull;
    case 11: return 0b100000000101ull;
    case 13: return 0b10000000011011ull;
    case 15: return 0b1000000000000011ull;
    default: throw std::invalid_argument("modulus_for_degree: no shipped modulus for this degree");
  }
}

static int poly_degree(std::uint64_t p) { return p == 0 ? -1 : 63 - std::countl_zero(p); }

static std::uint64_t poly_mod(std::uint64_t a, std::uint64_t g) {  // gf2.hpp:181-185
  const int dg = poly_degree(g);
  for (int da = poly_degree(a); da >= dg; da = poly_degree(a)) a ^= g << (da - dg);
  return a;
}

bool verify_irreducible(std::uint64_t poly, int degree) {  // gf2.hpp:192-200
  if (degree < 1) throw std::invalid_argument("verify_irreducible: degree must be >= 1");
  if (poly_degree(poly) != degree)
    throw std::invalid_argument("verify_irreducible: leading coefficient not at stated degree");
  for (std::uint64_t g = 2; poly_degree(g) <= degree / 2; ++g)
    if (poly_mod(poly, g) == 0) return false;
  return true;
}

std::uint64_t field_mul(int q, std::uint64_t modulus, std::uint64_t a, std::uint64_t b) {
  // gf2.hpp:251-261: accumulate a*x^i for set bits of b, reducing a on overflow.
  const std::uint64_t top = std::uint64_t{1} << q;
  std::uint64_t acc = 0, aa = a;
  for (std::uint64_t bb = b; bb != 0; bb >>= 1) {
    if (bb & 1u) acc ^= aa;
    aa <<= 1;
    if (aa & top) aa ^= modulus;
  }
  return acc;
}

int field_trace(int q, std::uint64_t modulus, std::uint64_t a) {  // gf2.hpp:264-274
  std::uint64_t acc = a, pw = a;
  for (int i = 1; i < q; ++i) {
    pw = field_mul(q, modulus, pw, pw);
    acc ^= pw;
  }
  if (acc > 1) throw std::logic_error("field_trace: trace left the prime subfield");
  return static_cast<int>(acc);
}

int gf2_rank(const std::uint64_t* in, int dim) {  // gf2.hpp:148-172
  std::vector<std::uint64_t> rows(in, in + dim);
  int rank = 0;
  for (int col = 0; col < dim; ++col) {
    const std::uint64_t bit = std::uint64_t{1} << col;
    int pivot = -1;
    for (int r = rank; r < dim; ++r)
      if (rows[r] & bit) { pivot = r; break; }
    if (pivot < 0) continue;
    std::swap(rows[rank], rows[pivot]);
    for (int r = 0; r < dim; ++r)
      if (r != rank && (rows[r] & bit)) rows[r] ^= rows[rank];
    ++rank;
  }
  return rank;
}

std::uint64_t coords_of_position(std::uint64_t p, int k) {  // gf2.hpp:65-69
  std::uint64_t w = 0;
  for (int c = 0; c < k; ++c)
    if ((p >> (k - 1 - c)) & 1u) w |= std::uint64_t{1} << c;
  return w;
}

std::uint64_t position_of_coords(std::uint64_t w, int k) {  // gf2.hpp:72-78
  std::uint64_t p = 0;
  for (int c = 0; c < k; ++c)
    if ((w >> c) & 1u) p |= std::uint64_t{1} << (k - 1 - c);
  return p;
}

// -------------------------------------------------------------- kerdock ----

DesignParams DesignParams::make(int k) {  // kerdock.hpp:26-31
  if (k < 2 || k % 2 != 0) throw std::invalid_argument("DesignParams: k must be a positive even integer");
  if (k > 16) throw std::invalid_argument("DesignParams: k > 16 is not supported");
  DesignParams p;
  p.k = k;
  p.d = std::int64_t{1} << k;
  p.L = p.d * (p.d / 2 + 1);
  p.modulus = modulus_for_degree(k - 1);
  if (!verify_irreducible(p.modulus, k - 1)) throw std::invalid_argument("FieldCtx: modulus is reducible");
  return p;
}

int quadratic_form(const std::uint64_t* rows, int dim, std::uint64_t xw) {  // kerdock.hpp:38-49
  int acc = 0;
  for (std::uint64_t rest = xw; rest != 0; rest &= rest - 1) {
    const int i = std::countr_zero(rest);
    if (i + 1 >= 64) break;
    if (i >= dim) break;
    const std::uint64_t above = ~std::uint64_t{0} << (i + 1);
    acc ^= std::popcount(rows[i] & xw & above) & 1;
  }
  return acc;
}

std::vector<std::uint64_t> kerdock_matrix(const DesignParams& p, std::uint64_t s) {
  // kerdock.hpp:55-84: (M_s)_{r,c} = tr(a^r f_c) for r < q, row q = t_c, where
  // (f_c, t_c) = L_s(basis_c), basis a^0..a^(q-1) then (0,1).
  const int q = p.k - 1;
  const int k = p.k;
  const std::uint64_t mod = p.modulus;
  if (s >= (std::uint64_t{1} << q)) throw std::invalid_argument("kerdock_matrix: field index out of range");
  const std::uint64_t s2 = field_mul(q, mod, s, s);
  std::vector<std::uint64_t> f(k), t(k);
  for (int c = 0; c < q; ++c) {
    const std::uint64_t ac = std::uint64_t{1} << c;
    t[c] = static_cast<std::uint64_t>(field_trace(q, mod, field_mul(q, mod, s, ac)));
    f[c] = field_mul(q, mod, s2, ac) ^ (t[c] ? s : 0);
  }
  f[q] = s;
  t[q] = 0;
  std::vector<std::uint64_t> m(k, 0);
  for (int c = 0; c < k; ++c) {
    for (int r = 0; r < q; ++r) {
      const std::uint64_t ar = std::uint64_t{1} << r;
      if (field_trace(q, mod, field_mul(q, mod, ar, f[c])) != 0) m[r] |= std::uint64_t{1} << c;
    }
    if (t[c]) m[q] |= std::uint64_t{1} << c;
  }
  return m;
}

DecodedIndex decode_index(const DesignParams& p, std::int64_t ell) {  // kerdock.hpp:121-129
  if (ell < 0 || ell >= p.L) throw std::out_of_range("DesignIndex: linear index out of range");
  const std::int64_t kb = p.kerdock_bases() * p.d;
  if (ell < kb)
    return {false, static_cast<std::uint64_t>(ell / p.d), static_cast<std::uint64_t>(ell % p.d)};
  return {true, 0, static_cast<std::uint64_t>(ell - kb)};
}

std::vector<double> projected_design_column(const DesignParams& p, std::int64_t n, std::int64_t ell) {
  // kerdock.hpp:134-167: entry j of u_{M,w} is 2^(-k/2) (-1)^(Q_M(coords(j)) + w.j);
  // s_ell = sqrt(d) * head(n); identity -> sqrt(d) e_w (0 past n).
  if (n < 1 || n > p.d) throw std::invalid_argument("projected_design_column: n out of [1,d]");
  const DecodedIndex idx = decode_index(p, ell);
  const double sqrt_d = std::sqrt(static_cast<double>(p.d));
  std::vector<double> v(static_cast<std::size_t>(n), 0.0);
  if (idx.identity) {
    if (static_cast<std::int64_t>(idx.wpos) < n) v[idx.wpos] = sqrt_d;
    return v;
  }
  const auto m = kerdock_matrix(p, idx.s);
  const double scale = 1.0 / std::sqrt(static_cast<double>(p.d));
  for (std::int64_t j = 0; j < n; ++j) {
    const int sign = quadratic_form(m.data(), p.k, coords_of_position(static_cast<std::uint64_t>(j), p.k)) ^
                     (std::popcount(idx.wpos & static_cast<std::uint64_t>(j)) & 1);
    v[j] = sqrt_d * (sign ? -scale : scale);
  }
  return v;
}

// ----------------------------------------------------------------- fwht ----

template <typename T>
void fwht_unnormalized(T* data, std::size_t len) {  // fwht.hpp:17-30
  if (len == 0 || (len & (len - 1)) != 0) throw std::invalid_argument("fwht: length is not a power of two");
  for (std::size_t h = 1; h < len; h <<= 1)
    for (std::size_t i = 0; i < len; i += h << 1)
      for (std::size_t j = i; j < i + h; ++j) {
        const T x = data[j];
        const T y = data[j + h];
        data[j] = x + y;
        data[j + h] = x - y;
      }
}

template <typename T>
void fwht_normalized(T* data, std::size_t len) {  // fwht.hpp:35-39
  fwht_unnormalized(data, len);
  const T scale = T(1) / std::sqrt(static_cast<T>(len));
  for (std::size_t i = 0; i < len; ++i) data[i] *= scale;
}

template void fwht_unnormalized<double>(double*, std::size_t);
template void fwht_unnormalized<float>(float*, std::size_t);
template void fwht_normalized<double>(double*, std::size_t);
template void fwht_normalized<float>(float*, std::size_t);

// --------------------------------------------------------------- sketch ----

int even_log2_ceil(std::int64_t n) {  // sketch.hpp:58-63
  if (n < 1) throw std::invalid_argument("even_log2_ceil: n must be positive");
  int k = 2;
  while ((std::int64_t{1} << k) < n) k += 2;
  return k;
}

template <typename T>
const T* Sketch<T>::column(std::int64_t ell) const {  // sketch.hpp:114-117
  if (ell < 0 || ell >= design.L) throw std::out_of_range("Sketch::column: index out of range");
  return columns.data() + ell * m;
}

// sketch.hpp:171-196 for one Kerdock basis: signs Q_s(pos) (176-179), rows in
// 32-row tiles masked + zero padded (182-186), unnormalised FWHT (187),
// transposed write into the basis' d columns of m values (191-196).
template <typename T>
void kerdock_block(const T* a, std::int64_t m, std::int64_t n, const DesignParams& design, const std::uint64_t* mat,
                   T* block, std::vector<T>& sign, std::vector<T>& tile) {
  constexpr std::int64_t kRowTile = 32;
  const std::int64_t d = design.d;
  sign.resize(static_cast<std::size_t>(d));
  tile.resize(static_cast<std::size_t>(kRowTile * d));
  for (std::int64_t j = 0; j < d; ++j)
    sign[j] = quadratic_form(mat, design.k, coords_of_position(static_cast<std::uint64_t>(j), design.k)) ? T(-1) : T(1);
  for (std::int64_t i0 = 0; i0 < m; i0 += kRowTile) {
    const std::int64_t rows = std::min(kRowTile, m - i0);
    for (std::int64_t r = 0; r < rows; ++r) {
      T* buf = tile.data() + r * d;
      const T* arow = a + (i0 + r) * n;
      for (std::int64_t j = 0; j < n; ++j) buf[j] = sign[j] * arow[j];
      std::fill(buf + n, buf + d, T(0));
      fwht_unnormalized(buf, static_cast<std::size_t>(d));
    }
    for (std::int64_t w = 0; w < d; ++w) {
      T* dst = block + w * m + i0;
      const T* src = tile.data() + w;
      for (std::int64_t r = 0; r < rows; ++r) dst[r] = src[r * d];
    }
  }
}
template void kerdock_block<double>(const double*, std::int64_t, std::int64_t, const DesignParams&,
                                    const std::uint64_t*, double*, std::vector<double>&, std::vector<double>&);
template void kerdock_block<float>(const float*, std::int64_t, std::int64_t, const DesignParams&,
                                   const std::uint64_t*, float*, std::vector<float>&, std::vector<float>&);

template <typename T>
Sketch<T> preprocess(const T* a, std::int64_t m, std::int64_t n, int threads) {
  // sketch.hpp:149-211. Per Kerdock basis s: sign table (176-179), 32-row tiles
  // masked + zero padded (182-186), unnormalised FWHT (187), transposed write
  // into column s*d + w (191-196). Identity block sqrt(d) * A[:,w] (200-208).
  if (m < 1 || n < 1) throw std::invalid_argument("preprocess: matrix must be nonempty");
  for (std::int64_t i = 0; i < m * n; ++i)
    if (!std::isfinite(static_cast<double>(a[i])))
      throw std::invalid_argument("preprocess: matrix entries must be finite");
  Sketch<T> sk;
  sk.design = DesignParams::make(even_log2_ceil(n));
  sk.m = m;
  sk.n = n;
  sk.a.assign(a, a + m * n);
  const std::int64_t d = sk.design.d, L = sk.design.L, nk = sk.design.kerdock_bases();
  try {
    sk.columns.assign(static_cast<std::size_t>(m) * static_cast<std::size_t>(L), T(0));
  } catch (const std::bad_alloc&) {
    throw std::runtime_error("preprocess: cannot allocate sketch of " +
                             std::to_string(static_cast<std::uint64_t>(m) * L * sizeof(T)) + " bytes");
  }
  sk.kerdock.resize(static_cast<std::size_t>(nk));
  for (std::int64_t s = 0; s < nk; ++s) sk.kerdock[s] = kerdock_matrix(sk.design, static_cast<std::uint64_t>(s));

  T* cols = sk.columns.data();
  auto work = [&](std::int64_t s_first, std::int64_t s_last) {
    std::vector<T> sign, tile;
    for (std::int64_t s = s_first; s < s_last; ++s)
      kerdock_block(a, m, n, sk.design, sk.kerdock[s].data(), cols + s * d * m, sign, tile);
  };
  // sketch.hpp:37-53: fork-join over disjoint basis ranges (schedule-invariant).
  threads = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(threads, nk)));
  if (threads <= 1) {
    work(0, nk);
  } else {
    std::vector<std::thread> pool;
    const std::int64_t per = (nk + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
      const std::int64_t f = t * per, l = std::min(nk, f + per);
      if (f >= l) break;
      pool.emplace_back([&work, f, l] { work(f, l); });
    }
    for (auto& th : pool) th.join();
  }
  const T sqrt_d = static_cast<T>(std::sqrt(static_cast<double>(d)));
  for (std::int64_t w = 0; w < d; ++w) {
    T* dst = cols + (nk * d + w) * m;
    if (w < n)
      for (std::int64_t i = 0; i < m; ++i) dst[i] = sqrt_d * a[i * n + w];
  }
  // sketch.hpp:126-131 — row_norm_max over the embedded matrix (norm in double).
  double rn = 0;
  for (std::int64_t i = 0; i < m; ++i) {
    double acc = 0;
    for (std::int64_t j = 0; j < n; ++j) acc += static_cast<double>(a[i * n + j]) * static_cast<double>(a[i * n + j]);
    rn = std::max(rn, std::sqrt(acc));
  }
  sk.row_norm_max = rn;
  return sk;
}

template struct Sketch<double>;
template struct Sketch<float>;
template Sketch<double> preprocess<double>(const double*, std::int64_t, std::int64_t, int);
template Sketch<float> preprocess<float>(const float*, std::int64_t, std::int64_t, int);

// ------------------------------------------------------------------ rng ----

std::uint64_t SeededRng::index(std::uint64_t bound) {  // rng.hpp:20-23
  return static_cast<std::uint64_t>((static_cast<unsigned __int128>(eng_()) * bound) >> 64);
}

double SeededRng::unit_double() {  // rng.hpp:26-28
  return (static_cast<double>(eng_() >> 11) + 1.0) * 0x1.0p-53;
}

double SeededRng::gaussian() {  // rng.hpp:31-43
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  const double u1 = unit_double();
  const double u2 = unit_double();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
  spare_ = r * std::sin(theta);
  have_spare_ = true;
  return r * std::cos(theta);
}

std::uint64_t mix_seed(std::uint64_t z) {  // rng.hpp:54-59
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// --------------------------------------------------------------- stream ----

void StreamParams::validate() const {  // stream.hpp:30-38
  if (!(epsilon > delta) || delta < 0) throw std::invalid_argument("StreamParams: need epsilon > delta >= 0");
  if (s < 1) throw std::invalid_argument("StreamParams: need s >= 1");
  if (J < 1 || K < 1) throw std::invalid_argument("StreamParams: need J, K >= 1");
  if (widen < 1) throw std::invalid_argument("StreamParams: need widen >= 1");
  if (J > std::numeric_limits<std::int64_t>::max() / K) throw std::overflow_error("StreamParams: J*K overflows");
}

std::pair<std::int64_t, std::int64_t> choose_params(double r, double gamma, double eta, std::int64_t m) {
  // stream.hpp:58-69
  if (!(gamma > 0)) throw std::invalid_argument("choose_params: gamma must be positive");
  if (!(eta > 0) || eta > 1) throw std::invalid_argument("choose_params: eta must be in (0,1]");
  if (m < 1) throw std::invalid_argument("choose_params: m must be positive");
  const double e2 = 7.38905609893065;
  const double j_real = 4.0 * e2 * r * r / (gamma * gamma);
  const auto j = static_cast<std::int64_t>(std::max(1.0, std::ceil(j_real)));
  const double k_real = 2.0 * std::log(static_cast<double>(m) / eta);
  const auto k = std::max<std::int64_t>(1, static_cast<std::int64_t>(std::ceil(k_real)));
  return {j, k};
}

void reversed_q_rows(const std::uint64_t* rows, int k, std::uint64_t* rev) {  // stream.hpp:76-84
  for (int a = 0; a < k; ++a) {
    std::uint64_t row = 0;
    for (int b = 0; b < k; ++b)
      if ((rows[k - 1 - a] >> (k - 1 - b)) & 1u) row |= std::uint64_t{1} << b;
    rev[a] = row;
  }
}

template <typename T>
T kerdock_inner_product(const T* x, std::int64_t n, std::int64_t d, const std::uint64_t* rev_rows,
                        std::uint64_t wpos) {
  // stream.hpp:89-103: Gray-code walk pos = t ^ (t >> 1); Q updated by polarization.
  T acc = 0;
  std::uint64_t pos = 0;
  int sign = 0;
  for (std::uint64_t t = 0;; ++t) {
    if (static_cast<std::int64_t>(pos) < n) acc += sign ? -x[pos] : x[pos];
    if (t + 1 == static_cast<std::uint64_t>(d)) break;
    const int b = std::countr_zero(t + 1);
    sign ^= std::popcount(rev_rows[b] & pos) & 1;
    sign ^= static_cast<int>((wpos >> b) & 1u);
    pos ^= std::uint64_t{1} << b;
  }
  return acc;
}
template double kerdock_inner_product<double>(const double*, std::int64_t, std::int64_t, const std::uint64_t*, std::uint64_t);
template float kerdock_inner_product<float>(const float*, std::int64_t, std::int64_t, const std::uint64_t*, std::uint64_t);

double inner_product_with_design(const double* x, std::int64_t n, const DesignParams& p, std::int64_t ell) {
  // stream.hpp:109-121
  if (n < 1 || n > p.d) throw std::invalid_argument("inner_product_with_design: bad vector length");
  const DecodedIndex idx = decode_index(p, ell);
  if (idx.identity)
    return static_cast<std::int64_t>(idx.wpos) < n ? std::sqrt(static_cast<double>(p.d)) * x[idx.wpos] : 0.0;
  const auto m = kerdock_matrix(p, idx.s);
  std::uint64_t rev[16];
  reversed_q_rows(m.data(), p.k, rev);
  return kerdock_inner_product(x, n, p.d, rev, idx.wpos);
}

template <typename T>
std::vector<T> median_of_batch_means(const T* means, std::int64_t m, std::int64_t K) {
  // stream.hpp:126-143: nth_element at K/2; even K -> 0.5*(max(lower half) + nth).
  std::vector<T> mu(static_cast<std::size_t>(m));
  std::vector<T> scratch(static_cast<std::size_t>(K));
  for (std::int64_t i = 0; i < m; ++i) {
    for (std::int64_t b = 0; b < K; ++b) scratch[b] = means[b * m + i];
    const auto h = scratch.begin() + K / 2;
    std::nth_element(scratch.begin(), h, scratch.end());
    if (K % 2 == 1) {
      mu[i] = *h;
    } else {
      const T lower = *std::max_element(scratch.begin(), h);
      mu[i] = T(0.5) * (lower + *h);
    }
  }
  return mu;
}
template std::vector<double> median_of_batch_means<double>(const double*, std::int64_t, std::int64_t);
template std::vector<float> median_of_batch_means<float>(const float*, std::int64_t, std::int64_t);

std::vector<std::int64_t> draw_samples(std::int64_t L, const StreamParams& p) {  // stream.hpp:173-182
  p.validate();
  std::vector<std::int64_t> out(static_cast<std::size_t>(p.J * p.K));
  SeededRng rng(p.seed);
  for (auto& ell : out) ell = static_cast<std::int64_t>(rng.index(static_cast<std::uint64_t>(L)));
  return out;
}

std::int64_t candidate_count(std::int64_t s, std::int64_t widen, std::int64_t m) {  // stream.hpp:245-246
  return (s > m / widen) ? m : std::min(widen * s, m);
}

template <typename T>
TransformResult<T> transform_with_samples(const Sketch<T>& sk, const T* x, const StreamParams& p,
                                          const std::vector<std::int64_t>& indices) {
  // stream.hpp:197-268
  p.validate();
  if (static_cast<std::int64_t>(indices.size()) != p.J * p.K)
    throw std::invalid_argument("transform: drawn sample count does not match J*K");
  const std::int64_t m = sk.m, n = sk.n;
  const DesignParams& design = sk.design;
  const std::int64_t kb = design.kerdock_bases() * design.d;
  const T sqrt_d = static_cast<T>(std::sqrt(static_cast<double>(design.d)));

  std::vector<T> means(static_cast<std::size_t>(m * p.K), T(0));
  std::uint64_t rev[16];
  std::int64_t cached_s = -1;
  for (std::int64_t b = 0; b < p.K; ++b) {
    T* col_sum = means.data() + b * m;
    for (std::int64_t j = 0; j < p.J; ++j) {
      const std::int64_t ell = indices[static_cast<std::size_t>(b * p.J + j)];
      if (ell < 0 || ell >= design.L) throw std::out_of_range("Sketch::column: index out of range");
      T t;
      if (ell >= kb) {
        const std::int64_t pos = ell - kb;
        t = pos < n ? sqrt_d * x[pos] : T(0);
      } else {
        const std::int64_t s = ell / design.d;
        if (s != cached_s) {
          reversed_q_rows(sk.kerdock[s].data(), design.k, rev);
          cached_s = s;
        }
        t = kerdock_inner_product(x, n, design.d, rev, static_cast<std::uint64_t>(ell % design.d));
      }
      if (t == T(0)) continue;  // stream.hpp:230
      const T* col = sk.column(ell);
      for (std::int64_t i = 0; i < m; ++i) col_sum[i] += t * col[i];  // mul, round, add, round
    }
  }
  for (auto& v : means) v /= static_cast<T>(p.J);  // stream.hpp:237: divide, not reciprocal

  TransformResult<T> res;
  res.mu = median_of_batch_means(means.data(), m, p.K);
  res.samples_used = p.J * p.K;
  const std::int64_t want = candidate_count(p.s, p.widen, m);
  std::vector<std::int64_t> order(static_cast<std::size_t>(m));
  std::iota(order.begin(), order.end(), std::int64_t{0});
  const auto& mu = res.mu;
  const auto by_mag = [&mu](std::int64_t a, std::int64_t b) {  // stream.hpp:248-255
    const T ma = std::abs(mu[a]), mb = std::abs(mu[b]);
    return ma != mb ? ma > mb : a < b;
  };
  std::nth_element(order.begin(), order.begin() + want, order.end(), by_mag);
  res.candidate_set.assign(order.begin(), order.begin() + want);
  std::sort(res.candidate_set.begin(), res.candidate_set.end());
  for (const std::int64_t i : res.candidate_set) {  // stream.hpp:259-266
    T v = 0;
    const T* row = sk.a.data() + i * n;
    for (std::int64_t j = 0; j < n; ++j) v += row[j] * x[j];
    if (std::abs(v) >= static_cast<T>(p.epsilon)) {
      res.support.push_back(i);
      res.values.push_back(v);
    }
  }
  return res;
}
template TransformResult<double> transform_with_samples<double>(const Sketch<double>&, const double*,
                                                                const StreamParams&, const std::vector<std::int64_t>&);
template TransformResult<float> transform_with_samples<float>(const Sketch<float>&, const float*,
                                                              const StreamParams&, const std::vector<std::int64_t>&);

template <typename T>
TransformResult<T> transform_gathered(const T* a, std::int64_t m, std::int64_t n, const T* x, const StreamParams& p,
                                      const std::vector<std::int64_t>& indices, const T* gathered,
                                      const std::vector<std::vector<std::uint64_t>>* kerdock_set) {
  // Same steps as transform_with_samples; sk.column(ell) replaced by the
  // gathered copy (stream.hpp:235-236).
  p.validate();
  if (static_cast<std::int64_t>(indices.size()) != p.J * p.K)
    throw std::invalid_argument("transform: drawn sample count does not match J*K");
  const DesignParams design = DesignParams::make(even_log2_ceil(n));
  const std::int64_t kb = design.kerdock_bases() * design.d;
  const T sqrt_d = static_cast<T>(std::sqrt(static_cast<double>(design.d)));
  std::vector<T> means(static_cast<std::size_t>(m * p.K), T(0));
  std::uint64_t rev[16];
  std::int64_t cached_s = -1;
  for (std::int64_t b = 0; b < p.K; ++b) {
    T* col_sum = means.data() + b * m;
    for (std::int64_t j = 0; j < p.J; ++j) {
      const std::int64_t jj = b * p.J + j;
      const std::int64_t ell = indices[static_cast<std::size_t>(jj)];
      if (ell < 0 || ell >= design.L) throw std::out_of_range("Sketch::column: index out of range");
      T t;
      if (ell >= kb) {
        const std::int64_t pos = ell - kb;
        t = pos < n ? sqrt_d * x[pos] : T(0);
      } else {
        const std::int64_t s = ell / design.d;
        if (s != cached_s) {  // the reference reads sk.kerdock_set() (built once, sketch.hpp:130)
          if (kerdock_set != nullptr) {
            reversed_q_rows((*kerdock_set)[static_cast<std::size_t>(s)].data(), design.k, rev);
          } else {
            const auto mat = kerdock_matrix(design, static_cast<std::uint64_t>(s));
            reversed_q_rows(mat.data(), design.k, rev);
          }
          cached_s = s;
        }
        t = kerdock_inner_product(x, n, design.d, rev, static_cast<std::uint64_t>(ell % design.d));
      }
      if (t == T(0)) continue;
      const T* col = gathered + jj * m;
      for (std::int64_t i = 0; i < m; ++i) col_sum[i] += t * col[i];
    }
  }
  for (auto& v : means) v /= static_cast<T>(p.J);
  TransformResult<T> res;
  res.mu = median_of_batch_means(means.data(), m, p.K);
  res.samples_used = p.J * p.K;
  const std::int64_t want = candidate_count(p.s, p.widen, m);
  std::vector<std::int64_t> order(static_cast<std::size_t>(m));
  std::iota(order.begin(), order.end(), std::int64_t{0});
  const auto& mu = res.mu;
  std::nth_element(order.begin(), order.begin() + want, order.end(), [&mu](std::int64_t u, std::int64_t w) {
    const T mu_u = std::abs(mu[u]), mu_w = std::abs(mu[w]);
    return mu_u != mu_w ? mu_u > mu_w : u < w;
  });
  res.candidate_set.assign(order.begin(), order.begin() + want);
  std::sort(res.candidate_set.begin(), res.candidate_set.end());
  for (const std::int64_t i : res.candidate_set) {
    T v = 0;
    for (std::int64_t j = 0; j < n; ++j) v += a[i * n + j] * x[j];
    if (std::abs(v) >= static_cast<T>(p.epsilon)) {
      res.support.push_back(i);
      res.values.push_back(v);
    }
  }
  return res;
}
template TransformResult<double> transform_gathered<double>(const double*, std::int64_t, std::int64_t, const double*,
                                                            const StreamParams&, const std::vector<std::int64_t>&,
                                                            const double*,
                                                            const std::vector<std::vector<std::uint64_t>>*);
template TransformResult<float> transform_gathered<float>(const float*, std::int64_t, std::int64_t, const float*,
                                                          const StreamParams&, const std::vector<std::int64_t>&,
                                                          const float*, const std::vector<std::vector<std::uint64_t>>*);

// ----------------------------------------------------------- generators ----

std::vector<double> gen_orthogonal(std::int64_t n, std::uint64_t seed) {
  // generators.hpp:20-33. G filled row by row from SeededRng::gaussian; Q of
  // G = QR with diag(R) > 0 is unique, so this Householder restatement agrees
  // with Eigen::HouseholderQR + sign fix up to rounding.
  if (n < 1) throw std::invalid_argument("gen_orthogonal: n must be positive");
  SeededRng rng(seed);
  std::vector<double> g(static_cast<std::size_t>(n * n));  // column-major working copy
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t j = 0; j < n; ++j) g[j * n + i] = rng.gaussian();
  std::vector<double> vs(static_cast<std::size_t>(n * n), 0.0), betas(static_cast<std::size_t>(n), 0.0),
      rdiag(static_cast<std::size_t>(n), 0.0);
  for (std::int64_t kcol = 0; kcol < n; ++kcol) {
    double* col = g.data() + kcol * n;
    double norm2 = 0;
    for (std::int64_t i = kcol; i < n; ++i) norm2 += col[i] * col[i];
    const double norm = std::sqrt(norm2);
    const double alpha = col[kcol] >= 0 ? -norm : norm;
    double* v = vs.data() + kcol * n;
    for (std::int64_t i = kcol; i < n; ++i) v[i] = col[i];
    v[kcol] -= alpha;
    double vn2 = 0;
    for (std::int64_t i = kcol; i < n; ++i) vn2 += v[i] * v[i];
    const double beta = vn2 > 0 ? 2.0 / vn2 : 0.0;
    betas[kcol] = beta;
    for (std::int64_t c = kcol; c < n; ++c) {
      double* cc = g.data() + c * n;
      double dot = 0;
      for (std::int64_t i = kcol; i < n; ++i) dot += v[i] * cc[i];
      dot *= beta;
      for (std::int64_t i = kcol; i < n; ++i) cc[i] -= dot * v[i];
    }
    rdiag[kcol] = g[kcol * n + kcol];
  }
  // Q = H_0 H_1 ... H_{n-1} applied to I (column-major).
  std::vector<double> q(static_cast<std::size_t>(n * n), 0.0);
  for (std::int64_t i = 0; i < n; ++i) q[i * n + i] = 1.0;
  for (std::int64_t kcol = n - 1; kcol >= 0; --kcol) {
    const double* v = vs.data() + kcol * n;
    const double beta = betas[kcol];
    for (std::int64_t c = 0; c < n; ++c) {
      double* qc = q.data() + c * n;
      double dot = 0;
      for (std::int64_t i = kcol; i < n; ++i) dot += v[i] * qc[i];
      dot *= beta;
      for (std::int64_t i = kcol; i < n; ++i) qc[i] -= dot * v[i];
    }
  }
  std::vector<double> out(static_cast<std::size_t>(n * n));
  for (std::int64_t j = 0; j < n; ++j) {
    const double sgn = rdiag[j] < 0 ? -1.0 : 1.0;
    for (std::int64_t i = 0; i < n; ++i) out[i * n + j] = sgn * q[j * n + i];
  }
  return out;
}

std::vector<double> gen_exact_sparse(const double* a, std::int64_t m, std::int64_t n, std::int64_t s,
                                     std::uint64_t seed, double* x_out) {
  // generators.hpp:38-55: partial Fisher-Yates for s distinct rows, value
  // +-1/sqrt(s) by coin; x = A^T truth.
  if (s < 1 || s > m) throw std::invalid_argument("gen_exact_sparse: need 1 <= s <= m");
  SeededRng rng(seed);
  std::vector<std::int64_t> perm(static_cast<std::size_t>(m));
  std::iota(perm.begin(), perm.end(), std::int64_t{0});
  std::vector<double> truth(static_cast<std::size_t>(m), 0.0);
  const double mag = 1.0 / std::sqrt(static_cast<double>(s));
  for (std::int64_t i = 0; i < s; ++i) {
    const auto j = i + static_cast<std::int64_t>(rng.index(static_cast<std::uint64_t>(m - i)));
    std::swap(perm[i], perm[j]);
    truth[perm[i]] = rng.coin() ? mag : -mag;
  }
  for (std::int64_t j = 0; j < n; ++j) {
    double acc = 0;
    for (std::int64_t i = 0; i < m; ++i) acc += a[i * n + j] * truth[i];
    x_out[j] = acc;
  }
  return truth;
}

// ----------------------------------------------- kerdock.hpp:198-317 verifiers --

std::vector<double> materialize_design(const DesignParams& p) {  // kerdock.hpp:160-188
  const std::int64_t d = p.d, nk = p.kerdock_bases();
  std::vector<double> u(static_cast<std::size_t>(d * p.L), 0.0);
  const double scale = 1.0 / std::sqrt(static_cast<double>(d));
  std::vector<double> sign(static_cast<std::size_t>(d));
  for (std::int64_t s = 0; s < nk; ++s) {
    const auto m = kerdock_matrix(p, static_cast<std::uint64_t>(s));
    for (std::int64_t j = 0; j < d; ++j)
      sign[j] = quadratic_form(m.data(), p.k, coords_of_position(static_cast<std::uint64_t>(j), p.k)) ? -scale : scale;
    for (std::int64_t w = 0; w < d; ++w) {
      double* col = u.data() + (s * d + w) * d;
      for (std::int64_t j = 0; j < d; ++j) col[j] = (std::popcount(static_cast<std::uint64_t>(w & j)) & 1) ? -sign[j] : sign[j];
    }
  }
  for (std::int64_t w = 0; w < d; ++w) u[static_cast<std::size_t>((nk * d + w) * d + w)] = 1.0;  // identity block last
  return u;
}

namespace {

// G = B1^T B2 for two d-column blocks of a column-major d x L matrix.
void block_gram(const double* b1, const double* b2, std::int64_t d, std::vector<double>& g) {
  g.assign(static_cast<std::size_t>(d * d), 0.0);
  for (std::int64_t i = 0; i < d; ++i)
    for (std::int64_t j = 0; j < d; ++j) {
      const double* x = b1 + i * d;
      const double* y = b2 + j * d;
      double acc = 0;
      for (std::int64_t t = 0; t < d; ++t) acc += x[t] * y[t];
      g[static_cast<std::size_t>(i * d + j)] = acc;
    }
}

}  // namespace

MubReport verify_mub(const DesignParams& p, int cap) {  // kerdock.hpp:213-256
  if (p.k > cap) throw std::invalid_argument("verify_mub: k exceeds the verification cap");
  const std::int64_t d = p.d, nb = p.kerdock_bases() + 1;
  const std::vector<double> u = materialize_design(p);
  MubReport rep;
  rep.min_cross_sq = std::numeric_limits<double>::infinity();
  rep.max_cross_sq = -std::numeric_limits<double>::infinity();
  std::vector<double> g;
  for (std::int64_t b = 0; b < nb; ++b) {
    const double* blk = u.data() + b * d * d;
    block_gram(blk, blk, d, g);
    for (std::int64_t i = 0; i < d; ++i)
      for (std::int64_t j = 0; j < d; ++j)
        rep.max_within_gram_dev =
            std::max(rep.max_within_gram_dev, std::abs(g[static_cast<std::size_t>(i * d + j)] - (i == j ? 1.0 : 0.0)));
  }
  auto check_cross = [&](std::int64_t b, std::int64_t b2) {
    block_gram(u.data() + b * d * d, u.data() + b2 * d * d, d, g);
    for (const double c : g) {
      const double sq = c * c;
      rep.min_cross_sq = std::min(rep.min_cross_sq, sq);
      rep.max_cross_sq = std::max(rep.max_cross_sq, sq);
      rep.max_cross_dev = std::max(rep.max_cross_dev, std::abs(sq - 1.0 / static_cast<double>(d)));
    }
  };
  if (p.k <= 6) {
    for (std::int64_t b = 0; b < nb; ++b)
      for (std::int64_t b2 = b + 1; b2 < nb; ++b2) check_cross(b, b2);
  } else {
    rep.exhaustive = false;
    std::mt19937_64 rng(0x6d7562u);  // the reference's fixed seed
    for (int i = 0; i < 256; ++i) {
      const auto b = static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(nb));
      auto b2 = static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(nb - 1));
      if (b2 >= b) ++b2;
      check_cross(b, b2);
    }
  }
  if (!std::isfinite(rep.min_cross_sq)) rep.min_cross_sq = rep.max_cross_sq = 0;
  return rep;
}

double design_moment_target(std::int64_t d, int k) {  // kerdock.hpp:267-276
  double num = 1, den = 1;
  for (int i = 0; i < k; ++i) {
    num *= static_cast<double>(2 * i + 1);
    den *= static_cast<double>(d + 2 * i);
  }
  return num / den;
}

MomentReport design_moments_of(const double* u, std::int64_t d, std::int64_t L) {  // kerdock.hpp:280-297
  MomentReport rep;
  double sum2 = 0, sum4 = 0;
  for (std::int64_t a = 0; a < L; ++a)
    for (std::int64_t b = 0; b < L; ++b) {
      const double* x = u + a * d;
      const double* y = u + b * d;
      double ip = 0;
      for (std::int64_t t = 0; t < d; ++t) ip += x[t] * y[t];
      const double sq = ip * ip;
      sum2 += sq;
      sum4 += sq * sq;
    }
  const double pairs = static_cast<double>(L) * static_cast<double>(L);
  rep.m1 = sum2 / pairs;
  rep.m2 = sum4 / pairs;
  return rep;
}

MomentReport verify_design_moments(const DesignParams& p, int cap) {  // kerdock.hpp:301-315
  if (p.k > cap) throw std::invalid_argument("verify_design_moments: k exceeds the verification cap");
  const std::vector<double> u = materialize_design(p);
  if (p.k <= 6) return design_moments_of(u.data(), p.d, p.L);
  MomentReport rep;
  rep.exact = false;
  std::mt19937_64 rng(0x6d6f6du);
  const int samples = 4'000'000;
  double sum2 = 0, sum4 = 0;
  for (int i = 0; i < samples; ++i) {
    const auto a = static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(p.L));
    const auto b = static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(p.L));
    const double* x = u.data() + a * p.d;
    const double* y = u.data() + b * p.d;
    double ip = 0;
    for (std::int64_t t = 0; t < p.d; ++t) ip += x[t] * y[t];
    const double sq = ip * ip;
    sum2 += sq;
    sum4 += sq * sq;
  }
  rep.m1 = sum2 / samples;
  rep.m2 = sum4 / samples;
  return rep;
}

void verify_kerdock_set(const DesignParams& p, bool* skew, std::int64_t* bad_pairs) {  // cli.hpp:45-60
  const std::int64_t nk = p.kerdock_bases();
  std::vector<std::vector<std::uint64_t>> mats(static_cast<std::size_t>(nk));
  bool ok = true;
  for (std::int64_t s = 0; s < nk; ++s) {
    mats[s] = kerdock_matrix(p, static_cast<std::uint64_t>(s));
    for (int i = 0; i < p.k && ok; ++i) ok = ((mats[s][i] >> i) & 1) == 0;
    for (int i = 0; i < p.k && ok; ++i)
      for (int j = 0; j < p.k && ok; ++j) ok = ((mats[s][i] >> j) & 1) == ((mats[s][j] >> i) & 1);
  }
  std::int64_t bad = 0;
  std::vector<std::uint64_t> sum(static_cast<std::size_t>(p.k));
  for (std::int64_t a = 0; a < nk; ++a)
    for (std::int64_t b = a + 1; b < nk; ++b) {
      for (int i = 0; i < p.k; ++i) sum[i] = mats[a][i] ^ mats[b][i];
      if (gf2_rank(sum.data(), p.k) != p.k) ++bad;
    }
  *skew = ok;
  *bad_pairs = bad;
}

}  // namespace fst_oracle
