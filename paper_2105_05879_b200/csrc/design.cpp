// Host-side Kerdock design tables (see design.hpp).
#include "design.hpp"

#include <algorithm>
#include <cmath>

namespace fstg {

int even_log2_ceil(std::int64_t n) {
  if (n < 1) throw InvalidArgument("even_log2_ceil: n must be positive");
  int k = 2;
  while ((std::int64_t{1} << k) < n) k += 2;
  return k;
}

static std::uint64_t shipped_modulus(int q) {
  // The moduli the reference ships (gf2.hpp:205-218); every sign bit of the
  // design depends on these exact polynomials.
  static const std::uint64_t table[16] = {0,      0x3,   0, 0xB,    0, 0x25,   0, 0x83,
                                          0,      0x211, 0, 0x805,  0, 0x201B, 0, 0x8003};
  if (q < 1 || q > 15 || (q % 2) == 0) throw InvalidArgument("modulus_for_degree: no shipped modulus for this degree");
  return table[q];
}

Design Design::make(int k) {
  if (k < 2 || k % 2 != 0) throw InvalidArgument("DesignParams: k must be a positive even integer");
  if (k > 16) throw InvalidArgument("DesignParams: k > 16 is not supported");
  Design d;
  d.k = k;
  d.d = std::int64_t{1} << k;
  d.L = d.d * (d.d / 2 + 1);
  d.modulus = shipped_modulus(k - 1);
  return d;
}

Field::Field(int q, std::uint64_t modulus) : q_(q), mod_(modulus) {
  // The trace is GF(2)-linear: tr(a) = parity(a & mask) with mask bit i =
  // tr(alpha^i), each computed once as the sum of the Frobenius orbit.
  for (int i = 0; i < q; ++i) {
    std::uint64_t a = std::uint64_t{1} << i, acc = a, pw = a;
    for (int j = 1; j < q; ++j) {
      pw = mul(pw, pw);
      acc ^= pw;
    }
    if (acc > 1) throw std::logic_error("field trace left the prime subfield");
    trace_mask_ |= acc << i;
  }
}

std::uint64_t Field::mul(std::uint64_t a, std::uint64_t b) const {
  // Carry-less product (degree < 2q) then reduction from the top bit down.
  unsigned __int128 prod = 0;
  for (int i = 0; i < q_; ++i)
    if ((b >> i) & 1u) prod ^= static_cast<unsigned __int128>(a) << i;
  for (int bit = 2 * q_ - 2; bit >= q_; --bit)
    if ((prod >> bit) & 1u) prod ^= static_cast<unsigned __int128>(mod_) << (bit - q_);
  return static_cast<std::uint64_t>(prod);
}

std::vector<std::uint64_t> kerdock_matrix(const Design& d, const Field& f, std::uint64_t s) {
  // M_s in the basis {(alpha^0,0)..(alpha^(q-1),0),(0,1)} of GF(2^q) x GF(2):
  // columns are the images (f_c, t_c) = L_s(basis_c) with
  // L_s(x, a) = (s^2 x + s tr(sx) + a s, tr(sx)); row r < q is tr(alpha^r f_c),
  // row q is t_c.
  const int q = d.k - 1;
  if (s >= (std::uint64_t{1} << q)) throw InvalidArgument("kerdock_matrix: field index out of range");
  const std::uint64_t s2 = f.mul(s, s);
  std::vector<std::uint64_t> rows(static_cast<std::size_t>(d.k), 0);
  for (int c = 0; c < d.k; ++c) {
    std::uint64_t fc;
    int tc;
    if (c < q) {
      const std::uint64_t ac = std::uint64_t{1} << c;
      tc = f.trace(f.mul(s, ac));
      fc = f.mul(s2, ac) ^ (tc ? s : 0);
    } else {
      fc = s;
      tc = 0;
    }
    for (int r = 0; r < q; ++r)
      if (f.trace(f.mul(std::uint64_t{1} << r, fc))) rows[r] |= std::uint64_t{1} << c;
    if (tc) rows[q] |= std::uint64_t{1} << c;
  }
  return rows;
}

void reversed_rows(const std::uint64_t* rows, int k, std::uint32_t* rev) {
  for (int a = 0; a < k; ++a) {
    std::uint32_t row = 0;
    for (int b = 0; b < k; ++b)
      if ((rows[k - 1 - a] >> (k - 1 - b)) & 1u) row |= 1u << b;
    rev[a] = row;
  }
}

std::vector<std::uint32_t> reversed_row_table(const Design& d) {
  const Field f(d.k - 1, d.modulus);
  std::vector<std::uint32_t> table(static_cast<std::size_t>(d.kerdock_bases()) * 16, 0);
  for (std::int64_t s = 0; s < d.kerdock_bases(); ++s) {
    const auto rows = kerdock_matrix(d, f, static_cast<std::uint64_t>(s));
    reversed_rows(rows.data(), d.k, table.data() + s * 16);
  }
  return table;
}

void choose_params(double r, double gamma, double eta, std::int64_t m, std::int64_t* J, std::int64_t* K) {
  if (!(gamma > 0)) throw InvalidArgument("choose_params: gamma must be positive");
  if (!(eta > 0) || eta > 1) throw InvalidArgument("choose_params: eta must be in (0,1]");
  if (m < 1) throw InvalidArgument("choose_params: m must be positive");
  const double e2 = 7.38905609893065;  // e^2 as the reference hard-codes it
  const double j_real = 4.0 * e2 * r * r / (gamma * gamma);
  *J = static_cast<std::int64_t>(std::max(1.0, std::ceil(j_real)));
  const double k_real = 2.0 * std::log(static_cast<double>(m) / eta);
  *K = std::max<std::int64_t>(1, static_cast<std::int64_t>(std::ceil(k_real)));
}

std::int64_t candidate_count(std::int64_t s, std::int64_t widen, std::int64_t m) {
  if (widen < 1) return m;
  return (s > m / widen) ? m : std::min(widen * s, m);
}

}  // namespace fstg
