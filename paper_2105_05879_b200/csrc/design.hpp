// Host-side Kerdock design tables for the B200 path (product code).
//
// Independent implementation of the bit-exact host prerequisites of the hot
// path: GF(2^q) arithmetic (schoolbook carry-less product + top-down
// reduction; trace as a linear functional), the Kerdock matrices M_s
// (reference kerdock.hpp:55-84), and their position-reversed rows
// (stream.hpp:76-84). The device expands these rows into the sign-bit tables
// consumed by the kernels. Cross-checked against the oracle in tests/.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

namespace fstg {

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct OutOfRange : std::out_of_range {
  using std::out_of_range::out_of_range;
};
struct Overflow : std::overflow_error {
  using std::overflow_error::overflow_error;
};
struct NotSupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// sketch.hpp:58-63 — smallest even k with 2^k >= n.
int even_log2_ceil(std::int64_t n);

/// kerdock.hpp:20-34 — d = 2^k points per basis, d/2 Kerdock bases + identity.
struct Design {
  int k = 0;
  std::int64_t d = 0;
  std::int64_t L = 0;
  std::uint64_t modulus = 0;  // GF(2^(k-1)), gf2.hpp:205-218
  std::int64_t kerdock_bases() const { return d / 2; }
  static Design make(int k);
};

/// GF(2^q) with the shipped modulus (gf2.hpp:205-218).
class Field {
 public:
  Field(int q, std::uint64_t modulus);
  std::uint64_t mul(std::uint64_t a, std::uint64_t b) const;
  int trace(std::uint64_t a) const { return __builtin_parityll(a & trace_mask_); }
  int degree() const { return q_; }

 private:
  int q_;
  std::uint64_t mod_;
  std::uint64_t trace_mask_ = 0;  // bit i = tr(alpha^i)
};

/// kerdock.hpp:55-84: k rows, bit c of row r = (M_s)_{r,c}.
std::vector<std::uint64_t> kerdock_matrix(const Design& d, const Field& f, std::uint64_t s);
/// stream.hpp:76-84: rev[a] bit b = M_{k-1-a, k-1-b}.
void reversed_rows(const std::uint64_t* rows, int k, std::uint32_t* rev);

/// Reversed rows of every Kerdock matrix, (d/2) x 16 words (rows >= k zero).
std::vector<std::uint32_t> reversed_row_table(const Design& d);

/// stream.hpp:58-69
void choose_params(double row_norm_max, double gamma, double eta, std::int64_t m, std::int64_t* J,
                   std::int64_t* K);
/// stream.hpp:245-246
std::int64_t candidate_count(std::int64_t s, std::int64_t widen, std::int64_t m);

}  // namespace fstg
