// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Eigen-free CPU restatement of the reference `fst` hot path (arXiv 2105.05879
// reference, /root/reference/proj/include/fst/*.hpp). Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load this code, and only as the checker / CPU baseline. The product
// (paper_2105_05879_b200/) never links or calls it.
//
// Pinning: the restatement is checked against (1) every known-answer and
// property test the reference's own suites hold for this path
// (proj/tests/test_{gf2,fwht,kerdock,sketch,stream,...}.cpp, acceptance.cpp), and
// (2) golden vectors produced by the reference's own gf2.hpp / rng.hpp compiled
// unmodified from /root/reference (oracle/ref_golden.cpp -> oracle/_ref/). The
// rest of the reference needs Eigen (absent, not shimmed). See DESIGN.md §4.
//
// Compile with -ffp-contract=off: the reference builds without -march, i.e.
// SSE2 with no FMA, so every a*b+c is two roundings.
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace fst_oracle {

// ---------------------------------------------------------------- gf2.hpp --

/// gf2.hpp:205-218 — the shipped irreducible moduli (q odd, 1..15).
std::uint64_t modulus_for_degree(int q);
/// gf2.hpp:192-200 — exhaustive trial division.
bool verify_irreducible(std::uint64_t poly, int degree);
/// gf2.hpp:251-261 — shift-and-reduce product in GF(2^q).
std::uint64_t field_mul(int q, std::uint64_t modulus, std::uint64_t a, std::uint64_t b);
/// gf2.hpp:264-274 — trace a + a^2 + ... + a^(2^(q-1)).
int field_trace(int q, std::uint64_t modulus, std::uint64_t a);
/// gf2.hpp:148-172 — rank by bit-packed elimination (rows: bit j of row i = entry (i,j)).
int gf2_rank(const std::uint64_t* rows, int dim);
/// gf2.hpp:65-69 — coordinate c is bit (k-1-c) of p (big-endian).
std::uint64_t coords_of_position(std::uint64_t p, int k);
/// gf2.hpp:72-78
std::uint64_t position_of_coords(std::uint64_t w, int k);

// ------------------------------------------------------------ kerdock.hpp --

/// kerdock.hpp:20-34
struct DesignParams {
  int k = 0;
  std::int64_t d = 0;
  std::int64_t L = 0;
  std::uint64_t modulus = 0;  // FieldCtx(k-1)
  static DesignParams make(int k);
  std::int64_t kerdock_bases() const { return d / 2; }
};

/// kerdock.hpp:38-49 — Q_M(x) = sum_{i<j} M_ij x_i x_j over GF(2).
int quadratic_form(const std::uint64_t* rows, int dim, std::uint64_t x);
/// kerdock.hpp:55-84 — M_s of the standard Kerdock set, k rows.
std::vector<std::uint64_t> kerdock_matrix(const DesignParams& p, std::uint64_t s);

/// kerdock.hpp:102-130 — linear index -> (kerdock?, s, wpos).
struct DecodedIndex {
  bool identity;
  std::uint64_t s;
  std::uint64_t wpos;  // position of w (big-endian coords -> integer)
};
DecodedIndex decode_index(const DesignParams& p, std::int64_t ell);

/// kerdock.hpp:132-167 — s_ell = sqrt(d) * first n coordinates of u_ell.
std::vector<double> projected_design_column(const DesignParams& p, std::int64_t n, std::int64_t ell);

// --------------------------------------------------------------- fwht.hpp --

/// fwht.hpp:17-30 — radix-2, h = 1, 2, 4, ..., butterflies (x+y, x-y).
template <typename T>
void fwht_unnormalized(T* data, std::size_t len);
/// fwht.hpp:35-39
template <typename T>
void fwht_normalized(T* data, std::size_t len);

// ------------------------------------------------------------- sketch.hpp --

/// sketch.hpp:58-63
int even_log2_ceil(std::int64_t n);

/// sketch.hpp:149-211 — columns are column-major m x L (column ell at ell*m).
template <typename T>
struct Sketch {
  DesignParams design;
  std::int64_t m = 0, n = 0;
  std::vector<T> a;        // embedded A, row-major m x n
  std::vector<T> columns;  // m * L
  double row_norm_max = 0;
  std::vector<std::vector<std::uint64_t>> kerdock;  // d/2 matrices, k rows each
  const T* column(std::int64_t ell) const;
};
template <typename T>
Sketch<T> preprocess(const T* a, std::int64_t m, std::int64_t n, int threads = 1);
/// sketch.hpp:171-196 for one basis: block = its d columns of m values.
template <typename T>
void kerdock_block(const T* a, std::int64_t m, std::int64_t n, const DesignParams& design, const std::uint64_t* mat,
                   T* block, std::vector<T>& sign, std::vector<T>& tile);

// ---------------------------------------------------------------- rng.hpp --

/// rng.hpp:13-52 — std::mt19937_64 + multiply-shift bounded draws + Box-Muller.
class SeededRng {
 public:
  explicit SeededRng(std::uint64_t seed) : eng_(seed) {}
  std::uint64_t next_u64() { return eng_(); }
  std::uint64_t index(std::uint64_t bound);
  double unit_double();
  double gaussian();
  bool coin() { return (eng_() >> 63) != 0; }

 private:
  std::mt19937_64 eng_;
  double spare_ = 0;
  bool have_spare_ = false;
};
/// rng.hpp:54-59 — SplitMix64 step.
std::uint64_t mix_seed(std::uint64_t z);

// ------------------------------------------------------------- stream.hpp --

/// stream.hpp:22-39
struct StreamParams {
  double epsilon = 0;
  double delta = 0;
  std::int64_t s = 1;
  std::int64_t J = 1;
  std::int64_t K = 1;
  std::int64_t widen = 10;
  std::uint64_t seed = 0;
  void validate() const;
};

/// stream.hpp:58-69
std::pair<std::int64_t, std::int64_t> choose_params(double row_norm_max, double gamma, double eta,
                                                    std::int64_t m);
/// stream.hpp:76-84
void reversed_q_rows(const std::uint64_t* rows, int k, std::uint64_t* rev_rows);
/// stream.hpp:89-103 — Gray-code walk, sequential summation order.
template <typename T>
T kerdock_inner_product(const T* x, std::int64_t n, std::int64_t d, const std::uint64_t* rev_rows,
                        std::uint64_t wpos);
/// stream.hpp:109-121
double inner_product_with_design(const double* x, std::int64_t n, const DesignParams& p,
                                 std::int64_t ell);
/// stream.hpp:126-143 — means column-major m x K.
template <typename T>
std::vector<T> median_of_batch_means(const T* means, std::int64_t m, std::int64_t K);
/// stream.hpp:173-182
std::vector<std::int64_t> draw_samples(std::int64_t L, const StreamParams& p);
/// stream.hpp:245-246
std::int64_t candidate_count(std::int64_t s, std::int64_t widen, std::int64_t m);

template <typename T>
struct TransformResult {
  std::vector<std::int64_t> support;
  std::vector<T> values;
  std::vector<std::int64_t> candidate_set;
  std::vector<T> mu;
  std::int64_t samples_used = 0;
};

/// stream.hpp:197-268
template <typename T>
TransformResult<T> transform_with_samples(const Sketch<T>& sk, const T* x, const StreamParams& p,
                                          const std::vector<std::int64_t>& indices);

/// The draw_and_gather path (stream.hpp:184-191, 197-268 with
/// drawn.use_gathered): identical arithmetic, columns supplied by the caller
/// (gathered: N x m, row j = column ell_j). Used to check full-size (n=4096)
/// GPU runs without materialising the 275 GB fp64 sketch.
/// kerdock_set: the Kerdock matrices of every basis, built once as the reference's
/// Sketch constructor does (sketch.hpp:130); nullptr rebuilds them per basis change.
template <typename T>
TransformResult<T> transform_gathered(const T* a, std::int64_t m, std::int64_t n, const T* x, const StreamParams& p,
                                      const std::vector<std::int64_t>& indices, const T* gathered,
                                      const std::vector<std::vector<std::uint64_t>>* kerdock_set = nullptr);

// ----------------------------------------------- kerdock.hpp:198-317 verifiers --

/// kerdock.hpp:160-188 (detail::materialize_design): all L unit design vectors
/// as a column-major d x L matrix (column c at c*d), Kerdock blocks first.
std::vector<double> materialize_design(const DesignParams& p);

/// kerdock.hpp:199-208
struct MubReport {
  double max_within_gram_dev = 0;
  double min_cross_sq = 0;
  double max_cross_sq = 0;
  double max_cross_dev = 0;
  bool exhaustive = true;
  bool pass(double tol) const { return max_within_gram_dev <= tol && max_cross_dev <= tol; }
};
/// kerdock.hpp:213-256 (exhaustive for k <= 6, 256 sampled basis pairs above).
MubReport verify_mub(const DesignParams& p, int cap = 8);

/// kerdock.hpp:261-278
struct MomentReport {
  double m1 = 0;
  double m2 = 0;
  bool exact = true;
};
double design_moment_target(std::int64_t d, int k);
/// kerdock.hpp:280-297 — u column-major d x L.
MomentReport design_moments_of(const double* u, std::int64_t d, std::int64_t L);
/// kerdock.hpp:301-315 (exact for k <= 6, 4M sampled pairs above).
MomentReport verify_design_moments(const DesignParams& p, int cap = 8);
/// cli.hpp:45-60: zero-diagonal symmetric matrices, number of basis pairs whose
/// sum is rank-deficient (must be 0 for a Kerdock set).
void verify_kerdock_set(const DesignParams& p, bool* skew, std::int64_t* bad_pairs);

// --------------------------------------------------------- generators.hpp --

/// generators.hpp:20-33 — Haar orthogonal: Householder QR of a SeededRng
/// Gaussian matrix, Q columns sign-fixed so that diag(R) > 0 (unique Q).
std::vector<double> gen_orthogonal(std::int64_t n, std::uint64_t seed);
/// generators.hpp:38-55 — returns truth (m) ; x = A^T truth written to x_out.
std::vector<double> gen_exact_sparse(const double* a, std::int64_t m, std::int64_t n, std::int64_t s,
                                     std::uint64_t seed, double* x_out);

/// experiment.hpp:133-136
inline std::uint64_t gen_seed(std::uint64_t trial_seed) { return mix_seed(trial_seed ^ 0x67656eull); }
inline std::uint64_t stream_seed(std::uint64_t trial_seed) { return mix_seed(trial_seed ^ 0x747278ull); }

}  // namespace fst_oracle
