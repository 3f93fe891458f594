// ORACLE — TEST INFRASTRUCTURE ONLY.
// Golden-vector generator built from the reference's OWN sources: the two
// reference headers on the path that compile without Eigen
// (/root/reference/proj/include/fst/gf2.hpp and rng.hpp) are included
// unmodified from where they lie. Build: `make -C oracle ref` -> oracle/_ref/.
// Output (stdout): one JSON document; tests/golden/make_golden.py stores it as
// tests/golden/ref_gf2_rng.json, which the CPU tests compare the restatement
// against (the GPU box never reads /root/reference).
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "fst/gf2.hpp"
#include "fst/rng.hpp"

static void print_u64_list(const char* key, const std::vector<std::uint64_t>& v, bool last = false) {
  std::printf("\"%s\": [", key);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s\"%llu\"", i ? "," : "", (unsigned long long)v[i]);
  std::printf("]%s\n", last ? "" : ",");
}

int main() {
  std::printf("{\n");
  // Raw engine, bounded index draws (the stream's sampling path, rng.hpp:20-23).
  const std::uint64_t seeds[] = {0ull, 1ull, 42ull, 9000ull, 8080ull, 0x747278ull, 0xdeadbeefcafef00dull};
  std::printf("\"rng\": [\n");
  for (std::size_t si = 0; si < sizeof(seeds) / sizeof(seeds[0]); ++si) {
    const std::uint64_t seed = seeds[si];
    std::printf("{\"seed\": \"%llu\",\n", (unsigned long long)seed);
    {
      fst::SeededRng r(seed);
      std::vector<std::uint64_t> v;
      for (int i = 0; i < 1000; ++i) v.push_back(r.next_u64());
      print_u64_list("u64", v);
    }
    const std::uint64_t bounds[] = {12ull, 33024ull, 525312ull, 8392704ull, 134234112ull};
    std::printf("\"index\": {");
    for (int b = 0; b < 5; ++b) {
      fst::SeededRng r(seed);
      std::printf("%s\"%llu\": [", b ? "," : "", (unsigned long long)bounds[b]);
      for (int i = 0; i < 800; ++i) std::printf("%s%llu", i ? "," : "", (unsigned long long)r.index(bounds[b]));
      std::printf("]");
    }
    std::printf("},\n");
    {
      fst::SeededRng r(seed);
      std::printf("\"gaussian\": [");
      for (int i = 0; i < 64; ++i) std::printf("%s%.17g", i ? "," : "", r.gaussian());
      std::printf("],\n");
    }
    {
      fst::SeededRng r(seed);
      std::printf("\"unit_double\": [");
      for (int i = 0; i < 64; ++i) std::printf("%s%.17g", i ? "," : "", r.unit_double());
      std::printf("],\n");
    }
    {
      fst::SeededRng r(seed);
      std::printf("\"coin\": [");
      for (int i = 0; i < 64; ++i) std::printf("%s%d", i ? "," : "", r.coin() ? 1 : 0);
      std::printf("],\n");
    }
    std::printf("\"mix_seed\": \"%llu\"}%s\n", (unsigned long long)fst::mix_seed(seed),
                si + 1 < sizeof(seeds) / sizeof(seeds[0]) ? "," : "");
  }
  std::printf("],\n");

  // GF(2^q) arithmetic for every shipped degree (gf2.hpp:205-274).
  std::printf("\"field\": [\n");
  const int qs[] = {1, 3, 5, 7, 9, 11, 13, 15};
  for (int qi = 0; qi < 8; ++qi) {
    const int q = qs[qi];
    fst::FieldCtx ctx(q);
    std::printf("{\"q\": %d, \"modulus\": \"%llu\", \"irreducible\": %d,\n", q,
                (unsigned long long)ctx.modulus(), fst::verify_irreducible(ctx.modulus(), q) ? 1 : 0);
    fst::SeededRng r(1000 + q);
    std::vector<std::uint64_t> as, bs, prods;
    std::vector<std::uint64_t> traces;
    for (int i = 0; i < 200; ++i) {
      const std::uint64_t a = r.index(ctx.order()), b = r.index(ctx.order());
      as.push_back(a);
      bs.push_back(b);
      prods.push_back(fst::field_mul(ctx, {a}, {b}).repr);
      traces.push_back(static_cast<std::uint64_t>(fst::field_trace(ctx, {a})));
    }
    print_u64_list("a", as);
    print_u64_list("b", bs);
    print_u64_list("mul", prods);
    print_u64_list("trace", traces, true);
    std::printf("}%s\n", qi + 1 < 8 ? "," : "");
  }
  std::printf("],\n");

  // Big-endian coordinate map (gf2.hpp:65-78) and rank (gf2.hpp:148-172).
  std::printf("\"coords\": [");
  for (int k : {2, 4, 8, 12}) {
    for (std::uint64_t p : {0ull, 1ull, 5ull, 6ull, 15ull})
      std::printf("%s[%d,%llu,%llu]", (k == 2 && p == 0) ? "" : ",", k, (unsigned long long)p,
                  (unsigned long long)fst::coords_of_position(p & ((1ull << k) - 1), k).word());
  }
  std::printf("],\n");
  std::printf("\"rank\": [");
  {
    fst::SeededRng r(77);
    for (int t = 0; t < 50; ++t) {
      const int dim = 1 + static_cast<int>(r.index(16));
      fst::BitMatrix m(dim);
      std::printf("%s{\"dim\": %d, \"rows\": [", t ? "," : "", dim);
      for (int i = 0; i < dim; ++i) {
        m.set_row(i, r.next_u64() & r.next_u64());
        std::printf("%s\"%llu\"", i ? "," : "", (unsigned long long)m.row(i));
      }
      std::printf("], \"rank\": %d}", fst::gf2_rank(m));
    }
  }
  std::printf("]\n}\n");
  return 0;
}
