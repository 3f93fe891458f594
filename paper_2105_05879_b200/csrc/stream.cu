// Fused streaming estimator + support refinement (reference stream.hpp:197-268).
//
// One persistent CTA per SM works through vectors v = blockIdx.x, += gridDim.x,
// with warp-specialised roles (see the role map above stream_kernel):
//   * producer (P lanes of the last warp): streams the sampled sketch columns
//     C[:, ell_j] (16 KiB segments) HBM -> shared memory with 1-D bulk copies
//     (cp.async.bulk, SASS UBLKCP) into an S-stage ring guarded by full/empty
//     mbarriers, evict-first in L2, running ahead across vector boundaries.
//   * coefficient warps: t_j = s_ell^T x (stream.hpp:89-103, 218-229) from the
//     lane-transposed Kerdock sign tables and x in shared memory, 8 samples per
//     pass over x, into a 64-slot ring.
//   * consumer warps: per-batch running sums acc += t_j * C[:, ell_j]
//     (stream.hpp:231-234) in registers, / J (stream.hpp:237) into a
//     double-buffered scratch slot (PARTIAL mode: into means_io).
//   * tail warps, overlapping the next vector: entrywise median of the K batch
//     means (stream.hpp:126-143), the `want` largest |mu| with ties to the
//     smaller index by an MSB radix select plus an index-ordered ballot scan
//     (stream.hpp:245-257), the exact fp64-accumulated refinement of those rows
//     of A through a TMA row ring (A L2-resident, evict-last; stream.hpp:259-266)
//     — in fp32 preceded by a screening pass with a rigorous rounding bound, so
//     only candidates not proven below eps pay for the exact dot — and the
//     ordered compaction of the |v| >= eps support.
// STRICT mode reproduces the reference's operation order exactly: Gray-code
// sequential coefficient sums and separately-rounded multiply/add.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "fst_common.cuh"
#include "kernels.hpp"

namespace fstg {

#ifndef FSTG_NCW
#define FSTG_NCW 8
#endif
constexpr int kNCW = FSTG_NCW;              // consumer warps
constexpr int kNC = kNCW * 32;              // consumer threads
#ifndef FSTG_CW
#define FSTG_CW 8
#endif
constexpr int kCW = FSTG_CW;                // coefficient warps
constexpr int kTLW = 7;                     // tail warps (median / select / refine / compact); 24 warps total
constexpr int kTL = kTLW * 32;              // tail threads
constexpr int kThreads = kNC + kCW * 32 + kTL + 32;  // + producer warp (768 threads with 8 consumer warps: 80 regs)
constexpr int kWarpCoef = kNCW, kWarpTail = kNCW + kCW, kWarpProd = kNCW + kCW + kTLW;
#ifndef FSTG_TRING
#define FSTG_TRING 64
#endif
constexpr int kTRing = FSTG_TRING;          // slots of the coefficient ring
static_assert((kTRing & (kTRing - 1)) == 0, "coefficient ring: power of two");
// Samples per coefficient-warp group: one x read from shared memory serves kNS
// samples (8 vs 4: +8% at config 3, profiles/r01_stream_pipeline.txt; 16 spills).
#ifndef FSTG_NS
#define FSTG_NS 8
#endif
constexpr int kNS = FSTG_NS;
constexpr int kSegBytes = 16384;            // one ring stage at most
// samples per consumer iteration for small columns: FAST mode (config 2, fp32 m = 1024:
// 3 / 4 / 5 / 6 -> 1.12M / 1.21M / 1.25M / 1.28M vectors/s) and STRICT mode (config 1, fp64
// m = 256: 4 / 5 / 6 -> 405k / 384k / 364k), profiles/r01_stream_pipeline.txt
#ifndef FSTG_SMALL_GROUP_FAST
#define FSTG_SMALL_GROUP_FAST 6
#endif
#ifndef FSTG_SMALL_GROUP_STRICT
#define FSTG_SMALL_GROUP_STRICT 4
#endif
constexpr int kSmallGroupFast = FSTG_SMALL_GROUP_FAST, kSmallGroupStrict = FSTG_SMALL_GROUP_STRICT;
constexpr int kMaxStages = 64;
// x buffers: coefficients on v+1 while the tail refines v. A third buffer (coefficients two
// vectors ahead) measured 5% slower at config 3 (profiles/r01_stream_pipeline.txt).
constexpr int kXBuf = 3;   // barriers for up to 3; buffers in use: kXBufUse (FSTG_XBUFS for experiments)
constexpr int kXBufUse = 2;
constexpr int kSmemBudget = 227 * 1024;
constexpr int kInflightBytes = 8 * 16384;    // cap on column bytes in flight per SM (shared memory decides)
constexpr int kBarCoef = 2, kBarTail = 3;   // named barrier ids
#ifndef FSTG_RSTAGES
#define FSTG_RSTAGES 6
#endif
constexpr int kRStages = FSTG_RSTAGES;       // refinement ring: tail warp 0 issues, warps 1..kRStages consume
static_assert(kRStages >= 1 && kRStages <= kTLW - 1, "refinement stages are owned by tail warps 1..kTLW-1");
// Stages in use at run time: one fewer for small candidate sets, so the column ring gets a
// sixth 16 KiB stage (config 3, want = 320: 455k -> 464k vectors/s); large sets (config 5 at
// s = 256) keep all kRStages (they are refinement-bound: 172k vs 189k with 5).
#ifndef FSTG_RSTAGES_SMALL_WANT
#define FSTG_RSTAGES_SMALL_WANT 512
#endif
constexpr int64_t kRSmallWant = FSTG_RSTAGES_SMALL_WANT;
// bf16 screening rows per refinement-ring stage (one x pass screens them together)
constexpr int kRRowsBf16 = 2;

// Experiment instrumentation (FSTG_STREAM_DEBUG bit 8): cycles each warp role
// spends in each mbarrier wait, summed over warps (lane 0) into g_wait_cycles.
enum WaitSite {
  kWProdEmpty, kWCoefXEmpty, kWCoefTEmpty, kWTailMFull, kWTailXFull, kWTailREmpty, kWTailRFull,
  kWConsT, kWConsCol, kWConsMEmpty, kWTotProd, kWTotCoef, kWTotTail, kWTotCons, kWSites
};
__device__ unsigned long long g_wait_cycles[kWSites];

#ifndef FSTG_WAIT_PROFILE
#define FSTG_WAIT_PROFILE 0
#endif
// Compiled out unless built with -DFSTG_WAIT_PROFILE=1 (then FSTG_STREAM_DEBUG bit 8
// turns it on): a runtime check on every wait costs the small-d configs ~20%.
constexpr bool kWaitProfile = FSTG_WAIT_PROFILE != 0;
struct WaitProf {
  bool on;
  unsigned long long* acc;  // kWSites shared-memory counters, acc[kWSites] = warps finished
  __device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity, int site) {
    if constexpr (kWaitProfile) {
      if (on) {
        const long long t0 = clock64();
        mbar_wait(bar, parity);
        if ((threadIdx.x & 31) == 0) atomicAdd(&acc[site], static_cast<unsigned long long>(clock64() - t0));
        return;
      }
    }
    mbar_wait(bar, parity);
  }
  // called once per warp when its role ends; the last warp publishes the CTA's totals
  __device__ __forceinline__ void done(int site, long long t_start) {
    if constexpr (kWaitProfile) {
      if (!on || (threadIdx.x & 31) != 0) return;
      atomicAdd(&acc[site], static_cast<unsigned long long>(clock64() - t_start));
      __threadfence_block();
      if (atomicAdd(&acc[kWSites], 1ull) == static_cast<unsigned long long>(blockDim.x / 32 - 1)) {
        for (int i = 0; i < kWSites; ++i) atomicAdd(&g_wait_cycles[i], atomicAdd(&acc[i], 0ull));
      }
    }
  }
};

template <typename T>
struct KeyOf;
template <>
struct KeyOf<float> {
  using K = uint32_t;
  static constexpr int BITS = 32;
  __device__ static K key(float v) { return __float_as_uint(v) & 0x7fffffffu; }
};
template <>
struct KeyOf<double> {
  using K = unsigned long long;
  static constexpr int BITS = 64;
  __device__ static K key(double v) { return static_cast<K>(__double_as_longlong(v)) & 0x7fffffffffffffffull; }
};

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int N = 4;
  using V = float4;
  __device__ static void get(const V& v, float (&o)[4]) {
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
  }
};
template <>
struct Vec<double> {
  static constexpr int N = 2;
  using V = double2;
  __device__ static void get(const V& v, double (&o)[2]) {
    o[0] = v.x;
    o[1] = v.y;
  }
};

// x widened to fp64 for the exact refinement dots (fp32, d <= 4096, large candidate sets only:
// the 32 KiB cost two column stages, which is worth it only when the exact dots dominate --
// config 5 at s = 256, want = 2560: 199k -> 230k vectors/s; at s = 64, want = 640, it loses 5-12%)
constexpr int64_t kX64MaxD = 4096, kX64MinWant = 1025;
template <typename T>
__host__ __device__ inline int64_t x64_elems(int64_t d, int64_t want) {
  return (sizeof(T) == 4 && d <= kX64MaxD && want >= kX64MinWant) ? (d < 4 ? 4 : d) : 0;
}

struct SmemLayout {
  size_t ring, x, tbuf, bars, hist, scan, misc, cand, cval, cflag, rring, x64, total;
};

template <typename T>
__host__ __device__ inline SmemLayout smem_layout(int64_t d, int stages, int stage_stride, int64_t want,
                                                  int rstride, int xbufs, int rstages) {
  SmemLayout L{};
  size_t off = 0;
  auto take = [&off](size_t bytes, size_t align) {
    off = (off + align - 1) / align * align;
    const size_t at = off;
    off += bytes;
    return at;
  };
  L.ring = take(size_t(stages) * stage_stride, 1024);
  L.x = take(size_t(xbufs) * size_t(d < 4 ? 4 : d) * sizeof(T), 16);
  L.tbuf = take(kTRing * sizeof(T), 16);
  L.bars = take((2 * kMaxStages + 2 * kTRing + 2 * kXBuf + 4 + 2 * kRStages) * sizeof(uint64_t), 8);
  L.hist = take(256 * sizeof(uint32_t), 16);
  L.scan = take(2 * 32 * sizeof(uint32_t), 16);
  L.misc = take(16 * sizeof(unsigned long long), 16);
  L.cand = take(size_t(want) * sizeof(int32_t), 16);
  L.cval = take(size_t(want) * sizeof(T), 16);
  L.cflag = take(size_t(want) * sizeof(uint8_t), 16);
  L.rring = take(size_t(rstages) * rstride, 128);  // rstride 0: refinement reads A directly
  // x widened to fp64 once per vector for the exact refinement dots (x64_elems)
  L.x64 = take(x64_elems<T>(d, want) * sizeof(double), 16);
  L.total = (off + 15) / 16 * 16;
  return L;
}

// Exclusive scan of a uint32 over the NWARPS warps of one role (named barrier
// `bar`, local warp index `lw`). *total gets the sum over the group.
template <int NWARPS>
__device__ __forceinline__ uint32_t group_scan(uint32_t v, uint32_t* scan_smem, int parity, uint32_t bar, int lw,
                                               uint32_t* total) {
  const int lane = threadIdx.x % 32;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  uint32_t* tot = scan_smem + parity * 32;
  if (lane == 31) tot[lw] = inc;
  named_bar_sync(bar, NWARPS * 32);
  uint32_t wpre = 0, all = 0;
#pragma unroll
  for (int w = 0; w < NWARPS; ++w) {
    const uint32_t t = tot[w];
    wpre += (w < lw) ? t : 0u;
    all += t;
  }
  *total = all;
  return wpre + inc - v;
}

// ------------------------------------------------ sample coefficients ----
// Fast path (d >= 128), NS samples at once: lane owns positions 128 i + 4 lane + e; the sign of
// x[pos] in s_ell is Q_s(pos) ^ parity(w & pos) (kerdock.hpp:132-152). The x loads are shared by the
// NS samples and the NS accumulation chains are independent, so one warp keeps
// NS sign-table loads and NS FADD chains in flight. ells[k] >= kb (identity
// block) are handled by the caller.
template <typename T, int NS>
__device__ __forceinline__ void coeff_fast_multi(const StreamArgs<T>& A, const T* xs, const uint32_t* wbase,
                                                 const uint32_t (&ells)[NS], int lane, T (&out)[NS]) {
#ifndef FSTG_TWC
#define FSTG_TWC 1
#endif
  constexpr int TWC = FSTG_TWC;  // sign-table words per sample in flight (1 keeps kNS = 8 spill-free)
  const int64_t rows128 = A.d / 128;
  const int tw = static_cast<int>(A.d >= 1024 ? A.d / 1024 : 1);
  // per sample: 32-bit word offset into qtrans, the Walsh base mask with the lane's
  // fix folded in, and the high Walsh bits (flip of word t = parity(whi & 8t))
  uint32_t whi[NS], base[NS], qoff[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    const uint32_t ell = static_cast<int64_t>(ells[k]) >= A.kb ? 0u : ells[k];
    const uint32_t s = ell >> A.k, w = ell & static_cast<uint32_t>(A.d - 1);
    whi[k] = w >> 7;
    const uint32_t fix = __popc(((w >> 2) & 31u) & static_cast<uint32_t>(lane)) & 1u;
    base[k] = wbase[((whi[k] & 7u) << 2) | (w & 3u)] ^ (fix ? 0xffffffffu : 0u);
    qoff[k] = s * static_cast<uint32_t>(tw) * 32u + static_cast<uint32_t>(lane);
  }
  T acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = T(0);
  // fp32: acc[k] collects the entries whose sign bit is set (one predicated FADD per entry and
  // sample: LOP3.P + @P FADD, instead of shift + sign-XOR + FADD) and tot all entries, shared by
  // the NS samples; the lane's partial is tot - 2 acc[k] (2 acc exact: one rounding)
  T tot = T(0);
  for (int t0 = 0; t0 < tw; t0 += TWC) {
    uint32_t raw[TWC][NS];
#pragma unroll
    for (int tt = 0; tt < TWC; ++tt)
#pragma unroll
      for (int k = 0; k < NS; ++k) raw[tt][k] = (t0 + tt < tw) ? __ldg(A.qtrans + qoff[k] + (t0 + tt) * 32) : 0u;
#pragma unroll
    for (int tt = 0; tt < TWC; ++tt) {
      const int t = t0 + tt;
      if (t < tw) {
        uint32_t M[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const uint32_t hiflip = __popc(whi[k] & (8u * t)) & 1u;
          M[k] = raw[tt][k] ^ base[k] ^ (hiflip ? 0xffffffffu : 0u);
        }
#pragma unroll
        for (int ip = 0; ip < 8; ++ip) {
          const int64_t i = 8 * t + ip;
          if (i < rows128) {
            const T* xp = xs + 128 * i + 4 * lane;
            if constexpr (sizeof(T) == 4) {
              const float4 xv = *reinterpret_cast<const float4*>(xp);
              const float xe[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                tot += xe[e];
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %2, %3;\n\tsetp.ne.u32 p, t, 0;\n\t"
                      "@p add.f32 %0, %0, %1;\n\t}"
                      : "+f"(acc[k])
                      : "f"(xe[e]), "r"(M[k]), "r"(1u << (4 * ip + e)));
                }
              }
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const T xvv = xp[e];
#pragma unroll
                for (int k = 0; k < NS; ++k) acc[k] += ((M[k] >> (4 * ip + e)) & 1u) ? -xvv : xvv;
              }
            }
          }
        }
      }
    }
  }
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int k = 0; k < NS; ++k) acc[k] = fmaf(-2.f, acc[k], tot);
  }
#pragma unroll
  for (int k = 0; k < NS; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    if (static_cast<int64_t>(ells[k]) >= A.kb) {
      const int64_t pos = static_cast<int64_t>(ells[k]) - A.kb;
      acc[k] = pos < A.n ? static_cast<T>(sqrt(static_cast<double>(A.d))) * xs[pos] : T(0);
    }
    out[k] = acc[k];
  }
}

// Generic warp path (any d): lane owns positions lane + 32 r.
template <typename T>
__device__ __forceinline__ T coeff_generic(const StreamArgs<T>& A, const T* xs, uint32_t ell, int lane) {
  if (static_cast<int64_t>(ell) >= A.kb) {
    const int64_t pos = static_cast<int64_t>(ell) - A.kb;
    return pos < A.n ? static_cast<T>(sqrt(static_cast<double>(A.d))) * xs[pos] : T(0);
  }
  const uint32_t s = ell >> A.k, w = ell & static_cast<uint32_t>(A.d - 1);
  const int64_t wpb = A.d >= 32 ? A.d / 32 : 1;
  T acc = T(0);
  for (int64_t pos = lane; pos < A.d; pos += 32) {
    const uint32_t qb = (__ldg(A.qplain + s * wpb + pos / 32) >> (pos % 32)) & 1u;
    const uint32_t sg = qb ^ (__popc(w & static_cast<uint32_t>(pos)) & 1u);
    const T xv = xs[pos];
    acc += sg ? -xv : xv;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Strict path: one thread, Gray-code walk in the reference's order
// (stream.hpp:89-103), separately rounded adds.
template <typename T>
__device__ __forceinline__ T coeff_strict(const StreamArgs<T>& A, const T* xs, uint32_t ell) {
  if (static_cast<int64_t>(ell) >= A.kb) {
    const int64_t pos = static_cast<int64_t>(ell) - A.kb;
    const T sqrt_d = static_cast<T>(sqrt(static_cast<double>(A.d)));
    return pos < A.n ? (sizeof(T) == 8 ? T(__dmul_rn(double(sqrt_d), double(xs[pos])))
                                       : T(__fmul_rn(float(sqrt_d), float(xs[pos]))))
                     : T(0);
  }
  const uint32_t s = ell >> A.k, wpos = ell & static_cast<uint32_t>(A.d - 1);
  uint32_t rev[16];
#pragma unroll
  for (int a = 0; a < 16; ++a) rev[a] = __ldg(A.revtab + static_cast<int64_t>(s) * 16 + a);
  T acc = T(0);
  uint32_t pos = 0;
  uint32_t sign = 0;
  const uint32_t d = static_cast<uint32_t>(A.d);
  for (uint32_t t = 0;; ++t) {
    if (static_cast<int64_t>(pos) < A.n) {
      const T xv = xs[pos];
      if constexpr (sizeof(T) == 8)
        acc = __dadd_rn(acc, sign ? -xv : xv);
      else
        acc = __fadd_rn(acc, sign ? -xv : xv);
    }
    if (t + 1 == d) break;
    const int b = __ffs(t + 1) - 1;
    sign ^= __popc(rev[b] & pos) & 1u;
    sign ^= (wpos >> b) & 1u;
    pos ^= 1u << b;
  }
  return acc;
}

// ----------------------------------------------------------- refinement ----
__device__ __forceinline__ bool screen_decide(float d, float s, int64_t nv, double eps) {
  const double k = 4.0 * static_cast<double>((nv + 63) / 64) + 6.0;
  const double bound = 1.01 * (k + 2.0) * 0x1.0p-24 * static_cast<double>(s) + 1e-30;
  return !(fabs(static_cast<double>(d)) + bound < eps);  // true: needs the exact dot (NaN included)
}
// Exact refinement dot v_i = a_i . x for fp32 rows (stream.hpp:261): every
// product a_j x_j is exact in fp64 and accumulated in fp64 (lane chunks
// q = lane + 32 i, two accumulators alternating with i, then a warp tree).
// Reads the row from global memory (L2-resident A, evict-last policy).
__device__ __forceinline__ double refine_dot_exact(const float* __restrict__ arow, const float* xs, int64_t n,
                                                   int lane, uint64_t pol_keep) {
  constexpr int kRB = 4;
  double dot = 0.0, dot2 = 0.0;
  const int64_t nv = (n + 3) / 4;
  const float4* a4 = reinterpret_cast<const float4*>(arow);
  const float4* x4 = reinterpret_cast<const float4*>(xs);
  for (int64_t q0 = lane; q0 < nv; q0 += 32 * kRB) {
    float4 av[kRB];
#pragma unroll
    for (int u = 0; u < kRB; ++u)
      av[u] = (q0 + 32 * u < nv) ? ldg_f4_policy(a4 + q0 + 32 * u, pol_keep) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < kRB; ++u) {
      if (q0 + 32 * u < nv) {
        const float4 xv4 = x4[q0 + 32 * u];
        double& acc = (u & 1) ? dot2 : dot;
        acc = fma(static_cast<double>(av[u].x), static_cast<double>(xv4.x), acc);
        acc = fma(static_cast<double>(av[u].y), static_cast<double>(xv4.y), acc);
        acc = fma(static_cast<double>(av[u].z), static_cast<double>(xv4.z), acc);
        acc = fma(static_cast<double>(av[u].w), static_cast<double>(xv4.w), acc);
      }
    }
  }
  dot += dot2;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  return dot;
}

// The same dot with x already widened to fp64 in shared memory (one conversion per
// element instead of two; identical operations and order, so identical values).
__device__ __forceinline__ double refine_dot_exact_x64(const float* __restrict__ arow, const double* x64, int64_t n,
                                                       int lane, uint64_t pol_keep) {
  constexpr int kRB = 4;
  double dot = 0.0, dot2 = 0.0;
  const int64_t nv = (n + 3) / 4;
  const float4* a4 = reinterpret_cast<const float4*>(arow);
  const double2* x2 = reinterpret_cast<const double2*>(x64);
  for (int64_t q0 = lane; q0 < nv; q0 += 32 * kRB) {
    float4 av[kRB];
#pragma unroll
    for (int u = 0; u < kRB; ++u)
      av[u] = (q0 + 32 * u < nv) ? ldg_f4_policy(a4 + q0 + 32 * u, pol_keep) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < kRB; ++u) {
      if (q0 + 32 * u < nv) {
        const double2 xa = x2[2 * (q0 + 32 * u)], xb = x2[2 * (q0 + 32 * u) + 1];
        double& acc = (u & 1) ? dot2 : dot;
        acc = fma(static_cast<double>(av[u].x), xa.x, acc);
        acc = fma(static_cast<double>(av[u].y), xa.y, acc);
        acc = fma(static_cast<double>(av[u].z), xb.x, acc);
        acc = fma(static_cast<double>(av[u].w), xb.y, acc);
      }
    }
  }
  dot += dot2;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  return dot;
}

// fp32 screening pass of the refinement: d = fl(a . x) by FFMA chains and
// S = fl(sum |a_j x_j|), in the same chunk order (depth k = 4 ceil(nv / 64) + 6
// roundings per result). Rounding-error analysis of FMA dot products gives
// |d - a.x| <= gamma_k S_true with gamma_k = k u / (1 - k u), u = 2^-24, and
// S_true <= S / (1 - gamma_k); so |a.x| < eps is PROVEN when
// |d| + 1.01 (k + 2) u S < eps (plus an absolute 1e-30 for underflow). Only
// the remaining candidates (the support and its neighbourhood; NaN / inf fall
// through as well) need the exact fp64 dot, whose value is the one reported:
// outputs are identical to refining every candidate exactly.
__device__ __forceinline__ bool refine_screen_f32(const float4* a4, const float4* x4, int64_t n, int lane,
                                                  double eps) {
  const int64_t nv = (n + 3) / 4;
  float d0 = 0.f, d1 = 0.f, s0 = 0.f, s1 = 0.f;
#pragma unroll 4
  for (int64_t q = lane; q < nv; q += 32) {
    const float4 av = a4[q], xv = x4[q];
    const bool odd = (q >> 5) & 1;
    float& d = odd ? d1 : d0;
    float& s = odd ? s1 : s0;
    d = fmaf(av.x, xv.x, d);
    d = fmaf(av.y, xv.y, d);
    d = fmaf(av.z, xv.z, d);
    d = fmaf(av.w, xv.w, d);
    s = fmaf(fabsf(av.x), fabsf(xv.x), s);
    s = fmaf(fabsf(av.y), fabsf(xv.y), s);
    s = fmaf(fabsf(av.z), fabsf(xv.z), s);
    s = fmaf(fabsf(av.w), fabsf(xv.w), s);
  }
  float d = d0 + d1, s = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return screen_decide(d, s, nv, eps);
}

// The same screening pass with the row read from global memory (rows longer
// than one ring stage, n > 4096 fp32): kRB 16-byte loads in flight per lane.
__device__ __forceinline__ bool refine_screen_f32_global(const float4* a4, const float4* x4, int64_t n, int lane,
                                                         double eps, uint64_t pol_keep) {
  constexpr int kRB = 4;
  const int64_t nv = (n + 3) / 4;
  float d0 = 0.f, d1 = 0.f, s0 = 0.f, s1 = 0.f;
  for (int64_t q0 = lane; q0 < nv; q0 += 32 * kRB) {
    float4 av[kRB];
#pragma unroll
    for (int u = 0; u < kRB; ++u)
      av[u] = (q0 + 32 * u < nv) ? ldg_f4_policy(a4 + q0 + 32 * u, pol_keep) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < kRB; ++u) {
      if (q0 + 32 * u < nv) {
        const float4 xv = x4[q0 + 32 * u];
        float& d = (u & 1) ? d1 : d0;
        float& s = (u & 1) ? s1 : s0;
        d = fmaf(av[u].x, xv.x, d);
        d = fmaf(av[u].y, xv.y, d);
        d = fmaf(av[u].z, xv.z, d);
        d = fmaf(av[u].w, xv.w, d);
        s = fmaf(fabsf(av[u].x), fabsf(xv.x), s);
        s = fmaf(fabsf(av[u].y), fabsf(xv.y), s);
        s = fmaf(fabsf(av[u].z), fabsf(xv.z), s);
        s = fmaf(fabsf(av[u].w), fabsf(xv.w), s);
      }
    }
  }
  float d = d0 + d1, s = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return screen_decide(d, s, nv, eps);
}

// Screening from the bf16 copy of A (fstg_sketch::ab, RN-rounded, 2 bytes per
// entry: half the refinement's row traffic, an L2-resident table half the size).
// With a^ = bf16(a): |a_j - a^_j| <= 2^-8 |a^_j| (unit roundoff of an 8-bit
// significand) + 2^-134 below the normal range. d = fl(a^.x) is evaluated with
// packed FFMA2 chains of depth k = ceil(nv/32) + 7 (nv = ceil(n/4) four-entry
// chunks, lane chunks q = lane + 32 i, two packed accumulators), so
// |d - a^.x| <= gamma_k sum|a^_j x_j|, and by Cauchy-Schwarz
//   |a.x| <= |d| + (gamma_k + 2^-8) |a^|_2 |x|_2 + 2^-134 |x|_1.
// |a^_i|_2 is precomputed per row (rounded up, fstg_sketch::abn); |x|_2 and
// |x|_1 per vector in fp64. |a.x| < eps is PROVEN when
//   |d| + 1.001 (1.01 (k + 2) 2^-24 + 2^-8) N_i X2 + 2^-125 X1 + 1e-30 < eps
// (2^-125 also covers subnormal a^_j flushed to zero). No second (|a| |x|)
// accumulation: one FFMA2 per two entries. Candidates it cannot rule out
// (support, eps-neighbourhood, NaN / inf) get the exact fp64 dot over the fp32
// row, so outputs are unchanged.
struct XNorms {
  double x2, x1;  // |x|_2, |x|_1 (fp64, all lanes)
};
template <typename T>
__device__ __forceinline__ XNorms warp_x_norms(const T* xs, int64_t n, int lane) {
  double s2 = 0.0, s1 = 0.0;
  for (int64_t j = lane; j < n; j += 32) {
    const double v = static_cast<double>(xs[j]);
    s2 = fma(v, v, s2);
    s1 += fabs(v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  return {sqrt(s2), s1};
}
__device__ __forceinline__ bool screen_decide_bf16(float d, float rown, const XNorms& xn, int64_t nv, double eps) {
  const double k = static_cast<double>((nv + 31) / 32) + 7.0;
  const double bound = 1.001 * (1.01 * (k + 2.0) * 0x1.0p-24 + 0x1.0p-8) * static_cast<double>(rown) * xn.x2 +
                       0x1.0p-125 * xn.x1 + 1e-30;
  return !(fabs(static_cast<double>(d)) + bound < eps);  // true: needs the exact dot (NaN included)
}
__device__ __forceinline__ float2 bf16x2_f32(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
// d += a^[4q .. 4q+3] . x[4q .. 4q+3] on two packed accumulators
__device__ __forceinline__ void bf16_chunk(uint2 aw, float4 xv, float2& p0, float2& p1) {
  p0 = __ffma2_rn(bf16x2_f32(aw.x), make_float2(xv.x, xv.y), p0);
  p1 = __ffma2_rn(bf16x2_f32(aw.y), make_float2(xv.z, xv.w), p1);
}
__device__ __forceinline__ float bf16_reduce(float2 p0, float2 p1) {
  float d = (p0.x + p0.y) + (p1.x + p1.y);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  return d;
}

// one bf16 row from the refinement ring
__device__ __forceinline__ bool refine_screen_bf16(const uint2* a4, const float4* x4, int64_t n, int lane, float rown,
                                                   const XNorms& xn, double eps) {
  const int64_t nv = (n + 3) / 4;
  float2 p0 = make_float2(0.f, 0.f), p1 = p0;
#pragma unroll 4
  for (int64_t q = lane; q < nv; q += 32) bf16_chunk(a4[q], x4[q], p0, p1);
  return screen_decide_bf16(bf16_reduce(p0, p1), rown, xn, nv, eps);
}

// two bf16 rows of one ring stage screened in one pass over x (half the shared-memory x reads)
__device__ __forceinline__ void refine_screen_bf16_pair(const uint2* a4, const uint2* b4, const float4* x4, int64_t n,
                                                        int lane, float rowa, float rowb, const XNorms& xn, double eps,
                                                        bool& ma, bool& mb) {
  const int64_t nv = (n + 3) / 4;
  float2 pa0 = make_float2(0.f, 0.f), pa1 = pa0, pb0 = pa0, pb1 = pa0;
#pragma unroll 4
  for (int64_t q = lane; q < nv; q += 32) {
    const float4 xv = x4[q];
    bf16_chunk(a4[q], xv, pa0, pa1);
    bf16_chunk(b4[q], xv, pb0, pb1);
  }
  ma = screen_decide_bf16(bf16_reduce(pa0, pa1), rowa, xn, nv, eps);
  mb = screen_decide_bf16(bf16_reduce(pb0, pb1), rowb, xn, nv, eps);
}

// the same with the bf16 row read from global memory (rows longer than one ring stage)
__device__ __forceinline__ bool refine_screen_bf16_global(const uint2* a4, const float4* x4, int64_t n, int lane,
                                                          float rown, const XNorms& xn, double eps, uint64_t pol_keep) {
  constexpr int kRB = 8;
  const int64_t nv = (n + 3) / 4;
  float2 p0 = make_float2(0.f, 0.f), p1 = p0;
  for (int64_t q0 = lane; q0 < nv; q0 += 32 * kRB) {
    uint2 aw[kRB];
#pragma unroll
    for (int u = 0; u < kRB; ++u) aw[u] = (q0 + 32 * u < nv) ? ldg_u2_policy(a4 + q0 + 32 * u, pol_keep) : make_uint2(0u, 0u);
#pragma unroll
    for (int u = 0; u < kRB; ++u)
      if (q0 + 32 * u < nv) bf16_chunk(aw[u], x4[q0 + 32 * u], p0, p1);
  }
  return screen_decide_bf16(bf16_reduce(p0, p1), rown, xn, nv, eps);
}

// --------------------------------------------------------------- kernel ----
// One persistent CTA per SM; warp roles (24 warps, 768 threads):
//   [0, 8)   consumers   : wait t_j and the column ring, acc += t_j * C[:, ell_j],
//                          per-batch means -> L2 scratch slot (lv & 1)
//   [8, 16)  coefficients: x -> smem (2 buffers), t_j -> 64-slot ring
//   [16, 23) tail        : median, radix select, candidate compaction,
//                          refinement (warp 16 issues the row copies, 17-22
//                          own the 6 ring stages), support compaction for
//                          vector lv while the consumers already stream lv + 1
//   23       producer    : bulk copies of the sampled columns (16 KiB stages)
template <typename T, bool STRICT, int NSEG, bool SPLIT>
__global__ void __launch_bounds__(kThreads, 1) stream_kernel(const StreamArgs<T> A) {
  using KT = typename KeyOf<T>::K;
  constexpr int VEC = Vec<T>::N;
  constexpr int SEG = kSegBytes / static_cast<int>(sizeof(T));  // rows per segment
  constexpr int CPS = SEG / VEC;                                  // 16-byte chunks per segment
  // NSEG == 0: small columns (m_pad <= kNC * VEC): one 16-byte chunk per consumer thread
  // and kSmallGroupFast / kSmallGroupStrict samples per consumer iteration (the per-sample handshake, not
  // bandwidth, bounds small-m configs; the ring has >= 32 stages there).
  constexpr bool SMALL = NSEG == 0;
  constexpr int NSG = SMALL ? 1 : NSEG;                          // segments held per column
  constexpr int CPT = SMALL ? 1 : CPS / kNC;                      // chunks per consumer thread per segment
  constexpr int CG = SMALL ? (STRICT ? kSmallGroupStrict : kSmallGroupFast) : 1;  // samples per consumer iteration

  extern __shared__ __align__(1024) unsigned char smem[];
  const SmemLayout Ls = smem_layout<T>(A.d, A.stages, A.stage_stride, A.want, A.rstride, A.xbufs, A.rstages);
  unsigned char* ring = smem + Ls.ring;
  T* xbuf = reinterpret_cast<T*>(smem + Ls.x);
  T* tring = reinterpret_cast<T*>(smem + Ls.tbuf);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Ls.bars);
  uint64_t* empty = full + kMaxStages;
  uint64_t* t_full = empty + kMaxStages;
  uint64_t* t_empty = t_full + kTRing;
  uint64_t* x_full = t_empty + kTRing;
  uint64_t* x_empty = x_full + kXBuf;
  uint64_t* m_full = x_empty + kXBuf;
  uint64_t* m_empty = m_full + 2;
  uint64_t* r_full = m_empty + 2;
  uint64_t* r_empty = r_full + kRStages;
  unsigned char* rring = smem + Ls.rring;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + Ls.hist);
  uint32_t* scan = reinterpret_cast<uint32_t*>(smem + Ls.scan);
  unsigned long long* misc = reinterpret_cast<unsigned long long*>(smem + Ls.misc);
  int32_t* cand = reinterpret_cast<int32_t*>(smem + Ls.cand);
  T* cval = reinterpret_cast<T*>(smem + Ls.cval);
  uint8_t* cflag = reinterpret_cast<uint8_t*>(smem + Ls.cflag);
  double* x64 = reinterpret_cast<double*>(smem + Ls.x64);
  __shared__ uint32_t wbase[32];
  __shared__ unsigned long long wait_acc[kWSites + 1];
  const long long t_start = kWaitProfile ? clock64() : 0;
  WaitProf wp{kWaitProfile && (A.debug & 8) != 0, wait_acc};
  if (kWaitProfile && threadIdx.x <= kWSites) wait_acc[threadIdx.x] = 0;

  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const int S = A.stages;
  // Work items: vectors, or (vector, batch) pairs when A.batch_split (small batches).
  constexpr bool split = SPLIT;  // (vector, batch) work items: compile-time, so the normal path pays nothing
  const int64_t items = split ? A.B * A.K : A.B;
  const int64_t NI = split ? A.J : A.N;  // samples per item
  auto item_vec = [&](int64_t w) { return split ? w / A.K : w; };
  auto item_j0 = [&](int64_t w) { return split ? (w % A.K) * A.J : int64_t(0); };
  const int64_t dx = A.d < 4 ? 4 : A.d;
  const int64_t seg_last_rows = A.m_pad - int64_t(A.nseg - 1) * SEG;
  const uint32_t stage_bytes_full = static_cast<uint32_t>((A.nseg > 1 ? SEG : A.m_pad) * sizeof(T));
  const uint32_t stage_bytes_last = static_cast<uint32_t>(seg_last_rows * sizeof(T));
  const int64_t slot_elems = (A.K + 1) * A.m_pad;  // K batch means + mu
  T* scratch = A.means + int64_t(blockIdx.x) * 2 * slot_elems;

  if (tid < S) {
    mbar_init(&full[tid], 1);
    mbar_init(&empty[tid], kNCW);
  }
  if (tid < kTRing) {
    mbar_init(&t_full[tid], 1);
    mbar_init(&t_empty[tid], kNCW);
  }
  if (tid < kXBuf) {
    mbar_init(&x_full[tid], 1);
    mbar_init(&x_empty[tid], 1);
  }
  if (tid < 2) {
    mbar_init(&m_full[tid], kNCW);
    mbar_init(&m_empty[tid], 1);
  }
  if (tid < A.rstages) {
    mbar_init(&r_full[tid], 1);
    mbar_init(&r_empty[tid], 1);
  }
  if (tid < 32) {
    // Walsh base masks: bit f (i' = f/4, e = f%4) = parity(hi3 & i') ^ parity(lo2 & e).
    const uint32_t hi3 = static_cast<uint32_t>(tid) >> 2, lo2 = static_cast<uint32_t>(tid) & 3u;
    uint32_t m = 0;
    for (int f = 0; f < 32; ++f)
      m |= static_cast<uint32_t>((__popc(hi3 & static_cast<uint32_t>(f >> 2)) ^ __popc(lo2 & static_cast<uint32_t>(f & 3))) & 1) << f;
    wbase[tid] = m;
  }
  fence_mbar_init();
  __syncthreads();

  if (warp == kWarpProd) {
    // ======================= producer warp =======================
    // P lanes issue the bulk copies in lockstep (one lane's back-to-back copies
    // serialise at ~4 TB/s chip-wide, profiles/r01_tma_issue.txt); lane l owns the
    // ring stages s = l (mod P), P | S, so every stage is refilled in order by one
    // thread and its empty-barrier parity never runs two phases ahead. Each lane
    // loads the sample index of its next copy while issuing the current one.
    int P = 1;
    for (int c = S < 32 ? S : 32; c > 1; --c)
      if (S % c == 0) {
        P = c;
        break;
      }
    if (lane < P && !(A.debug & 2) && A.means_mode != kMeansTail) {
      const uint64_t pol = policy_evict_first();
      const int nseg = A.nseg;
      int64_t w = blockIdx.x, j = 0;  // work item, sample within the item
      int sg = 0;
      auto advance = [&](int by) {
        sg += by;
        while (sg >= nseg) {
          sg -= nseg;
          if (++j == NI) {
            j = 0;
            w += gridDim.x;
          }
        }
      };
      // flat sample position v * N + j0 + j of the current copy
      auto flat = [&](int64_t ww, int64_t jj) { return item_vec(ww) * A.N + item_j0(ww) + jj; };
      advance(lane);
      uint32_t ell_next = (w < items && !A.gathered) ? __ldg(A.idx + flat(w, j)) : 0u;
      int stage = lane;
      uint32_t phase = 0, used = 0;
      while (w < items) {
        // everything for this copy is ready before the wait; the next index load and
        // the bookkeeping happen after the copy is issued (the wait ends when a
        // consumer frees the slot, so nothing else sits on the refill path)
        const int sgc = sg;
        const T* col = (A.gathered ? A.gathered + flat(w, j) * A.ldc : A.cols + static_cast<int64_t>(ell_next) * A.ldc) +
                       int64_t(sgc) * SEG;
        const uint32_t bytes = (sgc == nseg - 1) ? stage_bytes_last : stage_bytes_full;
        if (used) wp.wait(&empty[stage], phase ^ 1u, kWProdEmpty);
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(ring + size_t(stage) * A.stage_stride, col, bytes, &full[stage], pol);
        advance(P);
        if (w < items && !A.gathered) ell_next = __ldg(A.idx + flat(w, j));
        stage += P;
        if (stage >= S) {
          stage -= S;
          phase ^= 1u;
          used = 1;
        }
      }
    }
    wp.done(kWTotProd, t_start);
    return;
  }

  if (warp >= kWarpCoef && warp < kWarpTail) {
    // ======================= coefficient warps =======================
    const int cw = warp - kWarpCoef;
    const int ctid = tid - kWarpCoef * 32;  // 0 .. kCW*32-1
    uint32_t lv = 0;
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x, ++lv) {
      const int64_t v = item_vec(w);
      const uint32_t xb = lv % static_cast<uint32_t>(A.xbufs), xu = lv / static_cast<uint32_t>(A.xbufs);
      // (PARTIAL: no tail reads x; this role's own end-of-vector barrier orders the reuse)
      if (xu > 0 && A.means_mode != kMeansPartial) wp.wait(&x_empty[xb], (xu - 1) & 1u, kWCoefXEmpty);
      T* xs = xbuf + xb * dx;
      const T* xv = A.X + v * A.ldx;
      for (int64_t p = ctid; p < A.d; p += kCW * 32) xs[p] = (p < A.n) ? xv[p] : T(0);
      named_bar_sync(kBarCoef, kCW * 32);
      if (ctid == 0) mbar_arrive(&x_full[xb]);
      const uint32_t* vidx = A.idx + v * A.N + item_j0(w);
      const uint64_t g0 = uint64_t(lv) * uint64_t(NI);
      if ((A.debug & 1) || A.means_mode == kMeansTail) {
        // TAIL mode (no columns) or the column-pipeline experiment: no coefficients
      } else if constexpr (STRICT) {
        // One producing thread per ring slot (stride = kTRing): a slot's uses are
        // produced in order by the same thread, so a parity wait is never two
        // phases ahead.
        static_assert(kCW * 32 >= kTRing, "strict producers need kTRing threads");
        for (int64_t j = ctid; ctid < kTRing && j < NI; j += kTRing) {
          const uint64_t g = g0 + uint64_t(j);
          const uint32_t slot = static_cast<uint32_t>(g % kTRing), u = static_cast<uint32_t>(g / kTRing);
          const T t = coeff_strict<T>(A, xs, __ldg(vidx + j));
          if (u > 0) wp.wait(&t_empty[slot], (u - 1) & 1u, kWCoefTEmpty);
          tring[slot] = t;
          mbar_arrive(&t_full[slot]);
        }
      } else if (A.d >= 128) {
        // groups of kNS samples j = cw + kCW * (kNS * grp + k)
        uint32_t nxt[kNS];
#pragma unroll
        for (int k = 0; k < kNS; ++k) {
          const int64_t j = cw + int64_t(kCW) * k;
          nxt[k] = j < NI ? __ldg(vidx + j) : 0u;
        }
        for (int64_t j0 = cw; j0 < NI; j0 += int64_t(kCW) * kNS) {
          uint32_t ells[kNS];
          T t[kNS];
#pragma unroll
          for (int k = 0; k < kNS; ++k) {
            ells[k] = nxt[k];
            const int64_t jn = j0 + int64_t(kCW) * (kNS + k);  // prefetch the next group's indices
            nxt[k] = jn < NI ? __ldg(vidx + jn) : 0u;
          }
          coeff_fast_multi<T, kNS>(A, xs, wbase, ells, lane, t);
#pragma unroll
          for (int k = 0; k < kNS; ++k) {
            const int64_t j = j0 + int64_t(kCW) * k;
            if (j < NI) {
              const uint64_t g = g0 + uint64_t(j);
              const uint32_t slot = static_cast<uint32_t>(g % kTRing), u = static_cast<uint32_t>(g / kTRing);
              if (u > 0) wp.wait(&t_empty[slot], (u - 1) & 1u, kWCoefTEmpty);
              if (lane == 0) {
                tring[slot] = t[k];
                mbar_arrive(&t_full[slot]);
              }
            }
          }
          __syncwarp();
        }
      } else {
        for (int64_t j = cw; j < NI; j += kCW) {
          const uint64_t g = g0 + uint64_t(j);
          const uint32_t slot = static_cast<uint32_t>(g % kTRing), u = static_cast<uint32_t>(g / kTRing);
          const T t = coeff_generic<T>(A, xs, __ldg(vidx + j), lane);
          if (u > 0) wp.wait(&t_empty[slot], (u - 1) & 1u, kWCoefTEmpty);
          if (lane == 0) {
            tring[slot] = t;
            mbar_arrive(&t_full[slot]);
          }
          __syncwarp();
        }
      }
      named_bar_sync(kBarCoef, kCW * 32);
    }
    wp.done(kWTotCoef, t_start);
    return;
  }

  if (warp >= kWarpTail) {
    // ======================= tail warps =======================
    if (A.means_mode == kMeansPartial) {
      wp.done(kWTotTail, t_start);
      return;
    }
    const int ttid = tid - kWarpTail * 32, tw = warp - kWarpTail;
    const uint64_t pol_keep = policy_evict_last();
    // fp32 refinement screening (refine_screen_f32); FSTG_STREAM_DEBUG bit 16 refines every candidate exactly
    const bool screen = !(A.debug & 16);
    int parity = 0;
    uint32_t rg = 0;  // running index of refinement rows through the ring (all tail threads agree)
    uint32_t lv = 0;
    for (int64_t v = blockIdx.x; v < A.B; v += gridDim.x, ++lv) {
      const uint32_t slot = lv & 1u, su = lv >> 1, xb = lv % static_cast<uint32_t>(A.xbufs),
                     xu = lv / static_cast<uint32_t>(A.xbufs);
      T* means = A.means_mode == kMeansTail
                     ? A.means_io + v * (A.means_vstride > 0 ? A.means_vstride : (A.K + 1) * A.m_pad)
                     : scratch + slot * slot_elems;
      T* mus = means + A.K * A.m_pad;
      wp.wait(&m_full[slot], su & 1u, kWTailMFull);

      // ---- median of the K batch means (stream.hpp:126-143) ----
      for (int64_t c = ttid; int64_t(c) * VEC < A.m_pad; c += kTL) {
        const int64_t row0 = c * VEC;
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const int64_t row = row0 + e;
          T mu = T(0);
          if (row < A.m) {
            if (A.K == 1) {
              mu = means[row];
            } else if (A.K == 2) {
              const T x0 = means[row], x1 = means[A.m_pad + row];
              const T lo = x0 < x1 ? x0 : x1, hi = x0 < x1 ? x1 : x0;
              mu = T(0.5) * (lo + hi);
            } else {
              // order statistics K/2 (and K/2-1 for even K), ties by batch index
              const int64_t hK = A.K / 2;
              T up = T(0), lo = T(0);
              for (int64_t i = 0; i < A.K; ++i) {
                const T xi = means[i * A.m_pad + row];
                int64_t rank = 0;
                for (int64_t q = 0; q < A.K; ++q) {
                  const T xq = means[q * A.m_pad + row];
                  rank += (xq < xi || (xq == xi && q < i)) ? 1 : 0;
                }
                if (rank == hK) up = xi;
                if (rank == hK - 1) lo = xi;
              }
              mu = (A.K % 2 == 1) ? up : T(0.5) * (lo + up);
            }
            if (A.mu != nullptr) A.mu[v * A.m + row] = mu;
          }
          mus[row] = mu;
        }
      }
      named_bar_sync(kBarTail, kTL);
      if (ttid == 0) mbar_arrive(&m_empty[slot]);  // batch means consumed; mus stays private

      // ---- MSB radix select of the want-th largest |mu| ----
      KT prefix = 0, kmask = 0;
      int64_t remaining = A.want;
      for (int shift = KeyOf<T>::BITS - 8; shift >= 0; shift -= 8) {
        for (int b = ttid; b < 256; b += kTL) hist[b] = 0;
        named_bar_sync(kBarTail, kTL);
        for (int64_t row = ttid; row < A.m_pad + kTL; row += kTL) {
          // uniform trip count across the warp (row bound checked inside)
          if (row - ttid >= A.m_pad) break;
          const bool inr = row < A.m;
          const KT key = inr ? KeyOf<T>::key(mus[row]) : KT(0);
          const bool act = inr && ((key & kmask) == prefix);
          const uint32_t digit = static_cast<uint32_t>((key >> shift) & 0xffu);
          const uint32_t am = __ballot_sync(0xffffffffu, act);
          if (act) {
            const uint32_t peers = __match_any_sync(am, digit);
            if (lane == __ffs(peers) - 1) atomicAdd(&hist[digit], static_cast<uint32_t>(__popc(peers)));
          }
        }
        named_bar_sync(kBarTail, kTL);
        if (tw == 0) {
          uint32_t h[8], sum = 0;
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            h[b] = hist[255 - 8 * lane - b];
            sum += h[b];
          }
          uint32_t inc = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
          }
          const uint32_t exc = inc - sum;
          if (exc < static_cast<uint32_t>(remaining) && inc >= static_cast<uint32_t>(remaining)) {
            uint32_t cum = exc;
            int b = 0;
            for (; b < 8; ++b) {
              if (cum + h[b] >= static_cast<uint32_t>(remaining)) break;
              cum += h[b];
            }
            misc[0] = static_cast<unsigned long long>(255 - 8 * lane - b);
            misc[1] = static_cast<unsigned long long>(remaining - cum);
          }
        }
        named_bar_sync(kBarTail, kTL);
        const KT dg = static_cast<KT>(misc[0]);
        remaining = static_cast<int64_t>(misc[1]);
        prefix |= dg << shift;
        kmask |= static_cast<KT>(0xff) << shift;
      }
      const KT thr = prefix;
      const uint32_t quota = static_cast<uint32_t>(remaining);

      // ---- index-ordered compaction of the candidate set (sorted ascending) ----
      {
        uint32_t base_gt = 0, base_eq = 0;
        for (int64_t r0 = 0; r0 < A.m_pad; r0 += int64_t(kTL) * VEC) {
          const int64_t row0 = r0 + int64_t(ttid) * VEC;
          uint32_t ngt = 0, neq = 0;
          KT kk[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const int64_t row = row0 + e;
            kk[e] = (row < A.m) ? KeyOf<T>::key(mus[row]) : KT(0);
            if (row < A.m) {
              ngt += kk[e] > thr;
              neq += kk[e] == thr;
            }
          }
          uint32_t total;
          const uint32_t pre = group_scan<kTLW>((neq << 16) | ngt, scan, parity, kBarTail, tw, &total);
          parity ^= 1;
          uint32_t gt_before = base_gt + (pre & 0xffffu), eq_before = base_eq + (pre >> 16);
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const int64_t row = row0 + e;
            if (row < A.m) {
              if (kk[e] > thr) {
                cand[gt_before + (eq_before < quota ? eq_before : quota)] = static_cast<int32_t>(row);
                ++gt_before;
              } else if (kk[e] == thr) {
                if (eq_before < quota) cand[gt_before + eq_before] = static_cast<int32_t>(row);
                ++eq_before;
              }
            }
          }
          base_gt += total & 0xffffu;
          base_eq += total >> 16;
        }
      }
      named_bar_sync(kBarTail, kTL);

      // ---- refinement: v_i = a_i . x, fp64 accumulation (stream.hpp:259-266); fp32 rows are
      //      screened first (refine_screen_f32) and only the unresolved ones refined exactly ----
      wp.wait(&x_full[xb], xu & 1u, kWTailXFull);
      const T* xs = xbuf + xb * dx;
      if (A.debug & 4) {
        // experiment: no refinement (no A-row traffic)
        for (int64_t ci = tw * 32 + lane; ci < A.want; ci += kTLW * 32) cflag[ci] = 0;
      } else if (A.rstride > 0) {
        // Gather-GEMV staged through TMA: tail warp 0 bulk-copies the candidate
        // rows of A (L2-resident, evict-last) into a kRStages-deep ring; warp
        // 1 + st owns stage st and takes the rows whose running index g
        // satisfies g % kRStages == st, so each stage's uses stay in order on
        // one warp (mbarrier parity never aliases).
        // fp32 with the bf16 screening table: the ring holds bf16 rows, A.rrows (2) per stage so one
        // pass over x in shared memory screens both (exact dots re-read the fp32 rows from L2)
        const bool bf = sizeof(T) == 4 && A.ab != nullptr;
        const uint32_t rbytes = bf ? static_cast<uint32_t>(A.ldab * 2) : static_cast<uint32_t>(A.lda * sizeof(T));
        const uint32_t rst = static_cast<uint32_t>(A.rstages);
        const int64_t rps = bf ? A.rrows : 1;            // rows per ring stage (unit)
        const int64_t nun = (A.want + rps - 1) / rps;    // units of this vector
        if (tw == 0) {
          // lane st issues the units of stage st (one issuing thread per stage, like its consumer)
          if (lane < rst) {
            const uint32_t st = static_cast<uint32_t>(lane);
            const uint32_t first = (st + rst - rg % rst) % rst;
            for (int64_t ui = first; ui < nun; ui += rst) {
              const uint32_t g = rg + static_cast<uint32_t>(ui);
              const uint32_t u = g / rst;
              if (u > 0) wp.wait(&r_empty[st], (u - 1) & 1u, kWTailREmpty);
              const int64_t r0 = ui * rps, r1 = min(A.want, r0 + rps);
              mbar_arrive_expect_tx(&r_full[st], rbytes * static_cast<uint32_t>(r1 - r0));
              for (int64_t ci = r0; ci < r1; ++ci) {
                const void* src = bf ? static_cast<const void*>(A.ab + int64_t(cand[ci]) * A.ldab)
                                     : static_cast<const void*>(A.a + int64_t(cand[ci]) * A.lda);
                bulk_g2s(rring + size_t(st) * A.rstride + size_t(ci - r0) * rbytes, src, rbytes, &r_full[st], pol_keep);
              }
            }
          }
          __syncwarp();
        } else if (tw - 1 < static_cast<int>(rst)) {
          const uint32_t st = static_cast<uint32_t>(tw - 1);
          const uint32_t first = (st + rst - rg % rst) % rst;  // first unit with (rg + ui) % rst == st
          const XNorms xn = bf ? warp_x_norms(xs, A.n, lane) : XNorms{0.0, 0.0};
          for (int64_t ui = first; ui < nun; ui += rst) {
            const uint32_t g = rg + static_cast<uint32_t>(ui);
            const int64_t ci = ui * rps;
            wp.wait(&r_full[st], (g / rst) & 1u, kWTailRFull);
            if constexpr (sizeof(T) == 4) {
              if (bf) {
                // bf16 screening pass (refine_screen_bf16); unresolved candidates get the exact dot below
                const uint2* a0 = reinterpret_cast<const uint2*>(rring + size_t(st) * A.rstride);
                bool m0 = false, m1 = false;
                if (A.debug & 64) {
                  // experiment: row traffic without the screening arithmetic
                } else if (ci + 1 < A.want && rps == 2)
                  refine_screen_bf16_pair(a0, reinterpret_cast<const uint2*>(rring + size_t(st) * A.rstride + rbytes),
                                          reinterpret_cast<const float4*>(xs), A.n, lane, A.abn[cand[ci]],
                                          A.abn[cand[ci + 1]], xn, A.epsilon, m0, m1);
                else
                  m0 = refine_screen_bf16(a0, reinterpret_cast<const float4*>(xs), A.n, lane, A.abn[cand[ci]], xn,
                                          A.epsilon);
                __syncwarp();
                if (lane == 0) {
                  mbar_arrive(&r_empty[st]);
                  cflag[ci] = m0 ? 2 : 0;
                  if (ci + 1 < A.want && rps == 2) cflag[ci + 1] = m1 ? 2 : 0;
                }
                continue;
              }
              if (screen) {
                // fp32 screening pass; candidates it cannot rule out get the exact dot below
                const bool maybe = refine_screen_f32(reinterpret_cast<const float4*>(rring + size_t(st) * A.rstride),
                                                     reinterpret_cast<const float4*>(xs), A.n, lane, A.epsilon);
                __syncwarp();
                if (lane == 0) {
                  mbar_arrive(&r_empty[st]);
                  cflag[ci] = maybe ? 2 : 0;
                }
                continue;
              }
            }
            double dot = 0.0, dot2 = 0.0;
            if constexpr (sizeof(T) == 4) {
              const int64_t nv = (A.n + 3) / 4;
              const float4* a4 = reinterpret_cast<const float4*>(rring + size_t(st) * A.rstride);
              const float4* x4 = reinterpret_cast<const float4*>(xs);
#pragma unroll 4
              for (int64_t q = lane; q < nv; q += 32) {
                const float4 av = a4[q], xv4 = x4[q];
                double& acc = ((q >> 5) & 1) ? dot2 : dot;
                acc = fma(static_cast<double>(av.x), static_cast<double>(xv4.x), acc);
                acc = fma(static_cast<double>(av.y), static_cast<double>(xv4.y), acc);
                acc = fma(static_cast<double>(av.z), static_cast<double>(xv4.z), acc);
                acc = fma(static_cast<double>(av.w), static_cast<double>(xv4.w), acc);
              }
            } else {
              const int64_t nv = (A.n + 1) / 2;
              const double2* a2 = reinterpret_cast<const double2*>(rring + size_t(st) * A.rstride);
              const double2* x2 = reinterpret_cast<const double2*>(xs);
#pragma unroll 4
              for (int64_t q = lane; q < nv; q += 32) {
                const double2 av = a2[q], xv2 = x2[q];
                double& acc = ((q >> 5) & 1) ? dot2 : dot;
                acc = fma(av.x, xv2.x, acc);
                acc = fma(av.y, xv2.y, acc);
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&r_empty[st]);
            dot += dot2;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            if (lane == 0) {
              cval[ci] = static_cast<T>(dot);
              cflag[ci] = fabs(dot) >= A.epsilon ? 1 : 0;
            }
          }
        }
        rg += static_cast<uint32_t>(nun);
        if constexpr (sizeof(T) == 4) {
          if (screen || bf) {
            named_bar_sync(kBarTail, kTL);  // every screening flag is written
            const bool wide = x64_elems<T>(A.d, A.want) > 0;
            if (wide) {
              // x widened to fp64 once for this vector's exact dots
              for (int64_t j = ttid; j < x64_elems<T>(A.d, A.want); j += kTL) x64[j] = static_cast<double>(xs[j]);
              named_bar_sync(kBarTail, kTL);
            }
            for (int64_t ci = tw; ci < A.want; ci += kTLW) {
              if (cflag[ci] != 2) continue;  // warp-uniform
              if (A.debug & 32) {  // experiment: no exact dots
                if (lane == 0) cflag[ci] = 0;
                continue;
              }
              const float* arow = reinterpret_cast<const float*>(A.a + int64_t(cand[ci]) * A.lda);
              const double dot = wide ? refine_dot_exact_x64(arow, x64, A.n, lane, pol_keep)
                                      : refine_dot_exact(arow, reinterpret_cast<const float*>(xs), A.n, lane, pol_keep);
              if (lane == 0) {
                cval[ci] = static_cast<T>(dot);
                cflag[ci] = fabs(dot) >= A.epsilon ? 1 : 0;
              }
            }
          }
        }
      } else {
        // rows longer than one stage: direct 16-byte loads from L2
        const bool bf = sizeof(T) == 4 && A.ab != nullptr;
        const XNorms xn = bf ? warp_x_norms(xs, A.n, lane) : XNorms{0.0, 0.0};
        for (int64_t ci = tw; ci < A.want; ci += kTLW) {
          const int64_t row = cand[ci];
          const T* arow = A.a + row * A.lda;
          double dot = 0.0, dot2 = 0.0;
          if constexpr (sizeof(T) == 4) {
            const bool maybe =
                bf ? refine_screen_bf16_global(reinterpret_cast<const uint2*>(A.ab + row * A.ldab),
                                               reinterpret_cast<const float4*>(xs), A.n, lane, A.abn[row], xn,
                                               A.epsilon, pol_keep)
                   : (!screen || refine_screen_f32_global(reinterpret_cast<const float4*>(arow),
                                                          reinterpret_cast<const float4*>(xs), A.n, lane, A.epsilon,
                                                          pol_keep));
            if (!maybe) {
              if (lane == 0) cflag[ci] = 0;  // proven |a_i . x| < eps
              continue;
            }
            dot = refine_dot_exact(arow, xs, A.n, lane, pol_keep);
          } else {
            constexpr int kRB = 4;
            const int64_t nv = (A.n + 1) / 2;
            const double2* a2 = reinterpret_cast<const double2*>(arow);
            const double2* x2 = reinterpret_cast<const double2*>(xs);
            for (int64_t q0 = lane; q0 < nv; q0 += 32 * kRB) {
              double2 av[kRB];
#pragma unroll
              for (int u = 0; u < kRB; ++u)
                av[u] = (q0 + 32 * u < nv) ? ldg_d2_policy(a2 + q0 + 32 * u, pol_keep) : make_double2(0.0, 0.0);
#pragma unroll
              for (int u = 0; u < kRB; ++u) {
                if (q0 + 32 * u < nv) {
                  const double2 xv2 = x2[q0 + 32 * u];
                  double& acc = (u & 1) ? dot2 : dot;
                  acc = fma(av[u].x, xv2.x, acc);
                  acc = fma(av[u].y, xv2.y, acc);
                }
              }
            }
            dot += dot2;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
          }
          if (lane == 0) {
            cval[ci] = static_cast<T>(dot);
            cflag[ci] = fabs(dot) >= A.epsilon ? 1 : 0;
          }
        }
      }
      named_bar_sync(kBarTail, kTL);
      if (ttid == 0) mbar_arrive(&x_empty[xb]);

      // ---- ordered compaction of the support ----
      uint32_t out_base = 0;
      for (int64_t c0 = 0; c0 < A.want; c0 += kTL) {
        const int64_t ci = c0 + ttid;
        const uint32_t f = (ci < A.want) ? cflag[ci] : 0u;
        uint32_t total;
        const uint32_t pre = group_scan<kTLW>(f, scan, parity, kBarTail, tw, &total);
        parity ^= 1;
        if (f) {
          const int64_t o = v * A.want + out_base + pre;
          A.support[o] = cand[ci];
          A.values[o] = cval[ci];
        }
        if (A.cands != nullptr && ci < A.want) A.cands[v * A.want + ci] = cand[ci];
        out_base += total;
      }
      if (ttid == 0) A.counts[v] = static_cast<int32_t>(out_base);
      named_bar_sync(kBarTail, kTL);  // cand/cval/cflag reuse by the next vector
    }
    wp.done(kWTotTail, t_start);
    return;
  }

  // ======================= consumer warps =======================
  int stage = 0;
  uint32_t phase = 0;
  uint32_t lv = 0;
  for (int64_t w = blockIdx.x; w < items; w += gridDim.x, ++lv) {
    const int64_t v = item_vec(w);
    const uint32_t slot = lv & 1u, su = lv >> 1;
    if (A.means_mode == kMeansTail) {  // means come from means_io: only the slot handshake
      if (su > 0) wp.wait(&m_empty[slot], (su - 1) & 1u, kWConsMEmpty);
      __syncwarp();
      if (lane == 0) mbar_arrive(&m_full[slot]);
      continue;
    }
    const bool partial = A.means_mode == kMeansPartial;
    // PARTIAL: rows [row0, row0 + m) of vector v's K batch means in means_io
    const int64_t vstride = A.means_vstride > 0 ? A.means_vstride : (A.K + 1) * A.m_io;
    T* means = partial ? A.means_io + v * vstride + A.row0 : scratch + slot * slot_elems;
    const int64_t bstride = partial ? A.m_io : A.m_pad;
    const int64_t rows_out = partial ? A.m : A.m_pad;
    const uint64_t g0 = uint64_t(lv) * uint64_t(NI);

    T acc[NSG][CPT][VEC];
#pragma unroll
    for (int sg = 0; sg < NSG; ++sg)
#pragma unroll
      for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[sg][c][e] = T(0);

    auto accumulate = [&](T& a, T t, T x) {
      if constexpr (STRICT) {
        if constexpr (sizeof(T) == 8)
          a = __dadd_rn(a, __dmul_rn(t, x));
        else
          a = __fadd_rn(a, __fmul_rn(t, x));
      } else {
        a = fma(t, x, a);
      }
    };
    int64_t jb = 0, b = split ? w % A.K : 0;  // position inside the batch, batch index
    const bool cons_fast = (A.debug & 3) == 0 && seg_last_rows == SEG;
    uint32_t tslot = static_cast<uint32_t>(g0 % kTRing), tphase = static_cast<uint32_t>((g0 / kTRing) & 1);
    bool item_done = false;
    if constexpr (NSEG == 1 && !SMALL) {
      if (cons_fast && A.J < (int64_t(1) << 30)) {
        // Full-height single-segment columns (config 3): a tight per-batch sample loop with
        // 32-bit counters, the batch end outside it. Per sample: the coefficient and column
        // waits, the loads, the stage and the coefficient slot released BEFORE the FMAs use the
        // loaded values (mbarrier.arrive orders the loads), then the updates in j order.
        const int J = static_cast<int>(A.J), nb = static_cast<int>(NI / A.J);
        const T Jt = static_cast<T>(A.J);
        for (int bb = 0; bb < nb; ++bb) {
          for (int jj = 0; jj < J; ++jj) {
            wp.wait(&t_full[tslot], tphase, kWConsT);
            const T t = tring[tslot];
            wp.wait(&full[stage], phase, kWConsCol);
            const typename Vec<T>::V* src =
                reinterpret_cast<const typename Vec<T>::V*>(ring + size_t(stage) * A.stage_stride);
            T vv[CPT][VEC];
#pragma unroll
            for (int c = 0; c < CPT; ++c) Vec<T>::get(src[tid + c * kNC], vv[c]);
            __syncwarp();
            if (lane == 0) {
              mbar_arrive(&empty[stage]);
              mbar_arrive(&t_empty[tslot]);
            }
#pragma unroll
            for (int c = 0; c < CPT; ++c)
#pragma unroll
              for (int e = 0; e < VEC; ++e) accumulate(acc[0][c][e], t, vv[c][e]);
            if (++stage == S) {
              stage = 0;
              phase ^= 1u;
            }
            tslot = (tslot + 1) & static_cast<uint32_t>(kTRing - 1);
            tphase ^= tslot == 0 ? 1u : 0u;
          }
          // batch b complete: mean = sum / J (IEEE division, stream.hpp:237)
          if (b == 0 && su > 0 && !partial) wp.wait(&m_empty[slot], (su - 1) & 1u, kWConsMEmpty);
          T* mb = means + b * bstride;
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            const int64_t row0 = int64_t(tid + c * kNC) * VEC;
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              if (row0 + e < rows_out) mb[row0 + e] = acc[0][c][e] / Jt;
              acc[0][c][e] = T(0);
            }
          }
          ++b;
        }
        item_done = true;
      }
    }
    for (int64_t j = 0; j < NI && !item_done;) {
      bool grouped = false;
      if constexpr (CG > 1) {
        if (jb + CG <= A.J && !(A.debug & 3)) {
          // CG samples of the same batch: all waits, all loads, then the updates in j
          // order (per element the same sequence as one sample at a time)
          uint32_t ts[CG], tp[CG], ph[CG];
          int st[CG];
#pragma unroll
          for (int g = 0; g < CG; ++g) {
            ts[g] = tslot;
            tp[g] = tphase;
            if (++tslot == kTRing) {
              tslot = 0;
              tphase ^= 1u;
            }
            st[g] = stage;
            ph[g] = phase;
            if (++stage == S) {
              stage = 0;
              phase ^= 1u;
            }
          }
          T tg[CG];
#pragma unroll
          for (int g = 0; g < CG; ++g) {
            wp.wait(&t_full[ts[g]], tp[g], kWConsT);
            tg[g] = tring[ts[g]];
          }
          T vv[CG][VEC];
          const bool have = int64_t(tid) * VEC < seg_last_rows;
#pragma unroll
          for (int g = 0; g < CG; ++g) {
            wp.wait(&full[st[g]], ph[g], kWConsCol);
            if (have)
              Vec<T>::get(reinterpret_cast<const typename Vec<T>::V*>(ring + size_t(st[g]) * A.stage_stride)[tid], vv[g]);
          }
          if (have) {
#pragma unroll
            for (int g = 0; g < CG; ++g)
#pragma unroll
              for (int e = 0; e < VEC; ++e) accumulate(acc[0][0][e], tg[g], vv[g][e]);
          }
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int g = 0; g < CG; ++g) {
              mbar_arrive(&empty[st[g]]);
              mbar_arrive(&t_empty[ts[g]]);
            }
          }
          j += CG;
          jb += CG - 1;  // + 1 below
          grouped = true;
        }
      }
      if constexpr (NSEG == 1 && !SMALL) {
        if (!grouped && cons_fast) {
          // one full-height segment per sample, every chunk in range (config 3): the loads first,
          // the stage and the coefficient slot released before the FMAs use the loaded values
          wp.wait(&t_full[tslot], tphase, kWConsT);
          const T t = tring[tslot];
          wp.wait(&full[stage], phase, kWConsCol);
          const typename Vec<T>::V* src =
              reinterpret_cast<const typename Vec<T>::V*>(ring + size_t(stage) * A.stage_stride);
          T vv[CPT][VEC];
#pragma unroll
          for (int c = 0; c < CPT; ++c) Vec<T>::get(src[tid + c * kNC], vv[c]);
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&empty[stage]);
            mbar_arrive(&t_empty[tslot]);
          }
#pragma unroll
          for (int c = 0; c < CPT; ++c)
#pragma unroll
            for (int e = 0; e < VEC; ++e) accumulate(acc[0][c][e], t, vv[c][e]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
          if (++tslot == kTRing) {
            tslot = 0;
            tphase ^= 1u;
          }
          ++j;
          grouped = true;
        }
      }
      if (!grouped) {
        T t = T(1);
        if (!(A.debug & 1)) {
          wp.wait(&t_full[tslot], tphase, kWConsT);
          t = tring[tslot];
        }
#pragma unroll
        for (int sg = 0; sg < NSG; ++sg) {
          if (sg < A.nseg && !(A.debug & 2)) {
            wp.wait(&full[stage], phase, kWConsCol);
            const typename Vec<T>::V* src =
                reinterpret_cast<const typename Vec<T>::V*>(ring + size_t(stage) * A.stage_stride);
            const int64_t rows_here = (sg == A.nseg - 1) ? seg_last_rows : SEG;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
              const int chunk = tid + c * kNC;
              if (int64_t(chunk) * VEC < rows_here) {
                T vv[VEC];
                Vec<T>::get(src[chunk], vv);
#pragma unroll
                for (int e = 0; e < VEC; ++e) accumulate(acc[sg][c][e], t, vv[e]);
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == S) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
        if (lane == 0 && !(A.debug & 1)) mbar_arrive(&t_empty[tslot]);
        if (++tslot == kTRing) {
          tslot = 0;
          tphase ^= 1u;
        }
        ++j;
      }
      if (++jb == A.J) {
        // batch b complete: mean = sum / J (IEEE division, stream.hpp:237)
        if (b == 0 && su > 0 && !partial) wp.wait(&m_empty[slot], (su - 1) & 1u, kWConsMEmpty);
        T* mb = means + b * bstride;
        const T Jt = static_cast<T>(A.J);
#pragma unroll
        for (int sg = 0; sg < NSG; ++sg)
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            const int64_t row0 = int64_t(sg) * SEG + int64_t(tid + c * kNC) * VEC;
            if (sg < A.nseg && row0 < A.m_pad) {
#pragma unroll
              for (int e = 0; e < VEC; ++e) {
                if (row0 + e < rows_out) mb[row0 + e] = acc[sg][c][e] / Jt;
                acc[sg][c][e] = T(0);
              }
            }
          }
        jb = 0;
        ++b;
      }
    }
    __syncwarp();
    if (lane == 0 && !partial) mbar_arrive(&m_full[slot]);
  }
  wp.done(kWTotCons, t_start);
}

// Experiment readout for FSTG_STREAM_DEBUG bit 8 (reset after reading).
void stream_wait_profile(unsigned long long* out, int count) {
  unsigned long long h[kWSites] = {};
  cudaMemcpyFromSymbol(h, g_wait_cycles, sizeof(h));
  const unsigned long long z[kWSites] = {};
  cudaMemcpyToSymbol(g_wait_cycles, z, sizeof(z));
  for (int i = 0; i < count && i < kWSites; ++i) out[i] = h[i];
}

// ------------------------------------------------------------- launching --
template <typename T>
int stream_grid_size(StreamArgs<T>& args, bool strict, int64_t B, size_t* smem_bytes, int* stages,
                     int* stage_stride, int* rstride_out, int* xbufs_out) {
  const int64_t stage_bytes = (args.m_pad * int64_t(sizeof(T)) < kSegBytes) ? args.m_pad * int64_t(sizeof(T)) : kSegBytes;
  const int stride = static_cast<int>((stage_bytes + 127) / 128 * 128);
  // the refinement ring holds bf16 screening rows when the sketch has them (fp32), two per stage
  // when they fit (one pass over x screens both)
  const bool bf = sizeof(T) == 4 && args.ab != nullptr;
  const int64_t row_bytes = bf ? args.ldab * 2 : args.lda * int64_t(sizeof(T));
  args.rrows = (bf && 2 * row_bytes <= kSegBytes) ? kRRowsBf16 : 1;
  if (const char* e = std::getenv("FSTG_RROWS")) args.rrows = bf && 2 * row_bytes <= kSegBytes ? std::max(1, std::min(2, std::atoi(e))) : 1;  // experiments
  const int64_t unit_bytes = row_bytes * args.rrows;
  const int rstride = unit_bytes <= kSegBytes ? static_cast<int>((unit_bytes + 127) / 128 * 128) : 0;
  *rstride_out = rstride;
  int xbufs = kXBufUse;
  if (const char* e = std::getenv("FSTG_XBUFS")) xbufs = std::max(1, std::min(kXBuf, std::atoi(e)));  // experiments
  *xbufs_out = xbufs;
  int rst = (args.want <= kRSmallWant && kRStages > 1) ? kRStages - 1 : kRStages;
  if (const char* e = std::getenv("FSTG_RSTAGES_RT")) rst = std::max(1, std::min(kRStages, std::atoi(e)));  // experiments
  args.rstages = rst;
  const SmemLayout L0 = smem_layout<T>(args.d, 0, stride, args.want, rstride, xbufs, rst);
  int S = static_cast<int>((kSmemBudget - static_cast<int64_t>(L0.total) - 1024) / stride);
  // ~64 KiB in flight per SM is enough (profiles/r01_stream_stages.txt: 3-5 x 16 KiB stages beat 10)
  S = std::min(S, std::max(4, static_cast<int>(kInflightBytes / stride)));
  if (const char* e = std::getenv("FSTG_STREAM_STAGES")) S = std::min(S, std::max(2, std::atoi(e)));  // experiments
  if (S > kMaxStages) S = kMaxStages;
  if (S < 2) S = 2;
  const SmemLayout L = smem_layout<T>(args.d, S, stride, args.want, rstride, xbufs, rst);
  *smem_bytes = L.total;
  *stages = S;
  *stage_stride = stride;
  (void)strict;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = sms;
  if (grid > B) grid = B;
  if (grid < 1) grid = 1;
  return static_cast<int>(grid);
}

template <typename T>
int64_t stream_scratch_elems(const StreamArgs<T>& args, int grid) {
  return int64_t(grid) * 2 * (args.K + 1) * args.m_pad;
}

template <typename T, bool STRICT, int NSEG>
static cudaError_t launch_one(const StreamArgs<T>& args, int grid, size_t smem, cudaStream_t st) {
  auto kern = args.batch_split ? stream_kernel<T, STRICT, NSEG, true> : stream_kernel<T, STRICT, NSEG, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, st>>>(args);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_stream(const StreamArgs<T>& args, bool strict, int grid, cudaStream_t st) {
  const SmemLayout L = smem_layout<T>(args.d, args.stages, args.stage_stride, args.want, args.rstride, args.xbufs,
                                      args.rstages);
  if (L.total > static_cast<size_t>(kSmemBudget)) return cudaErrorInvalidConfiguration;
  if (args.nseg <= 1 && args.m_pad <= int64_t(kNC) * (16 / int64_t(sizeof(T))) &&
      args.stages >= 4 * (strict ? kSmallGroupStrict : kSmallGroupFast)) {
    return strict ? launch_one<T, true, 0>(args, grid, L.total, st) : launch_one<T, false, 0>(args, grid, L.total, st);
  }
  if (args.nseg <= 1) {
    return strict ? launch_one<T, true, 1>(args, grid, L.total, st) : launch_one<T, false, 1>(args, grid, L.total, st);
  }
  if (args.nseg <= 4) {
    return strict ? launch_one<T, true, 4>(args, grid, L.total, st) : launch_one<T, false, 4>(args, grid, L.total, st);
  }
  return cudaErrorNotSupported;
}

template cudaError_t launch_stream<float>(const StreamArgs<float>&, bool, int, cudaStream_t);
template cudaError_t launch_stream<double>(const StreamArgs<double>&, bool, int, cudaStream_t);
template int stream_grid_size<float>(StreamArgs<float>&, bool, int64_t, size_t*, int*, int*, int*, int*);
template int stream_grid_size<double>(StreamArgs<double>&, bool, int64_t, size_t*, int*, int*, int*, int*);
template int64_t stream_scratch_elems<float>(const StreamArgs<float>&, int);
template int64_t stream_scratch_elems<double>(const StreamArgs<double>&, int);

}  // namespace fstg
