// Design verifiers on the GPU (reference kerdock.hpp:198-317, cli.hpp:45-60).
//
// Every entry of a unit design vector is +-2^(-k/2) (Kerdock) or 0/1
// (identity), so every inner product is F/d with F an integer, and the
// reference's Gram-matrix checks reduce to exact integer statistics:
//   * Kerdock bases s, s': <u_{s,w}, u_{s',w'}> = F[w ^ w'] / d with
//     F = WHT((-1)^(Q_s + Q_s')) — one d-point integer FWHT per basis pair
//     yields all d^2 entries of the cross Gram (s == s': the within-basis Gram).
//   * Kerdock vs identity: +-2^(-k/2) by construction (|F| = 2^(k/2)).
// pair_fwht_kernel runs the FWHT per basis pair from the same sign-bit tables
// (qplain) the preprocessing kernels use and accumulates, exactly, max |F - d
// delta| (within), min/max F^2 (cross) and the sums of F^2 and F^4 (design
// moments); moment_samples_kernel evaluates F for sampled column pairs (the
// reference's k > 6 Monte Carlo estimate); kerdock_rank_kernel counts basis
// pairs whose matrix sum is rank-deficient (cli.hpp:52-56).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace fstg {

namespace {

using u128 = unsigned __int128;

__device__ __forceinline__ void add_u128(unsigned long long* dst, u128 v) {
  const unsigned long long lo = static_cast<unsigned long long>(v), hi = static_cast<unsigned long long>(v >> 64);
  const unsigned long long old = atomicAdd(dst, lo);
  atomicAdd(dst + 1, hi + ((old + lo) < old ? 1ull : 0ull));
}

// Upper-triangle pair p -> (b, b2), b <= b2 < nk (diag = true) or b < b2 (diag = false).
__device__ __forceinline__ void decode_pair(int64_t p, int64_t nk, bool diag, int64_t& b, int64_t& b2) {
  const int64_t rowlen0 = diag ? nk : nk - 1;
  auto start = [&](int64_t r) { return r * rowlen0 - r * (r - 1) / 2; };
  const double t = 2.0 * double(rowlen0) + 1.0;
  int64_t r = static_cast<int64_t>((t - sqrt(t * t - 8.0 * double(p))) / 2.0);
  if (r < 0) r = 0;
  while (r > 0 && start(r) > p) --r;
  while (start(r + 1) <= p) ++r;
  b = r;
  b2 = r + (p - start(r)) + (diag ? 0 : 1);
}

template <int KB>
struct PairCfg {
  static constexpr int D = 1 << KB;
  static constexpr int NT = D < 256 ? D : 256;
  static constexpr int E = D / NT;
  static constexpr int WPB = D >= 32 ? D / 32 : 1;
};

// pairs: explicit (pb[i], pb2[i]) list, or (pb == nullptr) the upper triangle
// including the diagonal. acc[0..7] = u128 sums {F^2 within, F^4 within,
// F^2 cross, F^4 cross}; stats[0] = max |F - d delta| within, [1] = min F^2
// cross, [2] = max F^2 cross.
template <int KB>
__global__ void __launch_bounds__(PairCfg<KB>::NT) pair_fwht_kernel(const uint32_t* __restrict__ qplain, int64_t nk,
                                                                   int64_t npairs, const int32_t* __restrict__ pb,
                                                                   const int32_t* __restrict__ pb2,
                                                                   unsigned long long* acc, int* stats) {
  using C = PairCfg<KB>;
  constexpr int D = C::D, NT = C::NT, E = C::E, WPB = C::WPB;
  extern __shared__ __align__(16) int f[];
  const int t = threadIdx.x;
  u128 x2w = 0, x4w = 0, x2c = 0, x4c = 0;
  int bad = 0, f2min = INT32_MAX, f2max = 0;
  for (int64_t p = blockIdx.x; p < npairs; p += gridDim.x) {
    int64_t b, b2;
    if (pb != nullptr) {
      b = pb[p];
      b2 = pb2[p];
    } else {
      decode_pair(p, nk, true, b, b2);
    }
    const uint32_t* qa = qplain + b * WPB;
    const uint32_t* qb = qplain + b2 * WPB;
    int v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int pos = t * E + e;
      const uint32_t w = __ldg(qa + (pos >> 5)) ^ __ldg(qb + (pos >> 5));
      v[e] = ((w >> (pos & 31)) & 1u) ? -1 : 1;
    }
    // stages h < E in registers, then h >= E through shared memory (fwht.hpp:20-29 order)
#pragma unroll
    for (int h = 1; h < E; h <<= 1)
#pragma unroll
      for (int i = 0; i < E; ++i)
        if ((i & h) == 0) {
          const int x = v[i], y = v[i + h];
          v[i] = x + y;
          v[i + h] = x - y;
        }
#pragma unroll
    for (int e = 0; e < E; ++e) f[t * E + e] = v[e];
    __syncthreads();
    for (int h = E; h < D; h <<= 1) {
      for (int bt = t; bt < D / 2; bt += NT) {
        const int i = (bt / h) * 2 * h + (bt % h);
        const int x = f[i], y = f[i + h];
        f[i] = x + y;
        f[i + h] = x - y;
      }
      __syncthreads();
    }
    u128 s2 = 0, s4 = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int u = t * E + e;
      const int F = f[u];
      const unsigned long long F2 = static_cast<unsigned long long>(static_cast<long long>(F) * F);
      s2 += F2;
      s4 += static_cast<u128>(F2) * F2;
      if (b == b2) {
        const int dev = abs(F - (u == 0 ? D : 0));
        bad = max(bad, dev);
      } else {
        f2min = min(f2min, static_cast<int>(F2 > INT32_MAX ? INT32_MAX : F2));
        f2max = max(f2max, static_cast<int>(F2 > INT32_MAX ? INT32_MAX : F2));
      }
    }
    if (b == b2) {
      x2w += s2;
      x4w += s4;
    } else {
      x2c += s2;
      x4c += s4;
    }
    __syncthreads();  // f is rewritten by the next pair
  }
  add_u128(acc + 0, x2w);
  add_u128(acc + 2, x4w);
  add_u128(acc + 4, x2c);
  add_u128(acc + 6, x4c);
  atomicMax(stats + 0, bad);
  atomicMin(stats + 1, f2min);
  atomicMax(stats + 2, f2max);
}

// F = d <u_a, u_b> for sampled column pairs (kerdock.hpp:305-312); acc[0..3] =
// u128 sums of F^2 and F^4.
__global__ void moment_samples_kernel(const uint32_t* __restrict__ qplain, int k, const int64_t* __restrict__ ia,
                                      const int64_t* __restrict__ ib, int64_t count, unsigned long long* acc) {
  const int64_t d = int64_t(1) << k, nk = d / 2;
  const int wpb = d >= 32 ? static_cast<int>(d / 32) : 1;
  const uint32_t valid = d >= 32 ? 0xffffffffu : ((1u << d) - 1u);
  constexpr uint32_t kWalsh[5] = {0xAAAAAAAAu, 0xCCCCCCCCu, 0xF0F0F0F0u, 0xFF00FF00u, 0xFFFF0000u};
  u128 x2 = 0, x4 = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t a = ia[i], b = ib[i];
    const bool ida = a >= nk * d, idb = b >= nk * d;
    int64_t F;
    if (ida && idb) {
      F = (a == b) ? d : 0;
    } else if (ida || idb) {
      F = int64_t(1) << (k / 2);  // +-2^(k/2): entry of a Kerdock vector times a unit vector, times d
    } else {
      const uint32_t* qa = qplain + (a / d) * wpb;
      const uint32_t* qb = qplain + (b / d) * wpb;
      const uint32_t x = static_cast<uint32_t>((a % d) ^ (b % d));
      uint32_t low = 0;
#pragma unroll
      for (int c = 0; c < 5; ++c)
        if ((x >> c) & 1u) low ^= kWalsh[c];
      int64_t neg = 0;
      for (int w = 0; w < wpb; ++w) {
        const uint32_t hi = (__popc(x & (static_cast<uint32_t>(w) << 5)) & 1) ? 0xffffffffu : 0u;
        neg += __popc((__ldg(qa + w) ^ __ldg(qb + w) ^ low ^ hi) & valid);
      }
      F = d - 2 * neg;
    }
    const unsigned long long F2 = static_cast<unsigned long long>(F * F);
    x2 += F2;
    x4 += static_cast<u128>(F2) * F2;
  }
  add_u128(acc + 0, x2);
  add_u128(acc + 2, x4);
}

// rows: nk x k words (bit c of row r = M_{r,c}); counts pairs a < b with
// rank(M_a + M_b) < k (gf2.hpp:148-172 rank; cli.hpp:52-56).
template <int KB>
__global__ void kerdock_rank_kernel(const uint32_t* __restrict__ rows, int64_t nk, unsigned long long* bad) {
  const int64_t npairs = nk * (nk - 1) / 2;
  unsigned long long local = 0;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < npairs; p += int64_t(gridDim.x) * blockDim.x) {
    int64_t a, b;
    decode_pair(p, nk, false, a, b);
    uint32_t basis[KB];
#pragma unroll
    for (int i = 0; i < KB; ++i) basis[i] = 0;
    int rank = 0;
#pragma unroll
    for (int r = 0; r < KB; ++r) {
      uint32_t v = __ldg(rows + a * KB + r) ^ __ldg(rows + b * KB + r);
#pragma unroll
      for (int bit = KB - 1; bit >= 0; --bit) {
        if ((v >> bit) & 1u) {
          if (basis[bit]) {
            v ^= basis[bit];
          } else {
            basis[bit] = v;
            v = 0;
            ++rank;
          }
        }
      }
    }
    if (rank != KB) ++local;
  }
  if (local) atomicAdd(bad, local);
}

template <int KB>
cudaError_t launch_pairs_k(const uint32_t* qplain, int64_t nk, int64_t npairs, const int32_t* pb, const int32_t* pb2,
                           unsigned long long* acc, int* stats, cudaStream_t st) {
  using C = PairCfg<KB>;
  const size_t smem = size_t(C::D) * sizeof(int);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(pair_fwht_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t grid = npairs < 148 * 16 ? npairs : 148 * 16;
  if (grid <= 0) return cudaSuccess;
  pair_fwht_kernel<KB><<<static_cast<unsigned>(grid), C::NT, smem, st>>>(qplain, nk, npairs, pb, pb2, acc, stats);
  return cudaGetLastError();
}

template <int KB>
cudaError_t launch_rank_k(const uint32_t* rows, int64_t nk, unsigned long long* bad, cudaStream_t st) {
  const int64_t npairs = nk * (nk - 1) / 2;
  if (npairs <= 0) return cudaSuccess;
  const int64_t blocks = (npairs + 255) / 256 < 148 * 32 ? (npairs + 255) / 256 : 148 * 32;
  kerdock_rank_kernel<KB><<<static_cast<unsigned>(blocks), 256, 0, st>>>(rows, nk, bad);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_verify_pairs(int k, const uint32_t* qplain, int64_t nk, int64_t npairs, const int32_t* pb,
                                const int32_t* pb2, unsigned long long* acc, int* stats, cudaStream_t st) {
  switch (k) {
    case 2: return launch_pairs_k<2>(qplain, nk, npairs, pb, pb2, acc, stats, st);
    case 4: return launch_pairs_k<4>(qplain, nk, npairs, pb, pb2, acc, stats, st);
    case 6: return launch_pairs_k<6>(qplain, nk, npairs, pb, pb2, acc, stats, st);
    case 8: return launch_pairs_k<8>(qplain, nk, npairs, pb, pb2, acc, stats, st);
    case 10: return launch_pairs_k<10>(qplain, nk, npairs, pb, pb2, acc, stats, st);
    case 12: return launch_pairs_k<12>(qplain, nk, npairs, pb, pb2, acc, stats, st);
    case 14: return launch_pairs_k<14>(qplain, nk, npairs, pb, pb2, acc, stats, st);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t launch_verify_samples(int k, const uint32_t* qplain, const int64_t* ia, const int64_t* ib, int64_t count,
                                  unsigned long long* acc, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int64_t blocks = (count + 255) / 256 < 148 * 16 ? (count + 255) / 256 : 148 * 16;
  moment_samples_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(qplain, k, ia, ib, count, acc);
  return cudaGetLastError();
}

cudaError_t launch_verify_ranks(int k, const uint32_t* rows, int64_t nk, unsigned long long* bad, cudaStream_t st) {
  switch (k) {
    case 2: return launch_rank_k<2>(rows, nk, bad, st);
    case 4: return launch_rank_k<4>(rows, nk, bad, st);
    case 6: return launch_rank_k<6>(rows, nk, bad, st);
    case 8: return launch_rank_k<8>(rows, nk, bad, st);
    case 10: return launch_rank_k<10>(rows, nk, bad, st);
    case 12: return launch_rank_k<12>(rows, nk, bad, st);
    case 14: return launch_rank_k<14>(rows, nk, bad, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace fstg
