// Small public helpers of the reference's stream / design API on the GPU
// (stream.hpp:86-162, kerdock.hpp:156-167). They are not on the throughput path;
// they complete the drop-in surface the reference's tests and harness call.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace fstg {

namespace {

// stream.hpp:89-103: s_ell^T x for a Kerdock index by the reference's Gray-code
// walk (position order and sign updates identical, fp64, one thread: bit-exact).
__global__ void inner_product_kernel(const double* __restrict__ x, int64_t n, int64_t d,
                                     const uint32_t* __restrict__ rev, uint64_t wpos, double* out) {
  double acc = 0;
  uint64_t pos = 0;
  int sign = 0;
  for (uint64_t t = 0;; ++t) {
    if (static_cast<int64_t>(pos) < n) acc += sign ? -x[pos] : x[pos];
    if (t + 1 == static_cast<uint64_t>(d)) break;
    const int b = __ffsll(static_cast<long long>(t + 1)) - 1;
    sign ^= __popcll(static_cast<uint64_t>(rev[b]) & pos) & 1;
    sign ^= static_cast<int>((wpos >> b) & 1u);
    pos ^= uint64_t{1} << b;
  }
  *out = acc;
}

// stream.hpp:126-155: per row, K batch means of J columns each (sequential sum in
// column order, then / J), then the median (odd K: order statistic K/2; even K:
// 0.5 * (max of the lower half + element K/2)). Samples m x N, column j at j * m.
__global__ void median_of_means_kernel(const double* __restrict__ samples, int64_t m, int64_t J, int64_t K,
                                       double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t hK = K / 2;
    double up = 0, lo = 0;
    // order statistics by rank with ties broken by batch index (nth_element semantics on values)
    for (int64_t b = 0; b < K; ++b) {
      double sb = 0;
      for (int64_t j = 0; j < J; ++j) sb += samples[(b * J + j) * m + i];
      const double mb = sb / static_cast<double>(J);
      int64_t rank = 0;
      for (int64_t q = 0; q < K; ++q) {
        if (q == b) continue;
        double sq = 0;
        for (int64_t j = 0; j < J; ++j) sq += samples[(q * J + j) * m + i];
        const double mq = sq / static_cast<double>(J);
        rank += (mq < mb || (mq == mb && q < b)) ? 1 : 0;
      }
      if (rank == hK) up = mb;
      if (rank == hK - 1) lo = mb;
    }
    out[i] = (K % 2 == 1) ? up : 0.5 * (lo + up);
  }
}

// stream.hpp:158-162 (|t| = eps kept).
__global__ void hard_threshold_kernel(const double* __restrict__ v, int64_t len, double eps, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = fabs(v[i]) >= eps ? v[i] : 0.0;
}

// kerdock.hpp:156-167: s_ell = sqrt(d) * (first n entries of u_ell): Kerdock entries
// (-1)^(Q_s(pos) + w.pos) from the reversed rows (Q evaluated on position bits,
// stream.hpp:76-84), identity sqrt(d) e_w or 0 once projected away.
__global__ void design_column_kernel(int64_t n, int64_t d, int identity, const uint32_t* __restrict__ rev, int k,
                                     uint64_t wpos, double sqrt_d, double* __restrict__ out) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    if (identity) {
      out[p] = (static_cast<uint64_t>(p) == wpos) ? sqrt_d : 0.0;
      continue;
    }
    // Q(pos) = sum_{a<b} M'_{ab} pos_a pos_b over position bits (rev[a] bit b = M'_{a,b})
    int q = 0;
    const uint64_t pos = static_cast<uint64_t>(p);
    for (int a = 0; a < k; ++a)
      if ((pos >> a) & 1u) q ^= __popcll(static_cast<uint64_t>(rev[a]) & pos & ~((uint64_t{2} << a) - 1)) & 1;
    q ^= __popcll(wpos & pos) & 1;
    out[p] = q ? -1.0 : 1.0;
  }
}

unsigned blocks_for(int64_t count) {
  const int64_t b = (count + 255) / 256;
  return static_cast<unsigned>(b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b));
}

}  // namespace

cudaError_t launch_inner_product(const double* x, int64_t n, int64_t d, const uint32_t* rev, uint64_t wpos,
                                 double* out, cudaStream_t st) {
  inner_product_kernel<<<1, 1, 0, st>>>(x, n, d, rev, wpos, out);
  return cudaGetLastError();
}

cudaError_t launch_median_of_means(const double* samples, int64_t m, int64_t J, int64_t K, double* out,
                                   cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  median_of_means_kernel<<<blocks_for(m), 256, 0, st>>>(samples, m, J, K, out);
  return cudaGetLastError();
}

cudaError_t launch_hard_threshold(const double* v, int64_t len, double eps, double* out, cudaStream_t st) {
  if (len <= 0) return cudaSuccess;
  hard_threshold_kernel<<<blocks_for(len), 256, 0, st>>>(v, len, eps, out);
  return cudaGetLastError();
}

cudaError_t launch_design_column(int64_t n, int64_t d, int identity, const uint32_t* rev, int k, uint64_t wpos,
                                 double sqrt_d, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  design_column_kernel<<<blocks_for(n), 256, 0, st>>>(n, d, identity, rev, k, wpos, sqrt_d, out);
  return cudaGetLastError();
}

}  // namespace fstg
