// Index draws: draw_samples (reference stream.hpp:173-182) for a batch of
// vectors. Vector v runs std::mt19937_64(seed[v]) (rng.hpp:15) and maps each
// 64-bit output y to ell = (y * L) >> 64 (rng.hpp:20-23), in draw order.
// One warp per vector: lane 0 seeds, the warp regenerates the 312-word state
// in parallel and tempers 32 outputs at a time.
#include <cuda_runtime.h>

#include <cstdint>

#include "fst_common.cuh"
#include "kernels.hpp"

namespace fstg {

template <typename IdxT>
__global__ void __launch_bounds__(128) draw_kernel(const uint64_t* __restrict__ seeds, uint64_t seed_base,
                                                   int64_t B, int64_t N, uint64_t L, IdxT* __restrict__ out) {
  __shared__ uint64_t state[4][kMtN];
  const int lane = threadIdx.x % 32, wib = threadIdx.x / 32;
  uint64_t* mt = state[wib];
  const int64_t warps = int64_t(gridDim.x) * 4;
  for (int64_t v = int64_t(blockIdx.x) * 4 + wib; v < B; v += warps) {
    const uint64_t seed = seeds ? seeds[v] : seed_base;
    mt_seed_warp(mt, seed, lane);
    IdxT* dst = out + v * N;
    for (int64_t base = 0; base < N; base += kMtN) {
      mt_twist_warp(mt, lane);
      const int64_t cnt = (N - base < kMtN) ? (N - base) : kMtN;
      for (int64_t i = lane; i < cnt; i += 32) dst[base + i] = static_cast<IdxT>(__umul64hi(mt_temper(mt[i]), L));
      __syncwarp();
    }
  }
}

template <typename IdxT>
cudaError_t launch_draw(const uint64_t* seeds, uint64_t seed_base, int64_t B, int64_t N, uint64_t L, IdxT* out,
                        cudaStream_t st) {
  if (B <= 0 || N <= 0) return cudaSuccess;
  int64_t blocks = (B + 3) / 4;
  if (blocks > 148 * 16) blocks = 148 * 16;
  draw_kernel<IdxT><<<static_cast<unsigned>(blocks), 128, 0, st>>>(seeds, seed_base, B, N, L, out);
  return cudaGetLastError();
}

template cudaError_t launch_draw<uint32_t>(const uint64_t*, uint64_t, int64_t, int64_t, uint64_t, uint32_t*,
                                           cudaStream_t);
template cudaError_t launch_draw<int64_t>(const uint64_t*, uint64_t, int64_t, int64_t, uint64_t, int64_t*,
                                          cudaStream_t);

// int64 (API) -> uint32 (device) indices with range validation; flags[0] is
// set when an index is outside [0, L) (reported as std::out_of_range).
__global__ void narrow_indices_kernel(const int64_t* __restrict__ in, int64_t count, int64_t L,
                                      uint32_t* __restrict__ out, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = in[i];
    if (v < 0 || v >= L) {
      atomicExch(bad, 1);
      out[i] = 0;
    } else {
      out[i] = static_cast<uint32_t>(v);
    }
  }
}

cudaError_t launch_narrow_indices(const int64_t* in, int64_t count, int64_t L, uint32_t* out, int* bad,
                                  cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  narrow_indices_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(in, count, L, out, bad);
  return cudaGetLastError();
}

}  // namespace fstg
