// Bisect helper (tools only): the ldg_read micro with the stream kernel's sample-index
// ring (a producer warp stages random indices in shared memory, chunks of 64, 8 chunks,
// mbarrier full/empty) feeding 8 loader warps that keep D columns in flight.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2105_05879_b200/csrc/fst_common.cuh"
using namespace fstg;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <int D, int MODE, int VAR>
__global__ void __launch_bounds__(288, 1) kern(const float4* __restrict__ cols, uint64_t ncols, const uint32_t* idx,
                                               int64_t G, float* out) {
  __shared__ uint32_t ring[512];
  __shared__ uint64_t full[8], empty[8];
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  if (tid < 8) {
    mbar_init(&full[tid], 1);
    mbar_init(&empty[tid], 8);
  }
  fence_mbar_init();
  __syncthreads();
  if (warp == 8) {  // producer
    for (int64_t c = 0; c * 64 < G; ++c) {
      const int slot = c % 8;
      const uint32_t u = c / 8;
      if (u > 0 && !(VAR & 1)) mbar_wait(&empty[slot], (u - 1) & 1u);
      for (int h = 0; h < 2; ++h) {
        const int64_t g = c * 64 + lane + 32 * h;
        ring[slot * 64 + lane + 32 * h] =
            MODE == 1 ? __ldg(idx + blockIdx.x * G + g) : static_cast<uint32_t>(__umul64hi(mix64(blockIdx.x * G + g), ncols));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[slot]);
    }
    return;
  }
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  float4 buf[D][4];
  int64_t gl = 0;
  auto issue = [&](float4(&b)[4]) {
    if ((VAR & 4) || gl < G) {
      const uint32_t pos = gl % 64, slot = (gl / 64) % 8;
      if (pos == 0 && !(VAR & 2)) mbar_wait(&full[slot], (gl / 512) & 1u);
      const uint32_t ell = ring[slot * 64 + pos];
      const float4* c = cols + uint64_t(ell) * 1024 + 2 * tid;
      ldg_stream8(c, b[0], b[1]);
      ldg_stream8(c + 512, b[2], b[3]);
      if (pos == 63 && !(VAR & 1)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
    }
    ++gl;
  };
#pragma unroll
  for (int d = 0; d < D; ++d) issue(buf[d]);
  for (int64_t g = 0; g < G;) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if ((VAR & 4) || g < G) {
        const float t = (VAR & 8) ? 1.0f + 1e-7f * float(d) : 1.0f + 1e-7f * float(g);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc[4 * k + 0] = fmaf(t, buf[d][k].x, acc[4 * k + 0]);
          acc[4 * k + 1] = fmaf(t, buf[d][k].y, acc[4 * k + 1]);
          acc[4 * k + 2] = fmaf(t, buf[d][k].z, acc[4 * k + 2]);
          acc[4 * k + 3] = fmaf(t, buf[d][k].w, acc[4 * k + 3]);
        }
        issue(buf[d]);
        ++g;
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * 256 + tid] = s;
}

template <int D, int MODE, int VAR>
void run(const float4* cols, uint64_t ncols, const uint32_t* idx, int64_t G, float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<D, MODE, VAR><<<148, 288>>>(cols, ncols, idx, 512, out);
  cudaEventRecord(e0);
  kern<D, MODE, VAR><<<148, 288>>>(cols, ncols, idx, G, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("D=%d mode=%d var=%d  %.1f GB/s (%.2f ms) %s\n", D, MODE, VAR, 148.0 * G * 16384.0 / ms / 1e6, ms,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const uint64_t bytes = 128ull << 30, ncols = bytes / 16384;
  const int64_t G = 20000;
  float4* cols;
  float* out;
  uint32_t* idx;
  if (cudaMalloc(&cols, bytes) != cudaSuccess) return 1;
  cudaMemset(cols, 0, bytes);
  cudaMalloc(&out, 148 * 256 * sizeof(float));
  cudaMalloc(&idx, 148 * G * sizeof(uint32_t));
  uint32_t* h = (uint32_t*)malloc(148 * G * 4);
  uint64_t z = 1;
  for (int64_t i = 0; i < 148 * G; ++i) {
    z = z * 6364136223846793005ull + 1442695040888963407ull;
    h[i] = (uint32_t)((z >> 33) % ncols);
  }
  cudaMemcpy(idx, h, 148 * G * 4, cudaMemcpyHostToDevice);
  const int v = getenv("VAR") ? atoi(getenv("VAR")) : 0;
  if (v == 0) run<4, 0, 0>(cols, ncols, idx, G, out);
  if (v == 2) run<4, 0, 2>(cols, ncols, idx, G, out);
  if (v == 3) run<4, 0, 3>(cols, ncols, idx, G, out);
  if (v == 7) run<4, 0, 7>(cols, ncols, idx, G, out);
  if (v == 11) run<4, 0, 11>(cols, ncols, idx, G, out);
  if (v == 15) run<4, 0, 15>(cols, ncols, idx, G, out);
  return 0;
}
