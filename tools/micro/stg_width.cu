// Store-request shape for the sketch write-back (tools only): each CTA writes 8 rows
// of every column of 128 bases (columns 16 KiB apart), 1 CTA/SM, as
//   A: st.global.b32  - lane = (row r, column group): 4 columns x 8 rows per warp request
//   B: st.global.v4   - lane = (4-row half, column):  16 columns x 8 rows per warp request
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) st32(float* cols, int64_t ldc, int d, int bpc, int nb) {
  extern __shared__ float dummy[];
  const int64_t i0 = int64_t(blockIdx.x) * 8;
  const int r = threadIdx.x % 8, c = threadIdx.x / 8;
  for (int s = blockIdx.y * bpc; s < min(nb, int(blockIdx.y) * bpc + bpc); ++s)
    for (int w = c; w < d; w += 64) cols[(int64_t(s) * d + w) * ldc + i0 + r] = float(w);
}

__global__ void __launch_bounds__(512, 1) st128(float* cols, int64_t ldc, int d, int bpc, int nb) {
  extern __shared__ float dummy[];
  const int64_t i0 = int64_t(blockIdx.x) * 8;
  const int h = threadIdx.x % 2, c = threadIdx.x / 2;  // 256 columns per pass, 2 threads per column
  for (int s = blockIdx.y * bpc; s < min(nb, int(blockIdx.y) * bpc + bpc); ++s)
    for (int w = c; w < d; w += 256)
      *reinterpret_cast<float4*>(cols + (int64_t(s) * d + w) * ldc + i0 + 4 * h) = make_float4(w, w, w, w);
}

int main() {
  const int64_t m = 4096, d = 4096, nb = 2048, ldc = m;
  const size_t bytes = size_t(nb) * d * ldc * 4;
  float* cols;
  if (cudaMalloc(&cols, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(cols, 0, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int bpc = 128;
  dim3 grid(unsigned(m / 8), unsigned(nb / bpc));
  for (auto k : {st32, st128}) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    for (int which = 0; which < 2; ++which) {
      auto k = which ? st128 : st32;
      k<<<grid, 512, 120 * 1024>>>(cols, ldc, int(d), bpc, int(nb));
      cudaEventRecord(a);
      k<<<grid, 512, 120 * 1024>>>(cols, ldc, int(d), bpc, int(nb));
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%s: %.2f ms %.0f GB/s\n", which ? "st.v4 (16 B/thread)" : "st.b32 (4 B/thread)", ms, bytes / ms / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
