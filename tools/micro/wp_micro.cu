// Store-pattern microbenchmark for the sketch write-back (tools only, not product).
// Each CTA owns R rows of every column of a range of bases (column-major, ldc rows
// per column, d columns per basis) and writes them, like fwht12_tmem_kernel's
// transposed write-back. R = 8 (current: 32-B segments), 16 (64 B), 32 (128 B).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int R, int NT>
__global__ void __launch_bounds__(NT) wp_kernel(float* cols, int64_t ldc, int64_t m, int d, int bpc, int nb,
                                                int basis_major) {
  extern __shared__ float dummy[];
  const unsigned bx = basis_major ? blockIdx.y : blockIdx.x, by = basis_major ? blockIdx.x : blockIdx.y;
  const int64_t i0 = int64_t(bx) * R;
  const int s0 = by * bpc;
  const int tid = threadIdx.x;
  // thread -> (row r, column group): R rows x (NT/R) columns per store wave
  const int r = tid % R, c = tid / R;
  constexpr int CPW = NT / R;
  for (int s = s0; s < min(nb, s0 + bpc); ++s) {
    float* base = cols + int64_t(s) * d * ldc + i0 + r;
    for (int w = c; w < d; w += CPW) __stcs(base + int64_t(w) * ldc, float(w + s));
  }
}

template <int R>
float run(float* cols, int64_t ldc, int64_t m, int d, int nb, int bpc, int smem = 0, int basis_major = 0) {
  constexpr int NT = 512;
  cudaFuncSetAttribute(wp_kernel<R, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  dim3 grid(unsigned(m / R), unsigned((nb + bpc - 1) / bpc));
  if (basis_major) grid = dim3(grid.y, grid.x);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  wp_kernel<R, NT><<<grid, NT, smem>>>(cols, ldc, m, d, bpc, nb, basis_major);
  cudaEventRecord(a);
  wp_kernel<R, NT><<<grid, NT, smem>>>(cols, ldc, m, d, bpc, nb, basis_major);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

__global__ void fill_kernel(float4* p, int64_t n4) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x)
    __stcs(p + i, make_float4(1, 2, 3, 4));
}

int main() {
  const int64_t m = 4096, d = 4096, nb = 2048;
  const int64_t ldc = m;
  const size_t bytes = size_t(nb) * d * ldc * 4;
  float* cols;
  if (cudaMalloc(&cols, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  fill_kernel<<<148 * 8, 512>>>(reinterpret_cast<float4*>(cols), bytes / 16);
  cudaEventRecord(a);
  fill_kernel<<<148 * 8, 512>>>(reinterpret_cast<float4*>(cols), bytes / 16);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("contiguous fill %.2f ms %.0f GB/s\n", ms, bytes / ms / 1e6);
  for (int bpc : {32, 128}) {
    float t8 = run<8>(cols, ldc, m, d, nb, bpc);
    float t16 = run<16>(cols, ldc, m, d, nb, bpc);
    float t32 = run<32>(cols, ldc, m, d, nb, bpc);
    float t64 = run<64>(cols, ldc, m, d, nb, bpc);
    printf("bpc %d: R=8 %.2f ms (%.0f GB/s)  R=16 %.2f (%.0f)  R=32 %.2f (%.0f)  R=64 %.2f (%.0f)\n", bpc, t8,
           bytes / t8 / 1e6, t16, bytes / t16 / 1e6, t32, bytes / t32 / 1e6, t64, bytes / t64 / 1e6);
  }
  for (int smem : {0, 60 * 1024, 120 * 1024}) {
    for (int bm : {0, 1}) {
      float t8 = run<8>(cols, ldc, m, d, nb, 32, smem, bm);
      float t16 = run<16>(cols, ldc, m, d, nb, 32, smem, bm);
      float t32 = run<32>(cols, ldc, m, d, nb, 32, smem, bm);
      printf("smem %dK basis_major %d: R=8 %.2f ms  R=16 %.2f  R=32 %.2f\n", smem / 1024, bm, t8, t16, t32);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
