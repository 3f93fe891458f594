// Store-path microbenchmark (tools only): the sketch write-back (8 rows x every column
// of a basis per CTA, columns 16 KiB apart) issued as TMA 2-D tensor stores of
// [8 rows x BOXC columns] boxes from shared memory vs plain st.global.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int BOXC>
__global__ void __launch_bounds__(256, 1) tma_store_kernel(const __grid_constant__ CUtensorMap map, int d, int bpc, int nb) {
  __shared__ __align__(128) float stage[2][BOXC * 8];
  const int i0 = blockIdx.x * 8;
  const int s0 = blockIdx.y * bpc;
  for (int k = threadIdx.x; k < BOXC * 8; k += blockDim.x) { stage[0][k] = 1.f; stage[1][k] = 2.f; }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  int buf = 0;
  for (int s = s0; s < min(nb, s0 + bpc); ++s) {
    for (int c0 = 0; c0 < d; c0 += BOXC) {
      if (threadIdx.x == 0) {
        const int col = s * d + c0;
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                     :: "l"(&map), "r"(i0), "r"(col), "r"(smem_u32(stage[buf])) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // the other buffer is free
      }
      buf ^= 1;
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(512, 1) stg_kernel(float* cols, int64_t ldc, int d, int bpc, int nb) {
  extern __shared__ float dummy[];
  const int64_t i0 = int64_t(blockIdx.x) * 8;
  const int r = threadIdx.x % 8, c = threadIdx.x / 8;
  for (int s = blockIdx.y * bpc; s < min(nb, int(blockIdx.y) * bpc + bpc); ++s)
    for (int w = c; w < d; w += 64) __stcs(cols + (int64_t(s) * d + w) * ldc + i0 + r, float(w));
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
  auto timeit = [&](auto launch) {
    launch();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  };
  const int bpc = 32;
  dim3 grid(unsigned(m / 8), unsigned(nb / bpc));
  cudaFuncSetAttribute(stg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  float t = timeit([&] { stg_kernel<<<grid, 512, 120 * 1024>>>(cols, ldc, int(d), bpc, int(nb)); });
  printf("st.global R=8, 1 CTA/SM: %.2f ms %.0f GB/s\n", t, bytes / t / 1e6);
  auto run_tma = [&](auto kern, int boxc) {
    CUtensorMap map;
    cuuint64_t gdim[2] = {cuuint64_t(ldc), cuuint64_t(nb * d)};
    cuuint64_t gstride[1] = {cuuint64_t(ldc * 4)};
    cuuint32_t box[2] = {8, cuuint32_t(boxc)};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, cols, gdim, gstride, box, estride,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return; }
    for (int extra_smem : {0, 100 * 1024}) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, extra_smem);
      float tt = timeit([&] { kern<<<grid, 256, extra_smem>>>(map, int(d), bpc, int(nb)); });
      printf("TMA store box 8 x %d, extra smem %dK: %.2f ms %.0f GB/s\n", boxc, extra_smem / 1024, tt, bytes / tt / 1e6);
    }
  };
  run_tma(tma_store_kernel<256>, 256);
  run_tma(tma_store_kernel<128>, 128);
  run_tma(tma_store_kernel<64>, 64);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
