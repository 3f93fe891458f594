// Random 16 KiB column reads straight into registers (tools only, not product):
// the alternative to the stream kernel's TMA ring. Persistent CTAs of 8 warps
// (256 threads, 16 rows = 4 x 16-byte chunks per thread per column), each
// thread keeping D columns of loads in flight (register ring, unrolled), FMA
// accumulating like the consumer warps. Reports GB/s per D.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2105_05879_b200/csrc/fst_common.cuh"

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// 256-bit load (two float4), L2 evict-first: sm_100 takes .L2::evict_first only on v8.b32 / v4.b64
__device__ __forceinline__ void ldg_stream8(const float4* p, float4& a, float4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
               : "l"(p));
}

template <int D>
__global__ void __launch_bounds__(768, 1) ldg_kernel(const float4* __restrict__ cols, uint64_t ncols, int per_cta,
                                                     float* out) {
  const int tid = threadIdx.x;
  __shared__ uint64_t never, done;
  if (tid == 0) {
    fstg::mbar_init(&never, 1);
    fstg::mbar_init(&done, 256);
  }
  __syncthreads();
  if (tid >= 256) {
    // SPIN: extra warps wait on an mbarrier (like the kernel's idle roles) until the loaders finish
#ifdef SETMAXNREG
    if (tid < 512) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;" ::: "memory");
    else asm volatile("setmaxnreg.dec.sync.aligned.u32 64;" ::: "memory");
#endif
    if (out == nullptr) return;
    while (!fstg::mbar_try_wait(&done, 0)) {
    }
    return;
  }
#ifdef SETMAXNREG
  asm volatile("setmaxnreg.inc.sync.aligned.u32 104;" ::: "memory");
#endif
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  float4 buf[D][4];
  uint64_t seed = blockIdx.x * 1000003ull;
  __shared__ uint32_t zeros[64];
  if (tid < 64) zeros[tid] = 0;
  __syncthreads();
#ifdef WITH_LDS
  // the column address depends on a shared-memory load (like an index ring)
  auto col_of = [&](int j) { return __umul64hi(mix64(seed + j), ncols) ^ zeros[j & 63]; };
#else
  auto col_of = [&](int j) { return __umul64hi(mix64(seed + j), ncols); };
#endif
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const float4* c = cols + col_of(d) * 1024;
#pragma unroll
    for (int k = 0; k < 2; ++k) ldg_stream8(c + 2 * tid + 512 * k, buf[d][2 * k], buf[d][2 * k + 1]);
  }
  for (int j = 0; j < per_cta; j += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const float t = 1.0f + 1e-7f * (j + d);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[4 * k + 0] = fmaf(t, buf[d][k].x, acc[4 * k + 0]);
        acc[4 * k + 1] = fmaf(t, buf[d][k].y, acc[4 * k + 1]);
        acc[4 * k + 2] = fmaf(t, buf[d][k].z, acc[4 * k + 2]);
        acc[4 * k + 3] = fmaf(t, buf[d][k].w, acc[4 * k + 3]);
      }
      const float4* c = cols + col_of(j + d + D) * 1024;
#pragma unroll
      for (int k = 0; k < 2; ++k) ldg_stream8(c + 2 * tid + 512 * k, buf[d][2 * k], buf[d][2 * k + 1]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * 256 + tid] = s;
  fstg::mbar_arrive(&done);
}

template <int D>
void run(const float4* cols, uint64_t ncols, float* out, int ctas) {
  const int per_cta = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = getenv("SMEM_KB") ? atoi(getenv("SMEM_KB")) * 1024 : 0;
  cudaFuncSetAttribute(ldg_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int thr = getenv("THREADS") ? atoi(getenv("THREADS")) : 256;
  ldg_kernel<D><<<ctas, thr, smem>>>(cols, ncols, 512, out);
  cudaEventRecord(e0);
  ldg_kernel<D><<<ctas, thr, smem>>>(cols, ncols, per_cta, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = double(ctas) * ((per_cta + D - 1) / D * D + D) * 16384.0;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, ldg_kernel<D>);
  printf("D=%2d ctas=%d smem=%dK regs=%d spill=%zu  %.1f GB/s  (%.2f ms) %s\n", D, ctas, smem / 1024, fa.numRegs,
         fa.localSizeBytes, bytes / ms / 1e6, ms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const uint64_t bytes = (getenv("GIB") ? strtoull(getenv("GIB"), 0, 10) : 64ull) << 30;
  const uint64_t ncols = bytes / 16384;
  float4* cols;
  float* out;
  if (cudaMalloc(&cols, bytes) != cudaSuccess) return 1;
  cudaMemset(cols, 0, bytes);
  cudaMalloc(&out, 148 * 2 * 256 * sizeof(float));
  for (int ctas : {148}) {
    run<2>(cols, ncols, out, ctas);
    run<4>(cols, ncols, out, ctas);
    run<6>(cols, ncols, out, ctas);
    run<8>(cols, ncols, out, ctas);
    run<10>(cols, ncols, out, ctas);
  }
  return 0;
}
