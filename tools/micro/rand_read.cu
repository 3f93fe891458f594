// Ceiling of the stream kernel's DRAM access pattern (tools only, not product):
// persistent CTAs issue 1-D TMA bulk copies of random 16 KiB columns into an
// mbarrier ring; a consumer warp releases slots. Reports GB/s for ring depth,
// CTAs per SM and split requests.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2105_05879_b200/csrc/fst_common.cuh"
using namespace fstg;

// wait variants: 0 = try_wait with the 10 ms suspend hint (fst_common.cuh), 1 = try_wait without a hint,
// 2 = test_wait spin
__device__ __forceinline__ bool try_wait_nohint(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait_mode(uint64_t* bar, uint32_t parity, int mode) {
  if (mode == 0) {
    while (!mbar_try_wait(bar, parity)) {
    }
  } else if (mode == 1) {
    while (!try_wait_nohint(bar, parity)) {
    }
  } else {
    while (!test_wait(bar, parity)) {
    }
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void rr_kernel(const char* __restrict__ buf, uint64_t ncols, int stages, int iters, int split, int seq,
                          float* sink, int pmode, int cmode, int nprod) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 32;
  unsigned char* ring = smem + 1024;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  if (nprod < 0) {
    if (warp == 0 && lane < -nprod) {
      for (int i = lane; i < iters; i += -nprod) {
        const int s = i % stages;
        if (i >= stages) wait_mode(empty + s, ((i / stages) - 1) & 1, pmode);
        const uint64_t col = mix64(uint64_t(blockIdx.x) * 1000003ull + i) % ncols;
        mbar_arrive_expect_tx(full + s, 16384);
        bulk_g2s(ring + s * 16384, buf + col * 16384, 16384, full + s, pol);
      }
    } else if (warp == 1) {
      float acc = 0;
      for (int i = 0; i < iters; ++i) {
        const int s = i % stages;
        wait_mode(full + s, (i / stages) & 1, cmode);
        acc += reinterpret_cast<const float*>(ring + s * 16384)[lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
      }
      if (acc == 12345.f) sink[0] = acc;
    }
    return;
  }
  if (warp < nprod && lane == 0) {
    for (int i = warp; i < iters; i += nprod) {
      const int s = i % stages;
      if (i >= stages) wait_mode(empty + s, ((i / stages) - 1) & 1, pmode);
      const uint64_t col = seq ? (uint64_t(blockIdx.x) * iters + i) % ncols : mix64(uint64_t(blockIdx.x) * 1000003ull + i) % ncols;
      const char* src = buf + col * 16384;
      mbar_arrive_expect_tx(full + s, 16384);
      const uint32_t part = 16384 / split;
      for (int q = 0; q < split; ++q) bulk_g2s(ring + s * 16384 + q * part, src + q * part, part, full + s, pol);
    }
  } else if (warp == nprod) {
    float acc = 0;
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      wait_mode(full + s, (i / stages) & 1, cmode);
      acc += reinterpret_cast<const float*>(ring + s * 16384)[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
    if (acc == 12345.f) sink[0] = acc;
  }
}

int main() {
  const size_t bytes = size_t(128) << 30;
  char* buf;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 1, bytes);
  float* sink;
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(rr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const uint64_t ncols = bytes / 16384;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct V { int stages, ctas_per_sm, split, seq, pmode, cmode, nprod; uint64_t cols; };
  const uint64_t l2c = (uint64_t(64) << 20) / 16384;   // 64 MiB: L2-resident
  V vs[] = {{5, 1, 1, 0, 0, 0, -5, ncols}, {8, 1, 1, 0, 0, 0, -4, ncols}, {5, 1, 1, 0, 0, 0, -5, l2c},
            {8, 1, 1, 0, 0, 0, -8, l2c}, {6, 2, 1, 0, 0, 0, -6, l2c}, {12, 1, 1, 0, 0, 0, -12, l2c},
            {4, 3, 1, 0, 0, 0, -4, l2c}, {6, 1, 1, 0, 0, 0, -6, (uint64_t(32) << 20) / 16384}};
  for (const V& v : vs) {
    const int grid = 148 * v.ctas_per_sm;
    const int iters = int((size_t(48) << 30) / 16384 / grid);
    const size_t smem = 1024 + size_t(v.stages) * 16384;
    rr_kernel<<<grid, 32 * ((v.nprod < 0 ? 1 : v.nprod) + 1), smem>>>(buf, v.cols, v.stages, iters / 4, v.split, v.seq, sink, v.pmode, v.cmode, v.nprod);  // warm
    cudaEventRecord(a);
    rr_kernel<<<grid, 32 * ((v.nprod < 0 ? 1 : v.nprod) + 1), smem>>>(buf, v.cols, v.stages, iters, v.split, v.seq, sink, v.pmode, v.cmode, v.nprod);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double gb = double(grid) * iters * 16384 / 1e9;
    printf("buf %6.0f MiB producers %d pwait %d cwait %d stages %2d ctas/SM %d split %d %s: %.2f ms  %.0f GB/s  (%.0f KiB in flight/SM)\n", v.cols * 16384.0 / 1048576, v.nprod, v.pmode, v.cmode, v.stages,
           v.ctas_per_sm, v.split, v.seq ? "seq " : "rand", ms, gb / ms * 1e3, v.stages * 16.0 * v.ctas_per_sm);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
