// L2-exchange write-path microbenchmark (tools only, not product).
// Question: can 4 CTAs that each own 8 rows of a 32-row group turn their 32-byte
// column pieces into full 128-byte column lines by exchanging their tiles through
// an L2-resident scratch area (contiguous 128 KiB tile write, flag hand-off,
// 4 x 32-byte piece reads per line), and is that faster than writing the
// 32-byte pieces directly? Store pattern only, no FWHT arithmetic.
//
//   mode 0: direct 32-B pieces (the current kernel's write-back), 1 CTA/SM, persistent
//   mode 1: L2 exchange (scratch tiles double-buffered per CTA, release/acquire flags)
//   mode 2: like 1 without the flag waits (exchange traffic only; data race, timing only)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 512, R = 8, G = 4, D = 4096;

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st4_pol(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld4_pol(const float4* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// work item = (32-row group, basis range of bpc bases); CTA group g = blockIdx.x / 4 takes items g, g + ngroups, ...
__global__ void __launch_bounds__(NT, 1) l2x_kernel(float* cols, int64_t ldc, int64_t m, int nb, int bpc, int mode,
                                                    float* scratch, unsigned* ready, unsigned* done) {
  extern __shared__ float smem_dummy[];
  const int tid = threadIdx.x, cta = blockIdx.x, rank = cta % G, grp = cta / G;
  const int ngroups = gridDim.x / G;
  const int64_t rgroups = m / (R * G), items = rgroups * ((nb + bpc - 1) / bpc);
  const uint64_t pl = pol_last(), pf = pol_first();
  unsigned seq = 0;  // bases processed by this CTA (uniform in the group)
  for (int64_t it = grp; it < items; it += ngroups) {
    const int64_t rg = it % rgroups, s0 = (it / rgroups) * bpc;
    const int64_t i0 = rg * (R * G);  // first row of the 32-row group
    for (int64_t s = s0; s < s0 + bpc && s < nb; ++s, ++seq) {
      float* colbase = cols + s * D * ldc;
      if (mode == 0) {
        // direct: thread (r = tid % 8, q = tid / 8) writes rows i0 + 8 rank + r of columns e*64 + q
        const int r = tid % R, q = tid / R;
        float* p = colbase + int64_t(q) * ldc + i0 + R * rank + r;
#pragma unroll
        for (int e = 0; e < 64; ++e) p[int64_t(e) * 64 * ldc] = float(e + s);
        continue;
      }
      const int buf = seq & 1;
      float* mine = scratch + (size_t(cta) * 2 + buf) * (D * R);
      // WAR: the peers finished reading this buffer's previous use (basis seq - 2)
      if (mode == 1 && seq >= 2) {
        if (tid < G && tid != rank) {
          const unsigned* f = done + (grp * G + tid);
          while (ld_acquire(f) < seq - 1) {
          }
        }
        __syncthreads();
      }
      // tile -> scratch as [w][8 rows]: a warp writes 4 x 32 B = 128 B contiguous per e
      {
        const int r = tid % R, q = tid / R;
#pragma unroll
        for (int e = 0; e < 64; e += 4) {
          // thread t of the warp stores 16 B = 4 floats of one row? keep it simple: scalar stores, coalesced
#pragma unroll
          for (int u = 0; u < 4; ++u) mine[(size_t(e + u) * 64 + q) * R + r] = float(e + u + s);
        }
      }
      __syncthreads();
      if (mode == 1) {
        if (tid == 0) {
          __threadfence();
          st_release(ready + cta, seq + 1);
        }
        if (tid < G && tid != rank) {
          const unsigned* f = ready + (grp * G + tid);
          while (ld_acquire(f) < seq + 1) {
          }
        }
        __syncthreads();
      }
      // this CTA writes columns w in [1024 rank, 1024 rank + 1024): 32 rows = 4 tiles x 8 rows,
      // 8 threads x 16 B per column line
      {
        const int sub = tid % 8, c0 = tid / 8;  // 64 columns per pass
        const int src = sub / 2, half = sub % 2;
        const float* peer = scratch + (size_t(grp * G + src) * 2 + buf) * (D * R);
        float4 v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int w = 1024 * rank + c0 + 64 * k;
          v[k] = ld4_pol(reinterpret_cast<const float4*>(peer + size_t(w) * R + 4 * half), pl);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int w = 1024 * rank + c0 + 64 * k;
          st4_pol(reinterpret_cast<float4*>(colbase + int64_t(w) * ldc + i0 + 4 * sub), v[k], pf);
        }
      }
      if (mode == 1) {
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          st_release(done + cta, seq + 1);
        }
      }
    }
  }
}

int main() {
  const int64_t m = 4096, nb = 2048, ldc = m;
  const size_t bytes = size_t(nb) * D * ldc * 4;
  float* cols;
  if (cudaMalloc(&cols, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms / G * G;
  float* scratch;
  unsigned *ready, *done;
  cudaMalloc(&scratch, size_t(grid) * 2 * D * R * 4);
  cudaMalloc(&ready, grid * 4);
  cudaMalloc(&done, grid * 4);
  cudaFuncSetAttribute(l2x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaMemset(cols, 0, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode)
      for (int bpc : {32, 128}) {
        cudaMemset(ready, 0, grid * 4);
        cudaMemset(done, 0, grid * 4);
        const int g = mode == 0 ? sms : grid;
        cudaEventRecord(a);
        l2x_kernel<<<g, NT, 160 * 1024>>>(cols, ldc, m, int(nb), bpc, mode, scratch, ready, done);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("mode %d bpc %3d grid %d: %.2f ms  %.2f TB/s  %s\n", mode, bpc, g, ms, bytes / ms / 1e9,
               cudaGetErrorString(e));
      }
  return 0;
}
