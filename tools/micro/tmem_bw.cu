// TMEM read / write throughput per SM (tools only): the config-4 FWHT kernels re-read
// their A row from tensor memory for every basis (64 KiB per basis-row at k = 14).
// W warps per CTA (W % 4 == 0), 1 CTA per SM, 128 TMEM columns per warp-quarter
// group; each warp repeatedly issues tcgen05.ld.32x32b.x32 (4 KiB per warp-instruction)
// or tcgen05.st of the same shape. Prints bytes/clk/SM from clock64 of warp 0.
// (Round 1's version consumed the loaded values with a run-time register index, which
// put the 128-value buffer in local memory and measured that traffic: ~32 B/clk/SM.)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int W, bool STORE>
__global__ void __launch_bounds__(W * 32, 1) tmem_kernel(float* out, int iters, long long* cycles) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x / 32;
  constexpr int COLS = 512;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&base)), "n"(COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w: lanes 32 (w % 4), columns 32 * (w / 4) .. (x32 per instruction, 4 column groups rotate)
  const uint32_t t = base + (static_cast<uint32_t>(32 * (warp % 4)) << 16);
  const uint32_t cg = static_cast<uint32_t>((warp / 4) % (COLS / 128));
  float acc = 0.f;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = float(threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t addr = t + 128 * cg + 32 * (it & 3);
    if constexpr (STORE) {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
          "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
          "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
          "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
          "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
          "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
          : "memory");
    } else {
      // 4 loads in flight (like the FWHT kernels: a 128-value row per thread), then wait
      float w[4][32];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
            "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=f"(w[k][0]), "=f"(w[k][1]), "=f"(w[k][2]), "=f"(w[k][3]), "=f"(w[k][4]), "=f"(w[k][5]), "=f"(w[k][6]),
              "=f"(w[k][7]), "=f"(w[k][8]), "=f"(w[k][9]), "=f"(w[k][10]), "=f"(w[k][11]), "=f"(w[k][12]),
              "=f"(w[k][13]), "=f"(w[k][14]), "=f"(w[k][15]), "=f"(w[k][16]), "=f"(w[k][17]), "=f"(w[k][18]),
              "=f"(w[k][19]), "=f"(w[k][20]), "=f"(w[k][21]), "=f"(w[k][22]), "=f"(w[k][23]), "=f"(w[k][24]),
              "=f"(w[k][25]), "=f"(w[k][26]), "=f"(w[k][27]), "=f"(w[k][28]), "=f"(w[k][29]), "=f"(w[k][30]),
              "=f"(w[k][31])
            : "r"(t + 128 * cg + 32 * k)
            : "memory");
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 4; ++k) acc += w[k][0] + w[k][13] + w[k][31];  // static indices: w stays in registers
    }
  }
  if constexpr (STORE) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  else asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  long long t1 = clock64();
  for (int i = 0; i < 32; ++i) acc += v[i];
  if (acc == 1234.5f) out[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS) : "memory");
}

template <int W, bool STORE>
void run(float* out, long long* cyc_d, int sms) {
  const int iters = 4096;
  tmem_kernel<W, STORE><<<sms, W * 32>>>(out, iters, cyc_d);
  tmem_kernel<W, STORE><<<sms, W * 32>>>(out, iters, cyc_d);
  cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, cyc_d, sizeof(cyc), cudaMemcpyDeviceToHost);
  const double bytes = double(W) * iters * 32 * 32 * 4 * (STORE ? 1 : 4);  // per CTA (= per SM)
  printf("%s warps/CTA %2d: %.1f bytes/clk/SM (%lld cycles)\n", STORE ? "tcgen05.st" : "tcgen05.ld", W, bytes / cyc, cyc);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&cyc, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, false>(out, cyc, sms);
  run<8, false>(out, cyc, sms);
  run<16, false>(out, cyc, sms);
  run<4, true>(out, cyc, sms);
  run<8, true>(out, cyc, sms);
  run<16, true>(out, cyc, sms);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
