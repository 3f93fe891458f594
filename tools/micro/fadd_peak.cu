// FP32 add-rate ceiling on the CUDA cores (tools only): the denominator of the
// config-4 Kerdock-pass roofline. Independent chains of
//   A: FADD   (scalar, 1 add per lane)
//   B: FADD2  (packed, 2 adds per lane)
//   C: FADD2 + FFMA2(y, -1, x) pairs, the butterfly mix of preprocess.cu
// with 8 resident warps per SMSP, 1 CTA of 1024 threads per SM (grid = 148 x 2).
// Prints adds/clk/SM (from the SM clock read during the run) and Tadd/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 16;    // independent chains per thread
constexpr int IT = 4096;  // iterations

__global__ void __launch_bounds__(1024, 1) k_fadd(float* out, float a, float b) {
  float v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-7f + c;
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = v[c] + a;
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = v[c] + b;
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(1024, 1) k_fadd2(float* out, float a, float b) {
  float2 v[CH / 2];
#pragma unroll
  for (int c = 0; c < CH / 2; ++c) v[c] = make_float2(threadIdx.x * 1e-7f + c, c);
  const float2 A = make_float2(a, b), B = make_float2(b, a);
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) v[c] = __fadd2_rn(v[c], A);
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) v[c] = __fadd2_rn(v[c], B);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH / 2; ++c) s += v[c].x + v[c].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}

// butterfly mix: (x, y) -> (x + y, x - y) on packed pairs, 4 independent pairs of pairs
__global__ void __launch_bounds__(1024, 1) k_bfly2(float* out, float a, float b) {
  float2 x[CH / 4], y[CH / 4];
#pragma unroll
  for (int c = 0; c < CH / 4; ++c) {
    x[c] = make_float2(threadIdx.x * 1e-7f + c, a);
    y[c] = make_float2(b, c * 0.5f);
  }
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH / 4; ++c) {
      const float2 s = __fadd2_rn(x[c], y[c]);
      const float2 d = __ffma2_rn(y[c], make_float2(-1.f, -1.f), x[c]);
      x[c] = __fmul2_rn(s, make_float2(0.5f, 0.5f));  // keep values bounded (2 FP ops counted as adds below)
      y[c] = d;
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH / 4; ++c) s += x[c].x + y[c].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct K {
    const char* name;
    void (*f)(float*, float, float);
    double lane_ops_per_iter;  // FP32 lane-ops per thread per iteration
  } ks[] = {{"FADD  (scalar)", k_fadd, 2.0 * CH}, {"FADD2 (packed)", k_fadd2, 2.0 * CH},
            {"FADD2+FFMA2+FMUL2 butterfly", k_bfly2, 6.0 * (CH / 4)}};
  for (int rep = 0; rep < 2; ++rep)
    for (auto& k : ks) {
      const dim3 grid(sms), block(1024);
      k.f<<<grid, block>>>(out, 1e-9f, -1e-9f);
      cudaEventRecord(e0);
      k.f<<<grid, block>>>(out, 1e-9f, -1e-9f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = double(sms) * 1024 * IT * k.lane_ops_per_iter;
      const double rate = ops / (ms * 1e-3);
      if (rep == 1)
        printf("%-30s %8.3f ms  %7.2f T lane-ops/s  %6.1f lane-ops/clk/SM at the %d MHz max clock\n", k.name, ms,
               rate / 1e12, rate / sms / (clk_khz * 1e3), clk_khz / 1000);
    }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
