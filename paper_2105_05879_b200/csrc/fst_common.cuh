// Device helpers shared by the sm_100a kernels: mbarrier / bulk-copy (TMA)
// PTX wrappers, L2 cache policies, and the MT19937-64 engine the reference's
// SeededRng is built on (rng.hpp:15, std::mt19937_64).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fstg {

// ------------------------------------------------------------ mbarriers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// try_wait with a suspend-time hint: a waiting thread is parked by the
// hardware (up to the hint, in ns) instead of re-issuing the probe, so waiting
// warps do not steal issue slots from the warps doing the work.
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ------------------------------------------------------ cache policies ----
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// -------------------------------------------------- bulk copy (1-D TMA) ----
// Global -> shared bulk copy completing on an mbarrier (cp.async.bulk; SASS
// UBLKCP). bytes and both addresses must be 16-byte multiples.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// ------------------------------------------------- cached global loads ----
__device__ __forceinline__ float4 ldg_f4_policy(const float4* p, uint64_t policy) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(policy));
  return v;
}

__device__ __forceinline__ uint2 ldg_u2_policy(const uint2* p, uint64_t policy) {
  uint2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(policy));
  return v;
}

__device__ __forceinline__ double2 ldg_d2_policy(const double2* p, uint64_t policy) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(policy));
  return v;
}

__device__ __forceinline__ void stg_f32_policy(float* p, float v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(policy) : "memory");
}

__device__ __forceinline__ void stg_f64_policy(double* p, double v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(policy) : "memory");
}

// Named barrier over `count` threads (consumer warps only; the producer warp
// never joins). id 0 is __syncthreads.
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// --------------------------------------------------------- MT19937-64 ----
// Standard 64-bit Mersenne Twister (std::mt19937_64, rng.hpp:15): n = 312,
// m = 156, r = 31, a = 0xB5026F5AA96619E9, u = 29 (d = 0x5555555555555555),
// s = 17 (b = 0x71D67FFFEDA60000), t = 37 (c = 0xFFF7EEE000000000), l = 43,
// f = 6364136223846793005.
constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kMtUpper = 0xFFFFFFFF80000000ull;
constexpr uint64_t kMtLower = 0x000000007FFFFFFFull;

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= (y >> 43);
  return y;
}

__device__ __forceinline__ uint64_t mt_twist_one(uint64_t cur, uint64_t next, uint64_t far) {
  const uint64_t x = (cur & kMtUpper) | (next & kMtLower);
  uint64_t xa = x >> 1;
  if (x & 1ull) xa ^= kMtA;
  return far ^ xa;
}

// Seeds `mt` (312 words in shared memory) from `seed`: lane 0 runs the
// sequential initialisation, then the warp syncs.
__device__ __forceinline__ void mt_seed_warp(uint64_t* mt, uint64_t seed, int lane) {
  if (lane == 0) {
    uint64_t prev = seed;
    mt[0] = prev;
    for (int i = 1; i < kMtN; ++i) {
      prev = 6364136223846793005ull * (prev ^ (prev >> 62)) + static_cast<uint64_t>(i);
      mt[i] = prev;
    }
  }
  __syncwarp();
}

// One full regeneration of the 312-word state by a warp, identical to the
// sequential twist: words [0,156) read only old words; [156,311) read old
// words and new words i-156; word 311 reads new word 0 and new word 155.
__device__ __forceinline__ void mt_twist_warp(uint64_t* mt, int lane) {
  for (int base = 0; base < kMtM; base += 32) {
    const int i = base + lane;
    uint64_t v = 0;
    if (i < kMtM) v = mt_twist_one(mt[i], mt[i + 1], mt[i + kMtM]);
    __syncwarp();
    if (i < kMtM) mt[i] = v;
    __syncwarp();
  }
  for (int base = kMtM; base < kMtN - 1; base += 32) {
    const int i = base + lane;
    uint64_t v = 0;
    if (i < kMtN - 1) v = mt_twist_one(mt[i], mt[i + 1], mt[i - kMtM]);
    __syncwarp();
    if (i < kMtN - 1) mt[i] = v;
    __syncwarp();
  }
  if (lane == 0) mt[kMtN - 1] = mt_twist_one(mt[kMtN - 1], mt[0], mt[kMtN - 1 - kMtM]);
  __syncwarp();
}

}  // namespace fstg
