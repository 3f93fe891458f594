// Preprocessing kernels: the Kerdock-sketch {A s_l} (reference sketch.hpp:144-211).
//
//  * qtable_kernel   — expands each basis' position-reversed Kerdock rows into
//                      sign-bit tables Q_s(coords(pos)) (sketch.hpp:176-179,
//                      kerdock.hpp:38-49), in two layouts: plain (bit pos%32 of
//                      word pos/32) for the FWHT, and lane-transposed for the
//                      streaming coefficient kernel.
//  * fwht_sketch_kernel — per (row tile, basis range): sign-mask R rows of A,
//                      one unnormalised FWHT per row in registers + one shared
//                      memory transpose, written transposed into columns
//                      s*d + w (sketch.hpp:180-196). Butterfly stages run in
//                      the reference order h = 1, 2, 4, ... with (x+y, x-y)
//                      (fwht.hpp:20-29), so fp64 output is bit-identical to the
//                      reference and fp32 output to the same algorithm in fp32.
//  * identity_kernel — column (d/2)*d + w = sqrt(d) * A[:, w] (sketch.hpp:200-208).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "fst_common.cuh"
#include "kernels.hpp"

namespace fstg {

// ---------------------------------------------------------------------------
// Sign tables. One thread per (basis, 32-position word).
// plain:  qplain[s * wpb + w]   bit b = Q_s(pos = 32 w + b)            (wpb = max(1, d/32))
// trans:  qtrans[(s * tw + t) * 32 + lane] bit f = Q_s(pos = 128*(f/4 + 8 t) + 4*lane + f%4)
//         (tw = d/1024 words per lane, d >= 128; f in [0,32) covers i = 8t..8t+7, e = 0..3)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int q_of_pos(const uint32_t* rev, int k, uint32_t pos) {
  // Q_M(coords(pos)) evaluated on the position bits with reversed rows
  // (stream.hpp:76-84, kerdock.hpp:38-49): sum_{a<b} R_ab pos_a pos_b.
  int acc = 0;
  for (uint32_t rest = pos; rest != 0; rest &= rest - 1) {
    const int a = __ffs(rest) - 1;
    const uint32_t above = (a + 1 >= 32) ? 0u : (~0u << (a + 1));
    acc ^= __popc(rev[a] & pos & above) & 1;
  }
  (void)k;
  return acc;
}

__global__ void qtable_kernel(const uint32_t* __restrict__ revtab, int k, int64_t nbases,
                              uint32_t* __restrict__ qplain) {
  const int64_t d = int64_t{1} << k;
  const int64_t wpb = d >= 32 ? d / 32 : 1;
  const int64_t total = nbases * wpb;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = g / wpb;
    const uint32_t w = static_cast<uint32_t>(g % wpb);
    uint32_t rev[16];
#pragma unroll
    for (int a = 0; a < 16; ++a) rev[a] = revtab[s * 16 + a];
    uint32_t word = 0;
    const int nbits = d >= 32 ? 32 : static_cast<int>(d);
    for (int b = 0; b < nbits; ++b) word |= static_cast<uint32_t>(q_of_pos(rev, k, w * 32u + b)) << b;
    qplain[s * wpb + w] = word;
  }
}

// Lane-transposed layout for the streaming coefficient kernel (d >= 128):
// word (s, t, lane), t < tw = max(1, d/1024): bit f <-> position
// 128 * (8 t + f / 4) + 4 * lane + f % 4.
__global__ void qtrans_kernel(const uint32_t* __restrict__ revtab, int k, int64_t nbases,
                              uint32_t* __restrict__ qtrans) {
  const int64_t d = int64_t{1} << k;
  const int64_t tw = d >= 1024 ? d / 1024 : 1;
  const int64_t total = nbases * tw * 32;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = g / (tw * 32);
    const uint32_t t = static_cast<uint32_t>((g / 32) % tw), lane = static_cast<uint32_t>(g % 32);
    uint32_t rev[16];
#pragma unroll
    for (int a = 0; a < 16; ++a) rev[a] = revtab[s * 16 + a];
    uint32_t word = 0;
    for (int f = 0; f < 32; ++f) {
      const uint32_t pos = 128u * (8u * t + static_cast<uint32_t>(f / 4)) + 4u * lane + static_cast<uint32_t>(f % 4);
      if (pos < d) word |= static_cast<uint32_t>(q_of_pos(rev, k, pos)) << f;
    }
    qtrans[g] = word;
  }
}

// ---------------------------------------------------------------------------
// FWHT sketch kernel.
// KB = k (even), E = 2^(KB/2) elements per thread per row, P = E threads per
// row, R = NT / E rows per CTA. Phase 1: thread (r = tid / P, p = tid % P)
// owns positions p*E + e (bits 0..KB/2-1 in registers). Phase 2: thread
// (r = tid % R, q = tid / R) owns positions e*E + q (bits KB/2..KB-1).
// ---------------------------------------------------------------------------
template <typename T, int KB, int NT>
struct FwhtCfg {
  static constexpr int HALF = KB / 2;
  static constexpr int E = 1 << HALF;
  static constexpr int D = 1 << KB;
  static constexpr int R = NT / E;
  static constexpr int PAD = (R <= 32) ? (32 / R) : 1;
  static constexpr int RS = D + PAD;  // row stride (elements) of the smem tile
  static constexpr int SW = (E < 32 ? E : 32) - 1;
  static constexpr size_t SMEM = size_t(R) * RS * sizeof(T);
};

template <typename T>
__device__ __forceinline__ void bfly(T& x, T& y) {
  const T a = x, b = y;
  x = a + b;
  y = a - b;
}

// Butterflies over register bits [0, HALF) in ascending bit order.
template <typename T, int HALF>
__device__ __forceinline__ void reg_fwht(T (&v)[1 << HALF]) {
  constexpr int E = 1 << HALF;
#pragma unroll
  for (int hb = 0; hb < HALF; ++hb) {
    const int h = 1 << hb;
#pragma unroll
    for (int i = 0; i < E; ++i)
      if ((i & h) == 0) bfly(v[i], v[i + h]);
  }
}

// fp32 specialisation with packed FADD2 for stages h >= 2 (pairs (i, i+1)).
template <>
__device__ __forceinline__ void reg_fwht<float, 6>(float (&v)[64]) {
  // stage h = 1 (scalar)
#pragma unroll
  for (int i = 0; i < 64; i += 2) bfly(v[i], v[i + 1]);
#pragma unroll
  for (int hb = 1; hb < 6; ++hb) {
    const int h = 1 << hb;
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
      if ((i & h) == 0) {
        const float2 x = make_float2(v[i], v[i + 1]);
        const float2 y = make_float2(v[i + h], v[i + h + 1]);
        const float2 s = __fadd2_rn(x, y);
        const float2 d = __ffma2_rn(y, make_float2(-1.f, -1.f), x);
        v[i] = s.x;
        v[i + 1] = s.y;
        v[i + h] = d.x;
        v[i + h + 1] = d.y;
      }
    }
  }
}

template <typename T, int KB, int NT>
__global__ void __launch_bounds__(NT) fwht_sketch_kernel(const T* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                                         const uint32_t* __restrict__ qplain, int64_t basis_begin,
                                                         int64_t basis_end, int bases_per_cta, T* __restrict__ cols,
                                                         int64_t ldc) {
  using C = FwhtCfg<T, KB, NT>;
  constexpr int E = C::E, R = C::R, RS = C::RS, D = C::D, SW = C::SW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);

  const int tid = threadIdx.x;
  const int64_t i0 = int64_t(blockIdx.x) * R;
  const int64_t s_first = basis_begin + int64_t(blockIdx.y) * bases_per_cta;
  const int64_t s_last = min(basis_end, s_first + bases_per_cta);
  const uint64_t pol_keep = policy_evict_last();
  const uint64_t pol_stream = policy_evict_first();

  // Phase-1 coordinates.
  const int r1 = tid / E, p1 = tid % E;
  const int64_t row1 = i0 + r1;
  // Phase-2 coordinates.
  const int r2 = tid % R, q2 = tid / R;
  const int64_t row2 = i0 + r2;
  constexpr int WPB = D >= 32 ? D / 32 : 1;

  for (int64_t s = s_first; s < s_last; ++s) {
    T v[E];
    // ---- load + sign mask + zero padding (sketch.hpp:182-186) ----
    uint32_t qw[(E + 31) / 32];
    if constexpr (E >= 32) {
#pragma unroll
      for (int w = 0; w < E / 32; ++w) qw[w] = __ldg(qplain + s * WPB + (int64_t(p1) * E) / 32 + w);
    } else {
      const int64_t pos0 = int64_t(p1) * E;
      qw[0] = (__ldg(qplain + s * WPB + pos0 / 32) >> (pos0 % 32));
    }
    if (row1 < m) {
      const T* arow = a + row1 * lda;
      const int64_t pos0 = int64_t(p1) * E;
      if (pos0 + E <= n && (reinterpret_cast<uintptr_t>(arow + pos0) % 16) == 0) {
        if constexpr (sizeof(T) == 4) {
#pragma unroll
          for (int e = 0; e < E; e += 4) {
            const float4 f = ldg_f4_policy(reinterpret_cast<const float4*>(arow + pos0 + e), pol_keep);
            v[e] = f.x;
            v[e + 1] = f.y;
            v[e + 2] = f.z;
            v[e + 3] = f.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; e += 2) {
            const double2 f = ldg_d2_policy(reinterpret_cast<const double2*>(arow + pos0 + e), pol_keep);
            v[e] = f.x;
            v[e + 1] = f.y;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = (pos0 + e < n) ? arow[pos0 + e] : T(0);
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = T(0);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t bit = (qw[e / 32] >> (e % 32)) & 1u;
      v[e] = bit ? -v[e] : v[e];  // sign[j] * a_ij with sign = +-1 (exact)
    }
    // ---- stages h = 1 .. E/2 in registers ----
    reg_fwht<T, C::HALF>(v);
    // ---- transpose through shared memory ----
    __syncthreads();  // previous basis' phase-2 reads are done
    {
      T* dst = tile + r1 * RS + p1 * E;
#pragma unroll
      for (int e = 0; e < E; ++e) dst[e ^ (p1 & SW)] = v[e];
    }
    __syncthreads();
    {
      const T* src = tile + r2 * RS;
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = src[e * E + (q2 ^ (e & SW))];
    }
    // ---- stages h = E .. D/2 (register index bit j <-> position bit HALF + j) ----
    reg_fwht<T, C::HALF>(v);
    // ---- transposed write-back: column s*d + w, row i0 + r2 (sketch.hpp:191-196) ----
    if (row2 < m) {
      T* ptr = cols + (s * D + q2) * ldc + row2;
      const int64_t step = int64_t(E) * ldc;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if constexpr (sizeof(T) == 4)
          stg_f32_policy(reinterpret_cast<float*>(ptr), static_cast<float>(v[e]), pol_stream);
        else
          stg_f64_policy(reinterpret_cast<double*>(ptr), static_cast<double>(v[e]), pol_stream);
        ptr += step;
        asm volatile("" : "+l"(ptr));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k = 12 fp32 specialisation (the n = 4096 headline): the CTA's 8 rows of A
// are parked in tensor memory (TMEM, 128 KiB of the SM's 256 KiB) once and
// re-read with tcgen05.ld for every basis, so the per-basis loop has no
// global loads; butterflies on register bits >= 1 use packed FADD2 / FFMA2
// (x - y as fma(y, -1, x), exactly rounded like the reference's x - y); the
// smem transpose uses 16-byte chunk-swizzled stores.
// Thread layout as in the generic kernel: E = 64, R = 8 rows, 512 threads.
// TMEM: warp w owns lanes 32*(w%4) .. +31 and columns 64*(w/4) .. +63.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_ld_x32(uint32_t taddr, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
        "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]), "=f"(v[16]),
        "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]),
        "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Butterflies over register-index bits [0, 6) of v[64], ascending; bit 0
// scalar, bits >= 1 as packed pairs (i, i+1) with FADD2 / FFMA2(-1).
__device__ __forceinline__ void reg_fwht64_packed(float (&v)[64]) {
#pragma unroll
  for (int i = 0; i < 64; i += 2) {
    const float a = v[i], b = v[i + 1];
    v[i] = a + b;
    v[i + 1] = a - b;
  }
#pragma unroll
  for (int hb = 1; hb < 6; ++hb) {
    const int h = 1 << hb;
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
      if ((i & h) == 0) {
        const float2 x = make_float2(v[i], v[i + 1]);
        const float2 y = make_float2(v[i + h], v[i + h + 1]);
        const float2 s = __fadd2_rn(x, y);
        const float2 d = __ffma2_rn(y, make_float2(-1.f, -1.f), x);
        v[i] = s.x;
        v[i + 1] = s.y;
        v[i + h] = d.x;
        v[i + h + 1] = d.y;
      }
    }
  }
}

__global__ void __launch_bounds__(512, 1) fwht12_tmem_kernel(const float* __restrict__ a, int64_t lda, int64_t m,
                                                             int64_t n, const uint32_t* __restrict__ qplain,
                                                             int64_t basis_begin, int64_t basis_end,
                                                             int bases_per_cta, float* __restrict__ cols,
                                                             int64_t ldc, int store_mode) {
  constexpr int E = 64, R = 8, RS = 4096 + 4, D = 4096, WPB = 128;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tile = reinterpret_cast<float*>(smem_raw);
  __shared__ uint32_t tmem_base_slot;

  const int tid = threadIdx.x, warp = tid / 32;
  const int64_t i0 = int64_t(blockIdx.x) * R;
  const int64_t s_first = basis_begin + int64_t(blockIdx.y) * bases_per_cta;
  const int64_t s_last = min(basis_end, s_first + bases_per_cta);

  const int r1 = tid / E, p1 = tid % E;
  const int64_t row1 = i0 + r1;
  const int r2 = tid % R, q2 = tid / R;
  const int64_t row2 = i0 + r2;

  // ---- TMEM: allocate 256 columns, park the A tile ----
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = tmem_base_slot + (static_cast<uint32_t>(32 * (warp % 4)) << 16) +
                         static_cast<uint32_t>(64 * (warp / 4));
  {
    float v[E];
    const int64_t pos0 = int64_t(p1) * E;
    if (row1 < m) {
      const float* arow = a + row1 * lda;
      if (pos0 + E <= n) {
#pragma unroll
        for (int e = 0; e < E; e += 4) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(arow + pos0 + e));
          v[e] = f.x;
          v[e + 1] = f.y;
          v[e + 2] = f.z;
          v[e + 3] = f.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = (pos0 + e < n) ? arow[pos0 + e] : 0.f;
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = 0.f;
    }
    tmem_st_x32(taddr, v);
    tmem_st_x32(taddr + 32, v + 32);
    tmem_wait_st();
  }

  // sign words of the next basis are prefetched one iteration ahead (L2 latency)
  uint32_t q0n = 0, q1n = 0;
  if (s_first < s_last) {
    q0n = __ldg(qplain + s_first * WPB + 2 * p1);
    q1n = __ldg(qplain + s_first * WPB + 2 * p1 + 1);
  }
  for (int64_t s = s_first; s < s_last; ++s) {
    float v[E];
    tmem_ld_x32(taddr, v);
    tmem_ld_x32(taddr + 32, v + 32);
    const uint32_t q0 = q0n, q1 = q1n;
    if (s + 1 < s_last) {
      q0n = __ldg(qplain + (s + 1) * WPB + 2 * p1);
      q1n = __ldg(qplain + (s + 1) * WPB + 2 * p1 + 1);
    }
    tmem_wait_ld();
    // sign mask (sketch.hpp:185): flip the sign bit where Q_s(pos) = 1 (exact)
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(__float_as_uint(v[e]) ^ ((q0 << (31 - e)) & 0x80000000u));
#pragma unroll
    for (int e = 0; e < 32; ++e)
      v[32 + e] = __uint_as_float(__float_as_uint(v[32 + e]) ^ ((q1 << (31 - e)) & 0x80000000u));
    if (store_mode < 2) reg_fwht64_packed(v);  // position bits 0..5 (store_mode 2: write-path experiment)
    __syncthreads();       // previous basis' phase-2 reads done
    {
      float* dst = tile + r1 * RS + p1 * E;
#pragma unroll
      for (int c = 0; c < 16; ++c)
        *reinterpret_cast<float4*>(dst + 4 * (c ^ (p1 & 15))) =
            make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
    __syncthreads();
    {
      const float* src = tile + r2 * RS + (q2 & 3);
      const int cq = q2 >> 2;
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = src[e * E + 4 * (cq ^ (e & 15))];
    }
    if (store_mode < 2) reg_fwht64_packed(v);  // position bits 6..11
    if (row2 < m) {
      // incremental addressing keeps 64 hoisted 64-bit offsets out of registers
      float* ptr = cols + (s * D + q2) * ldc + row2;
      const int64_t step = int64_t(E) * ldc;
      if (store_mode == 0) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          ptr[0] = v[e];  // default policy: L2 merges the 4 CTAs' 32-byte sectors of a line
          ptr += step;
          asm volatile("" : "+l"(ptr));
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          __stcs(ptr, v[e]);  // streaming store (evict-first)
          ptr += step;
          asm volatile("" : "+l"(ptr));
        }
      }
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base_slot) : "memory");
}

// ---------------------------------------------------------------------------
// k = 12 fp32, row-pair variant: 256 threads, 8 rows per CTA; thread (rp, p)
// owns rows (2rp, 2rp+1) x positions p*64 .. p*64+63 as 64 float2 pairs, so
// every butterfly stage is one FADD2 (x+y) + one FFMA2(y, -1, x) per pair
// butterfly on natural register pairs, the Kerdock sign mask is shared by the
// two rows, and the write-back is STG.64 (two consecutive rows of a column).
// smem tile: row-pair block rp at rp * RSP floats, pair of position pos at
// 2*pos, 16-byte chunk c of thread p stored at chunk c ^ (p & 7);
// RSP = 8192 + 8 makes both the STS.128 and the LDS.64 patterns conflict-free.
// TMEM: warp w owns lanes 32*(w%4) .. +31, columns 128*(w/4) .. +127.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1) fwht12_pairs_kernel(const float* __restrict__ a, int64_t lda, int64_t m,
                                                              int64_t n, const uint32_t* __restrict__ qplain,
                                                              int64_t basis_begin, int64_t basis_end,
                                                              int bases_per_cta, float* __restrict__ cols,
                                                              int64_t ldc) {
  constexpr int E = 64, D = 4096, WPB = 128, RSP = 8192 + 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tile = reinterpret_cast<float*>(smem_raw);
  __shared__ uint32_t tmem_base_slot;

  const int tid = threadIdx.x, warp = tid / 32;
  const int64_t i0 = int64_t(blockIdx.x) * 8;
  const int64_t s_first = basis_begin + int64_t(blockIdx.y) * bases_per_cta;
  const int64_t s_last = min(basis_end, s_first + bases_per_cta);

  const int rp = tid / E, p1 = tid % E;    // phase 1: row pair, position group
  const int rp2 = tid % 4, q2 = tid / 4;   // phase 2: row pair, position residue
  const int64_t row_a = i0 + 2 * rp, row2 = i0 + 2 * rp2;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = tmem_base_slot + (static_cast<uint32_t>(32 * (warp % 4)) << 16) +
                         static_cast<uint32_t>(128 * (warp / 4));
  {
    // park the two rows' 64 values as interleaved pairs (v[2e], v[2e+1]) = (row_a, row_a+1)
    float v[2 * E];
    const int64_t pos0 = int64_t(p1) * E;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int64_t row = row_a + r;
      if (row < m && pos0 + E <= n) {
        const float* arow = a + row * lda + pos0;
#pragma unroll
        for (int e = 0; e < E; e += 4) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(arow + e));
          v[2 * e + r] = f.x;
          v[2 * (e + 1) + r] = f.y;
          v[2 * (e + 2) + r] = f.z;
          v[2 * (e + 3) + r] = f.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[2 * e + r] = (row < m && pos0 + e < n) ? a[row * lda + pos0 + e] : 0.f;
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_st_x32(taddr + 32 * c, v + 32 * c);
    tmem_wait_st();
  }

  uint32_t q0n = 0, q1n = 0;
  if (s_first < s_last) {
    q0n = __ldg(qplain + s_first * WPB + 2 * p1);
    q1n = __ldg(qplain + s_first * WPB + 2 * p1 + 1);
  }
  for (int64_t s = s_first; s < s_last; ++s) {
    float2 V[E];
    {
      float* vf = reinterpret_cast<float*>(V);
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_x32(taddr + 32 * c, vf + 32 * c);
    }
    const uint32_t q0 = q0n, q1 = q1n;
    if (s + 1 < s_last) {
      q0n = __ldg(qplain + (s + 1) * WPB + 2 * p1);
      q1n = __ldg(qplain + (s + 1) * WPB + 2 * p1 + 1);
    }
    tmem_wait_ld();
    // Kerdock sign mask (sketch.hpp:185), shared by both rows of the pair
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t msk = ((e < 32 ? q0 : q1) << (31 - (e & 31))) & 0x80000000u;
      V[e].x = __uint_as_float(__float_as_uint(V[e].x) ^ msk);
      V[e].y = __uint_as_float(__float_as_uint(V[e].y) ^ msk);
    }
    // position bits 0..5 (h = 1 .. 32), reference stage order
#pragma unroll
    for (int hb = 0; hb < 6; ++hb) {
      const int h = 1 << hb;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if ((e & h) == 0) {
          const float2 x = V[e], y = V[e + h];
          V[e] = __fadd2_rn(x, y);
          V[e + h] = __ffma2_rn(y, make_float2(-1.f, -1.f), x);
        }
      }
    }
    __syncthreads();  // previous basis' phase-2 reads done
    {
      float* dst = tile + rp * RSP + p1 * (2 * E);
#pragma unroll
      for (int c = 0; c < 32; ++c)
        *reinterpret_cast<float4*>(dst + 4 * (c ^ (p1 & 7))) = make_float4(V[2 * c].x, V[2 * c].y, V[2 * c + 1].x,
                                                                          V[2 * c + 1].y);
    }
    __syncthreads();
    {
      const float* src = tile + rp2 * RSP + 2 * (q2 & 1);
      const int cq = q2 >> 1;
#pragma unroll
      for (int e = 0; e < E; ++e) V[e] = *reinterpret_cast<const float2*>(src + e * (2 * E) + 4 * (cq ^ (e & 7)));
    }
    // position bits 6..11 (h = 64 .. 2048)
#pragma unroll
    for (int hb = 0; hb < 6; ++hb) {
      const int h = 1 << hb;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if ((e & h) == 0) {
          const float2 x = V[e], y = V[e + h];
          V[e] = __fadd2_rn(x, y);
          V[e + h] = __ffma2_rn(y, make_float2(-1.f, -1.f), x);
        }
      }
    }
    // transposed write-back (sketch.hpp:191-196): column s*d + e*64 + q2, rows row2, row2+1
    if (row2 + 1 < m) {
      float* ptr = cols + (s * D + q2) * ldc + row2;
      const int64_t step = int64_t(E) * ldc;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        __stcs(reinterpret_cast<float2*>(ptr), V[e]);
        ptr += step;
        asm volatile("" : "+l"(ptr));
      }
    } else if (row2 < m) {
      float* ptr = cols + (s * D + q2) * ldc + row2;
      const int64_t step = int64_t(E) * ldc;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        __stcs(ptr, V[e].x);
        ptr += step;
        asm volatile("" : "+l"(ptr));
      }
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base_slot) : "memory");
}

// ---------------------------------------------------------------------------
// Identity block: column nk*d + w = sqrt(d) * A[:, w] for w < n, zero for
// n <= w < d. 32x32 tiles transposed through shared memory.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void identity_kernel(const T* __restrict__ a, int64_t lda, int64_t m, int64_t n, int64_t d,
                                int64_t nk, T sqrt_d, T* __restrict__ cols, int64_t ldc) {
  __shared__ T tile[32][33];
  const int64_t w0 = int64_t(blockIdx.x) * 32, i0 = int64_t(blockIdx.y) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = i0 + r, w = w0 + tx;
    tile[r][tx] = (i < m && w < n) ? sqrt_d * a[i * lda + w] : T(0);
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t w = w0 + r, i = i0 + tx;
    if (w < d && i < m) cols[(nk * d + w) * ldc + i] = tile[tx][r];
  }
}

// Per-row 2-norm in double (sketch.hpp:126-131), one warp per row.
template <typename T>
__global__ void row_norm_kernel(const T* __restrict__ a, int64_t lda, int64_t m, int64_t n, double* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= m) return;
  double acc = 0;
  for (int64_t j = lane; j < n; j += 32) {
    const double v = static_cast<double>(a[int64_t(warp) * lda + j]);
    acc += v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[warp] = sqrt(acc);
}

// ----------------------------------------------------------------- launch --
cudaError_t launch_qtables(const uint32_t* revtab, int k, int64_t nbases, uint32_t* qplain, uint32_t* qtrans,
                           cudaStream_t st) {
  const int64_t d = int64_t{1} << k;
  const int threads = 256;
  const int64_t cap = 148 * 64;
  int64_t total = nbases * (d >= 32 ? d / 32 : 1);
  int64_t blocks = (total + threads - 1) / threads;
  qtable_kernel<<<static_cast<unsigned>(blocks < cap ? blocks : cap), threads, 0, st>>>(revtab, k, nbases, qplain);
  if (qtrans != nullptr && d >= 128) {
    total = nbases * (d >= 1024 ? d / 1024 : 1) * 32;
    blocks = (total + threads - 1) / threads;
    qtrans_kernel<<<static_cast<unsigned>(blocks < cap ? blocks : cap), threads, 0, st>>>(revtab, k, nbases, qtrans);
  }
  return cudaGetLastError();
}

template <typename T, int KB>
static cudaError_t launch_fwht_k(const T* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                                 int64_t b0, int64_t b1, T* cols, int64_t ldc, cudaStream_t st) {
  constexpr int NT = (sizeof(T) == 8 && KB >= 12) ? 256 : ((KB >= 14) ? 256 : 512);
  using C = FwhtCfg<T, KB, NT>;
  static_assert(C::R >= 1, "rows per CTA");
  auto kern = fwht_sketch_kernel<T, KB, NT>;
  if (C::SMEM > 227 * 1024) return cudaErrorNotSupported;
  if (C::SMEM > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
  }
  const int64_t nb = b1 - b0;
  if (nb <= 0) return cudaSuccess;
  const int64_t row_tiles = (m + C::R - 1) / C::R;
  // Bases per CTA: enough CTAs for >= 4 waves, at most 16 bases each.
  int bpc = 16;
  while (bpc > 1 && row_tiles * ((nb + bpc - 1) / bpc) < 148 * 8) bpc /= 2;
  const int64_t gy = (nb + bpc - 1) / bpc;
  if (row_tiles > 0x7fffffff || gy > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid(static_cast<unsigned>(row_tiles), static_cast<unsigned>(gy));
  kern<<<grid, NT, C::SMEM, st>>>(a, lda, m, n, qplain, b0, b1, bpc, cols, ldc);
  return cudaGetLastError();
}

static cudaError_t launch_fwht12_tmem(const float* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                                      int64_t b0, int64_t b1, float* cols, int64_t ldc, cudaStream_t st) {
  constexpr size_t smem = size_t(8) * (4096 + 4) * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(fwht12_tmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const int64_t nb = b1 - b0;
  if (nb <= 0) return cudaSuccess;
  const int64_t row_tiles = (m + 7) / 8;
  int bpc = 32;
  if (const char* b = std::getenv("FSTG_FWHT_BPC")) bpc = std::max(1, std::atoi(b));  // A/B experiments only
  while (bpc > 1 && row_tiles * ((nb + bpc - 1) / bpc) < 148 * 8) bpc /= 2;
  const int64_t gy = (nb + bpc - 1) / bpc;
  if (row_tiles > 0x7fffffff || gy > 65535) return cudaErrorInvalidConfiguration;
  const char* sm = std::getenv("FSTG_FWHT_STORE");  // A/B experiments only
  const int store_mode = (sm && std::string(sm) == "cs") ? 1 : (sm && std::string(sm) == "nofwht") ? 2 : 0;
  fwht12_tmem_kernel<<<dim3(static_cast<unsigned>(row_tiles), static_cast<unsigned>(gy)), 512, smem, st>>>(
      a, lda, m, n, qplain, b0, b1, bpc, cols, ldc, store_mode);
  return cudaGetLastError();
}

static cudaError_t launch_fwht12_pairs(const float* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                                       int64_t b0, int64_t b1, float* cols, int64_t ldc, cudaStream_t st) {
  constexpr size_t smem = size_t(4) * (8192 + 8) * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(fwht12_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const int64_t nb = b1 - b0;
  if (nb <= 0) return cudaSuccess;
  const int64_t row_tiles = (m + 7) / 8;
  int bpc = 32;
  while (bpc > 1 && row_tiles * ((nb + bpc - 1) / bpc) < 148 * 8) bpc /= 2;
  const int64_t gy = (nb + bpc - 1) / bpc;
  if (row_tiles > 0x7fffffff || gy > 65535) return cudaErrorInvalidConfiguration;
  fwht12_pairs_kernel<<<dim3(static_cast<unsigned>(row_tiles), static_cast<unsigned>(gy)), 256, smem, st>>>(
      a, lda, m, n, qplain, b0, b1, bpc, cols, ldc);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fwht_sketch(int k, const T* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                               int64_t b0, int64_t b1, T* cols, int64_t ldc, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    if (k == 12 && (lda % 4) == 0) {
      const char* var = std::getenv("FSTG_FWHT_VARIANT");  // A/B experiments only
      if (var && std::string(var) == "pairs") return launch_fwht12_pairs(a, lda, m, n, qplain, b0, b1, cols, ldc, st);
      return launch_fwht12_tmem(a, lda, m, n, qplain, b0, b1, cols, ldc, st);
    }
  }
  switch (k) {
    case 2: return launch_fwht_k<T, 2>(a, lda, m, n, qplain, b0, b1, cols, ldc, st);
    case 4: return launch_fwht_k<T, 4>(a, lda, m, n, qplain, b0, b1, cols, ldc, st);
    case 6: return launch_fwht_k<T, 6>(a, lda, m, n, qplain, b0, b1, cols, ldc, st);
    case 8: return launch_fwht_k<T, 8>(a, lda, m, n, qplain, b0, b1, cols, ldc, st);
    case 10: return launch_fwht_k<T, 10>(a, lda, m, n, qplain, b0, b1, cols, ldc, st);
    case 12: return launch_fwht_k<T, 12>(a, lda, m, n, qplain, b0, b1, cols, ldc, st);
    case 14: return launch_fwht_k<T, 14>(a, lda, m, n, qplain, b0, b1, cols, ldc, st);
    default: return cudaErrorNotSupported;
  }
}

template <typename T>
cudaError_t launch_identity(const T* a, int64_t lda, int64_t m, int64_t n, int64_t d, int64_t nk, T* cols,
                            int64_t ldc, cudaStream_t st) {
  const T sqrt_d = static_cast<T>(sqrt(static_cast<double>(d)));
  dim3 grid(static_cast<unsigned>((d + 31) / 32), static_cast<unsigned>((m + 31) / 32));
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  identity_kernel<T><<<grid, dim3(32, 8), 0, st>>>(a, lda, m, n, d, nk, sqrt_d, cols, ldc);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_row_norms(const T* a, int64_t lda, int64_t m, int64_t n, double* out, cudaStream_t st) {
  const int threads = 256;
  const int64_t blocks = (m * 32 + threads - 1) / threads;
  row_norm_kernel<T><<<static_cast<unsigned>(blocks), threads, 0, st>>>(a, lda, m, n, out);
  return cudaGetLastError();
}

template cudaError_t launch_fwht_sketch<float>(int, const float*, int64_t, int64_t, int64_t, const uint32_t*,
                                               int64_t, int64_t, float*, int64_t, cudaStream_t);
template cudaError_t launch_fwht_sketch<double>(int, const double*, int64_t, int64_t, int64_t, const uint32_t*,
                                                int64_t, int64_t, double*, int64_t, cudaStream_t);
template cudaError_t launch_identity<float>(const float*, int64_t, int64_t, int64_t, int64_t, int64_t, float*,
                                            int64_t, cudaStream_t);
template cudaError_t launch_identity<double>(const double*, int64_t, int64_t, int64_t, int64_t, int64_t, double*,
                                             int64_t, cudaStream_t);
template cudaError_t launch_row_norms<float>(const float*, int64_t, int64_t, int64_t, double*, cudaStream_t);
template cudaError_t launch_row_norms<double>(const double*, int64_t, int64_t, int64_t, double*, cudaStream_t);

}  // namespace fstg
