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
//  * fwht_tmem_kernel<k> — the fp32 k = 12 / 14 path of the same computation:
//                      the CTA's A rows are parked in TMEM (tcgen05.st once,
//                      tcgen05.ld per basis) and the next basis' sign words are
//                      prefetched; RETAIN mode walks only bases holding a
//                      requested column and keeps just those (fstg_sample_columns,
//                      rows [row0, m) for the row-blocked design transform).
//  * fwht12_sketch_ws_kernel — the k = 12 full-sketch build (config 3) with
//                      store warps: butterfly warps park their results in
//                      the free half of tensor memory and a fifth warpgroup
//                      issues the scattered column stores; 2-CTA clusters
//                      start each basis' stores together.
//  * fwht14_retain_ws_kernel — the k = 14 RETAIN pass (config 4) with warp
//                      specialisation: two butterfly warpgroups + a copy
//                      warpgroup that also evaluates the last two stages for
//                      the requested positions (setmaxnreg), and the retained values of a 4-CTA
//                      cluster's rows merged into 16-byte column segments
//                      through distributed shared memory (st.async).
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

// fp32: stage h = 1 scalar, stages h >= 2 as packed pairs (i, i+1) with FADD2
// (x + y) and FFMA2(y, -1, x) (x - y, one rounding) — same values as scalar.
template <int HALF>
__device__ __forceinline__ void reg_fwht_f32_packed(float (&v)[1 << HALF]) {
  constexpr int E = 1 << HALF;
#pragma unroll
  for (int i = 0; i < E; i += 2) bfly(v[i], v[i + 1]);
#pragma unroll
  for (int hb = 1; hb < HALF; ++hb) {
    const int h = 1 << hb;
#pragma unroll
    for (int i = 0; i < E; i += 2) {
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

template <typename T, int HALF>
__device__ __forceinline__ void reg_fwht_any(T (&v)[1 << HALF]) {
  if constexpr (sizeof(T) == 4 && HALF >= 2)
    reg_fwht_f32_packed<HALF>(v);
  else
    reg_fwht<T, HALF>(v);
}

// RETAIN = false: write every column s*d + w (the full sketch).
// RETAIN = true (retain-sampled, SURVEY.md §8(e) for n = 16384): only the
// requested columns are kept — requests sorted by ell, basis s owning
// [req_start[s], req_start[s+1]); request r writes column ell_r into slot
// req_pos[r] of `cols` (stride ldc), i.e. the draw_and_gather buffer
// (stream.hpp:184-191). Bases without requests are skipped.
template <typename T, int KB, int NT, bool RETAIN>
__global__ void __launch_bounds__(NT) fwht_sketch_kernel(const T* __restrict__ a, int64_t lda, int64_t m, int64_t n,
                                                         const uint32_t* __restrict__ qplain, int64_t basis_begin,
                                                         int64_t basis_end, int bases_per_cta, T* __restrict__ cols,
                                                         int64_t ldc, const int64_t* __restrict__ req_start,
                                                         const int64_t* __restrict__ req_ell,
                                                         const int64_t* __restrict__ req_pos, int64_t row0) {
  using C = FwhtCfg<T, KB, NT>;
  constexpr int E = C::E, R = C::R, RS = C::RS, D = C::D, SW = C::SW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);

  const int tid = threadIdx.x;
  const int64_t i0 = row0 + int64_t(blockIdx.x) * R;  // rows [row0, m): retain-sampled row blocks
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
  // Small rows (E * sizeof(T) <= 128 B per thread: fp32 k <= 10, fp64 k <= 8): the thread's E
  // values of A are loaded once and kept in registers for all of the CTA's bases, so the basis
  // loop issues no global loads (config 2: the per-basis L2 reloads left it latency-bound).
  constexpr bool CACHE_A = E * sizeof(T) <= 128;
  T areg[CACHE_A ? E : 1];
  auto load_row = [&](T (&dst)[E]) {
    if (row1 < m) {
      const T* arow = a + row1 * lda;
      const int64_t pos0 = int64_t(p1) * E;
      if (pos0 + E <= n && (reinterpret_cast<uintptr_t>(arow + pos0) % 16) == 0) {
        if constexpr (sizeof(T) == 4) {
#pragma unroll
          for (int e = 0; e < E; e += 4) {
            const float4 f = ldg_f4_policy(reinterpret_cast<const float4*>(arow + pos0 + e), pol_keep);
            dst[e] = f.x;
            dst[e + 1] = f.y;
            dst[e + 2] = f.z;
            dst[e + 3] = f.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; e += 2) {
            const double2 f = ldg_d2_policy(reinterpret_cast<const double2*>(arow + pos0 + e), pol_keep);
            dst[e] = f.x;
            dst[e + 1] = f.y;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) dst[e] = (pos0 + e < n) ? arow[pos0 + e] : T(0);
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) dst[e] = T(0);
    }
  };
  if constexpr (CACHE_A) load_row(areg);

  for (int64_t s = s_first; s < s_last; ++s) {
    if constexpr (RETAIN) {
      if (req_start[s] == req_start[s + 1]) continue;  // no sample in this basis (uniform per CTA)
    }
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
    if constexpr (CACHE_A) {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = areg[e];
    } else {
      load_row(v);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t bit = (qw[e / 32] >> (e % 32)) & 1u;
      v[e] = bit ? -v[e] : v[e];  // sign[j] * a_ij with sign = +-1 (exact)
    }
    // ---- stages h = 1 .. E/2 in registers ----
    reg_fwht_any<T, C::HALF>(v);
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
    reg_fwht_any<T, C::HALF>(v);
    if constexpr (RETAIN) {
      // stage the R x D result as [w][r] in the (now free) tile, then copy the
      // requested columns' R-row segments to their slots.
      __syncthreads();
#pragma unroll
      for (int e = 0; e < E; ++e) tile[(int64_t(e) * E + q2) * R + r2] = v[e];
      __syncthreads();
      const int64_t r_lo = req_start[s], r_hi = req_start[s + 1];
      for (int64_t it = tid; it < (r_hi - r_lo) * R; it += NT) {
        const int64_t r = r_lo + it / R;
        const int rr = static_cast<int>(it % R);
        const int64_t w = req_ell[r] - s * D;
        if (i0 + rr < m) cols[req_pos[r] * ldc + (i0 - row0) + rr] = tile[w * R + rr];
      }
      continue;  // the next basis' first __syncthreads orders the tile reuse
    }
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
// fp32 TMEM-resident FWHT for k = 12 (n = 4096 headline) and k = 14 (n = 16384):
// the CTA's R rows of A are parked in tensor memory once (tcgen05.st; 128 KiB
// of the SM's 256 KiB) and re-read with tcgen05.ld for every basis, so the
// per-basis loop issues no global loads (at k = 14 A is 1 GiB and would
// otherwise be re-read from HBM for every basis). Butterflies on register bits
// >= 1 are packed FADD2 / FFMA2(y, -1, x) (exactly rounded x - y); the smem
// transpose uses 16-byte chunk swizzling (conflict-free both ways).
//   k = 12: E = 64 elements/thread, R = 8 rows, 512 threads.
//   k = 14: E = 128, R = 2 rows, 256 threads.
// TMEM: warp w owns lanes 32*(w%4) .. +31 and columns E*(w/4) .. +E-1.
// RETAIN: keep only requested columns (see fwht_sketch_kernel).
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

__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
        "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr)
      : "memory");
}

// 8-byte cp.async (LDGSTS) for the request-record prefetch
__device__ __forceinline__ void cp_async_8(void* dst_smem, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Distributed shared memory (thread-block cluster) helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Cluster hand-over without cluster-scope fences (a release / acquire at
// cluster scope compiles to MEMBAR.ALL.GPU / CCTL.IVALL, which drain this
// SM's outstanding global stores): data moves with st.async (completes bytes
// on the receiver's mbarrier), slots are released with relaxed remote arrivals.
__device__ __forceinline__ void st_async_f32(uint32_t local_dst, float v, uint32_t rank, uint32_t local_bar) {
  asm volatile(
      "{\n\t.reg .b32 rd, rb;\n\t"
      "mapa.shared::cluster.u32 rd, %0, %2;\n\t"
      "mapa.shared::cluster.u32 rb, %3, %2;\n\t"
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [rd], %1, [rb];\n\t}" ::"r"(local_dst),
      "f"(v), "r"(rank), "r"(local_bar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t local_bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(local_bar),
      "r"(rank)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cta(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void stg_f32x4(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int KB>
struct TmemCfg {
  static constexpr int HALF = KB / 2;
  static constexpr int E = 1 << HALF;
  static constexpr int D = 1 << KB;
  // k = 14: one row per CTA (128 threads, 65 KiB tile) so two CTAs share an SM and
  // overlap each other's transpose barriers (register-limited to 2 x 128 x 256).
#ifndef FSTG_K14_NT
#define FSTG_K14_NT 128
#endif
  static constexpr int NT = (KB == 12) ? 512 : FSTG_K14_NT;
  static constexpr int MIN_CTAS = (KB == 12 || NT > 128) ? 1 : 2;
  static constexpr int R = NT / E;
  static constexpr int TCOLS = E * ((NT / 32 + 3) / 4);  // TMEM columns: E per warp, 4 warps share a column range
  static constexpr int RS = D + 32 / R;          // row stride (floats): phase-2 reads conflict-free
  static constexpr int WPT = E / 32;             // sign words per thread
  static constexpr int CH = E / 4;               // 16-byte chunks per thread
  static constexpr int SWC = CH - 1;             // chunk swizzle mask
  static constexpr size_t SMEM = size_t(R) * RS * sizeof(float);
  static constexpr int RCAP = 1024;              // RETAIN: request records per basis held in shared memory
  static constexpr int MAXBPC = 256;             // RETAIN: bases per CTA (request ranges cached in shared memory)
};

// CL > 1 (k = 14 RETAIN, one row per CTA): the CL CTAs of a cluster hold CL
// consecutive rows and walk the same bases; every CTA writes 1/CL of the
// requests as CL-row column segments (two lanes x 16-byte stores per request)
// assembled in its shared receive ring through distributed shared memory — full 32-byte
// sectors instead of one scattered 4-byte store per request and row. Each CTA
// pushes its row's value of request j with st.async into CTA j % CL's receive
// slot (bytes complete on that CTA's full barrier); reader warps release a slot
// with relaxed remote arrivals on every writer's empty barrier. No cluster-wide
// barrier per basis: a CTA may run up to SS - 1 slots ahead of its slowest peer.
template <int KB, bool RETAIN, int CL = 1>
__global__ void __launch_bounds__(TmemCfg<KB>::NT, TmemCfg<KB>::MIN_CTAS) fwht_tmem_kernel(
    const float* __restrict__ a, int64_t lda, int64_t m, int64_t n, const uint32_t* __restrict__ qplain,
    int64_t basis_begin, int64_t basis_end, int bases_per_cta, float* __restrict__ cols, int64_t ldc,
    const int64_t* __restrict__ req_start, const int64_t* __restrict__ req_ell, const int64_t* __restrict__ req_pos,
    int64_t row0, const uint2* __restrict__ req_rec) {
  static_assert(CL == 1 || (RETAIN && (CL == 4 || CL == 8) && TmemCfg<KB>::R == 1),
                "cluster merge: one row per CTA, 4 or 8 CTAs");
  constexpr bool kMerge = CL > 1;
  using C = TmemCfg<KB>;
  constexpr int E = C::E, R = C::R, RS = C::RS, D = C::D, NT = C::NT, WPT = C::WPT, CH = C::CH, SWC = C::SWC;
  constexpr int WPB = D / 32, RCAP = C::RCAP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tile = reinterpret_cast<float*>(smem_raw);
  __shared__ uint32_t tmem_base_slot;
  // RETAIN: (w, slot) records of the current / next visited basis (double buffer,
  // filled by cp.async one basis ahead so the copy loop reads no global memory)
  __shared__ __align__(16) uint2 reqbuf[RETAIN ? 2 * RCAP : 2];
  // RETAIN: req_start[s_first .. s_last] (the CTA's request ranges; read every basis)
  __shared__ int64_t rstart[RETAIN ? C::MAXBPC + 1 : 1];
  // CL > 1: receive ring (SS slots of [request][row] values pushed by the cluster's CTAs) and its barriers
  constexpr int SS = 4, NW = NT / 32;
  __shared__ __align__(16) float recv[CL > 1 ? SS * RCAP : 1];
  __shared__ __align__(8) uint64_t full_bar[CL > 1 ? SS : 1], empty_bar[CL > 1 ? SS : 1];
  __shared__ uint32_t rslot[CL > 1 ? SS * (RCAP / CL) : 1];  // output slot of each received request
  __shared__ int rmine[CL > 1 ? SS : 1];                     // received requests per slot use
  constexpr uint32_t DL = 2;  // uses between a push and its write-back (< SS; 3 measured the same)

  const int tid = threadIdx.x, warp = tid / 32;
  const int64_t i0 = row0 + int64_t(blockIdx.x) * R;  // rows [row0, m): retain-sampled row blocks
  const int64_t s_first = basis_begin + int64_t(blockIdx.y) * bases_per_cta;
  const int64_t s_last = min(basis_end, s_first + bases_per_cta);
  const int r1 = tid / E, p1 = tid % E;
  const int64_t row1 = i0 + r1;
  const int r2 = tid % R, q2 = tid / R;
  const int64_t row2 = i0 + r2;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_slot)),
                 "n"(C::TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = tmem_base_slot + (static_cast<uint32_t>(32 * (warp % 4)) << 16) +
                         static_cast<uint32_t>(E * (warp / 4));
  {
    float v[E];
    const int64_t pos0 = int64_t(p1) * E;
    if (row1 < m && pos0 + E <= n) {
      const float* arow = a + row1 * lda;
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
      for (int e = 0; e < E; ++e) v[e] = (row1 < m && pos0 + e < n) ? a[row1 * lda + pos0 + e] : 0.f;
    }
#pragma unroll
    for (int c = 0; c < E / 32; ++c) tmem_st_x32(taddr + 32 * c, v + 32 * c);
    tmem_wait_st();
  }

  if constexpr (RETAIN) {
    for (int64_t j = tid; j <= s_last - s_first; j += NT) rstart[j] = req_start[s_first + j];
    __syncthreads();
  }
  if constexpr (kMerge) {
    if (tid == 0) {
      for (int i = 0; i < SS; ++i) {
        mbar_init(&full_bar[i], 1);          // this CTA's expect_tx arrival + the pushed bytes
        mbar_init(&empty_bar[i], CL * NW);   // every reader warp of the cluster
      }
      fence_mbar_init();
    }
    cluster_sync_all();  // every peer's barriers are initialised before any remote arrive
  }
  auto rs = [&](int64_t sb) { return rstart[sb - s_first]; };  // req_start[sb], sb in [s_first, s_last]
  // staged transform value at position w of row rr (layouts written after phase 2)
  auto staged = [&](uint32_t w, int rr) -> float { return tile[w * R + rr]; };
  // RETAIN visits only bases holding a requested column (uniform per CTA)
  auto next_basis = [&](int64_t s) {
    if constexpr (RETAIN) {
      while (s < s_last && rs(s) == rs(s + 1)) ++s;
    }
    return s;
  };
  // request records of basis sb into reqbuf[buf] (one commit group per call, possibly empty)
  auto prefetch_req = [&](int64_t sb, int buf) {
    if constexpr (RETAIN) {
      if (sb < s_last) {
        const int64_t lo = rs(sb), cnt = rs(sb + 1) - lo;
        if (cnt <= RCAP)
          for (int j = tid; j < cnt; j += NT) cp_async_8(&reqbuf[buf * RCAP + j], req_rec + lo + j);
      }
      cp_async_commit();
    }
  };
  const uint32_t crank = CL > 1 ? cluster_ctarank() : 0;
  const int64_t cbase = i0 - crank;  // CL > 1: the cluster's first row
  // CL > 1: write back use ud of the receive ring (CL-row segments of this CTA's
  // requests), then release the slot to every writer in the cluster
  auto drain_use = [&](uint32_t ud) {
    if constexpr (kMerge) {
      const int slot = static_cast<int>(ud % SS);
      mbar_wait(&full_bar[slot], (ud / SS) & 1);  // all CL rows of this use landed
      const float* const rv = recv + slot * RCAP;
      const uint32_t* const rsl = rslot + slot * (RCAP / CL);
      float* const cout = cols + (cbase - row0);
      constexpr int QD = CL / 4;  // 4-row quads (16-byte stores) per request
      const int mine = rmine[slot];
      for (int t = tid; t < QD * mine; t += NT) {
        const int jj = t / QD, h = t % QD;
        const float4 val = *reinterpret_cast<const float4*>(rv + jj * CL + 4 * h);
        float* dst = cout + int64_t(rsl[jj]) * ldc + 4 * h;
        const int64_t r4 = cbase + 4 * h;
        if (r4 + 3 < m) {
          stg_f32x4(dst, val);
        } else {
          if (r4 + 0 < m) dst[0] = val.x;
          if (r4 + 1 < m) dst[1] = val.y;
          if (r4 + 2 < m) dst[2] = val.z;
        }
      }
      __syncwarp();
      if ((tid & 31) == 0)  // this warp's reads of the slot are done: release it to every writer
        for (int r = 0; r < CL; ++r) mbar_arrive_remote_relaxed(smem_u32(&empty_bar[slot]), r);
    }
  };
  // sign words of the next visited basis are prefetched one iteration ahead (L2 latency)
  int64_t s = next_basis(s_first);
  uint32_t qn[WPT];
#pragma unroll
  for (int w = 0; w < WPT; ++w) qn[w] = (s < s_last) ? __ldg(qplain + s * WPB + WPT * p1 + w) : 0u;
  int buf = 0;
  uint32_t use = 0;  // CL > 1: staging-slot uses so far (uniform across the cluster)
  (void)use;
  if (req_rec != nullptr) prefetch_req(s, 0);
  while (s < s_last) {
    const int64_t s_next = next_basis(s + 1);
    float v[E];
#pragma unroll
    for (int c = 0; c < E / 32; ++c) tmem_ld_x32(taddr + 32 * c, v + 32 * c);
    uint32_t q[WPT];
#pragma unroll
    for (int w = 0; w < WPT; ++w) q[w] = qn[w];
    if (s_next < s_last) {
#pragma unroll
      for (int w = 0; w < WPT; ++w) qn[w] = __ldg(qplain + s_next * WPB + WPT * p1 + w);
    }
    tmem_wait_ld();
    // Kerdock sign mask (sketch.hpp:185): flip the sign bit where Q_s(pos) = 1 (exact)
#pragma unroll
    for (int e = 0; e < E; ++e)
      v[e] = __uint_as_float(__float_as_uint(v[e]) ^ ((q[e / 32] << (31 - (e % 32))) & 0x80000000u));
    reg_fwht_f32_packed<C::HALF>(v);  // position bits 0 .. HALF-1
    __syncthreads();                  // previous basis' tile reads done
    if (RETAIN && req_rec != nullptr) prefetch_req(s_next, buf ^ 1);  // its buffer's readers are past the barrier
    {
      float* dst = tile + r1 * RS + p1 * E;
#pragma unroll
      for (int c = 0; c < CH; ++c)
        *reinterpret_cast<float4*>(dst + 4 * (c ^ (p1 & SWC))) =
            make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
    __syncthreads();
    {
      const float* src = tile + r2 * RS + (q2 & 3);
      const int cq = q2 >> 2;
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = src[e * E + 4 * (cq ^ (e & SWC))];
    }
    reg_fwht_f32_packed<C::HALF>(v);  // position bits HALF .. KB-1
    if constexpr (RETAIN) {
      __syncthreads();
#pragma unroll
      // (a thread-contiguous 16-byte-swizzled layout with 32 STS.128 measured 5% slower)
#pragma unroll
      for (int e = 0; e < E; ++e) tile[(int64_t(e) * E + q2) * R + r2] = v[e];
      if (req_rec != nullptr) cp_async_wait_1();  // this basis' records landed (the next basis' may be in flight)
      __syncthreads();
      const int64_t r_lo = rs(s), r_hi = rs(s + 1);
      float* const out = cols + (i0 - row0);
      if constexpr (kMerge) {
        // req_rec is non-null on this path (host); records from shared memory when they fit
        const int cnt = static_cast<int>(r_hi - r_lo);
        const uint2* recs = cnt <= RCAP ? reqbuf + buf * RCAP : req_rec + r_lo;
        for (int c0 = 0; c0 < cnt; c0 += RCAP) {
          const int nc = min(RCAP, cnt - c0);
          const int slot = static_cast<int>(use % SS);
          const uint32_t round = use / SS;
          // this CTA receives requests j = crank (mod CL) of the chunk: CL row values each
          const int mine = (nc - static_cast<int>(crank) + CL - 1) / CL;
          if (tid == 0) {
            mbar_arrive_expect_tx_cta(&full_bar[slot], static_cast<uint32_t>(4 * CL * mine));
            rmine[slot] = mine;
          }
          for (int jj = tid; jj < mine; jj += NT) rslot[slot * (RCAP / CL) + jj] = recs[c0 + jj * CL + static_cast<int>(crank)].y;
          // every reader has released this slot's previous round (its warps arrived here)
          if (round >= 1) mbar_wait(&empty_bar[slot], (round - 1) & 1);
          // push: value of request j (this CTA's row) -> reader j % CL, slot entry (j / CL, row crank)
          const uint32_t rbase = smem_u32(recv + slot * RCAP) + 4u * crank, fbar = smem_u32(&full_bar[slot]);
          constexpr int U = 8;  // batches: all shared-memory reads first, then the pushes
          for (int j0 = tid; j0 < nc; j0 += U * NT) {
            float val[U];
#pragma unroll
            for (int u = 0; u < U; ++u) val[u] = staged(recs[c0 + min(j0 + u * NT, nc - 1)].x, 0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int j = j0 + u * NT;
              if (j < nc)
                st_async_f32(rbase + 4u * static_cast<uint32_t>((j / CL) * CL), val[u], static_cast<uint32_t>(j % CL),
                             fbar);
            }
          }
          ++use;
          if (use > DL) drain_use(use - 1 - DL);  // write back an older use: its peers are most likely done
          if (c0 + RCAP < cnt) __syncthreads();   // next chunk reuses rslot / rmine entries (uniform)
        }
      } else if (req_rec != nullptr && r_hi - r_lo <= RCAP) {
        // batches of U items: all shared-memory reads first, then the stores
        constexpr int U = 8;
        const uint2* rb = reqbuf + buf * RCAP;
        const int nit = static_cast<int>(r_hi - r_lo) * R;
        for (int it0 = tid; it0 < nit; it0 += U * NT) {
          uint32_t slot[U];
          float val[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int it = it0 + u * NT;
            const uint2 rec = rb[min(it, nit - 1) / R];
            slot[u] = rec.y;
            val[u] = staged(rec.x, it % R);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int it = it0 + u * NT, rr = it % R;
            if (it < nit && i0 + rr < m) out[int64_t(slot[u]) * ldc + rr] = val[u];
          }
        }
      } else {
        for (int64_t it = tid; it < (r_hi - r_lo) * R; it += NT) {
          const int64_t r = r_lo + it / R;
          const int rr = static_cast<int>(it % R);
          const int64_t w = req_ell[r] - s * D;
          if (i0 + rr < m) out[req_pos[r] * ldc + rr] = staged(static_cast<uint32_t>(w), rr);
        }
      }
      buf ^= 1;
    } else if (row2 < m) {
      // transposed write-back (sketch.hpp:191-196): column s*d + e*E + q2, row row2
      float* ptr = cols + (s * D + q2) * ldc + row2;
      const int64_t step = int64_t(E) * ldc;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        ptr[0] = v[e];
        ptr += step;
        asm volatile("" : "+l"(ptr));
      }
    }
    s = s_next;
  }

  if constexpr (kMerge) {
    __syncthreads();  // the last pushes' rslot / rmine entries are visible to every thread
    for (uint32_t u = use > DL ? use - DL : 0; u < use; ++u) drain_use(u);
    // peers may still read this CTA's slots: wait for the last use of each slot to be released
    for (uint32_t u = use > SS ? use - SS : 0; u < use; ++u) mbar_wait(&empty_bar[u % SS], (u / SS) & 1);
    cluster_sync_all();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_slot), "n"(C::TCOLS) : "memory");
}

// ---------------------------------------------------------------------------
// Warp-specialised k = 14 retain kernel (config 4): the cluster-merged
// write-back of fwht_tmem_kernel<14, true, CL>, with the request handling moved
// off the butterfly warps. 384 threads per CTA, one row, CL-CTA clusters, two
// CTAs per SM:
//   warpgroups 0-1 (256 threads x 64 values, setmaxnreg 96): TMEM row -> sign
//     mask -> position bits 0-5 in registers -> swizzled shared transpose
//     (each 64-thread quarter of the row transposes on its own: barriers 5-8)
//     -> bits 6-11 in registers -> staged in place (each thread rewrites the
//     tile words it read, so no barrier before it);
//   warpgroup 2 (setmaxnreg 48): record prefetch (cp.async), the last two
//     stages (bits 12, 13) for the requested positions only, st.async pushes
//     of those values to the cluster, deferred 16-byte write-back of the
//     receive ring:
//       out(w) = (S0 +- S1) +- (S2 +- S3), S_h = staged[h * 4096 + (w & 4095)],
//     inner sign = bit 12 of w, outer sign = bit 13 — the same additions in
//     the same order as stages h = 4096, 8192 of fwht_unnormalized
//     (fwht.hpp:20-29), so every retained value is bit-identical to the full
//     transform's.
// Hand-over per basis with named barriers: STAGED (id 1: butterfly warps
// arrive, copy warps sync) and FREED (id 2: copy warps arrive once they hold
// their requested values in registers, butterfly warps sync before the next
// transpose overwrites the tile); the copy warpgroup's internal barrier is
// id 4. The copy of basis s overlaps the butterflies of basis s + 1.
// (Round 2 measured the previous shape — 128 butterfly threads x 128 values,
// all 14 stages — within 1% of this one, and five ways of overlapping its
// phases without gain: profiles/r02_k14_retain.txt.)
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

#ifdef FSTG_WS_PROF  // experiments: per-phase cycle counts of one butterfly / copy thread per CTA (tools/prof_k14.py)
__device__ unsigned long long g_wsprof[16];
__device__ __forceinline__ long long ws_clock() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  return t;
}
#define WS_PROF_BEGIN() long long wsacc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, wst = ws_clock()
#define WS_T(i)                         \
  do {                                  \
    const long long tn_ = ws_clock();   \
    wsacc[i] += tn_ - wst;              \
    wst = tn_;                          \
  } while (0)
#define WS_PROF_END(base)                                                                              \
  do {                                                                                                 \
    if (t0 == 0)                                                                                       \
      for (int i = 0; i < 8; ++i) atomicAdd(&g_wsprof[(base) + i], static_cast<unsigned long long>(wsacc[i])); \
  } while (0)
#else
#define WS_PROF_BEGIN() do { } while (0)
#define WS_T(i) do { } while (0)
#define WS_PROF_END(base) do { } while (0)
#endif
// receive-ring depth (4 and 6 slots measured the same, profiles/r01_k14_retain.txt)
constexpr int kWsSlots = 4;
constexpr size_t kWsRecvBytes = size_t(kWsSlots) * TmemCfg<14>::RCAP * sizeof(float);

template <int CL>
__global__ void __launch_bounds__(384, 2) fwht14_retain_ws_kernel(
    const float* __restrict__ a, int64_t lda, int64_t m, int64_t n, const uint32_t* __restrict__ qplain,
    int64_t basis_end, int bases_per_cta, float* __restrict__ cols, int64_t ldc, const int64_t* __restrict__ req_start,
    const uint2* __restrict__ req_rec, int64_t row0) {
  using C = TmemCfg<14>;
  constexpr int E = 64, HALF = 6, D = C::D, WPT = E / 32, CH = E / 4, SWC = CH - 1, TCOLS = 128;
  constexpr int WPB = D / 32, RCAP = C::RCAP, SS = kWsSlots, NW1 = 4, NB = 256, NALL = 384;
  constexpr uint32_t DL = 2;
  static_assert(DL < SS && (CL == 4 || CL == 8), "write-back lag below the ring depth; 4- or 8-CTA clusters");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tile = reinterpret_cast<float*>(smem_raw);
  __shared__ uint32_t tmem_base_slot;
  __shared__ __align__(16) uint2 reqbuf[2 * RCAP];
  __shared__ int64_t rstart[C::MAXBPC + 1];
  float* const recv = tile + C::SMEM / sizeof(float);  // receive ring: dynamic, after the tile
  __shared__ __align__(8) uint64_t full_bar[SS], empty_bar[SS];
  __shared__ uint32_t rslot[SS * (RCAP / CL)];
  __shared__ int rmine[SS];

  const int tid = threadIdx.x, warp = tid / 32;
  const bool bfly = __shfl_sync(0xffffffffu, tid / 128, 0) < 2;  // warp-uniform by construction (setmaxnreg regions)
  const int64_t i0 = row0 + int64_t(blockIdx.x);
  const int64_t s_first = int64_t(blockIdx.y) * bases_per_cta;
  const int64_t s_last = min(basis_end, s_first + bases_per_cta);
  const uint32_t crank = cluster_ctarank();
  const int64_t cbase = i0 - crank;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_slot)),
                 "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int64_t j = tid; j <= s_last - s_first; j += NALL) rstart[j] = req_start[s_first + j];
  if (tid == 0) {
    for (int i = 0; i < SS; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], CL * NW1);
    }
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  cluster_sync_all();  // peers' barriers initialised before any remote arrive

  auto rs = [&](int64_t sb) { return rstart[sb - s_first]; };
  auto next_basis = [&](int64_t sb) {
    while (sb < s_last && rs(sb) == rs(sb + 1)) ++sb;
    return sb;
  };

  if (bfly) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 96;" ::: "memory");  // 256 x 96 + 128 x 48 = 384 x 80
    const uint32_t taddr = tmem_base_slot + (static_cast<uint32_t>(32 * (warp % 4)) << 16) +
                           static_cast<uint32_t>(E * (warp / 4));
    const int p1 = tid;  // phase 1: positions p1 * 64 + e
    {
      float v[E];
      const int64_t pos0 = int64_t(p1) * E;
      if (i0 < m && pos0 + E <= n) {
        const float* arow = a + i0 * lda;
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
        for (int e = 0; e < E; ++e) v[e] = (i0 < m && pos0 + e < n) ? a[i0 * lda + pos0 + e] : 0.f;
      }
#pragma unroll
      for (int c = 0; c < E / 32; ++c) tmem_st_x32(taddr + 32 * c, v + 32 * c);
      tmem_wait_st();
    }
    // phase 2: thread (hi2 = tid / 64, lo6 = tid % 64) owns positions hi2 * 4096 + e * 64 + lo6
    float* const src = tile + (tid >> 6) * (E * E) + (tid & 3);
    const int cq = (tid & 63) >> 2;
    int64_t s = next_basis(s_first);
    uint32_t qn[WPT];
#pragma unroll
    for (int w = 0; w < WPT; ++w) qn[w] = (s < s_last) ? __ldg(qplain + s * WPB + WPT * p1 + w) : 0u;
    bool first = true;
    WS_PROF_BEGIN();
    const int t0 = tid;  // (phase counters)
    (void)t0;
    while (s < s_last) {
      const int64_t s_next = next_basis(s + 1);
      float v[E];
      WS_T(0);
#pragma unroll
      for (int c = 0; c < E / 32; ++c) tmem_ld_x32(taddr + 32 * c, v + 32 * c);
      uint32_t q[WPT];
#pragma unroll
      for (int w = 0; w < WPT; ++w) q[w] = qn[w];
      if (s_next < s_last) {
#pragma unroll
        for (int w = 0; w < WPT; ++w) qn[w] = __ldg(qplain + s_next * WPB + WPT * p1 + w);
      }
      tmem_wait_ld();
      WS_T(1);
      // Kerdock sign mask (sketch.hpp:185): flip the sign bit where Q_s(pos) = 1 (exact)
#pragma unroll
      for (int e = 0; e < E; ++e)
        v[e] = __uint_as_float(__float_as_uint(v[e]) ^ ((q[e / 32] << (31 - (e % 32))) & 0x80000000u));
      reg_fwht_f32_packed<HALF>(v);  // position bits 0-5
      WS_T(2);
      if (!first) named_sync(2, NALL);  // FREED: the copy warps' reads of the previous staging are done
      first = false;
      WS_T(3);
      {
        float* dst = tile + p1 * E;
#pragma unroll
        for (int c = 0; c < CH; ++c)
          *reinterpret_cast<float4*>(dst + 4 * (c ^ (p1 & SWC))) =
              make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      }
      named_sync(5 + (tid >> 6), 64);  // the quarter's transpose only (two warps)
      WS_T(4);
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = src[e * E + 4 * (cq ^ (e & SWC))];
      reg_fwht_f32_packed<HALF>(v);  // position bits 6-11
      WS_T(5);
#pragma unroll
      for (int e = 0; e < E; ++e) src[e * E + 4 * (cq ^ (e & SWC))] = v[e];  // in place (bits 12, 13 left to the copy warps)
      named_arrive(1, NALL);  // STAGED
      WS_T(6);
      s = s_next;
    }
    WS_PROF_END(0);
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 48;" ::: "memory");  // 256 x 96 + 128 x 48 = 384 x 80
    const int t0 = tid & 127;
    uint32_t use = 0;
    int buf = 0;
    float* const cout = cols + (cbase - row0);
    auto prefetch = [&](int64_t sb, int b) {  // records of basis sb into reqbuf[b]; one commit group
      if (sb < s_last) {
        const int64_t lo = rs(sb), cnt = rs(sb + 1) - lo;
        if (cnt <= RCAP)
          for (int j = t0; j < cnt; j += 128) cp_async_8(&reqbuf[b * RCAP + j], req_rec + lo + j);
      }
      cp_async_commit();
    };
    // (transform value at position w: stages 4096 and 8192 over the four staged quarter values,
    //  (S0 +- S1) +- (S2 +- S3), evaluated in the chunk loop below)
    auto drain_use = [&](uint32_t ud) {
      const int slot = static_cast<int>(ud % SS);
      mbar_wait(&full_bar[slot], (ud / SS) & 1);
      const float* const rv = recv + slot * RCAP;
      const uint32_t* const rsl = rslot + slot * (RCAP / CL);
      constexpr int QD = CL / 4;
      const int mine = rmine[slot];
      for (int t = t0; t < QD * mine; t += 128) {
        const int jj = t / QD, h = t % QD;
        const float4 val = *reinterpret_cast<const float4*>(rv + jj * CL + 4 * h);
        float* dst = cout + int64_t(rsl[jj]) * ldc + 4 * h;
        const int64_t r4 = cbase + 4 * h;
        if (r4 + 3 < m) {
          stg_f32x4(dst, val);
        } else {
          if (r4 + 0 < m) dst[0] = val.x;
          if (r4 + 1 < m) dst[1] = val.y;
          if (r4 + 2 < m) dst[2] = val.z;
        }
      }
      __syncwarp();
      if ((tid & 31) == 0)
        for (int r = 0; r < CL; ++r) mbar_arrive_remote_relaxed(smem_u32(&empty_bar[slot]), r);
    };
    int64_t s = next_basis(s_first);
    prefetch(s, 0);
    WS_PROF_BEGIN();
    while (s < s_last) {
      const int64_t s_next = next_basis(s + 1);
      cp_async_wait_all();
      named_sync(4, 128);  // every copy thread finished basis s - 1 and its records of basis s are visible
      prefetch(s_next, buf ^ 1);  // next basis' records, issued while the tile is still being staged
      const int64_t r_lo = rs(s), r_hi = rs(s + 1);
      const int cnt = static_cast<int>(r_hi - r_lo);
      const uint2* recs = cnt <= RCAP ? reqbuf + buf * RCAP : req_rec + r_lo;
      // Everything that does not need the tile happens before STAGED: the requested positions of
      // the first chunk (RCAP / 128 = 8 per thread) are in registers when the tile arrives, so the
      // stretch between STAGED and FREED — which the butterfly warps wait out before their next
      // transpose — is the staged reads and three adds per request only.
      constexpr int U = RCAP / 128;
      uint32_t wv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = t0 + u * 128;
        wv[u] = j < min(RCAP, cnt) ? recs[j].x : 0u;
      }
      named_sync(1, NALL);  // STAGED: basis s is in the tile
      WS_T(0);
      for (int c0 = 0; c0 < cnt; c0 += RCAP) {
        const int nc = min(RCAP, cnt - c0);
        const int slot = static_cast<int>(use % SS);
        const uint32_t round = use / SS;
        const int mine = (nc - static_cast<int>(crank) + CL - 1) / CL;
        if (c0 > 0) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = t0 + u * 128;
            wv[u] = j < nc ? recs[c0 + j].x : 0u;
          }
        }
        float val[U];
#pragma unroll
        for (int h = 0; h < U; h += 4) {  // four requests' staged reads in flight at a time
          float sv[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t w = wv[h + u], pe = (w >> 6) & 63u, lo6 = w & 63u;
            const float* b = tile + pe * E + (lo6 & 3u) + 4u * ((lo6 >> 2) ^ (pe & SWC));
            sv[u][0] = b[0];
            sv[u][1] = b[4096];
            sv[u][2] = b[8192];
            sv[u][3] = b[12288];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t w = wv[h + u];
            const uint32_t n12 = (w << 19) & 0x80000000u, n13 = (w << 18) & 0x80000000u;  // bits 12, 13 as sign flips
            const float x = sv[u][0] + __uint_as_float(__float_as_uint(sv[u][1]) ^ n12);
            const float y = sv[u][2] + __uint_as_float(__float_as_uint(sv[u][3]) ^ n12);
            val[h + u] = x + __uint_as_float(__float_as_uint(y) ^ n13);
          }
        }
        // ... so the butterfly warps can overwrite the tile while the pushes go out
        if (c0 + RCAP >= cnt && s_next < s_last) named_arrive(2, NALL);  // FREED (last chunk of this basis)
        WS_T(1);
        if (t0 == 0) {
          mbar_arrive_expect_tx_cta(&full_bar[slot], static_cast<uint32_t>(4 * CL * mine));
          rmine[slot] = mine;
        }
        for (int jj = t0; jj < mine; jj += 128)
          rslot[slot * (RCAP / CL) + jj] = recs[c0 + jj * CL + static_cast<int>(crank)].y;
        if (round >= 1) mbar_wait(&empty_bar[slot], (round - 1) & 1);
        WS_T(2);
        const uint32_t rbase = smem_u32(recv + slot * RCAP) + 4u * crank, fbar = smem_u32(&full_bar[slot]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = t0 + u * 128;
          if (j < nc)
            st_async_f32(rbase + 4u * static_cast<uint32_t>((j / CL) * CL), val[u], static_cast<uint32_t>(j % CL), fbar);
        }
        ++use;
        WS_T(3);
        if (use > DL) drain_use(use - 1 - DL);
        WS_T(4);
        if (c0 + RCAP < cnt) named_sync(4, 128);  // next chunk reuses rslot / rmine entries
      }
      buf ^= 1;
      s = s_next;
    }
    WS_PROF_END(8);
    named_sync(4, 128);  // the last pushes' rslot / rmine entries are visible
    for (uint32_t u = use > DL ? use - DL : 0; u < use; ++u) drain_use(u);
    for (uint32_t u = use > SS ? use - SS : 0; u < use; ++u) mbar_wait(&empty_bar[u % SS], (u / SS) & 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_slot), "n"(TCOLS) : "memory");
}

// ---------------------------------------------------------------------------
// k = 12 full-sketch kernel with store warps (config 3 preprocessing): the
// arithmetic of fwht_tmem_kernel<12, false> (same stages, same order, same
// bits), but the 64 scattered column stores per thread per basis are issued by
// a separate warpgroup. In the single-role kernel a warp sits in its 64 stores
// (four 128-byte lines per warp store, so ~4 L1 tag cycles each; the LSU queue
// is shallow: lg_throttle) before it can start the next basis, and the store
// drain (~4.1k cycles per basis per SM) and the butterfly chain (~4.5k) add up.
// Here the butterfly warps park their phase-2 registers in the free half of
// tensor memory (tcgen05.st, ~1 KB/clk) and go on; store warp j (lane quadrant
// j) reads them back 32 columns at a time and replays the stores of butterfly
// warps j, j + 4, j + 8, j + 12 while the next basis is computed.
//   warps 0-15 (setmaxnreg 104): TMEM A tile -> sign mask -> FWHT -> TMEM staging
//   warps 16-19 (setmaxnreg 64): TMEM staging -> st.global (transposed, sketch.hpp:191-196)
// Named barriers: STAGED (id 1: butterfly warps arrive, store warps sync) and
// DRAINED (id 2: store warps arrive once the staging half is in their
// registers, butterfly warps sync before the next tcgen05.st).
// ---------------------------------------------------------------------------
template <int CL>
__global__ void __launch_bounds__(640, 1) fwht12_sketch_ws_kernel(
    const float* __restrict__ a, int64_t lda, int64_t m, int64_t n, const uint32_t* __restrict__ qplain,
    int64_t basis_begin, int64_t basis_end, int bases_per_cta, float* __restrict__ cols, int64_t ldc) {
  using C = TmemCfg<12>;
  constexpr int E = C::E, R = C::R, RS = C::RS, D = C::D, WPT = C::WPT, CH = C::CH, SWC = C::SWC;
  constexpr int WPB = D / 32, NB = 512, NALL = 640, TCOLS = 2 * C::TCOLS;
  static_assert(TCOLS == 512 && E == 64 && R == 8, "A tile and staging fill tensor memory");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tile = reinterpret_cast<float*>(smem_raw);
  __shared__ uint32_t tmem_base_slot;
  __shared__ __align__(8) uint64_t peer_bar[2];  // CL > 1: one arrival per CTA of the cluster and basis (even / odd)

  const int tid = threadIdx.x, warp = tid / 32;
  const bool bfly = __shfl_sync(0xffffffffu, tid / 128, 0) < 4;  // warp-uniform by construction (setmaxnreg regions)
  const int64_t i0 = int64_t(blockIdx.x) * R;
  const int64_t s_first = basis_begin + int64_t(blockIdx.y) * bases_per_cta;
  const int64_t s_last = min(basis_end, s_first + bases_per_cta);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_slot)),
                 "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (CL > 1 && tid == 0) {
    mbar_init(&peer_bar[0], CL);
    mbar_init(&peer_bar[1], CL);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if constexpr (CL > 1) cluster_sync_all();  // peers' barriers initialised before any remote arrive

  if (bfly) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 104;" ::: "memory");  // 512 x 104 + 128 x 64 = 640 x 96
    const int r1 = tid / E, p1 = tid % E;
    const int64_t row1 = i0 + r1;
    const int r2 = tid % R, q2 = tid / R;
    const uint32_t taddr = tmem_base_slot + (static_cast<uint32_t>(32 * (warp % 4)) << 16) +
                           static_cast<uint32_t>(E * (warp / 4));
    const uint32_t tstage = taddr + C::TCOLS;
    {
      float v[E];
      const int64_t pos0 = int64_t(p1) * E;
      if (row1 < m && pos0 + E <= n) {
        const float* arow = a + row1 * lda;
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
        for (int e = 0; e < E; ++e) v[e] = (row1 < m && pos0 + e < n) ? a[row1 * lda + pos0 + e] : 0.f;
      }
#pragma unroll
      for (int c = 0; c < E / 32; ++c) tmem_st_x32(taddr + 32 * c, v + 32 * c);
      tmem_wait_st();
    }
    uint32_t qn[WPT];
#pragma unroll
    for (int w = 0; w < WPT; ++w) qn[w] = (s_first < s_last) ? __ldg(qplain + s_first * WPB + WPT * p1 + w) : 0u;
    for (int64_t s = s_first; s < s_last; ++s) {
      float v[E];
#pragma unroll
      for (int c = 0; c < E / 32; ++c) tmem_ld_x32(taddr + 32 * c, v + 32 * c);
      uint32_t q[WPT];
#pragma unroll
      for (int w = 0; w < WPT; ++w) q[w] = qn[w];
      if (s + 1 < s_last) {
#pragma unroll
        for (int w = 0; w < WPT; ++w) qn[w] = __ldg(qplain + (s + 1) * WPB + WPT * p1 + w);
      }
      tmem_wait_ld();
      // Kerdock sign mask (sketch.hpp:185): flip the sign bit where Q_s(pos) = 1 (exact)
#pragma unroll
      for (int e = 0; e < E; ++e)
        v[e] = __uint_as_float(__float_as_uint(v[e]) ^ ((q[e / 32] << (31 - (e % 32))) & 0x80000000u));
#ifndef FSTG_PRE_WS_NOCOMPUTE
      reg_fwht_f32_packed<C::HALF>(v);  // position bits 0 .. 5
      named_sync(3, NB);                // previous basis' tile reads done
      {
        float* dst = tile + r1 * RS + p1 * E;
#pragma unroll
        for (int c = 0; c < CH; ++c)
          *reinterpret_cast<float4*>(dst + 4 * (c ^ (p1 & SWC))) =
              make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      }
      named_sync(3, NB);
      if constexpr (CL > 1) {  // "this CTA is half-way through basis s" to every CTA of the cluster (incl. itself)
        if (tid == 0) {
          const uint32_t kb = static_cast<uint32_t>(s - s_first);
          for (int r = 0; r < CL; ++r) mbar_arrive_remote_relaxed(smem_u32(&peer_bar[kb & 1]), r);
        }
      }
      {
        const float* src = tile + r2 * RS + (q2 & 3);
        const int cq = q2 >> 2;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = src[e * E + 4 * (cq ^ (e & SWC))];
      }
      reg_fwht_f32_packed<C::HALF>(v);  // position bits 6 .. 11
#endif
      if (s > s_first) {                // DRAINED: the store warps hold the previous basis
        named_sync(2, NALL);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
#pragma unroll
      for (int c = 0; c < E / 32; ++c) tmem_st_x32(tstage + 32 * c, v + 32 * c);
      tmem_wait_st();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      named_arrive(1, NALL);  // STAGED
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;" ::: "memory");
    const int j = warp - 16, lane = tid & 31;  // lane quadrant j: butterfly warps j, j + 4, j + 8, j + 12
    const uint32_t tstage = tmem_base_slot + (static_cast<uint32_t>(32 * j) << 16) + C::TCOLS;
    const int64_t step = int64_t(E) * ldc;
    for (int64_t s = s_first; s < s_last; ++s) {
      named_sync(1, NALL);  // STAGED
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if constexpr (CL > 1) {
        // The CL CTAs of a cluster hold the 8-row pieces of the same 32 * CL-byte column segments:
        // start this basis' stores together, so the 32-byte sectors of a segment reach L2 within a
        // short window and leave it as one DRAM burst (no data is exchanged: relaxed arrivals only,
        // sent by the butterfly warps half a basis earlier so the hand-shake is off the store path).
        // Uncoupled CTAs drift and the build time becomes bimodal (31 ms or 39-58 ms); 4-CTA
        // clusters only place on 132 of the 148 SMs; profiles/r02_preprocess_storewarps.txt.
        // (Two barriers, even / odd basis: a waiter can never see its barrier wrap a second time.)
        const uint32_t kb = static_cast<uint32_t>(s - s_first);
        mbar_wait(&peer_bar[kb & 1], (kb >> 1) & 1u);
      }
      // 16 pieces of 16 staged columns (piece p: butterfly warp 4 * (p / 4) + j, its registers
      // 16 * (p % 4) .. + 15), double-buffered: piece p + 1 is in flight while piece p is stored
      float vb[2][16];
      float* ptr = nullptr;
      const bool live = i0 + (lane % R) < m;  // the replayed thread's row: (32 * w + lane) % 8 = lane % 8
      tmem_ld_x16(tstage, vb[0]);
      tmem_wait_ld();
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        const int g = p / 4, c16 = p % 4;
        if (p + 1 < 16) tmem_ld_x16(tstage + E * ((p + 1) / 4) + 16 * ((p + 1) % 4), vb[(p + 1) & 1]);
        // the butterfly thread whose registers this lane replays: phase-2 row r2, column group q2
        if (c16 == 0) {
          const int tb = 32 * (4 * g + j) + lane;
          ptr = cols + (s * D + tb / R) * ldc + (i0 + tb % R);
        }
#ifndef FSTG_PRE_WS_NOSTORE
        if (live) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            ptr[0] = vb[p & 1][e];
            ptr += step;
            asm volatile("" : "+l"(ptr));
          }
        }
#else
        if (live && vb[p & 1][0] == 1.2345e-33f) ptr[0] = vb[p & 1][1];
#endif
        if (p + 1 < 16) {
          tmem_wait_ld();
          if (p + 1 == 15 && s + 1 < s_last) {  // the staging half is in registers: free again
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            named_arrive(2, NALL);  // DRAINED
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();  // no peer arrives on an exited CTA's barrier
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_slot), "n"(TCOLS) : "memory");
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

template <typename T, int KB, bool RETAIN = false>
static cudaError_t launch_fwht_k(const T* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                                 int64_t b0, int64_t b1, T* cols, int64_t ldc, cudaStream_t st,
                                 const int64_t* req_start = nullptr, const int64_t* req_ell = nullptr,
                                 const int64_t* req_pos = nullptr, int64_t row0 = 0) {
  constexpr int NT = (sizeof(T) == 8 && KB >= 12) ? 256 : ((KB >= 14) ? 256 : 512);
  using C = FwhtCfg<T, KB, NT>;
  static_assert(C::R >= 1, "rows per CTA");
  static_assert(!RETAIN || size_t(C::D) * C::R <= size_t(C::R) * C::RS, "retain staging fits the tile");
  auto kern = fwht_sketch_kernel<T, KB, NT, RETAIN>;
  if (C::SMEM > 227 * 1024) return cudaErrorNotSupported;
  if (C::SMEM > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
  }
  const int64_t nb = b1 - b0;
  if (nb <= 0) return cudaSuccess;
  const int64_t row_tiles = (m - row0 + C::R - 1) / C::R;
  // Bases per CTA: enough CTAs for >= 4 waves, at most 16 bases each.
  int bpc = 16;
  while (bpc > 1 && row_tiles * ((nb + bpc - 1) / bpc) < 148 * 8) bpc /= 2;
  const int64_t gy = (nb + bpc - 1) / bpc;
  if (row_tiles > 0x7fffffff || gy > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid(static_cast<unsigned>(row_tiles), static_cast<unsigned>(gy));
  kern<<<grid, NT, C::SMEM, st>>>(a, lda, m, n, qplain, b0, b1, bpc, cols, ldc, req_start, req_ell, req_pos, row0);
  return cudaGetLastError();
}

template <int KB, bool RETAIN>
static cudaError_t launch_fwht_tmem(const float* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                                    int64_t b0, int64_t b1, float* cols, int64_t ldc, cudaStream_t st,
                                    const int64_t* req_start, const int64_t* req_ell, const int64_t* req_pos,
                                    int64_t row0, const uint2* req_rec = nullptr);

template <typename T>
cudaError_t launch_fwht_retain(int k, const T* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                               int64_t nbases, T* out, int64_t ldc, const int64_t* req_start, const int64_t* req_ell,
                               const int64_t* req_pos, cudaStream_t st, int64_t row0, const uint2* req_rec) {
  if constexpr (sizeof(T) == 4) {
    if (k == 12 && (lda % 4) == 0)
      return launch_fwht_tmem<12, true>(a, lda, m, n, qplain, 0, nbases, out, ldc, st, req_start, req_ell, req_pos, row0,
                                        req_rec);
    if (k == 14 && (lda % 4) == 0)
      return launch_fwht_tmem<14, true>(a, lda, m, n, qplain, 0, nbases, out, ldc, st, req_start, req_ell, req_pos, row0,
                                        req_rec);
  }
  switch (k) {
    case 2: return launch_fwht_k<T, 2, true>(a, lda, m, n, qplain, 0, nbases, out, ldc, st, req_start, req_ell, req_pos, row0);
    case 4: return launch_fwht_k<T, 4, true>(a, lda, m, n, qplain, 0, nbases, out, ldc, st, req_start, req_ell, req_pos, row0);
    case 6: return launch_fwht_k<T, 6, true>(a, lda, m, n, qplain, 0, nbases, out, ldc, st, req_start, req_ell, req_pos, row0);
    case 8: return launch_fwht_k<T, 8, true>(a, lda, m, n, qplain, 0, nbases, out, ldc, st, req_start, req_ell, req_pos, row0);
    case 10: return launch_fwht_k<T, 10, true>(a, lda, m, n, qplain, 0, nbases, out, ldc, st, req_start, req_ell, req_pos, row0);
    case 12: return launch_fwht_k<T, 12, true>(a, lda, m, n, qplain, 0, nbases, out, ldc, st, req_start, req_ell, req_pos, row0);
    case 14: return launch_fwht_k<T, 14, true>(a, lda, m, n, qplain, 0, nbases, out, ldc, st, req_start, req_ell, req_pos, row0);
    default: return cudaErrorNotSupported;
  }
}
template cudaError_t launch_fwht_retain<float>(int, const float*, int64_t, int64_t, int64_t, const uint32_t*, int64_t,
                                               float*, int64_t, const int64_t*, const int64_t*, const int64_t*,
                                               cudaStream_t, int64_t, const uint2*);
template cudaError_t launch_fwht_retain<double>(int, const double*, int64_t, int64_t, int64_t, const uint32_t*, int64_t,
                                                double*, int64_t, const int64_t*, const int64_t*, const int64_t*,
                                                cudaStream_t, int64_t, const uint2*);

template <int KB, bool RETAIN>
static cudaError_t launch_fwht_tmem(const float* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                                    int64_t b0, int64_t b1, float* cols, int64_t ldc, cudaStream_t st,
                                    const int64_t* req_start, const int64_t* req_ell, const int64_t* req_pos,
                                    int64_t row0, const uint2* req_rec) {
  using C = TmemCfg<KB>;
  auto kern = fwht_tmem_kernel<KB, RETAIN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
  if (e != cudaSuccess) return e;
  const int64_t nb = b1 - b0;
  if (nb <= 0) return cudaSuccess;
  const int64_t row_tiles = (m - row0 + C::R - 1) / C::R;
  // the A tile is reused across bpc bases (TMEM); full sketch: 128 (32/64/128/256 measured
  // 37.5/37.0/36.3/36.8 ms at n = 4096, profiles/r01_preprocess_writepath.txt)
  bool sketch_ws = false;  // k = 12 full sketch: store-warp kernel (default), 2-CTA clusters
  int sketch_cl = 2;
  if constexpr (KB == 12 && !RETAIN) {
    sketch_ws = row0 == 0;
    if (const char* ev = std::getenv("FSTG_SKETCH_WS")) sketch_ws = sketch_ws && std::atoi(ev) != 0;  // experiments
    if (const char* ev = std::getenv("FSTG_SKETCH_CL")) sketch_cl = std::atoi(ev);                    // experiments
    if (sketch_cl != 2 && sketch_cl != 4) sketch_cl = 1;
  }
  // 128 bases per CTA for both k = 12 sketch kernels (store-warp kernel with CTA pairs: 32 / 64 / 128 / 256 / 512
  // measured 32.6 / 31.8 / 31.4 / 31.5 / 31.5 ms, profiles/r02_preprocess_storewarps.txt)
  int bpc = RETAIN ? C::MAXBPC : 128;
  if (const char* ev = std::getenv("FSTG_SKETCH_BPC")) {  // experiments
    if (!RETAIN && std::atoi(ev) > 0) bpc = std::atoi(ev);
  }
  while (bpc > 1 && row_tiles * ((nb + bpc - 1) / bpc) < 148 * 8) bpc /= 2;
  const int64_t gy = (nb + bpc - 1) / bpc;
  if (row_tiles > 0x7fffffff || gy > 65535) return cudaErrorInvalidConfiguration;
  if constexpr (KB == 12 && !RETAIN) {
    if (sketch_ws) {
      const int cl = sketch_cl;
      auto kw = cl == 4 ? fwht12_sketch_ws_kernel<4> : cl == 2 ? fwht12_sketch_ws_kernel<2> : fwht12_sketch_ws_kernel<1>;
      e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
      if (e != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>((row_tiles + cl - 1) / cl * cl), static_cast<unsigned>(gy));
      cfg.blockDim = dim3(640);
      cfg.dynamicSmemBytes = C::SMEM;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = static_cast<unsigned>(cl);
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, kw, a, lda, m, n, qplain, b0, b1, bpc, cols, ldc);
    }
  }
  if constexpr (RETAIN && C::R == 1) {
    // cluster-merged write-back (8 rows per cluster): needs the packed records and
    // 16-byte aligned 4-row column segments
    bool merge = req_rec != nullptr && (ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(cols) % 16) == 0;
    // 4 CTAs (16-byte segments): config-4 pass 145 -> 134 ms per 1024 rows; 8 CTAs (32-byte
    // segments) 147 ms — the merge's fixed per-basis cost grows with the cluster
    // (profiles/r01_k14_retain.txt)
    int CL = 4;
    if (const char* ev = std::getenv("FSTG_RETAIN_CLUSTER")) {  // experiments: 0 = off, 4 or 8 CTAs
      CL = std::atoi(ev);
      merge = merge && (CL == 4 || CL == 8);
    }
    bool ws = KB == 14;  // warp-specialised variant (copy warps off the butterfly warps)
    if (const char* ev = std::getenv("FSTG_RETAIN_WS")) ws = ws && std::atoi(ev) != 0;  // experiments
    if (merge && ws) {
      auto kw = CL == 4 ? fwht14_retain_ws_kernel<4> : fwht14_retain_ws_kernel<8>;
      e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM + kWsRecvBytes));
      if (e != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>((row_tiles + CL - 1) / CL * CL), static_cast<unsigned>(gy));
      cfg.blockDim = dim3(384);
      cfg.dynamicSmemBytes = C::SMEM + kWsRecvBytes;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = CL;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, kw, a, lda, m, n, qplain, b1, bpc, cols, ldc, req_start, req_rec, row0);
    }
    if (merge) {
      auto kc = CL == 4 ? fwht_tmem_kernel<KB, RETAIN, 4> : fwht_tmem_kernel<KB, RETAIN, 8>;
      e = cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
      if (e != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>((row_tiles + CL - 1) / CL * CL), static_cast<unsigned>(gy));
      cfg.blockDim = dim3(C::NT);
      cfg.dynamicSmemBytes = C::SMEM;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = CL;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, kc, a, lda, m, n, qplain, b0, b1, bpc, cols, ldc, req_start, req_ell, req_pos,
                                row0, req_rec);
    }
  }
  kern<<<dim3(static_cast<unsigned>(row_tiles), static_cast<unsigned>(gy)), C::NT, C::SMEM, st>>>(
      a, lda, m, n, qplain, b0, b1, bpc, cols, ldc, req_start, req_ell, req_pos, row0, req_rec);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fwht_sketch(int k, const T* a, int64_t lda, int64_t m, int64_t n, const uint32_t* qplain,
                               int64_t b0, int64_t b1, T* cols, int64_t ldc, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    if (k == 12 && (lda % 4) == 0)
      return launch_fwht_tmem<12, false>(a, lda, m, n, qplain, b0, b1, cols, ldc, st, nullptr, nullptr, nullptr, 0);
    if (k == 14 && (lda % 4) == 0)
      return launch_fwht_tmem<14, false>(a, lda, m, n, qplain, b0, b1, cols, ldc, st, nullptr, nullptr, nullptr, 0);
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

#ifdef FSTG_WS_PROF
extern "C" int fstg_debug_wsprof(unsigned long long* out) {  // experiments only: read and clear the phase counters
  unsigned long long z[16] = {};
  if (cudaMemcpyFromSymbol(out, fstg::g_wsprof, sizeof(z)) != cudaSuccess) return 1;
  return cudaMemcpyToSymbol(fstg::g_wsprof, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
#endif
