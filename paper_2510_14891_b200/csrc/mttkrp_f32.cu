// Float32 MTTKRP on the 5th-generation tensor cores (tcgen05, kind::tf32),
// the north star's optional float32 path (<= 1e-4 relative Frobenius).
//
// Same contraction and chunking as the FP64 kernels (mttkrp.cu header): a
// chunk is BK = 32 consecutive values of the fastest non-k mode f with the
// other non-k indices fixed, and its Khatri-Rao rows are
// Z[c, j] = A_f[i_f0 + c, j] * prod_o A_o[o_m, j].  Per CTA tile of 128
// output rows x 128 rank columns:
//
//   warp 0 (one lane)  TMA: tensor tile, 32 rows of A_f, the o-rows -> raw
//                      stage (2 stages)
//   warp 1             TMEM allocation (two fp32 group accumulators + the
//                      running sum, 384 of 512 columns);
//                      one lane issues the UMMAs
//   warps 2-9          transform: Y and Z into "3xTF32" operands, each value
//                      v split as hi = v's top 11 significand bits (exactly
//                      a TF32, tf32_hi), lo = v - hi (exact), in the K-major
//                      SWIZZLE_128B layout UMMA reads (2 operand stages)
//   warps 10-17        drain: the tensor core's fp32 accumulation truncates,
//                      a bias that grows with the number of accumulations
//                      (1.1e-4 after ~4k MMAs into one accumulator), so the
//                      MMAs of every F_GROUP chunks go to one of two TMEM
//                      accumulators (ping-pong) and these warps add each
//                      finished group into a running sum kept in TMEM
//                      (round-to-nearest fp32 adds) while the other
//                      accumulator fills; then the epilogue
//
// Each chunk is 4 k-steps x {Yhi.Zhi, Yhi.Zlo, Ylo.Zhi} = 12
// tcgen05.mma.cta_group::1.kind::tf32 (M = 128, N = 128, K = 8) into one fp32
// TMEM accumulator; the dropped Ylo.Zlo term is ~2^-22 relative, so the
// result carries fp32-level accuracy (a single TF32 pass would not meet
// 1e-4: the hardware truncates fp32 operands to TF32, a biased ~1e-3 error;
// tools/umma_tf32_probe.cu).  Split-K partials are fp32; their merge sums
// in FP64 and writes fp32.
#include "common.cuh"
#include "mttkrp_internal.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

namespace cpk {
namespace {

constexpr int F_BM = 128, F_BN = 128, F_BK = 32;  // rows, rank columns, chunk depth (128 B of fp32)
// warp 0 TMA, warp 1 MMA, warps 2-9 transform, warps 10-17 drain
constexpr int F_XFORM_WARPS = 8, F_DRAIN_WARPS = 8;
constexpr int F_THREADS = (2 + F_XFORM_WARPS + F_DRAIN_WARPS) * 32;
constexpr int F_GROUP = 4;  // chunks (48 MMAs) per TMEM accumulator before a drain
// TMEM columns: two group accumulators [0, 256) and the running sum [256, 384)
constexpr int F_SUM_COL = 2 * F_BN, F_TMEM_COLS = 512;
constexpr int F_OP_STAGES = 2;
constexpr int F_TILE_BYTES = F_BM * F_BK * 4;  // 16 KB: one 128 x 32 fp32 operand tile
static_assert(F_BM == F_BN, "A and B operand tiles share one size");

struct alignas(64) F32Params {
  CUtensorMap tm_y;
  CUtensorMap tm_f;
  CUtensorMap tm_o[3];
  int64_t dim_o[3];
  int64_t chunks_per_f, n_chunks, chunks_per_split;
  int32_t Ik, R, k;
  float* out;  // partials [splits][Ik][ldo] or G
  int64_t ldo, out_split_stride;
  const float* lam;  // folded in the epilogue only when writing G directly
};

// KMAJ (mode > 0): TMA lands Y K-major with the 128-B swizzle, which is
// already the UMMA A layout, and the tensor core's fp32 -> TF32 truncation is
// exactly tf32_hi(): the UMMAs read Y_hi from the raw stage itself, so only
// Y_lo is written (the op stage drops A_hi) and the raw stage stays busy
// until the MMAs have read it -- hence 3 raw stages.  Mode 0 transposes.
template <int NO, bool KMAJ>
struct F32Cfg {
  static constexpr int RAW_STAGES = KMAJ ? 3 : 2;
  static constexpr int RAW_Y = 0;
  static constexpr int RAW_F = RAW_Y + F_TILE_BYTES;        // [32 k][128 n] fp32
  static constexpr int RAW_P = RAW_F + F_BK * F_BN * 4;     // NO x 128 fp32
  static constexpr int RAW_BYTES = ((RAW_P + NO * F_BN * 4 + 1023) / 1024) * 1024;
  static constexpr int TX = F_TILE_BYTES + F_BK * F_BN * 4 + NO * F_BN * 4;
  // operand stage: [A_hi (mode 0 only)], A_lo, B_hi, B_lo (K-major SW128)
  static constexpr int A_HI = 0;
  static constexpr int A_LO = KMAJ ? 0 : F_TILE_BYTES;
  static constexpr int B_HI = A_LO + F_TILE_BYTES, B_LO = B_HI + F_TILE_BYTES;
  static constexpr int OP_BYTES = B_LO + F_TILE_BYTES;
  static constexpr int OP_BASE = RAW_STAGES * RAW_BYTES;
  static constexpr int BAR_BASE = OP_BASE + F_OP_STAGES * OP_BYTES;
  static constexpr size_t SMEM = size_t(BAR_BASE) + 256;
};

// ---------------------------------------------------------------- PTX
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P;\nWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
template <int RANK>
__device__ __forceinline__ void tma(void* dst, const CUtensorMap* map, uint64_t* bar, const int (&c)[RANK]) {
  const unsigned d = su32(dst), b = su32(bar);
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  if constexpr (RANK == 2)
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
                 ::"r"(d), "l"(m), "r"(b), "r"(c[0]), "r"(c[1]) : "memory");
  else if constexpr (RANK == 3)
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n"
                 ::"r"(d), "l"(m), "r"(b), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory");
  else if constexpr (RANK == 4)
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n"
                 ::"r"(d), "l"(m), "r"(b), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];\n"
                 ::"r"(d), "l"(m), "r"(b), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
}
// K-major SWIZZLE_128B UMMA operand descriptor (rows of 128 B, 8-row atoms)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
         (uint64_t(2) << 61);
}
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(F_BN >> 3) << 17) | (uint32_t(F_BM >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// float offset of (row r, k) in a K-major SW128 tile of 32-float rows
__device__ __forceinline__ int swz(int r, int k4) { return r * 32 + (((k4 ^ (r & 7))) << 2); }

// v = hi + lo with hi = v's top 11 significand bits (exactly a TF32) and
// lo = v - hi exact in fp32; the tensor core truncates lo to TF32, an error
// below 2^-21 |v|, and the dropped lo*lo term is below 2^-20 |y z|.
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ void split_store(float* hi_tile, float* lo_tile, int off, float4 v) {
  float4 h, l;
  h.x = tf32_hi(v.x);
  h.y = tf32_hi(v.y);
  h.z = tf32_hi(v.z);
  h.w = tf32_hi(v.w);
  l.x = v.x - h.x;
  l.y = v.y - h.y;
  l.z = v.z - h.z;
  l.w = v.w - h.w;
  *reinterpret_cast<float4*>(hi_tile + off) = h;
  *reinterpret_cast<float4*>(lo_tile + off) = l;
}

// ---------------------------------------------------------------- kernel
template <bool KMAJ, int NO>
__global__ void __launch_bounds__(F_THREADS, 1) mttkrp_f32_umma_sm100(const __grid_constant__ F32Params p) {
  using C = F32Cfg<NO, KMAJ>;
  constexpr int RS = C::RAW_STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_BASE);
  uint64_t* raw_full = bars;                          // [RS] TMA landed
  uint64_t* raw_empty = bars + 3;                     // [RS] raw stage consumed (transform, + MMA if KMAJ)
  uint64_t* op_full = bars + 6;                       // [2] operands written
  uint64_t* op_empty = bars + 8;                      // [2] UMMAs done reading
  uint64_t* acc_full = bars + 10;                     // [2] accumulator group done
  uint64_t* acc_empty = bars + 12;                    // [2] accumulator drained
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q0 = int64_t(blockIdx.z) * p.chunks_per_split;
  const int nst = int(min(p.n_chunks, q0 + p.chunks_per_split) - q0);
  const int j0 = blockIdx.x * F_BN, n0 = blockIdx.y * F_BM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      bar_init(&raw_full[s], 1);
      bar_init(&raw_empty[s], F_XFORM_WARPS + (KMAJ ? 1 : 0));
    }
    for (int s = 0; s < 2; ++s) {
      bar_init(&op_full[s], F_XFORM_WARPS);
      bar_init(&op_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      bar_init(&acc_full[b], 1);
      bar_init(&acc_empty[b], F_DRAIN_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)),
                 "r"(F_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA
    if (lane == 0) {
      int qf = int(q0 % p.chunks_per_f), od[NO > 0 ? NO : 1];
      {
        int64_t rest = q0 / p.chunks_per_f;
#pragma unroll
        for (int i = 0; i < NO; ++i) {
          od[i] = int(rest % p.dim_o[i]);
          rest /= p.dim_o[i];
        }
      }
      constexpr int D = NO + 2;
      for (int it = 0; it < nst; ++it) {
        const int s = it % RS;
        if (it >= RS) bar_wait(&raw_empty[s], ((it / RS) - 1) & 1);
        uint8_t* st = smem + s * C::RAW_BYTES;
        bar_expect_tx(&raw_full[s], C::TX);
        const int if0 = qf * F_BK;
        int c[D];
        if constexpr (!KMAJ) {
          c[0] = n0;
          c[1] = if0;
#pragma unroll
          for (int m = 2; m < D; ++m) c[m] = od[m - 2];
        } else {
          c[0] = if0;
#pragma unroll
          for (int m = 1; m < D; ++m) {
            const int lo_i = m - 1 < NO ? m - 1 : NO - 1;
            const int hi_i = m >= 2 ? m - 2 : 0;
            c[m] = (m == p.k) ? n0 : (m > p.k ? od[hi_i] : od[lo_i]);
          }
        }
        tma<D>(st + C::RAW_Y, &p.tm_y, &raw_full[s], c);
        const int cf[2] = {j0, if0};
        tma<2>(st + C::RAW_F, &p.tm_f, &raw_full[s], cf);
#pragma unroll
        for (int i = 0; i < NO; ++i) {
          const int co[2] = {j0, od[i]};
          tma<2>(st + C::RAW_P + i * F_BN * 4, &p.tm_o[i], &raw_full[s], co);
        }
        if (++qf == int(p.chunks_per_f)) {
          qf = 0;
#pragma unroll
          for (int i = 0; i < NO; ++i) {
            if (++od[i] < int(p.dim_o[i])) break;
            od[i] = 0;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA
    if (lane == 0) {
      for (int it = 0; it < nst; ++it) {
        const int o = it & 1, g = it / F_GROUP, b = g & 1;
        const bool first = it % F_GROUP == 0;
        if (first && g >= 2) bar_wait(&acc_empty[b], ((g >> 1) - 1) & 1);
        bar_wait(&op_full[o], (it >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t base = su32(smem + C::OP_BASE + o * C::OP_BYTES);
        const int s = it % RS;
        const uint64_t a_hi = KMAJ ? sw128_desc(su32(smem + s * C::RAW_BYTES + C::RAW_Y)) : sw128_desc(base + C::A_HI);
        const uint64_t a_lo = sw128_desc(base + C::A_LO);
        const uint64_t b_hi = sw128_desc(base + C::B_HI), b_lo = sw128_desc(base + C::B_LO);
        const uint32_t acc_t = tmem + uint32_t(b * F_BN);
#pragma unroll
        for (int ks = 0; ks < F_BK / 8; ++ks) {  // UMMA_K = 8 tf32 = 32 B: +2 in the 16-B address units
          const uint64_t adv = uint64_t(ks * 2);
          umma_tf32(acc_t, a_hi + adv, b_hi + adv, (first && ks == 0) ? 0u : 1u);
          umma_tf32(acc_t, a_hi + adv, b_lo + adv, 1u);
          umma_tf32(acc_t, a_lo + adv, b_hi + adv, 1u);
        }
        umma_commit(&op_empty[o]);  // operand stage free once these MMAs have read it
        if constexpr (KMAJ) umma_commit(&raw_empty[s]);  // and the raw stage (Y_hi)
        if (it % F_GROUP == F_GROUP - 1 || it == nst - 1) umma_commit(&acc_full[b]);
      }
    }
  } else if (warp < 2 + F_XFORM_WARPS) {
    // ------------------------------------------------------------ transform
    // 256 threads: operand row r = t % 128 (m for Y, n for Z), float4
    // groups k4 in [4h, 4h + 4) with h = t / 128
    const int t = threadIdx.x - 64, r = t & (F_BM - 1), k4_0 = (t >> 7) * 4;
    for (int it = 0; it < nst; ++it) {
      const int s = it % RS, o = it & 1;
      bar_wait(&raw_full[s], (it / RS) & 1);
      if (it >= 2) bar_wait(&op_empty[o], ((it >> 1) - 1) & 1);
      const uint8_t* st = smem + s * C::RAW_BYTES;
      uint8_t* op = smem + C::OP_BASE + o * C::OP_BYTES;
      float* a_hi = reinterpret_cast<float*>(op + C::A_HI);
      float* a_lo = reinterpret_cast<float*>(op + C::A_LO);
      float* b_hi = reinterpret_cast<float*>(op + C::B_HI);
      float* b_lo = reinterpret_cast<float*>(op + C::B_LO);
      const float* ry = reinterpret_cast<const float*>(st + C::RAW_Y);
      if constexpr (KMAJ) {
        // Y_hi is the raw tile itself (see F32Cfg): write Y_lo only, at the
        // same swizzled offsets
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int off = (t + 256 * i) * 4;  // float4 chunk index * 4
          const float4 v = *reinterpret_cast<const float4*>(ry + off);
          float4 l;
          l.x = v.x - tf32_hi(v.x);
          l.y = v.y - tf32_hi(v.y);
          l.z = v.z - tf32_hi(v.z);
          l.w = v.w - tf32_hi(v.w);
          *reinterpret_cast<float4*>(a_lo + off) = l;
        }
      } else {
        // Y landed M-major [32 k][128 m]: transpose row m = t into K-major
#pragma unroll
        for (int k4 = k4_0; k4 < k4_0 + 4; ++k4) {
          float4 v;
          v.x = ry[(4 * k4 + 0) * F_BM + r];
          v.y = ry[(4 * k4 + 1) * F_BM + r];
          v.z = ry[(4 * k4 + 2) * F_BM + r];
          v.w = ry[(4 * k4 + 3) * F_BM + r];
          split_store(a_hi, a_lo, swz(r, k4), v);
        }
      }
      // Z^T row n = r: Z[k][n] = A_f[f0 + k][n] * prod_o A_o[o][n]
      const float* rf = reinterpret_cast<const float*>(st + C::RAW_F);
      float pr = 1.0f;
      if constexpr (NO > 0) {
        const float* rp = reinterpret_cast<const float*>(st + C::RAW_P);
        pr = rp[r];
#pragma unroll
        for (int i = 1; i < NO; ++i) pr *= rp[i * F_BN + r];
      }
#pragma unroll
      for (int k4 = k4_0; k4 < k4_0 + 4; ++k4) {
        float4 v;
        v.x = rf[(4 * k4 + 0) * F_BN + r] * pr;
        v.y = rf[(4 * k4 + 1) * F_BN + r] * pr;
        v.z = rf[(4 * k4 + 2) * F_BN + r] * pr;
        v.w = rf[(4 * k4 + 3) * F_BN + r] * pr;
        split_store(b_hi, b_lo, swz(r, k4), v);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> UMMA reads
      __syncwarp();
      if (lane == 0) {
        bar_arrive(&op_full[o]);
        bar_arrive(&raw_empty[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ drain + epilogue
    // two warps per TMEM lane quarter (rows 32q..32q+31), 64 columns each;
    // the running sum lives in TMEM too (columns F_SUM_COL..), updated with
    // round-to-nearest fp32 adds on the CUDA cores
    constexpr int HALF = F_BN / 2;
    const int quarter = warp & 3, c_base = ((warp - 2 - F_XFORM_WARPS) >> 2) * HALF;
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    const int groups = (nst + F_GROUP - 1) / F_GROUP;
    for (int g = 0; g < groups; ++g) {
      const int b = g & 1;
      bar_wait(&acc_full[b], (g >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int c0 = 0; c0 < HALF; c0 += 16) {
        uint32_t v[16], w[16];
        tmem_ld16(lane_base + uint32_t(b * F_BN + c_base + c0), v);
        if (g > 0) tmem_ld16(lane_base + uint32_t(F_SUM_COL + c_base + c0), w);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int jj = 0; jj < 16; ++jj)
          w[jj] = g > 0 ? __float_as_uint(__uint_as_float(w[jj]) + __uint_as_float(v[jj])) : v[jj];
        tmem_st16(lane_base + uint32_t(F_SUM_COL + c_base + c0), w);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&acc_empty[b]);
    }
    const int n = n0 + quarter * 32 + lane;
    const int jb = j0 + c_base;
#pragma unroll 1
    for (int c0 = 0; c0 < HALF; c0 += 16) {
      uint32_t w[16];
      tmem_ld16(lane_base + uint32_t(F_SUM_COL + c_base + c0), w);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (n < p.Ik) {
        float* dst = p.out + int64_t(blockIdx.z) * p.out_split_stride + int64_t(n) * p.ldo + jb + c0;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = jb + c0 + jj;
          if (j < p.R) dst[jj] = p.lam ? __uint_as_float(w[jj]) * p.lam[j] : __uint_as_float(w[jj]);
        }
      }
    }
  }
  // teardown: everyone done with TMEM before warp 1 frees it
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(F_TMEM_COLS));
  }
}

// split-K merge in FP64 (split order), lam folded once, fp32 out
__global__ void splitk_reduce_f32(const float* __restrict__ w, int splits, int64_t Ik, int64_t R, int64_t ldw,
                                  int64_t split_stride, const float* __restrict__ lam, float* __restrict__ G,
                                  int64_t ldg) {
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < Ik * R;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n = idx / R, j = idx - n * R;
    const float* src = w + n * ldw + j;
    double s = 0.0;
    for (int sp = 0; sp < splits; ++sp) s += double(src[sp * split_stride]);
    if (lam) s *= double(lam[j]);
    G[n * ldg + j] = float(s);
  }
}

// ---------------------------------------------------------------- host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn32() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

int encode32(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
             const cuuint32_t* box, CUtensorMapSwizzle swz) {
  auto fn = encode_fn32();
  if (!fn) return fail(CPK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CPK_ERR_CUDA, "cuTensorMapEncodeTiled (fp32) failed (%d)", int(r));
  return CPK_OK;
}

template <bool KMAJ, int NO>
void f32_kernel(const void** fn, size_t* smem) {
  static_assert(F32Cfg<NO, KMAJ>::SMEM <= 227 * 1024, "shared memory budget");
  *fn = reinterpret_cast<const void*>(&mttkrp_f32_umma_sm100<KMAJ, NO>);
  *smem = F32Cfg<NO, KMAJ>::SMEM;
}

struct F32Problem {
  int d, k, f, n_o;
  int64_t dims[CPK_MAX_MODES];
  int o_modes[3];
  int64_t chunks, tiles;
};

int f32_problem(int d, const int64_t* dims, int mode, int64_t rank, F32Problem* pr) {
  if (d < 2 || d > 5) return fail(CPK_ERR_PARAM, "float32 MTTKRP supports 2 <= d <= 5 (got %d)", d);
  if (!dims) return fail(CPK_ERR_SHAPE, "dims is NULL");
  if (mode < 0 || mode >= d) return fail(CPK_ERR_INDEX, "mode %d out of range [0, %d]", mode, d - 1);
  if (rank < 1) return fail(CPK_ERR_PARAM, "rank must be >= 1");
  pr->d = d;
  pr->k = mode;
  pr->f = mode == 0 ? 1 : 0;
  pr->n_o = 0;
  for (int m = 0; m < d; ++m) {
    if (dims[m] < 1) return fail(CPK_ERR_SHAPE, "extent %d is %lld", m, (long long)dims[m]);
    if (dims[m] >= (int64_t(1) << 31)) return fail(CPK_ERR_PARAM, "extent %d too large for the fp32 kernel", m);
    pr->dims[m] = dims[m];
    if (m != mode && m != pr->f) pr->o_modes[pr->n_o++] = m;
  }
  pr->chunks = (dims[pr->f] + F_BK - 1) / F_BK;
  for (int i = 0; i < pr->n_o; ++i) pr->chunks *= dims[pr->o_modes[i]];
  pr->tiles = ((dims[mode] + F_BM - 1) / F_BM) * ((rank + F_BN - 1) / F_BN);
  return CPK_OK;
}

// splits: <= 512 chunks per CTA, fill whole waves, workspace <= 2 GiB (as the FP64 planner)
int f32_splits(const F32Problem& pr, int64_t rank, int sms) {
  const int64_t ldw = (rank + 3) & ~int64_t(3);
  const double per = double(pr.dims[pr.k]) * double(ldw) * 4.0;
  const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(4096, int64_t(2.0 * (1 << 30) / per)));
  const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(pr.chunks, cap));
  const int64_t lo = std::min<int64_t>(max_s, std::max<int64_t>(1, (pr.chunks + 511) / 512));
  double best = -1.0;
  int64_t best_s = lo;
  for (int64_t s = lo; s <= max_s; ++s) {
    const int64_t work = pr.tiles * s, waves = (work + sms - 1) / sms;
    const double eff = double(work) / double(waves * sms);
    if (eff > best + 5e-3) {
      best = eff;
      best_s = s;
    }
  }
  const int64_t cps = (pr.chunks + best_s - 1) / best_s;
  return int((pr.chunks + cps - 1) / cps);
}

}  // namespace
}  // namespace cpk

using namespace cpk;

extern "C" int cpk_mttkrp_f32_workspace_bytes(int d, const int64_t* dims, int mode, int64_t rank, int splits,
                                              size_t* bytes) {
  if (!bytes) return fail(CPK_ERR_PARAM, "NULL argument");
  F32Problem pr;
  int rc = f32_problem(d, dims, mode, rank, &pr);
  if (rc) return rc;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int s = splits > 0 ? int(std::min<int64_t>(splits, pr.chunks)) : f32_splits(pr, rank, sms);
  const int64_t ldw = (rank + 3) & ~int64_t(3);
  *bytes = s > 1 ? size_t(s) * size_t(dims[mode]) * size_t(ldw) * sizeof(float) : 0;
  return CPK_OK;
}

extern "C" int cpk_mttkrp_f32(const float* y, int d, const int64_t* dims, int mode, const float* const* factors,
                              const int64_t* ld, const float* lam, int64_t rank, float* G, int64_t ldg, int splits,
                              void* workspace, size_t ws_bytes, void* stream) {
  F32Problem pr;
  int rc = f32_problem(d, dims, mode, rank, &pr);
  if (rc) return rc;
  if (!y || !G || !factors) return fail(CPK_ERR_PARAM, "NULL pointer");
  if (ldg < rank) return fail(CPK_ERR_PARAM, "ldg < rank");
  // TMA: 16-byte aligned bases and strides (I_0 and every ld a multiple of 4)
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (!al16(y) || pr.dims[0] % 4 != 0)
    return fail(CPK_ERR_PARAM, "float32 kernel needs a 16-byte aligned tensor and I_0 %% 4 == 0");
  for (int m = 0; m < d; ++m) {
    if (m == mode) continue;
    const int64_t l = ld ? ld[m] : rank;
    if (!factors[m] || l < rank || l % 4 != 0 || !al16(factors[m]))
      return fail(CPK_ERR_PARAM, "float32 kernel needs 16-byte aligned factors with ld %% 4 == 0 (mode %d)", m);
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int s = splits > 0 ? int(std::min<int64_t>(splits, pr.chunks)) : f32_splits(pr, rank, sms);
  const int64_t ldw = (rank + 3) & ~int64_t(3);
  const size_t need = s > 1 ? size_t(s) * size_t(dims[mode]) * size_t(ldw) * sizeof(float) : 0;
  if (need && (!workspace || ws_bytes < need))
    return fail(CPK_ERR_RESOURCE, "fp32 split-K workspace needs %zu bytes, got %zu", need, ws_bytes);

  F32Params p;
  memset(&p, 0, sizeof(p));
  cuuint64_t gdim[5], gstr[4];
  int64_t st = 1;
  for (int m = 0; m < d; ++m) {
    gdim[m] = cuuint64_t(dims[m]);
    if (m > 0) gstr[m - 1] = cuuint64_t(st * 4);
    st *= dims[m];
  }
  cuuint32_t box[5] = {1, 1, 1, 1, 1};
  if (mode == 0) {
    box[0] = F_BM;  // 128 rows (m contiguous), 32 chunk values
    box[1] = F_BK;
    rc = encode32(&p.tm_y, y, d, gdim, gstr, box, CU_TENSOR_MAP_SWIZZLE_NONE);
  } else {
    box[0] = F_BK;  // 32 fp32 = 128 B: the K-major SW128 row
    box[mode] = F_BM;
    rc = encode32(&p.tm_y, y, d, gdim, gstr, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (rc) return rc;
  {
    const cuuint64_t fd[2] = {cuuint64_t(rank), cuuint64_t(dims[pr.f])};
    const cuuint64_t fs[1] = {cuuint64_t((ld ? ld[pr.f] : rank) * 4)};
    const cuuint32_t fb[2] = {cuuint32_t(F_BN), cuuint32_t(F_BK)};
    rc = encode32(&p.tm_f, factors[pr.f], 2, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
  }
  for (int i = 0; i < pr.n_o; ++i) {
    const int m = pr.o_modes[i];
    const cuuint64_t od[2] = {cuuint64_t(rank), cuuint64_t(dims[m])};
    const cuuint64_t os[1] = {cuuint64_t((ld ? ld[m] : rank) * 4)};
    const cuuint32_t ob[2] = {cuuint32_t(F_BN), 1};
    rc = encode32(&p.tm_o[i], factors[m], 2, od, os, ob, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
    p.dim_o[i] = dims[m];
  }
  p.chunks_per_f = (dims[pr.f] + F_BK - 1) / F_BK;
  p.n_chunks = pr.chunks;
  p.chunks_per_split = (pr.chunks + s - 1) / s;
  p.Ik = int32_t(dims[mode]);
  p.R = int32_t(rank);
  p.k = mode;
  const bool direct = s == 1;
  p.out = direct ? G : static_cast<float*>(workspace);
  p.ldo = direct ? ldg : ldw;
  p.out_split_stride = direct ? 0 : int64_t(dims[mode]) * ldw;
  p.lam = direct ? lam : nullptr;

  const void* fn = nullptr;
  size_t smem = 0;
  const bool kmaj = mode != 0;
  switch (pr.n_o) {
    case 0: kmaj ? f32_kernel<true, 0>(&fn, &smem) : f32_kernel<false, 0>(&fn, &smem); break;
    case 1: kmaj ? f32_kernel<true, 1>(&fn, &smem) : f32_kernel<false, 1>(&fn, &smem); break;
    case 2: kmaj ? f32_kernel<true, 2>(&fn, &smem) : f32_kernel<false, 2>(&fn, &smem); break;
    default: kmaj ? f32_kernel<true, 3>(&fn, &smem) : f32_kernel<false, 3>(&fn, &smem); break;
  }
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return check_launch("fp32 set smem");
  dim3 grid(unsigned((rank + F_BN - 1) / F_BN), unsigned((dims[mode] + F_BM - 1) / F_BM), unsigned(s));
  if (grid.y > 65535u || grid.z > 65535u) return fail(CPK_ERR_PARAM, "grid too large");
  cudaStream_t cs = as_stream(stream);
  void* args[] = {&p};
  cudaError_t e = cudaLaunchKernel(fn, grid, dim3(F_THREADS), args, smem, cs);
  if (e != cudaSuccess) return fail(CPK_ERR_CUDA, "fp32 launch: %s", cudaGetErrorString(e));
  if (!direct) {
    const int64_t total = int64_t(dims[mode]) * rank;
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, int64_t(sms) * 16)));
    splitk_reduce_f32<<<blocks, 256, 0, cs>>>(static_cast<const float*>(workspace), s, dims[mode], rank, ldw,
                                              int64_t(dims[mode]) * ldw, lam, G, ldg);
  }
  return check_launch("mttkrp_f32");
}
