// Warp-specialized TMA variant of the sm_100a FP64 MTTKRP (the aligned fast
// path: I_0 even, even leading dimensions, 16-byte aligned bases, d <= 5).
//
// Same math and chunking as mttkrp.cu (see the header comment there); what
// changes is who moves the data:
//
//   * warp 8 (producer): one elected lane issues TMA (cp.async.bulk.tensor)
//     for the tensor tile, the BK factor rows of A_f and the o-mode rows of
//     every chunk, STAGES-1 chunks ahead, completing on an mbarrier; the
//     whole warp then forms the Khatri-Rao rows in place,
//     B[k][j] = A_f[i_f0 + k][j] * prod_o A_o[o][j], and publishes the stage.
//   * warps 0-7 (consumers): wait for a stage, run the 8x8-per-thread DFMA
//     outer products straight out of shared memory, release the stage.
//
// No __syncthreads in the main loop: full/empty mbarrier pairs per stage.
// The consumer instruction stream is LDS.128 + DFMA only.  TMA zero-fills
// out-of-range rows / chunk tails / rank tails, so there is no masking.
//
// Tensor tile layouts in shared memory:
//   mode 0 (M-major): DFMA consumers: box {BM, BK} -> As[k][m], no swizzle;
//     DMMA consumers: BM / 16 boxes {16, BK} with the 128-byte swizzle ->
//     panels [k][16] (and the factor rows likewise, BN / 16 boxes {16, BK}).
//   mode k>0 (K-major): two boxes {16, BM} (one per 16-deep panel) with the
//     128-byte swizzle -> panel[m][16] where the 16-byte chunk c of row m
//     lives at chunk c ^ (m & 7).
// The DMMA consumers' fragment mapping keeps every shared load at one
// wavefront per quarter warp (see ws_dmma_loop).
#include "common.cuh"
#include "mttkrp_internal.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace cpk {

constexpr int WS_CONSUMERS = 8;  // warps (warpgroups 0-1)
// + one producer warpgroup (warps 8-11; warp 8 works, 9-11 retire at once).
// setmaxnreg moves registers from the producer warpgroup to the consumers:
// per SMSP 2 x 232 + 1 x 40 registers x 32 lanes <= 16384 (see WsRegs).
constexpr int WS_THREADS = (WS_CONSUMERS + 4) * 32;
// 12-row tiles need 240 consumer registers (192 accumulators); their producer
// warpgroup then runs in 24 (2 x 240 + 24 <= 512 per SMSP, x 32 lanes).
template <int TM>
struct WsRegs {
  static constexpr int consumer = TM == 12 ? 240 : 232;
  static constexpr int producer = TM == 12 ? 24 : 40;
};

struct alignas(64) WsParams {
  CUtensorMap tm_y;
  CUtensorMap tm_f;
  CUtensorMap tm_o[3];
  int64_t dim_o[3];
  int64_t chunks_per_f, n_chunks, chunks_per_split;
  int32_t Ik, If, R, k;
  double* out;
  int64_t ldo, out_split_stride;
  const double* lam;
  int32_t y0, z0;  // first row block / split of this launch
  int32_t a_one_box;  // mode 0, DMMA: tm_y views the tensor as (16, I_1, I_0 / 16, ...) -> one box per stage
  int32_t b_one_box;  // DMMA, R % 16 == 0: tm_f views the factor as (16, rows, R / 16) -> one box per stage
  int* sem;           // split-K chain counters (one per output tile), or nullptr: partials / direct
  int32_t n_splits;
  // Khatri-Rao fold (DMMA only): the factor map holds W = KR(A_f, A_o0)
  // (rows i_f + I_f i_o0) and the first o-mode's factor is all ones, so
  // P_o stops changing with i_o0: an o-group runs og_len = chunks_per_f x
  // dim_o[0] chunks instead of chunks_per_f
  int32_t fold;
  int64_t og_len;  // chunks per o-group (the consumers' flush period)
};

// Epilogue prologue of the split-K chain (consumer threads only: the
// producer warpgroup may have retired, so a named barrier over the 256
// consumer threads).
__device__ __forceinline__ OutMode ws_chain_enter(const WsParams& p, int z, int tile) {
  const OutMode m = chain_mode(p.sem != nullptr, z, p.n_splits, p.lam != nullptr);
  if (p.sem) {
    if (threadIdx.x == 0) chain_wait(p.sem + tile, z);
    asm volatile("bar.sync 2, %0;\n" ::"n"(8 * 32) : "memory");
  }
  return m;
}
__device__ __forceinline__ void ws_chain_leave(const WsParams& p, int z, int tile) {
  if (!p.sem) return;
  asm volatile("bar.sync 2, %0;\n" ::"n"(8 * 32) : "memory");
  if (threadIdx.x == 0) {
    __threadfence();  // cumulative: the barrier ordered the consumers' stores before it
    st_release_gpu(p.sem + tile, z + 1);
  }
}

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// d += a * b as one DFMA whose position in the instruction stream ptxas keeps
// (volatile asm), so the snake order below survives scheduling.
__device__ __forceinline__ void dfma_ordered(double& d, double a, double b) {
  asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(d) : "d"(a), "d"(b));
}

// D += A (8x4, row) * B (4x8, col) on the FP64 tensor path.  Fragments
// (PTX ISA, mma.m8n8k4 .f64): a = A[lane / 4][lane % 4],
// b = B[lane % 4][lane / 4], d = D[lane / 4][2 (lane % 4) + {0, 1}].
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int RANK>
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, const int (&c)[RANK]) {
  const unsigned d = smem_u32(dst), b = smem_u32(bar);
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  if constexpr (RANK == 2)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(d),
        "l"(m), "r"(b), "r"(c[0]), "r"(c[1])
        : "memory");
  else if constexpr (RANK == 3)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(d),
        "l"(m), "r"(b), "r"(c[0]), "r"(c[1]), "r"(c[2])
        : "memory");
  else if constexpr (RANK == 4)
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(d),
        "l"(m), "r"(b), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3])
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];\n" ::"r"(d),
        "l"(m), "r"(b), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
        : "memory");
}

// DMMA consumer (TM == 0): warp tile 32 rows x 64 rank columns = 4 x 8
// m8n8k4 fragments, 64 accumulators per thread.  A DMMA moves 256 FMA per
// warp instruction against 32 for a DFMA, and its fragments are spread over
// the lanes without replication, so shared-memory wavefronts per flop fall
// ~6x below the DFMA outer product and the FP64 pipe (the same pipe: a mixed
// DFMA + DMMA stream never exceeds the DMMA peak, tools/microbench4.cu)
// becomes the only limit.  Each 8-deep k block runs as two k-steps, even k
// then odd k (the contraction order is free), so on the K-major swizzled
// panels one LDS.128 yields a thread's A fragments for both steps.
// o-group accumulation (OG): a chunk's Khatri-Rao rows are A_f rows times
// P_o, the product of the o-rows, and P_o only changes when the o-digits do
// -- every chunks_per_f chunks (an "o-group").  So the consumers run their
// DMMAs on the raw A_f rows and, at the end of each o-group, fold the
// group's accumulators into a running total kept in TMEM: total += acc o P_o.
// The same FP64 work as scaling every staged row, but issued by the
// consumers themselves at group ends instead of by the producer warps,
// whose DMULs starved behind the DMMAs and held up stages (c3: consumers
// waited ~6 % on `full`).  TMEM: 256 columns; warp w uses lanes
// 32 (w % 4).. and columns 128 (w / 4).. (its 64 doubles as 128 words).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// total (TMEM) += acc o P for one o-group, acc := 0.  p_s: the stage's o-rows
// (NO x BN); first: the total is still empty (no TMEM read).  The warp's
// 4 x NF fragments are 16 NF words per thread, moved 32 words (8 fragments)
// at a time: fragment (mf, nf) is words 4 (mf NF + nf) .. + 3.
template <int NO, int BN, int NF>
__device__ __forceinline__ void og_flush(double (&acc)[4][NF][2], uint32_t tbase, const double* p_s, int wn0, int lk,
                                         bool first) {
  // fragment nf = 2 q + e, accumulator v sits at column 16 q + 4 lk + 2 v + e
  // (dmma_col): the thread's columns of a fragment pair are 4 contiguous doubles
  double pj[NF][2];
#pragma unroll
  for (int q = 0; q < NF / 2; ++q)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int c = wn0 + 16 * q + 4 * lk + 2 * v;
      double2 x = *reinterpret_cast<const double2*>(p_s + c);
#pragma unroll
      for (int i = 1; i < NO; ++i) {
        const double2 w = *reinterpret_cast<const double2*>(p_s + i * BN + c);
        x.x *= w.x;
        x.y *= w.y;
      }
      pj[2 * q][v] = x.x;
      pj[2 * q + 1][v] = x.y;
    }
  constexpr int GROUPS = NF / 2;  // 32-word groups
#pragma unroll
  for (int g = 0; g < GROUPS; ++g) {
    uint32_t t[32];
    if (!first) {
      tmem_ld32(tbase + g * 32, t);
      tmem_wait_ld();
    }
#pragma unroll
    for (int f = 0; f < 8; ++f) {
      const int idx = g * 8 + f, mf = idx / NF, nf = idx % NF;
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int w = (f * 2 + v) * 2;
        const double old = first ? 0.0 : __hiloint2double(int(t[w + 1]), int(t[w]));
        const double nw = fma(acc[mf][nf][v], pj[nf][v], old);
        t[w] = uint32_t(__double2loint(nw));
        t[w + 1] = uint32_t(__double2hiint(nw));
        acc[mf][nf][v] = 0.0;
      }
    }
    tmem_st32(tbase + g * 32, t);
  }
  tmem_wait_st();
}

// The main loop over a CTA's chunks.  NA: fragments that do math (a warp
// whose 8 NF columns straddle the rank R runs only its live 16-column pairs:
// the rank tail of R = 2000 at tile 64 is 16 columns, 2 of 8 fragments; a
// warp with no live column, NA = 0, only keeps the stage protocol).  NA is a
// template argument so every variant is a fully unrolled, branch-free loop.
//
// Shared-memory layout and fragment mapping (conflict-free, every load an
// LDS.128 at its minimum of one wavefront per quarter warp):
//   * the k order inside each 16-deep panel is free, so k-step s in {0, 1}
//     of a panel gives lane quad lk the 16-byte k chunk
//     c = 2 lk + ((lk >> 1) ^ s) (s = 0: chunks 0 2 5 7, s = 1: 1 3 4 6),
//     i.e. k = 2 c + ph for the two DMMAs ph of the step;
//   * K-major tensor tiles (modes k > 0, TMA 128-byte swizzle, 16-deep
//     panels [m][16]): row m = 8 mf + lane / 4 reads chunk c ^ (m & 7); the
//     chunk set of a step holds no pair {x, x ^ 1}, so the two rows of a
//     quarter warp land on disjoint banks;
//   * M-major tensor tiles (mode 0) and the factor rows arrive as 16-wide
//     panels [k][16] (TMA boxes {16, BK}, 128-byte swizzle): row k holds
//     16 rows (columns) of the tile, chunk j at j ^ (k & 7); lanes read the
//     pair 2 (lane / 4), +1, so fragment 2 q + e covers tile rows (columns)
//     16 q + 2 (lane / 4) + e (dmma_row / dmma_col); k & 7 = (2 c + ph) & 7
//     takes 4 distinct even/odd values per step, so again no conflicts.
// The epilogue and the o-group scaling use the same row / column maps.
template <bool KMAJ>
__device__ __forceinline__ int dmma_row(int mf, int lr) {
  return KMAJ ? mf * 8 + lr : 16 * (mf >> 1) + 2 * lr + (mf & 1);
}
__device__ __forceinline__ int dmma_kchunk(int lk, int s) { return 2 * lk + ((lk >> 1) ^ s); }

template <bool KMAJ, int NA, bool OG, int NO, int BM, int BN, int NF, int BK, int STAGE_BYTES, int A_BYTES>
__device__ __forceinline__ void ws_dmma_loop(double (&acc)[4][NF][2], const uint8_t* smem, uint64_t* full,
                                             uint64_t* empty, int nst, int stages, int wm0, int wn0, int lane,
                                             uint32_t tbase, int64_t q0, int64_t og_len) {
  const int lr = lane >> 2, lk = lane & 3;
  bool first = true;
  int64_t qf = OG ? q0 % og_len : 0;  // position inside the o-group (og_len chunks long)
  for (int it = 0; it < nst; ++it) {
    const int s = it % stages;
    mbar_wait(&full[s], (it / stages) & 1);
    const uint8_t* st = smem + s * STAGE_BYTES;
    const double* a_s = reinterpret_cast<const double*>(st);
    const double* b_s = reinterpret_cast<const double*>(st + A_BYTES) + (wn0 >> 4) * (16 * BK);
#pragma unroll 2
    for (int kk = 0; kk < (NA > 0 ? BK : 0); kk += 8) {
      const int c = dmma_kchunk(lk, (kk >> 3) & 1);
      const int kr0 = (kk & ~15) + 2 * c;  // tile k of this lane's ph = 0 DMMA
      double a[4][2], b[NF][2];
      if constexpr (KMAJ) {
        const double* panel = a_s + (kk >> 4) * (BM * 16) + (wm0 + lr) * 16 + ((c ^ lr) << 1);
#pragma unroll
        for (int mf = 0; mf < 4; ++mf) {
          const double2 v = *reinterpret_cast<const double2*>(panel + mf * 8 * 16);
          a[mf][0] = v.x;
          a[mf][1] = v.y;
        }
      } else {
        const double* panel = a_s + (wm0 >> 4) * (16 * BK);
#pragma unroll
        for (int ph = 0; ph < 2; ++ph) {
          const int kr = kr0 + ph;
          const double* row = panel + kr * 16 + ((lr ^ (kr & 7)) << 1);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double2 v = *reinterpret_cast<const double2*>(row + q * (16 * BK));
            a[2 * q][ph] = v.x;
            a[2 * q + 1][ph] = v.y;
          }
        }
      }
#pragma unroll
      for (int ph = 0; ph < 2; ++ph) {
        const int kr = kr0 + ph;
        const double* row = b_s + kr * 16 + ((lr ^ (kr & 7)) << 1);
#pragma unroll
        for (int q = 0; q < NA / 2; ++q) {
          const double2 v = *reinterpret_cast<const double2*>(row + q * (16 * BK));
          b[2 * q][ph] = v.x;
          b[2 * q + 1][ph] = v.y;
        }
      }
#pragma unroll
      for (int ph = 0; ph < 2; ++ph)
#pragma unroll
        for (int mf = 0; mf < 4; ++mf)
#pragma unroll
          for (int nf = 0; nf < NA; ++nf) dmma_8x8x4(acc[mf][nf], a[mf][ph], b[nf][ph]);
    }
    if constexpr (OG && NA > 0) {
      if (++qf == og_len || it == nst - 1) {  // o-group ends: fold it into the total
        og_flush<NO, BN, NF>(acc, tbase, reinterpret_cast<const double*>(st + A_BYTES + BK * BN * 8), wn0, lk,
                             first);
        first = false;
        qf = 0;
      }
    }
    __syncwarp();
    if ((lane & 31) == 0) mbar_arrive(&empty[s]);
  }
}

// DMMA warp tiles: 32 rows x 8 NF rank columns, NF = min(8, BN / 8); narrow
// rank tiles (BN = 16, 32) keep 8 warps along the rows (BM = 256) with 16 /
// 32 accumulators per thread, and their small stages let more of them be in
// flight (the low-rank end streams the tensor at HBM rate).
template <int BN>
struct DmmaWarps {
  static constexpr int NF = BN >= 64 ? 8 : BN / 8;
  static constexpr int WARPS_N = BN >= 64 ? BN / 64 : 1;
};

template <bool KMAJ, bool OG, int NO, int BM, int BN, int BK, int STAGE_BYTES, int A_BYTES>
__device__ __forceinline__ void ws_consume_dmma(const uint8_t* smem, uint64_t* full, uint64_t* empty, int nst,
                                                const WsParams& p, int n0, int j0, int warp, int lane,
                                                int stages, uint32_t tmem, int64_t q0) {
  constexpr int WARPS_N = DmmaWarps<BN>::WARPS_N, NF = DmmaWarps<BN>::NF;
  const int wm0 = (warp / WARPS_N) * 32, wn0 = (warp % WARPS_N) * (8 * NF);
  const int lr = lane >> 2, lk = lane & 3;
  double acc[4][NF][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // this warp's live rank columns (warp-uniform; <= 0: none)
  const int live = p.R - j0 - wn0;
  // this warp's TMEM window: lanes 32 (warp % 4).., columns 128 (warp / 4)..
  const uint32_t tbase = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 128);
  const int64_t og_len = p.og_len;
#define CPK_DMMA_LOOP(NA_)                                                                                     \
  ws_dmma_loop<KMAJ, NA_, OG, NO, BM, BN, NF, BK, STAGE_BYTES, A_BYTES>(acc, smem, full, empty, nst, stages, wm0, \
                                                                        wn0, lane, tbase, q0, og_len)
  // every branch runs exactly one loop (a warp that skipped it would never
  // release its stages); plain compares, the last case catches the rest
  if (live <= 0) {
    CPK_DMMA_LOOP(0);
  } else if constexpr (NF == 2) {
    CPK_DMMA_LOOP(2);
  } else if constexpr (NF == 4) {
    if (live <= 16) CPK_DMMA_LOOP(2);
    else CPK_DMMA_LOOP(4);
  } else {
    if (live <= 16) CPK_DMMA_LOOP(2);
    else if (live <= 32) CPK_DMMA_LOOP(4);
    else if (live <= 48) CPK_DMMA_LOOP(6);
    else CPK_DMMA_LOOP(8);
  }
#undef CPK_DMMA_LOOP
  if constexpr (OG) {
    if (nst > 0 && live > 0) {  // the total -> acc registers for the epilogue
#pragma unroll
      for (int g = 0; g < NF / 2; ++g) {
        uint32_t t[32];
        tmem_ld32(tbase + g * 32, t);
        tmem_wait_ld();
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const int idx = g * 8 + f, mf = idx / NF, nf = idx % NF;
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int w = (f * 2 + v) * 2;
            acc[mf][nf][v] = __hiloint2double(int(t[w + 1]), int(t[w]));
          }
        }
      }
    }
  }

  const int zs = blockIdx.z + p.z0, tile = blockIdx.x + gridDim.x * (blockIdx.y + p.y0);
  double* out = p.out + (p.sem ? 0 : int64_t(zs) * p.out_split_stride);
  const OutMode om = ws_chain_enter(p, zs, tile);
#pragma unroll
  for (int mf = 0; mf < 4; ++mf) {
    const int n = n0 + wm0 + dmma_row<KMAJ>(mf, lr);
    if (n >= p.Ik) continue;
#pragma unroll
    for (int q = 0; q < NF / 2; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        // fragments 2q, 2q + 1 hold columns j, j + 1 (dmma_col)
        const int j = j0 + wn0 + 16 * q + 4 * lk + 2 * v;
        store_pair(out + int64_t(n) * p.ldo + j, j, p.R, (p.ldo & 1) == 0, acc[mf][2 * q][v], acc[mf][2 * q + 1][v],
                   p.lam, om);
      }
  }
  ws_chain_leave(p, zs, tile);
}

// ---------------------------------------------------------------- kernel
// Tile shapes (per-thread TM x 8 accumulators, 256 consumer threads):
//   TM = 8,  BN = 128 -> BM = 128 (16 x 16 threads), BK = 32
//   TM = 12, BN = 256 -> BM = 96  ( 8 x 32 threads), BK = 16
//   TM = 8,  BN = 64  -> BM = 256 (32 x  8 threads), BK = 16
// TM = 12 cuts shared-memory wavefronts per DFMA from 0.375 to 0.29: the A
// fragment (lane quads share a row -> 1 wavefront per 8 B) grows, the B
// fragment (4 distinct columns per quad -> 2 wavefronts per 8 B) does not.
// TM = 0 selects the DMMA consumer (mma.sync m8n8k4 f64): 8 warps of 32 x 64
// warp tiles, BN / 64 warps across the rank tile -> BM = 32 * 8 / (BN / 64):
//   BN = 64 -> BM = 256, BN = 128 -> BM = 128, BN = 256 -> BM = 64.
template <int TM, int BN>
struct WsTile {
  static constexpr int TX = BN / 8, TY = 256 / TX, BM = TY * TM;
};
template <int BN>
struct WsTile<0, BN> {
  static constexpr int WARPS_N = DmmaWarps<BN>::WARPS_N, WARPS_M = 8 / WARPS_N;
  static constexpr int TX = 8, TY = 0, BM = 32 * WARPS_M;
};

template <bool KMAJ, int NO, int TM, int BN, int BK, int STAGES>
struct WsCfg {
  static constexpr int D = NO + 2;  // tensor order
  static constexpr int TX = WsTile<TM, BN>::TX, TY = WsTile<TM, BN>::TY, BM = WsTile<TM, BN>::BM;
  static constexpr int A_ELEMS = BM * BK;
  static constexpr int B_ELEMS = BK * BN;
  static constexpr int P_ELEMS = NO * BN;
  static constexpr int A_BYTES = A_ELEMS * 8, B_BYTES = B_ELEMS * 8, P_BYTES = P_ELEMS * 8;
  static constexpr int STAGE_BYTES = ((A_BYTES + B_BYTES + P_BYTES + 1023) / 1024) * 1024;
  static constexpr int TX_BYTES = A_BYTES + B_BYTES + P_BYTES;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 256 /*barriers*/;
  static_assert(TM % 2 == 0 && BK % 16 == 0 && BM <= 256 && BN <= 256, "tile shape");
  static_assert(TM != 0 || BN == 16 || BN == 32 || (BN >= 64 && BN % 64 == 0), "DMMA rank tile 16, 32 or 64 k");
  static_assert((TX >= 8) && (TX % 8 == 0), "8 lanes per warp row");
};

template <bool KMAJ, int NO, int TM, int BN, int BK, int STAGES>
__global__ void __launch_bounds__(WS_THREADS, 1) mttkrp_f64_ws_sm100(const __grid_constant__ WsParams p) {
  using C = WsCfg<KMAJ, NO, TM, BN, BK, STAGES>;
  constexpr int BM = C::BM, TY = C::TY, TX = C::TX;
  // dynamic shared memory starts at the CTA window base (no static smem), so
  // it is 1024-byte aligned as the 128-byte swizzle requires; indexing the
  // __shared__ array directly keeps every access an LDS (not a generic LD)
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* full_tma = bar;             // TMA bytes landed
  uint64_t* full = bar + STAGES;        // Khatri-Rao rows formed
  uint64_t* empty = bar + 2 * STAGES;   // consumers done

  // DMMA tiles with o-modes fold the o-row product per o-group (OG, see
  // og_flush); the producer warps then only issue TMA
  constexpr bool OG = TM == 0 && NO > 0;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 3 * STAGES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q0 = int64_t(blockIdx.z + p.z0) * p.chunks_per_split;
  const int nst = int(min(p.n_chunks, q0 + p.chunks_per_split) - q0);
  const int j0 = blockIdx.x * BN;
  const int n0 = (blockIdx.y + p.y0) * BM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_tma[s], 1);
      mbar_init(&full[s], 4);  // one arrive per producer warp
      mbar_init(&empty[s], WS_CONSUMERS);
    }
    fence_barrier_init();
  }
  if constexpr (OG) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  }
  __syncthreads();
  uint32_t tmem = 0;
  if constexpr (OG) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    tmem = *tslot;
  }

  if (warp >= WS_CONSUMERS) {
    // ================================================================ producer
    // warp 8 issues the TMA loads; all four producer warps form the
    // Khatri-Rao rows of a landed stage, one column pair per thread
    setmaxnreg_dec<WsRegs<TM>::producer>();
    const int pt = threadIdx.x - WS_CONSUMERS * 32;  // 0..127
    const bool issuer = warp == WS_CONSUMERS;
    if (issuer && lane == 0) {
      prefetch_tmap(&p.tm_y);
      prefetch_tmap(&p.tm_f);
#pragma unroll
      for (int i = 0; i < NO; ++i) prefetch_tmap(&p.tm_o[i]);
    }
    // extents are < 2^31 (tensor-map coordinates), so the cursor is 32-bit
    int qf, od[NO > 0 ? NO : 1];
    {
      qf = int(q0 % p.chunks_per_f);
      int64_t rest = q0 / p.chunks_per_f;
#pragma unroll
      for (int i = 0; i < NO; ++i) {
        od[i] = int(rest % p.dim_o[i]);
        rest /= p.dim_o[i];
      }
    }
    auto issue = [&](int t) {
      const int s = t % STAGES;
      if (t >= STAGES) mbar_wait(&empty[s], ((t / STAGES) - 1) & 1);
      if (lane == 0) {
        uint8_t* st = smem + s * C::STAGE_BYTES;
        double* a_s = reinterpret_cast<double*>(st);
        double* b_s = reinterpret_cast<double*>(st + C::A_BYTES);
        double* p_s = reinterpret_cast<double*>(st + C::A_BYTES + C::B_BYTES);
        mbar_expect_tx(&full_tma[s], C::TX_BYTES);
        const int if0 = qf * BK;
        // tensor-map coordinates, mode 0 first; o digits fill the non-k,
        // non-f slots in ascending mode order (closed form, no local arrays)
        int c[C::D];
        if constexpr (!KMAJ) {
          c[0] = n0;
          c[1] = if0;
#pragma unroll
          for (int m = 2; m < C::D; ++m) c[m] = od[m - 2];
        } else {
          c[0] = if0;
#pragma unroll
          for (int m = 1; m < C::D; ++m) {
            const int lo_i = m - 1 < NO ? m - 1 : NO - 1;  // o index when m < k
            const int hi_i = m >= 2 ? m - 2 : 0;            // o index when m > k
            c[m] = (m == p.k) ? n0 : (m > p.k ? od[hi_i] : od[lo_i]);
          }
        }
        if (KMAJ) {
#pragma unroll
          for (int pn = 0; pn < BK / 16; ++pn) {  // one 16-deep swizzled panel per box
            c[0] = if0 + 16 * pn;
            tma_load<C::D>(a_s + pn * (BM * 16), &p.tm_y, &full_tma[s], c);
          }
        } else if (TM == 0) {
          bool done = false;
          if constexpr (C::D < 5) {
            if (p.a_one_box) {  // all BM / 16 panels as one box {16, BK, BM / 16}
              int c1[C::D + 1];
              c1[0] = 0;
              c1[1] = if0;
              c1[2] = n0 >> 4;
#pragma unroll
              for (int m = 2; m < C::D; ++m) c1[m + 1] = od[m - 2];
              tma_load<C::D + 1>(a_s, &p.tm_y, &full_tma[s], c1);
              done = true;
            }
          }
          if (!done) {
#pragma unroll
            for (int pm = 0; pm < BM / 16; ++pm) {  // 16-row swizzled panels [k][16] (DMMA layout)
              c[0] = n0 + 16 * pm;
              tma_load<C::D>(a_s + pm * (16 * BK), &p.tm_y, &full_tma[s], c);
            }
          }
        } else {
          tma_load<C::D>(a_s, &p.tm_y, &full_tma[s], c);
        }
        // factor rows of the chunk: A_f rows, or (fold) W rows i_f + I_f i_o0
        const int ifb = p.fold ? (qf + int(p.chunks_per_f) * od[0]) * BK : if0;
        if (TM == 0 && p.b_one_box) {  // all BN / 16 column panels as one box {16, BK, BN / 16}
          const int cf[3] = {0, ifb, j0 >> 4};
          tma_load<3>(b_s, &p.tm_f, &full_tma[s], cf);
        } else if (TM == 0) {
#pragma unroll
          for (int pc = 0; pc < BN / 16; ++pc) {  // 16-column swizzled panels [k][16]
            const int cf[2] = {j0 + 16 * pc, ifb};
            tma_load<2>(b_s + pc * (16 * BK), &p.tm_f, &full_tma[s], cf);
          }
        } else {
          const int cf[2] = {j0, if0};
          tma_load<2>(b_s, &p.tm_f, &full_tma[s], cf);
        }
#pragma unroll
        for (int i = 0; i < NO; ++i) {
          const int co[2] = {j0, od[i]};
          tma_load<2>(p_s + i * BN, &p.tm_o[i], &full_tma[s], co);
        }
      }
      // advance the odometer (in-slice walk, _kernels.py:135-147)
      if (++qf == int(p.chunks_per_f)) {
        qf = 0;
#pragma unroll
        for (int i = 0; i < NO; ++i) {
          if (++od[i] < int(p.dim_o[i])) break;
          od[i] = 0;
        }
      }
    };
    if (issuer)
      for (int t = 0; t < STAGES - 1 && t < nst; ++t) issue(t);
    if constexpr (OG) {  // nothing to scale: just keep the TMA ring full
      if (issuer)
        for (int t = STAGES - 1; t < nst; ++t) issue(t);
      return;
    }
    constexpr int PAIRS = BN / 2;                  // column pairs per row
    constexpr int ROW_STEP = 128 / PAIRS;          // producer threads per pair
    const int pair = pt % PAIRS, row0 = pt / PAIRS;
    // Scale a stage as soon as its bytes land (consumers are still on the
    // previous one), then (warp 8) refill the slot the consumers released.
    for (int it = 0; it < nst; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full_tma[s], (it / STAGES) & 1);
      if (NO > 0) {
        // Khatri-Rao rows: B[k][j] *= prod_o A_o[o][j]
        uint8_t* st = smem + s * C::STAGE_BYTES;
        double* b_s = reinterpret_cast<double*>(st + C::A_BYTES);
        const double* p_s = reinterpret_cast<const double*>(st + C::A_BYTES + C::B_BYTES);
        double2 pr = *reinterpret_cast<const double2*>(p_s + 2 * pair);
#pragma unroll
        for (int i = 1; i < NO; ++i) {
          const double2 v = *reinterpret_cast<const double2*>(p_s + i * BN + 2 * pair);
          pr.x *= v.x;
          pr.y *= v.y;
        }
        // loads of a batch of rows first, then the DMULs, then the stores:
        // one round trip of shared-memory latency per batch instead of one
        // per row (c3: 4.26 -> 4.11 ms per mode); batches of 8 rows keep the
        // producer inside its setmaxnreg budget
        constexpr int NR = (BK + ROW_STEP - 1) / ROW_STEP, NB = NR < 8 ? NR : 8;
#pragma unroll
        for (int b0 = 0; b0 < NR; b0 += NB) {
          double2 v[NB];
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            const int k = row0 + (b0 + i) * ROW_STEP;
            if (b0 + i < NR && k < BK) v[i] = *reinterpret_cast<const double2*>(b_s + k * BN + 2 * pair);
          }
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            v[i].x *= pr.x;
            v[i].y *= pr.y;
          }
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            const int k = row0 + (b0 + i) * ROW_STEP;
            if (b0 + i < NR && k < BK) *reinterpret_cast<double2*>(b_s + k * BN + 2 * pair) = v[i];
          }
        }
        // generic-proxy writes must be ordered before the next TMA into this buffer
        fence_proxy_async();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
      if (issuer && it + STAGES - 1 < nst) issue(it + STAGES - 1);
    }
    return;
  }

  // ================================================================== consumers
  setmaxnreg_inc<WsRegs<TM>::consumer>();
  if constexpr (TM == 0) {
    // with OG the consumers take a stage as soon as its bytes land
    ws_consume_dmma<KMAJ, OG, NO, BM, BN, BK, C::STAGE_BYTES, C::A_BYTES>(smem, OG ? full_tma : full, empty, nst, p,
                                                                          n0, j0, warp, lane, STAGES, tmem, q0);
    if constexpr (OG) {  // all consumers are done with TMEM before warp 0 frees it
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      asm volatile("bar.sync 1, %0;\n" ::"n"(WS_CONSUMERS * 32) : "memory");
      if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
      }
    }
    return;
  }
  if constexpr (TM != 0) {
  constexpr int WX = 8, WY = 4, WARPS_X = TX / WX;
  const int ty = (warp / WARPS_X) * WY + lane / WX;
  const int tx = (warp % WARPS_X) * WX + lane % WX;

  double acc[TM > 0 ? TM : 1][8];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;

  for (int it = 0; it < nst; ++it) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const uint8_t* st = smem + s * C::STAGE_BYTES;
    const double* a_s = reinterpret_cast<const double*>(st);
    const double* b_s = reinterpret_cast<const double*>(st + C::A_BYTES);
    if constexpr (TM == 8) {
      // k pairs: one LDS.128 gives (m, k..k+1) in the K-major layout
#pragma unroll 4
      for (int kk = 0; kk < BK; kk += 2) {
        double a[8][2];
        if (KMAJ) {
          const double* panel = a_s + (kk >> 4) * (BM * 16);
          const int chunk = (kk & 15) >> 1;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int m = 2 * ty + (r & 1) + 2 * TY * (r >> 1);
            const double2 v = *reinterpret_cast<const double2*>(panel + m * 16 + ((chunk ^ (m & 7)) << 1));
            a[r][0] = v.x;
            a[r][1] = v.y;
          }
        } else {
#pragma unroll
          for (int kq = 0; kq < 2; ++kq)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const double2 v = *reinterpret_cast<const double2*>(a_s + (kk + kq) * BM + 2 * ty + 2 * TY * i);
              a[2 * i][kq] = v.x;
              a[2 * i + 1][kq] = v.y;
            }
        }
#pragma unroll
        for (int kq = 0; kq < 2; ++kq) {
          double b[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double2 v = *reinterpret_cast<const double2*>(b_s + (kk + kq) * BN + 2 * tx + 2 * TX * i);
            b[2 * i] = v.x;
            b[2 * i + 1] = v.y;
          }
          // snake order: every DFMA shares one operand with the previous one,
          // so one of its 64-bit sources comes from the operand-reuse cache
          // (register-only outer product: 32.5 vs 31.1 TFLOP/s for row order,
          // 24.6 with no sharing -- tools/microbench3.cu)
#pragma unroll
          for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const int c = (r & 1) ? 7 - cc : cc;
              dfma_ordered(acc[r][c], a[r][kq], b[c]);
            }
        }
      }
    } else {
      // single k: B fragment first, then the TM rows streamed through.  Rows
      // 2ty+p+2TY*i share (m & 7) across i, so the swizzled column offset is
      // one value per (k, p) and the row offsets are compile-time strides.
      const double* arow0 = a_s + (2 * ty) * 16;
      const double* arow1 = arow0 + 16;
      const int swz0 = (2 * ty) & 7, swz1 = (2 * ty + 1) & 7;
#pragma unroll 1
      for (int k = 0; k < BK; ++k) {
        double b[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 v = *reinterpret_cast<const double2*>(b_s + k * BN + 2 * tx + 2 * TX * i);
          b[2 * i] = v.x;
          b[2 * i + 1] = v.y;
        }
#pragma unroll
        for (int i = 0; i < TM / 2; ++i) {
          double a0, a1;
          if (KMAJ) {
            static_assert(!KMAJ || (2 * TY) % 8 == 0, "row stride keeps the swizzle phase");
            const int pofs = (k >> 4) * (BM * 16) + 2 * TY * 16 * i;
            const int chunk = (k & 15) >> 1, odd = k & 1;
            a0 = arow0[pofs + ((chunk ^ swz0) << 1) + odd];
            a1 = arow1[pofs + ((chunk ^ swz1) << 1) + odd];
          } else {
            const double2 v = *reinterpret_cast<const double2*>(a_s + k * BM + 2 * ty + 2 * TY * i);
            a0 = v.x;
            a1 = v.y;
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[2 * i][c] = fma(a0, b[c], acc[2 * i][c]);
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[2 * i + 1][c] = fma(a1, b[c], acc[2 * i + 1][c]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // epilogue: partial, chained or final (lam-folded) tile -> out
  const int zs = blockIdx.z + p.z0, tile = blockIdx.x + gridDim.x * (blockIdx.y + p.y0);
  double* out = p.out + (p.sem ? 0 : int64_t(zs) * p.out_split_stride);
  const OutMode om = ws_chain_enter(p, zs, tile);
#pragma unroll
  for (int r = 0; r < TM; ++r) {
    const int n = n0 + 2 * ty + (r & 1) + 2 * TY * (r >> 1);
    if (n >= p.Ik) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = j0 + 2 * tx + 2 * TX * i;
      store_pair(out + int64_t(n) * p.ldo + j, j, p.R, (p.ldo & 1) == 0, acc[r][2 * i], acc[r][2 * i + 1], p.lam,
                 om);
    }
  }
  ws_chain_leave(p, zs, tile);
  }  // TM != 0
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

static int encode(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                  const cuuint32_t* box, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) return fail(CPK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CPK_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return CPK_OK;
}

template <bool KMAJ, int NO, int TM, int BN, int BK>
static void ws_kernel(const void** fn, size_t* smem) {
  constexpr int stage = WsCfg<KMAJ, NO, TM, BN, BK, 1>::STAGE_BYTES;
  constexpr int fit = (227 * 1024 - 256) / stage;
  // narrow rank tiles are HBM-bound: more of their (small) stages in flight
  constexpr int cap = (TM == 0 && BN < 64) ? 6 : 4;
  constexpr int S = fit > cap ? cap : fit;
  static_assert(S >= 2, "two stages must fit");
  *fn = reinterpret_cast<const void*>(&mttkrp_f64_ws_sm100<KMAJ, NO, TM, BN, BK, S>);
  *smem = WsCfg<KMAJ, NO, TM, BN, BK, S>::SMEM;
}

template <int TM, int BN, int BK>
static void ws_pick(bool kmaj, int no, const void** fn, size_t* smem) {
  if (kmaj) {
    if (no == 0) ws_kernel<true, 0, TM, BN, BK>(fn, smem);
    else if (no == 1) ws_kernel<true, 1, TM, BN, BK>(fn, smem);
    else if (no == 2) ws_kernel<true, 2, TM, BN, BK>(fn, smem);
    else ws_kernel<true, 3, TM, BN, BK>(fn, smem);
  } else {
    if (no == 0) ws_kernel<false, 0, TM, BN, BK>(fn, smem);
    else if (no == 1) ws_kernel<false, 1, TM, BN, BK>(fn, smem);
    else if (no == 2) ws_kernel<false, 2, TM, BN, BK>(fn, smem);
    else ws_kernel<false, 3, TM, BN, BK>(fn, smem);
  }
}

bool ws_shape(int rank_tile, int math, int* block_rows, int* block_k) {
  if (math == WS_MATH_DMMA) {
    switch (rank_tile) {
      case 16: *block_rows = 256; *block_k = 16; return true;
      case 32: *block_rows = 256; *block_k = 16; return true;
      case 64: *block_rows = 256; *block_k = 16; return true;
      case 128: *block_rows = 128; *block_k = 32; return true;
      case 256: *block_rows = 64; *block_k = 16; return true;
      default: return false;
    }
  }
  switch (rank_tile) {
    case 64: *block_rows = 256; *block_k = 16; return true;   // TM 8
    case 128: *block_rows = 128; *block_k = 32; return true;  // TM 8
    case 256: *block_rows = 96; *block_k = 16; return true;   // TM 12
    default: return false;
  }
}

bool ws_eligible(const WsRequest& r) {
  int bm, bk;
  if (!ws_shape(r.rank_tile, r.math, &bm, &bk)) return false;
  if (r.d < 2 || r.d > 5 || r.n_o > 3) return false;
  if (r.block_k != bk) return false;
  if (r.dims[0] % 2 != 0) return false;
  for (int m = 0; m < r.d; ++m)
    if (r.dims[m] >= (int64_t(1) << 31)) return false;
  if ((reinterpret_cast<uintptr_t>(r.y) & 15) != 0) return false;
  for (int m = 0; m < r.d; ++m) {
    if (m == r.k) continue;
    if ((reinterpret_cast<uintptr_t>(r.factors[m]) & 15) != 0 || (r.ld[m] % 2) != 0) return false;
  }
  return true;
}

int launch_ws(const WsRequest& r, cudaStream_t st) {
  int BM, BK;
  if (!ws_shape(r.rank_tile, r.math, &BM, &BK)) return fail(CPK_ERR_PARAM, "no TMA tile for rank_tile %d", r.rank_tile);
  const int BN = r.rank_tile;
  WsParams p;
  memset(&p, 0, sizeof(p));
  const int d = r.d, k = r.k, f = k == 0 ? 1 : 0;
  cuuint64_t gdim[5], gstr[4];
  int64_t s = 1;
  for (int m = 0; m < d; ++m) {
    gdim[m] = cuuint64_t(r.dims[m]);
    if (m > 0) gstr[m - 1] = cuuint64_t(s * 8);
    s *= r.dims[m];
  }
  cuuint32_t box[5];
  int rc;
  const bool dmma = r.math == WS_MATH_DMMA;  // DMMA consumers read 16-wide swizzled panels
  static const bool one_box_off = getenv("CPK_WS_PANEL_BOXES") != nullptr;  // A/B switch: per-panel boxes
  if (k == 0 && dmma && d < 5 && r.dims[0] % 16 == 0 && !one_box_off) {
    // (i_0 mod 16, i_1, i_0 / 16, i_2, ...): one box {16, BK, BM / 16} lands
    // the BM / 16 swizzled panels [k][16] of a stage in order
    cuuint64_t pdim[5], pstr[4];
    cuuint32_t pbox[5];
    pdim[0] = 16;
    pdim[1] = gdim[1];
    pdim[2] = gdim[0] / 16;
    pstr[0] = gstr[0];  // i_1
    pstr[1] = 16 * 8;   // i_0 / 16
    pbox[0] = 16;
    pbox[1] = cuuint32_t(BK);
    pbox[2] = cuuint32_t(BM / 16);
    for (int m = 2; m < d; ++m) {
      pdim[m + 1] = gdim[m];
      pstr[m] = gstr[m - 1];
      pbox[m + 1] = 1;
    }
    rc = encode(&p.tm_y, r.y, d + 1, pdim, pstr, pbox, CU_TENSOR_MAP_SWIZZLE_128B);
    p.a_one_box = 1;
  } else if (k == 0) {
    for (int m = 0; m < d; ++m) box[m] = 1;
    box[0] = cuuint32_t(dmma ? 16 : BM);
    box[1] = cuuint32_t(BK);
    rc = encode(&p.tm_y, r.y, d, gdim, gstr, box, dmma ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
  } else {
    for (int m = 0; m < d; ++m) box[m] = 1;
    box[0] = 16;
    box[k] = cuuint32_t(BM);
    rc = encode(&p.tm_y, r.y, d, gdim, gstr, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (rc) return rc;
  int o0 = -1;  // the first o-mode (the fold's second KR factor)
  for (int m = 0; m < d; ++m)
    if (m != k && m != f) {
      o0 = m;
      break;
    }
  if (r.fold && (r.math != WS_MATH_DMMA || o0 < 0 || r.dims[f] % BK != 0))
    return fail(CPK_ERR_PARAM, "Khatri-Rao fold needs the DMMA engine, an o-mode and I_f %% %d == 0", BK);
  p.fold = r.fold ? 1 : 0;
  p.og_len = 0;  // set below from chunks_per_f
  {
    // fold: factors[f] is W (I_f I_o0 rows) -- see WsParams::fold
    const cuuint64_t frows = cuuint64_t(r.fold ? r.dims[f] * r.dims[o0] : r.dims[f]);
    static const bool b_boxes_off = getenv("CPK_WS_PANEL_BOXES") != nullptr;  // A/B: per-panel boxes
    if (dmma && r.rank % 16 == 0 && !b_boxes_off) {
      // (column mod 16, row, column / 16): every panel column < R, so the
      // view never reads past a row; panels past R zero-fill
      const cuuint64_t fd[3] = {16, frows, cuuint64_t(r.rank / 16)};
      const cuuint64_t fs[2] = {cuuint64_t(r.ld[f] * 8), 16 * 8};
      const cuuint32_t fb[3] = {16, cuuint32_t(BK), cuuint32_t(BN / 16)};
      rc = encode(&p.tm_f, r.factors[f], 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_128B);
      p.b_one_box = 1;
    } else {
      const cuuint64_t fd[2] = {cuuint64_t(r.rank), frows};
      const cuuint64_t fs[1] = {cuuint64_t(r.ld[f] * 8)};
      const cuuint32_t fb[2] = {cuuint32_t(dmma ? 16 : BN), cuuint32_t(BK)};
      rc = encode(&p.tm_f, r.factors[f], 2, fd, fs, fb, dmma ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
    }
    if (rc) return rc;
  }
  int oi = 0;
  for (int m = 0; m < d; ++m) {
    if (m == k || m == f) continue;
    const cuuint64_t od[2] = {cuuint64_t(r.rank), cuuint64_t(r.dims[m])};
    const cuuint64_t os[1] = {cuuint64_t(r.ld[m] * 8)};
    const cuuint32_t ob[2] = {cuuint32_t(BN), 1};
    rc = encode(&p.tm_o[oi], r.factors[m], 2, od, os, ob, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
    p.dim_o[oi] = r.dims[m];
    ++oi;
  }
  p.chunks_per_f = (r.dims[f] + BK - 1) / BK;
  p.n_chunks = p.chunks_per_f;
  for (int i = 0; i < oi; ++i) p.n_chunks *= p.dim_o[i];
  p.chunks_per_split = (p.n_chunks + r.splits - 1) / r.splits;
  p.og_len = p.fold ? p.chunks_per_f * p.dim_o[0] : p.chunks_per_f;
  p.Ik = int(r.dims[k]);
  p.If = int(r.dims[f]);
  p.R = int(r.rank);
  p.k = k;
  p.out = r.out;
  p.ldo = r.ldo;
  p.out_split_stride = r.out_split_stride;
  p.lam = r.lam;
  p.y0 = r.y0;
  p.z0 = r.z0;
  p.sem = r.sem;
  p.n_splits = r.splits;

  const void* fn = nullptr;
  size_t smem = 0;
  const bool kmaj = k != 0;
  const int no = r.n_o;
  if (r.math == WS_MATH_DMMA) {
    if (BN == 128) ws_pick<0, 128, 32>(kmaj, no, &fn, &smem);
    else if (BN == 256) ws_pick<0, 256, 16>(kmaj, no, &fn, &smem);
    else if (BN == 32) ws_pick<0, 32, 16>(kmaj, no, &fn, &smem);
    else if (BN == 16) ws_pick<0, 16, 16>(kmaj, no, &fn, &smem);
    else ws_pick<0, 64, 16>(kmaj, no, &fn, &smem);
  } else if (BN == 128) ws_pick<8, 128, 32>(kmaj, no, &fn, &smem);
  else if (BN == 256) ws_pick<12, 256, 16>(kmaj, no, &fn, &smem);
  else ws_pick<8, 64, 16>(kmaj, no, &fn, &smem);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return check_launch("ws set smem");
  const int64_t gx = (r.rank + BN - 1) / BN;
  if (r.z1 - r.z0 > 65535) return fail(CPK_ERR_PARAM, "too many splits for one launch");
  // row blocks beyond the 65535 grid-y limit (I_k > 16.7 M rows at 256-row
  // tiles) go in several launches; p.y0 keeps the global row block
  for (int32_t y = r.y0; y < r.y1; y += 65535) {
    p.y0 = y;
    dim3 grid(unsigned(gx), unsigned(std::min(r.y1 - y, 65535)), unsigned(r.z1 - r.z0));
    void* args[] = {&p};
    cudaError_t e = cudaLaunchKernel(fn, grid, dim3(WS_THREADS), args, smem, st);
    if (e != cudaSuccess) return fail(CPK_ERR_CUDA, "ws launch: %s", cudaGetErrorString(e));
  }
  return CPK_OK;
}

}  // namespace cpk
