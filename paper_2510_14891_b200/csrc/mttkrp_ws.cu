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
//   mode 0 (M-major): box {BM, BK} -> As[k][m], no swizzle.
//   mode k>0 (K-major): two boxes {16, BM} (one per 16-deep panel) with the
//     128-byte swizzle -> panel[m][16] where the 16-byte chunk c of row m
//     lives at chunk c ^ (m & 7): the 4 rows a warp quarter reads land in
//     distinct banks.
#include "common.cuh"
#include "mttkrp_internal.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

namespace cpk {

constexpr int WS_BM = 128, WS_BN = 128, WS_BK = 32;
constexpr int WS_CONSUMERS = 8;  // warps (warpgroups 0-1)
// + one producer warpgroup (warps 8-11; warp 8 works, 9-11 retire at once).
// setmaxnreg moves registers from the producer warpgroup to the consumers:
// per SMSP 2 x 232 + 1 x 40 registers x 32 lanes <= 16384.
constexpr int WS_THREADS = (WS_CONSUMERS + 4) * 32;
constexpr int WS_CONSUMER_REGS = 232, WS_PRODUCER_REGS = 40;

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
};

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

// ---------------------------------------------------------------- kernel
template <bool KMAJ, int NO, int STAGES>
struct WsCfg {
  static constexpr int D = NO + 2;                       // tensor order
  static constexpr int A_ELEMS = WS_BM * WS_BK;          // 32 KiB
  static constexpr int B_ELEMS = WS_BK * WS_BN;          // 32 KiB
  static constexpr int P_ELEMS = NO * WS_BN;
  static constexpr int A_BYTES = A_ELEMS * 8, B_BYTES = B_ELEMS * 8, P_BYTES = P_ELEMS * 8;
  static constexpr int STAGE_BYTES = ((A_BYTES + B_BYTES + P_BYTES + 1023) / 1024) * 1024;
  static constexpr int TX_BYTES = A_BYTES + B_BYTES + P_BYTES;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 256 /*barriers*/;
};

template <bool KMAJ, int NO, int STAGES>
__global__ void __launch_bounds__(WS_THREADS, 1) mttkrp_f64_ws_sm100(const __grid_constant__ WsParams p) {
  using C = WsCfg<KMAJ, NO, STAGES>;
  // dynamic shared memory starts at the CTA window base (no static smem), so
  // it is 1024-byte aligned as the 128-byte swizzle requires; indexing the
  // __shared__ array directly keeps every access an LDS (not a generic LD)
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* full_tma = bar;             // TMA bytes landed
  uint64_t* full = bar + STAGES;        // Khatri-Rao rows formed
  uint64_t* empty = bar + 2 * STAGES;   // consumers done

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q0 = int64_t(blockIdx.z) * p.chunks_per_split;
  const int nst = int(min(p.n_chunks, q0 + p.chunks_per_split) - q0);
  const int j0 = blockIdx.x * WS_BN;
  const int n0 = blockIdx.y * WS_BM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_tma[s], 1);
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WS_CONSUMERS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp >= WS_CONSUMERS) {
    // ================================================================ producer
    setmaxnreg_dec<WS_PRODUCER_REGS>();
    if (warp != WS_CONSUMERS) return;
    if (lane == 0) {
      prefetch_tmap(&p.tm_y);
      prefetch_tmap(&p.tm_f);
#pragma unroll
      for (int i = 0; i < NO; ++i) prefetch_tmap(&p.tm_o[i]);
    }
    // chunk cursor for the TMA issue side (runs STAGES-1 chunks ahead)
    int64_t qf, od[NO > 0 ? NO : 1];
    {
      qf = q0 % p.chunks_per_f;
      int64_t rest = q0 / p.chunks_per_f;
#pragma unroll
      for (int i = 0; i < NO; ++i) {
        od[i] = rest % p.dim_o[i];
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
        const int if0 = int(qf) * WS_BK;
        int c[C::D];
        // o digits fill the non-k, non-f slots in ascending mode order
        {
          int oi = 0;
#pragma unroll
          for (int m = 0; m < C::D; ++m) {
            const bool is_k = KMAJ ? (m == p.k) : (m == 0);
            const bool is_f = KMAJ ? (m == 0) : (m == 1);
            if (is_k) {
              c[m] = n0;
            } else if (is_f) {
              c[m] = if0;
            } else {
              int v = 0;
#pragma unroll
              for (int i = 0; i < NO; ++i)
                if (i == oi) v = int(od[i]);
              c[m] = v;
              ++oi;
            }
          }
        }
        if (KMAJ) {
          tma_load<C::D>(a_s, &p.tm_y, &full_tma[s], c);
          c[0] = if0 + 16;
          tma_load<C::D>(a_s + WS_BM * 16, &p.tm_y, &full_tma[s], c);
        } else {
          tma_load<C::D>(a_s, &p.tm_y, &full_tma[s], c);
        }
        const int cf[2] = {j0, if0};
        tma_load<2>(b_s, &p.tm_f, &full_tma[s], cf);
#pragma unroll
        for (int i = 0; i < NO; ++i) {
          const int co[2] = {j0, int(od[i])};
          tma_load<2>(p_s + i * WS_BN, &p.tm_o[i], &full_tma[s], co);
        }
      }
      // advance the odometer (in-slice walk, _kernels.py:135-147)
      if (++qf == p.chunks_per_f) {
        qf = 0;
#pragma unroll
        for (int i = 0; i < NO; ++i) {
          if (++od[i] < p.dim_o[i]) break;
          od[i] = 0;
        }
      }
    };
    for (int t = 0; t < STAGES - 1 && t < nst; ++t) issue(t);
    // Scale a stage as soon as its bytes land (consumers are still on the
    // previous one), then refill the slot the consumers released last.
    for (int it = 0; it < nst; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full_tma[s], (it / STAGES) & 1);
      if (NO > 0) {
        // Khatri-Rao rows: B[k][j] *= prod_o A_o[o][j]; lane owns column
        // pairs 2*lane and 2*lane + 64
        uint8_t* st = smem + s * C::STAGE_BYTES;
        double* b_s = reinterpret_cast<double*>(st + C::A_BYTES);
        const double* p_s = reinterpret_cast<const double*>(st + C::A_BYTES + C::B_BYTES);
        double2 pa = *reinterpret_cast<const double2*>(p_s + 2 * lane);
        double2 pb = *reinterpret_cast<const double2*>(p_s + 64 + 2 * lane);
#pragma unroll
        for (int i = 1; i < NO; ++i) {
          const double2 qa = *reinterpret_cast<const double2*>(p_s + i * WS_BN + 2 * lane);
          const double2 qb = *reinterpret_cast<const double2*>(p_s + i * WS_BN + 64 + 2 * lane);
          pa.x *= qa.x;
          pa.y *= qa.y;
          pb.x *= qb.x;
          pb.y *= qb.y;
        }
#pragma unroll 8
        for (int k = 0; k < WS_BK; ++k) {
          double2* ra = reinterpret_cast<double2*>(b_s + k * WS_BN + 2 * lane);
          double2* rb = reinterpret_cast<double2*>(b_s + k * WS_BN + 64 + 2 * lane);
          double2 va = *ra, vb = *rb;
          va.x *= pa.x;
          va.y *= pa.y;
          vb.x *= pb.x;
          vb.y *= pb.y;
          *ra = va;
          *rb = vb;
        }
        // generic-proxy writes must be ordered before the next TMA into this buffer
        fence_proxy_async();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
      if (it + STAGES - 1 < nst) issue(it + STAGES - 1);
    }
    return;
  }

  // ================================================================== consumers
  setmaxnreg_inc<WS_CONSUMER_REGS>();
  constexpr int TY = WS_BM / 8, TX = WS_BN / 8;  // 16 x 16 threads, 8x8 each
  constexpr int WX = 8, WY = 4, WARPS_X = TX / WX;
  const int ty = (warp / WARPS_X) * WY + lane / WX;
  const int tx = (warp % WARPS_X) * WX + lane % WX;

  double acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;

  for (int it = 0; it < nst; ++it) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const uint8_t* st = smem + s * C::STAGE_BYTES;
    const double* a_s = reinterpret_cast<const double*>(st);
    const double* b_s = reinterpret_cast<const double*>(st + C::A_BYTES);
#pragma unroll 4
    for (int kk = 0; kk < WS_BK; kk += 2) {
      double a[8][2];
      if (KMAJ) {
        const double* panel = a_s + (kk >> 4) * (WS_BM * 16);
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
            const double2 v = *reinterpret_cast<const double2*>(a_s + (kk + kq) * WS_BM + 2 * ty + 2 * TY * i);
            a[2 * i][kq] = v.x;
            a[2 * i + 1][kq] = v.y;
          }
      }
#pragma unroll
      for (int kq = 0; kq < 2; ++kq) {
        double b[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 v = *reinterpret_cast<const double2*>(b_s + (kk + kq) * WS_BN + 2 * tx + 2 * TX * i);
          b[2 * i] = v.x;
          b[2 * i + 1] = v.y;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = fma(a[r][kq], b[c], acc[r][c]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // epilogue: partial (or final, lam-folded) tile -> out
  double* out = p.out + int64_t(blockIdx.z) * p.out_split_stride;
  const bool fold = p.lam != nullptr;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int n = n0 + 2 * ty + (r & 1) + 2 * TY * (r >> 1);
    if (n >= p.Ik) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = j0 + 2 * tx + 2 * TX * i;
      double v0 = acc[r][2 * i], v1 = acc[r][2 * i + 1];
      if (fold) {
        if (j < p.R) v0 *= p.lam[j];
        if (j + 1 < p.R) v1 *= p.lam[j + 1];
      }
      double* dst = out + int64_t(n) * p.ldo + j;
      if (j + 1 < p.R && ((p.ldo & 1) == 0)) {
        *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
      } else {
        if (j < p.R) dst[0] = v0;
        if (j + 1 < p.R) dst[1] = v1;
      }
    }
  }
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

template <bool KMAJ, int NO>
static void ws_kernel(const void** fn, size_t* smem, int* stages) {
  constexpr int S = (3 * WsCfg<KMAJ, NO, 3>::STAGE_BYTES + 256 <= 227 * 1024) ? 3 : 2;
  *fn = reinterpret_cast<const void*>(&mttkrp_f64_ws_sm100<KMAJ, NO, S>);
  *smem = WsCfg<KMAJ, NO, S>::SMEM;
  *stages = S;
}

bool ws_eligible(const WsRequest& r) {
  if (r.d < 2 || r.d > 5 || r.n_o > 3) return false;
  if (r.rank_tile != WS_BN || r.block_k != WS_BK) return false;
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
  if (k == 0) {
    for (int m = 0; m < d; ++m) box[m] = 1;
    box[0] = WS_BM;
    box[1] = WS_BK;
    rc = encode(&p.tm_y, r.y, d, gdim, gstr, box, CU_TENSOR_MAP_SWIZZLE_NONE);
  } else {
    for (int m = 0; m < d; ++m) box[m] = 1;
    box[0] = 16;
    box[k] = WS_BM;
    rc = encode(&p.tm_y, r.y, d, gdim, gstr, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (rc) return rc;
  {
    const cuuint64_t fd[2] = {cuuint64_t(r.rank), cuuint64_t(r.dims[f])};
    const cuuint64_t fs[1] = {cuuint64_t(r.ld[f] * 8)};
    const cuuint32_t fb[2] = {WS_BN, WS_BK};
    rc = encode(&p.tm_f, r.factors[f], 2, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
  }
  int oi = 0;
  for (int m = 0; m < d; ++m) {
    if (m == k || m == f) continue;
    const cuuint64_t od[2] = {cuuint64_t(r.rank), cuuint64_t(r.dims[m])};
    const cuuint64_t os[1] = {cuuint64_t(r.ld[m] * 8)};
    const cuuint32_t ob[2] = {WS_BN, 1};
    rc = encode(&p.tm_o[oi], r.factors[m], 2, od, os, ob, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
    p.dim_o[oi] = r.dims[m];
    ++oi;
  }
  p.chunks_per_f = (r.dims[f] + WS_BK - 1) / WS_BK;
  p.n_chunks = p.chunks_per_f;
  for (int i = 0; i < oi; ++i) p.n_chunks *= p.dim_o[i];
  p.chunks_per_split = (p.n_chunks + r.splits - 1) / r.splits;
  p.Ik = int(r.dims[k]);
  p.If = int(r.dims[f]);
  p.R = int(r.rank);
  p.k = k;
  p.out = r.out;
  p.ldo = r.ldo;
  p.out_split_stride = r.out_split_stride;
  p.lam = r.lam;

  const void* fn = nullptr;
  size_t smem = 0;
  int stages = 0;
  const int no = r.n_o;
  if (k == 0) {
    if (no == 0) ws_kernel<false, 0>(&fn, &smem, &stages);
    else if (no == 1) ws_kernel<false, 1>(&fn, &smem, &stages);
    else if (no == 2) ws_kernel<false, 2>(&fn, &smem, &stages);
    else ws_kernel<false, 3>(&fn, &smem, &stages);
  } else {
    if (no == 0) ws_kernel<true, 0>(&fn, &smem, &stages);
    else if (no == 1) ws_kernel<true, 1>(&fn, &smem, &stages);
    else if (no == 2) ws_kernel<true, 2>(&fn, &smem, &stages);
    else ws_kernel<true, 3>(&fn, &smem, &stages);
  }
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return check_launch("ws set smem");
  const int64_t gx = (r.rank + WS_BN - 1) / WS_BN, gy = (r.dims[k] + WS_BM - 1) / WS_BM;
  dim3 grid(unsigned(gx), unsigned(gy), unsigned(r.splits));
  void* args[] = {&p};
  cudaError_t e = cudaLaunchKernel(fn, grid, dim3(WS_THREADS), args, smem, st);
  if (e != cudaSuccess) return fail(CPK_ERR_CUDA, "ws launch: %s", cudaGetErrorString(e));
  return CPK_OK;
}

}  // namespace cpk
