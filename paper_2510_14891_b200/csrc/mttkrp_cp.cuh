// The cp.async MTTKRP kernel template (DFMA or DMMA consumers) and its
// launch descriptors, shared by mttkrp.cu (host logic) and the two
// instantiation units mttkrp_cp_dfma.cu / mttkrp_cp_dmma.cu (split so the
// build compiles them in parallel).  Design notes: mttkrp.cu.
#pragma once

#include "common.cuh"

namespace cpk {

constexpr int KPAD = 2;  // K-major As row pad (doubles)

struct MttkrpParams {
  const double* y;
  const double* fac_f;
  const double* fac_o[CPK_MAX_MODES];
  int64_t ld_f;
  int64_t ld_o[CPK_MAX_MODES];
  int64_t dim_o[CPK_MAX_MODES];
  int64_t stride_o[CPK_MAX_MODES];
  int64_t Ik, stride_k;
  int64_t If, stride_f;
  int64_t chunks_per_f;      // ceil(If / BK)
  int64_t n_chunks;          // chunks_per_f * prod(dim_o)
  int64_t chunks_per_split;
  int64_t R;
  double* out;
  int64_t ldo;
  int64_t out_split_stride;
  const double* lam;         // folded in the epilogue when direct, or by the chain's last split
  int32_t y0, z0;            // first row block / split of this launch
  int* sem;                  // split-K chain counters (common.cuh), or nullptr
  int32_t n_splits;
};

// Loader state: the chunk being staged next, as an odometer over
// (q_f, o digits) -- the in-slice walk of accum_tile (_kernels.py:135-147),
// advanced one chunk per pipeline stage without any div/mod.
template <int NO>
struct ChunkCursor {
  int64_t qf;
  int64_t od[NO > 0 ? NO : 1];
  int64_t base;  // sum od[i] * stride_o[i]

  __device__ void init(const MttkrpParams& p, int64_t q) {
    qf = q % p.chunks_per_f;
    int64_t rest = q / p.chunks_per_f;
    base = 0;
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      od[i] = rest % p.dim_o[i];
      rest /= p.dim_o[i];
      base += od[i] * p.stride_o[i];
    }
  }
  __device__ void advance(const MttkrpParams& p) {
    if (++qf < p.chunks_per_f) return;
    qf = 0;
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      base += p.stride_o[i];
      if (++od[i] < p.dim_o[i]) return;
      base -= od[i] * p.stride_o[i];
      od[i] = 0;
    }
  }
};

template <int BM, int BN, int BK, bool KMAJ, int VEC, int STAGES, int NO>
struct TileCfg {
  static constexpr int TY = BM / 8, TX = BN / 8, NT = TY * TX;
  static constexpr int WX = TX < 8 ? TX : 8, WY = 32 / WX;
  static constexpr int APITCH = KMAJ ? (BK + KPAD) : BM;
  static constexpr int A_ELEMS = KMAJ ? BM * (BK + KPAD) : BK * BM;
  static constexpr int B_ELEMS = BK * BN;
  static constexpr int P_ELEMS = NO * NT * VEC;
  static constexpr int CPA = KMAJ ? BK / VEC : BM / VEC;  // A chunks per staged row
  static constexpr int NA = BM * BK / VEC / NT;           // A chunks per thread
  static constexpr int CPB = BN / VEC;
  static constexpr int NB = BK * BN / VEC / NT;
  static constexpr size_t STAGE_BYTES = sizeof(double) * size_t(A_ELEMS + B_ELEMS + P_ELEMS);
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(NT % 32 == 0, "whole warps");
  static_assert(NT % CPB == 0, "uniform B-chunk ownership (scale pass)");
  static_assert((BM * BK / VEC) % NT == 0 && (BK * BN / VEC) % NT == 0, "even split");
  static_assert(BK % 2 == 0, "k pairs");
};

template <int VEC>
__device__ __forceinline__ int64_t clamp_vec(int64_t left) {
  return left < VEC ? left : VEC;
}

template <int VEC>
__device__ __forceinline__ void cp_chunk(double* dst, const double* src, int valid_elems) {
  int v = valid_elems < 0 ? 0 : (valid_elems > VEC ? VEC : valid_elems);
  if (VEC == 2)
    cp_async16(dst, src, v * 8);
  else
    cp_async8(dst, src, v * 8);
}

// DMMA consumer for the cp.async tiles (256 threads = 8 warps of 32 x 64 warp
// tiles, as the TMA kernel's, mttkrp_ws.cu): m8n8k4 fragments read from the
// staged layouts, each 8-deep k block as two k-steps (even k, odd k).  TAIL:
// the warp's columns straddle R; only its first nf_act 8-column fragments
// issue DMMAs.
template <bool KMAJ, bool TAIL, int BM, int BN, int BK, int APITCH>
__device__ __forceinline__ void cp_dmma_stage(double (&acc)[4][8][2], const double* a_s, const double* b_s, int wm0,
                                              int wn0, int lane, int nf_act) {
  const int lr = lane >> 2, lk = lane & 3;
#pragma unroll 2
  for (int kk = 0; kk < BK; kk += 8) {
    double a[4][2], b[8][2];
#pragma unroll
    for (int mf = 0; mf < 4; ++mf) {
      const int m = wm0 + mf * 8 + lr;
      if constexpr (KMAJ) {
        const double2 v = *reinterpret_cast<const double2*>(a_s + m * APITCH + kk + 2 * lk);
        a[mf][0] = v.x;
        a[mf][1] = v.y;
      } else {
        a[mf][0] = a_s[(kk + 2 * lk) * BM + m];
        a[mf][1] = a_s[(kk + 2 * lk + 1) * BM + m];
      }
    }
    const double* brow = b_s + (kk + 2 * lk) * BN + wn0 + lr;
#pragma unroll
    for (int nf = 0; nf < 8; ++nf) {
      if (TAIL && nf >= nf_act) break;
      b[nf][0] = brow[nf * 8];
      b[nf][1] = brow[BN + nf * 8];
    }
#pragma unroll
    for (int ph = 0; ph < 2; ++ph)
#pragma unroll
      for (int mf = 0; mf < 4; ++mf)
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) {
          if (TAIL && nf >= nf_act) break;
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[mf][nf][0]), "+d"(acc[mf][nf][1])
                       : "d"(a[mf][ph]), "d"(b[nf][ph]));
        }
  }
}

template <int BM, int BN, int BK, bool KMAJ, int VEC, int STAGES, int NO, bool DMMA = false>
__global__ void __launch_bounds__((BM / 8) * (BN / 8), 1)
    mttkrp_f64_sm100(const __grid_constant__ MttkrpParams p) {
  using C = TileCfg<BM, BN, BK, KMAJ, VEC, STAGES, NO>;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = As + STAGES * C::A_ELEMS;
  double* Ps = Bs + STAGES * C::B_ELEMS;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int WARPS_X = C::TX / C::WX;
  const int ty = (warp / WARPS_X) * C::WY + lane / C::WX;
  const int tx = (warp % WARPS_X) * C::WX + lane % C::WX;

  const int64_t j0 = int64_t(blockIdx.x) * BN;
  const int64_t n0 = int64_t(blockIdx.y + p.y0) * BM;
  const int64_t q0 = int64_t(blockIdx.z + p.z0) * p.chunks_per_split;
  const int64_t q1 = min(p.n_chunks, q0 + p.chunks_per_split);
  const int nst = int(q1 - q0);

  ChunkCursor<NO> cur;
  cur.init(p, q0);

  // --- stage loader: tensor tile + A_f rows + private P_o slots ----------
  auto load_stage = [&](int buf) {
    const int64_t if0 = cur.qf * BK;
    double* a_s = As + buf * C::A_ELEMS;
    double* b_s = Bs + buf * C::B_ELEMS;
#pragma unroll
    for (int c = 0; c < C::NA; ++c) {
      const int idx = tid + c * C::NT;
      if (!KMAJ) {
        const int k = idx / C::CPA, m = (idx % C::CPA) * VEC;
        const bool kv = if0 + k < p.If;
        const int64_t off = cur.base + (if0 + k) * p.stride_f + n0 + m;
        const int valid = kv ? int(clamp_vec<VEC>(p.Ik - (n0 + m))) : 0;
        cp_chunk<VEC>(a_s + k * BM + m, valid > 0 ? p.y + off : p.y, valid);
      } else {
        const int m = idx / C::CPA, k = (idx % C::CPA) * VEC;
        const bool mv = n0 + m < p.Ik;
        const int64_t off = cur.base + (n0 + m) * p.stride_k + if0 + k;
        const int valid = mv ? int(clamp_vec<VEC>(p.If - (if0 + k))) : 0;
        cp_chunk<VEC>(a_s + m * C::APITCH + k, valid > 0 ? p.y + off : p.y, valid);
      }
    }
    const int jc = (tid % C::CPB) * VEC;
    const int jvalid = int(clamp_vec<VEC>(p.R - (j0 + jc)));
#pragma unroll
    for (int c = 0; c < C::NB; ++c) {
      const int k = (tid + c * C::NT) / C::CPB;
      const bool kv = if0 + k < p.If;
      const int valid = kv ? jvalid : 0;
      const double* src = p.fac_f + (if0 + k) * p.ld_f + j0 + jc;
      cp_chunk<VEC>(b_s + k * BN + jc, valid > 0 ? src : p.fac_f, valid);
    }
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      const double* src = p.fac_o[i] + cur.od[i] * p.ld_o[i] + j0 + jc;
      cp_chunk<VEC>(Ps + (buf * NO + i) * C::NT * VEC + tid * VEC, jvalid > 0 ? src : p.fac_o[i],
                    jvalid);
    }
  };

  double acc[8][8];  // DFMA: 8 x 8 per thread; DMMA: [4 m-frags][8 n-frags][2]
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
  double(&dacc)[4][8][2] = *reinterpret_cast<double(*)[4][8][2]>(&acc);
  static_assert(!DMMA || C::NT == 256, "DMMA tiles run 8 warps");
  constexpr int DWARPS_N = BN / 64 > 0 ? BN / 64 : 1;
  const int dwm0 = (warp / DWARPS_N) * 32, dwn0 = (warp % DWARPS_N) * 64;
  const int dnf_act = int((p.R - j0 - dwn0 + 7) >> 3);

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nst) {
      load_stage(s);
      cur.advance(p);
    }
    cp_async_commit();
  }

  for (int it = 0; it < nst; ++it) {
    const int buf = it % STAGES;
    cp_async_wait<STAGES - 2>();
    if (NO > 0) {
      // Khatri-Rao row formation: B[k][j] = A_f[i_f0+k][j] * prod_o A_o[o][j],
      // on this thread's own chunks (same column pair for all of them).
      const double* ps = Ps + buf * NO * C::NT * VEC + tid * VEC;
      double pp[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) pp[v] = ps[v];
#pragma unroll
      for (int i = 1; i < NO; ++i)
#pragma unroll
        for (int v = 0; v < VEC; ++v) pp[v] *= ps[i * C::NT * VEC + v];
      double* b_s = Bs + buf * C::B_ELEMS;
      const int jc = (tid % C::CPB) * VEC;
#pragma unroll
      for (int c = 0; c < C::NB; ++c) {
        const int k = (tid + c * C::NT) / C::CPB;
        double* bp = b_s + k * BN + jc;
        if (VEC == 2) {
          double2 v = *reinterpret_cast<double2*>(bp);
          v.x *= pp[0];
          v.y *= pp[VEC - 1];
          *reinterpret_cast<double2*>(bp) = v;
        } else {
          bp[0] *= pp[0];
        }
      }
    }
    __syncthreads();
    if (it + STAGES - 1 < nst) {
      load_stage((it + STAGES - 1) % STAGES);
      cur.advance(p);
    }
    cp_async_commit();

    const double* a_s = As + buf * C::A_ELEMS;
    const double* b_s = Bs + buf * C::B_ELEMS;
    if constexpr (DMMA) {
      if (dnf_act >= 8)
        cp_dmma_stage<KMAJ, false, BM, BN, BK, C::APITCH>(dacc, a_s, b_s, dwm0, dwn0, lane, 8);
      else
        cp_dmma_stage<KMAJ, true, BM, BN, BK, C::APITCH>(dacc, a_s, b_s, dwm0, dwn0, lane, dnf_act);
    } else {
#pragma unroll
    for (int kk = 0; kk < BK; kk += 2) {
      double a[8][2];
      if (KMAJ) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int m = 2 * ty + (r & 1) + 2 * C::TY * (r >> 1);
          const double2 v = *reinterpret_cast<const double2*>(a_s + m * C::APITCH + kk);
          a[r][0] = v.x;
          a[r][1] = v.y;
        }
      } else {
#pragma unroll
        for (int kq = 0; kq < 2; ++kq)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double2 v =
                *reinterpret_cast<const double2*>(a_s + (kk + kq) * BM + 2 * ty + 2 * C::TY * i);
            a[2 * i][kq] = v.x;
            a[2 * i + 1][kq] = v.y;
          }
      }
#pragma unroll
      for (int kq = 0; kq < 2; ++kq) {
        double b[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 v =
              *reinterpret_cast<const double2*>(b_s + (kk + kq) * BN + 2 * tx + 2 * C::TX * i);
          b[2 * i] = v.x;
          b[2 * i + 1] = v.y;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = fma(a[r][kq], b[c], acc[r][c]);
      }
    }
    }  // DFMA
  }
  cp_async_wait<0>();

  // --- epilogue: partial (or final, lam-folded) tile -> out --------------
  const int zs = blockIdx.z + p.z0, tile = blockIdx.x + gridDim.x * (blockIdx.y + p.y0);
  double* out = p.out + (p.sem ? 0 : int64_t(zs) * p.out_split_stride);
  const OutMode om = chain_mode(p.sem != nullptr, zs, p.n_splits, p.lam != nullptr);
  if (p.sem) {
    if (threadIdx.x == 0) chain_wait(p.sem + tile, zs);
    __syncthreads();
  }
  const bool vec = (p.ldo & 1) == 0;
  if constexpr (DMMA) {
    const int lr = lane >> 2, lk = lane & 3;
#pragma unroll
    for (int mf = 0; mf < 4; ++mf) {
      const int64_t n = n0 + dwm0 + mf * 8 + lr;
      if (n >= p.Ik) continue;
#pragma unroll
      for (int nf = 0; nf < 8; ++nf) {
        const int64_t j = j0 + dwn0 + nf * 8 + 2 * lk;
        store_pair(out + n * p.ldo + j, j, p.R, vec, dacc[mf][nf][0], dacc[mf][nf][1], p.lam, om);
      }
    }
  } else {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t n = n0 + 2 * ty + (r & 1) + 2 * C::TY * (r >> 1);
    if (n >= p.Ik) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t j = j0 + 2 * tx + 2 * C::TX * i;
      store_pair(out + n * p.ldo + j, j, p.R, vec, acc[r][2 * i], acc[r][2 * i + 1], p.lam, om);
    }
  }
  }  // DFMA epilogue
  if (p.sem) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();  // cumulative: the barrier ordered the CTA's stores before it
      st_release_gpu(p.sem + tile, zs + 1);
    }
  }
}

// Tile configurations: (BM, BN, threads) = (128,128,256) | (128,64,128) | (64,32,32);
// BK = 16 (any shape) or 32 (16-byte path only); as many stages (<= 3) as fit
// in 227 KiB of shared memory.
template <int BM, int BN, int BK, bool KMAJ, int VEC, int NO>
struct Pick {
  static constexpr size_t stage_bytes = TileCfg<BM, BN, BK, KMAJ, VEC, 1, NO>::STAGE_BYTES;
  static constexpr int stages = (3 * stage_bytes <= 227 * 1024) ? 3 : 2;
  using Cfg = TileCfg<BM, BN, BK, KMAJ, VEC, stages, NO>;
};

struct KernelInfo {
  const void* fn;
  size_t smem;
  int threads;
  int stages;
};

template <int BM, int BN, int BK, bool KMAJ, int VEC, int NO, bool DMMA>
inline KernelInfo info() {
  using P = Pick<BM, BN, BK, KMAJ, VEC, NO>;
  return {reinterpret_cast<const void*>(&mttkrp_f64_sm100<BM, BN, BK, KMAJ, VEC, P::stages, NO, DMMA>), P::Cfg::SMEM,
          P::Cfg::NT, P::stages};
}

template <int BM, int BN, int BK, bool KMAJ, int VEC, bool DMMA>
inline KernelInfo pick_no(int no) {
  switch (no) {
    case 0: return info<BM, BN, BK, KMAJ, VEC, 0, DMMA>();
    case 1: return info<BM, BN, BK, KMAJ, VEC, 1, DMMA>();
    case 2: return info<BM, BN, BK, KMAJ, VEC, 2, DMMA>();
    case 3: return info<BM, BN, BK, KMAJ, VEC, 3, DMMA>();
    default: return {nullptr, 0, 0, 0};
  }
}

template <int BM, int BN, bool DMMA = false>
inline KernelInfo pick_layout(int bk, bool kmaj, int vec, int no) {
  if (bk == 32) {
    if (vec != 2) return {nullptr, 0, 0, 0};
    return kmaj ? pick_no<BM, BN, 32, true, 2, DMMA>(no) : pick_no<BM, BN, 32, false, 2, DMMA>(no);
  }
  if (kmaj) return vec == 2 ? pick_no<BM, BN, 16, true, 2, DMMA>(no) : pick_no<BM, BN, 16, true, 1, DMMA>(no);
  return vec == 2 ? pick_no<BM, BN, 16, false, 2, DMMA>(no) : pick_no<BM, BN, 16, false, 1, DMMA>(no);
}

// one instantiation unit each (mttkrp_cp_dfma.cu, mttkrp_cp_dmma.cu)
KernelInfo pick_kernel_dfma(int rank_tile, int bk, bool kmaj, int vec, int no);
KernelInfo pick_kernel_dmma(int rank_tile, int bk, bool kmaj, int vec, int no);

}  // namespace cpk
