// Dimension-tree CP-ALS: the in-group contraction (cpk_dimtree_contract_f64).
//
// The sweep (als_sweep.run_sweeps, tree mode) splits the modes into a left
// group {0..p-1} and a right group {p..d-1}.  Before the first mode of a
// group of two or more modes it runs ONE matrix-free MTTKRP over a view of
// the tensor in which the group is a single merged mode (mttkrp_ws.cu):
//
//   W_G[i_G, r] = sum_{i_rest} Y[i_G, i_rest] * prod_{m not in G} A_m[i_m, r]
//
// and each mode k of the group then reads its MTTKRP out of W_G:
//
//   G_k[i_k, r] = sum_{i_l, l in G, l != k} W_G[i_G, r] * prod_{l != k} A_l[i_l, r]
//
// which is the reference sweep's unit-weight mode-k MTTKRP (cpals.py:121-124,
// mt.run with KruskalTensor(unit, factors)) with the sum over the tensor split
// in two.  A_m outside the group are the factors the reference's update of
// mode k sees (the group's first mode runs before any of them change); inside
// the group, the current ones.  W_G is I_G x R, written once, read once per mode of the group: an
// HBM-bound pass (2 flops per 8 bytes read), here one CTA per (output row,
// 32 rank columns), 8 warps splitting the summed rows, lanes on consecutive
// columns (256-byte coalesced rows of W_G), a fixed-order shared-memory
// reduction (deterministic, run-to-run reproducible).
#include <type_traits>

#include "common.cuh"

namespace cpk {

struct GroupFactors {
  const double* A[CPK_MAX_MODES];
  int64_t lda[CPK_MAX_MODES];
  int64_t ext[CPK_MAX_MODES];
};

constexpr int DT_WARPS = 8;
constexpr int DT_UNROLL = 8;

// Two-mode group (every group of a 3- or 4-way tensor): one of J_lo / J_hi is
// 1, so a summed row is s * stride_s + i_j * stride_j and its Khatri-Rao
// weight is the other mode's factor row s -- no index arithmetic.  V columns
// per lane (V = 2: 16-byte loads, 512-byte warp rows when every row start is
// 16-byte aligned), DT_UNROLL rows in flight per warp.
template <int V>
__global__ void __launch_bounds__(DT_WARPS * 32)
dimtree_contract2_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ B, int64_t ldb,
                         int64_t S, int64_t stride_s, int64_t stride_j, int64_t rows_out, int64_t rank,
                         double* __restrict__ out, int64_t ldo) {
  using vec = typename std::conditional<V == 2, double2, double>::type;
  __shared__ vec red[DT_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t chunks = (rank + 32 * V - 1) / (32 * V);
  for (int64_t b = blockIdx.x; b < rows_out * chunks; b += gridDim.x) {
    const int64_t ij = b / chunks;
    const int64_t c = (b - ij * chunks) * (32 * V) + V * lane;
    const int64_t cc = c < rank ? c : rank - V;  // dead lanes read a live column, never write
    const double* wp = W + ij * stride_j * ldw + cc;
    const double* bp = B + cc;
    const int64_t ws = stride_s * ldw;
    vec acc = vec{};
    int64_t s = w;
    for (; s + (DT_UNROLL - 1) * DT_WARPS < S; s += DT_UNROLL * DT_WARPS) {
      vec wv[DT_UNROLL], bv[DT_UNROLL];
#pragma unroll
      for (int u = 0; u < DT_UNROLL; ++u) {
        const int64_t su = s + u * DT_WARPS;
        wv[u] = __ldg(reinterpret_cast<const vec*>(wp + su * ws));
        bv[u] = __ldg(reinterpret_cast<const vec*>(bp + su * ldb));
      }
#pragma unroll
      for (int u = 0; u < DT_UNROLL; ++u) {
        if constexpr (V == 2) {
          acc.x = fma(wv[u].x, bv[u].x, acc.x);
          acc.y = fma(wv[u].y, bv[u].y, acc.y);
        } else {
          acc = fma(wv[u], bv[u], acc);
        }
      }
    }
    for (; s < S; s += DT_WARPS) {
      const vec wv = __ldg(reinterpret_cast<const vec*>(wp + s * ws));
      const vec bv = __ldg(reinterpret_cast<const vec*>(bp + s * ldb));
      if constexpr (V == 2) {
        acc.x = fma(wv.x, bv.x, acc.x);
        acc.y = fma(wv.y, bv.y, acc.y);
      } else {
        acc = fma(wv, bv, acc);
      }
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0) {
      vec t = red[0][lane];
#pragma unroll
      for (int q = 1; q < DT_WARPS; ++q) {
        if constexpr (V == 2) {
          t.x += red[q][lane].x;
          t.y += red[q][lane].y;
        } else {
          t += red[q][lane];
        }
      }
      if (c < rank) {
        if constexpr (V == 2) {
          out[ij * ldo + c] = t.x;
          out[ij * ldo + c + 1] = t.y;
        } else {
          out[ij * ldo + c] = t;
        }
      }
    }
    __syncthreads();
  }
}

// Any group size: the summed row index s enumerates (i_lo, i_hi), i_lo over
// the modes before j (fastest first), i_hi over the modes after it.
__global__ void __launch_bounds__(DT_WARPS * 32)
dimtree_contract_kernel(const double* __restrict__ W, int64_t ldw, GroupFactors gf, int g, int j, int64_t j_lo,
                        int64_t S, int64_t rows_out, int64_t rank, double* __restrict__ out, int64_t ldo) {
  __shared__ double red[DT_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t chunks = (rank + 31) / 32;
  const int64_t j_ext = gf.ext[j];
  for (int64_t b = blockIdx.x; b < rows_out * chunks; b += gridDim.x) {
    const int64_t ij = b / chunks;
    const int64_t c = (b - ij * chunks) * 32 + lane;
    const int64_t cc = c < rank ? c : rank - 1;
    double acc = 0.0;
    for (int64_t s = w; s < S; s += DT_WARPS) {
      const int64_t i_lo = s % j_lo, i_hi = s / j_lo;
      const int64_t row = i_lo + j_lo * (ij + j_ext * i_hi);
      double kr = 1.0;
      int64_t t = i_lo;
      for (int l = 0; l < j; ++l) {
        const int64_t il = t % gf.ext[l];
        t /= gf.ext[l];
        kr *= __ldg(gf.A[l] + il * gf.lda[l] + cc);
      }
      t = i_hi;
      for (int l = j + 1; l < g; ++l) {
        const int64_t il = t % gf.ext[l];
        t /= gf.ext[l];
        kr *= __ldg(gf.A[l] + il * gf.lda[l] + cc);
      }
      acc = fma(__ldg(W + row * ldw + cc), kr, acc);
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0) {
      double t = red[0][lane];
#pragma unroll
      for (int q = 1; q < DT_WARPS; ++q) t += red[q][lane];
      if (c < rank) out[ij * ldo + c] = t;
    }
    __syncthreads();
  }
}

}  // namespace cpk

using namespace cpk;

extern "C" int cpk_dimtree_contract_f64(const double* W, int64_t ldw, int g, const int64_t* ext, int j,
                                        const double* const* factors, const int64_t* lda, int64_t rank, double* out,
                                        int64_t ldo, void* stream) {
  if (!W || !ext || !factors || !lda || !out) return fail(CPK_ERR_PARAM, "NULL pointer");
  if (g < 2 || g > CPK_MAX_MODES || j < 0 || j >= g) return fail(CPK_ERR_PARAM, "bad group (g=%d, j=%d)", g, j);
  if (rank < 1 || ldw < rank || ldo < rank) return fail(CPK_ERR_SHAPE, "bad rank / leading dimensions");
  GroupFactors gf{};
  int64_t j_lo = 1, j_hi = 1;
  for (int l = 0; l < g; ++l) {
    if (ext[l] < 1) return fail(CPK_ERR_SHAPE, "group extent %d is %lld", l, (long long)ext[l]);
    gf.ext[l] = ext[l];
    if (l == j) continue;
    if (!factors[l]) return fail(CPK_ERR_PARAM, "factor %d of the group is NULL", l);
    if (lda[l] < rank) return fail(CPK_ERR_SHAPE, "factor %d: lda %lld < rank", l, (long long)lda[l]);
    gf.A[l] = factors[l];
    gf.lda[l] = lda[l];
    (l < j ? j_lo : j_hi) *= ext[l];
  }
  const int64_t S = j_lo * j_hi, rows_out = ext[j];
  const int64_t blocks = rows_out * ((rank + 31) / 32);
  const unsigned grid = unsigned(blocks < 148 * 64 ? blocks : 148 * 64);
  cudaStream_t st = as_stream(stream);
  if (g == 2) {
    const int o = 1 - j;  // the other mode of the pair
    const int64_t stride_s = (j == 0) ? ext[0] : 1, stride_j = (j == 0) ? 1 : ext[0];
    const bool v2 = rank % 2 == 0 && ldw % 2 == 0 && lda[o] % 2 == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(factors[o]) & 15) == 0;
    if (v2) {
      const int64_t blocks2 = rows_out * ((rank + 63) / 64);
      dimtree_contract2_kernel<2><<<unsigned(blocks2 < 148 * 64 ? blocks2 : 148 * 64), DT_WARPS * 32, 0, st>>>(
          W, ldw, factors[o], lda[o], S, stride_s, stride_j, rows_out, rank, out, ldo);
    } else {
      dimtree_contract2_kernel<1><<<grid, DT_WARPS * 32, 0, st>>>(W, ldw, factors[o], lda[o], S, stride_s,
                                                                  stride_j, rows_out, rank, out, ldo);
    }
  } else {
    dimtree_contract_kernel<<<grid, DT_WARPS * 32, 0, st>>>(W, ldw, gf, g, j, j_lo, S, rows_out, rank, out, ldo);
  }
  return check_launch("dimtree contract");
}
