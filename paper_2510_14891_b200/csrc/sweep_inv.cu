// Gamma^-1 for the CP-ALS normal equations X Gamma = G (cpals.py:75-89),
// R > 256: a multi-CTA blocked Gauss-Jordan sweep with FP64 tensor-core
// (DMMA, mma.sync m8n8k4) tile updates, one cooperative launch.
//
// The reference solves with scipy cho_factor / cho_solve.  Here the
// factorization side (which needs only Gamma) produces Gamma^-1 itself, so
// the side that needs G -- on the CP-ALS critical path -- is one GEMM,
// X = G Gamma^-1, run by the MTTKRP kernel (a 2-way MTTKRP: the tensor is G
// read as the R x rows first-mode-fastest array, the factor is Gamma^-1).
// The factorization side runs on a side stream while the mode's MTTKRP
// produces G (cp_als), off the critical path.
//
// Algorithm (symmetric block sweep, 32 x 32 tiles, lower triangle stored):
// for each diagonal block k
//   (A) S = A_kk; Cholesky S = L L^T (LAPACK's positivity test: the first
//       failing pivot of the Schur complements is potrf's failing column,
//       reported 1-based as potrf's info); D = S^-1 = L^-T L^-1; A_kk <- -D
//   (B) for i != k: V_i = A_ik (old), U_i = V_i D
//   (C) for i >= j, i, j != k: A_ij -= U_i V_j^T; then A_ik <- U_i
// after the last block A = -Gamma^-1.  (A) of block k + 1 only needs tile
// (k+1, k+1) after (C) of block k, so the CTA that owns it updates that tile
// first and factors it while the others finish (C): two grid barriers per
// block.  Tiles are staged in shared memory (rows padded to 36 doubles: the
// m8n8k4 fragment loads are conflict-free) and every global access goes
// through L2 (.cg): tiles written by one SM are read by another after a
// barrier, and L1 is not coherent.  R is padded to whole tiles with an
// identity block, which the sweep leaves an identity.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "sweep_inv.cuh"

namespace cg = cooperative_groups;

namespace cpk {
namespace {

constexpr int SB = 32, SLD = 36, ST = 128;

struct SweepArgs {
  const double* gamma;
  int R, Rp, N;
  double eps;
  double* A;  // Rp x Rp row-major; lower tiles hold the sweep, then W = Gamma^-1 (full)
  double* U;  // N tiles of 32 x 32 (tile i at U + 1024 i, ld 32)
  double* V;
  double* D;  // 32 x 32
  int* info;
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// s[r][t] = trans ? g[t][r] : g[r][t] for a 32 x 32 tile (reads coalesced along g's rows)
__device__ __forceinline__ void load_tile(double* s, const double* g, int64_t ld, bool trans) {
#pragma unroll
  for (int e = threadIdx.x; e < SB * SB; e += ST) {
    const int hi = e >> 5, lo = e & 31;
    const double v = __ldcg(g + hi * ld + lo);
    if (trans)
      s[lo * SLD + hi] = v;
    else
      s[hi * SLD + lo] = v;
  }
}

// Warp w owns the 16 x 16 quadrant (w >> 1, w & 1); acc[fr][fc] is the
// m8n8 fragment (fr, fc) of it: element e at row r0 + 8 fr + g, column
// c0 + 8 fc + 2 t + e (g = lane / 4, t = lane % 4).
using Acc = double[2][2][2];

__device__ __forceinline__ void zero(Acc& acc) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// acc += As Bs^T  (As[r][t], Bs[c][t])
__device__ __forceinline__ void mma_tile(const double* As, const double* Bs, Acc& acc) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, t = l & 3;
  const int r0 = (w >> 1) * 16, c0 = (w & 1) * 16;
#pragma unroll
  for (int kk = 0; kk < SB; kk += 4) {
    double a[2], b[2];
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      a[f] = As[(r0 + 8 * f + g) * SLD + kk + t];
      b[f] = Bs[(c0 + 8 * f + g) * SLD + kk + t];
    }
#pragma unroll
    for (int fr = 0; fr < 2; ++fr)
#pragma unroll
      for (int fc = 0; fc < 2; ++fc) dmma(acc[fr][fc], a[fr], b[fc]);
  }
}

template <typename F>
__device__ __forceinline__ void for_acc(F f) {  // f(fr, fc, e, row, col)
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, t = l & 3;
  const int r0 = (w >> 1) * 16, c0 = (w & 1) * 16;
#pragma unroll
  for (int fr = 0; fr < 2; ++fr)
#pragma unroll
    for (int fc = 0; fc < 2; ++fc)
#pragma unroll
      for (int e = 0; e < 2; ++e) f(fr, fc, e, r0 + 8 * fr + g, c0 + 8 * fc + 2 * t + e);
}

struct DiagSmem {
  double lt[SB * 33];  // L, then M = L^-1 (row i, column j at [i * 33 + j])
  double mt[SB * 33];
  double colk[SB];
  double rdg[SB];
  int bad;
};

// (A): Cholesky of the (updated) diagonal tile k, D = S^-1, A_kk <- -D.
// Whole CTA; returns false (info set) when a pivot is not positive.
__device__ bool diag_step(const SweepArgs& a, int k, DiagSmem& sm) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* Akk = a.A + int64_t(k) * SB * a.Rp + int64_t(k) * SB;
  if (warp == 0) {
    // unblocked Cholesky in registers: lane = row, r[c] = S[lane][c]
    double r[SB];
#pragma unroll
    for (int c = 0; c < SB; ++c) r[c] = c <= lane ? __ldcg(Akk + int64_t(lane) * a.Rp + c) : 0.0;
    int bad = 0;
#pragma unroll
    for (int kk = 0; kk < SB; ++kk) {
      if (bad == 0) {  // warp-uniform
        const double dkk = __shfl_sync(~0u, r[kk], kk);
        if (!(dkk > 0.0)) {  // also catches NaN
          bad = kk + 1;
        } else {
          const double rl = rsqrt(dkk);
          r[kk] = lane == kk ? dkk * rl : (lane > kk ? r[kk] * rl : 0.0);
          sm.colk[lane] = r[kk];
          __syncwarp();
#pragma unroll
          for (int c = 1; c < SB; ++c) {
            if (c <= kk) continue;
            r[c] = fma(-r[kk], sm.colk[c], r[c]);
          }
          __syncwarp();
        }
      }
    }
#pragma unroll
    for (int c = 0; c < SB; ++c) sm.lt[lane * 33 + c] = c <= lane ? r[c] : 0.0;
    if (lane == 0) sm.bad = bad;
    __syncwarp();
    sm.rdg[lane] = 1.0 / sm.lt[lane * 34];
  }
  __syncthreads();
  if (sm.bad) {
    if (tid == 0) *a.info = k * SB + sm.bad;  // potrf's 1-based failing column
    return false;
  }
  if (warp == 0) {
    // M = L^-1 by forward substitution on e_lane: lane = column of M
    double x[SB];
#pragma unroll
    for (int i = 0; i < SB; ++i) {
      double v = i == lane ? 1.0 : 0.0;
#pragma unroll
      for (int u = 0; u < i; ++u) v = fma(-sm.lt[i * 33 + u], x[u], v);  // x[u] = 0 for u < lane
      x[i] = i >= lane ? v * sm.rdg[i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < SB; ++i) sm.mt[i * 33 + lane] = x[i];
  }
  __syncthreads();
  // D = M^T M: D[p][q] = sum_{i >= p} M[i][p] M[i][q] (p >= q), mirrored exactly
  const int q = lane;
#pragma unroll
  for (int pp = 0; pp < SB / 4; ++pp) {
    const int p = warp * (SB / 4) + pp;
    if (p >= q) {
      double s = 0.0;
      for (int i = p; i < SB; ++i) s = fma(sm.mt[i * 33 + p], sm.mt[i * 33 + q], s);
      __stcg(a.D + p * SB + q, s);
      __stcg(a.D + q * SB + p, s);
      __stcg(Akk + int64_t(p) * a.Rp + q, -s);
      __stcg(Akk + int64_t(q) * a.Rp + p, -s);
    }
  }
  return true;
}

__device__ __forceinline__ bool failed(const SweepArgs& a) { return __ldcg(a.info) != 0; }

__global__ void __launch_bounds__(ST) sweep_inverse_kernel(SweepArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ __align__(16) double As[SB * SLD];
  __shared__ __align__(16) double Bs[SB * SLD];
  __shared__ DiagSmem dsm;
  __shared__ double red[ST / 32];
  const int tid = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const int Rp = a.Rp, N = a.N, R = a.R;

  // ---- A = Gamma + (eps tr(Gamma) / R) I on the lower tiles, identity padding
  double shift = 0.0;
  if (a.eps != 0.0) {  // cpals.py:84
    double t = 0.0;
    for (int i = tid; i < R; i += ST) t += a.gamma[int64_t(i) * R + i];
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_down_sync(~0u, t, o);
    if ((tid & 31) == 0) red[tid >> 5] = t;
    __syncthreads();
    double tr = 0.0;
#pragma unroll
    for (int w = 0; w < ST / 32; ++w) tr += red[w];
    shift = a.eps * tr / double(R);
  }
  if (b == 0 && tid == 0) __stcg(a.info, 0);
  const int64_t total = int64_t(Rp) * Rp;
  for (int64_t idx = int64_t(b) * ST + tid; idx < total; idx += int64_t(G) * ST) {
    const int i = int(idx / Rp), j = int(idx % Rp);
    if (j / SB > i / SB) continue;  // strictly upper tiles are never read
    double v = (i < R && j < R) ? a.gamma[int64_t(i) * R + j] : 0.0;
    if (i == j) v += i < R ? shift : 1.0;
    __stcg(a.A + idx, v);
  }
  grid.sync();
  if (b == 0) diag_step(a, 0, dsm);
  grid.sync();

  for (int k = 0; k < N; ++k) {
    if (failed(a)) return;
    // ---- (B) V_i = A_ik, U_i = V_i D
    bool have_d = false;
    for (int i = b; i < N; i += G) {
      if (i == k) continue;
      if (!have_d) {
        load_tile(Bs, a.D, SB, false);
        have_d = true;
      }
      if (i > k)
        load_tile(As, a.A + int64_t(i) * SB * Rp + int64_t(k) * SB, Rp, false);
      else
        load_tile(As, a.A + int64_t(k) * SB * Rp + int64_t(i) * SB, Rp, true);
      __syncthreads();
      double* Vi = a.V + int64_t(i) * SB * SB;
      double* Ui = a.U + int64_t(i) * SB * SB;
      for (int e = tid; e < SB * SB; e += ST) __stcg(Vi + e, As[(e >> 5) * SLD + (e & 31)]);
      Acc acc;
      zero(acc);
      mma_tile(As, Bs, acc);
      for_acc([&](int fr, int fc, int e, int r, int c) { __stcg(Ui + r * SB + c, acc[fr][fc][e]); });
      __syncthreads();
    }
    grid.sync();
    // ---- (C) A_ij -= U_i V_j^T (i >= j; i, j != k), then A_ik <- U_i
    const int n = N - 1;
    const int ntile = n * (n + 1) / 2, items = ntile + n;
    const int la = k + 1 < N ? k * (k + 1) / 2 + k : -1;  // tile (k+1, k+1), reduced index (k, k)
    auto do_tile = [&](int e) {
      int ip = int((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((ip + 1) * (ip + 2) / 2 <= e) ++ip;
      while (ip * (ip + 1) / 2 > e) --ip;
      const int jp = e - ip * (ip + 1) / 2;
      const int i = ip + (ip >= k), j = jp + (jp >= k);
      load_tile(As, a.U + int64_t(i) * SB * SB, SB, false);
      load_tile(Bs, a.V + int64_t(j) * SB * SB, SB, false);
      __syncthreads();
      Acc acc;
      zero(acc);
      mma_tile(As, Bs, acc);
      double* Aij = a.A + int64_t(i) * SB * Rp + int64_t(j) * SB;
      for_acc([&](int fr, int fc, int e2, int r, int c) {
        double* p = Aij + int64_t(r) * Rp + c;
        __stcg(p, __ldcg(p) - acc[fr][fc][e2]);
      });
      __syncthreads();
    };
    auto do_writeback = [&](int ip) {
      const int i = ip + (ip >= k);
      const double* Ui = a.U + int64_t(i) * SB * SB;
      if (i > k) {
        double* dst = a.A + int64_t(i) * SB * Rp + int64_t(k) * SB;
        for (int e = tid; e < SB * SB; e += ST) __stcg(dst + int64_t(e >> 5) * Rp + (e & 31), __ldcg(Ui + e));
      } else {
        load_tile(As, Ui, SB, true);  // As = U_i^T
        __syncthreads();
        double* dst = a.A + int64_t(k) * SB * Rp + int64_t(i) * SB;
        for (int e = tid; e < SB * SB; e += ST) __stcg(dst + int64_t(e >> 5) * Rp + (e & 31), As[(e >> 5) * SLD + (e & 31)]);
        __syncthreads();
      }
    };
    if (b == 0 && la >= 0) {  // look-ahead: the next diagonal tile, then its factorization
      do_tile(la);
      diag_step(a, k + 1, dsm);
    }
    const int others = items - (la >= 0 ? 1 : 0);
    for (int s = G > 1 ? b - 1 : 0; s < others; s += (G > 1 ? G - 1 : 1)) {
      if (G > 1 && b == 0) break;  // CTA 0 only runs the look-ahead when others can take the rest
      const int e = (la >= 0 && s >= la) ? s + 1 : s;
      if (e < ntile)
        do_tile(e);
      else
        do_writeback(e - ntile);
    }
    grid.sync();
  }
  if (failed(a)) return;
  // ---- W = -A, both triangles
  const int ntl = N * (N + 1) / 2;
  for (int e = b; e < ntl; e += G) {
    int i = int((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    while (i * (i + 1) / 2 > e) --i;
    const int j = e - i * (i + 1) / 2;
    double* Aij = a.A + int64_t(i) * SB * Rp + int64_t(j) * SB;
    load_tile(As, Aij, Rp, false);
    __syncthreads();
    double* Aji = a.A + int64_t(j) * SB * Rp + int64_t(i) * SB;
    for (int x = tid; x < SB * SB; x += ST) {
      const int r = x >> 5, c = x & 31;
      if (i == j) {
        __stcg(Aij + int64_t(r) * Rp + c, -As[max(r, c) * SLD + min(r, c)]);
      } else {
        __stcg(Aij + int64_t(r) * Rp + c, -As[r * SLD + c]);
        __stcg(Aji + int64_t(r) * Rp + c, -As[c * SLD + r]);
      }
    }
    __syncthreads();
  }
}

}  // namespace

int64_t sweep_padded(int64_t R) { return (R + SB - 1) / SB * SB; }

size_t sweep_factor_bytes(int64_t R) {
  const int64_t Rp = sweep_padded(R), N = Rp / SB;
  const size_t a = size_t(Rp) * Rp, uv = size_t(2) * N * SB * SB, d = SB * SB;
  return ((a + uv + d) * sizeof(double) + 255) / 256 * 256 + 256;  // + info
}

static int max_coop_ctas() {
  static int cached = 0;
  if (cached) return cached;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sweep_inverse_kernel, ST, 0);
  cached = std::max(1, sms * std::max(1, per));
  return cached;
}

int sweep_default_ctas(int64_t R) {
  const int64_t N = sweep_padded(R) / SB;
  const int64_t work = std::max<int64_t>(1, N * (N - 1) / 2 + N);  // items of one (C) phase
  return int(std::min<int64_t>(work + 1, max_coop_ctas()));
}

int sweep_inverse(const double* gamma, int64_t R, double eps, void* work, size_t work_bytes, int* info, int ctas,
                  cudaStream_t st) {
  if (work_bytes < sweep_factor_bytes(R)) return fail(CPK_ERR_RESOURCE, "sweep workspace too small");
  const int64_t Rp = sweep_padded(R), N = Rp / SB;
  SweepArgs a;
  a.gamma = gamma;
  a.R = int(R);
  a.Rp = int(Rp);
  a.N = int(N);
  a.eps = eps;
  a.A = static_cast<double*>(work);
  a.U = a.A + Rp * Rp;
  a.V = a.U + N * SB * SB;
  a.D = a.V + N * SB * SB;
  a.info = info;
  const int g = std::max(1, std::min(ctas > 0 ? ctas : sweep_default_ctas(R), max_coop_ctas()));
  void* args[] = {&a};
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(sweep_inverse_kernel), dim3(g), dim3(ST),
                                                    args, 0, st);
  if (e != cudaSuccess) return fail(CPK_ERR_CUDA, "sweep_inverse launch: %s", cudaGetErrorString(e));
  return check_launch("sweep_inverse");
}

const double* sweep_inverse_matrix(const void* work) { return static_cast<const double*>(work); }

}  // namespace cpk
