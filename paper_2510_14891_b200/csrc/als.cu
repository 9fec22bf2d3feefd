// On-device CP-ALS step kernels: Gram, Hadamard of Grams, the normal-equation
// solve with the reference's regularization ladder, column normalization and
// the factored fit terms.  Reference: pkg/src/cpkern/cpals.py:75-152 and
// kruskal.py:74-114.  Every reduction runs in a fixed order, so a sweep is
// bit-reproducible run to run (README.md "same seed, same trajectory").
#include "common.cuh"
#include "sweep_inv.cuh"

#include <cusolverDn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace cpk {

// ---------------------------------------------------------------- Gram
// A^T A for A (rows x R, row-major, lda): 64x64 output tiles, 256 threads with
// 4x4 register micro-tiles, rows staged GK at a time with cp.async into two
// buffers (the next slab loads behind the current slab's FMAs; a plain
// load-then-sync loop waited out the L2 latency every 16 rows: c3's 128 x 256
// Gram took ~30 us).  Only tiles on or above the diagonal are launched; every
// (a <= b) entry is written to both (a, b) and (b, a) -- exact symmetry as
// kruskal.gram (kruskal.py:110-114).  Each entry sums its rows in order.
constexpr int GT = 64, GK = 32, GLD = GT + 1;
constexpr size_t GRAM_SMEM = size_t(2) * 2 * GK * GLD * sizeof(double);

__global__ void __launch_bounds__(256) gram_kernel(const double* __restrict__ A, int64_t rows, int64_t R,
                                                   int64_t lda, double* __restrict__ G) {
  // map the linear block id onto the upper-triangular tile (ti <= tj)
  const int64_t nt = (R + GT - 1) / GT;
  int64_t b = blockIdx.x, ti = 0;
  while (b >= nt - ti) {
    b -= nt - ti;
    ++ti;
  }
  const int64_t tj = ti + b;
  extern __shared__ double gsm[];  // [buf][panel a/b][GK][GLD]
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  const int64_t a0 = ti * GT, b0 = tj * GT;
  auto issue = [&](int64_t r0, int buf) {
    double* sa = gsm + buf * 2 * GK * GLD;
    double* sb = sa + GK * GLD;
    for (int e = threadIdx.x; e < GK * GT; e += 256) {
      const int kr = e / GT, c = e % GT;
      const int64_t r = r0 + kr;
      const bool oka = r < rows && a0 + c < R, okb = r < rows && b0 + c < R;
      cp_async8(sa + kr * GLD + c, oka ? A + r * lda + a0 + c : A, oka ? 8 : 0);
      cp_async8(sb + kr * GLD + c, okb ? A + r * lda + b0 + c : A, okb ? 8 : 0);
    }
    cp_async_commit();
  };
  issue(0, 0);
  int buf = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += GK, buf ^= 1) {
    if (r0 + GK < rows) {
      issue(r0 + GK, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* sa = gsm + buf * 2 * GK * GLD;
    const double* sb = sa + GK * GLD;
#pragma unroll 8
    for (int kr = 0; kr < GK; ++kr) {
      double x[4], y[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[i] = sa[kr * GLD + ty + 16 * i];
        y[i] = sb[kr * GLD + tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(x[i], y[j], acc[i][j]);
    }
    __syncthreads();  // this buffer is refilled two slabs on
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t a = a0 + ty + 16 * i, c = b0 + tx + 16 * j;
      if (a < R && c < R && a <= c) {
        G[a * R + c] = acc[i][j];
        G[c * R + a] = acc[i][j];
      }
    }
}

// ---------------------------------------------------------------- Hadamard
struct GramList {
  const double* g[CPK_MAX_MODES];
  int n;
  int skip;
};

__global__ void hadamard_kernel(const __grid_constant__ GramList gl, int64_t RR, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < RR; i += int64_t(gridDim.x) * blockDim.x) {
    double v = 1.0;
    for (int m = 0; m < gl.n; ++m)
      if (m != gl.skip) v *= gl.g[m][i];
    out[i] = v;
  }
}

// ---------------------------------------------------------------- column norms
// normsq[j] = sum_i A[i, j]^2: 32 columns x 8 row groups per block, row
// groups combined in a fixed order.
__global__ void __launch_bounds__(256) colnorms_kernel(const double* __restrict__ A, int64_t rows, int64_t R,
                                                       int64_t lda, double* __restrict__ normsq) {
  __shared__ double part[8][33];
  const int cx = threadIdx.x % 32, gy = threadIdx.x / 32;
  const int64_t j = blockIdx.x * 32 + cx;
  double s = 0.0;
  if (j < R)
    for (int64_t i = gy; i < rows; i += 8) {
      const double v = A[i * lda + j];
      s = fma(v, v, s);
    }
  part[gy][cx] = s;
  __syncthreads();
  if (gy == 0 && j < R) {
    double t = part[0][cx];
    for (int g = 1; g < 8; ++g) t += part[g][cx];
    normsq[j] = t;
  }
}

__global__ void scale_columns_kernel(double* __restrict__ A, int64_t rows, int64_t R, int64_t lda,
                                     const double* __restrict__ normsq, double* __restrict__ lam) {
  const int64_t total = rows * R;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx / R, j = idx - i * R;
    const double nrm = sqrt(normsq[j]);
    if (nrm > 0.0) A[i * lda + j] /= nrm;
    if (i == 0 && lam) lam[j] = nrm > 0.0 ? nrm : 0.0;
  }
}

// ---------------------------------------------------------------- reductions
template <int NT>
__device__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
#pragma unroll
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// out[0] = lam^T H lam  (cpals.py:146 forms (lam @ H) @ lam), out[1] = sum((G*lam)*A)
__global__ void __launch_bounds__(1024) fit_terms_kernel(const double* __restrict__ H,
                                                         const double* __restrict__ lam,
                                                         const double* __restrict__ G,
                                                         const double* __restrict__ A, int64_t rows,
                                                         int64_t R, double* __restrict__ out) {
  __shared__ double sh[1024];
  // lam^T (H lam): warp a-rows, lanes stride the (coalesced) columns, so the
  // loads are independent of the accumulation chain (H is symmetric)
  // (one CTA, so every loop keeps several loads in flight: independent
  // partial sums, combined in a fixed order)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s0 = 0.0;
  for (int64_t a = warp; a < R; a += 32) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t b = lane;
    for (; b + 96 < R; b += 128)
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = fma(H[a * R + b + 32 * u], lam[b + 32 * u], v[u]);
    for (; b < R; b += 32) v[0] = fma(H[a * R + b], lam[b], v[0]);
    s0 = fma(lam[a], (v[0] + v[1]) + (v[2] + v[3]), s0);
  }
  double s1 = 0.0;
  if (G && A) {
    double p[4] = {0.0, 0.0, 0.0, 0.0};
    const int64_t n = rows * R;
    int64_t idx = threadIdx.x;
    for (; idx + 3 * 1024 < n; idx += 4 * 1024)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = idx + 1024 * u;
        p[u] = fma(G[i] * lam[i % R], A[i], p[u]);
      }
    for (; idx < n; idx += 1024) p[0] = fma(G[idx] * lam[idx % R], A[idx], p[0]);
    s1 = (p[0] + p[1]) + (p[2] + p[3]);
  }
  const double t0 = block_sum<1024>(s0, sh);
  const double t1 = block_sum<1024>(s1, sh);
  if (threadIdx.x == 0) {
    out[0] = t0;
    out[1] = t1;
  }
}

__global__ void __launch_bounds__(256) sumsq_partial_kernel(const double* __restrict__ x, int64_t n,
                                                            double* __restrict__ part) {
  __shared__ double sh[256];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += 256) s = fma(x[i], x[i], s);
  const double t = block_sum<256>(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) sumsq_final_kernel(const double* __restrict__ part, int n,
                                                           double* __restrict__ out) {
  __shared__ double sh[1024];
  const double t = block_sum<1024>(threadIdx.x < n ? part[threadIdx.x] : 0.0, sh);
  if (threadIdx.x == 0) out[0] = t;
}

// ---------------------------------------------------------------- solve helpers
__global__ void copy_regularize_kernel(const double* __restrict__ gamma, int64_t R, double eps,
                                       double* __restrict__ out) {
  // out = gamma + (eps * trace(gamma) / R) I   (cpals.py:84); eps = 0: plain copy
  __shared__ double tr_sh[256];
  double t = 0.0;
  if (eps != 0.0)
    for (int64_t i = threadIdx.x; i < R; i += 256) t += gamma[i * R + i];
  const double tr = block_sum<256>(t, tr_sh);
  const double shift = eps * tr / double(R);
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < R * R;
       idx += int64_t(gridDim.x) * blockDim.x) {
    double v = gamma[idx];
    if (eps != 0.0 && idx / R == idx % R) v += shift;
    out[idx] = v;
  }
}

// ---------------------------------------------------------------- small-R Cholesky
// For R <= CHOL_SMALL_MAX the normal-equation solve runs as two of our own
// launches instead of cuSOLVER potrf + potrs (~20 latency-bound launches).  Same algorithm as cho_factor / cho_solve
// (cpals.py:79-85): Gamma = L L^T, then X L L^T = G row by row; only the
// blocking and the summation order differ.
//
// chol_small_kernel: one CTA, right-looking over 32-column blocks.  Warp 0
// factors the diagonal block in registers (lane = row, shuffles carry the
// pivot column), the CTA solves the panel below it against that block (one
// thread per row), and 64-thread groups apply the symmetric rank-32 update
// to the trailing lower triangle in 32 x 32 tiles (4 x 4 per thread), with a
// look-ahead: the next block column's tiles first, then warp 0 factors the
// next diagonal block while the other groups finish the trailing update (the
// serial factorization was a third of the kernel, profiles/r02_chol_small.md).  The
// matrix lives in the caller's workspace (L2-resident); the panel is staged
// in shared memory for the update.  On exit the lower triangle holds L and
// the upper triangle of each 32 x 32 diagonal block the transposed strictly
// lower part of that block's inverse (for chol_rows); the rest of the upper
// triangle is not written.  info = 0, or the 1-based column whose pivot was
// not positive (LAPACK's potrf convention).
constexpr int CB = 32, CHOL_THREADS = 512;
// The kernels handle R <= CHOL_KERNEL_CAP; by default they replace cuSOLVER
// up to CHOL_SMALL_MAX, where they stop winning (single CTA: the trailing
// updates grow as R^3).  tools/solve_bench.py, B200: R = 32 19 vs 40 us,
// 64 34 vs 81, 128 81 vs 172, 256 258 vs 363, 384 597 vs 558 (rows = 128).
constexpr int CHOL_KERNEL_CAP = 512, CHOL_SMALL_MAX = 256;

static size_t chol_smem(int64_t R) {
  const int64_t np = std::max<int64_t>(0, R - CB);
  return size_t(CB * 33 + ((np + CB - 1) / CB) * CB * 33) * sizeof(double);
}

__global__ void __launch_bounds__(CHOL_THREADS, 1) chol_small_kernel(const double* __restrict__ gamma, int R,
                                                                     double eps, double* __restrict__ L,
                                                                     int* __restrict__ info) {
  extern __shared__ double csm[];
  double* dg = csm;             // [32][33] the factored diagonal block
  double* pan = csm + CB * 33;  // [round32(R - 32)][33] the solved panel
  __shared__ double red[CHOL_THREADS / 32], rdg[CB];
  __shared__ __align__(16) double colk[CB];
  __shared__ int fail;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double shift = 0.0;
  if (eps != 0.0) {  // Gamma + (eps tr(Gamma) / R) I  (cpals.py:84)
    double t = 0.0;
    for (int i = tid; i < R; i += CHOL_THREADS) t += gamma[int64_t(i) * R + i];
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_down_sync(~0u, t, o);
    if (lane == 0) red[warp] = t;
    __syncthreads();
    double tr = 0.0;
    for (int w = 0; w < CHOL_THREADS / 32; ++w) tr += red[w];
    shift = eps * tr / double(R);
  }
  // no copy of Gamma: step 0 reads Gamma (+ shift on the diagonal) wherever
  // later steps read L, and every lower element is written by step 0
  if (tid == 0) fail = 0;
  __syncthreads();

  const int nblk = (R + CB - 1) / CB;
  // unblocked Cholesky of diagonal block jb by warp 0 in registers: lane =
  // row, a[c] = A[lane][c]; every loop is unrolled, so a[] never leaves the
  // register file, and shuffles carry the pivot column.  Block 0 reads Gamma
  // (+ shift), later blocks the trailing-updated L.
  auto factor_diag = [&](int jb) {
    const int j0 = jb * CB, bw = min(CB, R - j0);
    const double* src = jb == 0 ? gamma : L;
    const double dshift = jb == 0 ? shift : 0.0;
    double a[CB];
    const bool in = lane < bw;
#pragma unroll
    for (int c = 0; c < CB; ++c)
      a[c] = (in && c <= lane) ? src[int64_t(j0 + lane) * R + j0 + c] + (c == lane ? dshift : 0.0) : 0.0;
    int bad = 0;
#pragma unroll
    for (int k = 0; k < CB; ++k) {
      if (k < bw && bad == 0) {  // warp-uniform
        const double dkk = __shfl_sync(~0u, a[k], k);
        if (!(dkk > 0.0)) {  // also catches NaN
          bad = k + 1;
        } else {
          // potf2 scales the column by 1 / sqrt(pivot); rsqrt is one MUFU
          // + Newton steps, shorter than sqrt then a reciprocal
          const double rl = rsqrt(dkk);
          a[k] = lane == k ? dkk * rl : (lane > k ? a[k] * rl : 0.0);
          colk[lane] = a[k];  // column k, read back as broadcasts
          __syncwarp();
          // unpredicated: lanes < c only touch their (unused) upper entries
#pragma unroll
          for (int c = 1; c < CB; ++c) {  // constant trip count: unrolls fully
            if (c <= k) continue;
            a[c] = fma(-a[k], colk[c], a[c]);
          }
          __syncwarp();
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CB; ++c) dg[lane * 33 + c] = a[c];
    __syncwarp();
    if (bad) {
      if (lane == 0) fail = j0 + bad;
    } else {
#pragma unroll
      for (int c = 0; c < CB; ++c)
        if (in && c <= lane) L[int64_t(j0 + lane) * R + j0 + c] = a[c];
      rdg[lane] = lane < bw ? 1.0 / dg[lane * 33 + lane] : 0.0;
    }
  };
  // the last warp inverts a factored diagonal block for the row solve: lane
  // j = column j of L_bb^-1 (forward substitution on e_j); its strictly-lower
  // part goes, transposed, into the unused upper triangle of the block:
  // L[j0 + j][j0 + i] = (L_bb^-1)[i][j], i > j
  auto invert_diag = [&](int j0, int bw) {
    double x[CB];
#pragma unroll
    for (int i = 0; i < CB; ++i) {
      double v = i == lane ? 1.0 : 0.0;
#pragma unroll
      for (int u = 0; u < i; ++u) v = fma(-dg[i * 33 + u], x[u], v);  // x[u] = 0 for u < lane
      x[i] = i >= lane ? v * rdg[i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < CB; ++i)
      if (i > lane && i < bw) L[int64_t(j0 + lane) * R + j0 + i] = x[i];
  };
  // One copy of each unrolled helper in the code (instruction cache): the
  // loop starts at j = -1, whose only work is factoring diagonal block 0.
  const int grp = tid >> 6, gl = tid & 63, ty = gl >> 3, tx = gl & 7;
  constexpr int NGRP = CHOL_THREADS / 64;
  int p0 = 0, np = 0, nb2 = 0;
  const double* src = gamma;
  double dshift = 0.0;
  // trailing lower triangle -= P P^T in 32 x 32 tiles (bi, bl), bl <= bi,
  // one tile per 64-thread group (4 x 4 per thread)
  auto update_tile = [&](int bi, int bl) {
    const int r0 = bi * CB + ty * 4, c0 = bl * CB + tx * 4;
    double acc[4][4];  // starts as the old values, loaded before the products
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int rr = r0 + i, cc = c0 + jj;
        acc[i][jj] = (rr < np && cc <= rr) ? src[int64_t(p0 + rr) * R + p0 + cc] + (rr == cc ? dshift : 0.0) : 0.0;
      }
#pragma unroll 8
    for (int u = 0; u < CB; ++u) {
      double pr[4], pc[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        pr[i] = pan[(r0 + i) * 33 + u];
        pc[i] = pan[(c0 + i) * 33 + u];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fma(-pr[i], pc[jj], acc[i][jj]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int rr = r0 + i, cc = c0 + jj;
        if (rr < np && cc <= rr) L[int64_t(p0 + rr) * R + p0 + cc] = acc[i][jj];
      }
  };
  auto tri = [](int t, int& bi, int& bl) {  // t-th tile of a lower triangle, row-major
    bi = 0;
    bl = t;
    while (bl > bi) {
      bl -= bi + 1;
      ++bi;
    }
  };
#pragma unroll 1
  for (int j = -1; j < nblk; ++j) {
    // look-ahead when the trailing matrix has >= 4 block rows: the next block
    // column's tiles first, then warp 0 factors the next diagonal block while
    // groups 1.. update the rest (a shorter trailing matrix: all tiles, then
    // the factorization; the extra barrier would cost more than it hides)
    bool la = false;
    if (j >= 0) {
      const int j0 = j * CB;
      src = j == 0 ? gamma : L;
      dshift = j == 0 ? shift : 0.0;
      // panel rows p0..: X L_jj^T = A, solved in place in shared memory (none
      // for the last block: every loop below is empty)
      p0 = j0 + CB;
      np = max(0, R - p0);
      const int npr = ((np + CB - 1) / CB) * CB;
      for (int t0 = warp; t0 < npr; t0 += 8 * (CHOL_THREADS / 32)) {  // 8 rows in flight per warp
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + u * (CHOL_THREADS / 32);
          v[u] = t < np ? src[int64_t(p0 + t) * R + j0 + lane] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int t = t0 + u * (CHOL_THREADS / 32);
          if (t < npr) pan[t * 33 + lane] = v[u];
        }
      }
      __syncthreads();
      static_assert(CHOL_KERNEL_CAP - CB <= CHOL_THREADS - 32, "one panel row per thread, last warp free");
      if (warp == CHOL_THREADS / 32 - 1) invert_diag(j0, min(CB, R - j0));  // meanwhile
      if (tid < np) {  // not a loop: the dg reads would be hoisted and spill
        const int t = tid;
        double x[CB];  // fully unrolled: stays in registers
#pragma unroll
        for (int c = 0; c < CB; ++c) x[c] = pan[t * 33 + c];
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          double v = x[c];
#pragma unroll
          for (int u = 0; u < c; ++u) v = fma(-x[u], dg[c * 33 + u], v);
          x[c] = v * rdg[c];
        }
#pragma unroll
        for (int c = 0; c < CB; ++c) pan[t * 33 + c] = x[c];
      }
      __syncthreads();
      for (int idx = tid; idx < np * CB; idx += CHOL_THREADS) {
        const int t = idx >> 5, c = idx & 31;
        L[int64_t(p0 + t) * R + j0 + c] = pan[t * 33 + c];
      }
      nb2 = npr / CB;
      la = nb2 >= 4;
      const int n1 = la ? nb2 : nb2 * (nb2 + 1) / 2;
      for (int t = grp; t < n1; t += NGRP) {
        int bi = t, bl = 0;
        if (!la) tri(t, bi, bl);
        update_tile(bi, bl);
      }
      __syncthreads();
    }
    if (j + 1 < nblk) {
      if (warp == 0) {
        factor_diag(j + 1);  // its block is trailing tile (0, 0), already updated
      } else if (la && grp > 0) {
        const int m = nb2 - 1, nt = m * (m + 1) / 2;  // tiles 1 <= bl <= bi
        for (int t = grp - 1; t < nt; t += NGRP - 1) {
          int bi, bl;
          tri(t, bi, bl);
          update_tile(bi + 1, bl + 1);
        }
      }
      __syncthreads();
      if (fail) {
        if (tid == 0) *info = fail;
        return;
      }
    }
  }
  if (tid == 0) *info = 0;
}

// X L L^T = G for every row of G (rows x R, row-major, ld R), skipped when
// *info != 0.  RW rows per warp, ROWS_WARPS warps per CTA; the rows live in
// shared memory interleaved (z[c][q]), lane j owns column tb * 32 + j of the
// current 32-column block.  The 2 nblk steps (forward blocks 0.., backward
// blocks ..0) each need a strip of L and the raw diagonal block (its lower
// triangle L_bb, its upper the transposed inverse chol_small parks there);
// they are staged with cp.async into two buffers, the next step's while the
// current one computes (DB; one buffer when two do not fit, R > 256).  Each
// warp then runs the dot-product part from shared memory (RW independent
// chains per strip element) and the in-block solve as a 32 x 32 GEMV with
// the inverse.  Forward Z L^T = G needs L[t][u] (u < t), backward X L = Z
// needs L[c][t] (c > t): both from the lower triangle.
constexpr int ROWS_WARPS = 4;

template <int RW>
__device__ __forceinline__ void zrow(const double* z, double (&v)[RW]) {  // one interleaved row of z
  if constexpr (RW == 4) {
    const double4 t = *reinterpret_cast<const double4*>(z);
    v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
  } else if constexpr (RW == 2) {
    const double2 t = *reinterpret_cast<const double2*>(z);
    v[0] = t.x, v[1] = t.y;
  } else {
    v[0] = z[0];
  }
}

static size_t rows_smem(int64_t R, int rw, bool db) {
  const int64_t rp = (R + 31) / 32 * 32;
  const int64_t nb = db ? 2 : 1;
  return size_t(nb * (rp * 33 + 32 * 33) + int64_t(ROWS_WARPS) * rw * rp + 32) * sizeof(double);
}

template <int RW, bool DB>
__global__ void __launch_bounds__(ROWS_WARPS * 32) chol_rows_kernel(const double* __restrict__ LU, int R,
                                                                    double* __restrict__ G, int64_t rows,
                                                                    const int* __restrict__ info) {
  if (*info != 0) return;
  extern __shared__ __align__(16) double rsm[];
  const int rp = (R + 31) / 32 * 32;
  double* zall = rsm;                                    // [warp][rp][RW]
  double* rdiag = zall + ROWS_WARPS * RW * rp;           // [32]
  double* bufs = rdiag + 32;                             // DB ? 2 : 1 x {strip [rp][33], dblk [32][33]}
  const int buf_elems = rp * 33 + 32 * 33;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q0 = (int64_t(blockIdx.x) * ROWS_WARPS + warp) * RW;
  const bool active = q0 < rows;  // inactive warps still help stage strips
  double* z = zall + int64_t(warp) * rp * RW;
  for (int c = lane; c < rp; c += 32)
#pragma unroll
    for (int q = 0; q < RW; ++q) z[c * RW + q] = (active && q0 + q < rows && c < R) ? G[(q0 + q) * R + c] : 0.0;
  const int nblk = rp / 32, nsteps = 2 * nblk;
  // step s: forward block s, then backward blocks nblk-1 .. 0
  auto block_of = [&](int s) { return s < nblk ? s : 2 * nblk - 1 - s; };
  auto issue = [&](int s, int b) {
    const int b0 = block_of(s) * 32;
    double* strip = bufs + b * buf_elems;
    double* dblk = strip + rp * 33;
    for (int e = threadIdx.x; e < 32 * 32; e += ROWS_WARPS * 32) {  // raw diagonal block
      const int r = e >> 5, c = e & 31;
      const bool ok = b0 + r < R && b0 + c < R;
      cp_async8(dblk + r * 33 + c, ok ? LU + int64_t(b0 + r) * R + b0 + c : LU, ok ? 8 : 0);
    }
    if (s < nblk) {  // forward: strip[u][t] = L[b0 + t][u], u < b0 (lanes along u)
      for (int t = warp; t < 32; t += ROWS_WARPS)
        for (int u = lane; u < b0; u += 32) {
          const bool ok = b0 + t < R;
          cp_async8(strip + u * 33 + t, ok ? LU + int64_t(b0 + t) * R + u : LU, ok ? 8 : 0);
        }
    } else {  // backward: strip[c][t] = L[c][b0 + t], c >= b0 + 32 (lanes along t)
      for (int c = b0 + 32 + warp; c < rp; c += ROWS_WARPS) {
        const bool ok = c < R && b0 + lane < R;
        cp_async8(strip + c * 33 + lane, ok ? LU + int64_t(c) * R + b0 + lane : LU, ok ? 8 : 0);
      }
    }
    cp_async_commit();
  };
  issue(0, 0);
  for (int s = 0; s < nsteps; ++s) {
    const int b = DB ? (s & 1) : 0;
    if (DB && s + 1 < nsteps) {
      issue(s + 1, (s + 1) & 1);  // the next step's strip, behind this one's math
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* strip = bufs + b * buf_elems;
    const double* dblk = strip + rp * 33;
    const int b0 = block_of(s) * 32, t = b0 + lane;
    if (threadIdx.x < 32) rdiag[threadIdx.x] = b0 + threadIdx.x < R ? 1.0 / dblk[threadIdx.x * 34] : 0.0;
    __syncthreads();
    if (active) {
      double acc[RW];
#pragma unroll
      for (int q = 0; q < RW; ++q) acc[q] = z[t * RW + q];
      if (s < nblk) {
        // forward: z_t = (g_t - sum_{u<t} z_u L[t][u]) / L[t][t]
#pragma unroll 8
        for (int u = 0; u < b0; ++u) {
          const double w = strip[u * 33 + lane];
          double zu[RW];
          zrow<RW>(z + u * RW, zu);
#pragma unroll
          for (int q = 0; q < RW; ++q) acc[q] = fma(-zu[q], w, acc[q]);
        }
        // in-block: z_b = L_bb^-1 rhs_b (a 32 x 32 GEMV, no sequential chain)
#pragma unroll
        for (int q = 0; q < RW; ++q) z[t * RW + q] = acc[q];
        __syncwarp();
        const double rd = rdiag[lane];
#pragma unroll
        for (int q = 0; q < RW; ++q) acc[q] *= rd;
#pragma unroll
        for (int u = 0; u < 31; ++u) {
          const double w = u < lane ? dblk[u * 33 + lane] : 0.0;  // (L_bb^-1)[t][u]
          double zu[RW];
          zrow<RW>(z + (b0 + u) * RW, zu);
#pragma unroll
          for (int q = 0; q < RW; ++q) acc[q] = fma(w, zu[q], acc[q]);
        }
      } else {
        // backward: x_t = (z_t - sum_{c>t} x_c L[c][t]) / L[t][t]
#pragma unroll 8
        for (int c = b0 + 32; c < R; ++c) {
          const double w = strip[c * 33 + lane];
          double zc[RW];
          zrow<RW>(z + c * RW, zc);
#pragma unroll
          for (int q = 0; q < RW; ++q) acc[q] = fma(-zc[q], w, acc[q]);
        }
        // in-block: x_b = rhs_b L_bb^-1, x_t = sum_{u >= t} rhs_u (L_bb^-1)[u][t]
#pragma unroll
        for (int q = 0; q < RW; ++q) z[t * RW + q] = acc[q];
        __syncwarp();
        const double rd = rdiag[lane];
#pragma unroll
        for (int q = 0; q < RW; ++q) acc[q] *= rd;
#pragma unroll
        for (int u = 1; u < 32; ++u) {
          const double w = u > lane ? dblk[lane * 33 + u] : 0.0;  // (L_bb^-1)[u][t]
          double zu[RW];
          zrow<RW>(z + (b0 + u) * RW, zu);
#pragma unroll
          for (int q = 0; q < RW; ++q) acc[q] = fma(w, zu[q], acc[q]);
        }
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < RW; ++q) z[t * RW + q] = acc[q];
      __syncwarp();
    }
    __syncthreads();  // buffer b is refilled two steps on (one, without DB)
    if (!DB && s + 1 < nsteps) issue(s + 1, 0);
  }
  if (!active) return;
  for (int c = lane; c < R; c += 32)
#pragma unroll
    for (int q = 0; q < RW; ++q)
      if (q0 + q < rows) G[(q0 + q) * R + c] = z[c * RW + q];
}

// Solve paths: R <= CHOL_SMALL_MAX the one-CTA Cholesky + row solve above;
// larger R the multi-CTA sweep (sweep_inv.cu: Gamma^-1 on the factor side,
// X = G Gamma^-1 as one MTTKRP-kernel GEMM on the apply side); cuSOLVER
// potrf / potrs only when forced.  CPK_SOLVE=kernel / sweep / cusolver
// force a path (A/B comparisons and tests; `kernel` up to CHOL_KERNEL_CAP).
enum class SolvePath { Small, Sweep, Cusolver };

static SolvePath solve_path(int64_t R) {
  const char* e = getenv("CPK_SOLVE");
  if (e && strcmp(e, "cusolver") == 0) return SolvePath::Cusolver;
  if (e && strcmp(e, "sweep") == 0) return SolvePath::Sweep;
  if (e && strcmp(e, "kernel") == 0 && R <= CHOL_KERNEL_CAP) return SolvePath::Small;
  return R <= CHOL_SMALL_MAX ? SolvePath::Small : SolvePath::Sweep;
}

static bool use_small_chol(int64_t R) { return solve_path(R) == SolvePath::Small; }

static int chol_small(const double* gamma, int64_t R, double eps, double* L, int* info, cudaStream_t st) {
  const cudaError_t attr = cudaFuncSetAttribute(chol_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                int(chol_smem(CHOL_KERNEL_CAP)));
  if (attr != cudaSuccess) return fail(CPK_ERR_CUDA, "chol smem attribute: %s", cudaGetErrorString(attr));
  chol_small_kernel<<<1, CHOL_THREADS, chol_smem(R), st>>>(gamma, int(R), eps, L, info);
  return check_launch("chol_small");
}

template <int RW, bool DB>
static int chol_rows_launch(const double* LU, int64_t R, double* G, int64_t rows, const int* info, cudaStream_t st) {
  const size_t smem = rows_smem(R, RW, DB);
  if (cudaFuncSetAttribute(chol_rows_kernel<RW, DB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) !=
      cudaSuccess)
    return check_launch("chol_rows smem attribute");
  const unsigned grid = unsigned((rows + ROWS_WARPS * RW - 1) / (ROWS_WARPS * RW));
  chol_rows_kernel<RW, DB><<<grid, ROWS_WARPS * 32, smem, st>>>(LU, int(R), G, rows, info);
  return check_launch("chol_rows");
}

static int chol_rows(const double* LU, int64_t R, double* G, int64_t rows, const int* info, cudaStream_t st) {
  if (rows <= 0) return CPK_OK;
  // few rows: one row per warp (more CTAs, the strips' loads are hidden);
  // many: 4 per warp (each strip element feeds 4 chains).  R = 256
  // (tools/solve_bench.py, factor + rows): 128 rows 233 / 244 / 252 us for
  // RW = 1 / 2 / 4, 1024 rows 285 / 244 / 252, 4096 rows 542 / 430 / 324.
  if (rows <= 256 && rows_smem(R, 1, true) <= 227 * 1024) return chol_rows_launch<1, true>(LU, R, G, rows, info, st);
  if (rows <= 1024 && rows_smem(R, 2, true) <= 227 * 1024)
    return chol_rows_launch<2, true>(LU, R, G, rows, info, st);
  if (rows_smem(R, 4, true) <= 227 * 1024) return chol_rows_launch<4, true>(LU, R, G, rows, info, st);
  return chol_rows_launch<4, false>(LU, R, G, rows, info, st);
}

struct SolverCtx {
  cusolverDnHandle_t h = nullptr;
  int dev = -1;
};
static thread_local SolverCtx g_solver;

static int solver_for(cudaStream_t st, cusolverDnHandle_t* out) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_solver.h == nullptr || g_solver.dev != dev) {
    if (g_solver.h) cusolverDnDestroy(g_solver.h);
    g_solver.h = nullptr;
    if (cusolverDnCreate(&g_solver.h) != CUSOLVER_STATUS_SUCCESS) return fail(CPK_ERR_LIB, "cusolverDnCreate failed");
    g_solver.dev = dev;
  }
  if (cusolverDnSetStream(g_solver.h, st) != CUSOLVER_STATUS_SUCCESS) return fail(CPK_ERR_LIB, "cusolverDnSetStream");
  *out = g_solver.h;
  return CPK_OK;
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace cpk

using namespace cpk;

extern "C" int cpk_gram_f64(const double* A, int64_t rows, int64_t rank, int64_t lda, double* gram, void* stream) {
  if (!A || !gram) return fail(CPK_ERR_PARAM, "NULL pointer");
  if (rows < 1 || rank < 1 || lda < rank) return fail(CPK_ERR_SHAPE, "bad gram shape");
  const int64_t nt = (rank + GT - 1) / GT;
  if (cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(GRAM_SMEM)) != cudaSuccess)
    return check_launch("gram smem attribute");
  gram_kernel<<<unsigned(nt * (nt + 1) / 2), 256, GRAM_SMEM, as_stream(stream)>>>(A, rows, rank, lda, gram);
  return check_launch("gram");
}

extern "C" int cpk_hadamard_f64(const double* const* grams, int n, int skip, int64_t rank, double* out,
                                void* stream) {
  if (!grams || !out || n < 0 || n > CPK_MAX_MODES) return fail(CPK_ERR_PARAM, "bad hadamard arguments");
  GramList gl{};
  gl.n = n;
  gl.skip = skip;
  for (int m = 0; m < n; ++m) {
    gl.g[m] = grams[m];
    if (m != skip && !grams[m]) return fail(CPK_ERR_PARAM, "gram %d is NULL", m);
  }
  const int64_t rr = rank * rank;
  const unsigned blocks = unsigned(std::min<int64_t>((rr + 255) / 256, 148 * 8));
  hadamard_kernel<<<std::max(blocks, 1u), 256, 0, as_stream(stream)>>>(gl, rr, out);
  return check_launch("hadamard");
}

extern "C" int cpk_colnorms_sq_f64(const double* A, int64_t rows, int64_t rank, int64_t lda, double* normsq,
                                   void* stream) {
  if (!A || !normsq || rank < 1 || lda < rank || rows < 0) return fail(CPK_ERR_PARAM, "bad colnorms arguments");
  colnorms_kernel<<<unsigned((rank + 31) / 32), 256, 0, as_stream(stream)>>>(A, rows, rank, lda, normsq);
  return check_launch("colnorms");
}

extern "C" int cpk_scale_columns_f64(double* A, int64_t rows, int64_t rank, int64_t lda, const double* normsq,
                                     double* lam, void* stream) {
  if (!A || !normsq || rank < 1 || lda < rank || rows < 0) return fail(CPK_ERR_PARAM, "bad scale arguments");
  if (rows == 0) return CPK_OK;
  const int64_t total = rows * rank;
  const unsigned blocks = unsigned(std::min<int64_t>((total + 255) / 256, 148 * 8));
  scale_columns_kernel<<<blocks, 256, 0, as_stream(stream)>>>(A, rows, rank, lda, normsq, lam);
  return check_launch("scale_columns");
}

extern "C" int cpk_normalize_columns_f64(double* A, int64_t rows, int64_t rank, int64_t lda, double* lam,
                                         double* normsq_work, void* stream) {
  int rc = cpk_colnorms_sq_f64(A, rows, rank, lda, normsq_work, stream);
  if (rc) return rc;
  return cpk_scale_columns_f64(A, rows, rank, lda, normsq_work, lam, stream);
}

extern "C" int cpk_fit_terms_f64(const double* H, const double* lam, const double* G, const double* A,
                                 int64_t rows, int64_t rank, double* out2, void* stream) {
  if (!H || !lam || !out2) return fail(CPK_ERR_PARAM, "NULL pointer");
  fit_terms_kernel<<<1, 1024, 0, as_stream(stream)>>>(H, lam, G, A, rows, rank, out2);
  return check_launch("fit_terms");
}

extern "C" int cpk_sumsq_f64(const double* x, int64_t n, double* work, double* out, void* stream) {
  if (!x || !work || !out || n < 0) return fail(CPK_ERR_PARAM, "bad sumsq arguments");
  sumsq_partial_kernel<<<CPK_SUMSQ_PARTIALS, 256, 0, as_stream(stream)>>>(x, n, work);
  sumsq_final_kernel<<<1, 1024, 0, as_stream(stream)>>>(work, CPK_SUMSQ_PARTIALS, out);
  return check_launch("sumsq");
}

// work layout (cuSOLVER / small-R paths): [gamma copy R*R][potrf lwork][info int]
static int solve_layout(int64_t rows, int64_t rank, int lwork, size_t* total, size_t* off_lwork, size_t* off_info) {
  (void)rows;
  const size_t g = align_up(size_t(rank) * size_t(rank) * sizeof(double));
  const size_t w = align_up(size_t(std::max(lwork, 1)) * sizeof(double));
  *off_lwork = g;
  *off_info = g + w;
  *total = g + w + 256;
  return CPK_OK;
}

// work layout (sweep path): [sweep_factor_bytes: Gamma^-1 (Rp x Rp) ...]
// [copy of G: rows x R][MTTKRP workspace of the apply GEMM]
static int apply_mttkrp_bytes(int64_t rows, int64_t rank, size_t* bytes) {
  *bytes = 0;
  if (rows <= 0) return CPK_OK;
  // The split-K layout depends on the output-tile count (split chain vs
  // partial copies, mttkrp.cu), so the size is not monotone in rows, and a
  // caller sizes one workspace for its largest mode: take the maximum over
  // every row count up to `rows` (tile boundaries are multiples of 64).
  const int64_t step = std::max<int64_t>(64, (rows / 256 + 63) / 64 * 64);
  for (int64_t i = -1, r = rows; r > 0; ++i, r = rows / step * step - i * step) {
    if (i >= 0 && r == rows) continue;  // already counted
    const int64_t dims[2] = {rank, r};
    size_t b = 0;
    const int rc = cpk_mttkrp_workspace_bytes(2, dims, 1, rank, nullptr, &b);
    if (rc) return rc;
    *bytes = std::max(*bytes, b);
  }
  return CPK_OK;
}

static int* info_d_sweep(void* work, int64_t rank) {  // the info word at the end of the factor block
  return reinterpret_cast<int*>(static_cast<char*>(work) + sweep_factor_bytes(rank) - 256);
}

static int sweep_layout_bytes(int64_t rows, int64_t rank, size_t* total) {
  size_t m = 0;
  const int rc = apply_mttkrp_bytes(rows, rank, &m);
  if (rc) return rc;
  *total = sweep_factor_bytes(rank) + align_up(size_t(std::max<int64_t>(rows, 0)) * size_t(rank) * sizeof(double)) +
           align_up(m);
  return CPK_OK;
}

// X Gamma = G in place as X = G Gamma^-1: G is copied aside and read back as
// the R x rows first-mode-fastest tensor T[c, i] = G[i][c] whose mode-1
// MTTKRP with the factor Gamma^-1 (ld Rp) is X[i][j] = sum_c G[i][c] W[c][j]
// -- the hot MTTKRP kernel does the GEMM.
static int sweep_apply(double* G, int64_t rows, int64_t rank, void* work, size_t work_bytes, cudaStream_t st) {
  if (rows <= 0) return CPK_OK;
  size_t need = 0;
  int rc = sweep_layout_bytes(rows, rank, &need);
  if (rc) return rc;
  if (work_bytes < need) return fail(CPK_ERR_RESOURCE, "solve workspace needs %zu bytes, got %zu", need, work_bytes);
  char* base = static_cast<char*>(work);
  double* tmp = reinterpret_cast<double*>(base + sweep_factor_bytes(rank));
  const size_t tmp_bytes = align_up(size_t(rows) * size_t(rank) * sizeof(double));
  void* mws = base + sweep_factor_bytes(rank) + tmp_bytes;
  const size_t mws_bytes = work_bytes - sweep_factor_bytes(rank) - tmp_bytes;
  if (cudaMemcpyAsync(tmp, G, size_t(rows) * size_t(rank) * sizeof(double), cudaMemcpyDeviceToDevice, st) !=
      cudaSuccess)
    return fail(CPK_ERR_CUDA, "solve apply copy failed");
  const int64_t dims[2] = {rank, rows};
  const double* fac[2] = {sweep_inverse_matrix(work), nullptr};
  const int64_t ld[2] = {sweep_padded(rank), rank};
  return cpk_mttkrp_f64(tmp, 2, dims, 1, fac, ld, nullptr, rank, G, rank, nullptr, mws, mws_bytes, st);
}

static int potrf_lwork(int64_t rank, int* lwork) {
  cusolverDnHandle_t h;
  int rc = solver_for(nullptr, &h);
  if (rc) return rc;
  if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, int(rank), nullptr, int(rank), lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(CPK_ERR_LIB, "potrf_bufferSize failed");
  return CPK_OK;
}

extern "C" int cpk_solve_workspace_bytes(int64_t rows, int64_t rank, size_t* bytes) {
  if (!bytes || rank < 1 || rank > (1 << 30)) return fail(CPK_ERR_PARAM, "bad solve arguments");
  int lwork = 0;
  int rc = potrf_lwork(rank, &lwork);
  if (rc) return rc;
  size_t a, b, sw = 0;
  rc = solve_layout(rows, rank, lwork, bytes, &a, &b);
  if (rc) return rc;
  // room for every path (CPK_SOLVE may switch between calls)
  if (rank > CHOL_SMALL_MAX || getenv("CPK_SOLVE")) {
    rc = sweep_layout_bytes(rows, rank, &sw);
    if (rc) return rc;
    *bytes = std::max(*bytes, sw);
  }
  return CPK_OK;
}

extern "C" int cpk_solve_normal_f64(const double* gamma, double* G, int64_t rows, int64_t rank, void* work,
                                    size_t work_bytes, void* stream) {
  if (!gamma || !G || !work || rank < 1 || rows < 0) return fail(CPK_ERR_PARAM, "bad solve arguments");
  cudaStream_t st = as_stream(stream);
  cusolverDnHandle_t h;
  int rc = solver_for(st, &h);
  if (rc) return rc;
  int lwork = 0;
  if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, int(rank), nullptr, int(rank), &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(CPK_ERR_LIB, "potrf_bufferSize failed");
  size_t total, off_w, off_info;
  solve_layout(rows, rank, lwork, &total, &off_w, &off_info);
  if (work_bytes < total) return fail(CPK_ERR_RESOURCE, "solve workspace needs %zu bytes, got %zu", total, work_bytes);
  char* base = static_cast<char*>(work);
  double* L = reinterpret_cast<double*>(base);
  double* w = reinterpret_cast<double*>(base + off_w);
  int* info_d = reinterpret_cast<int*>(base + off_info);
  const unsigned cblocks = unsigned(std::min<int64_t>((rank * rank + 255) / 256, 148 * 4));
  // Rung 0 is the plain Cholesky; rungs 1..5 add eps tr/R I, eps = 1e-12 * 1e3^i
  double eps = 0.0;
  const SolvePath path = solve_path(rank);
  const bool small = path == SolvePath::Small;
  for (int rung = 0; rung <= 5; ++rung) {
    if (path == SolvePath::Sweep) {
      rc = sweep_inverse(gamma, rank, eps, work, work_bytes, info_d_sweep(work, rank), 0, st);
      if (rc) return rc;
      int info = 0;
      if (cudaMemcpyAsync(&info, info_d_sweep(work, rank), sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess)
        return fail(CPK_ERR_CUDA, "sweep info readback failed");
      if (info == 0) return sweep_apply(G, rows, rank, work, work_bytes, st);
      eps = rung == 0 ? 1e-12 : eps * 1e3;
      continue;
    }
    if (small) {
      rc = chol_small(gamma, rank, eps, L, info_d, st);
      if (rc) return rc;
      int info = 0;
      if (cudaMemcpyAsync(&info, info_d, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess)
        return fail(CPK_ERR_CUDA, "chol info readback failed");
      if (info == 0) return chol_rows(L, rank, G, rows, info_d, st);
      eps = rung == 0 ? 1e-12 : eps * 1e3;
      continue;
    }
    copy_regularize_kernel<<<std::max(cblocks, 1u), 256, 0, st>>>(gamma, rank, eps, L);
    rc = check_launch("copy_regularize");
    if (rc) return rc;
    // Gamma is symmetric, so row-major == column-major; UPPER as scipy's
    // cho_factor(lower=False) (cpals.py:79)
    if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, int(rank), L, int(rank), w, lwork, info_d) !=
        CUSOLVER_STATUS_SUCCESS)
      return fail(CPK_ERR_LIB, "potrf failed");
    int info = 0;
    if (cudaMemcpyAsync(&info, info_d, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return fail(CPK_ERR_CUDA, "potrf info readback failed");
    if (info == 0) {
      // X Gamma = G  <=>  Gamma X^T = G^T; row-major G is column-major G^T
      if (rows > 0 && cusolverDnDpotrs(h, CUBLAS_FILL_MODE_UPPER, int(rank), int(rows), L, int(rank), G, int(rank),
                                       info_d) != CUSOLVER_STATUS_SUCCESS)
        return fail(CPK_ERR_LIB, "potrs failed");
      return check_launch("potrs");
    }
    eps = rung == 0 ? 1e-12 : eps * 1e3;
  }
  return fail(CPK_ERR_NOT_PD, "Gamma is not positive definite after 5 regularization rungs");
}

extern "C" int cpk_solve_factor_spec_f64(const double* gamma, int64_t rank, void* work, size_t work_bytes,
                                         int* info_out, void* stream) {
  if (!gamma || !work || !info_out || rank < 1) return fail(CPK_ERR_PARAM, "bad solve arguments");
  cudaStream_t st = as_stream(stream);
  cusolverDnHandle_t h;
  int rc = solver_for(st, &h);
  if (rc) return rc;
  int lwork = 0;
  if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, int(rank), nullptr, int(rank), &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(CPK_ERR_LIB, "potrf_bufferSize failed");
  size_t total, off_w, off_info;
  solve_layout(0, rank, lwork, &total, &off_w, &off_info);
  if (work_bytes < total) return fail(CPK_ERR_RESOURCE, "solve workspace needs %zu bytes, got %zu", total, work_bytes);
  char* base = static_cast<char*>(work);
  double* L = reinterpret_cast<double*>(base);
  double* w = reinterpret_cast<double*>(base + off_w);
  if (use_small_chol(rank)) return chol_small(gamma, rank, 0.0, L, info_out, st);
  if (solve_path(rank) == SolvePath::Sweep) {
    // On the side stream the sweep runs beside the mode's MTTKRP: a
    // full-machine cooperative grid fights it for SMs, 16 CTAs stay hidden
    // behind it (128^4, R = 300: 21.2 ms per sweep either way; small-tensor
    // R = 512 runs 4.7 -> 4.4 ms; c5 hides either; profiles/r02_sweep_ctas*.log).
    // CPK_SWEEP_CTAS overrides (0 = full machine).
    const char* c = getenv("CPK_SWEEP_CTAS");
    const int ctas = c ? atoi(c) : std::min(16, sweep_default_ctas(rank));
    return sweep_inverse(gamma, rank, 0.0, work, work_bytes, info_out, ctas, st);
  }
  const unsigned cblocks = unsigned(std::min<int64_t>((rank * rank + 255) / 256, 148 * 4));
  copy_regularize_kernel<<<std::max(cblocks, 1u), 256, 0, st>>>(gamma, rank, 0.0, L);
  rc = check_launch("copy_regularize");
  if (rc) return rc;
  // rung 0 only, and no readback: the caller checks *info_out later
  if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, int(rank), L, int(rank), w, lwork, info_out) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(CPK_ERR_LIB, "potrf failed");
  return check_launch("potrf");
}

extern "C" int cpk_solve_apply_spec_f64(double* G, int64_t rows, int64_t rank, void* work, size_t work_bytes,
                                        const int* info_out, void* stream) {
  if (!G || !work || !info_out || rank < 1 || rows < 0) return fail(CPK_ERR_PARAM, "bad solve arguments");
  cudaStream_t st = as_stream(stream);
  cusolverDnHandle_t h;
  int rc = solver_for(st, &h);
  if (rc) return rc;
  int lwork = 0;
  if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, int(rank), nullptr, int(rank), &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(CPK_ERR_LIB, "potrf_bufferSize failed");
  size_t total, off_w, off_info;
  solve_layout(rows, rank, lwork, &total, &off_w, &off_info);
  if (work_bytes < total) return fail(CPK_ERR_RESOURCE, "solve workspace needs %zu bytes, got %zu", total, work_bytes);
  char* base = static_cast<char*>(work);
  double* L = reinterpret_cast<double*>(base);
  int* info_d = reinterpret_cast<int*>(base + off_info);
  if (use_small_chol(rank)) return chol_rows(L, rank, G, rows, info_out, st);
  // a failed factor (sweep or potrf) just produces garbage, which the caller discards
  if (solve_path(rank) == SolvePath::Sweep) return sweep_apply(G, rows, rank, work, work_bytes, st);
  // potrs on a failed factor just produces garbage, which the caller discards
  if (rows > 0 && cusolverDnDpotrs(h, CUBLAS_FILL_MODE_UPPER, int(rank), int(rows), L, int(rank), G, int(rank),
                                   info_d) != CUSOLVER_STATUS_SUCCESS)
    return fail(CPK_ERR_LIB, "potrs failed");
  return check_launch("potrs");
}

extern "C" int cpk_solve_normal_spec_f64(const double* gamma, double* G, int64_t rows, int64_t rank, void* work,
                                         size_t work_bytes, int* info_out, void* stream) {
  if (!gamma || !G || !work || !info_out || rank < 1 || rows < 0) return fail(CPK_ERR_PARAM, "bad solve arguments");
  const int rc = cpk_solve_factor_spec_f64(gamma, rank, work, work_bytes, info_out, stream);
  if (rc) return rc;
  return cpk_solve_apply_spec_f64(G, rows, rank, work, work_bytes, info_out, stream);
}
