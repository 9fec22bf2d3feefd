// On-device CP-ALS step kernels: Gram, Hadamard of Grams, the normal-equation
// solve with the reference's regularization ladder, column normalization and
// the factored fit terms.  Reference: pkg/src/cpkern/cpals.py:75-152 and
// kruskal.py:74-114.  Every reduction runs in a fixed order, so a sweep is
// bit-reproducible run to run (README.md "same seed, same trajectory").
#include "common.cuh"

#include <cusolverDn.h>

#include <algorithm>
#include <vector>

namespace cpk {

// ---------------------------------------------------------------- Gram
// A^T A for A (rows x R, row-major, lda): 64x64 output tiles, 256 threads with
// 4x4 register micro-tiles, rows staged 16 at a time.  Only tiles on or above
// the diagonal are launched; every (a <= b) entry is written to both (a, b)
// and (b, a) -- exact symmetry as kruskal.gram (kruskal.py:110-114).
constexpr int GT = 64, GK = 16;

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
  __shared__ double sa[GK][GT + 1], sb[GK][GT + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  const int64_t a0 = ti * GT, b0 = tj * GT;
  for (int64_t r0 = 0; r0 < rows; r0 += GK) {
    for (int e = threadIdx.x; e < GK * GT; e += 256) {
      const int kr = e / GT, c = e % GT;
      const int64_t r = r0 + kr;
      sa[kr][c] = (r < rows && a0 + c < R) ? A[r * lda + a0 + c] : 0.0;
      sb[kr][c] = (r < rows && b0 + c < R) ? A[r * lda + b0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kr = 0; kr < GK; ++kr) {
      double x[4], y[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[i] = sa[kr][ty + 16 * i];
        y[i] = sb[kr][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(x[i], y[j], acc[i][j]);
    }
    __syncthreads();
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

// out[0] = lam^T H lam  ((lam @ H) @ lam as cpals.py:146), out[1] = sum((G*lam)*A)
__global__ void __launch_bounds__(1024) fit_terms_kernel(const double* __restrict__ H,
                                                         const double* __restrict__ lam,
                                                         const double* __restrict__ G,
                                                         const double* __restrict__ A, int64_t rows,
                                                         int64_t R, double* __restrict__ out) {
  __shared__ double sh[1024];
  double s0 = 0.0;
  for (int64_t b = threadIdx.x; b < R; b += 1024) {
    double v = 0.0;
    for (int64_t a = 0; a < R; ++a) v = fma(lam[a], H[a * R + b], v);
    s0 = fma(v, lam[b], s0);
  }
  double s1 = 0.0;
  if (G && A)
    for (int64_t idx = threadIdx.x; idx < rows * R; idx += 1024) {
      const int64_t j = idx % R;
      s1 = fma(G[idx] * lam[j], A[idx], s1);
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
  gram_kernel<<<unsigned(nt * (nt + 1) / 2), 256, 0, as_stream(stream)>>>(A, rows, rank, lda, gram);
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

// work layout: [gamma copy R*R][potrf lwork][info int]
static int solve_layout(int64_t rows, int64_t rank, int lwork, size_t* total, size_t* off_lwork, size_t* off_info) {
  (void)rows;
  const size_t g = align_up(size_t(rank) * size_t(rank) * sizeof(double));
  const size_t w = align_up(size_t(std::max(lwork, 1)) * sizeof(double));
  *off_lwork = g;
  *off_info = g + w;
  *total = g + w + 256;
  return CPK_OK;
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
  size_t a, b;
  return solve_layout(rows, rank, lwork, bytes, &a, &b);
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
  for (int rung = 0; rung <= 5; ++rung) {
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

extern "C" int cpk_solve_normal_spec_f64(const double* gamma, double* G, int64_t rows, int64_t rank, void* work,
                                         size_t work_bytes, int* info_out, void* stream) {
  if (!gamma || !G || !work || !info_out || rank < 1 || rows < 0) return fail(CPK_ERR_PARAM, "bad solve arguments");
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
  copy_regularize_kernel<<<std::max(cblocks, 1u), 256, 0, st>>>(gamma, rank, 0.0, L);
  rc = check_launch("copy_regularize");
  if (rc) return rc;
  // rung 0 only, and no readback: the caller checks *info_out later
  if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, int(rank), L, int(rank), w, lwork, info_out) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(CPK_ERR_LIB, "potrf failed");
  if (rows > 0 && cusolverDnDpotrs(h, CUBLAS_FILL_MODE_UPPER, int(rank), int(rows), L, int(rank), G, int(rank),
                                   info_d) != CUSOLVER_STATUS_SUCCESS)
    return fail(CPK_ERR_LIB, "potrs failed");
  return check_launch("potrs");
}
