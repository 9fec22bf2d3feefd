// Status plumbing, the synthetic-tensor generator and the FP64 peak probe.
#include "common.cuh"

#include <string.h>
#include <algorithm>

namespace cpk {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// splitmix64 finalizer (Steele, Lea, Flood 2014); CPU twin: oracle/gen.py.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_uniform_kernel(double* __restrict__ x, int64_t n, uint64_t key, int64_t offset) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const uint64_t c = uint64_t(offset + i);
    const uint64_t z = mix64(key + (c + 1) * 0x9E3779B97F4A7C15ull);
    x[i] = double(z >> 11) * 0x1.0p-53;
  }
}

// Slab of a larger splitmix tensor: local element (first mode fastest, local
// dims) gets the value of its GLOBAL flat index, the shard mode offset by lo.
struct SlabDims {
  int64_t local[CPK_MAX_MODES];
  int64_t gstride[CPK_MAX_MODES];
  int d, mode;
  int64_t lo;
};

__global__ void fill_slab_kernel(double* __restrict__ x, int64_t n, const __grid_constant__ SlabDims sd,
                                 uint64_t key) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    int64_t rem = i, g = 0;
    for (int m = 0; m < sd.d; ++m) {
      const int64_t q = rem / sd.local[m];
      int64_t sub = rem - q * sd.local[m];
      rem = q;
      if (m == sd.mode) sub += sd.lo;
      g += sub * sd.gstride[m];
    }
    const uint64_t z = mix64(key + (uint64_t(g) + 1) * 0x9E3779B97F4A7C15ull);
    x[i] = double(z >> 11) * 0x1.0p-53;
  }
}

static uint64_t seed_key(uint64_t seed) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Independent DFMA chains, register resident: the FP64 pipe ceiling.
constexpr int PROBE_CHAINS = 16;
__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, int iters, double b, double c) {
  double a[PROBE_CHAINS];
#pragma unroll
  for (int i = 0; i < PROBE_CHAINS; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < PROBE_CHAINS; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < PROBE_CHAINS; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// The same FP64 pipe through mma.sync m8n8k4 (256 FMA per warp instruction):
// 8 independent accumulator pairs per warp.
__global__ void __launch_bounds__(256) dmma_probe_kernel(double* out, int iters, double b, double c) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 1e-3 * (threadIdx.x + i);
  const double a = b * threadIdx.x, bb = c * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(bb));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace cpk

using namespace cpk;

extern "C" const char* cpk_last_error(void) { return g_err; }

extern "C" const char* cpk_version(void) { return "cpk_b200 0.1.0 sm_100a"; }

extern "C" int cpk_fill_uniform_f64(double* x, int64_t n, uint64_t seed, int64_t offset, void* stream) {
  if (n < 0 || offset < 0) return fail(CPK_ERR_PARAM, "negative length or offset");
  if (n == 0) return CPK_OK;
  if (!x) return fail(CPK_ERR_PARAM, "x is NULL");
  const uint64_t key = seed_key(seed);  // decorrelates neighbouring seeds
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 32);
  fill_uniform_kernel<<<unsigned(blocks), 256, 0, as_stream(stream)>>>(x, n, key, offset);
  return check_launch("fill_uniform");
}

extern "C" int cpk_fill_uniform_slab_f64(double* x, int d, const int64_t* global_dims, int mode, int64_t lo,
                                         int64_t hi, uint64_t seed, void* stream) {
  if (d < 1 || d > CPK_MAX_MODES || !global_dims) return fail(CPK_ERR_PARAM, "bad order or dims");
  if (mode < 0 || mode >= d) return fail(CPK_ERR_INDEX, "mode %d out of range", mode);
  if (lo < 0 || hi < lo || hi > global_dims[mode]) return fail(CPK_ERR_PARAM, "bad slab [%lld, %lld)", (long long)lo,
                                                               (long long)hi);
  SlabDims sd{};
  sd.d = d;
  sd.mode = mode;
  sd.lo = lo;
  int64_t g = 1, n = 1;
  for (int m = 0; m < d; ++m) {
    sd.local[m] = m == mode ? hi - lo : global_dims[m];
    sd.gstride[m] = g;
    g *= global_dims[m];
    n *= sd.local[m];
  }
  if (n == 0) return CPK_OK;
  if (!x) return fail(CPK_ERR_PARAM, "x is NULL");
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 32);
  fill_slab_kernel<<<unsigned(blocks), 256, 0, as_stream(stream)>>>(x, n, sd, seed_key(seed));
  return check_launch("fill_slab");
}

extern "C" int cpk_fp64_peak_probe(double* flops_per_s, double* seconds) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return fail(CPK_ERR_CUDA, "device query failed");
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return fail(CPK_ERR_CUDA, "cudaMalloc");
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // best of 5 for each form of the FP64 pipe: DFMA chains and DMMA
  auto time_best = [&](auto launch) {
    launch(256);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      launch(-1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    return double(best) * 1e-3;
  };
  const int it_f = 1 << 14, it_m = 1 << 12;
  const double t_f = time_best([&](int n) { dfma_probe_kernel<<<blocks, threads>>>(out, n < 0 ? it_f : n, 1.0000001, 1e-9); });
  const double t_m = time_best([&](int n) { dmma_probe_kernel<<<blocks, threads>>>(out, n < 0 ? it_m : n, 1e-3, 2e-3); });
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  int rc = check_launch("fp64 probe");
  if (rc) return rc;
  const double f_f = 2.0 * PROBE_CHAINS * double(it_f) * double(blocks) * threads / t_f;
  const double f_m = 2.0 * 256 * 8 * double(it_m) * double(blocks) * (threads / 32) / t_m;
  if (seconds) *seconds = f_m > f_f ? t_m : t_f;
  if (flops_per_s) *flops_per_s = std::max(f_f, f_m);
  return CPK_OK;
}

// ---------------------------------------------------------------- ELEM
// The paper's baseline matrix-free GPU MTTKRP, MTTKRP-ELEM (
// CPU restatement _kernels.py:60-93): every element adds lam_j y prod_m
// A_m(i_m, j) into its output row with one FP64 atomic per column -- N R
// logical atomics (mttkrp.py:309).  One warp per element, lanes over the
// rank columns (coalesced factor rows and atomics).  A comparison variant
// only: results are not bit-reproducible (atomic order).
namespace cpk {
struct ElemParams {
  const double* y;
  const double* fac[CPK_MAX_MODES];
  int64_t ld[CPK_MAX_MODES];
  int64_t dims[CPK_MAX_MODES];
  int d, k;
  int64_t n, R, ldg;
  const double* lam;
  double* G;
};

__global__ void __launch_bounds__(256) mttkrp_elem_atomic_f64(const __grid_constant__ ElemParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < p.n; i += warps) {
    int64_t sub[CPK_MAX_MODES], rem = i;
    for (int m = 0; m < p.d; ++m) {
      sub[m] = rem % p.dims[m];
      rem /= p.dims[m];
    }
    const double yv = p.y[i];
    double* grow = p.G + sub[p.k] * p.ldg;
    for (int64_t j = lane; j < p.R; j += 32) {
      double v = p.lam ? p.lam[j] * yv : yv;
      for (int m = 0; m < p.d; ++m)
        if (m != p.k) v *= p.fac[m][sub[m] * p.ld[m] + j];
      atomicAdd(grow + j, v);
    }
  }
}
}  // namespace cpk

extern "C" int cpk_mttkrp_elem_f64(const double* y, int d, const int64_t* dims, int mode,
                                   const double* const* factors, const int64_t* ld, const double* lam, int64_t rank,
                                   double* G, int64_t ldg, void* stream) {
  if (!y || !dims || !factors || !G) return fail(CPK_ERR_PARAM, "NULL argument");
  if (d < 1 || d > CPK_MAX_MODES) return fail(CPK_ERR_PARAM, "order d=%d unsupported", d);
  if (mode < 0 || mode >= d) return fail(CPK_ERR_INDEX, "mode %d out of range [0, %d]", mode, d - 1);
  if (rank < 1 || ldg < rank) return fail(CPK_ERR_PARAM, "bad rank / ldg");
  ElemParams p{};
  p.y = y;
  p.d = d;
  p.k = mode;
  p.n = 1;
  for (int m = 0; m < d; ++m) {
    if (dims[m] < 1) return fail(CPK_ERR_SHAPE, "extent %d is %lld", m, (long long)dims[m]);
    p.dims[m] = dims[m];
    p.n *= dims[m];
    p.fac[m] = m == mode ? nullptr : factors[m];
    p.ld[m] = ld ? ld[m] : rank;
    if (m != mode && !factors[m]) return fail(CPK_ERR_PARAM, "factor %d is NULL", m);
  }
  p.R = rank;
  p.ldg = ldg;
  p.lam = lam;
  p.G = G;
  cudaStream_t st = as_stream(stream);
  if (cudaMemset2DAsync(G, size_t(ldg) * sizeof(double), 0, size_t(rank) * sizeof(double), size_t(dims[mode]), st) !=
      cudaSuccess)
    return fail(CPK_ERR_CUDA, "memset G");
  const int64_t blocks = std::min<int64_t>((p.n + 7) / 8, 148 * 16);
  mttkrp_elem_atomic_f64<<<unsigned(std::max<int64_t>(blocks, 1)), 256, 0, st>>>(p);
  return check_launch("mttkrp_elem_atomic");
}
