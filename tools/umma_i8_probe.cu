// Validation + rate probe for tcgen05.mma kind::i8 (the building block an
// Ozaki-style FP64 emulation of the MTTKRP would run on):
// D[128 x N] (s32, TMEM) += A[128 x K] * B[N x K]^T with signed int8 K-major
// SWIZZLE_128B smem operands (128 int8 per row = one swizzle row), UMMA_K =
// 32.  Checks exact int32 accumulation against the CPU over `reps` repeats,
// then the rate of back-to-back MMAs from shared memory on 148 CTAs for
// N = 32, 64, 128, 256 (whether small rank tiles are shared-memory bound).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_probe tools/umma_i8_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, K = 128;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
// K-major SW128: row r at r * 128 bytes, 16-byte chunk c at chunk c ^ (r & 7)
__host__ __device__ inline int swz_off(int r, int k) { return r * 128 + ((((k >> 4) ^ (r & 7))) << 4) + (k & 15); }
__device__ __forceinline__ uint64_t sdesc(const void* p) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
         (uint64_t(2) << 61);
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4)     // D = S32
         | (1u << 7)   // A = signed int8
         | (1u << 10)  // B = signed int8
         | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

template <int N>
__global__ void __launch_bounds__(128, 1) probe(const int8_t* A, const int8_t* B, int32_t* D, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  int8_t* As = reinterpret_cast<int8_t*>(smem);          // 16 KB
  int8_t* Bs = reinterpret_cast<int8_t*>(smem + 16384);  // N x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + N * 128);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += 128) As[swz_off(i / K, i % K)] = A[i];
  for (int i = tid; i < N * K; i += 128) Bs[swz_off(i / K, i % K)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  constexpr int COLS = N < 32 ? 32 : N;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "r"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  constexpr uint32_t id = idesc_i8(M, N);
  if (tid == 0) {
    const uint64_t da0 = sdesc(As), db0 = sdesc(Bs);
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < K / 32; ++k) {  // UMMA_K = 32 int8 = 32 bytes: +2 in 16-byte units
        const uint32_t acc = (r > 0 || k > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da0 + uint64_t(2 * k)), "l"(db0 + uint64_t(2 * k)), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P;\nW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n}\n" ::"r"(smem_u32(bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    const int row = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) D[size_t(blockIdx.x) * M * N + row * N + c0 + j] = int32_t(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(COLS));
}

template <int N>
static void run(const std::vector<int8_t>& A, const std::vector<int8_t>& B) {
  int8_t *dA, *dB;
  int32_t* dD;
  const int blocks = 148;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, size_t(N) * K);
  cudaMalloc(&dD, size_t(blocks) * M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), size_t(N) * K, cudaMemcpyHostToDevice);
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int check_reps = 3;
  probe<N><<<1, 128, smem>>>(dA, dB, dD, check_reps);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int32_t> D(size_t(M) * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  long long bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      long long ref = 0;
      for (int k = 0; k < K; ++k) ref += int(A[m * K + k]) * int(B[n * K + k]);
      if (ref * check_reps != D[size_t(m) * N + n]) ++bad;
    }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20000;
  probe<N><<<blocks, 128, smem>>>(dA, dB, dD, 10);
  cudaEventRecord(e0);
  probe<N><<<blocks, 128, smem>>>(dA, dB, dD, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * M * N * K * double(reps) * blocks;
  printf("{\"N\": %d, \"launch\": \"%s\", \"exact\": %s, \"mismatches\": %lld, \"tops\": %.1f, "
         "\"smem_bytes_per_mma\": %d, \"macs_per_mma\": %d}\n",
         N, cudaGetErrorString(e), bad == 0 ? "true" : "false", bad, ops / (ms * 1e-3) / 1e12,
         (M + N) * 32, M * N * 32);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
}


// Ozaki-shaped loop: NDIAG int32 accumulators of N columns in TMEM (one per
// slice diagonal), PER_GROUP MMAs per o-group spread over them, then 8 drain
// warps read every accumulator (tcgen05.ld), fold them into an FP64 running
// sum (scale 2^-7d, times a per-column o-row product) while the MMA warp
// waits -- no double buffering (7 x 64 columns leave no room).  The rate
// counted is the int8 work of the MMAs; /28 it is the FP64-equivalent rate
// of a 7-slice emulation.
template <int N, int NDIAG, int PER_GROUP>
__global__ void __launch_bounds__(320, 1) ozaki_sim(const int8_t* A, const int8_t* B, double* out, int groups) {
  extern __shared__ __align__(1024) uint8_t smem[];
  int8_t* As = reinterpret_cast<int8_t*>(smem);
  int8_t* Bs = reinterpret_cast<int8_t*>(smem + 16384);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 16384 + N * 128);  // [0] acc full, [1] drained
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) As[swz_off(i / K, i % K)] = A[i];
  for (int i = tid; i < N * K; i += blockDim.x) Bs[swz_off(i / K, i % K)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bars[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;\n" ::"r"(smem_u32(&bars[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  constexpr uint32_t id = idesc_i8(M, N);
  auto wait = [](uint64_t* b, unsigned ph) {
    asm volatile(
        "{\n\t.reg .pred P;\nW%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(ph)
        : "memory");
  };
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t da0 = sdesc(As), db0 = sdesc(Bs);
      for (int g = 0; g < groups; ++g) {
        if (g > 0) wait(&bars[1], (g - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        for (int it = 0; it < PER_GROUP / NDIAG; ++it) {  // no divisions in the issue loop
          const int k = it & 3;
          const uint32_t acc = it > 0 ? 1u : 0u;
#pragma unroll
          for (int dgl = 0; dgl < NDIAG; ++dgl)
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + uint32_t(dgl * N)),
                "l"(da0 + uint64_t(2 * k)), "l"(db0 + uint64_t(2 * k)), "r"(id), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&bars[0]))
                     : "memory");
      }
    }
  } else if (warp >= 2) {
    // 8 drain warps: lane quarter (warp & 3), column half ((warp - 2) >> 2)
    constexpr int HALF = N / 2;
    const int quarter = warp & 3, c_base = ((warp - 2) >> 2) * HALF;
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    double sum[HALF];
#pragma unroll
    for (int j = 0; j < HALF; ++j) sum[j] = 0.0;
    for (int g = 0; g < groups; ++g) {
      wait(&bars[0], g & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const double po = 1.0 + 1e-3 * g;  // stands in for the o-rows' product
#pragma unroll
      for (int c0 = 0; c0 < HALF; c0 += 16) {
        double t[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) t[j] = 0.0;
#pragma unroll
        for (int dd = NDIAG - 1; dd >= 0; --dd) {  // smallest terms first
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(lane_base + uint32_t(dd * N + c_base + c0)));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          const double sc = ldexp(1.0, -7 * dd);
#pragma unroll
          for (int j = 0; j < 16; ++j) t[j] = fma(double(int32_t(v[j])), sc, t[j]);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) sum[c0 + j] = fma(po, t[j], sum[c0 + j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bars[1]))
                                  : "memory");
    }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < HALF; ++j) acc += sum[j];
    out[size_t(blockIdx.x) * 256 + (warp - 2) * 32 + lane] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

template <int N, int NDIAG, int PER_GROUP>
static void run_ozaki(const std::vector<int8_t>& A, const std::vector<int8_t>& B) {
  int8_t *dA, *dB;
  double* dO;
  const int blocks = 148, groups = 200;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, size_t(N) * K);
  cudaMalloc(&dO, size_t(blocks) * 256 * 8);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), size_t(N) * K, cudaMemcpyHostToDevice);
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(ozaki_sim<N, NDIAG, PER_GROUP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ozaki_sim<N, NDIAG, PER_GROUP><<<blocks, 320, smem>>>(dA, dB, dO, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ozaki_sim<N, NDIAG, PER_GROUP><<<blocks, 320, smem>>>(dA, dB, dO, groups);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * M * N * 32 * double(PER_GROUP) * groups * blocks;
  printf("{\"ozaki_sim\": true, \"N\": %d, \"diagonals\": %d, \"mmas_per_group\": %d, \"launch\": \"%s\", "
         "\"int8_tops\": %.1f, \"fp64_equiv_tflops_28_products\": %.1f, \"fp64_equiv_tflops_21_products\": %.1f}\n",
         N, NDIAG, PER_GROUP, cudaGetErrorString(cudaGetLastError()), ops / (ms * 1e-3) / 1e12,
         ops / (ms * 1e-3) / 1e12 / 28, ops / (ms * 1e-3) / 1e12 / 21);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
}

int main() {
  std::vector<int8_t> A(size_t(M) * K), B(size_t(256) * K);
  srand(1);
  for (auto& x : A) x = int8_t((rand() & 255) - 128);
  for (auto& x : B) x = int8_t((rand() & 255) - 128);
  run<32>(A, B);
  run<64>(A, B);
  run<128>(A, B);
  run<256>(A, B);
  // o-group of I_f = 1024: 28 slice products x 32 K-steps = 896 MMAs (7 slices), 21 x 32 = 672 (6 slices)
  run_ozaki<64, 7, 896>(A, B);
  run_ozaki<64, 6, 672>(A, B);
  run_ozaki<64, 7, 1792>(A, B);  // I_f = 2048
  run_ozaki<64, 7, 3584>(A, B);  // I_f = 4096
  return 0;
}
