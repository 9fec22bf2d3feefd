// Validation + rate probe for the tcgen05 kind::tf32 building blocks used by
// the float32 MTTKRP: K-major SWIZZLE_128B smem operands written by threads,
// UMMA smem descriptors, the instruction descriptor, TMEM alloc / ld, and
// commit-to-mbarrier.  D[128 x N] = A[128 x K] * B[N x K]^T, K = 32 per stage.
// Modes: 0 = A K-major (works; the fp32 kernel's layout); 1/2 = A in the
// MN-major SWIZZLE_128B canonical layout with the transpose-A bit set (and
// LBO/SBO swapped): both return all zeros on this B200/driver, which is why
// the fp32 kernel transposes mode-0 tiles itself.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_tf32_probe tools/umma_tf32_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 128, K = 32;  // one 128-byte swizzle row of fp32 per operand row

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

// K-major SW128 layout: row r (M or N index) at r * 128 bytes; 16-byte chunk
// c of the row stored at chunk c ^ (r & 7) (1024-byte aligned atoms)
__device__ __forceinline__ int swz_off(int r, int k) {  // float index
  return r * 32 + ((((k >> 2) ^ (r & 7)) << 2) | (k & 3));
}

__device__ __forceinline__ uint64_t sdesc(const void* p) {
  const uint64_t a = smem_u32(p);
  uint64_t d = 0;
  d |= (a >> 4) & 0x3FFF;             // start address
  d |= uint64_t(1) << 16;             // LBO (unused for swizzled K-major), 16 B
  d |= uint64_t(1024 >> 4) << 32;     // SBO: 8-row group stride
  d |= uint64_t(1) << 46;             // version (sm100)
  d |= uint64_t(2) << 61;             // SWIZZLE_128B
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, int a_mn = 0) {
  return (1u << 4)            // D = F32
         | (2u << 7)          // A = TF32
         | (2u << 10)         // B = TF32
         | (uint32_t(a_mn) << 15)  // A K-major (0) / MN-major (1)
         | (0u << 16)         // B K-major
         | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
// MN-major SW128: 32-m groups of 32 k-rows x 128 B (4096 B), 8-row atoms
__device__ __forceinline__ int mn_off(int m, int k) {
  return (m / 32) * 1024 + k * 32 + ((((m % 32) >> 2) ^ (k & 7)) << 2) + (m & 3);
}
__device__ __forceinline__ uint64_t sdesc_mn(const void* p, int swap) {
  const uint64_t a = smem_u32(p);
  const uint64_t lbo = swap ? 1024 : 4096, sbo = swap ? 4096 : 1024;
  return ((a >> 4) & 0x3FFF) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

__global__ void __launch_bounds__(128, 1) probe(const float* A, const float* B, float* D, int reps, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* As = reinterpret_cast<float*>(smem);            // 16 KB
  float* Bs = reinterpret_cast<float*>(smem + 16384);    // 16 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += 128) As[mode ? mn_off(i / K, i % K) : swz_off(i / K, i % K)] = A[i];
  for (int i = tid; i < N * K; i += 128) Bs[swz_off(i / K, i % K)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)), "r"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t id = idesc_tf32(M, N, mode ? 1 : 0);
  if (tid == 0) {
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < K / 8; ++k) {  // UMMA_K = 8 tf32 = 32 bytes: advance the start address
        const uint64_t da = mode ? sdesc_mn(As, mode == 2) + uint64_t(k * 64) : sdesc(As) + uint64_t((k * 32) >> 4);
        const uint64_t db = sdesc(Bs) + uint64_t((k * 32) >> 4);
        const uint32_t acc = (r > 0 || k > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
  }
  // wait for the MMAs
  asm volatile(
      "{\n\t.reg .pred P;\nW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n}\n" ::"r"(smem_u32(bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // warp w reads TMEM lanes 32w..32w+31 (= rows), 16 columns at a time
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
    for (int j = 0; j < 16; ++j) D[size_t(blockIdx.x) * M * N + row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(N));
}

int main() {
  std::vector<float> A(M * K), B(N * K);
  srand(1);
  for (auto& x : A) x = float(rand()) / RAND_MAX;
  for (auto& x : B) x = float(rand()) / RAND_MAX;
  float *dA, *dB, *dD;
  const int blocks = 148;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, size_t(blocks) * M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 32768 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 3; ++mode) {
  probe<<<1, 128, smem>>>(dA, dB, dD, 1, mode);
  cudaError_t e = cudaDeviceSynchronize();
  printf("mode %d (0 K-major, 1 MN-major, 2 MN swapped) launch: %s\n", mode, cudaGetErrorString(e));
  std::vector<float> D(M * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxrel = 0, maxabs = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += double(A[m * K + k]) * double(B[n * K + k]);
      maxabs = std::max(maxabs, std::fabs(ref - D[m * N + n]));
      maxrel = std::max(maxrel, std::fabs(ref - D[m * N + n]) / std::fabs(ref));
    }
  printf("D[0][0]=%f  max rel err vs fp64 = %.3e (tf32 expected ~1e-3), max abs %.3e\n", D[0], maxrel, maxabs);
  }
  // rate: reps MMAs of 128x128x32 per CTA, 148 CTAs
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20000;
  probe<<<blocks, 128, smem>>>(dA, dB, dD, 10, 0);
  cudaEventRecord(e0);
  probe<<<blocks, 128, smem>>>(dA, dB, dD, reps, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("tf32 UMMA M128 N128: %.1f TFLOP/s (%s)\n", 2.0 * M * N * K * reps * double(blocks) / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
