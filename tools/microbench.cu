// Microbenchmarks that size the MTTKRP inner loop on B200 (run under gpurun):
//   1. DFMA throughput (register-resident chains)      -> FP64 CUDA-core peak
//   2. DMMA m8n8k4 throughput (mma.sync f64)            -> FP64 tensor peak
//   3. LDS.128 cost with the MTTKRP broadcast patterns  -> shared-memory bound
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1e-3 * threadIdx.x, b = 2e-3 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

// Shared-load patterns: address(lane) in 8-byte units; W = 128 or 64 bits.
// ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum
// gives wavefronts per instruction; clock64 gives SM-cycles per warp-LDS.
template <int PAT, int W>
__global__ void lds_pattern(double* out, long long* cyc, int iters) {
  __shared__ __align__(16) double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int a;  // in doubles
  switch (PAT) {
    case 0: a = 0; break;                                // full broadcast
    case 1: a = (lane >> 3) * 2; break;                  // quarter-uniform, 4 distinct (current A)
    case 2: a = (lane & 7) * 2; break;                   // 8 distinct, same in every quarter (current B)
    case 3: a = ((lane >> 2) & 3) * 2; break;            // 4 distinct per half-warp (4x4 ty)
    case 4: a = (lane & 3) * 2; break;                   // 4 distinct, lane%4 (4x4 tx)
    case 5: a = lane * 2; break;                         // all distinct, contiguous
    case 6: a = (lane >> 2) * 2; break;                  // 8 distinct, groups of 4 lanes
    case 7: a = (lane & 15) * 2; break;                  // 16 distinct, halves identical
    default: a = 0;
  }
  if (W == 64) a = a / 2;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int off = (a + j * 128 + (it & 3) * 1024) & 4095;
      if (W == 128) {
        const double2 v = *reinterpret_cast<const double2*>(&sm[off & ~1]);
        acc += v.x + v.y;
      } else {
        acc += sm[off];
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 1.2345) out[0] = acc;
}

template <int PAT, int W>
void run_lds(int sms, double* out, long long* cyc) {
  const int iters = 2048, warps = 8;
  lds_pattern<PAT, W><<<sms, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("LDS.%d pattern %d: %.2f SM-cycles per warp-LDS (8 warps/SM)\n", W, PAT, double(h) / (iters * 8.0 * warps));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, sizeof(long long) * 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  {
    const int iters = 1 << 14, blocks = sms * 8, th = 256;
    dfma_kernel<<<blocks, th>>>(out, 64);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, th>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA: %.2f TFLOP/s\n", 2.0 * 16 * iters * double(blocks) * th / (ms * 1e-3) / 1e12);
  }
  {
    const int iters = 1 << 13, blocks = sms * 8, th = 256;
    dmma_kernel<<<blocks, th>>>(out, 64);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, th>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    // one m8n8k4 = 256 FMA per warp
    printf("DMMA m8n8k4: %.2f TFLOP/s\n", 2.0 * 256 * 8 * double(iters) * blocks * (th / 32) / (ms * 1e-3) / 1e12);
  }
  run_lds<0, 128>(sms, out, cyc); run_lds<1, 128>(sms, out, cyc); run_lds<2, 128>(sms, out, cyc);
  run_lds<3, 128>(sms, out, cyc); run_lds<4, 128>(sms, out, cyc); run_lds<5, 128>(sms, out, cyc);
  run_lds<6, 128>(sms, out, cyc); run_lds<7, 128>(sms, out, cyc);
  run_lds<0, 64>(sms, out, cyc); run_lds<1, 64>(sms, out, cyc); run_lds<2, 64>(sms, out, cyc);
  run_lds<3, 64>(sms, out, cyc); run_lds<4, 64>(sms, out, cyc); run_lds<5, 64>(sms, out, cyc);
  run_lds<6, 64>(sms, out, cyc); run_lds<7, 64>(sms, out, cyc);
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
