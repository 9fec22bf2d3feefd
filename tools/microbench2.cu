// Inner-loop ceilings for the 8x8-per-thread FP64 outer product on B200.
//   reg:  a[8], b[8] fixed in registers, 64 DFMA per step (RF/reuse ceiling)
//   lds:  fragments re-read from shared memory each k (the MTTKRP consumer loop)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench2 tools/microbench2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) outer_reg(double* out, int iters) {
  double acc[8][8];
  double a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = 1e-3 * (threadIdx.x + i);
    b[i] = 1.0 + 1e-9 * i;
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] += 1e-12;  // keep a live and changing (8 DADD / 64 DFMA)
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[r][c];
  if (s == 1.2345) out[0] = s;
}

// The consumer loop of mttkrp_ws: A [k][128] (M-major), B [k][128], 16x16 threads of 8x8.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) outer_lds(double* out, int iters) {
  extern __shared__ __align__(16) double sm[];
  double* A = sm;               // 32 x 128
  double* B = sm + 32 * 128;    // 32 x 128
  for (int i = threadIdx.x; i < 2 * 32 * 128; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ty = (warp / 2) * 4 + lane / 8, tx = (warp % 2) * 8 + lane % 8;
  double acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int kk = 0; kk < 32; kk += 2) {
      double a[8][2];
#pragma unroll
      for (int kq = 0; kq < 2; ++kq)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 v = *reinterpret_cast<const double2*>(A + (kk + kq) * 128 + 2 * ty + 32 * i);
          a[2 * i][kq] = v.x;
          a[2 * i + 1][kq] = v.y;
        }
#pragma unroll
      for (int kq = 0; kq < 2; ++kq) {
        double b[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 v = *reinterpret_cast<const double2*>(B + (kk + kq) * 128 + 2 * tx + 32 * i);
          b[2 * i] = v.x;
          b[2 * i + 1] = v.y;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = fma(a[r][kq], b[c], acc[r][c]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[r][c];
  if (s == 1.2345) out[0] = s;
}

template <typename K>
double rate(K kernel, int blocks, int threads, size_t smem, int iters, double flops_per_thread_iter) {
  double* out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  kernel<<<blocks, threads, smem>>>(out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kernel<<<blocks, threads, smem>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  return flops_per_thread_iter * iters * double(blocks) * threads / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("outer_reg 4 warps/SM : %.2f TFLOP/s\n", rate(outer_reg<4>, sms, 128, 0, 20000, 128.0));
  printf("outer_reg 8 warps/SM : %.2f TFLOP/s\n", rate(outer_reg<8>, sms, 256, 0, 20000, 128.0));
  printf("outer_lds 8 warps/SM : %.2f TFLOP/s\n", rate(outer_lds<8>, sms, 256, 65536, 1000, 32 * 128.0));
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
