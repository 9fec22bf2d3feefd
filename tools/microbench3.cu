// Does operand reuse limit the FP64 outer product on B200?  Register-only
// 8x8 outer products (no loads) in different DFMA orders, 8 warps/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench3 tools/microbench3.cu
#include <cstdio>
#include <cuda_runtime.h>

// ORDER 0: row-major (a reused along c), 1: snake (a shared, then b at the
// row boundary), 2: column-major (b reused), 3: "scattered" (no operand shared
// between consecutive DFMAs)
template <int ORDER>
__global__ void __launch_bounds__(256, 1) outer(double* out, int iters) {
  double acc[8][8];
  double a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = 1e-3 * (threadIdx.x + i);
    b[i] = 1.0 + 1e-9 * (i + blockIdx.x);
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 64; ++s) {
      int r, c;
      if (ORDER == 0) {
        r = s / 8;
        c = s % 8;
      } else if (ORDER == 1) {
        r = s / 8;
        c = (r & 1) ? 7 - s % 8 : s % 8;
      } else if (ORDER == 2) {
        c = s / 8;
        r = s % 8;
      } else {
        r = s % 8;
        c = (s / 8 + s % 8) % 8;  // consecutive s differ in both r and c
      }
      asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc[r][c]) : "d"(a[r]), "d"(b[c]));
    }
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[r][c];
  if (s == 1.2345) out[0] = s;
}

template <int ORDER>
void run(int sms) {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000;
  outer<ORDER><<<sms, 256>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  outer<ORDER><<<sms, 256>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("outer product order %d: %.2f TFLOP/s\n", ORDER, 128.0 * iters * sms * 256.0 / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>(sms);
  run<1>(sms);
  run<2>(sms);
  run<3>(sms);
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
